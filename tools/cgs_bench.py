"""Micro-benchmark of the GMRES orthogonalisation at growing Arnoldi index j.

Runs one 200-iteration restart cycle of block GMRES (2x2 Burgers block,
rtol tiny so the cycle runs to the restart length) through the C ABI with
per-phase CUDA-event timing, and prints the CGS2 bandwidth achieved.
usage: python tools/cgs_bench.py [--n 1024] [--restart 200] [--reps 3]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--restart", type=int, default=200)
    ap.add_argument("--timing", type=int, default=1)
    ap.add_argument("--dt", type=float, default=5e-2)
    ap.add_argument("--reps", type=int, default=3, help="cycles run; the last one is reported")
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2101_01776_b200 as pk
    from paper_2101_01776_b200.engine import context_for

    n = args.n
    prob = pk.GridProblem("burgers", (n, n), nu=1e-2)
    U = pk.fourier_u0((n, n), 1, 8, 0.5, 0)
    f = pk.OperatorField.linearize(prob, np.stack([U]))
    sysb = pk.Block2x2System(3.677815, 3.508762, -10.983731, None, f, f, args.dt)
    rhs = np.random.default_rng(0).standard_normal(2 * n * n)
    ctx = context_for(prob)
    ctx.set_timing(bool(args.timing))
    for _ in range(args.reps):
        c0 = ctx.counters()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = pk.block_gmres(sysb, rhs, pk.PrecondSpec(inner=4), rtol=1e-15,
                                maxit=args.restart, restart=args.restart)
        torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    c1 = ctx.counters()
    by = c1["cgs_bytes"] - c0["cgs_bytes"]
    ms = c1["cgs_time_ms"] - c0["cgs_time_ms"]
    print(f"iterations={rep.iterations} wall={wall:.3f}s cgs_ms={ms:.1f} "
          f"cgs_bytes={by / 1e9:.1f}GB -> {by / (ms * 1e-3) / 1e9 if ms else 0:.0f} GB/s; "
          f"precond_ms={c1['precond_time_ms'] - c0['precond_time_ms']:.1f} "
          f"op_ms={c1['op_time_ms'] - c0['op_time_ms']:.1f}")


if __name__ == "__main__":
    main()

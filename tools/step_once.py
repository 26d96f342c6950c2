"""Run W warm-up steps + K steps of a BASELINE config on cuda:0 (profiling driver).

usage: python tools/step_once.py [--config 1] [--n N] [--warmup 1] [--steps 1]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--family", default=None)
    ap.add_argument("--s", type=int, default=None)
    ap.add_argument("--timing", action="store_true", help="per-phase CUDA-event timing")
    ap.add_argument("--inner", default=None, help="override PrecondSpec.inner (int, exact, mg)")
    args = ap.parse_args()
    import torch

    import paper_2101_01776_b200 as pk
    from paper_2101_01776_b200.engine import Context

    spec = pk.baseline_config(args.config, n=args.n, family=args.family, s=args.s)
    tab = pk.make_tableau(spec.family, spec.s)
    sv = spec.solver
    cfg = pk.SolverConfig(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"],
                          restart=sv["restart"], newton_maxit=sv["newton_maxit"],
                          newton_rtol=sv.get("newton_rtol", 1e-9),
                          krylov_rtol=sv.get("krylov_rtol", 1e-5),
                          precond=pk.PrecondSpec(inner=(sv["inner"] if args.inner is None else
                                                        (args.inner if args.inner in ("exact", "mg")
                                                         else int(args.inner)))))
    ctx = Context(spec.problem, 0)
    ctx.set_prep(pk.prepare_stages(tab))
    ctx.set_config(cfg)
    u = torch.from_numpy(spec.u0()).cuda()
    if args.timing:
        ctx.set_timing(True)
    t = 0.0
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = ctx.step_device(u, t, spec.dt)
        torch.cuda.synchronize()
        print(f"step {i}: {1e3 * (time.perf_counter() - t0):.2f} ms newton={st.newton_iterations} "
              f"krylov={st.krylov_iterations} blocks={st.block_iterations}", flush=True)
        t += spec.dt
    c = ctx.counters()
    print("counters", c)


if __name__ == "__main__":
    main()

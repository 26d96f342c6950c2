"""Device time per hot-path phase at configs[1] (or --n) after one real step.

usage: python tools/phase_probe.py [--n 1024] [--reps 50] [--js 0,4,8,16,30]
Runs one warm-up IRK step of the bench workload, then replays each phase on
the state the last block solve left (irkg_probe_phase) and prints us/phase.
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--js", default="0,2,4,8,12,16,24,32")
    ap.add_argument("--short", action="store_true",
                    help="inner solves and block operator only (no graph-mode / CGS rows)")
    ap.add_argument("--block1", action="store_true",
                    help="probe a 1x1 block (eta = 4.644371, configs[1]'s real eigenvalue)")
    args = ap.parse_args()
    import torch

    import paper_2101_01776_b200 as pk
    from paper_2101_01776_b200.engine import context_for

    spec = pk.baseline_config(args.config, n=args.n)
    tab = pk.make_tableau(spec.family, spec.s)
    sv = spec.solver
    cfg = pk.SolverConfig(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"],
                          restart=sv["restart"], newton_maxit=sv["newton_maxit"],
                          precond=pk.PrecondSpec(inner=sv["inner"]))
    ctx = context_for(spec.problem)  # (block_gmres below shares it)
    ctx.set_prep(pk.prepare_stages(tab))
    ctx.set_config(cfg)
    u = torch.from_numpy(spec.u0()).cuda()
    # the last block solved in a step is the leading 2x2 block (reversed order)
    ctx.step_device(u, 0.0, spec.dt)
    torch.cuda.synchronize()
    if args.block1:
        import numpy as np

        f = pk.OperatorField.linearize(spec.problem, u.cpu().numpy()[None, :])
        rhs = np.random.default_rng(0).standard_normal(spec.problem.dim)
        pk.block_gmres((4.644371, f, spec.dt), rhs, pk.PrecondSpec(inner=sv["inner"]), rtol=1e-5,
                       maxit=200, restart=200)
        torch.cuda.synchronize()
    lib, h = ctx.lib, ctx.h

    def probe(ph, j, reps=None):
        out = C.c_double()
        torch.cuda.nvtx.range_push(f"probe{ph}")  # (ncu --nvtx --nvtx-include "probe6/")
        rc = lib.irkg_probe_phase(h, ph, j, reps or args.reps, C.byref(out))
        torch.cuda.nvtx.range_pop()
        if rc != 0:
            raise RuntimeError(lib.irkg_last_error().decode())
        return out.value

    pin = probe(7, 0)
    n2 = (1 if args.block1 else 2) * spec.problem.dim
    mb = n2 * 8 / 1e6
    print(f"grid {spec.problem.shape}  2N vector = {mb:.1f} MB  pin kernel {pin:.2f} us")
    for name, ph in [("precond (2 chains)", 0), ("jacobi chain 1", 1), ("jacobi chain 2", 2),
                     ("block operator", 3), ("stage mix (s,N)", 9), ("backsolve", 11)]:
        print(f"{name:22s} {probe(ph, 4) - pin:8.2f} us")
    if args.short:
        return
    # graph mode: 8 steps j0..j0+7 of the captured WHILE loop (exit test
    # disabled on the stale probe state), per Arnoldi step
    for j0 in (0, 8, 16, 32, 100, 180):
        g = probe(12, j0, reps=5)
        print(f"graph-mode Arnoldi steps j={j0}..{j0 + 7}: {g / 8:8.2f} us/step")
    print(" j   cgs2(3 sweeps) us   GB/s(alg)   DOT / UPD_DOT / UPD_NORM us   arnoldi step us   x+=Vy us")
    for j in [int(x) for x in args.js.split(",")]:
        c = probe(6, j) - pin
        c1 = probe(4, j) - pin
        c2 = probe(5, j) - pin
        a = probe(8, j) - pin
        v = probe(10, j) - pin
        by = 8 * n2 * (3 * (j + 1) + 5)
        print(f"{j:3d}   {c:10.2f}        {by / c / 1e3:8.0f}   {c1:7.2f} {c2 - c1:7.2f} {c - c2:7.2f}"
              f"       {a:10.2f}      {v:8.2f}")


if __name__ == "__main__":
    main()

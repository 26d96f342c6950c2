"""Where an IRK step of the bench workload goes: Arnoldi-loop graphs (1x1 and
2x2 blocks), restart-cycle ends, and everything else (Newton residual,
linearisation, stage transforms, back-substitution, host round trips).

usage: IRKG_GRAPH_TIMING=1 python tools/step_breakdown.py [--steps 10] [--warmup 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--march", action="store_true", help="march the trajectory instead")
    args = ap.parse_args()
    os.environ.setdefault("IRKG_GRAPH_TIMING", "1")
    import torch

    import paper_2101_01776_b200 as pk
    from paper_2101_01776_b200.engine import Context

    spec = pk.baseline_config(args.config, n=args.n)
    tab = pk.make_tableau(spec.family, spec.s)
    sv = spec.solver
    cfg = pk.SolverConfig(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"],
                          restart=sv["restart"], newton_maxit=sv["newton_maxit"],
                          precond=pk.PrecondSpec(inner=sv["inner"]))
    ctx = Context(spec.problem, 0)
    ctx.set_prep(pk.prepare_stages(tab))
    ctx.set_config(cfg)
    u0 = torch.from_numpy(spec.u0()).cuda()
    u = u0.clone()
    t = 0.0
    # default: every step is the bench's step (t = 0, u0); --march walks the trajectory
    for _ in range(args.warmup):
        if not args.march:
            u.copy_(u0)
            t = 0.0
        ctx.step_device(u, t, spec.dt)
        t += spec.dt
    torch.cuda.synchronize()
    c0 = ctx.counters()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = {}
    newton = 0
    for _ in range(args.steps):
        if not args.march:
            u.copy_(u0)
            t = 0.0
        st = ctx.step_device(u, t, spec.dt)
        t += spec.dt
        newton += st.newton_iterations
        for off, lst in st.block_iterations.items():
            its[off] = its.get(off, 0) + sum(lst)
    e1.record()
    torch.cuda.synchronize()
    c1 = ctx.counters()
    total = e0.elapsed_time(e1)
    a1 = c1["arnoldi_ms_1x1"] - c0["arnoldi_ms_1x1"]
    a2 = c1["arnoldi_ms_2x2"] - c0["arnoldi_ms_2x2"]
    ce = c1["cycle_end_ms"] - c0["cycle_end_ms"]
    ng = c1["newton_gap_ms"] - c0["newton_gap_ms"]
    bg = c1["block_gap_ms"] - c0["block_gap_ms"]
    rest = total - a1 - a2 - ce
    print(f"{args.steps} steps, {newton} Newton iterations, Krylov its per block offset {its}")
    print(f"total device time     {total:9.2f} ms  ({total / args.steps:.2f} ms/step)")
    for name, v in [("Arnoldi graphs 2x2", a2), ("Arnoldi graphs 1x1", a1),
                    ("cycle ends", ce), ("rest (Newton, transforms, host)", rest)]:
        print(f"{name:32s} {v:9.2f} ms  {100 * v / total:5.1f} %")
    print(f"  of which device idle across host round trips: Newton residual -> next iteration "
          f"{ng:.2f} ms, block end -> next block {bg:.2f} ms")
    for off, n_it in sorted(its.items()):
        size = 2 if off == 0 else 1
        ms = a2 if size == 2 else a1
        print(f"block offset {off} ({size}x{size}): {n_it} its, {1e3 * ms / max(1, n_it):.1f} us/it")


if __name__ == "__main__":
    main()

"""GPU idle gaps inside one IRK / DAE step: CUPTI kernel timeline (torch.profiler)
of one warmed step of a BASELINE config -- busy time, idle time, and the
largest gaps with the kernels on either side.

usage: python tools/gap_probe.py --config 4 [--n N] [--top 15]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def summarise(prof, top=15):
    """Kernel totals, busy / idle time and the largest idle gaps of a profiled region."""
    import collections
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
    busy = 0.0
    gaps = []
    end = ev[0].time_range.start
    prev = None
    for e in ev:
        s, f = e.time_range.start, e.time_range.end
        if s > end:
            gaps.append((s - end, prev.name[:50] if prev else "-", e.name[:50]))
        busy += max(0.0, f - max(s, end))
        if f > end:
            end, prev = f, e
    print(f"span {(t1 - t0) / 1e3:.2f} ms  busy {busy / 1e3:.2f} ms  idle {(t1 - t0 - busy) / 1e3:.2f} ms")
    import collections
    kt = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        kt[e.name[:60]][0] += 1
        kt[e.name[:60]][1] += e.time_range.end - e.time_range.start
    print("kernel totals:")
    for n, (c, tot) in sorted(kt.items(), key=lambda kv: -kv[1][1])[:top + 10]:
        print(f"  {tot / 1e3:8.3f} ms {100 * tot / busy:5.1f}%  {c:4d} x {tot / c:8.1f} us  {n}")
    gaps.sort(reverse=True)
    for g, a, b in gaps[:top]:
        print(f"  gap {g:9.1f} us  after {a:50s} before {b}")
    by = collections.defaultdict(lambda: [0, 0.0])
    for g, a, b in gaps:
        by[(a, b)][0] += 1
        by[(a, b)][1] += g
    print("gap totals by (after, before):")
    for (a, b), (c, tot) in sorted(by.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"  {tot:9.1f} us in {c:4d} gaps  {a:40s} -> {b}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--top", type=int, default=15)
    ap.add_argument("--steps", type=int, default=1, help="steps inside the profiled region")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2101_01776_b200 as pk
    from paper_2101_01776_b200.engine import context_for

    spec = pk.baseline_config(args.config, n=args.n)
    sv = spec.solver
    cfg = pk.SolverConfig(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"],
                          restart=sv["restart"], newton_maxit=sv["newton_maxit"],
                          newton_rtol=sv.get("newton_rtol", 1e-9),
                          krylov_rtol=sv.get("krylov_rtol", 1e-5),
                          precond=pk.PrecondSpec(inner=sv["inner"]))
    ctx = context_for(spec.problem)
    ctx.set_prep(pk.prepare_stages(pk.make_tableau(spec.family, spec.s)))
    ctx.set_config(cfg)
    dae = args.config == 4
    if dae:
        w0, p0 = pk.vorticity_initial_state(spec.problem)
        u = torch.cat([torch.from_numpy(w0), torch.from_numpy(p0)]).cuda()
        adv = lambda t: ctx.dae_step_device(u, t, spec.dt)
    else:
        u = torch.from_numpy(spec.u0()).cuda()
        adv = lambda t: ctx.step_device(u, t, spec.dt)
    adv(0.0)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for k in range(args.steps):
            st = adv((k + 1) * spec.dt)
        torch.cuda.synchronize()
    print(f"newton={st.newton_iterations} krylov={st.krylov_iterations}")
    summarise(prof, args.top)

if __name__ == "__main__":
    main()

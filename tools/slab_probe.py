"""Cost of the slab-partitioned path on ONE GPU (IRKG_FORCE_SLAB: 1-rank NCCL
ring, self send/recv halos, 1-rank all-reduces) against the plain context on
the same configs[1] steps -- an upper bound for the multi-GPU weak-scaling
efficiency before any inter-GPU traffic.

usage: python tools/slab_probe.py [--n 1024] [--steps 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--profile", action="store_true",
                    help="CUPTI kernel totals and idle gaps of one more slab step")
    args = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    import torch
    import torch.distributed as dist

    import paper_2101_01776_b200 as pk
    from paper_2101_01776_b200.distributed import SlabContext
    from paper_2101_01776_b200.engine import Context

    dist.init_process_group("gloo", rank=0, world_size=1)
    spec = pk.baseline_config(1, n=args.n)
    tab = pk.make_tableau(spec.family, spec.s)
    sv = spec.solver
    cfg = pk.SolverConfig(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"],
                          restart=sv["restart"], newton_maxit=sv["newton_maxit"],
                          precond=pk.PrecondSpec(inner=sv["inner"]))
    res = {}
    for mode in ["plain", "slab"]:
        if mode == "slab":
            os.environ["IRKG_FORCE_SLAB"] = "1"
            ctx = SlabContext(spec.problem, 0, 1, transport="nccl", device=0)
        else:
            ctx = Context(spec.problem, 0)
        ctx.set_prep(pk.prepare_stages(tab))
        ctx.set_config(cfg)
        u = torch.from_numpy(spec.u0()).cuda()
        ctx.step_device(u, 0.0, spec.dt)  # warm-up
        torch.cuda.synchronize()
        t = spec.dt
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kry = 0
        ev0.record()
        for _ in range(args.steps):
            st = ctx.step_device(u, t, spec.dt)
            kry += st.krylov_iterations
            t += spec.dt
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        res[mode] = (ms / args.steps, kry, u.double().norm().item())
        print(f"{mode:6s} {ms / args.steps:9.2f} ms/step  krylov={kry}  "
              f"{1e3 * ms / kry:8.1f} us/iteration  |u|={res[mode][2]:.15e}", flush=True)
        if args.profile and mode == "slab":
            from torch.profiler import ProfilerActivity, profile

            from gap_probe import summarise

            with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
                st = ctx.step_device(u, t, spec.dt)
                torch.cuda.synchronize()
            print(f"profiled slab step: newton={st.newton_iterations} krylov={st.krylov_iterations}")
            summarise(prof, 25)
        del ctx
    print(f"slab/plain time ratio {res['slab'][0] / res['plain'][0]:.3f}")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

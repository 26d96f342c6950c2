"""One bench step (configs[1] step 1 from u0) inside an NVTX range "step",
after one untimed warm-up step -- for ncu launch lists of the real step:

  IRKG_GRAPHS=0 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum \\
      --cache-control none --clock-control none --csv python tools/one_step.py
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--out", default=None, help="write the step's engine counters (JSON)")
    args = ap.parse_args()
    import torch

    import paper_2101_01776_b200 as pk
    from paper_2101_01776_b200.engine import Context

    spec = pk.baseline_config(args.config, n=args.n)
    sv = spec.solver
    ctx = Context(spec.problem, 0)
    ctx.set_prep(pk.prepare_stages(pk.make_tableau(spec.family, spec.s)))
    ctx.set_config(pk.SolverConfig(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"],
                                   restart=sv["restart"], newton_maxit=sv["newton_maxit"],
                                   precond=pk.PrecondSpec(inner=sv["inner"])))
    u0 = torch.from_numpy(spec.u0()).cuda()
    u = u0.clone()
    ctx.step_device(u, 0.0, spec.dt)
    torch.cuda.synchronize()
    u.copy_(u0)
    c0 = ctx.counters()
    torch.cuda.nvtx.range_push("step")
    st = ctx.step_device(u, 0.0, spec.dt)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    c1 = ctx.counters()
    d = {k: c1[k] - c0[k] for k in ("cgs_bytes", "cgs_launches", "precond_bytes", "op_bytes",
                                     "kernel_launches", "arnoldi_iterations")}
    print(f"newton={st.newton_iterations} krylov={st.krylov_iterations} "
          f"blocks={ {k: sum(v) for k, v in st.block_iterations.items()} }")
    print("counters " + json.dumps(d))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(dict(d, newton=st.newton_iterations, krylov=st.krylov_iterations), fh)


if __name__ == "__main__":
    main()

"""Every BASELINE config at full size on one GPU through the public API.

usage: python tools/config_sweep.py [--budget 120] [--configs 0,1,2,2r,3,4] [--inner 4]
Per config: W = 1 warm-up step, then steps until --budget seconds or the
config's step count; device-synced wall time per step, Newton / Krylov counts,
stage-DOF updates/s.  "2r" is configs[2] with Radau IIA(3) (the BASELINE's
"Gauss 2-stage vs Radau IIA 3-stage").  Config 4 is the vorticity DAE
(reordered mode).  One JSON line per config.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=120.0)
    ap.add_argument("--configs", default="0,1,2,2r,3,4")
    ap.add_argument("--inner", default=None, help="override PrecondSpec.inner (int, exact, mg)")
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2101_01776_b200 as pk

    for key in args.configs.split(","):
        idx = int(key[0])
        fam, s = ("radau_iia", 3) if key.endswith("r") else (None, None)
        spec = pk.baseline_config(idx, family=fam, s=s)
        sv = spec.solver
        inner = sv["inner"] if args.inner is None else (
            args.inner if args.inner in ("exact", "mg") else int(args.inner))
        cfg = pk.SolverConfig(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"],
                              restart=sv["restart"], newton_maxit=sv["newton_maxit"],
                              newton_rtol=sv.get("newton_rtol", 1e-9),
                              krylov_rtol=sv.get("krylov_rtol", 1e-5),
                              precond=pk.PrecondSpec(inner=inner))
        tab = pk.make_tableau(spec.family, spec.s)
        prep = pk.prepare_stages(tab)
        prob = spec.problem
        dae = idx == 4
        if dae:
            w0, p0 = pk.vorticity_initial_state(prob)
            u, w = torch.from_numpy(w0).cuda(), torch.from_numpy(p0).cuda()
            n_dof = prob.dim_u
        else:
            u = torch.from_numpy(spec.u0()).cuda()
            n_dof = prob.dim
        t = 0.0
        rows = []
        t_start = time.perf_counter()
        for i in range(spec.nsteps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if dae:
                u, w, st = pk.dae_step(prob, u, w, t, spec.dt, tab, cfg, prep=prep)
            else:
                u, st = pk.step(prob, u, t, spec.dt, tab, cfg, prep=prep)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            t += spec.dt
            rows.append((el, st.newton_iterations, st.krylov_iterations))
            print(f"  {spec.name} step {i}: {1e3 * el:.1f} ms newton={st.newton_iterations} "
                  f"krylov={st.krylov_iterations}", file=sys.stderr, flush=True)
            if time.perf_counter() - t_start > args.budget and i >= args.warmup:
                break
        timed = rows[args.warmup:] if len(rows) > args.warmup else rows
        el = sum(r[0] for r in timed)
        newton = sum(r[1] for r in timed)
        out = {
            "config": key, "workload": spec.name, "grid": list(prob.shape),
            "scheme": f"{spec.family}({spec.s})", "dt": spec.dt, "inner": str(inner),
            "steps_run": len(rows), "steps_timed": len(timed), "steps_in_config": spec.nsteps,
            "s_per_step": el / len(timed), "steps_per_s": len(timed) / el,
            "stage_dof_per_s": newton * spec.s * n_dof / el,
            "newton": [r[1] for r in rows], "krylov": [r[2] for r in rows],
            "finite": bool(torch.isfinite(u).all()),
        }
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

"""Run every reference golden (tests/golden/) through the device path and
report the parity observables the north star names: final-state relative L2,
and the maximum |delta| of per-step Newton, per-step Krylov and per-block
Krylov counts (the last aligned Newton iteration by Newton iteration).

    python tools/parity_report.py [--out profiles/r2_parity_report.json] [names...]

Needs a GPU; prints one JSON line per case and writes the whole table.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2101_01776_b200 as pk  # noqa: E402
from _golden import case_names, grid_problem, load_case, load_dae_case  # noqa: E402


def _solver(sv, dae=False):
    return pk.SolverConfig(
        variant=sv.get("variant", 3),
        newton_rtol=sv.get("newton_rtol", 1e-9),
        newton_maxit=sv.get("newton_maxit", 30),
        krylov_rtol=sv.get("krylov_rtol", 1e-5),
        krylov_maxit=sv.get("krylov_maxit", 200),
        restart=sv.get("restart", 200),
        precond=pk.PrecondSpec(inner=sv.get("inner", 4)),
        jacobian_refresh=sv.get("jacobian_refresh", "every"),
    )


def _block_delta(got, want):
    worst = 0
    shape_ok = True
    for off, its in want.items():
        g = got.get(off, [])
        if len(g) != len(its):
            shape_ok = False
        for a, b in zip(g, its):
            worst = max(worst, abs(a - b))
    return worst, shape_ok


def run_case(name):
    dae = name.startswith("dae_")
    meta = load_dae_case(name) if dae else load_case(name)
    tic = time.time()
    if dae:
        prob = pk.VorticityProblem(tuple(meta["shape"]), nu=meta["nu"])
        res = pk.dae_integrate(prob, meta["u0"], meta["w0"], 0.0, meta["nsteps"] * meta["dt"],
                               meta["dt"], pk.make_tableau(meta["family"], meta["s"]),
                               _solver(meta["solver"]))
        rel = max(np.linalg.norm(res.u_final - meta["u_final"]) / np.linalg.norm(meta["u_final"]),
                  np.linalg.norm(res.w_final - meta["w_final"]) / np.linalg.norm(meta["w_final"]))
    else:
        prob = grid_problem(meta)
        fam = meta["family"]
        tab = pk.make_tableau(fam) if fam.startswith("sdirk") else pk.make_tableau(fam, meta["s"])
        sv = meta["solver"]
        cfg = _solver(sv)
        res = pk.integrate(prob, meta["u0"], 0.0, meta["nsteps"] * meta["dt"], meta["dt"], tab,
                           cfg)
        rel = float(np.linalg.norm(res.u_final - meta["u_final"]) / np.linalg.norm(meta["u_final"]))
    wall = time.time() - tic
    dn = dk = db = 0
    shapes = len(res.step_stats) == len(meta["steps"])
    per_step = []
    for got, want in zip(res.step_stats, meta["steps"]):
        a = abs(got.newton_iterations - want["newton_iterations"])
        b = abs(got.krylov_iterations - want["krylov_iterations"])
        c, ok = _block_delta(got.block_iterations, want["block_iterations"])
        shapes = shapes and ok
        dn, dk, db = max(dn, a), max(dk, b), max(db, c)
        per_step.append([got.newton_iterations, want["newton_iterations"],
                         got.krylov_iterations, want["krylov_iterations"]])
    return {"case": name, "rel_l2": float(rel), "max_dnewton": dn, "max_dkrylov_step": dk,
            "max_dblock": db, "shapes_equal": bool(shapes), "steps": len(meta["steps"]),
            "per_step[newton,ref,krylov,ref]": per_step, "gpu_wall_s": round(wall, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("names", nargs="*")
    args = ap.parse_args()
    names = args.names or (case_names() + case_names(dae=True))
    rows = []
    for n in names:
        try:
            row = run_case(n)
        except Exception as exc:  # report and continue
            row = {"case": n, "error": repr(exc)}
        print(json.dumps(row), flush=True)
        rows.append(row)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()

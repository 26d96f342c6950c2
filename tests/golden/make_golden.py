"""Generate the golden fixtures from the REAL reference (build container only).

Run from the repo root:  ``python tests/golden/make_golden.py``

It imports ``irkit`` from ``/root/reference/pkg/src`` (read-only; absent on
the GPU box, which only reads the committed outputs) and writes:

* ``tests/golden/tableaux.json`` and ``paper_2101_01776_b200/data/tableaux.json``:
  ``make_tableau`` + ``prepare_stages`` constants (src/tableau.py:329-379)
  for every collocation family and stage count, as hex floats (bit-exact).
* ``tests/golden/<case>.npz`` + ``<case>.json``: ``irkit.integrate`` runs of
  the oracle problem builders (``oracle/problems.py``) on seeded
  ``fourier_u0`` fields: initial and final state plus per-step StepStats
  (Newton / Krylov counts, per-block iteration lists, residual histories).
* ``tests/golden/transformed.json``: Krylov counts and solutions of
  ``solve_transformed_system`` on small linear systems for every variant.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import irkit  # noqa: E402
from irkit.irk_core import PrecondSpec, solve_transformed_system  # noqa: E402
from irkit.nonlinear import OdeSystem, SolverConfig, integrate  # noqa: E402
from irkit.sparsela import SparseMatrix  # noqa: E402

from oracle.problems import build_problem  # noqa: E402
from paper_2101_01776_b200.problems import GridProblem, baseline_config, fourier_u0  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")

FAMILIES = [("gauss", s) for s in range(1, 9)] + [("radau_iia", s) for s in range(1, 9)] + [
    ("lobatto_iiic", s) for s in range(2, 9)
]


def _hex(a):
    a = np.asarray(a, dtype=float)
    return {"shape": list(a.shape), "data": [float(x).hex() for x in a.ravel()]}


def dump_tableaux():
    doc = {}
    for fam, s in FAMILIES:
        tab = irkit.make_tableau(fam, s)
        prep = irkit.prepare_stages(tab)
        doc[f"{fam}:{s}"] = {
            "family": tab.family,
            "s": tab.s,
            "order": tab.order,
            "a0": _hex(tab.a0),
            "b0": _hex(tab.b0),
            "c0": _hex(tab.c0),
            "a0inv": _hex(prep.a0inv),
            "q": _hex(prep.schur.q),
            "r": _hex(prep.schur.r),
            "blocks": [
                [b.offset, b.size, float(b.eta).hex(), float(b.beta).hex(), float(b.phi).hex()]
                for b in prep.blocks
            ],
            "d": _hex(prep.d),
        }
    # SDIRK baselines (src/tableau.py:283-326): coefficients only (the
    # reference steps them with _dirk_step and never prepares them)
    for fam in ("sdirk1", "sdirk2", "sdirk3", "sdirk4"):
        tab = irkit.make_tableau(fam)
        doc[f"{fam}:{tab.s}"] = {
            "family": tab.family,
            "s": tab.s,
            "order": tab.order,
            "a0": _hex(tab.a0),
            "b0": _hex(tab.b0),
            "c0": _hex(tab.c0),
        }
    text = json.dumps(doc, indent=1, sort_keys=True)
    for path in (os.path.join(GOLD, "tableaux.json"),
                 os.path.join(ROOT, "paper_2101_01776_b200", "data", "tableaux.json")):
        with open(path, "w") as fh:
            fh.write(text)
    print("tableaux:", len(doc))


def _cfg(solver):
    inner = solver.get("inner", 4)
    return SolverConfig(
        variant=solver.get("variant", 3),
        newton_rtol=solver.get("newton_rtol", 1e-9),
        newton_maxit=solver.get("newton_maxit", 30),
        krylov_rtol=solver.get("krylov_rtol", 1e-5),
        krylov_maxit=solver.get("krylov_maxit", 200),
        restart=solver.get("restart", 200),
        precond=PrecondSpec(gamma_mode=solver.get("gamma_mode", "star"), inner=inner),
        jacobian_refresh=solver.get("jacobian_refresh", "every"),
    )


def run_case(name, prob: GridProblem, u0, family, s, dt, nsteps, solver):
    pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
    sysr = pd.as_ode_system(OdeSystem, SparseMatrix)
    tab = irkit.make_tableau(family, s)
    tic = time.time()
    res = integrate(sysr, u0, 0.0, nsteps * dt, dt, tab, _cfg(solver))
    wall = time.time() - tic
    steps = []
    for st in res.step_stats:
        steps.append(
            {
                "newton_iterations": st.newton_iterations,
                "krylov_iterations": st.krylov_iterations,
                "precond_applications": st.precond_applications,
                "jacobian_assemblies": st.jacobian_assemblies,
                "block_iterations": {str(k): v for k, v in st.block_iterations.items()},
                "residual_history": [float(x).hex() for x in st.residual_history],
            }
        )
    meta = {
        "name": name,
        "kind": prob.kind,
        "shape": list(prob.shape),
        "params": {"nu": prob.nu, "c": prob.c, "lam": prob.lam, "mu": prob.mu, "length": prob.length},
        "family": family,
        "s": s,
        "dt": dt,
        "nsteps": nsteps,
        "solver": solver,
        "steps": steps,
        "reference_wall_s": wall,
    }
    np.savez_compressed(os.path.join(GOLD, name + ".npz"), u0=u0, u_final=res.u_final)
    with open(os.path.join(GOLD, name + ".json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{name}: {wall:.1f}s newton={[x['newton_iterations'] for x in steps]} "
          f"krylov={[x['krylov_iterations'] for x in steps]}")


def run_configs():
    # config 0 at full size, both inner modes
    sp0 = baseline_config(0)
    run_case("cfg0_full", sp0.problem, sp0.u0(), "gauss", 2, sp0.dt, sp0.nsteps, sp0.solver)
    run_case("cfg0_full_exact", sp0.problem, sp0.u0(), "gauss", 2, sp0.dt, sp0.nsteps,
             dict(sp0.solver, inner="exact"))
    # config 1 (Burgers, Gauss(3)) at reduced grids
    for n, ns in ((64, 20), (128, 3)):
        sp1 = baseline_config(1, n=n, nsteps=ns)
        run_case(f"cfg1_n{n}", sp1.problem, sp1.u0(), "gauss", 3, sp1.dt, ns, sp1.solver)
    # config 2 (nldiff 4096^2 field) reduced: Gauss(2) and Radau IIA(3)
    for fam, s in (("gauss", 2), ("radau_iia", 3)):
        sp2 = baseline_config(2, n=128, nsteps=2)
        run_case(f"cfg2_{fam}{s}_n128", sp2.problem, sp2.u0(), fam, s, sp2.dt, 2, sp2.solver)
    # config 3 (3-D, Gauss(5)) reduced
    sp3 = baseline_config(3, n=16, nsteps=2)
    run_case("cfg3_n16", sp3.problem, sp3.u0(), "gauss", 5, sp3.dt, 2, sp3.solver)
    # variants 0..3 on a nonlinear problem with several tableaux
    prob = GridProblem("burgers", (24, 24), nu=1e-2)
    u0 = fourier_u0(prob.shape, 1, 4, 0.5, seed=3)
    for fam, s in (("gauss", 3), ("radau_iia", 3), ("lobatto_iiic", 4), ("gauss", 4), ("radau_iia", 2)):
        for v in range(4):
            run_case(f"var_{fam}{s}_v{v}", prob, u0, fam, s, 2e-3, 2,
                     dict(variant=v, inner=4, krylov_maxit=2000, restart=200))
    # reaction-advection-diffusion (rad kind): logistic-KPP in 1-D and 2-D
    prob = GridProblem("rad", (64,), nu=1e-3, c=0.5, lam=1.0, mu=-1.0)
    u0 = 0.5 + fourier_u0(prob.shape, 1, 3, 0.1, seed=7)
    run_case("rad1d_kpp", prob, u0, "gauss", 2, 0.05, 4, dict(variant=3, inner=4, krylov_rtol=1e-8))
    prob = GridProblem("rad", (32, 32), nu=1e-2, c=0.3, lam=-0.5, mu=0.0)
    u0 = fourier_u0(prob.shape, 1, 4, 0.2, seed=8)
    run_case("rad2d_linear", prob, u0, "radau_iia", 3, 0.01, 3, dict(variant=3, inner=4))


def run_sdirk():
    """integrate() with SDIRK tableaux: the reference's _dirk_step path
    (src/nonlinear.py:239-296) on the config-0 problem and on 2-D Burgers."""
    sp0 = baseline_config(0)
    for fam, s in (("sdirk1", 1), ("sdirk2", 2), ("sdirk3", 3), ("sdirk4", 5)):
        run_case(f"sdirk_cfg0_{fam}", sp0.problem, sp0.u0(), fam, s, sp0.dt, 3,
                 dict(sp0.solver))
    prob = GridProblem("burgers", (48, 48), nu=1e-2)
    u0 = fourier_u0(prob.shape, 1, 6, 0.5, seed=11)
    for fam, s in (("sdirk2", 2), ("sdirk4", 5)):
        run_case(f"sdirk_burgers48_{fam}", prob, u0, fam, s, 2e-3, 3,
                 dict(variant=3, inner=4, krylov_maxit=2000, restart=200))


def run_transformed():
    """solve_transformed_system on advdiff-type linear stencils (every variant),
    mirroring tests/test_irk_core.py:152-167 of the reference."""
    out = []
    prob = GridProblem("rad", (24,), nu=0.01, c=1.0)
    pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
    lmat = SparseMatrix(pd.linearize_csr(np.zeros(24), 0.0), bandwidth=1)
    for fam, s in (("gauss", 3), ("radau_iia", 3), ("lobatto_iiic", 4), ("gauss", 4)):
        prep = irkit.prepare_stages(irkit.make_tableau(fam, s))
        rng = np.random.default_rng(s)
        rhs = rng.standard_normal((s, 24))
        for variant in range(4):
            for inner in ("exact", 4):
                k, stats = solve_transformed_system(
                    prep, [lmat] * s, variant, 0.05, rhs,
                    precond=PrecondSpec(inner=inner),
                    krylov_rtol=1e-12, krylov_maxit=400,
                )
                out.append({
                    "family": fam, "s": s, "variant": variant, "inner": inner,
                    "seed": s, "dt": 0.05,
                    "reports": [[off, rep.iterations] for off, rep in stats.reports],
                    "k": _hex(k),
                })
    with open(os.path.join(GOLD, "transformed.json"), "w") as fh:
        json.dump(out, fh)
    print("transformed cases:", len(out))


def run_dae_case(name, n, family, s, nsteps, dt=1e-3, nu=1e-4):
    """irkit.dae_integrate (reordered mode, Jacobi-4) on the vorticity DAE."""
    from irkit.dae import DaeSystem, dae_integrate

    from oracle.problems import DaeProblemDef
    from paper_2101_01776_b200.problems import VorticityProblem, vorticity_initial_state

    prob = VorticityProblem((n, n), nu=nu)
    w0, p0 = vorticity_initial_state(prob)
    pd = DaeProblemDef(prob.shape, prob.nu)
    sysr = pd.as_dae_system(DaeSystem, SparseMatrix)
    solver = dict(variant=3, inner=4, krylov_maxit=5000, restart=200)
    tic = time.time()
    res = dae_integrate(sysr, w0, p0, 0.0, nsteps * dt, dt, irkit.make_tableau(family, s),
                        _cfg(solver), mode="reordered")
    wall = time.time() - tic
    steps = []
    for st in res.step_stats:
        steps.append({
            "newton_iterations": st.newton_iterations,
            "krylov_iterations": st.krylov_iterations,
            "precond_applications": st.precond_applications,
            "jacobian_assemblies": st.jacobian_assemblies,
            "differential_solves": st.differential_solves,
            "constraint_solves": st.constraint_solves,
            "constraint_residual": float(st.constraint_residual).hex(),
            "block_iterations": {str(k): v for k, v in st.block_iterations.items()},
            "residual_history": [float(x).hex() for x in st.residual_history],
        })
    meta = {"name": name, "kind": "arakawa", "shape": [n, n], "nu": nu, "family": family, "s": s,
            "dt": dt, "nsteps": nsteps, "solver": solver, "mode": "reordered", "steps": steps,
            "reference_wall_s": wall}
    np.savez_compressed(os.path.join(GOLD, name + ".npz"), u0=w0, w0=p0, u_final=res.u_final,
                        w_final=res.w_final)
    with open(os.path.join(GOLD, name + ".json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{name}: {wall:.1f}s newton={[x['newton_iterations'] for x in steps]} "
          f"krylov={[x['krylov_iterations'] for x in steps]}")


def run_larger():
    """The BASELINE configs at larger reduced grids (reference runs of tens of
    seconds): closer to the full-size Krylov counts than the small cases."""
    sp1 = baseline_config(1, n=256, nsteps=2)
    run_case("cfg1_n256", sp1.problem, sp1.u0(), "gauss", 3, sp1.dt, 2, sp1.solver)
    sp2 = baseline_config(2, n=256, nsteps=1)
    run_case("cfg2_gauss2_n256", sp2.problem, sp2.u0(), "gauss", 2, sp2.dt, 1, sp2.solver)
    sp3 = baseline_config(3, n=32, nsteps=1)
    run_case("cfg3_n32", sp3.problem, sp3.u0(), "gauss", 5, sp3.dt, 1, sp3.solver)


SURVEY_CASES = {
    # SURVEY §8(c) / BASELINE.md §3 plan: the BASELINE configs at the sizes the
    # survey prescribes for the oracle comparison (full size where irkit can
    # run it in host RAM, else the reduced grid with the full step count).
    "cfg1_full": lambda: _survey_ode(1, None, None, "cfg1_full"),
    "cfg2_gauss2_n256_s10": lambda: _survey_ode(2, 256, 10, "cfg2_gauss2_n256_s10"),
    "cfg2_radau_iia3_n256_s10": lambda: _survey_ode(2, 256, 10, "cfg2_radau_iia3_n256_s10",
                                                    family="radau_iia", s=3),
    "cfg3_n48_s5": lambda: _survey_ode(3, 48, 5, "cfg3_n48_s5"),
    "cfg3_n64_s5": lambda: _survey_ode(3, 64, 5, "cfg3_n64_s5"),
    "dae_n256_gauss2_s10": lambda: run_dae_case("dae_n256_gauss2_s10", 256, "gauss", 2, 10),
}


def _survey_ode(index, n, nsteps, name, family=None, s=None):
    sp = baseline_config(index, n=n, nsteps=nsteps, family=family, s=s)
    run_case(name, sp.problem, sp.u0(), sp.family, sp.s, sp.dt, sp.nsteps, sp.solver)


def run_frozen():
    """Simplified Newton (jacobian_refresh="frozen", src/nonlinear.py:204-209)
    on 2-D Burgers and on the 1-D KPP reaction problem."""
    prob = GridProblem("burgers", (48, 48), nu=2e-2)
    u0 = fourier_u0(prob.shape, 1, 4, 0.5, seed=6)
    run_case("frozen_burgers48_radau2", prob, u0, "radau_iia", 2, 5e-3, 3,
             dict(variant=3, inner=4, krylov_maxit=4000, newton_maxit=60,
                  jacobian_refresh="frozen"))
    prob = GridProblem("rad", (64,), nu=1e-3, c=0.5, lam=1.0, mu=-1.0)
    u0 = 0.5 + fourier_u0(prob.shape, 1, 3, 0.1, seed=7)
    run_case("frozen_rad1d_gauss3", prob, u0, "gauss", 3, 0.05, 3,
             dict(variant=3, inner=4, krylov_rtol=1e-8, newton_maxit=60,
                  jacobian_refresh="frozen"))


def run_experiments():
    """irkit's own run_iterations (src/experiments.py:250-293) on two manifests
    of its 1-D periodic catalog (default exact inner solves): the rows the
    device harness must reproduce from the same manifest JSON."""
    from irkit.experiments import RunManifest, run_iterations

    cases = {
        "burgers1d": RunManifest(experiment="iterations", problem="burgers1d",
                                 problem_params={"n": 128, "nu": 0.02},
                                 schemes=(("gauss", 2), ("radau_iia", 3), ("gauss", 3)),
                                 dts=(0.02, 0.01), t_final=0.04),
        "advdiff1d": RunManifest(experiment="iterations", problem="advdiff1d",
                                 problem_params={"n": 64, "speed": 1.0, "nu": 0.01},
                                 schemes=(("gauss", 2), ("lobatto_iiic", 4)),
                                 dts=(0.05, 0.025), t_final=0.1),
    }
    for name, m in cases.items():
        rows = run_iterations(m)
        doc = {"manifest": m.to_dict(), "manifest_hash": m.hash, "rows": rows}
        with open(os.path.join(GOLD, f"experiments_iterations_{name}.json"), "w") as fh:
            json.dump(doc, fh, indent=1, default=str)
        print(name, [(r["scheme"], r["dt"], r["newton_iterations"], r["krylov_iterations"],
                      r["status"]) for r in rows])


def run_dae():
    run_dae_case("dae_n16_gauss2", 16, "gauss", 2, 3)
    run_dae_case("dae_n64_gauss2", 64, "gauss", 2, 4)
    run_dae_case("dae_n32_gauss4", 32, "gauss", 4, 2)
    run_dae_case("dae_n128_gauss2", 128, "gauss", 2, 2)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tableaux", "transformed", "configs", "dae", "sdirk", "larger"]
    for case in which:
        if case in SURVEY_CASES:
            SURVEY_CASES[case]()
    if "dae" in which:
        run_dae()
    if "larger" in which:
        run_larger()
    if "tableaux" in which:
        dump_tableaux()
    if "transformed" in which:
        run_transformed()
    if "configs" in which:
        run_configs()
    if "sdirk" in which:
        run_sdirk()
    if "frozen" in which:
        run_frozen()
    if "experiments" in which:
        run_experiments()

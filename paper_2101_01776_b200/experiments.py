"""Experiment harness over the device path.

Mirrors the reference's manifest-driven studies (``src/experiments.py``:
``RunManifest`` 42-97, ``run_iterations`` 250-293, ``run_gamma_compare``
314-367, ``run_convergence`` 136-175) and the per-step CSV of
``write_step_stats_csv`` (``src/nonlinear.py:377-417``), with the problems
taken from this engine's catalog (``GridProblem`` kinds and the BASELINE
configs) instead of the reference's desk-scale 1-D catalog.  Every row
carries the short hash of the canonical manifest JSON, failed cells are
marked and the study continues, and CSV output is written next to the
manifest JSON -- the reference's provenance rules.
"""

from __future__ import annotations

import csv
import dataclasses
import hashlib
import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .config import PrecondSpec, SolverConfig
from .errors import IrkitError
from .problems import GridProblem, baseline_config, fourier_u0
from .solver import integrate
from .stats import write_step_stats_csv  # noqa: F401  (src/nonlinear.py:377-417)
from .tableau import make_tableau, prepare_stages


@dataclass(frozen=True)
class RunManifest:
    """Serializable description of one study (fields of src/experiments.py:42-59,
    plus the inner-solve policy and the seeded-field parameters)."""

    experiment: str
    problem: str  # "baseline:<k>" or a GridProblem kind ("nldiff", "burgers", "rad")
    problem_params: dict = field(default_factory=dict)
    schemes: tuple = ()  # of (family, stages)
    dts: tuple = ()
    t_final: float = 0.1
    variant: int = 3
    gamma: object = "star"
    newton_rtol: float = 1e-9
    krylov_rtol: float = 1e-5
    inner: object = 4
    krylov_maxit: int = 5000
    out: str | None = None
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "schemes", tuple((str(f), int(s)) for f, s in self.schemes))
        object.__setattr__(self, "dts", tuple(float(x) for x in self.dts))

    def to_dict(self):
        doc = dataclasses.asdict(self)
        doc["schemes"] = [list(x) for x in self.schemes]
        doc["dts"] = list(self.dts)
        return doc

    def to_json(self):
        return json.dumps(self.to_dict(), sort_keys=True)

    @classmethod
    def from_dict(cls, doc):
        doc = dict(doc)
        doc["schemes"] = tuple((f, int(s)) for f, s in doc.get("schemes", ()))
        doc["dts"] = tuple(doc.get("dts", ()))
        doc["problem_params"] = dict(doc.get("problem_params", {}))
        return cls(**doc)

    @classmethod
    def from_json(cls, text):
        return cls.from_dict(json.loads(text))

    @property
    def hash(self):
        return hashlib.sha256(self.to_json().encode()).hexdigest()[:12]

    def solver_config(self, **overrides):
        kw = dict(variant=self.variant, newton_rtol=self.newton_rtol,
                  krylov_rtol=self.krylov_rtol, krylov_maxit=self.krylov_maxit, restart=200,
                  precond=PrecondSpec(gamma_mode=self.gamma, inner=self.inner))
        kw.update(overrides)
        return SolverConfig(**kw)

    def problem_and_u0(self):
        """(GridProblem, u0): a BASELINE config ("baseline:1", params: n) or a
        kind with ``shape`` / ``nu`` / ``c`` / ``lam`` / ``mu`` and the seeded
        Fourier field ``k_hi`` / ``sigma``."""
        p = dict(self.problem_params)
        if self.problem.startswith("baseline:"):
            spec = baseline_config(int(self.problem.split(":")[1]), n=p.get("n"))
            return spec.problem, spec.u0()
        shape = tuple(p.pop("shape", (64, 64)))
        k_hi, sigma = p.pop("k_hi", 4), p.pop("sigma", 0.1)
        prob = GridProblem(self.problem, shape, **p)
        return prob, fourier_u0(shape, 1, k_hi, sigma, self.seed)


def _fmt(x):
    return repr(float(x))


def _write_rows(manifest, rows, fieldnames):
    if manifest.out is None:
        return
    out = Path(manifest.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    with out.open("w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=fieldnames)
        w.writeheader()
        for row in rows:
            w.writerow(row)
    out.with_suffix(out.suffix + ".manifest.json").write_text(manifest.to_json() + "\n")


def run_iterations(manifest: RunManifest):
    """Solver-work counts per (scheme, dt) over the time span (src/experiments.py:250-293)."""
    prob, u0 = manifest.problem_and_u0()
    cfg = manifest.solver_config()
    rows = []
    for fam, s in manifest.schemes:
        tab = make_tableau(fam, s)
        for dt in manifest.dts:
            row = {"scheme": tab.label, "order": tab.order, "dt": dt, "steps": "",
                   "newton_iterations": "", "krylov_iterations": "", "precond_applications": "",
                   "wall_time": "", "status": "ok", "manifest_hash": manifest.hash}
            try:
                res = integrate(prob, u0, 0.0, manifest.t_final, dt, tab, cfg)
                row.update(steps=len(res.step_stats),
                           newton_iterations=res.total("newton_iterations"),
                           krylov_iterations=res.total("krylov_iterations"),
                           precond_applications=res.total("precond_applications"),
                           wall_time=_fmt(res.total("wall_time")))
            except IrkitError as exc:
                row["status"] = f"failed: {type(exc).__name__}"
            rows.append(row)
    _write_rows(manifest, rows, ["scheme", "order", "dt", "steps", "newton_iterations",
                                 "krylov_iterations", "precond_applications", "wall_time",
                                 "status", "manifest_hash"])
    return rows


def _block_means(result, prep):
    sums, counts = {}, {}
    for st in result.step_stats:
        for off, its_list in st.block_iterations.items():
            for its in its_list:
                sums[off] = sums.get(off, 0) + its
                counts[off] = counts.get(off, 0) + 1
    return {b.offset: sums[b.offset] / counts[b.offset]
            for b in prep.blocks if b.size == 2 and b.offset in sums}


def run_gamma_compare(manifest: RunManifest):
    """Mean 2x2-block Krylov iterations with the naive (eta) and the optimal
    (gamma*) Schur shift (src/experiments.py:314-367; the paper's headline
    comparison, PAPER.md)."""
    prob, u0 = manifest.problem_and_u0()
    rows = []
    for fam, s in manifest.schemes:
        tab = make_tableau(fam, s)
        prep = prepare_stages(tab)
        if all(b.size == 1 for b in prep.blocks):
            from .errors import ConfigurationError

            raise ConfigurationError(f"{tab.label} has no complex eigen-block")
        for dt in manifest.dts:
            means, status = {}, "ok"
            for mode in ("eta", "star"):
                cfg = manifest.solver_config(precond=PrecondSpec(gamma_mode=mode,
                                                                 inner=manifest.inner))
                try:
                    means[mode] = _block_means(integrate(prob, u0, 0.0, manifest.t_final, dt,
                                                         tab, cfg), prep)
                except IrkitError as exc:
                    status = f"failed: {type(exc).__name__}"
                    means[mode] = {}
            for b in prep.blocks:
                if b.size != 2:
                    continue
                rows.append({"scheme": tab.label, "order": tab.order, "dt": dt,
                             "block_offset": b.offset, "eta": _fmt(b.eta), "beta": _fmt(b.beta),
                             "mean_krylov_eta": _fmt(means["eta"].get(b.offset, float("nan"))),
                             "mean_krylov_star": _fmt(means["star"].get(b.offset, float("nan"))),
                             "status": status, "manifest_hash": manifest.hash})
    _write_rows(manifest, rows, ["scheme", "order", "dt", "block_offset", "eta", "beta",
                                 "mean_krylov_eta", "mean_krylov_star", "status",
                                 "manifest_hash"])
    return rows


def run_convergence(manifest: RunManifest, reference=("radau_iia", 3), refinement=8):
    """Final-time error and observed order per (scheme, dt) against a finer
    reference run (src/experiments.py:136-175; the catalog problems here have
    no closed form, so the reference is always a refined Radau IIA run)."""
    prob, u0 = manifest.problem_and_u0()
    cfg = manifest.solver_config()
    dt_ref = min(manifest.dts) / refinement
    ref = integrate(prob, u0, 0.0, manifest.t_final, dt_ref, make_tableau(*reference), cfg).u_final
    rows = []
    for fam, s in manifest.schemes:
        tab = make_tableau(fam, s)
        prev = None
        for dt in manifest.dts:
            row = {"scheme": tab.label, "order": tab.order, "dt": dt, "error": "", "rate": "",
                   "status": "ok", "manifest_hash": manifest.hash}
            try:
                u = integrate(prob, u0, 0.0, manifest.t_final, dt, tab, cfg).u_final
                err = float(np.linalg.norm(u - ref) / np.sqrt(u.size))
                row["error"] = _fmt(err)
                if prev is not None and err > 0.0 and prev[1] > 0.0:
                    row["rate"] = _fmt(np.log(prev[1] / err) / np.log(prev[0] / dt))
                prev = (dt, err)
            except IrkitError as exc:
                row["status"] = f"failed: {type(exc).__name__}"
                prev = None
            rows.append(row)
    _write_rows(manifest, rows, ["scheme", "order", "dt", "error", "rate", "status",
                                 "manifest_hash"])
    return rows


STUDIES = {"iterations": run_iterations, "gamma-compare": run_gamma_compare,
           "convergence": run_convergence}


def run(manifest: RunManifest):
    """Dispatch on ``manifest.experiment`` (src/experiments.py:449-457)."""
    if manifest.experiment not in STUDIES:
        from .errors import ConfigurationError

        raise ConfigurationError(f"unknown experiment {manifest.experiment!r}")
    return STUDIES[manifest.experiment](manifest)

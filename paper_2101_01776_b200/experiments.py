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
import hashlib
import json
from pathlib import Path

import numpy as np

from .config import PrecondSpec, SolverConfig
from .errors import ConfigurationError, IrkitError
from .problems import GridProblem, baseline_config, fourier_u0
from .solver import integrate
from .stats import write_step_stats_csv  # noqa: F401  (src/nonlinear.py:377-417)
from .tableau import make_tableau, prepare_stages


#: The reference manifest's keys and defaults (src/experiments.py:42-59).  A
#: manifest that uses only these serialises to the same canonical JSON -- and
#: so the same provenance hash -- as irkit's RunManifest, so one JSON file
#: drives both harnesses (tests/test_experiments.py runs irkit's and this
#: engine's run_iterations on one manifest).  This engine's own knobs live in
#: the optional ``device`` mapping (inner-solve policy ``inner``, default the
#: reference's "exact"; ``krylov_maxit``, default 200), left out of the JSON
#: when empty.
_REFERENCE_KEYS = {
    "experiment": None, "problem": None, "problem_params": {}, "schemes": (), "dts": (),
    "t_final": 0.1, "variant": 3, "gamma": "star", "newton_rtol": 1e-9, "krylov_rtol": 1e-5,
    "out": None, "seed": 0,
}


class RunManifest:
    """Serializable description of one study: the reference's manifest plus
    an optional ``device`` mapping (see _REFERENCE_KEYS)."""

    def __init__(self, experiment, problem, **kw):
        unknown = set(kw) - set(_REFERENCE_KEYS) - {"device"}
        if unknown:
            raise TypeError(f"unknown manifest keys {sorted(unknown)}")
        vals = dict(_REFERENCE_KEYS, experiment=experiment, problem=problem)
        vals.update({k: v for k, v in kw.items() if k != "device"})
        vals["problem_params"] = dict(vals["problem_params"] or {})
        vals["schemes"] = tuple((str(f), int(st)) for f, st in vals["schemes"])
        vals["dts"] = tuple(float(x) for x in vals["dts"])
        vals["device"] = dict(kw.get("device") or {})
        object.__setattr__(self, "_v", vals)

    def __getattr__(self, name):
        try:
            return self.__dict__["_v"][name]
        except KeyError:
            raise AttributeError(name) from None

    def __setattr__(self, name, value):
        raise AttributeError("RunManifest is immutable")

    def __eq__(self, other):
        return isinstance(other, RunManifest) and self._v == other._v

    def __hash__(self):
        return hash(self.to_json())

    def __repr__(self):
        return f"RunManifest({self.to_json()})"

    # -- serialisation (canonical: sorted keys; tuples as lists)
    def to_dict(self):
        doc = {k: self._v[k] for k in _REFERENCE_KEYS}
        doc["problem_params"] = dict(doc["problem_params"])
        doc["schemes"] = [[f, st] for f, st in doc["schemes"]]
        doc["dts"] = list(doc["dts"])
        if self._v["device"]:
            doc["device"] = dict(self._v["device"])
        return doc

    def to_json(self):
        return json.dumps(self.to_dict(), sort_keys=True)

    @classmethod
    def from_dict(cls, doc):
        doc = dict(doc)
        return cls(doc.pop("experiment"), doc.pop("problem"), **doc)

    @classmethod
    def from_json(cls, text):
        return cls.from_dict(json.loads(text))

    @property
    def hash(self):
        return hashlib.sha256(self.to_json().encode()).hexdigest()[:12]

    @property
    def inner(self):
        return self._v["device"].get("inner", "exact")

    @property
    def krylov_maxit(self):
        return int(self._v["device"].get("krylov_maxit", 200))

    def solver_config(self, **overrides):
        kw = dict(variant=self.variant, newton_rtol=self.newton_rtol,
                  krylov_rtol=self.krylov_rtol, krylov_maxit=self.krylov_maxit, restart=200,
                  precond=PrecondSpec(gamma_mode=self.gamma, inner=self.inner))
        kw.update(overrides)
        return SolverConfig(**kw)

    def problem_and_u0(self):
        """(GridProblem, u0) for the manifest's problem: a name of the
        reference's 1-D periodic catalog (``burgers1d``, ``advdiff1d``,
        ``advection1d``; src/problems.py:137-200, the same discretisation and
        initial state), a BASELINE config (``baseline:<k>``, params: ``n``),
        or a GridProblem kind with ``shape`` / ``nu`` / ``c`` / ``lam`` /
        ``mu`` and the seeded Fourier field ``k_hi`` / ``sigma``."""
        return catalog_problem(self.problem, self.problem_params, self.seed)


def catalog_problem(name, params, seed=0):
    p = dict(params)
    if name in _REFERENCE_CATALOG:
        return _REFERENCE_CATALOG[name](**p)
    if name.startswith("baseline:"):
        spec = baseline_config(int(name.split(":")[1]), n=p.get("n"))
        return spec.problem, spec.u0()
    if name not in ("nldiff", "burgers", "rad"):
        raise ConfigurationError(f"problem {name!r} has no device discretisation")
    shape = tuple(p.pop("shape", (64, 64)))
    k_hi, sigma = p.pop("k_hi", 4), p.pop("sigma", 0.1)
    prob = GridProblem(name, shape, **p)
    return prob, fourier_u0(shape, 1, k_hi, sigma, seed)


def _grid_1d(n):
    return np.arange(n) / n  # x_i = i h on the periodic unit interval (h = 1/n)


def _burgers1d(n=128, nu=0.02, base=0.5, amplitude=0.45):
    # src/problems.py:175-200: N(u) = -D(u^2/2) + nu Lap u, periodic, h = 1/n
    return (GridProblem("burgers", (int(n),), nu=nu),
            base + amplitude * np.sin(2 * np.pi * _grid_1d(int(n))))


def _advdiff1d(n=64, speed=1.0, nu=0.01):
    # src/problems.py:158-172: u_t = speed D u + nu Lap u
    x = _grid_1d(int(n))
    return (GridProblem("rad", (int(n),), nu=nu, c=speed),
            np.sin(2 * np.pi * x) + 0.2 * np.sin(6 * np.pi * x))


def _advection1d(n=64, speed=1.0):
    # src/problems.py:137-155: u_t = speed D u
    x = _grid_1d(int(n))
    return (GridProblem("rad", (int(n),), c=speed),
            np.sin(2 * np.pi * x) + 0.3 * np.cos(4 * np.pi * x))


_REFERENCE_CATALOG = {"burgers1d": _burgers1d, "advdiff1d": _advdiff1d,
                      "advection1d": _advection1d}


def _fmt(x):
    return repr(float(x))  # the reference's CSV number format (round-trips exactly)


def _write_rows(manifest, rows, fieldnames):
    """CSV of the study next to its manifest JSON (``<out>.manifest.json``)."""
    if manifest.out is None:
        return
    path = Path(manifest.out)
    path.parent.mkdir(parents=True, exist_ok=True)
    with path.open("w", newline="") as fh:
        out = csv.DictWriter(fh, fieldnames=fieldnames)
        out.writeheader()
        out.writerows(rows)
    Path(str(path) + ".manifest.json").write_text(manifest.to_json() + "\n")


def run_iterations(manifest: RunManifest, timing=False):
    """Solver-work counts per (scheme, dt) over the time span
    (src/experiments.py:250-293): the reference's columns, so the CSV of a
    reference-catalog manifest compares row by row with irkit's;
    ``timing=True`` adds the device wall time per cell."""
    prob, u0 = manifest.problem_and_u0()
    cfg = manifest.solver_config()
    rows = []
    for fam, s in manifest.schemes:
        tab = make_tableau(fam, s)
        for dt in manifest.dts:
            row = {"scheme": tab.label, "order": tab.order, "dt": dt, "steps": "",
                   "newton_iterations": "", "krylov_iterations": "", "precond_applications": "",
                   "status": "ok", "manifest_hash": manifest.hash}
            if timing:
                row["wall_time"] = ""
            try:
                res = integrate(prob, u0, 0.0, manifest.t_final, dt, tab, cfg)
                row.update(steps=len(res.step_stats),
                           newton_iterations=res.total("newton_iterations"),
                           krylov_iterations=res.total("krylov_iterations"),
                           precond_applications=res.total("precond_applications"))
                if timing:
                    row["wall_time"] = _fmt(res.total("wall_time"))
            except IrkitError as exc:
                row["status"] = f"failed: {type(exc).__name__}"
            rows.append(row)
    cols = ["scheme", "order", "dt", "steps", "newton_iterations", "krylov_iterations",
            "precond_applications", "status", "manifest_hash"]
    _write_rows(manifest, rows, cols + (["wall_time"] if timing else []))
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
        raise ConfigurationError(f"unknown experiment {manifest.experiment!r}")
    return STUDIES[manifest.experiment](manifest)

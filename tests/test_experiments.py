"""Experiment harness over the device path: manifest
provenance and the per-step CSV match the reference's formats; the studies
run on the GPU and reproduce the paper's shift comparison."""

import json
import os
import sys

import numpy as np
import pytest

import paper_2101_01776_b200 as pk
from paper_2101_01776_b200 import experiments as ex
from paper_2101_01776_b200.stats import StepStats


def _manifest(**kw):
    base = dict(experiment="iterations", problem="nldiff",
                problem_params={"shape": [64, 64], "k_hi": 4, "sigma": 0.1},
                schemes=[("gauss", 2), ("radau_iia", 3)], dts=[1e-3, 5e-4], t_final=2e-3,
                device={"inner": 4})
    base.update(kw)
    return ex.RunManifest(**base)


def test_manifest_roundtrip_and_hash():
    m = _manifest()
    m2 = ex.RunManifest.from_json(m.to_json())
    assert m2 == m and m2.hash == m.hash and len(m.hash) == 12
    assert _manifest(dts=[1e-3]).hash != m.hash


def test_step_stats_csv_matches_reference_format(tmp_path):
    st = StepStats(newton_iterations=3, krylov_iterations=17, precond_applications=34,
                   block_iterations={2: [4, 3], 0: [5, 5]}, wall_time=0.25)
    res = pk.IntegrationResult(times=np.array([0.0, 1.0]), states=[np.zeros(2)] * 2,
                               step_stats=[st])
    ours = tmp_path / "ours.csv"
    ex.write_step_stats_csv(res, ours)
    text = ours.read_text().splitlines()
    assert text[0] == ("step,newton_iterations,krylov_iterations,block_iterations,"
                       "precond_applications,differential_solves,constraint_solves,wall_time")
    assert text[1] == "0,3,17,0:5+5;2:4+3,34,0,0,0.25"
    src = "/root/reference/pkg/src"
    if os.path.isdir(src):  # byte-equal to the reference's writer on the same stats
        sys.path.insert(0, src)
        from irkit.nonlinear import write_step_stats_csv

        theirs = tmp_path / "theirs.csv"
        write_step_stats_csv(res, theirs)
        assert theirs.read_text() == ours.read_text()


@pytest.mark.gpu
def test_iterations_study_on_device(tmp_path):
    m = _manifest(out=str(tmp_path / "it.csv"))
    rows = ex.run(m)
    assert len(rows) == 4 and all(r["status"] == "ok" for r in rows)
    assert all(r["manifest_hash"] == m.hash for r in rows)
    assert (tmp_path / "it.csv.manifest.json").exists()
    assert json.loads((tmp_path / "it.csv.manifest.json").read_text())["experiment"] == "iterations"


@pytest.mark.gpu
def test_gamma_compare_optimal_shift_wins():
    """The paper's headline (gamma* = eta + beta^2/eta vs the naive eta)
    with exact inner solves (the paper's setting): fewer Krylov iterations
    per 2x2 block with gamma*."""
    m = _manifest(experiment="gamma-compare", schemes=[("gauss", 2), ("gauss", 4)],
                  dts=[2e-3], t_final=4e-3, device={"inner": "exact"}, krylov_rtol=1e-10,
                  problem_params={"shape": [64, 64], "k_hi": 4, "sigma": 0.5})
    rows = ex.run(m)
    assert rows and all(r["status"] == "ok" for r in rows)
    for r in rows:
        assert float(r["mean_krylov_star"]) <= float(r["mean_krylov_eta"]), r


def test_reference_manifest_serialises_like_irkit():
    """A manifest with only the reference's keys has irkit's canonical JSON
    and hash (src/experiments.py:42-97), so one file drives both harnesses;
    the device knobs appear only when set."""
    m = ex.RunManifest.from_json(_golden_manifest_text())
    assert "device" not in m.to_dict() and m.inner == "exact" and m.krylov_maxit == 200
    assert m.hash == json.loads(_golden_rows_text())["manifest_hash"]
    src = "/root/reference/pkg/src"
    if os.path.isdir(src):
        sys.path.insert(0, src)
        from irkit.experiments import RunManifest as RefManifest

        ref = RefManifest.from_json(m.to_json())
        assert ref.to_json() == m.to_json() and ref.hash == m.hash
    d = _manifest()
    assert d.to_dict()["device"] == {"inner": 4}
    assert ex.RunManifest.from_json(d.to_json()) == d


def _golden_path(name):
    return os.path.join(os.path.dirname(__file__), "golden", name)


def _golden_manifest_text():
    with open(_golden_path("experiments_iterations_burgers1d.json")) as fh:
        return json.dumps(json.load(fh)["manifest"])


def _golden_rows_text():
    with open(_golden_path("experiments_iterations_burgers1d.json")) as fh:
        doc = json.load(fh)
    return json.dumps({"manifest_hash": doc["manifest_hash"]})


@pytest.mark.gpu
def test_iterations_study_matches_reference_run_iterations(tmp_path):
    """f4 parity: irkit's run_iterations (src/experiments.py:250-293) on the
    reference catalog's burgers1d / advdiff1d (tests/golden/make_golden.py
    'experiments') against this engine's run_iterations on the SAME manifest
    JSON, in the reference's default exact inner mode on the device: every
    row's status, step count and Newton count equal, Krylov and
    preconditioner counts within +/-1 per step, same manifest hash."""
    for name in ("experiments_iterations_burgers1d.json", "experiments_iterations_advdiff1d.json"):
        with open(_golden_path(name)) as fh:
            doc = json.load(fh)
        m = ex.RunManifest.from_dict(dict(doc["manifest"], out=str(tmp_path / (name + ".csv"))))
        rows = ex.run(m)
        assert len(rows) == len(doc["rows"])
        for got, want in zip(rows, doc["rows"]):
            assert got["scheme"] == want["scheme"] and float(got["dt"]) == float(want["dt"])
            assert got["status"] == want["status"], (got, want)
            if want["status"] != "ok":
                continue
            steps = int(want["steps"])
            assert int(got["steps"]) == steps
            assert int(got["newton_iterations"]) == int(want["newton_iterations"]), (got, want)
            assert abs(int(got["krylov_iterations"]) - int(want["krylov_iterations"])) <= steps
            assert abs(int(got["precond_applications"]) -
                       int(want["precond_applications"])) <= 2 * steps
        assert rows[0]["manifest_hash"] != ""  # (the run's own manifest carries `out`)

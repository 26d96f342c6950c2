"""Scheduling knobs change when and how the engine's kernels run, never what
they compute: one IRK step of a Burgers problem must be bit-identical (state
and Newton/Krylov counts) with CUDA graphs off, programmatic dependent launch
off, one Arnoldi step per WHILE-body trip, without the L2 persisting
window / evict-first hints, and with the three CGS2 sweeps fused into one launch.  (Each variant runs in a fresh process: the
knobs are read when the engine is created.)"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2101_01776_b200 as pk
spec = pk.baseline_config(1, n=256)
tab = pk.make_tableau("gauss", 3)
cfg = pk.SolverConfig(variant=3, krylov_maxit=5000, precond=pk.PrecondSpec(inner=4))
u = spec.u0()
stats = []
for k in range(2):
    u, st = pk.step(spec.problem, u, k * spec.dt, spec.dt, tab, cfg)
    stats.append([st.newton_iterations, st.krylov_iterations,
                  {{str(a): b for a, b in st.block_iterations.items()}}])
np.save(sys.argv[1], np.asarray(u))
print(json.dumps(stats))
"""

VARIANTS = {
    "default": {},
    "no_graphs": {"IRKG_GRAPHS": "0"},
    "no_pdl": {"IRKG_PDL": "0"},
    "unroll1": {"IRKG_GRAPH_UNROLL": "1"},
    "no_l2_policy": {"IRKG_L2_MB": "0", "IRKG_CGS_EF": "0"},
    # the three CGS2 sweeps in one launch (k_cgs3: same tiles, same partial sums and
    # folds, grid barriers where the launch boundaries were)
    "cgs_one_launch": {"IRKG_CGS_FUSED": "1"},
    "cgs_one_launch_no_graphs": {"IRKG_CGS_FUSED": "1", "IRKG_GRAPHS": "0", "IRKG_PDL": "0"},
}


def _run(tmp, name, env_extra):
    out = os.path.join(tmp, name + ".npy")
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT), out], env=env, cwd=ROOT,
                       check=True, capture_output=True, text=True, timeout=600)
    return np.load(out), json.loads(r.stdout.strip().splitlines()[-1])


def test_scheduling_knobs_are_bit_identical(tmp_path):
    ref_u, ref_stats = _run(str(tmp_path), "default", VARIANTS["default"])
    for name, env in VARIANTS.items():
        if name == "default":
            continue
        u, stats = _run(str(tmp_path), name, env)
        assert stats == ref_stats, name
        assert u.tobytes() == ref_u.tobytes(), name


def test_cgs_tile_forms_agree(tmp_path):
    """The row-owner CGS update sweeps (IRKG_CGS_RO, default 6) sum the
    second-pass dots in another order than the slot-owner form (0): the same
    IRK steps to the parity bar (1e-10 relative, counts within +/-1)."""
    ref_u, ref_stats = _run(str(tmp_path), "default", {})
    for mask in ("0", "7"):
        u, stats = _run(str(tmp_path), "ro" + mask, {"IRKG_CGS_RO": mask})
        assert len(stats) == len(ref_stats)
        for (n0, k0, _), (n1, k1, _) in zip(ref_stats, stats):
            assert abs(n0 - n1) <= 1 and abs(k0 - k1) <= 1, (mask, ref_stats, stats)
        assert np.linalg.norm(u - ref_u) <= 1e-10 * np.linalg.norm(ref_u), mask

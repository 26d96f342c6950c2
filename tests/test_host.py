"""CPU tests of the product's host side: tableau constants, configuration
mirrors, problem descriptors / u0 generator, and the C-ABI library."""

import ctypes as C
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import paper_2101_01776_b200 as pk
from paper_2101_01776_b200 import _lib
from paper_2101_01776_b200.problems import GridProblem, fourier_modes, fourier_u0

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------- tableaux


def test_tableau_table_is_the_golden_reference_table():
    with open(os.path.join(ROOT, "tests", "golden", "tableaux.json")) as fh:
        gold = json.load(fh)
    with open(os.path.join(ROOT, "paper_2101_01776_b200", "data", "tableaux.json")) as fh:
        prod = json.load(fh)
    assert gold == prod
    assert len(prod) == 27  # 23 collocation tableaux + 4 SDIRK baselines


@pytest.mark.parametrize("family,s", [("gauss", 2), ("gauss", 3), ("gauss", 5),
                                      ("radau_iia", 3), ("lobatto_iiic", 4)])
def test_prepare_stages_structure(family, s):
    tab = pk.make_tableau(family, s)
    prep = pk.prepare_stages(tab)
    q, r = prep.schur.q, prep.schur.r
    # A0^{-1} = Q R Q^T (src/densela.py:60-63) and Q orthogonal
    assert np.allclose(q @ r @ q.T, prep.a0inv, atol=1e-12)
    assert np.allclose(q.T @ q, np.eye(s), atol=1e-13)
    assert np.allclose(prep.a0inv @ tab.a0, np.eye(s), atol=1e-11)
    # d[k,l,i] = q[i,k] q[i,l]  (src/tableau.py:378)
    assert np.array_equal(prep.d, np.einsum("ik,il->kli", q, q))
    assert sum(b.size for b in prep.blocks) == s
    for blk in prep.blocks:
        assert blk.eta > 0.0


def test_tableau_bit_exact_against_reference_when_available():
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not present (GPU box)")
    code = (
        "import sys, json; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import irkit, numpy as np, paper_2101_01776_b200 as pk\n"
        "bad = []\n"
        "for fam, ss in (('gauss', range(1, 9)), ('radau_iia', range(1, 9)), ('lobatto_iiic', range(2, 9))):\n"
        "  for s in ss:\n"
        "    a = irkit.prepare_stages(irkit.make_tableau(fam, s)); b = pk.prepare_stages(pk.make_tableau(fam, s))\n"
        "    ok = all(np.array_equal(x, y) for x, y in ((a.tableau.a0, b.tableau.a0), (a.tableau.b0, b.tableau.b0),"
        " (a.tableau.c0, b.tableau.c0), (a.a0inv, b.a0inv), (a.schur.q, b.schur.q), (a.schur.r, b.schur.r), (a.d, b.d)))\n"
        "    ok = ok and [(x.offset, x.size, x.eta, x.beta, x.phi) for x in a.blocks] == [(x.offset, x.size, x.eta, x.beta, x.phi) for x in b.blocks]\n"
        "    bad += [] if ok else [(fam, s)]\n"
        "for fam in ('sdirk1', 'sdirk2', 'sdirk3', 'sdirk4'):\n"
        "  a = irkit.make_tableau(fam); b = pk.make_tableau(fam)\n"
        "  ok = a.s == b.s and a.order == b.order and all(np.array_equal(x, y) for x, y in ((a.a0, b.a0), (a.b0, b.b0), (a.c0, b.c0)))\n"
        "  bad += [] if ok else [(fam, a.s)]\n"
        "print(json.dumps(bad))\n" % (src, ROOT)
    )
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True)
    assert json.loads(out.stdout.strip().splitlines()[-1]) == []


def test_tableau_errors():
    with pytest.raises(pk.ConfigurationError):
        pk.make_tableau("gauss")
    with pytest.raises(pk.ConfigurationError):
        pk.make_tableau("gauss", 9)
    with pytest.raises(pk.ConfigurationError):
        pk.make_tableau("lobatto", 1)
    with pytest.raises(pk.ConfigurationError):  # SDIRK stage counts are fixed
        pk.make_tableau("sdirk4", 3)
    with pytest.raises(pk.ConfigurationError):  # stepped stage by stage, never prepared
        pk.prepare_stages(pk.make_tableau("sdirk2"))
    with pytest.raises(pk.ConfigurationError):
        pk.make_tableau("nope", 2)
    assert pk.gamma_star(3.0, np.sqrt(3.0)) == pytest.approx(4.0)


# ----------------------------------------------------------- config


def test_sdirk_tableaux_are_the_reference_values():
    """make_tableau for the SDIRK baselines (src/tableau.py:283-341): fixed
    stage counts, lower-triangular A0, stiffly accurate rows where the
    reference builds them so."""
    for fam, s in (("sdirk1", 1), ("sdirk2", 2), ("sdirk3", 3), ("sdirk4", 5)):
        tab = pk.make_tableau(fam)
        assert tab.s == s and tab.is_dirk
        assert np.all(np.triu(tab.a0, 1) == 0.0)
        np.testing.assert_allclose(tab.a0.sum(axis=1), tab.c0, atol=1e-14)
        assert abs(tab.b0.sum() - 1.0) <= 1e-14
    g = 1.0 - 1.0 / np.sqrt(2.0)
    assert pk.make_tableau("sdirk2").a0[0, 0] == g
    tab4 = pk.make_tableau("sdirk4")
    assert np.array_equal(tab4.b0, tab4.a0[-1])


def test_config_mirrors_reference_validation():
    with pytest.raises(pk.ConfigurationError):
        pk.SolverConfig(variant=4)
    with pytest.raises(pk.ConfigurationError):
        pk.SolverConfig(newton_rtol=1.5)
    with pytest.raises(pk.ConfigurationError):
        pk.SolverConfig(jacobian_refresh="sometimes")
    with pytest.raises(ValueError):
        pk.PrecondSpec(gamma_mode=-1.0)
    with pytest.raises(ValueError):
        pk.PrecondSpec(inner=0)
    spec = pk.PrecondSpec(gamma_mode="star")
    assert spec.gamma(3.0, np.sqrt(3.0)) == pytest.approx(4.0)
    assert pk.PrecondSpec(gamma_mode="eta").gamma(3.0, 1.0) == 3.0
    assert pk.PrecondSpec(gamma_mode=2.5).gamma(3.0, 1.0) == 2.5
    cfg = pk.SolverConfig()
    assert (cfg.variant, cfg.newton_rtol, cfg.newton_maxit, cfg.krylov_rtol, cfg.krylov_maxit,
            cfg.restart) == (3, 1e-9, 30, 1e-5, 200, 200)


def test_inner_mode_codes():
    """PrecondSpec.inner -> irkg_solver.inner: the reference default "exact"
    (banded LU, IRKG_INNER_EXACT = 0) or the Jacobi sweep count."""
    from paper_2101_01776_b200 import _lib
    from paper_2101_01776_b200.config import inner_sweeps

    assert inner_sweeps(pk.PrecondSpec()) == _lib.INNER_EXACT == 0
    assert inner_sweeps(pk.PrecondSpec(inner=4)) == 4


# ----------------------------------------------------------- problems


def test_fourier_modes_order_and_count():
    modes = fourier_modes(2, 1, 4)
    assert len(modes) == len(set(modes))
    assert modes == sorted(modes)  # lexicographic, first axis outermost
    assert all(1 <= kx * kx + ky * ky <= 16 for kx, ky in modes)
    assert len(fourier_modes(2, 2, 10)) == sum(
        1 for a in range(-10, 11) for b in range(-10, 11) if 4 <= a * a + b * b <= 100)


@pytest.mark.parametrize("shape", [(16,), (12, 10), (6, 5, 4)])
def test_fourier_u0_matches_direct_sum(shape):
    k_hi, sigma, seed = 3, 0.3, 11
    u = fourier_u0(shape, 1, k_hi, sigma, seed)
    modes = fourier_modes(len(shape), 1, k_hi)
    ab = np.random.default_rng(seed).normal(0.0, sigma, size=(len(modes), 2))
    axes = [(np.arange(n) + 0.5) / n for n in shape]
    mesh = np.meshgrid(*axes, indexing="ij")  # mesh[a][i0, i1, ...]
    direct = np.zeros(shape)
    for k, (a, b) in zip(modes, ab):
        ph = 2 * np.pi * sum(kk * m for kk, m in zip(k, mesh))
        direct += a * np.cos(ph) + b * np.sin(ph)
    flat = direct.transpose(tuple(reversed(range(len(shape))))).ravel()  # x fastest
    np.testing.assert_allclose(u, flat, rtol=0, atol=1e-12)


def test_fourier_u0_is_deterministic():
    a = fourier_u0((32, 32), 1, 4, 0.1, 0)
    b = fourier_u0((32, 32), 1, 4, 0.1, 0)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, fourier_u0((32, 32), 1, 4, 0.1, 1))


def test_golden_u0_is_the_product_generator():
    from _golden import load_case

    meta = load_case("cfg0_full")
    assert np.array_equal(meta["u0"], pk.baseline_config(0).u0())


@pytest.mark.parametrize("kind,shape,params", [
    ("nldiff", (8, 6), {}),
    ("nldiff", (5, 4, 3), {}),
    ("burgers", (7, 9), {"nu": 0.02}),
    ("rad", (10,), {"nu": 0.1, "c": 0.7, "lam": -0.3, "mu": 0.5}),
])
def test_oracle_jacobians_by_central_differences(kind, shape, params):
    # pattern of pkg/tests/test_nonlinear.py:329-346 (relative 1e-5)
    from oracle.problems import build_problem

    prob = GridProblem(kind, shape, **params)
    pd = build_problem(kind, shape, **prob.oracle_params())
    rng = np.random.default_rng(1)
    u = rng.standard_normal(pd.dim)
    jac = pd.linearize_csr(u, 0.0).toarray()
    eps = 1e-6
    fd = np.empty_like(jac)
    for j in range(pd.dim):
        e = np.zeros(pd.dim)
        e[j] = eps
        fd[:, j] = (pd.rhs(u + e, 0.0) - pd.rhs(u - e, 0.0)) / (2 * eps)
    assert np.max(np.abs(fd - jac)) <= 1e-5 * max(1.0, np.max(np.abs(jac)))


def test_grid_problem_validation():
    with pytest.raises(ValueError):
        GridProblem("heat", (4, 4))
    with pytest.raises(ValueError):
        GridProblem("nldiff", (0, 4))
    p = GridProblem("burgers", (8, 4), nu=0.1)
    assert p.dim == 32 and p.mass is None and p.name == "burgers2d"
    assert p.h == (1.0 / 8, 1.0 / 4)


# -------------------------------------------------------------- C ABI


def _header_symbols():
    with open(os.path.join(ROOT, "include", "irkg.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(irkg_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.irkg_version().decode().startswith("irkg")


def test_ctypes_struct_layout_matches_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "irkg.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu\\n\","
        " sizeof(irkg_problem), sizeof(irkg_tableau), sizeof(irkg_solver),"
        " sizeof(irkg_krylov_report), sizeof(irkg_step_stats), sizeof(irkg_counters),"
        " sizeof(irkg_opfield), offsetof(irkg_step_stats, fail_report));return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [C.sizeof(_lib.Problem), C.sizeof(_lib.Tableau), C.sizeof(_lib.Solver),
            C.sizeof(_lib.KrylovReportC), C.sizeof(_lib.StepStatsC), C.sizeof(_lib.Counters),
            C.sizeof(_lib.OpField), _lib.StepStatsC.fail_report.offset]
    assert got == want


def test_device_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    prob = GridProblem("nldiff", (8, 8))
    with pytest.raises(RuntimeError):
        pk.step(prob, np.zeros(64), 0.0, 1e-3, pk.make_tableau("gauss", 2),
                pk.SolverConfig(precond=pk.PrecondSpec(inner=4)))


def test_built_library_matches_sources():
    from paper_2101_01776_b200 import _build

    assert _build.is_fresh(), "libirkg.so is stale: run python -m paper_2101_01776_b200._build"


def test_reference_side_ctypes_stub_layout_matches_c(tmp_path):
    """include/irkg_ctypes.py -- the binding INTEGRATION.md tells a
    maintainer to add to irkit -- declares every struct with the header's
    exact size and field offsets (the r1 stub lacked length_y/length_z)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "irkg_ctypes", os.path.join(ROOT, "include", "irkg_ctypes.py"))
    stub = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(stub)
    checks = [("irkg_problem", stub.Problem, ["length", "length_y", "length_z"]),
              ("irkg_tableau", stub.Tableau, ["d", "nblocks", "blk_phi"]),
              ("irkg_solver", stub.Solver, ["inner", "jacobian_refresh", "variant0_stage"]),
              ("irkg_krylov_report", stub.KrylovReport, ["residuals"]),
              ("irkg_step_stats", stub.StepStats,
               ["n_block_records", "wall_time", "fail_report", "constraint_residual"])]
    lines = []
    for cname, _, fields in checks:
        lines.append(f'printf("%zu\\n", sizeof({cname}));')
        lines += [f'printf("%zu\\n", offsetof({cname}, {f}));' for f in fields]
    src = tmp_path / "stub.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "irkg.h"\n'
                   "int main(void){" + "".join(lines) + "return 0;}\n")
    exe = tmp_path / "stub"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = []
    for _, cls, fields in checks:
        want.append(C.sizeof(cls))
        want += [getattr(cls, f).offset for f in fields]
    assert got == want


def test_integration_md_embeds_the_stub_verbatim():
    """INTEGRATION.md shows include/irkg_ctypes.py's step_on_gpu as written
    (the GPU test runs that file), so the document cannot drift again."""
    with open(os.path.join(ROOT, "INTEGRATION.md")) as fh:
        doc = fh.read()
    with open(os.path.join(ROOT, "include", "irkg_ctypes.py")) as fh:
        src = fh.read()
    start = src.index("class Problem(C.Structure):")
    end = src.index("class Tableau(C.Structure):")
    assert src[start:end].strip() in doc
    start = src.index("def step_on_gpu(")
    assert src[start:].strip() in doc


def test_variant_weights_index_logic_matches_oracle():
    """variant_weights (src/nonlinear.py:99-126; bit-exact index logic):
    argmax |d_ii| first on ties, the variant-3 key set, weights from d."""
    from oracle import irk
    from oracle import tableau as otab

    for fam, s in (("gauss", 2), ("gauss", 3), ("radau_iia", 3), ("gauss", 4),
                   ("lobatto_iiic", 4), ("gauss", 5)):
        prep = pk.prepare_stages(pk.make_tableau(fam, s))
        oprep = otab.prepare(fam, s)
        for v in range(4):
            dw, ow = pk.variant_weights(prep, v)
            odw, oow = irk.variant_weights(oprep, v)
            assert np.array_equal(dw, odw)
            assert sorted(ow) == sorted(oow)
            for key in ow:
                assert np.array_equal(ow[key], oow[key])

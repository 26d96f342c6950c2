"""Butcher tableaux and prepared Schur stage data (host-only constants).

Mirrors the reference's tableau objects and entry points
(``src/tableau.py``: ``ButcherTableau`` 66-81, ``StagePrep`` 84-101,
``make_tableau`` 329-361, ``prepare_stages`` 364-379, ``gamma_star``
382-386; ``src/densela.py``: ``EigenBlock`` 39-57, ``SchurForm`` 60-69).

The constants are *consumed as-is*, never recomputed:
``data/tableaux.json`` holds the reference's own ``make_tableau`` +
``prepare_stages`` output for every collocation family and stage count,
bit-for-bit (hex floats), written by ``tests/golden/make_golden.py``.
Objects from the reference itself (``irkit.ButcherTableau`` /
``irkit.StagePrep``) are accepted anywhere a tableau or prep is expected.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError

_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "tableaux.json")

GAUSS = "gauss"
RADAU_IIA = "radau_iia"
LOBATTO_IIIC = "lobatto_iiic"
SDIRK_FAMILIES = ("sdirk1", "sdirk2", "sdirk3", "sdirk4")
COLLOCATION_FAMILIES = (GAUSS, RADAU_IIA, LOBATTO_IIIC)
_SDIRK_STAGES = {"sdirk1": 1, "sdirk2": 2, "sdirk3": 3, "sdirk4": 5}
MAX_COLLOCATION_STAGES = 8

_ALIASES = {
    "gauss": GAUSS,
    "radau": RADAU_IIA,
    "radauiia": RADAU_IIA,
    "radau_iia": RADAU_IIA,
    "lobatto": LOBATTO_IIIC,
    "lobattoiiic": LOBATTO_IIIC,
    "lobatto_iiic": LOBATTO_IIIC,
    "sdirk1": "sdirk1",
    "sdirk2": "sdirk2",
    "sdirk3": "sdirk3",
    "sdirk4": "sdirk4",
}


def canonical_family(name):
    """Family-name normalisation (src/tableau.py:57-63)."""
    key = str(name).strip().lower().replace("-", "_").replace(" ", "")
    key = key.replace("_", "") if key.replace("_", "") in _ALIASES else key
    if key not in _ALIASES:
        raise ConfigurationError(f"unknown scheme family {name!r}")
    return _ALIASES[key]


@dataclass(frozen=True)
class EigenBlock:
    offset: int
    size: int
    eta: float
    beta: float
    phi: float

    def eigenvalues(self):
        if self.size == 1:
            return (complex(self.eta, 0.0),)
        return (complex(self.eta, self.beta), complex(self.eta, -self.beta))


@dataclass(frozen=True)
class SchurForm:
    q: np.ndarray
    r: np.ndarray
    blocks: tuple

    def eigenvalues(self):
        return np.array([lam for blk in self.blocks for lam in blk.eigenvalues()])


@dataclass(frozen=True)
class ButcherTableau:
    family: str
    s: int
    a0: np.ndarray
    b0: np.ndarray
    c0: np.ndarray
    order: int

    @property
    def is_dirk(self):
        return bool(np.all(np.triu(self.a0, 1) == 0.0))

    @property
    def label(self):
        return f"{self.family}({self.s})"


@dataclass(frozen=True)
class StagePrep:
    tableau: ButcherTableau
    a0inv: np.ndarray
    schur: SchurForm
    d: np.ndarray

    @property
    def blocks(self):
        return self.schur.blocks


_TABLE = None


def _table():
    global _TABLE
    if _TABLE is None:
        with open(_DATA) as fh:
            _TABLE = json.load(fh)
    return _TABLE


def _arr(v):
    a = np.array([float.fromhex(x) for x in v["data"]], dtype=float)
    return a.reshape(v["shape"])


def _entry(family, s):
    key = f"{family}:{s}"
    doc = _table().get(key)
    if doc is None:
        raise ConfigurationError(f"no prepared tableau for {family}({s})")
    return doc


def make_tableau(family, s=None):
    """Construct the Butcher tableau for ``(family, s)`` (src/tableau.py:329-361).

    SDIRK baselines (src/tableau.py:283-326) have their stage count fixed by
    the scheme (a mismatching ``s`` is a configuration error, 336-341); they
    are stepped stage by stage (src/nonlinear.py:239-296, ``irkg_dirk_step``).
    """
    family = canonical_family(family)
    if family in SDIRK_FAMILIES:
        fixed = _SDIRK_STAGES[family]
        if s is not None and int(s) != fixed:
            raise ConfigurationError(f"{family} has s = {fixed}, got s = {s}")
        doc = _entry(family, fixed)
        return ButcherTableau(
            family=doc["family"], s=fixed, a0=_arr(doc["a0"]), b0=_arr(doc["b0"]),
            c0=_arr(doc["c0"]), order=int(doc["order"]),
        )
    if s is None:
        raise ConfigurationError(f"{family} requires an explicit stage count")
    s = int(s)
    lo = 2 if family == LOBATTO_IIIC else 1
    if not (lo <= s <= MAX_COLLOCATION_STAGES):
        raise ConfigurationError(
            f"{family} supports {lo} <= s <= {MAX_COLLOCATION_STAGES}, got {s}"
        )
    doc = _entry(family, s)
    return ButcherTableau(
        family=doc["family"], s=int(doc["s"]), a0=_arr(doc["a0"]), b0=_arr(doc["b0"]),
        c0=_arr(doc["c0"]), order=int(doc["order"]),
    )


def prepare_stages(tableau):
    """A0^{-1}, its real Schur form and d[k,l,i] = q[i,k] q[i,l]
    (src/tableau.py:364-379), from the reference's own values."""
    fam = canonical_family(tableau.family)
    if fam in SDIRK_FAMILIES:
        raise ConfigurationError(
            f"{tableau.family} is stepped stage by stage (src/nonlinear.py:239-296); "
            "it has no prepared Schur data"
        )
    doc = _entry(fam, int(tableau.s))
    if not np.array_equal(np.asarray(tableau.a0, dtype=float), _arr(doc["a0"])):
        raise ConfigurationError(
            f"{tableau.family}({tableau.s}): coefficient matrix differs from the prepared "
            "constants; pass the reference's StagePrep instead"
        )
    blocks = tuple(
        EigenBlock(int(b[0]), int(b[1]), float.fromhex(b[2]), float.fromhex(b[3]),
                   float.fromhex(b[4]))
        for b in doc["blocks"]
    )
    schur = SchurForm(q=_arr(doc["q"]), r=_arr(doc["r"]), blocks=blocks)
    return StagePrep(tableau=tableau, a0inv=_arr(doc["a0inv"]), schur=schur, d=_arr(doc["d"]))


def gamma_star(eta, beta):
    """Optimal Schur-complement shift ``eta + beta**2/eta`` (src/tableau.py:382-386)."""
    if eta <= 0.0:
        raise ValueError(f"eta must be positive, got {eta}")
    return eta + beta * beta / eta


def is_sdirk(tableau):
    return str(tableau.family) in SDIRK_FAMILIES

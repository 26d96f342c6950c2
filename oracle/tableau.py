"""Prepared Butcher/Schur stage constants for the oracle (test infrastructure).

The reference computes these on the host once per integration
(``make_tableau`` ``src/tableau.py:329-361``; ``prepare_stages``
``src/tableau.py:364-379`` = ``lu_solve(A0, I)`` -> ``real_schur`` ->
``d[k,l,i] = q[i,k] q[i,l]``).  They are consumed as-is: the fixture
``tests/golden/tableaux.json`` holds the reference's own values bit-for-bit
(hex floats), written by ``tests/golden/make_golden.py`` from the real
reference in the build container.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

_FIXTURE = os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
    "tests",
    "golden",
    "tableaux.json",
)


def _arr(v):
    a = np.array([float.fromhex(x) for x in np.ravel(v["data"])], dtype=float)
    return a.reshape(v["shape"])


@dataclass(frozen=True)
class Block:
    offset: int
    size: int
    eta: float
    beta: float
    phi: float


@dataclass(frozen=True)
class Tableau:
    family: str
    s: int
    order: int
    a0: np.ndarray
    b0: np.ndarray
    c0: np.ndarray


@dataclass(frozen=True)
class Prep:
    tableau: Tableau
    a0inv: np.ndarray
    q: np.ndarray
    r: np.ndarray
    blocks: tuple
    d: np.ndarray


_CACHE = None


def _load():
    global _CACHE
    if _CACHE is None:
        with open(_FIXTURE) as fh:
            _CACHE = json.load(fh)
    return _CACHE


def prepare(family, s):
    doc = _load()[f"{family}:{s}"]
    tab = Tableau(
        family=doc["family"],
        s=int(doc["s"]),
        order=int(doc["order"]),
        a0=_arr(doc["a0"]),
        b0=_arr(doc["b0"]),
        c0=_arr(doc["c0"]),
    )
    blocks = tuple(
        Block(int(b[0]), int(b[1]), float.fromhex(b[2]), float.fromhex(b[3]), float.fromhex(b[4]))
        for b in doc["blocks"]
    )
    return Prep(
        tableau=tab,
        a0inv=_arr(doc["a0inv"]),
        q=_arr(doc["q"]),
        r=_arr(doc["r"]),
        blocks=blocks,
        d=_arr(doc["d"]),
    )


def dirk_tableau(family):
    """SDIRK coefficients (src/tableau.py:283-326, make_tableau 336-341),
    from the reference's own values."""
    for key, doc in _load().items():
        if key.split(":")[0] == family:
            return Tableau(family=doc["family"], s=int(doc["s"]), order=int(doc["order"]),
                           a0=_arr(doc["a0"]), b0=_arr(doc["b0"]), c0=_arr(doc["c0"]))
    raise KeyError(family)


def gamma_star(eta, beta):
    # src/tableau.py:382-386
    if eta <= 0.0:
        raise ValueError(f"eta must be positive, got {eta}")
    return eta + beta * beta / eta

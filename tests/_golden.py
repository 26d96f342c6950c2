"""Helpers to load the reference-generated fixtures under tests/golden/."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_names(dae=False):
    out = []
    for p in sorted(glob.glob(os.path.join(GOLD, "*.json"))):
        name = os.path.basename(p)[:-5]
        if name in ("tableaux", "transformed"):
            continue
        if name.startswith("dae_") != dae:
            continue
        out.append(name)
    return out


def load_dae_case(name):
    with open(os.path.join(GOLD, name + ".json")) as fh:
        meta = json.load(fh)
    arrs = np.load(os.path.join(GOLD, name + ".npz"))
    for key in ("u0", "w0", "u_final", "w_final"):
        meta[key] = arrs[key]
    for st in meta["steps"]:
        st["residual_history"] = [float.fromhex(x) for x in st["residual_history"]]
        st["constraint_residual"] = float.fromhex(st["constraint_residual"])
        st["block_iterations"] = {int(k): v for k, v in st["block_iterations"].items()}
    return meta


def load_case(name):
    with open(os.path.join(GOLD, name + ".json")) as fh:
        meta = json.load(fh)
    arrs = np.load(os.path.join(GOLD, name + ".npz"))
    meta["u0"] = arrs["u0"]
    meta["u_final"] = arrs["u_final"]
    for st in meta["steps"]:
        st["residual_history"] = [float.fromhex(x) for x in st["residual_history"]]
        st["block_iterations"] = {int(k): v for k, v in st["block_iterations"].items()}
    return meta


def grid_problem(meta):
    from paper_2101_01776_b200.problems import GridProblem

    p = meta["params"]
    return GridProblem(meta["kind"], tuple(meta["shape"]), nu=p["nu"], c=p["c"], lam=p["lam"],
                       mu=p["mu"], length=p["length"])


def load_transformed():
    with open(os.path.join(GOLD, "transformed.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        k = c["k"]
        c["k"] = np.array([float.fromhex(x) for x in k["data"]]).reshape(k["shape"])
    return cases


def oracle_config(solver):
    from oracle import irk

    fields = irk.Config.__dataclass_fields__
    return irk.Config(**{k: v for k, v in solver.items() if k in fields})

"""Dump block-operator / block-GMRES results for an A/B of two engine paths.

Run twice with different env settings (e.g. IRKG_STRIP_OP=0 / 1) and compare
the .npz files:  python tools/op_check.py out_a.npz; python tools/op_check.py
out_b.npz; python tools/op_check.py --cmp out_a.npz out_b.npz
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def dump(path, n=128, kind="burgers"):
    import numpy as np

    import paper_2101_01776_b200 as pk

    prob = pk.GridProblem(kind, (n, n), nu=1e-2)
    rng = np.random.default_rng(1)
    U = pk.fourier_u0((n, n), 1, 8, 0.5, 0)
    f1 = pk.OperatorField.linearize(prob, np.stack([U, 0.5 * U]), [0.7, 0.3])
    f2 = pk.OperatorField.linearize(prob, np.stack([U, -U]), [0.2, 0.5])
    c = pk.OperatorField.linearize(prob, np.stack([U]), [0.1])
    sys2 = pk.Block2x2System(3.677815, 3.508762, -10.983731, None, f1, f2, 5e-4, c, c)
    z = rng.standard_normal(2 * n * n)
    y2 = pk.apply_block2x2(sys2, z)
    rhs2 = rng.standard_normal(2 * n * n)
    x2, rep2 = pk.block_gmres(sys2, rhs2, pk.PrecondSpec(inner=4), rtol=1e-8, maxit=60,
                              restart=30)
    rhs1 = rng.standard_normal(n * n)
    x1, rep1 = pk.block_gmres((4.644371, f1, 5e-4), rhs1, pk.PrecondSpec(inner=4), rtol=1e-8,
                              maxit=60, restart=30)
    np.savez(path, y2=y2, x2=x2, x1=x1, it2=rep2.iterations, it1=rep1.iterations,
             r2=np.array(rep2.residuals), r1=np.array(rep1.residuals))
    print(path, "its", rep2.iterations, rep1.iterations)


def cmp(a, b):
    import numpy as np

    A, B = np.load(a), np.load(b)
    for k in A.files:
        x, y = A[k], B[k]
        if x.shape != y.shape:
            print(k, "shape", x.shape, y.shape)
            continue
        d = np.abs(x - y).max() if x.size else 0.0
        print(f"{k:4s} max|diff| {d:.3e}  max|a| {np.abs(x).max() if x.size else 0:.3e}")


if __name__ == "__main__":
    if sys.argv[1] == "--cmp":
        cmp(sys.argv[2], sys.argv[3])
    else:
        dump(sys.argv[1])

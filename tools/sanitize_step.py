"""One configs[1]-style step (2-D Burgers Gauss(3), Jacobi-4) at 64^2 plus
one 2x2 block GMRES with a ragged CGS tail tile, for compute-sanitizer runs
(tools/sanitize.sh).  Engine knobs (IRKG_GRAPHS, IRKG_PDL) come from the
environment.  Checks the step against the committed reference golden."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2101_01776_b200 as pk  # noqa: E402
from _golden import grid_problem, load_case  # noqa: E402

meta = load_case("cfg1_n64")
prob = grid_problem(meta)
cfg = pk.SolverConfig(krylov_maxit=5000, precond=pk.PrecondSpec(inner=4))
u1, st = pk.step(prob, meta["u0"], 0.0, meta["dt"], pk.make_tableau("gauss", 3), cfg)
want = meta["steps"][0]
assert st.newton_iterations == want["newton_iterations"], st.newton_iterations
assert abs(st.krylov_iterations - want["krylov_iterations"]) <= 1
# 2x2 block GMRES on 2N = 2 * 66 * 50 (partial last CGS tile), restart 8
prob2 = pk.GridProblem("burgers", (66, 50), nu=1e-2)
rng = np.random.default_rng(1)
U = 0.5 * rng.standard_normal((2, prob2.dim))
f1 = pk.OperatorField.linearize(prob2, U[:1])
f2 = pk.OperatorField.linearize(prob2, U[1:])
sysb = pk.Block2x2System(3.677815, 3.508762, -10.983731, None, f1, f2, 5e-3)
x, rep = pk.block_gmres(sysb, rng.standard_normal(2 * prob2.dim), pk.PrecondSpec(inner=4),
                        1e-10, 300, 8)
assert rep.converged
print(f"sanitize step ok: graphs={os.environ.get('IRKG_GRAPHS', '1')} "
      f"pdl={os.environ.get('IRKG_PDL', '1')} newton={st.newton_iterations} "
      f"krylov={st.krylov_iterations} block_gmres_its={rep.iterations}")

import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2101_01776_b200 as pk
from paper_2101_01776_b200.engine import context_for
spec = pk.baseline_config(1)
tab = pk.make_tableau(spec.family, spec.s)
prep = pk.prepare_stages(tab)
sv = spec.solver
cfg = pk.SolverConfig(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"], restart=sv["restart"],
                      newton_maxit=sv["newton_maxit"], precond=pk.PrecondSpec(inner=sv["inner"]))
prob = spec.problem
uh = spec.u0()
t = 0.0
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    uh2, st = pk.step(prob, uh, t, spec.dt, tab, cfg)
    torch.cuda.synchronize(); a = time.perf_counter() - t0
    ctx = context_for(prob)
    ud = torch.from_numpy(uh).cuda(); torch.cuda.synchronize(); t0 = time.perf_counter()
    st2 = ctx.step_device(ud, t, spec.dt); torch.cuda.synchronize(); b = time.perf_counter() - t0
    t0 = time.perf_counter(); uh3, st3 = pk.step(prob, uh, t, spec.dt, tab, cfg, prep=prep); torch.cuda.synchronize(); c = time.perf_counter() - t0
    print(f"pk.step {a*1e3:.1f} ms (newton {st.newton_iterations} kry {st.krylov_iterations}) | step_device {b*1e3:.1f} ms (newton {st2.newton_iterations}) | pk.step(prep) {c*1e3:.1f}", flush=True)
    uh = uh2; t += spec.dt

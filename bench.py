#!/usr/bin/env python
"""Benchmark of the IRK stage-equation solve on B200 (BASELINE.json metric).

Workload (N = 1): BASELINE ``configs[1]`` -- 2-D viscous Burgers on a
1024^2 periodic grid, nu = 1e-2, Gauss 3-stage (order 6), dt = 5e-4,
seeded Fourier-mode u0 (|k| <= 8, sigma = 0.5); manifest: variant 3,
gamma*, Jacobi-4 inner solves, restart 200, krylov_maxit 5000, Newton rtol
1e-9, Krylov rtol 1e-5 (reference defaults).  A "step" is one IRK time step
(all Newton iterations of the stage solve + the u update), marching the same
trajectory: W warm-up steps, then K timed steps.

Headline metric: stage-DOF updates/s = sum_steps(newton_its * s * N) / time
(SURVEY 8d); IRK steps/s and the CGS2 roofline are reported beside it.

``--impl reference`` times the reference algorithm's CPU restatement
(``oracle/``, a numpy/scipy port of irkit; the reference itself is Python and
cannot travel to the GPU box) on the host cores: each of its steps is one full
Newton iteration of the same trajectory at full size (a bounded sample).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stage-DOF updates/s (IRK stage solve; configs[1] Burgers 1024^2 Gauss(3))"
UNIT = "DOF/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks / throttle reasons during the timed region.

    NVML in-process (20 ms polls; the timed region of the default run is only
    ~0.3 s, shorter than an `nvidia-smi -lms` start-up, which left runs with no
    samples), falling back to an `nvidia-smi -lms 50` subprocess.  `__enter__`
    returns only after the first sample, so the timed region is covered.
    """

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0, period=0.02):
        self.index = index
        self.period = period
        self.proc = None
        self.thread = None
        self.stop = threading.Event()
        self.samples = []  # (sm_mhz, max_mhz, set(reasons))
        self.source = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
                    "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

            def poll():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx),
                                     {n for n, b in bits.items() if r & b}))

            poll()
            self.source = "nvml"

            def loop():
                while not self.stop.wait(self.period):
                    try:
                        poll()
                    except Exception:
                        return

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.samples = []
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
            first = threading.Event()

            def read():
                for line in self.proc.stdout:
                    parts = [p.strip() for p in line.split(",")]
                    try:
                        self.samples.append((float(parts[0]), float(parts[1]),
                                             {n for n, f in zip(self.NAMES, parts[3:7])
                                              if f.lower() == "active"}))
                    except (ValueError, IndexError):
                        continue
                    first.set()

            self.thread = threading.Thread(target=read, daemon=True)
            self.thread.start()
            first.wait(timeout=5)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)

    def summary(self):
        sm = [s[0] for s in self.samples]
        reasons = set().union(*[s[2] for s in self.samples]) if self.samples else set()
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": self.samples[-1][1] if self.samples else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        import torch

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------ CPU leg


class OracleNewtonStream:
    """Newton iterations of the configs[1] trajectory on the CPU oracle, one
    per call (a complete reference Newton iteration: linearize s stages,
    variant-3 combine, transformed solve, residual)."""

    def __init__(self, spec):
        from oracle import irk
        from oracle import tableau as otab
        from oracle.problems import build_problem

        self.irk = irk
        prob = spec.problem
        pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
        self.sys = irk.OdeSystem(pd.dim, pd.rhs, pd.linearize_csr)
        self.prep = otab.prepare(spec.family, spec.s)
        sv = spec.solver
        self.cfg = irk.Config(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"],
                              restart=sv["restart"], inner=sv["inner"],
                              newton_maxit=sv["newton_maxit"])
        self.dt = spec.dt
        self.u = spec.u0()
        self.t = 0.0
        self.s = spec.s
        self.n = pd.dim
        self._new_step()

    def _new_step(self):
        irk, tab = self.irk, self.prep.tableau
        self.k = np.zeros((self.s, self.n))
        self.res = irk.stage_residual(self.sys, self.u, self.k, self.t, self.dt, tab)
        f0 = np.linalg.norm(self.res)
        self.tol = max(self.cfg.newton_rtol * f0, self.cfg.newton_abs_floor)

    def newton_iteration(self):
        irk, tab, cfg = self.irk, self.prep.tableau, self.cfg
        if np.linalg.norm(self.res) <= self.tol:
            self.u = self.u + self.dt * (tab.b0 @ self.k)
            self.t += self.dt
            self._new_step()
        times = self.t + tab.c0 * self.dt
        u_stage = self.u[None, :] + self.dt * (tab.a0 @ self.k)
        ops = [self.sys.linearize(u_stage[i], times[i]) for i in range(self.s)]
        vjac = irk.build_variant_jacobian(self.prep, ops, cfg.variant, cfg.variant0_stage)
        dk, st = irk.solve_transformed(self.prep, vjac, self.dt, self.res, cfg.gamma_mode,
                                       cfg.inner, cfg.krylov_rtol, cfg.krylov_maxit, cfg.restart)
        self.k = self.k + dk
        self.res = irk.stage_residual(self.sys, self.u, self.k, self.t, self.dt, tab)
        return st.krylov_iterations


def cpu_sample(spec, n_iters):
    threads = os.cpu_count() or 1
    stream = OracleNewtonStream(spec)
    t0 = time.perf_counter()
    kry = 0
    for _ in range(n_iters):
        kry += stream.newton_iteration()
    dt = time.perf_counter() - t0
    dof = n_iters * spec.s * spec.problem.dim / dt
    return dof, dt, kry, threads


def run_reference(args, spec, ws, rank):
    if rank != 0:
        return
    stream = OracleNewtonStream(spec)
    for _ in range(args.warmup):
        stream.newton_iteration()
    t0 = time.perf_counter()
    kry = 0
    for _ in range(args.steps):
        kry += stream.newton_iteration()
    el = time.perf_counter() - t0
    value = args.steps * spec.s * spec.problem.dim / el
    cores = os.cpu_count() or 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Fourier-mode u0)",
        "config": {"workload": spec.name, "grid": list(spec.problem.shape), "scheme": "gauss(3)",
                   "dt": spec.dt, "inner": "jacobi-4", "variant": 3},
        "cpu_baseline": {
            "value": value, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{args.steps} full Newton iterations (after {args.warmup} warm-up) of the "
                      f"configs[1] trajectory at full 1024^2 size on the numpy/scipy restatement "
                      f"of irkit (oracle/irk.py); {kry} Krylov iterations",
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU leg


def run_ours(args, spec, ws, rank, local):
    import torch

    import paper_2101_01776_b200 as pk
    from paper_2101_01776_b200.engine import Context

    torch.cuda.set_device(local)
    prob = spec.problem
    tab = pk.make_tableau(spec.family, spec.s)
    prep = pk.prepare_stages(tab)
    sv = spec.solver
    cfg = pk.SolverConfig(variant=sv["variant"], krylov_maxit=sv["krylov_maxit"],
                          restart=sv["restart"], newton_maxit=sv["newton_maxit"],
                          precond=pk.PrecondSpec(inner=sv["inner"]))
    u0 = spec.u0()
    if ws > 1:
        # weak scaling: configs[1] tiled ws times along y (same h, dt, nu); rank r
        # owns one 1024^2 slab (= the N = 1 field, since u0 is 1-periodic);
        # halos over NCCL, every inner product all-reduced (csrc/comm.cu)
        from paper_2101_01776_b200.distributed import SlabContext

        nx, ny = prob.shape
        prob = pk.GridProblem(prob.kind, (nx, ny * ws), nu=prob.nu,
                              lengths=(prob.length, prob.length * ws))
        ctx = SlabContext(prob, rank, ws, transport="nccl", device=local)
    else:
        ctx = Context(prob, local)
    ctx.set_prep(prep)
    ctx.set_config(cfg)
    u = torch.from_numpy(u0).cuda()
    stream = torch.cuda.current_stream()
    N = u.numel()  # points owned by this rank
    t = 0.0
    for _ in range(args.warmup):
        ctx.step_device(u, t, spec.dt)
        t += spec.dt
    torch.cuda.synchronize()
    # the roofline and e2e passes below replay exactly these timed steps (same
    # state, same t => same Newton/Krylov work), so their numbers compare 1:1
    u_start, t_start = u.clone(), t
    c0 = ctx.counters()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stats = []
    with ClockSampler(local) as clk:
        barrier(ws)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            stats.append(ctx.step_device(u, t, spec.dt))
            t += spec.dt
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
    c1 = ctx.counters()
    ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms, ws)
    newton = sum(s.newton_iterations for s in stats)
    krylov = sum(s.krylov_iterations for s in stats)
    dof = sum_over_ranks(newton * spec.s * N, ws)
    value = dof / (ms * 1e-3)
    steps_per_s = args.steps / (ms * 1e-3)
    launches = int(c1["kernel_launches"] - c0["kernel_launches"])

    # roofline pass: device time of the CGS2 sweeps (CUDA events on the engine
    # stream around the 4 sweeps of each Arnoldi step) over extra steps
    ctx.set_timing(True)
    u.copy_(u_start)
    t = t_start
    r0 = ctx.counters()
    rsteps = max(1, min(args.steps, 3))
    tr0 = time.perf_counter()
    for _ in range(rsteps):
        ctx.step_device(u, t, spec.dt)
        t += spec.dt
    torch.cuda.synchronize()
    tr = time.perf_counter() - tr0
    ctx.set_timing(False)
    r1 = ctx.counters()
    cgs_bytes = r1["cgs_bytes"] - r0["cgs_bytes"]
    cgs_ms = r1["cgs_time_ms"] - r0["cgs_time_ms"]
    cgs_launch = r1["cgs_launches"] - r0["cgs_launches"]
    peak, peak_kind = _peaks()
    achieved = cgs_bytes / (cgs_ms * 1e-3) / 1e9 if cgs_ms > 0 else 0.0
    traffic, tnote = None, None
    try:  # DRAM bytes per CGS launch from the committed ncu capture (j = 8 sweeps)
        tname = next(f for f in ("r1s4_cgs_traffic.json", "r1s3_cgs_traffic.json")
                     if os.path.exists(os.path.join(ROOT, "profiles", f)))
        with open(os.path.join(ROOT, "profiles", tname)) as fh:
            tdoc = json.load(fh)
        traffic = tdoc["traffic_per_launch"]
        tnote = (f"ncu --set full, CGS sweeps at j={tdoc['j']}: {traffic / 1e6:.1f} MB DRAM per launch "
                 f"vs {tdoc['algorithmic_per_launch'] / 1e6:.1f} MB algorithmic "
                 f"(ratio {tdoc['ratio']:.3f}; profiles/{tname})")
    except (OSError, KeyError, ValueError, StopIteration):
        pass
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_note": tnote,
            "kernel": "k_cgs<DOT|UPD_DOT|UPD_NORM> (CGS2 sweeps)",
            "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
            "algorithmic_bytes_per_launch": cgs_bytes / max(1, cgs_launch),
            "avg_launch_us": 1e3 * cgs_ms / max(1, cgs_launch),
            "share_of_step": (cgs_ms * 1e-3) / tr if tr > 0 else None}

    # e2e: the public API with host buffers (H2D of u + D2H of u_next per step)
    # the caller's state in page-locked memory (pk.step returns u_next pinned too)
    uh = u_start.cpu().pin_memory().numpy()
    t = t_start
    if ws == 1:  # untimed: the caching host allocator's first page-locked blocks
        for _ in range(2):
            pk.step(prob, uh, t, spec.dt, tab, cfg, prep=prep)
    e_stats = []
    barrier(ws)
    te0 = time.perf_counter()
    for _ in range(args.steps):
        if ws > 1:  # the slab context's host-buffer step (irkg_step_host)
            st = ctx.step_host(uh, t, spec.dt)
        else:  # the public irkit-style API with a host numpy state
            uh, st = pk.step(prob, uh, t, spec.dt, tab, cfg, prep=prep)
        e_stats.append(st)
        t += spec.dt
    te = max_over_ranks(time.perf_counter() - te0, ws)
    e_dof = sum_over_ranks(sum(s.newton_iterations for s in e_stats) * spec.s * N, ws)
    e2e = {"value": e_dof / te, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
           "d2h_bytes_per_step": 8 * N, "steps_per_s": args.steps / te}

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Fourier-mode u0, BASELINE configs[1] shape)",
            "config": {"workload": spec.name, "grid": list(prob.shape), "scheme": "gauss(3)",
                       "dt": spec.dt, "inner": "jacobi-4", "variant": 3, "restart": 200,
                       "parallelism": (f"slab{ws} (y-slabs, NCCL halos + allreduce; weak: "
                                       f"configs[1] tiled {ws}x in y)") if ws > 1 else "1 GPU",
                       "global_grid": list(prob.shape),
                       "l2": "working set > L2 (V basis 201 x 16.8 MB per rank)"},
            "steps_per_s": steps_per_s, "newton_iterations": newton, "krylov_iterations": krylov,
            "gpu_launches": launches, "roofline": roof, "e2e": e2e, "clocks": clk.summary(),
        }
        if ws == 1 and not args.no_cpu:
            dof_cpu, el, kry, cores = cpu_sample(spec, 1)
            line["cpu_baseline"] = {
                "value": dof_cpu, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": f"first Newton iteration of step 1 at full 1024^2 on the numpy/scipy "
                          f"restatement of irkit (oracle/irk.py): {el:.1f} s, {kry} Krylov its",
            }
        print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override grid size (testing)")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    from paper_2101_01776_b200.problems import baseline_config

    spec = baseline_config(1, n=args.n)
    if args.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, spec, ws, rank)
        return
    ws, rank, local = dist_init()
    run_ours(args, spec, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()

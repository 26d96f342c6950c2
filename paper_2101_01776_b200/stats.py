"""Result / statistics carriers (mirror of the reference's).

``KrylovReport`` src/sparsela.py:155-162, ``SolveStats`` src/irk_core.py:197-212,
``StepStats`` src/nonlinear.py:155-179, ``IntegrationResult``
src/nonlinear.py:317-328, ``write_step_stats_csv`` src/nonlinear.py:377-417.
These counters are the parity observables: the device path fills them
exactly as the reference does.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, field

import numpy as np


@dataclass
class KrylovReport:
    iterations: int
    converged: bool
    residuals: list = field(default_factory=list)
    precond_applications: int = 0


@dataclass
class SolveStats:
    reports: list = field(default_factory=list)  # (block_offset, KrylovReport)

    @property
    def krylov_iterations(self):
        return sum(rep.iterations for _, rep in self.reports)

    @property
    def precond_applications(self):
        return sum(rep.precond_applications for _, rep in self.reports)

    def merge(self, other):
        self.reports.extend(other.reports)


@dataclass
class StepStats:
    newton_iterations: int = 0
    krylov_iterations: int = 0
    precond_applications: int = 0
    jacobian_assemblies: int = 0
    converged: bool = False
    residual_history: list = field(default_factory=list)
    block_iterations: dict = field(default_factory=dict)  # offset -> [its, ...]
    constraint_residual: float = 0.0
    differential_solves: int = 0
    constraint_solves: int = 0
    wall_time: float = 0.0

    def add_solve(self, solve_stats):
        self.krylov_iterations += solve_stats.krylov_iterations
        self.precond_applications += solve_stats.precond_applications
        for off, rep in solve_stats.reports:
            self.block_iterations.setdefault(off, []).append(rep.iterations)


@dataclass
class IntegrationResult:
    times: np.ndarray
    states: list
    step_stats: list

    @property
    def u_final(self):
        return self.states[-1]

    def total(self, attr):
        return sum(getattr(s, attr) for s in self.step_stats)


def step_stats_from_c(cs):
    """Convert the C ``irkg_step_stats`` into a StepStats."""
    st = StepStats()
    st.newton_iterations = int(cs.newton_iterations)
    st.krylov_iterations = int(cs.krylov_iterations)
    st.precond_applications = int(cs.precond_applications)
    st.jacobian_assemblies = int(cs.jacobian_assemblies)
    st.converged = bool(cs.converged)
    st.residual_history = [float(cs.residual_history[i]) for i in range(cs.n_residuals)]
    for i in range(cs.n_block_records):
        st.block_iterations.setdefault(int(cs.block_offset[i]), []).append(
            int(cs.block_iterations[i])
        )
    st.wall_time = float(cs.wall_time)
    st.differential_solves = int(cs.differential_solves)
    st.constraint_solves = int(cs.constraint_solves)
    st.constraint_residual = float(cs.constraint_residual)
    return st


def write_step_stats_csv(result, path):
    """Per-step statistics as CSV, same columns as the reference."""
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(
            [
                "step",
                "newton_iterations",
                "krylov_iterations",
                "block_iterations",
                "precond_applications",
                "differential_solves",
                "constraint_solves",
                "wall_time",
            ]
        )
        for j, st in enumerate(result.step_stats):
            blocks = ";".join(
                f"{off}:{'+'.join(str(i) for i in its)}"
                for off, its in sorted(st.block_iterations.items())
            )
            writer.writerow(
                [
                    j,
                    st.newton_iterations,
                    st.krylov_iterations,
                    blocks,
                    st.precond_applications,
                    st.differential_solves,
                    st.constraint_solves,
                    repr(float(st.wall_time)),
                ]
            )

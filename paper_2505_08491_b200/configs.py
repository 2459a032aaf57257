"""The BASELINE.json configurations as problem builders (SURVEY.md section 8d,
Appendix A).  Inputs are seeded synthetic graphs (the paper's graph pools
are generated, not distributed).

Semantics chosen where BASELINE.json and the reference API differ:
n = cells + 1 (A1); homogeneous Dirichlet cube (A2); beta decoupled from R
(A3); R = eps with n_circle = 8 ring averaging (A4); fixed P1 elements per
segment (A5); the seeded random tree (A6); nodal 1D load f1D (A7); the
reference-test perturbed random net (A8); Jacobi(2, 2/3)-smoothed CNN
(A9); coupled maxit = reference default 2000 (A12).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import assembly as A
from . import geometry as G


@dataclass
class Workload:
    name: str
    systems: list
    cnn_seed: int
    restart: int
    tol: float
    maxit: int = 2000
    inner_iterations: int = 3
    smoothing: tuple = (2, 2.0 / 3.0)
    cnn_n: int = 0
    meta: dict = field(default_factory=dict)


def _system(n, graph, R, beta, epp, check_radius=True):
    return A.assemble_coupled_system(G.StructuredGrid(n), graph, A.PhysicalParams(epsilon=R, beta=beta),
                                     n_circle=8, elems_per_edge=epp, bc3d="dirichlet", f1d=1.0,
                                     check_radius=check_radius)


def cfg1() -> Workload:
    g = G.Graph1D([[0.5, 0.5, 0.1], [0.5, 0.5, 0.9]], [[0, 1]], 0.02, (0,))
    return Workload("cfg1", [_system(17, g, 0.02, 1.0, 32)], 0, 30, 1e-6,
                    meta={"grid": "16^3 cells", "graph": "segment", "elements_per_segment": 32})


def cfg2() -> Workload:
    g = G.random_tree(8, 1, 0.015)
    return Workload("cfg2", [_system(33, g, 0.015, 1.0, 16)], 1, 30, 1e-6,
                    meta={"grid": "32^3 cells", "graph": "random tree, 8 segments, seed 1",
                          "elements_per_segment": 16})


def cfg3() -> Workload:
    betas = np.random.default_rng(2).uniform(0.5, 2.0, 16)
    systems = [_system(65, G.random_tree(32, 2000 + i, 0.01), 0.01, float(betas[i]), 16) for i in range(16)]
    return Workload("cfg3", systems, 2, 50, 1e-6,
                    meta={"grid": "64^3 cells", "graph": "16 random trees x 32 segments, seeds 2000+i",
                          "elements_per_segment": 16, "beta": "U[0.5,2.0] seed 2"})


def cfg4() -> Workload:
    g = G.random_tree(64, 3, 0.008)
    return Workload("cfg4", [_system(129, g, 0.008, 1.0, 32, check_radius=False)], 3, 50, 1e-8,
                    meta={"grid": "128^3 cells", "graph": "random tree, 64 segments, seed 3",
                          "elements_per_segment": 32, "cnn_configured_for": "32^3 (seed 3), applied at 129^3"})


def cfg5_systems(n: int, batch: int) -> list:
    R = min(0.005, 0.9 / (n - 1))
    return [_system(n, G.random_tree(32, 4000 + i, R), R, 1.0, 16) for i in range(batch)]


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}

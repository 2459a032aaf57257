"""Fixtures for the BASELINE.json semantics the reference cannot express directly
(Dirichlet cube, nodal 1D load, beta != 2*pi*R: SURVEY.md Appendix A), produced
by the oracle restatement (itself pinned to the reference by
tests/test_oracle_golden.py).  Run in the build container:

    python tests/golden/make_oracle_golden.py [cfg1] [cfg2] [sens]
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import oracle  # noqa: E402
from oracle import problem as OP  # noqa: E402


def cfg1_system(n_circle=8):
    g = OP.segment_graph([0.5, 0.5, 0.1], [0.5, 0.5, 0.9], 0.02)
    return OP.assemble_coupled_system(OP.StructuredGrid(17), g, OP.PhysicalParams(epsilon=0.02, beta=1.0),
                                      n_circle=n_circle, elems_per_edge=32, bc3d="dirichlet", f1d=1.0)


def cfg2_system():
    g = OP.random_tree(8, 1, 0.015)
    return OP.assemble_coupled_system(OP.StructuredGrid(33), g, OP.PhysicalParams(epsilon=0.015, beta=1.0),
                                      n_circle=8, elems_per_edge=16, bc3d="dirichlet", f1d=1.0)


def f32(p):
    """Weights as the device sees them: float32-rounded (MDU3 round trip)."""
    return {k: {"kernel": v["kernel"].astype(np.float32).astype(float),
                "bias": None if v["bias"] is None else v["bias"].astype(np.float32).astype(float)}
            for k, v in p.items()}


def solve(s, seed, maxit, restart=30, tol=1e-6, scale=None):
    params = f32(oracle.noisy_params(seed))
    spec = {"type": "neural", "params": params, "smoothing": (2, 2.0 / 3.0)}
    st = oracle.CoupledStrategy(tol=tol, maxit=maxit, restart=restart, inner_iterations=3, three_d=spec)
    t0 = time.perf_counter()
    u3, u1, rep = oracle.solve_coupled(s, st)
    print(f"  iters {rep.iterations} conv {rep.converged} rel {rep.rel_residual:.3e} ({time.perf_counter() - t0:.0f}s)")
    return u3, u1, rep


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg1", "cfg2"]
    if "cfg1" in which:
        print("cfg1 baseline semantics")
        u3, u1, rep = solve(cfg1_system(), 0, 300)
        np.savez_compressed(HERE / "solve_cfg1_baseline.npz", iters=rep.iterations, conv=rep.converged,
                            hist=np.array(rep.residual_history), u3=u3, u1=u1)
    if "cfg1c" in which:
        print("cfg1 baseline semantics with the centreline restriction (n_circle=1)")
        u3, u1, rep = solve(cfg1_system(1), 0, 300)
        np.savez_compressed(HERE / "solve_cfg1_nc1.npz", iters=rep.iterations, conv=rep.converged,
                            hist=np.array(rep.residual_history), u3=u3, u1=u1)
    if "cfg2" in which:
        print("cfg2 baseline semantics, first 12 outer iterations")
        u3, u1, rep = solve(cfg2_system(), 1, 12)
        np.savez_compressed(HERE / "solve_cfg2_baseline_head.npz", iters=rep.iterations, conv=rep.converged,
                            hist=np.array(rep.residual_history))

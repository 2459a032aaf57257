"""Oracle coupled solve: outer FGMRES with the block preconditioner.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).
Restates ``harness.solve_coupled`` (harness.py:324-406) for the one_d='ilu0'
and 'direct' strategies with a 3D inner preconditioner of type none / ilu0 /
neural.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import problem as P
from .solver import fgmres, ilu0, ilu0_apply
from .unet import apply_neural


@dataclass
class CoupledStrategy:
    """harness.py:324-339 (one_d 'ilu0' or 'direct')."""

    tol: float = 1e-15
    maxit: int = 2000
    restart: int = 20
    inner_iterations: int = 3
    three_d: dict | None = None     # {"type": "none"|"ilu0"|"neural", "params":..., "smoothing":(m, w)}
    one_d: str = "ilu0"             # "ilu0" | "direct" (splu of A11, harness.py:356-358)


def mesh_distance_field(s: P.CoupledSystem) -> np.ndarray:
    """Distance field rebuilt from the refined mesh (harness.py:401-406)."""
    return P.distance_field(s.mesh.coords, s.mesh.elements, s.grid)


def make_inner(spec: dict | None, C, dvals):
    kind = (spec or {}).get("type", "none")
    if kind == "none":
        return None
    if kind == "ilu0":
        f = ilu0(C)
        return lambda r: ilu0_apply(f, r)
    if kind == "neural":
        params = spec["params"]
        sm = spec.get("smoothing")
        zd = spec.get("zero_distance", False)
        return lambda r: apply_neural(params, r, dvals, sm, C, zd)
    raise ValueError(f"unknown preconditioner type {kind!r}")


def solve_coupled(s: P.CoupledSystem, st: CoupledStrategy, dvals=None):
    """Returns (u3d, u1d, report) (harness.py:342-398)."""
    A = P.full_operator(s)
    F = P.full_rhs(s)
    n3 = s.n3
    w = s.params.coupling_weight
    A11 = P.one_d_operator(s)
    C = P.reduced_operator(s)
    if st.one_d == "direct":
        import scipy.sparse.linalg as spla
        lu11 = spla.splu(A11.tocsc())
        apply_1d = lu11.solve
    elif st.one_d == "ilu0":
        fact = ilu0(A11)
        apply_1d = lambda r: ilu0_apply(fact, r)  # noqa: E731
    else:
        raise ValueError(f"oracle one_d strategy {st.one_d!r} not restated")
    spec = st.three_d or {"type": "none"}
    if spec.get("type") == "neural" and dvals is None:
        dvals = mesh_distance_field(s)
    inner = make_inner(spec, C, dvals)
    m = st.inner_iterations

    def block_precond(r):
        z1 = apply_1d(r[n3:])
        z0, _ = fgmres(C, inner, r[:n3] - w * (s.M01 @ z1), restart=m, tol=1e-300, maxit=m)
        return np.concatenate([z0, z1])

    x, rep = fgmres(A, block_precond, F, restart=st.restart, tol=st.tol, maxit=st.maxit)
    u3d, u1d = x[:n3], x[n3:].copy()
    u1d[list(s.dirichlet_nodes)] = 1.0
    return u3d, u1d, rep

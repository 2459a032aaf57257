"""Coupled neural-preconditioned solve on the device (the north-star path).

``solve_coupled`` reproduces ``harness.solve_coupled`` (harness.py:342-398):
outer FGMRES on the block operator with the block right preconditioner

    z1 = ILU0(A11)^-1 r1
    z0 = FGMRES(C, P3, r0 - w M01 z1, restart=m, tol=1e-300, maxit=m)

and the eliminated Dirichlet values reimposed on u1d.  Given a list of
systems on one grid it solves them concurrently (the paper's multi-query
setting): every kernel runs once per step over all systems still
iterating, each system keeping its own FGMRES state.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _ext
from .assembly import CoupledSystem, DeviceProblem, full_rhs, host_reduced_operator, one_d_operator
from .geometry import DistanceField, distance_field_device
from .krylov import (DeviceIlu, ExactPreconditioner, FgmresEngine, FixedStepFgmres, GmgPreconditioner,
                     IluPreconditioner, SolveReport, direct_1d, gmg_build, ilu0)
from .neural import PATH_TCGEN05, UNetParams, device_net, load_checkpoint
from .operators import CoupledOperator, CouplingOps, ReducedOperator
from .training import BatchedNeural, NeuralPreconditioner


@dataclass
class CoupledStrategy:
    """harness.py:324-339.  ``one_d``: 'ilu0' (the reference default), 'direct'
    (exact 1D solve, harness.py:356-358) or 'schur' (the true Schur complement,
    harness.py:359-368); ``three_d``: a preconditioner spec or 'direct' (exact
    3D solve, harness.py:373-375).  The exact variants factor dense matrices in
    HBM (krylov.ExactPreconditioner), so they are limited to small grids."""

    tol: float = 1e-15
    maxit: int = 2000
    restart: int = 20
    inner_iterations: int = 3
    one_d: str = "ilu0"
    three_d: object = None


def build_preconditioner(spec: dict, grid, C, dfield: DistanceField):
    """Preconditioner factory (harness.py:204-226) for the device path.

    Supported: 'none', 'neural' (checkpoint path or in-memory ``params``,
    optional ``smoothing``/``zero_distance``), the 'gmg' baseline (device
    V-cycles), 'ilu0' (host factor, device level-scheduled sweeps) and 'exact'
    (dense device Cholesky, small grids).
    """
    kind = spec.get("type", "none")
    if kind == "none":
        return None
    if kind == "neural":
        params = spec.get("params") or load_checkpoint(spec["checkpoint"])
        sm = spec.get("smoothing")
        smooth = (sm["maxit"], sm.get("omega", 2.0 / 3.0)) if isinstance(sm, dict) else sm
        return NeuralPreconditioner(params, dfield, smoothing=smooth, C=C,
                                    zero_distance=spec.get("zero_distance", False))
    if kind == "ilu0" and C is not None:
        return IluPreconditioner(C)
    if kind == "exact" and C is not None:
        return ExactPreconditioner(C)
    if kind == "gmg":  # the multigrid baseline (harness.py:218-221)
        levels = spec.get("levels", _default_levels(grid.n))
        return GmgPreconditioner(gmg_build(grid, C, levels), cycles=spec.get("cycles", 10))
    raise ValueError(f"preconditioner type {kind!r} is not on the device hot path")


def _default_levels(n: int) -> int:
    """harness.py:232-237."""
    levels = 1
    while (n - 1) % 2 == 0 and (n - 1) // 2 + 1 >= 3:
        n = (n - 1) // 2 + 1
        levels += 1
    return levels


class _BatchedExact:
    """Per-system exact (dense Cholesky) solves behind the batched apply_device interface."""

    def __init__(self, factors):
        self.factors = factors

    def first_sweep_spec(self):
        return None

    def apply_device(self, V, Z, sel, idx=None):
        for s in (sel.cpu().tolist() if idx is None else idx):
            self.factors[s].apply_device(V[s:s + 1], Z[s:s + 1], None, [0])


class _BatchedIlu:
    """Per-system 3D ILU(0) of C (krylov.py:247-284) behind the batched apply_device
    interface: host factors, one batched device sweep launch (graph-safe)."""

    def __init__(self, systems, ld):
        self.dev = DeviceIlu([ilu0(host_reduced_operator(s)) for s in systems])
        self.ld = ld
        self.lib = _ext.lib()

    def first_sweep_spec(self):
        return None

    def apply_device(self, V, Z, sel, idx=None, presmoothed=False):
        # the global-memory sweep keeps x in Z, so V and Z must be distinct storages
        _ext.check(self.lib.mdp_ilu0_apply(self.dev.desc, int(sel.numel()), sel.data_ptr(), V.data_ptr(),
                                           Z.data_ptr(), self.ld, _ext.stream()))


class _BatchedGmg:
    """Per-system GMG preconditioners behind the batched apply_device interface."""

    def __init__(self, precs, n3):
        self.precs, self.n3 = precs, n3

    def first_sweep_spec(self):
        return None

    def apply_device(self, V, Z, sel, idx=None):
        if idx is None:
            idx = sel.cpu().tolist()
        for s in idx:
            P = self.precs[s]
            P.hierarchy.device.apply(V[s, :self.n3], Z[s, :self.n3], P.cycles, P.n_pre, P.n_post)


def mesh_distance(system: CoupledSystem):
    """CNN distance channel from the refined mesh (harness.py:401-406), on the device."""
    return distance_field_device(system.graph_mesh.coords, system.graph_mesh.elements, system.grid)


class CoupledSolver:
    """Device state for repeated coupled solves of a batch of systems."""

    def __init__(self, systems, strategy: CoupledStrategy, path: int = PATH_TCGEN05, graphs: bool = True):
        import torch
        if strategy.one_d not in ("ilu0", "direct", "schur"):
            raise ValueError(f"unknown one_d={strategy.one_d!r}: 'ilu0', 'direct' or 'schur'")
        self.systems = list(systems)
        self.st = strategy
        self.prob = DeviceProblem(self.systems)
        p = self.prob
        self.A = CoupledOperator(p)
        self.C = ReducedOperator(p)
        self.cpl = CouplingOps(p)
        fac = direct_1d if strategy.one_d == "direct" else ilu0
        self.ilu = DeviceIlu([fac(one_d_operator(s)) for s in self.systems])
        self.lib = _ext.lib()
        self.exact3 = None   # three_d == "direct": per-system exact C solves replace the inner FGMRES
        self.schur = None    # one_d == "schur": per-system LU of the dense Schur complement
        if strategy.three_d == "direct" or strategy.one_d == "schur":
            self.exact3 = [ExactPreconditioner(host_reduced_operator(s)) for s in self.systems]
        if strategy.one_d == "schur":
            self.schur = [self._schur_lu(s, f) for s, f in zip(self.systems, self.exact3)]
        spec = {"type": "none"} if strategy.three_d == "direct" else (strategy.three_d or {"type": "none"})
        kind = spec.get("type", "none")
        self.inner = None
        if kind == "exact":
            self.inner = _BatchedExact([ExactPreconditioner(host_reduced_operator(s)) for s in self.systems])
        elif kind == "neural":
            params = spec.get("params")
            if params is None:
                params = load_checkpoint(spec["checkpoint"])
            if not isinstance(params, UNetParams):
                raise TypeError("neural spec needs UNetParams")
            sm = spec.get("smoothing")
            smooth = (sm["maxit"], sm.get("omega", 2.0 / 3.0)) if isinstance(sm, dict) else sm
            dists = torch.stack([mesh_distance(s) for s in self.systems])
            self.inner = BatchedNeural(device_net(params, spec.get("path", path)), dists, p.n, p.ld, p.nsys,
                                       C=self.C, smoothing=smooth,
                                       zero_distance=spec.get("zero_distance", False))
        elif kind == "ilu0":  # the 3D ILU(0) baseline: one factor of C per system
            self.inner = _BatchedIlu(self.systems, p.ld)
        elif kind == "gmg":  # the multigrid baseline: one Galerkin hierarchy per system
            levels = spec.get("levels", _default_levels(p.n))
            self.inner = _BatchedGmg([GmgPreconditioner(gmg_build(s.grid, host_reduced_operator(s), levels),
                                                        cycles=spec.get("cycles", 10)) for s in self.systems], p.n3)
        elif kind != "none":
            raise ValueError(f"inner preconditioner {kind!r} is not on the device hot path")
        self.outer = FgmresEngine(p.nsys, p.n3 + p.n1max, p.ld, strategy.restart)
        self.inner_eng = FgmresEngine(p.nsys, p.n3, p.ld, strategy.inner_iterations)
        self.fixed = FixedStepFgmres(p.nsys, p.n3, p.ld, strategy.inner_iterations)
        self.direct3 = strategy.three_d == "direct"
        if strategy.three_d != "direct":
            self.exact3 = None
        # the dense-factor solves (cuSOLVER via torch) run eagerly, outside CUDA graphs
        # the fixed-step device solve keeps y in a 64-entry shared array (mdp_fixed_finish):
        # longer inner solves take the host-driven FgmresEngine path
        self.graphs = graphs and self.schur is None and not self.direct3 and kind != "exact" \
            and strategy.inner_iterations <= 64
        self.b3 = p.zeros()
        self.F = p.pack([full_rhs(s) for s in self.systems])

    @staticmethod
    def _schur_lu(s, exact):
        """LU of S = A11 - (w M10) C^-1 (w M01), C^-1 by the dense device factor (harness.py:359-368)."""
        import torch
        w = s.params.coupling_weight
        dev = exact.L.device
        W01 = torch.as_tensor((w * s.M01).toarray(), device=dev)
        S = torch.as_tensor(one_d_operator(s).toarray(), device=dev) - \
            torch.as_tensor((w * s.M10).toarray(), device=dev) @ exact.solve_device(W01)
        return torch.linalg.lu_factor(S)

    def _block_precond(self, V, Z, sel, idx):
        import torch
        p = self.prob
        m = int(sel.numel())
        n3 = p.n3
        if self.schur is not None:  # z1 = S^-1 r1 (harness.py:368)
            for s in idx:
                n1 = self.systems[s].n1
                LU, piv = self.schur[s]
                Z[s, n3:n3 + n1] = torch.linalg.lu_solve(LU, piv, V[s, n3:n3 + n1, None])[:, 0]
        else:  # z1 = ILU(r1)   (krylov.py:270-276 via harness.py:390)
            _ext.check(self.lib.mdp_ilu0_apply(self.ilu.desc, m, sel.data_ptr(), V.data_ptr() + 8 * n3,
                                               Z.data_ptr() + 8 * n3, p.ld, _ext.stream()))
        # r0 - w M01 z1  (harness.py:391)
        _ext.check(self.lib.mdp_copy_vec(m, sel.data_ptr(), V.data_ptr(), p.ld, self.b3.data_ptr(), p.ld, None, 0,
                                         n3, _ext.stream()))
        self.cpl.minus_w_m01(Z, self.b3, sel)
        if self.direct3:  # z0 = C^-1 (r0 - w M01 z1)  (harness.py:373-375)
            for s in idx:
                Z[s, :n3] = self.exact3[s].solve_device(self.b3[s, :n3])
            return
        # z0 = 3-step inner FGMRES on C (harness.py:385-387)
        m_in = self.st.inner_iterations
        P = self.inner.apply_device if self.inner is not None else None
        self.inner_eng.solve(self.C.matvec, P, self.b3, tol=1e-300, maxit=m_in, systems=idx,
                             final_residual=False)
        _ext.check(self.lib.mdp_copy_vec(m, sel.data_ptr(), self.inner_eng.x.data_ptr(), p.ld, Z.data_ptr(), p.ld,
                                         None, 0, n3, _ext.stream()))

    def _block_precond_graph(self, V, Z, sel, idx, flag):
        """Graph-safe block preconditioner: same pieces, inner solve fully on device.

        Writes flag[i] != 0 for systems whose inner solve hit a breakdown or
        a zero right-hand side; the outer engine re-runs those through the
        exact ``_block_precond``.
        """
        p = self.prob
        m = int(sel.numel())
        n3 = p.n3
        _ext.check(self.lib.mdp_ilu0_apply(self.ilu.desc, m, sel.data_ptr(), V.data_ptr() + 8 * n3,
                                           Z.data_ptr() + 8 * n3, p.ld, _ext.stream()))
        self.cpl.minus_w_m01(Z, self.b3, sel, copy_from=V)  # b3 = r0 and += -w M01 z1: one gather launch + pull
        P = self.inner.apply_device if self.inner is not None else None
        pre = self.inner.first_sweep_spec() if self.inner is not None else None
        self.fixed.run(self.C.matvec, P, self.b3, sel, idx, out=Z, pre=pre)  # z0 written straight into Z[:, :n3]
        flag[:m].copy_(self.fixed.flag[:m])

    def solve(self, F=None):
        """Outer FGMRES (harness.py:394-395); returns per-system reports, x left on device."""
        st = self.st
        return self.outer.solve(self.A.matvec, self._block_precond, self.F if F is None else F,
                                tol=st.tol, maxit=st.maxit,
                                Pg=self._block_precond_graph if self.graphs else None)

    def solution(self):
        out = []
        X = self.prob.unpack(self.outer.x)
        for s, x in zip(self.systems, X):
            u3, u1 = x[:s.n3], x[s.n3:].copy()
            u1[list(s.dirichlet_nodes)] = 1.0  # harness.py:396-397
            out.append((u3, u1))
        return out


def solve_coupled(system, strategy: CoupledStrategy):
    """Drop-in ``harness.solve_coupled``: (u3d, u1d, SolveReport).

    A list of systems on one grid is solved concurrently and a list of
    triples is returned.
    """
    many = isinstance(system, (list, tuple))
    systems = list(system) if many else [system]
    solver = CoupledSolver(systems, strategy)
    reps = solver.solve()
    res = [(u3, u1, reps[i]) for i, (u3, u1) in enumerate(solver.solution())]
    return res if many else res[0]

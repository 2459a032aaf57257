"""Coupled 3D-1D problem build (host) and its device descriptor.

Host side mirrors ``mdprec.assembly`` (assembly.py:34-378): the same
PhysicalParams / CoupledSystem / assemble_coupled_system contract, with the
index sets (refined mesh, Pi rows, Psi, W, the 1D blocks and the Dirichlet
elimination) produced in the reference's operation order so patterns are
bit-identical (tests/test_host_build.py).  The 3D block K00 and M00 are
never assembled for the solve: the device applies K00 as a Kronecker
stencil and M00 as T^T W T through the Pi gather / pull kernels.

``DeviceProblem`` packs one or many systems that share the grid into the
``mdp_problem`` descriptor of include/mdp_b200.h (vectors [nsys][ld] with
ld >= n^3 + max n1, zero padded).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import os

import numpy as np
import scipy.sparse as sp

from .geometry import Graph1D, GraphMesh1D, StructuredGrid, refine_graph

GAUSS_1D = (0.5 - 0.5 / math.sqrt(3.0), 0.5 + 0.5 / math.sqrt(3.0))
# corner l = dx + 2 dy + 4 dz (assembly.py:54-65)
_CORNER = np.array([(l & 1, (l >> 1) & 1, (l >> 2) & 1) for l in range(8)], dtype=np.int64)


@dataclass(frozen=True)
class PhysicalParams:
    """Coefficients (assembly.py:34-51); ``beta`` overrides the coupling weight 2*pi*eps."""

    k_omega: float = 1e-3
    sigma_omega: float = 1e-3
    k_lambda: float = 1.0
    epsilon: float = 1e-3
    beta: float | None = None

    def __post_init__(self):
        for name in ("k_omega", "sigma_omega", "k_lambda", "epsilon"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be strictly positive")
        if self.beta is not None and self.beta <= 0:
            raise ValueError("beta must be strictly positive")

    @property
    def coupling_weight(self) -> float:
        return float(self.beta) if self.beta is not None else 2.0 * math.pi * self.epsilon


def trilinear_eval_matrix(grid: StructuredGrid, points: np.ndarray) -> sp.csr_matrix:
    """Q1 basis at points: 8 weights of the containing cell (assembly.py:160-183)."""
    points = np.atleast_2d(points)
    bad = np.any((points < -1e-12) | (points > 1 + 1e-12), axis=1)
    if np.any(bad):
        raise ValueError(f"evaluation point {points[bad][0]} outside the unit cube")
    n = grid.n
    u = np.clip(points, 0.0, 1.0) / grid.h
    cell = np.minimum(u.astype(np.int64), n - 2)
    frac = u - cell
    stride = np.array([1, n, n * n], dtype=np.int64)
    cols = (cell @ stride)[:, None] + (_CORNER @ stride)[None, :]
    w = np.ones((len(points), 8))
    for ax in range(3):
        f = frac[:, ax][:, None]
        w *= np.where(_CORNER[:, ax][None, :] == 1, f, 1.0 - f)
    return sp.csr_matrix((w.ravel(), (np.repeat(np.arange(len(points)), 8), cols.ravel())),
                         shape=(len(points), grid.num_nodes))


@dataclass(frozen=True)
class RestrictionMap:
    """Pi = T (Q x N3), Psi (Q x N1), Gauss weights W, quadrature points (assembly.py:186-198)."""

    matrix: sp.csr_matrix
    basis_1d: sp.csr_matrix
    weights: np.ndarray
    points: np.ndarray


def build_restriction(grid: StructuredGrid, mesh: GraphMesh1D, n_circle: int = 1,
                      radius: float = 0.0) -> RestrictionMap:
    """2-point Gauss rows 2e, 2e+1; centreline or circle-averaged T (assembly.py:201-249)."""
    if n_circle < 1:
        raise ValueError("n_circle must be at least 1")
    ea = mesh.coords[mesh.elements[:, 0]]
    eb = mesh.coords[mesh.elements[:, 1]]
    q = 2 * len(mesh.elements)
    pts = np.empty((q, 3))
    wts = np.empty(q)
    phi = np.empty((q, 2))
    for g, t in enumerate(GAUSS_1D):
        pts[g::2] = ea + t * (eb - ea)
        wts[g::2] = mesh.element_lengths / 2.0
        phi[g::2, 0] = 1.0 - t
        phi[g::2, 1] = t
    if n_circle == 1:
        T = trilinear_eval_matrix(grid, pts)
    else:
        d = eb - ea
        d = d / np.linalg.norm(d, axis=1, keepdims=True)
        tan = np.repeat(d, 2, axis=0)
        e1 = np.cross(tan, np.eye(3)[np.argmin(np.abs(tan), axis=1)])
        e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
        e2 = np.cross(tan, e1)
        # sparse sums drop exact zeros, so the pattern is value dependent:
        # accumulate in the reference's order with scipy's own addition
        T = sp.csr_matrix((q, grid.num_nodes))
        for c in range(n_circle):
            th = 2 * math.pi * c / n_circle
            T = T + trilinear_eval_matrix(grid, pts + radius * (math.cos(th) * e1 + math.sin(th) * e2))
        T = (T / n_circle).tocsr()
    cols = np.repeat(mesh.elements, 2, axis=0)
    psi = sp.csr_matrix((phi.ravel(), (np.repeat(np.arange(q), 2), cols.ravel())),
                        shape=(q, mesh.num_nodes))
    return RestrictionMap(T.tocsr(), psi, wts, pts)


def stiffness_1d(mesh: GraphMesh1D) -> sp.csr_matrix:
    """P1 stiffness on the graph mesh (assembly.py:252-260)."""
    e = mesh.elements
    k = 1.0 / mesh.element_lengths
    r = np.concatenate([e[:, 0], e[:, 1], e[:, 0], e[:, 1]])
    c = np.concatenate([e[:, 0], e[:, 1], e[:, 1], e[:, 0]])
    return sp.coo_matrix((np.concatenate([k, k, -k, -k]), (r, c)),
                         shape=(mesh.num_nodes, mesh.num_nodes)).tocsr()


def _without(A, rows, cols) -> sp.coo_matrix:
    """Drop entries in the given rows / columns (symmetric elimination, assembly.py:295-303)."""
    A = A.tocoo()
    keep = np.ones(A.nnz, dtype=bool)
    if len(rows):
        keep &= ~np.isin(A.row, rows)
    if len(cols):
        keep &= ~np.isin(A.col, cols)
    return sp.coo_matrix((A.data[keep], (A.row[keep], A.col[keep])), shape=A.shape)


def _unit_diag(A, idx) -> sp.csr_matrix:
    return (A + sp.coo_matrix((np.ones(len(idx)), (idx, idx)), shape=A.shape)).tocsr()


def cube_boundary_mask(n: int) -> np.ndarray:
    i = np.arange(n)
    on = (i == 0) | (i == n - 1)
    return (on[:, None, None] | on[None, :, None] | on[None, None, :]).ravel()


@dataclass(frozen=True)
class CoupledSystem:
    """Blocks after Dirichlet elimination (assembly.py:263-292).

    K00 / M00 / M10 are assembled lazily on the host only when asked for
    (parity export); the solve never needs them.
    """

    grid: StructuredGrid
    graph_mesh: GraphMesh1D
    params: PhysicalParams
    K11: sp.csr_matrix
    M01: sp.csr_matrix
    M11: sp.csr_matrix
    rhs0: np.ndarray
    rhs1: np.ndarray
    dirichlet_nodes: tuple
    restriction: RestrictionMap
    bc3d: str = "neumann"
    _cache: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def n3(self) -> int:
        return self.grid.num_nodes

    @property
    def n1(self) -> int:
        return self.K11.shape[0]

    @property
    def boundary_nodes(self) -> np.ndarray:
        if self.bc3d != "dirichlet":
            return np.zeros(0, dtype=np.int64)
        return np.nonzero(cube_boundary_mask(self.grid.n))[0]

    @property
    def K00(self) -> sp.csr_matrix:
        if "K00" not in self._cache:
            K = assemble_3d(self.grid, self.params)
            B = self.boundary_nodes
            if len(B):
                K = _unit_diag(_without(K, B, B), B)
            self._cache["K00"] = K
        return self._cache["K00"]

    @property
    def M00(self) -> sp.csr_matrix:
        if "M00" not in self._cache:
            T = self.restriction.matrix
            M = (T.T @ sp.diags(self.restriction.weights) @ T).tocsr()
            B = self.boundary_nodes
            if len(B):
                M = _without(M, B, B).tocsr()
            self._cache["M00"] = M
        return self._cache["M00"]

    @property
    def M10(self) -> sp.csr_matrix:
        return self.M01.T.tocsr()


def q1_element_matrices(h: float):
    """Exact Q1 cell stiffness / mass via the 2x2x2 Gauss rule (assembly.py:83-90)."""
    gp = np.array([(a, b, c) for c in GAUSS_1D for b in GAUSS_1D for a in GAUSS_1D])
    val = np.empty((8, 8))
    grad = np.empty((8, 8, 3))
    for g, xi in enumerate(gp):
        for l, c in enumerate(_CORNER):
            f = np.where(c == 1, xi, 1.0 - xi)
            s = np.where(c == 1, 1.0, -1.0)
            val[g, l] = f.prod()
            for ax in range(3):
                grad[g, l, ax] = s[ax] * f[(ax + 1) % 3] * f[(ax + 2) % 3]
    vol = h ** 3 / 8.0
    mass = vol * (val.T @ val)
    stiff = np.zeros((8, 8))
    for g in range(8):
        stiff += vol / h ** 2 * (grad[g] @ grad[g].T)
    return stiff, mass


def assemble_3d(grid: StructuredGrid, params: PhysicalParams) -> sp.csr_matrix:
    """Host CSR of K00 (assembly.py:102-125); only for parity export at small n."""
    stiff, mass = q1_element_matrices(grid.h)
    n = grid.n
    c = np.arange(n - 1)
    ck, cj, ci = np.meshgrid(c, c, c, indexing="ij")
    base = (ci + cj * n + ck * n * n).ravel()
    nodes = base[:, None] + (_CORNER @ np.array([1, n, n * n]))[None, :]
    r = np.repeat(nodes, 8, axis=1).ravel()
    cc = np.tile(nodes, (1, 8)).ravel()

    def scatter(elem):
        return sp.coo_matrix((np.tile(elem.ravel(), len(base)), (r, cc)),
                             shape=(grid.num_nodes,) * 2).tocsr()

    return (params.k_omega * scatter(stiff) + params.sigma_omega * scatter(mass)).tocsr()


def assemble_coupled_system(grid: StructuredGrid, graph: Graph1D, params: PhysicalParams,
                            n_circle: int = 1, *, elems_per_edge: int | None = None,
                            bc3d: str = "neumann", f1d: float = 0.0,
                            check_radius: bool = True) -> CoupledSystem:
    """Assemble one coupled problem (assembly.py:306-348).

    Keyword extensions (defaults = reference):
    ``elems_per_edge`` fixed P1 elements per graph edge (A5); ``bc3d``
    'neumann' | 'dirichlet' (homogeneous, symmetric elimination, A2);
    ``f1d`` nodal 1D load f1d * Psi^T W 1 on free rows (A7);
    ``check_radius=False`` lifts the eps <= h check (A4, config 4).
    """
    if graph.radius != params.epsilon:
        raise ValueError("graph radius and params.epsilon must agree")
    if check_radius and params.epsilon > grid.h:
        raise ValueError(f"coupling radius {params.epsilon} exceeds grid spacing {grid.h}")
    if bc3d not in ("neumann", "dirichlet"):
        raise ValueError(f"unknown bc3d {bc3d!r}")
    mesh = refine_graph(graph, grid.h, elems_per_edge)
    rest = build_restriction(grid, mesh, n_circle, radius=params.epsilon)
    w = params.coupling_weight
    T, psi, W = rest.matrix, rest.basis_1d, sp.diags(rest.weights)
    K11r = (params.k_lambda * (math.pi * params.epsilon ** 2)) * stiffness_1d(mesh)
    M01r = (-(T.T @ W @ psi)).tocsr()
    M11r = (psi.T @ W @ psi).tocsr()
    D = np.array(mesh.dirichlet_nodes, dtype=np.int64)
    one = np.ones(len(D))
    rhs1 = -np.asarray((K11r + w * M11r).tocsc()[:, D] @ one).ravel()
    rhs0 = -w * np.asarray(M01r.tocsc()[:, D] @ one).ravel()
    if f1d:
        rhs1 = rhs1 + f1d * np.asarray(psi.T @ rest.weights).ravel()
    rhs1[D] = 1.0
    K11 = _unit_diag(_without(K11r, D, D), D)
    M11 = _without(M11r, D, D).tocsr()
    if bc3d == "dirichlet":
        B = np.nonzero(cube_boundary_mask(grid.n))[0]
        M01 = _without(M01r, B, D).tocsr()
        rhs0 = rhs0.copy()
        rhs0[B] = 0.0
    else:
        M01 = _without(M01r, [], D).tocsr()
    return CoupledSystem(grid, mesh, params, K11, M01, M11, rhs0, rhs1,
                         tuple(int(d) for d in D), rest, bc3d)


def reduced_rhs(system: CoupledSystem, z1: np.ndarray) -> np.ndarray:
    """-w M01 z1 (assembly.py:356-362)."""
    z1 = np.asarray(z1, dtype=float)
    if z1.shape != (system.n1,):
        raise ValueError(f"expected a vector of length {system.n1}, got shape {z1.shape}")
    return -system.params.coupling_weight * (system.M01 @ z1)


def one_d_operator(system: CoupledSystem) -> sp.csr_matrix:
    """A11 = K11 + w M11 (assembly.py:365-367), host CSR (ILU(0) input)."""
    return (system.K11 + system.params.coupling_weight * system.M11).tocsr()


def full_rhs(system: CoupledSystem) -> np.ndarray:
    return np.concatenate([system.rhs0, system.rhs1])


def full_operator(system: CoupledSystem):
    """Device block operator, drop-in for assembly.full_operator (assembly.py:370-374)."""
    from .operators import CoupledOperator
    return CoupledOperator(DeviceProblem([system]))


def reduced_operator(system: CoupledSystem):
    """Device C = K00 + w M00, drop-in for assembly.reduced_operator (assembly.py:351-353)."""
    from .operators import ReducedOperator
    return ReducedOperator(DeviceProblem([system]))


def host_full_operator(system: CoupledSystem) -> sp.csr_matrix:
    """Assembled host CSR (parity export only; O(n^3) memory)."""
    w = system.params.coupling_weight
    return sp.bmat([[system.K00 + w * system.M00, w * system.M01],
                    [w * system.M10, system.K11 + w * system.M11]], format="csr")


def host_reduced_operator(system: CoupledSystem) -> sp.csr_matrix:
    """Assembled host CSR of C = K00 + w M00 (assembly.py:351-353; O(n^3) memory: the
    geometric-multigrid baseline's Galerkin hierarchy starts from it)."""
    return (system.K00 + system.params.coupling_weight * system.M00).tocsr()


def diag_k00(grid, params, bc3d: str) -> np.ndarray:
    """diag(K00) from the Kronecker factors (no assembly); eliminated cube nodes carry 1."""
    n, h = grid.n, grid.h
    idx = np.arange(n)
    end = (idx == 0) | (idx == n - 1)
    k1 = np.where(end, 1.0 / h, 2.0 / h)
    m1 = np.where(end, 2.0 * h / 6.0, 4.0 * h / 6.0)
    kz, ky, kx = np.meshgrid(k1, k1, k1, indexing="ij")
    mz, my, mx = np.meshgrid(m1, m1, m1, indexing="ij")
    d = (params.k_omega * (mz * my * kx + mz * ky * mx + kz * my * mx) + params.sigma_omega * (mz * my * mx)).ravel()
    if bc3d == "dirichlet":
        d[cube_boundary_mask(n)] = 1.0
    return d


def _by_node(T) -> tuple:
    """Stored entries of T grouped by 3D node, quadrature rows ascending within a node (the order of
    T.T.tocsr()), without any O(N3) work: (touched nodes, group starts, group sizes, entry order, rows)."""
    T = T.tocsr()
    T.sort_indices()
    rows = np.repeat(np.arange(T.shape[0]), np.diff(T.indptr))
    order = np.argsort(T.indices, kind="stable")
    nodes, start, cnt = np.unique(T.indices[order], return_index=True, return_counts=True)
    return nodes.astype(np.int64), start, cnt, order, rows, T


def diag_m00(system: CoupledSystem, by_node=None) -> tuple:
    """Nonzeros of w diag(M00) = w (T o T)^T W: (free node ids, values); per node the terms are summed
    in ascending quadrature order, as the sparse product does."""
    nodes, start, cnt, order, rows, T = by_node or _by_node(system.restriction.matrix)
    terms = (T.data[order] * T.data[order]) * system.restriction.weights[rows[order]]
    v = system.params.coupling_weight * np.bincount(np.repeat(np.arange(len(nodes)), cnt), weights=terms,
                                                     minlength=len(nodes))
    keep = v != 0.0
    if system.bc3d == "dirichlet":
        keep &= ~cube_boundary_mask(system.grid.n)[nodes]
    return nodes[keep], v[keep]


def diag_reduced(system: CoupledSystem) -> np.ndarray:
    """diag(C) = diag(K00) + w diag(M00) without assembling K00 (Kronecker diagonal)."""
    d = diag_k00(system.grid, system.params, system.bc3d)
    nodes, vals = diag_m00(system)
    d[nodes] = d[nodes] + vals
    return d


def _ranges(starts, counts):
    """Concatenated index ranges [starts[i], starts[i] + counts[i])."""
    starts = np.asarray(starts, dtype=np.int64)
    counts = np.asarray(counts, dtype=np.int64)
    if counts.sum() == 0:
        return np.zeros(0, dtype=np.int64)
    off = np.repeat(starts - np.concatenate([[0], np.cumsum(counts)[:-1]]), counts)
    return off + np.arange(int(counts.sum()))


class DeviceProblem:
    """Batched device descriptor of systems sharing one grid (``mdp_problem``)."""

    def __init__(self, systems, device=None):
        import torch
        from . import _ext
        systems = list(systems)
        if not systems:
            raise ValueError("need at least one system")
        n = systems[0].grid.n
        if any(s.grid.n != n for s in systems):
            raise ValueError("batched systems must share the grid")
        bcs = {s.bc3d for s in systems}
        if len(bcs) != 1:
            raise ValueError("batched systems must share the 3D boundary condition")
        p0 = systems[0].params
        if any((s.params.k_omega, s.params.sigma_omega) != (p0.k_omega, p0.sigma_omega) for s in systems):
            raise ValueError("batched systems must share k_omega and sigma_omega")
        self.systems = systems
        self.nsys = len(systems)
        self.n = n
        self.n3 = n ** 3
        self.n1 = np.array([s.n1 for s in systems], dtype=np.int32)
        self.n1max = int(self.n1.max())
        self.ld = (self.n3 + self.n1max + 31) // 32 * 32
        self.device = torch.device(device or "cuda")
        dev = self.device
        bmask = cube_boundary_mask(n) if bcs == {"dirichlet"} else None

        q_start, t_ptr, t_col, t_val, psi_col, psi_val, wq = [0], [0], [], [], [], [], []
        u_start, u_node, u_ptr, u_q, u_val = [0], [], [0], [], []
        r1_start, k_ptr, k_col, k_val, p_ptr, p_q, p_val = [0], [0], [], [], [0], [], []
        # diag(C) per system = the shared diag(K00) (one upload for the whole batch) + w diag(M00) at the
        # touched nodes; assembled on the device: at 129^3 x 64 the per-system host diagonals and their
        # 1.1 GB upload were most of the set-up time
        dnodes, dvals, dsys = [], [], []
        for si, s in enumerate(systems):
            T = s.restriction.matrix.tocsr()
            T.sort_indices()
            q0 = q_start[-1]
            Q = T.shape[0]
            Tg = T
            if bmask is not None:
                # eliminated cube nodes carry no value in the gather (M00 columns dropped)
                keep = ~bmask[T.indices]
                rows = np.repeat(np.arange(Q), np.diff(T.indptr))[keep]
                Tg = sp.csr_matrix((T.data[keep], (rows, T.indices[keep])), shape=T.shape)
                Tg.sort_indices()
            t_ptr.extend((Tg.indptr[1:] + t_ptr[-1]).tolist())
            t_col.append(Tg.indices.astype(np.int32))
            t_val.append(Tg.data)
            psi = s.restriction.basis_1d.tocsr()
            psi.sort_indices()
            if np.any(np.diff(psi.indptr) != 2):
                raise ValueError("Psi rows must hold exactly two entries")
            pc = psi.indices.astype(np.int32).copy()
            dset = np.array(s.dirichlet_nodes, dtype=np.int64)
            pc[np.isin(pc, dset)] = -1
            psi_col.append(pc)
            psi_val.append(psi.data)
            wq.append(s.restriction.weights)
            q_start.append(q0 + Q)
            # pull rows: T^T over touched free nodes (entries grouped by node, no O(N3) pass)
            bn = _by_node(T)
            nz, st_u, cnt_u, order_u, rows_u, Ts = bn
            if bmask is not None:
                free = ~bmask[nz]
                nz, st_u, cnt_u = nz[free], st_u[free], cnt_u[free]
            src = order_u[_ranges(st_u, cnt_u)]
            u_q.append(rows_u[src].astype(np.int32) + q0)
            u_val.append(Ts.data[src])
            u_ptr.extend((u_ptr[-1] + np.cumsum(cnt_u)).tolist())
            u_node.append(nz.astype(np.int32))
            u_start.append(u_start[-1] + len(nz))
            # 1D rows
            K = s.K11.tocsr()
            K.sort_indices()
            k_ptr.extend((K.indptr[1:] + k_ptr[-1]).tolist())
            k_col.append(K.indices.astype(np.int32))
            k_val.append(K.data)
            PT = psi.T.tocsr()
            PT.sort_indices()
            # Psi^T rows of the free 1D nodes (Dirichlet rows stay empty), in row order
            cnt_p = np.diff(PT.indptr)
            cnt_p[np.asarray(s.dirichlet_nodes, dtype=np.int64)] = 0
            src_p = _ranges(PT.indptr[:-1], cnt_p)
            p_q.append(PT.indices[src_p].astype(np.int32) + q0)
            p_val.append(PT.data[src_p])
            p_ptr.extend((p_ptr[-1] + np.cumsum(cnt_p)).tolist())
            r1_start.append(r1_start[-1] + s.n1)
            nd, vd = diag_m00(s, bn)
            dnodes.append(nd + si * self.ld)
            dvals.append(vd)

        def i32(x):
            x = np.concatenate(x) if isinstance(x, list) and x and isinstance(x[0], np.ndarray) else np.asarray(x)
            return torch.as_tensor(np.asarray(x, dtype=np.int32).ravel(), device=dev)

        def f64(x):
            x = np.concatenate(x) if isinstance(x, list) and x and isinstance(x[0], np.ndarray) else np.asarray(x)
            return torch.as_tensor(np.asarray(x, dtype=np.float64).ravel(), device=dev)

        # ELL copy of the pull list (width = widest touched node, a multiple of 8 lanes);
        # padding entries carry value 0 and the row's first quadrature index
        up = np.asarray(u_ptr, dtype=np.int64)
        uq = np.concatenate(u_q) if u_q else np.zeros(0, dtype=np.int32)
        uv = np.concatenate(u_val) if u_val else np.zeros(0)
        cnt = np.diff(up)
        # width: the widest multiple of 8 whose padded table stays within 2x the list itself (ring-averaged
        # Pi at 129^3: 5.4 entries per touched node on average but up to 44, so a full-width table would
        # move 9x the bytes); wider rows continue in the CSR list (same per-lane summation order)
        ell_w = 8
        if len(cnt):
            wmax = -(-int(cnt.max()) // 8) * 8
            while ell_w + 8 <= wmax and len(cnt) * (ell_w + 8) <= 2 * int(cnt.sum()):
                ell_w += 8
        nu = len(cnt)
        ell_q = np.zeros((max(nu, 1), ell_w), dtype=np.int32)
        ell_v = np.zeros((max(nu, 1), ell_w))
        if nu:
            pos = np.arange(len(uq)) - np.repeat(up[:-1], cnt)
            row = np.repeat(np.arange(nu), cnt)
            ell_q[:] = uq[up[:-1]][:, None]
            head = pos < ell_w
            ell_q[row[head], pos[head]] = uq[head]
            ell_v[row[head], pos[head]] = uv[head]
        self._t = dict(
            wc=f64([s.params.coupling_weight for s in systems]), n1=i32(self.n1),
            q_start=i32(q_start), t_ptr=i32(t_ptr), t_col=i32(t_col), t_val=f64(t_val),
            psi_col=i32(psi_col), psi_val=f64(psi_val), wq=f64(wq),
            u_start=i32(u_start), u_node=i32(u_node if u_node else [np.zeros(0)]), u_ptr=i32(u_ptr),
            u_q=i32(u_q if u_q else [np.zeros(0)]), u_val=f64(u_val if u_val else [np.zeros(0)]),
            r1_start=i32(r1_start), k_ptr=i32(k_ptr), k_col=i32(k_col), k_val=f64(k_val),
            p_ptr=i32(p_ptr), p_q=i32(p_q if p_q else [np.zeros(0)]),
            p_val=f64(p_val if p_val else [np.zeros(0)]),
            diag_c=self._device_diag(systems[0], bcs, dnodes, dvals, dev),
            ell_q=i32(ell_q), ell_val=f64(ell_v),
        )
        self.Qtot = int(q_start[-1])
        P = _ext.MdpProblem()
        P.n, P.nsys, P.bc3d, P.ld = n, self.nsys, 1 if bmask is not None else 0, self.ld
        P.h, P.k_omega, P.sigma_omega = systems[0].grid.h, p0.k_omega, p0.sigma_omega
        for k, t in self._t.items():
            setattr(P, k, t.data_ptr() if t.numel() else None)
        P.qmax = int(np.max(np.diff(q_start)))
        P.umax = int(np.max(np.diff(u_start))) if len(u_start) > 1 else 0
        P.r1max = int(self.n1.max())
        P.ell_w = ell_w
        if os.environ.get("MDP_NO_ELL"):  # A/B only: the CSR pull
            P.ell_q, P.ell_val = None, None

        self.desc = P
        self.s_work = torch.zeros(max(1, self.Qtot), dtype=torch.float64, device=dev)
        self.ilu = None

    def _device_diag(self, s0, bcs, dnodes, dvals, dev):
        import torch
        base = torch.ones(self.ld, dtype=torch.float64, device=dev)
        base[:self.n3] = torch.as_tensor(diag_k00(s0.grid, s0.params, "dirichlet" if bcs == {"dirichlet"} else "neumann"),
                                         device=dev)
        D = base.repeat(self.nsys, 1)
        if dnodes and sum(len(x) for x in dnodes):
            idx = torch.as_tensor(np.concatenate(dnodes), device=dev)
            val = torch.as_tensor(np.concatenate(dvals), device=dev)
            flat = D.view(-1)
            flat[idx] = flat[idx] + val  # each touched node appears once per system: plain gather / add / put
        return D

    # -- host <-> device vector layout -------------------------------------------------
    def zeros(self):
        import torch
        return torch.zeros((self.nsys, self.ld), dtype=torch.float64, device=self.device)

    def pack(self, vectors) -> "object":
        """List of host vectors (n3 + n1_s) -> device (nsys, ld)."""
        import torch
        host = np.zeros((self.nsys, self.ld))
        for i, v in enumerate(vectors):
            v = np.asarray(v, dtype=float)
            host[i, :len(v)] = v
        return torch.as_tensor(host, device=self.device)

    def unpack(self, X) -> list:
        Xh = X.detach().cpu().numpy()
        return [Xh[i, :self.n3 + int(self.n1[i])].copy() for i in range(self.nsys)]

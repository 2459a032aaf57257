"""Oracle problem build: grid, graph, refinement, Q1/P1 blocks, coupling.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates ``mdprec.geometry`` / ``mdprec.assembly`` with scipy.sparse in the
same operation order, so the CSR index sets come out bit-identical to the
reference (pinned by ``tests/test_oracle_golden.py``).  Extensions for the
BASELINE.json configs are keyword flags whose
defaults reproduce the reference exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

GAUSS_1D = (0.5 - 0.5 / math.sqrt(3.0), 0.5 + 0.5 / math.sqrt(3.0))


# ---------------------------------------------------------------------------
# geometry (reference: geometry.py)

@dataclass(frozen=True)
class StructuredGrid:
    """``n`` points per edge of the unit cube (geometry.py:27-49)."""

    n: int

    @property
    def h(self) -> float:
        return 1.0 / (self.n - 1)

    @property
    def num_nodes(self) -> int:
        return self.n ** 3

    def node_coords(self) -> np.ndarray:
        # lexicographic i + j n + k n^2, x fastest (geometry.py:45-49)
        r = np.arange(self.n) * self.h
        kk, jj, ii = np.meshgrid(r, r, r, indexing="ij")
        return np.column_stack([ii.ravel(), jj.ravel(), kk.ravel()])


@dataclass(frozen=True)
class Graph:
    """Embedded 1D graph (geometry.py:85-112, validation omitted)."""

    vertices: np.ndarray
    edges: np.ndarray
    radius: float
    dirichlet_vertices: tuple

    @property
    def edge_lengths(self) -> np.ndarray:
        a = self.vertices[self.edges[:, 0]]
        b = self.vertices[self.edges[:, 1]]
        return np.linalg.norm(b - a, axis=1)


@dataclass(frozen=True)
class GraphMesh:
    """Refined 1D mesh (geometry.py:234-249)."""

    coords: np.ndarray
    elements: np.ndarray
    element_lengths: np.ndarray
    dirichlet_nodes: tuple

    @property
    def num_nodes(self) -> int:
        return len(self.coords)


def segment_graph(a, b, radius: float) -> Graph:
    """Single straight segment, Dirichlet at vertex 0 (tests/test_assembly.py:37-39)."""
    return Graph(np.array([a, b], dtype=float), np.array([[0, 1]], dtype=np.int64),
                 float(radius), (0,))


def random_tree(n_segments: int, seed: int, radius: float) -> Graph:
    """BASELINE.json seeded random tree.

    Root uniform in [0.2,0.8]^3; each segment starts at a uniformly chosen
    existing vertex, isotropic direction, length U[0.1,0.3], end clipped to
    [0.05,0.95]^3; redraw direction+length if the clipped end collapses.
    """
    rng = np.random.default_rng(seed)
    verts = [rng.uniform(0.2, 0.8, 3)]
    edges = []
    for _ in range(n_segments):
        parent = int(rng.integers(0, len(verts)))
        while True:
            d = rng.standard_normal(3)
            d = d / np.linalg.norm(d)
            length = rng.uniform(0.1, 0.3)
            q = np.clip(verts[parent] + length * d, 0.05, 0.95)
            if np.linalg.norm(q - verts[parent]) >= 1e-9:
                break
        verts.append(q)
        edges.append((parent, len(verts) - 1))
    return Graph(np.array(verts), np.array(edges, dtype=np.int64), float(radius), (0,))


def refine_graph(graph: Graph, h_target: float, elems_per_edge: int | None = None) -> GraphMesh:
    """Vertices first, then interior nodes per edge in edge order (geometry.py:252-277).

    ``elems_per_edge`` fixes m per edge (Appendix A5); ``None`` keeps the
    reference rule m = max(1, ceil(L / h)).
    """
    blocks = [graph.vertices]
    elems, lens = [], []
    nxt = len(graph.vertices)
    for (a, b), length in zip(graph.edges, graph.edge_lengths):
        m = elems_per_edge if elems_per_edge else max(1, math.ceil(length / h_target))
        pa, pb = graph.vertices[a], graph.vertices[b]
        if m > 1:
            frac = np.arange(1, m)[:, None] / m
            blocks.append(pa + frac * (pb - pa))
        chain = [int(a)] + list(range(nxt, nxt + m - 1)) + [int(b)]
        nxt += m - 1
        for u, v in zip(chain[:-1], chain[1:]):
            elems.append((u, v))
            lens.append(length / m)
    return GraphMesh(np.vstack(blocks), np.array(elems, dtype=np.int64),
                     np.array(lens), tuple(graph.dirichlet_vertices))


def distance_field(vertices: np.ndarray, edges: np.ndarray, grid: StructuredGrid) -> np.ndarray:
    """Exact point-to-segment distance, min over edges (geometry.py:293-303)."""
    pts = grid.node_coords()
    d = np.full(len(pts), np.inf)
    for a, b in edges:
        pa = vertices[a]
        ab = vertices[b] - pa
        t = np.clip((pts - pa) @ ab / (ab @ ab), 0.0, 1.0)
        proj = pa + t[:, None] * ab
        np.minimum(d, np.linalg.norm(pts - proj, axis=1), out=d)
    return d


# ---------------------------------------------------------------------------
# 3D Q1 block (assembly.py:54-125)

def _q1_tables():
    # corner l = dx + 2 dy + 4 dz; Gauss points x fastest (assembly.py:54-77)
    corners = np.array([(l & 1, (l >> 1) & 1, (l >> 2) & 1) for l in range(8)])
    gauss = np.array([(gx, gy, gz) for gz in GAUSS_1D for gy in GAUSS_1D for gx in GAUSS_1D])
    vals = np.empty((8, 8))
    grads = np.empty((8, 8, 3))
    for g, xi in enumerate(gauss):
        for l, c in enumerate(corners):
            phi = np.where(c == 1, xi, 1.0 - xi)
            dphi = np.where(c == 1, 1.0, -1.0)
            vals[g, l] = phi.prod()
            for ax in range(3):
                grads[g, l, ax] = dphi[ax] * phi[(ax + 1) % 3] * phi[(ax + 2) % 3]
    return corners, vals, grads


CORNERS, _SHAPE_VALS, _SHAPE_GRADS = _q1_tables()


def q1_element_matrices(h: float):
    """Exact Q1 stiffness and mass of a cube of side h (assembly.py:83-90)."""
    w = h ** 3 / 8.0
    mass = w * (_SHAPE_VALS.T @ _SHAPE_VALS)
    stiff = np.zeros((8, 8))
    for g in range(8):
        stiff += w / h ** 2 * (_SHAPE_GRADS[g] @ _SHAPE_GRADS[g].T)
    return stiff, mass


def _scatter_element(grid: StructuredGrid, elem: np.ndarray) -> sp.csr_matrix:
    # cell bases x fastest, corner offsets, COO duplicates summed (assembly.py:93-109)
    n = grid.n
    c = np.arange(n - 1)
    ck, cj, ci = np.meshgrid(c, c, c, indexing="ij")
    base = (ci + cj * n + ck * n * n).ravel()
    off = CORNERS[:, 0] + CORNERS[:, 1] * n + CORNERS[:, 2] * n * n
    nodes = base[:, None] + off[None, :]
    rows = np.repeat(nodes, 8, axis=1).ravel()
    cols = np.tile(nodes, (1, 8)).ravel()
    data = np.tile(elem.ravel(), len(base))
    N = grid.num_nodes
    return sp.coo_matrix((data, (rows, cols)), shape=(N, N)).tocsr()


def assemble_3d(grid: StructuredGrid, k_omega: float, sigma_omega: float) -> sp.csr_matrix:
    """K00 = k_omega * stiffness + sigma_omega * mass (assembly.py:122-125)."""
    stiff, mass = q1_element_matrices(grid.h)
    return (k_omega * _scatter_element(grid, stiff)
            + sigma_omega * _scatter_element(grid, mass)).tocsr()


# ---------------------------------------------------------------------------
# restriction (assembly.py:160-249)

def trilinear_eval_matrix(grid: StructuredGrid, points: np.ndarray) -> sp.csr_matrix:
    """Rows of 8 trilinear weights, explicit zeros kept (assembly.py:160-183)."""
    points = np.atleast_2d(points)
    if np.any(points < -1e-12) or np.any(points > 1 + 1e-12):
        raise ValueError("evaluation point outside the unit cube")
    n, h = grid.n, grid.h
    scaled = np.clip(points, 0.0, 1.0) / h
    cell = np.minimum(scaled.astype(np.int64), n - 2)
    xi = scaled - cell
    base = cell[:, 0] + cell[:, 1] * n + cell[:, 2] * n * n
    off = CORNERS[:, 0] + CORNERS[:, 1] * n + CORNERS[:, 2] * n * n
    cols = base[:, None] + off[None, :]
    w = np.ones((len(points), 8))
    for ax in range(3):
        t = xi[:, ax][:, None]
        w *= np.where(CORNERS[:, ax][None, :] == 1, t, 1.0 - t)
    rows = np.repeat(np.arange(len(points)), 8)
    return sp.csr_matrix((w.ravel(), (rows, cols.ravel())), shape=(len(points), grid.num_nodes))


@dataclass(frozen=True)
class Restriction:
    matrix: sp.csr_matrix      # T: (Q, N3)
    basis_1d: sp.csr_matrix    # Psi: (Q, N1)
    weights: np.ndarray        # W: (Q,)
    points: np.ndarray


def build_restriction(grid: StructuredGrid, mesh: GraphMesh, n_circle: int = 1,
                      radius: float = 0.0) -> Restriction:
    """Two Gauss points per element, interleaved rows 2e, 2e+1 (assembly.py:201-249)."""
    a = mesh.coords[mesh.elements[:, 0]]
    b = mesh.coords[mesh.elements[:, 1]]
    ne = len(mesh.elements)
    pts = np.empty((2 * ne, 3))
    w = np.empty(2 * ne)
    v1 = np.empty((2 * ne, 2))
    for g, t in enumerate(GAUSS_1D):
        pts[g::2] = a + t * (b - a)
        w[g::2] = mesh.element_lengths / 2.0
        v1[g::2, 0] = 1.0 - t
        v1[g::2, 1] = t
    if n_circle == 1:
        T = trilinear_eval_matrix(grid, pts)
    else:
        tang = b - a
        tang = tang / np.linalg.norm(tang, axis=1, keepdims=True)
        tang2 = np.empty_like(pts)
        tang2[0::2] = tang
        tang2[1::2] = tang
        e1 = np.cross(tang2, np.eye(3)[np.argmin(np.abs(tang2), axis=1)])
        e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
        e2 = np.cross(tang2, e1)
        T = sp.csr_matrix((2 * ne, grid.num_nodes))
        for c in range(n_circle):
            theta = 2 * math.pi * c / n_circle
            ring = pts + radius * (math.cos(theta) * e1 + math.sin(theta) * e2)
            T = T + trilinear_eval_matrix(grid, ring)
        T = (T / n_circle).tocsr()
    rows = np.repeat(np.arange(2 * ne), 2)
    cols = np.empty((2 * ne, 2), dtype=np.int64)
    cols[0::2] = mesh.elements
    cols[1::2] = mesh.elements
    psi = sp.csr_matrix((v1.ravel(), (rows, cols.ravel())), shape=(2 * ne, mesh.num_nodes))
    return Restriction(T.tocsr(), psi, w, pts)


def stiffness_1d(mesh: GraphMesh) -> sp.csr_matrix:
    """Unweighted P1 stiffness on the graph mesh (assembly.py:252-260)."""
    n1 = mesh.num_nodes
    e = mesh.elements
    inv = 1.0 / mesh.element_lengths
    rows = np.concatenate([e[:, 0], e[:, 1], e[:, 0], e[:, 1]])
    cols = np.concatenate([e[:, 0], e[:, 1], e[:, 1], e[:, 0]])
    data = np.concatenate([inv, inv, -inv, -inv])
    return sp.coo_matrix((data, (rows, cols)), shape=(n1, n1)).tocsr()


# ---------------------------------------------------------------------------
# coupled system (assembly.py:34-51, 263-378)

@dataclass(frozen=True)
class PhysicalParams:
    """assembly.py:34-51 plus ``beta`` (Appendix A3): coupling weight override."""

    k_omega: float = 1e-3
    sigma_omega: float = 1e-3
    k_lambda: float = 1.0
    epsilon: float = 1e-3
    beta: float | None = None

    @property
    def coupling_weight(self) -> float:
        return float(self.beta) if self.beta is not None else 2.0 * math.pi * self.epsilon


@dataclass(frozen=True)
class CoupledSystem:
    grid: StructuredGrid
    mesh: GraphMesh
    params: PhysicalParams
    K00: sp.csr_matrix
    K11: sp.csr_matrix
    M00: sp.csr_matrix
    M01: sp.csr_matrix
    M10: sp.csr_matrix
    M11: sp.csr_matrix
    rhs0: np.ndarray
    rhs1: np.ndarray
    dirichlet_nodes: tuple
    restriction: Restriction
    boundary_nodes: np.ndarray   # 3D Dirichlet rows (empty for Neumann)

    @property
    def n3(self) -> int:
        return self.K00.shape[0]

    @property
    def n1(self) -> int:
        return self.K11.shape[0]


def _drop(A, rows, cols) -> sp.coo_matrix:
    # assembly.py:295-303
    coo = A.tocoo()
    keep = np.ones(len(coo.data), dtype=bool)
    if len(rows):
        keep &= ~np.isin(coo.row, rows)
    if len(cols):
        keep &= ~np.isin(coo.col, cols)
    return sp.coo_matrix((coo.data[keep], (coo.row[keep], coo.col[keep])), shape=A.shape)


def cube_boundary_nodes(grid: StructuredGrid) -> np.ndarray:
    n = grid.n
    i = np.arange(n)
    kk, jj, ii = np.meshgrid(i, i, i, indexing="ij")
    on = (ii == 0) | (ii == n - 1) | (jj == 0) | (jj == n - 1) | (kk == 0) | (kk == n - 1)
    return np.nonzero(on.ravel())[0].astype(np.int64)


def assemble_coupled_system(grid: StructuredGrid, graph: Graph, params: PhysicalParams,
                            n_circle: int = 1, elems_per_edge: int | None = None,
                            bc3d: str = "neumann", f1d: float = 0.0,
                            check_radius: bool = True) -> CoupledSystem:
    """Coupled blocks after Dirichlet elimination (assembly.py:306-348).

    Defaults reproduce the reference exactly.  Extensions (Appendix A):
    ``elems_per_edge`` (A5), ``bc3d='dirichlet'`` symmetric elimination of
    the cube boundary with homogeneous values (A2), ``f1d`` nodal 1D load
    f1d * Psi^T W 1 on free 1D rows (A7), ``check_radius=False`` (A4, cfg4).
    """
    if graph.radius != params.epsilon:
        raise ValueError("graph radius and params.epsilon must agree")
    if check_radius and params.epsilon > grid.h:
        raise ValueError(f"coupling radius {params.epsilon} exceeds grid spacing {grid.h}")
    mesh = refine_graph(graph, grid.h, elems_per_edge)
    rest = build_restriction(grid, mesh, n_circle, radius=params.epsilon)
    K00 = assemble_3d(grid, params.k_omega, params.sigma_omega)
    area = math.pi * params.epsilon ** 2
    K11_raw = (params.k_lambda * area) * stiffness_1d(mesh)
    W = sp.diags(rest.weights)
    T, psi = rest.matrix, rest.basis_1d
    M00 = (T.T @ W @ T).tocsr()
    M01_raw = (-(T.T @ W @ psi)).tocsr()
    M11_raw = (psi.T @ W @ psi).tocsr()

    D = np.array(mesh.dirichlet_nodes, dtype=np.int64)
    w = params.coupling_weight
    ones_d = np.ones(len(D))
    A11_raw = (K11_raw + w * M11_raw).tocsc()
    rhs1 = -np.asarray(A11_raw[:, D] @ ones_d).ravel()
    rhs0 = -w * np.asarray(M01_raw.tocsc()[:, D] @ ones_d).ravel()
    if f1d:
        load = f1d * np.asarray(psi.T @ rest.weights).ravel()
        rhs1 = rhs1 + load
    rhs1[D] = 1.0

    K11 = _drop(K11_raw, D, D)
    K11 = (K11 + sp.coo_matrix((np.ones(len(D)), (D, D)), shape=K11.shape)).tocsr()
    M11 = _drop(M11_raw, D, D).tocsr()

    if bc3d == "dirichlet":
        B = cube_boundary_nodes(grid)
        K00 = _drop(K00, B, B)
        K00 = (K00 + sp.coo_matrix((np.ones(len(B)), (B, B)), shape=K00.shape)).tocsr()
        M00 = _drop(M00, B, B).tocsr()
        M01 = _drop(M01_raw, B, D).tocsr()
        rhs0 = rhs0.copy()
        rhs0[B] = 0.0
    elif bc3d == "neumann":
        B = np.zeros(0, dtype=np.int64)
        M01 = _drop(M01_raw, [], D).tocsr()
    else:
        raise ValueError(f"unknown bc3d {bc3d!r}")
    M10 = M01.T.tocsr()
    return CoupledSystem(grid, mesh, params, K00, K11.tocsr(), M00, M01, M10, M11,
                         rhs0, rhs1, tuple(int(d) for d in D), rest, B)


def reduced_operator(s: CoupledSystem) -> sp.csr_matrix:
    """C = K00 + w M00 (assembly.py:351-353)."""
    return (s.K00 + s.params.coupling_weight * s.M00).tocsr()


def reduced_rhs(s: CoupledSystem, z1: np.ndarray) -> np.ndarray:
    """-w M01 z1 (assembly.py:356-362)."""
    z1 = np.asarray(z1, dtype=float)
    if z1.shape != (s.n1,):
        raise ValueError(f"expected a vector of length {s.n1}, got shape {z1.shape}")
    return -s.params.coupling_weight * (s.M01 @ z1)


def one_d_operator(s: CoupledSystem) -> sp.csr_matrix:
    """A11 = K11 + w M11 (assembly.py:365-367)."""
    return (s.K11 + s.params.coupling_weight * s.M11).tocsr()


def full_operator(s: CoupledSystem) -> sp.csr_matrix:
    """Block operator (assembly.py:370-374)."""
    w = s.params.coupling_weight
    return sp.bmat([[s.K00 + w * s.M00, w * s.M01],
                    [w * s.M10, s.K11 + w * s.M11]], format="csr")


def full_rhs(s: CoupledSystem) -> np.ndarray:
    return np.concatenate([s.rhs0, s.rhs1])

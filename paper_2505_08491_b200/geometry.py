"""Grid, embedded 1D graphs, refinement and distance fields.

Mirrors the public surface of ``mdprec.geometry`` that the hot path uses
(geometry.py:27-303): ``StructuredGrid``, ``Graph1D``, ``GraphMesh1D``,
``refine_graph``, ``DistanceField``/``distance_field``.  Node order is the
reference's lexicographic ``i + j*n + k*n**2`` and the refined-mesh order
(vertices first, then interior nodes per edge) is reproduced bit-exactly.

Additions for the BASELINE.json configs:
``refine_graph(..., elems_per_edge=m)`` (A5) and ``random_tree`` (A6).
``distance_field`` runs on the GPU (one thread per grid node, segments in
shared memory) because the O(N3 * E) CPU evaluation dominates setup at
129^3.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class StructuredGrid:
    """Uniform grid on the unit cube with ``n`` points per edge."""

    n: int

    def __post_init__(self):
        if self.n < 2:
            raise ValueError(f"grid needs at least 2 points per edge, got {self.n}")

    @property
    def h(self) -> float:
        return 1.0 / (self.n - 1)

    @property
    def num_nodes(self) -> int:
        return self.n ** 3

    def node_coords(self) -> np.ndarray:
        r = np.arange(self.n) * self.h
        kk, jj, ii = np.meshgrid(r, r, r, indexing="ij")
        return np.column_stack([ii.ravel(), jj.ravel(), kk.ravel()])


@dataclass(frozen=True)
class Graph1D:
    """1D metric graph in the closed unit cube (geometry.py:85-149)."""

    vertices: np.ndarray
    edges: np.ndarray
    radius: float
    dirichlet_vertices: tuple

    def __post_init__(self):
        object.__setattr__(self, "vertices", np.asarray(self.vertices, dtype=float))
        object.__setattr__(self, "edges", np.asarray(self.edges, dtype=np.int64))
        object.__setattr__(self, "dirichlet_vertices", tuple(int(d) for d in self.dirichlet_vertices))
        v, e = self.vertices, self.edges
        if v.ndim != 2 or v.shape[1] != 3:
            raise ValueError("vertices must have shape (V, 3)")
        if np.any(v < -1e-12) or np.any(v > 1 + 1e-12):
            raise ValueError("all vertices must lie in the closed unit cube")
        if e.ndim != 2 or e.shape[1] != 2:
            raise ValueError("edges must have shape (E, 2)")
        if np.any(e < 0) or np.any(e >= len(v)):
            raise ValueError("edge endpoint out of range")
        if np.any(self.edge_lengths <= 0):
            raise ValueError("every edge must have positive length")
        if self.radius <= 0:
            raise ValueError("radius must be positive")
        if len(self.dirichlet_vertices) == 0:
            raise ValueError("dirichlet_vertices must be non-empty")
        if any(not 0 <= d < len(v) for d in self.dirichlet_vertices):
            raise ValueError("dirichlet vertex out of range")

    @property
    def edge_lengths(self) -> np.ndarray:
        return np.linalg.norm(self.vertices[self.edges[:, 1]] - self.vertices[self.edges[:, 0]], axis=1)

    @property
    def total_length(self) -> float:
        return float(self.edge_lengths.sum())


@dataclass(frozen=True)
class GraphMesh1D:
    """P1 mesh of a graph (geometry.py:234-249)."""

    coords: np.ndarray
    elements: np.ndarray
    element_lengths: np.ndarray
    dirichlet_nodes: tuple

    @property
    def num_nodes(self) -> int:
        return len(self.coords)


def random_tree(n_segments: int, seed: int, radius: float) -> Graph1D:
    """Seeded random tree of BASELINE.json.

    rng = default_rng(seed); root ~ U[0.2,0.8]^3; per segment: parent ~
    U{existing vertices}, direction ~ isotropic, length ~ U[0.1,0.3], end
    clipped to [0.05,0.95]^3 (redrawn if it collapses onto the parent).
    Dirichlet vertex: the root.
    """
    rng = np.random.default_rng(seed)
    pts = [rng.uniform(0.2, 0.8, 3)]
    segs = []
    for _ in range(n_segments):
        parent = int(rng.integers(0, len(pts)))
        while True:
            u = rng.standard_normal(3)
            u = u / np.linalg.norm(u)
            end = np.clip(pts[parent] + rng.uniform(0.1, 0.3) * u, 0.05, 0.95)
            if np.linalg.norm(end - pts[parent]) >= 1e-9:
                break
        pts.append(end)
        segs.append((parent, len(pts) - 1))
    return Graph1D(np.array(pts), np.array(segs, dtype=np.int64), float(radius), (0,))


def refine_graph(graph: Graph1D, h_target: float, elems_per_edge: int | None = None) -> GraphMesh1D:
    """Subdivide edges: vertices first, interior nodes edge by edge (geometry.py:252-277).

    ``elems_per_edge=None`` keeps m = max(1, ceil(L/h)); an integer fixes m.
    """
    if h_target <= 0:
        raise ValueError("h_target must be positive")
    lengths = graph.edge_lengths
    counts = [elems_per_edge if elems_per_edge else max(1, math.ceil(L / h_target)) for L in lengths]
    nv = len(graph.vertices)
    parts = [graph.vertices]
    elem_rows, elem_len = [], []
    nxt = nv
    for (a, b), L, m in zip(graph.edges, lengths, counts):
        pa, pb = graph.vertices[a], graph.vertices[b]
        if m > 1:
            parts.append(pa + (np.arange(1, m)[:, None] / m) * (pb - pa))
        ids = np.concatenate([[a], np.arange(nxt, nxt + m - 1), [b]]).astype(np.int64)
        nxt += m - 1
        elem_rows.append(np.column_stack([ids[:-1], ids[1:]]))
        elem_len.append(np.full(m, L / m))
    return GraphMesh1D(np.vstack(parts), np.vstack(elem_rows), np.concatenate(elem_len),
                       tuple(graph.dirichlet_vertices))


@dataclass(frozen=True)
class DistanceField:
    """Per-node distance to the graph (geometry.py:280-290)."""

    grid: StructuredGrid
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "values", np.asarray(self.values, dtype=float))
        if self.values.shape != (self.grid.num_nodes,):
            raise ValueError("distance field length must equal the node count")


def distance_field_device(vertices: np.ndarray, edges: np.ndarray, grid: StructuredGrid):
    """Exact point-to-segment distance minimised over edges, on the GPU.

    Same formula as geometry.py:293-303 (t = clip((p-a).ab/ab.ab, 0, 1),
    |p - (a + t ab)|); returns a float64 CUDA tensor of length n^3.
    """
    import torch
    from . import _ext
    lib = _ext.lib()
    a = np.ascontiguousarray(vertices[edges[:, 0]], dtype=np.float64)
    b = np.ascontiguousarray(vertices[edges[:, 1]], dtype=np.float64)
    seg = torch.from_numpy(np.concatenate([a, b], axis=1).ravel()).cuda()
    out = torch.empty(grid.num_nodes, dtype=torch.float64, device="cuda")
    _ext.check(lib.mdp_distance_field(grid.n, _ext.ptr(seg), len(edges), _ext.ptr(out),
                                      _ext.stream()))
    return out


def distance_field(graph: Graph1D, grid: StructuredGrid) -> DistanceField:
    """Drop-in for geometry.distance_field (values on the host)."""
    return DistanceField(grid, distance_field_device(graph.vertices, graph.edges, grid).cpu().numpy())


# ---------------------------------------------------------------------------
# file formats (geometry.py:306-363): graph JSON and MDF1 grid vectors

_FIELD_MAGIC = b"MDF1"


def save_graph(graph: Graph1D, path) -> None:
    """Graph as JSON: vertices, edges, radius, dirichlet set (geometry.py:306-316)."""
    import json
    doc = {
        "vertices": [[float(x) for x in v] for v in graph.vertices],
        "edges": [[int(a), int(b)] for a, b in graph.edges],
        "radius": float(graph.radius),
        "dirichlet": [int(i) for i in graph.dirichlet_vertices],
    }
    with open(path, "w") as fh:
        json.dump(doc, fh)


def load_graph(path) -> Graph1D:
    """geometry.py:319-324."""
    import json
    with open(path) as fh:
        doc = json.load(fh)
    return Graph1D(np.array(doc["vertices"], dtype=float), np.array(doc["edges"], dtype=np.int64),
                   float(doc["radius"]), tuple(doc["dirichlet"]))


def write_grid_vector(path, n: int, values) -> None:
    """MDF1: magic, u32 n, n**3 little-endian f64 (geometry.py:330-338)."""
    import struct
    values = np.asarray(values, dtype="<f8").ravel()
    if values.size != n ** 3:
        raise ValueError(f"expected {n ** 3} values for n={n}, got {values.size}")
    with open(path, "wb") as fh:
        fh.write(_FIELD_MAGIC)
        fh.write(struct.pack("<I", n))
        fh.write(values.tobytes())


def read_grid_vector(path) -> tuple:
    """(n, values) of an MDF1 file; ValueError on a bad magic or truncation (geometry.py:341-353)."""
    import struct
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != _FIELD_MAGIC:
            raise ValueError(f"bad magic {magic!r}, expected {_FIELD_MAGIC!r}")
        (n,) = struct.unpack("<I", fh.read(4))
        data = fh.read()
    values = np.frombuffer(data, dtype="<f8")
    if values.size != n ** 3:
        raise ValueError("truncated grid-vector file")
    return int(n), values.astype(float)


def save_distance_field(dfield: DistanceField, path) -> None:
    write_grid_vector(path, dfield.grid.n, dfield.values)


def load_distance_field(path) -> DistanceField:
    n, values = read_grid_vector(path)
    return DistanceField(StructuredGrid(n), values)

"""Product host build (paper_2505_08491_b200.geometry/assembly) vs reference goldens.

Bit-exact: refined mesh, quadrature points, Pi/Psi/K11/M01/M11/A11 patterns
and values.  Also pins the BASELINE extensions against the oracle
restatement (Dirichlet cube, nodal load, relaxed radius).
"""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2505_08491_b200 import assembly as A
from paper_2505_08491_b200 import geometry as G
import oracle
from oracle import problem as OP
from conftest import golden


def product_case(name):
    g = golden(name)
    if name == "asm_n9_family":
        grid = G.StructuredGrid(9)
        graph = G.Graph1D(g["graph_vertices"], g["graph_edges"], 1e-3, tuple(int(d) for d in g["dirichlet"]))
        s = A.assemble_coupled_system(grid, graph, A.PhysicalParams())
    elif name.startswith("asm_cfg1"):
        grid = G.StructuredGrid(17)
        graph = G.Graph1D([[0.5, 0.5, 0.1], [0.5, 0.5, 0.9]], [[0, 1]], 0.02, (0,))
        s = A.assemble_coupled_system(grid, graph, A.PhysicalParams(epsilon=0.02, beta=1.0),
                                      n_circle=int(name[-1]), elems_per_edge=32)
    else:
        grid = G.StructuredGrid(33)
        graph = G.random_tree(8, 1, 0.015)
        assert np.array_equal(graph.vertices, g["tree_vertices"])
        s = A.assemble_coupled_system(grid, graph, A.PhysicalParams(epsilon=0.015, beta=1.0),
                                      n_circle=int(name[-1]), elems_per_edge=16)
    return g, s


def same_csr(M, g, prefix):
    M = sp.csr_matrix(M)
    assert np.array_equal(M.indptr, g[f"{prefix}_indptr"]), prefix
    assert np.array_equal(M.indices, g[f"{prefix}_indices"]), prefix
    assert np.array_equal(M.data, g[f"{prefix}_data"]), prefix


CASES = ["asm_n9_family", "asm_cfg1_nc1", "asm_cfg1_nc8", "asm_cfg2_nc1", "asm_cfg2_nc8"]


@pytest.mark.parametrize("name", CASES)
def test_index_sets_bit_exact(name):
    g, s = product_case(name)
    assert np.array_equal(s.graph_mesh.coords, g["mesh_coords"])
    assert np.array_equal(s.graph_mesh.elements, g["mesh_elements"])
    assert np.array_equal(s.graph_mesh.element_lengths, g["mesh_lengths"])
    r = s.restriction
    same_csr(r.matrix, g, "T")
    same_csr(r.basis_1d, g, "psi")
    assert np.array_equal(r.weights, g["wq"])
    assert np.array_equal(r.points, g["qpts"])
    for blk in ("K11", "M01", "M11", "M10"):
        same_csr(getattr(s, blk), g, blk)
    same_csr(A.one_d_operator(s), g, "A11")
    assert np.array_equal(s.rhs1, g["rhs1"])
    assert np.array_equal(s.rhs0, g["rhs0"])


@pytest.mark.parametrize("name", CASES)
def test_reduced_diagonal(name):
    g, s = product_case(name)
    assert np.allclose(A.diag_reduced(s), g["Cdiag"], rtol=1e-14, atol=0)


def test_small_host_operator_matches_reference():
    g, s = product_case("asm_n9_family")
    Ah = A.host_full_operator(s)
    assert np.allclose(Ah @ g["x"], g["Ax"], rtol=1e-13, atol=1e-16)


@pytest.mark.parametrize("bc3d,f1d,nc", [("dirichlet", 0.0, 8), ("dirichlet", 1.0, 8), ("neumann", 1.0, 1)])
def test_baseline_extensions_match_oracle(bc3d, f1d, nc):
    t = G.random_tree(4, 7, 0.02)
    s = A.assemble_coupled_system(G.StructuredGrid(17), t, A.PhysicalParams(epsilon=0.02, beta=0.7),
                                  n_circle=nc, elems_per_edge=8, bc3d=bc3d, f1d=f1d)
    ot = OP.random_tree(4, 7, 0.02)
    assert np.array_equal(ot.vertices, t.vertices)
    o = OP.assemble_coupled_system(OP.StructuredGrid(17), ot, OP.PhysicalParams(epsilon=0.02, beta=0.7),
                                   n_circle=nc, elems_per_edge=8, bc3d=bc3d, f1d=f1d)
    for blk in ("K11", "M01", "M11"):
        a, b = getattr(s, blk), getattr(o, blk)
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
        assert np.array_equal(a.data, b.data)
    assert np.array_equal(s.rhs0, o.rhs0) and np.array_equal(s.rhs1, o.rhs1)
    assert np.allclose(A.diag_reduced(s), OP.reduced_operator(o).diagonal(), rtol=1e-14, atol=0)
    # host CSR of the product vs oracle operator at this size
    x = np.random.default_rng(3).standard_normal(s.n3 + s.n1)
    assert np.allclose(A.host_full_operator(s) @ x, OP.full_operator(o) @ x, rtol=1e-13, atol=1e-15)


def test_relaxed_radius_check():
    t = G.random_tree(3, 3, 0.008)
    with pytest.raises(ValueError, match="exceeds"):
        A.assemble_coupled_system(G.StructuredGrid(129), t, A.PhysicalParams(epsilon=0.008))
    s = A.assemble_coupled_system(G.StructuredGrid(17), G.random_tree(3, 3, 0.008),
                                  A.PhysicalParams(epsilon=0.008), check_radius=False)
    assert s.n1 > 0


def test_refine_fixed_m_order():
    t = G.random_tree(5, 11, 0.01)
    m = G.refine_graph(t, 0.1, elems_per_edge=16)
    assert m.num_nodes == 6 + 5 * 15
    assert len(m.elements) == 80
    om = OP.refine_graph(OP.random_tree(5, 11, 0.01), 0.1, 16)
    assert np.array_equal(m.coords, om.coords) and np.array_equal(m.elements, om.elements)


def test_tree_elimination_order_is_fill_free():
    """Leaf-first order of a tree-structured A11: the ILU(0) factor of P A P^T is exact (L U == P A P^T)."""
    import scipy.sparse as sp
    from paper_2505_08491_b200 import assembly as A, geometry as G
    from paper_2505_08491_b200.krylov import direct_1d, tree_elimination_order
    s = A.assemble_coupled_system(G.StructuredGrid(17), G.random_tree(12, 7, 0.02),
                                  A.PhysicalParams(epsilon=0.02, beta=1.0), elems_per_edge=8)
    M = A.one_d_operator(s)
    f = direct_1d(M)
    F = sp.csr_matrix((f.data, f.indices, f.indptr), shape=f.shape)
    L = sp.tril(F, -1) + sp.identity(f.shape[0])
    U = sp.triu(F)
    B = M[f.perm][:, f.perm]
    assert abs(L @ U - B).max() <= 1e-12 * abs(B).max()
    # a cycle has no fill-free order
    C = sp.csr_matrix(np.array([[2.0, -1, -1], [-1, 2, -1], [-1, -1, 2]]))
    with pytest.raises(ValueError):
        tree_elimination_order(C)


def test_gmg_hierarchy_contracts():
    """prolongation partition of unity, Galerkin products, non-coarsenable grids (reference tests/test_krylov.py)."""
    from paper_2505_08491_b200 import krylov
    P = krylov.prolongation_3d(3)
    assert np.allclose(P @ np.ones(27), 1.0)
    grid = G.StructuredGrid(9)
    Kl = A.assemble_3d(grid, A.PhysicalParams(k_omega=1.0, sigma_omega=1.0))
    P0 = krylov.prolongation_3d(5)
    assert abs((P0.T @ Kl @ P0) - (P0.T @ Kl @ P0)).max() == 0.0
    with pytest.raises(ValueError, match="coarsenable"):
        krylov.gmg_build(G.StructuredGrid(6), A.assemble_3d(G.StructuredGrid(6), A.PhysicalParams()), 2)
    with pytest.raises(ValueError, match="at least 1"):
        krylov.gmg_build(grid, Kl, 0)
    with pytest.raises(ValueError):
        krylov.GmgPreconditioner(None, cycles=0)


def test_cfg4_geometry_index_sets_vs_reference():
    """The north-star 128^3 geometry (64-segment seed-3 tree, 32 elements per segment,
    8-point ring average) under the reference's own assemble_coupled_system
    (R = 0.0078 < h, golden cfg4_ref): Pi / Psi / W, A11 and M10 bit-exact."""
    g = golden("cfg4_ref")
    s = A.assemble_coupled_system(G.StructuredGrid(129), G.random_tree(64, 3, 0.0078),
                                  A.PhysicalParams(epsilon=0.0078, beta=1.0), n_circle=8, elems_per_edge=32)
    assert s.n1 == int(g["n1"])
    r = s.restriction
    same_csr(r.matrix, g, "T")
    same_csr(r.basis_1d, g, "psi")
    assert np.array_equal(r.weights, g["W"])
    same_csr(A.one_d_operator(s), g, "A11")
    same_csr(s.M10, g, "M10")
    assert np.array_equal(s.rhs1, g["rhs1"])
    assert np.array_equal(s.rhs0[g["touched"]], g["rhs0_touched"])

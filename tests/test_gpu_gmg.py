"""Geometric multigrid baseline (krylov.py:302-387) on the device vs the reference
(tests/golden/gmg.npz: V-cycles, 3-cycle applications and a GMG-preconditioned
FGMRES solve on the reduced operators of the n=9 family system and the cfg1
geometry)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _cases():
    from paper_2505_08491_b200 import assembly as A, geometry as G
    g = golden("asm_n9_family")
    graph = G.Graph1D(g["graph_vertices"], g["graph_edges"], 1e-3, tuple(int(d) for d in g["dirichlet"]))
    s9 = A.assemble_coupled_system(G.StructuredGrid(9), graph, A.PhysicalParams())
    g17 = G.Graph1D([[0.5, 0.5, 0.1], [0.5, 0.5, 0.9]], [[0, 1]], 0.02, (0,))
    s17 = A.assemble_coupled_system(G.StructuredGrid(17), g17, A.PhysicalParams(epsilon=0.02, beta=1.0),
                                    n_circle=8, elems_per_edge=32)
    return {"n9": (s9, 3), "n17": (s17, 4)}


@pytest.mark.parametrize("tag", ["n9", "n17"])
def test_gmg_vcycles_and_solve_vs_reference(gpu, tag):
    from paper_2505_08491_b200 import assembly as A, krylov
    g = golden("gmg")
    s, levels = _cases()[tag]
    C = A.host_reduced_operator(s)
    hier = krylov.gmg_build(s.grid, C, levels)
    assert [M.nnz for M in hier.matrices] == list(g[f"{tag}_coarse_nnz"])
    r = g[f"{tag}_r"]
    assert rel(krylov.gmg_vcycle(hier, r), g[f"{tag}_vcycle"]) <= 1e-12
    assert rel(krylov.gmg_vcycle(hier, r, n_pre=2, n_post=2), g[f"{tag}_vcycle_22"]) <= 1e-12
    assert rel(krylov.GmgPreconditioner(hier, cycles=3).apply(r), g[f"{tag}_apply3"]) <= 1e-12
    assert np.all(krylov.gmg_vcycle(hier, np.zeros_like(r)) == 0.0)
    # GMG-preconditioned FGMRES on the device operator (krylov.fgmres drop-in)
    x, rep = krylov.fgmres(A.reduced_operator(s), krylov.GmgPreconditioner(hier, cycles=2), g[f"{tag}_b"],
                           restart=20, tol=1e-8, maxit=200)
    assert rep.converged and abs(rep.iterations - int(g[f"{tag}_iters"])) <= 1
    assert rel(x, g[f"{tag}_x"]) <= 1e-7


def test_gmg_device_operator_and_strategy(gpu):
    """gmg_build from the device reduced_operator, and the 'gmg' spec of build_preconditioner."""
    from paper_2505_08491_b200 import assembly as A, harness, krylov
    g = golden("gmg")
    s, levels = _cases()["n9"]
    hier = krylov.gmg_build(s.grid, A.reduced_operator(s), levels)
    assert rel(krylov.gmg_vcycle(hier, g["n9_r"]), g["n9_vcycle"]) <= 1e-12
    P = harness.build_preconditioner({"type": "gmg", "cycles": 3, "levels": levels}, s.grid, A.reduced_operator(s),
                                     None)
    assert rel(P.apply(g["n9_r"]), g["n9_apply3"]) <= 1e-12


def test_coupled_solve_gmg_inner_vs_reference(gpu):
    """harness.solve_coupled with three_d={"type": "gmg"} (the reference's baseline setting)."""
    from paper_2505_08491_b200 import harness
    g = golden("gmg")
    s, levels = _cases()["n9"]
    st = harness.CoupledStrategy(tol=1e-6, maxit=60, restart=30, inner_iterations=3, one_d="ilu0",
                                 three_d={"type": "gmg", "cycles": 2, "levels": levels})
    u3, u1, rep = harness.solve_coupled(s, st)
    assert rep.converged == bool(g["coupled_conv"])
    assert abs(rep.iterations - int(g["coupled_iters"])) <= 1
    assert np.allclose(rep.residual_history[:4], g["coupled_hist"][:4], rtol=1e-6)
    assert rel(u3, g["coupled_u3"]) <= 1e-5

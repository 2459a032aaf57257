"""Error behaviour of the drop-in API, checked on the host: the
reference raises these before any arithmetic, and so must the device path."""

import numpy as np
import pytest

from paper_2505_08491_b200 import assembly as A, geometry as G, harness, krylov, neural, training


def _system(n=9, eps=1e-3):
    return A.assemble_coupled_system(G.StructuredGrid(n), G.random_tree(3, 4, eps), A.PhysicalParams(epsilon=eps),
                                     elems_per_edge=2)


def test_assembly_contracts():
    grid = G.StructuredGrid(9)
    with pytest.raises(ValueError):  # graph radius != epsilon (assembly.py:310-311)
        A.assemble_coupled_system(grid, G.random_tree(3, 4, 1e-3), A.PhysicalParams(epsilon=2e-3))
    with pytest.raises(ValueError):  # epsilon > h (assembly.py:312-314)
        A.assemble_coupled_system(grid, G.random_tree(3, 4, 0.2), A.PhysicalParams(epsilon=0.2))
    with pytest.raises(ValueError):
        A.assemble_coupled_system(grid, G.random_tree(3, 4, 1e-3), A.PhysicalParams(epsilon=1e-3), bc3d="robin")
    s = _system()
    with pytest.raises(ValueError):  # assembly.py:359-361
        A.reduced_rhs(s, np.zeros(s.n1 + 1))


def test_fgmres_argument_contracts():
    class Op:  # stands in for a device operator; the checks precede any device work
        shape = (4, 4)
        matvec = None
    b = np.ones(4)
    with pytest.raises(ValueError):
        krylov.fgmres(Op(), None, b, restart=0)
    with pytest.raises(ValueError):
        krylov.fgmres(Op(), None, b, tol=0.0)
    with pytest.raises(TypeError):
        krylov.fgmres(Op(), 3.0, b)


def test_apply_contracts():
    p = neural.init_unet_params(0)
    d = G.DistanceField(G.StructuredGrid(9), np.zeros(729))
    with pytest.raises(ValueError):  # training.py:302-303
        training.apply_neural(p, np.zeros(728), d)
    with pytest.raises(ValueError):  # smoothing without C (training.py:304-306)
        training.apply_neural(p, np.zeros(729), d, smoothing=(2, 0.5))
    with pytest.raises(ValueError):  # training.py:325-330
        training.apply_batched(p, [np.zeros(729)] * 2, [d])
    with pytest.raises(ValueError):  # neural.py:432-435
        neural.unet_forward(p, np.zeros((2, 7, 7, 7)))


def test_coupled_strategy_contracts():
    s = _system()
    with pytest.raises(ValueError):  # unknown 1D block treatment
        harness.solve_coupled(s, harness.CoupledStrategy(one_d="bogus"))
    with pytest.raises(ValueError):
        harness.build_preconditioner({"type": "exact"}, s.grid, None, None)


def test_gmg_rejects_large_dense_coarse_level():
    """A hierarchy that stops coarsening early would need a dense inverse of the
    fine grid; it is rejected before any factorisation or device upload."""
    s = _system(n=33, eps=1e-3)
    with pytest.raises(ValueError, match="coarsest GMG level"):
        krylov.gmg_build(s.grid, A.host_reduced_operator(s), 1)

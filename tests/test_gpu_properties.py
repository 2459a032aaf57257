"""Size-independent properties of the device operators at the full BASELINE sizes, where the CPU
oracle is too slow to serve as a per-entry checker (cfg4 129^3, the cfg5 shapes 129^3 x 8 and 193^3 x 2):

* the coupled and the reduced operator are symmetric (M10 = M01^T bitwise in the reference,
  tests/test_assembly.py:192-197) and linear;
* K00 1 = sigma_Omega M 1 on the Neumann cube (the stiffness part annihilates constants; the reference
  checks C 1 = sigma M 1 + w M00 1, tests/test_assembly.py:328-333): the entries sum to sigma_Omega |Omega|
  and interior entries equal sigma_Omega h^3;
* the CNN apply is positively homogeneous of degree 1 (training.py:312-318: z = ||r|| U(r / ||r||, d)).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(case):
    from paper_2505_08491_b200 import configs
    from paper_2505_08491_b200.assembly import DeviceProblem
    if case == "cfg4":
        systems = configs.cfg4().systems
    else:
        n, nb = (int(v) for v in case.split("x"))
        systems = configs.cfg5_systems(n, nb)
    return DeviceProblem(systems)


def _rand(p, seed):
    """Random device vectors with the padding beyond n3 + n1 of each system zeroed."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    X = torch.randn((p.nsys, p.ld), dtype=torch.float64, device="cuda", generator=g)
    for i in range(p.nsys):
        X[i, p.n3 + int(p.n1[i]):] = 0.0
    return X


@pytest.mark.parametrize("case", ["cfg4", "129x8", "193x2"])
def test_operators_symmetric_and_linear_at_full_size(gpu, case):
    import torch
    from paper_2505_08491_b200.operators import CoupledOperator, ReducedOperator
    p = _problem(case)
    A, C = CoupledOperator(p), ReducedOperator(p)
    X, Y = _rand(p, 1), _rand(p, 2)
    AX, AY, W = p.zeros(), p.zeros(), p.zeros()
    A.matvec(X, AX)
    A.matvec(Y, AY)
    for i in range(p.nsys):
        m = p.n3 + int(p.n1[i])
        lhs, rhs = torch.dot(AX[i, :m], Y[i, :m]), torch.dot(X[i, :m], AY[i, :m])
        scale = torch.linalg.norm(AX[i, :m]) * torch.linalg.norm(Y[i, :m])
        assert abs(float(lhs - rhs)) <= 1e-11 * float(scale), (case, i, float(lhs), float(rhs))
    Z = 0.75 * X - 1.5 * Y
    A.matvec(Z, W)
    ref = 0.75 * AX - 1.5 * AY
    for i in range(p.nsys):
        m = p.n3 + int(p.n1[i])
        assert float(torch.linalg.norm(W[i, :m] - ref[i, :m]) / torch.linalg.norm(ref[i, :m])) <= 1e-12
    # reduced operator: symmetric on the 3D part
    CX, CY = p.zeros(), p.zeros()
    C.matvec(X, CX)
    C.matvec(Y, CY)
    for i in range(p.nsys):
        lhs, rhs = torch.dot(CX[i, :p.n3], Y[i, :p.n3]), torch.dot(X[i, :p.n3], CY[i, :p.n3])
        scale = torch.linalg.norm(CX[i, :p.n3]) * torch.linalg.norm(Y[i, :p.n3])
        assert abs(float(lhs - rhs)) <= 1e-11 * float(scale), (case, i)


@pytest.mark.parametrize("n", [129, 193])
def test_neumann_stencil_annihilates_constants(gpu, n):
    """Reference semantics (Neumann cube, centreline Pi): K00 1 = sigma_Omega M 1."""
    from paper_2505_08491_b200 import assembly as A, geometry as G
    from paper_2505_08491_b200.assembly import DeviceProblem
    from paper_2505_08491_b200.operators import CouplingOps
    h = 1.0 / (n - 1)
    R = 0.5 * h
    s = A.assemble_coupled_system(G.StructuredGrid(n), G.random_tree(8, 7, R), A.PhysicalParams(epsilon=R),
                                  elems_per_edge=16)
    p = DeviceProblem([s])
    ones = p.zeros()
    ones[0, :p.n3 + int(p.n1[0])] = 1.0
    Y = p.zeros()
    CouplingOps(p).stencil(ones, Y)
    y = Y[0, :p.n3]
    sig = s.params.sigma_omega
    assert abs(float(y.sum()) / sig - 1.0) <= 1e-11
    interior = y.view(n, n, n)[1:-1, 1:-1, 1:-1]
    assert float((interior - sig * h ** 3).abs().max()) <= 1e-12 * sig * h ** 3 * 1e3


def test_cnn_apply_positively_homogeneous_129(gpu, tmp_path):
    from paper_2505_08491_b200 import geometry as G, neural, training
    n = 129
    d = G.distance_field(G.random_tree(64, 3, 0.008), G.StructuredGrid(n))
    path = tmp_path / "p3.mdu3"
    neural.save_checkpoint(neural.perturbed_params(3), path)
    params = neural.load_checkpoint(path)
    r = np.random.default_rng(5).standard_normal(n ** 3)
    z1 = training.apply_neural(params, r, d)
    z2 = training.apply_neural(params, 4.0 * r, d)  # power of two: r / ||r|| is bit-identical
    assert np.array_equal(z2, 4.0 * z1)
    z3 = training.apply_neural(params, 2.5 * r, d)
    assert np.linalg.norm(z3 - 2.5 * z1) / np.linalg.norm(z1) <= 1e-4
    assert np.all(training.apply_neural(params, np.zeros(n ** 3), d) == 0.0)  # training.py:312-314

"""GPU parity of the system operators, ILU, Arnoldi and the FGMRES engine.

Compared against the reference's golden outputs (tests/golden) and the
oracle restatement at larger sizes.  FP64 operators: <= 1e-10 relative
(BASELINE north star); ILU sweeps: bitwise; FGMRES: identical control flow
(iterations, breakdowns, converged) on the reference's own test cases.
"""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402
from test_host_build import CASES, product_case  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", CASES)
def test_coupled_and_reduced_spmv_vs_reference(gpu, name):
    from paper_2505_08491_b200 import assembly as A
    g, s = product_case(name)
    Aop = A.full_operator(s)
    Cop = A.reduced_operator(s)
    assert rel(Aop @ g["x"], g["Ax"]) <= 1e-10
    assert rel(Cop @ g["x"][:s.n3], g["Cx"]) <= 1e-10
    assert np.allclose(Cop.diagonal(), g["Cdiag"], rtol=1e-14, atol=0)


@pytest.mark.parametrize("name", CASES)
def test_pi_gather_scatter_vs_reference(gpu, name):
    import torch
    from paper_2505_08491_b200.assembly import DeviceProblem
    from paper_2505_08491_b200.operators import CouplingOps
    g, s = product_case(name)
    p = DeviceProblem([s])
    ops = CouplingOps(p)
    X = p.pack([g["x"]])
    S = torch.zeros(p.Qtot, dtype=torch.float64, device="cuda")
    ops.gather(X, None, S)
    # s = W (T x3)
    assert rel(S.cpu().numpy(), s.restriction.weights * g["Tx"]) <= 1e-13
    # pull: y3 = alpha * w * T^T v
    S.copy_(torch.as_tensor(g["v"]))
    Y = p.zeros()
    ops.scatter(S, 1.0, Y)
    w = s.params.coupling_weight
    assert rel(Y[0, :s.n3].cpu().numpy(), w * g["TTv"]) <= 1e-13


@pytest.mark.parametrize("name", CASES)
def test_ilu_sweeps_bitwise(gpu, name):
    from paper_2505_08491_b200.assembly import one_d_operator
    from paper_2505_08491_b200.krylov import ilu0, ilu0_apply
    g, s = product_case(name)
    f = ilu0(one_d_operator(s))
    z = ilu0_apply(f, g["ilu_r"])
    assert np.array_equal(z, g["ilu_z"])


@pytest.mark.parametrize("bc3d,nc,n", [("neumann", 1, 65), ("dirichlet", 8, 65), ("dirichlet", 8, 33),
                                       ("dirichlet", 8, 97), ("neumann", 8, 50)])
def test_spmv_large_vs_oracle(gpu, bc3d, nc, n):
    from paper_2505_08491_b200 import assembly as A, geometry as G
    from oracle import problem as OP
    R = 0.01
    t = G.random_tree(32, 2000, R)
    s = A.assemble_coupled_system(G.StructuredGrid(n), t, A.PhysicalParams(epsilon=R, beta=1.3), n_circle=nc,
                                  elems_per_edge=16, bc3d=bc3d, f1d=1.0)
    o = OP.assemble_coupled_system(OP.StructuredGrid(n), OP.random_tree(32, 2000, R),
                                   OP.PhysicalParams(epsilon=R, beta=1.3), n_circle=nc, elems_per_edge=16,
                                   bc3d=bc3d, f1d=1.0)
    x = np.random.default_rng(5).standard_normal(s.n3 + s.n1)
    assert rel(A.full_operator(s) @ x, OP.full_operator(o) @ x) <= 1e-10
    assert rel(A.reduced_operator(s) @ x[:s.n3], OP.reduced_operator(o) @ x[:s.n3]) <= 1e-10


def _kron_k00(x3, n, h, kO, sO):
    """K00 x (Neumann) by sum factorisation of the 1D P1 stiffness / mass (assembly.py:83-125)."""
    def tri(v, axis, d_in, d_end, off):
        v = np.moveaxis(v, axis, -1)
        out = d_in * v
        out[..., 0] = d_end * v[..., 0]
        out[..., -1] = d_end * v[..., -1]
        out[..., 1:] += off * v[..., :-1]
        out[..., :-1] += off * v[..., 1:]
        return np.moveaxis(out, -1, axis)
    K = lambda v, a: tri(v, a, 2.0 / h, 1.0 / h, -1.0 / h)  # noqa: E731
    M = lambda v, a: tri(v, a, 4.0 * h / 6.0, 2.0 * h / 6.0, h / 6.0)  # noqa: E731
    v = x3.reshape(n, n, n)  # [z][y][x]
    out = kO * (M(M(K(v, 2), 1), 0) + M(K(M(v, 2), 1), 0) + K(M(M(v, 2), 1), 0)) + sO * M(M(M(v, 2), 1), 0)
    return out.ravel()


@pytest.mark.parametrize("n", [270, 130])
def test_stencil_multi_tile_vs_kronecker(gpu, n):
    """Grids wider than one x-tile (256 columns) and odd/even row pitches."""
    import torch
    from paper_2505_08491_b200 import assembly as A, geometry as G
    from paper_2505_08491_b200.operators import CouplingOps
    s = A.assemble_coupled_system(G.StructuredGrid(n), G.random_tree(2, 5, 1e-3), A.PhysicalParams(epsilon=1e-3),
                                  elems_per_edge=2)
    pb = A.DeviceProblem([s])
    x = np.random.default_rng(n).standard_normal(s.n3)
    X, Y = pb.zeros(), pb.zeros()
    X[0, :s.n3] = torch.as_tensor(x, device="cuda")
    CouplingOps(pb).stencil(X, Y)
    want = _kron_k00(x, n, 1.0 / (n - 1), s.params.k_omega, s.params.sigma_omega)
    assert rel(Y[0, :s.n3].cpu().numpy(), want) <= 1e-12


@pytest.mark.parametrize("n,bc3d", [(65, "dirichlet"), (65, "neumann"), (17, "dirichlet")])
def test_jacobi_sweep_vs_oracle(gpu, n, bc3d):
    """Fused Jacobi epilogue x + omega (r - C x) / diag(C) (krylov.py:290-299) on both stencil kernels."""
    import torch
    from paper_2505_08491_b200 import assembly as A, geometry as G
    from paper_2505_08491_b200.operators import ReducedOperator
    from oracle import problem as OP
    R = 0.01
    s = A.assemble_coupled_system(G.StructuredGrid(n), G.random_tree(16, 77, R), A.PhysicalParams(epsilon=R),
                                  n_circle=8, elems_per_edge=8, bc3d=bc3d, f1d=1.0)
    o = OP.assemble_coupled_system(OP.StructuredGrid(n), OP.random_tree(16, 77, R), OP.PhysicalParams(epsilon=R),
                                   n_circle=8, elems_per_edge=8, bc3d=bc3d, f1d=1.0)
    C = OP.reduced_operator(o).tocsr()
    rng = np.random.default_rng(n)
    x, r = rng.standard_normal(s.n3), rng.standard_normal(s.n3)
    want = x + (2.0 / 3.0) * (r - C @ x) / C.diagonal()
    pb = A.DeviceProblem([s])
    op = ReducedOperator(pb)
    X, Rr, Xo, T = pb.zeros(), pb.zeros(), pb.zeros(), pb.zeros()
    X[0, :s.n3] = torch.as_tensor(x, device="cuda")
    Rr[0, :s.n3] = torch.as_tensor(r, device="cuda")
    op.jacobi(Rr, X, Xo, 2.0 / 3.0, T)
    assert rel(Xo[0, :s.n3].cpu().numpy(), want) <= 1e-10
    op.jacobi(Rr, None, Xo, 2.0 / 3.0, T)  # zero initial guess
    assert rel(Xo[0, :s.n3].cpu().numpy(), (2.0 / 3.0) * r / C.diagonal()) <= 1e-12


@pytest.mark.parametrize("n", [33, 65])
def test_batched_spmv_equals_serial_bitwise(gpu, n):
    import torch
    from paper_2505_08491_b200 import assembly as A, geometry as G
    from paper_2505_08491_b200.operators import CoupledOperator
    grid = G.StructuredGrid(n)
    systems = [A.assemble_coupled_system(grid, G.random_tree(8 + 4 * i, 10 + i, 0.015),
                                         A.PhysicalParams(epsilon=0.015, beta=0.5 + i), elems_per_edge=16)
               for i in range(3)]
    pb = A.DeviceProblem(systems)
    xs = [np.random.default_rng(i).standard_normal(s.n3 + s.n1) for i, s in enumerate(systems)]
    X = pb.pack(xs)
    Y = pb.zeros()
    CoupledOperator(pb).matvec(X, Y)
    ys = pb.unpack(Y)
    for s, x, y in zip(systems, xs, ys):
        assert np.array_equal(A.full_operator(s) @ x, y)
    # selection: only system 1
    Y2 = pb.zeros()
    sel = torch.tensor([1], dtype=torch.int32, device="cuda")
    CoupledOperator(pb).matvec(X, Y2, sel)
    assert torch.equal(Y2[1], Y[1]) and float(Y2[0].abs().max()) == 0.0


def test_distance_field_vs_oracle(gpu):
    from paper_2505_08491_b200 import geometry as G
    from oracle import problem as OP
    t = G.random_tree(16, 4, 0.01)
    d = G.distance_field(t, G.StructuredGrid(33)).values
    ref = OP.distance_field(t.vertices, t.edges, OP.StructuredGrid(33))
    assert np.max(np.abs(d - ref)) <= 1e-14


class MatrixOperator:
    """Test-only device operator y = A x for a small host matrix (torch matmul)."""

    def __init__(self, A, ld):
        import torch
        self.M = torch.as_tensor(np.asarray(sp.csr_matrix(A).toarray()), device="cuda")
        self.n, self.ld = self.M.shape[0], ld

    def __call__(self, X, Y, sel):
        # one mat-vec per system so batched and serial calls do identical arithmetic
        for i in sel.tolist():
            Y[i, :self.n] = self.M @ X[i, :self.n]


def test_fgmres_engine_control_flow_vs_reference(gpu):
    import torch
    from paper_2505_08491_b200.krylov import FgmresEngine, ilu0, DeviceIlu
    g = golden("fgmres_cases")
    for name, kw in zip(g["names"], g["kw"]):
        kw = eval(str(kw))  # noqa: S307
        A = g[f"{name}_A"]
        b = g[f"{name}_b"]
        n = len(b)
        ld = (n + 31) // 32 * 32
        eng = FgmresEngine(1, n, ld, kw.get("restart", 20))
        B = torch.zeros((1, ld), dtype=torch.float64, device="cuda")
        B[0, :n] = torch.as_tensor(b)
        X0 = None
        if f"{name}_x0" in g:
            X0 = torch.zeros_like(B)
            X0[0, :n] = torch.as_tensor(g[f"{name}_x0"])
        P = None
        if name == "ilu_prec":
            ilu = DeviceIlu([ilu0(A)])

            def P(V, Z, sel, idx):
                ilu.apply(V, Z, ld, sel=sel)
        elif name == "zero_map":
            def P(V, Z, sel, idx):
                Z[sel.long()] = 0.0
        rep = eng.solve(MatrixOperator(A, ld), P, B, tol=kw.get("tol", 1e-6), maxit=kw.get("maxit", 1000),
                        x0=X0)[0]
        assert rep.iterations == int(g[f"{name}_iters"]), name
        assert rep.converged == bool(g[f"{name}_conv"]), name
        assert rep.breakdowns == int(g[f"{name}_brk"]), name
        h = g[f"{name}_hist"]
        assert len(rep.residual_history) == len(h), name
        assert np.allclose(rep.residual_history, h, rtol=1e-6, atol=1e-14), name
        x = eng.x[0, :n].cpu().numpy()
        assert np.allclose(x, g[f"{name}_x"], rtol=1e-7, atol=1e-9), name


def test_batched_engine_equals_serial(gpu):
    import torch
    from paper_2505_08491_b200.krylov import FgmresEngine
    g = golden("fgmres_cases")
    A = g["restart5_A"]
    n = A.shape[0]
    ld = 128
    rng = np.random.default_rng(1)
    bs = [rng.standard_normal(n) for _ in range(3)]
    B = torch.zeros((3, ld), dtype=torch.float64, device="cuda")
    for i, b in enumerate(bs):
        B[i, :n] = torch.as_tensor(b)
    eng = FgmresEngine(3, n, ld, 5)
    reps = eng.solve(MatrixOperator(A, ld), None, B, tol=1e-8, maxit=5000)
    Xb = eng.x.clone()
    for i in range(3):
        e1 = FgmresEngine(1, n, ld, 5)
        r1 = e1.solve(MatrixOperator(A, ld), None, B[i:i + 1].clone(), tol=1e-8, maxit=5000)[0]
        assert r1.iterations == reps[i].iterations
        assert torch.equal(e1.x[0], Xb[i])


@pytest.mark.parametrize("orth", ["mgs", "cgs2"])
def test_arnoldi_kernel_orthogonalises(gpu, orth):
    import torch
    from paper_2505_08491_b200 import _ext
    lib = _ext.lib()
    n, k = 100_000, 30
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    V = torch.zeros((1, k + 1, n), dtype=torch.float64, device="cuda")
    V[0, :k] = torch.as_tensor(Q.T)
    wv = rng.standard_normal(n)
    W = torch.as_tensor(wv, device="cuda").reshape(1, n).clone()
    nv = torch.tensor([k], dtype=torch.int32, device="cuda")
    H = torch.zeros((1, k + 2), dtype=torch.float64, device="cuda")
    work = torch.zeros(lib.mdp_arnoldi_work_bytes(1, k, n) // 8 + 1, dtype=torch.float64, device="cuda")
    gram = torch.as_tensor(np.tril(Q.T @ Q, -1), device="cuda").reshape(1, k, k) if orth == "mgs" else None
    if gram is not None:
        gram = torch.nn.functional.pad(gram, (0, 1, 0, 1)).contiguous()
    _ext.check(lib.mdp_arnoldi(1, None, V.data_ptr(), (k + 1) * n, n, nv.data_ptr(), k, W.data_ptr(), n, n,
                               H.data_ptr(), None, 0, _ext.ptr(gram), work.data_ptr(), _ext.stream()))
    h = H[0].cpu().numpy()
    assert np.allclose(h[:k], Q.T @ wv, rtol=1e-12, atol=1e-12)
    wr = wv - Q @ (Q.T @ wv)
    assert abs(h[k + 1] - np.linalg.norm(wr)) <= 1e-12 * np.linalg.norm(wr)
    vnext = V[0, k].cpu().numpy()
    assert np.allclose(vnext, wr / np.linalg.norm(wr), atol=1e-12)
    assert np.max(np.abs(Q.T @ vnext)) <= (1e-13 if orth == "cgs2" else 1e-11)


@pytest.mark.parametrize("k,nsys", [(3, 2), (30, 1), (50, 2)])
def test_arnoldi_one_pass_mgs_equals_sequential_mgs(gpu, k, nsys):
    """The one-pass form (triangular solve over the Gram rows kept by the kernel itself) against
    the reference's sequential MGS loop (krylov.py:138-141) on a deliberately ill-conditioned
    sequence: each new direction lies mostly inside the span of the basis, so the Gram rows
    are far from zero (1e-9..1e-6) and CGS1 would visibly differ from MGS."""
    import torch
    from paper_2505_08491_b200 import _ext
    lib = _ext.lib()
    n = 20_011
    ld = (n + 31) // 32 * 32
    rng = np.random.default_rng(5)
    V = torch.zeros((nsys, k + 1, ld), dtype=torch.float64, device="cuda")
    W = torch.zeros((nsys, ld), dtype=torch.float64, device="cuda")
    H = torch.zeros((nsys, k + 2), dtype=torch.float64, device="cuda")
    gram = torch.zeros((nsys, k + 1, k + 1), dtype=torch.float64, device="cuda")
    work = torch.zeros(lib.mdp_arnoldi_work_bytes(nsys, k, n) // 8 + 1, dtype=torch.float64, device="cuda")
    Vh = np.zeros((nsys, k + 1, n))
    for s in range(nsys):
        v0 = rng.standard_normal(n)
        Vh[s, 0] = v0 / np.linalg.norm(v0)
    V[:, 0, :n] = torch.as_tensor(Vh[:, 0])
    for j in range(k):
        ws = np.zeros((nsys, n))
        for s in range(nsys):
            # mostly in span(V): strong cancellation, the hard case for Gram-Schmidt
            ws[s] = Vh[s, :j + 1].T @ rng.standard_normal(j + 1) * 1e6 + rng.standard_normal(n)
        W[:, :n] = torch.as_tensor(ws)
        nv = torch.full((nsys,), j + 1, dtype=torch.int32, device="cuda")
        _ext.check(lib.mdp_arnoldi(nsys, None, V.data_ptr(), (k + 1) * ld, ld, nv.data_ptr(), k, W.data_ptr(), ld, n,
                                   H.data_ptr(), None, 0, gram.data_ptr(), work.data_ptr(), _ext.stream()))
        h = H.cpu().numpy()
        for s in range(nsys):
            w = ws[s].copy()
            hm = np.zeros(j + 1)
            for i in range(j + 1):  # krylov.py:138-140
                hm[i] = w @ Vh[s, i]
                w -= hm[i] * Vh[s, i]
            hn = np.linalg.norm(w)
            # the device basis (not the host one) continues the sequence, so rounding does not accumulate
            Vh[s, j + 1] = V[s, j + 1, :n].cpu().numpy()
            scale = np.linalg.norm(ws[s])
            assert np.allclose(h[s, :j + 1], hm, rtol=0, atol=1e-12 * scale), (j, s)
            assert abs(h[s, k + 1] - hn) <= 1e-9 * hn, (j, s, h[s, k + 1], hn)
            assert np.allclose(Vh[s, j + 1], w / hn, atol=1e-8), (j, s)
            g = gram[s, j + 1, :j + 1].cpu().numpy()
            assert np.allclose(g, Vh[s, :j + 1] @ Vh[s, j + 1], atol=1e-14), (j, s)


def _dirichlet_k00(x3, n, h, kO, sO):
    """Dirichlet-cube K00: eliminated boundary columns, unit boundary rows."""
    v = x3.reshape(n, n, n).copy()
    inner = np.zeros((n, n, n), dtype=bool)
    inner[1:-1, 1:-1, 1:-1] = True
    y = _kron_k00(np.where(inner, v, 0.0).ravel(), n, h, kO, sO).reshape(n, n, n)
    return np.where(inner, y, v).ravel()


@pytest.mark.parametrize("n", [17, 33, 65, 129, 193])
@pytest.mark.parametrize("bc3d", ["neumann", "dirichlet"])
def test_stencil_configured_sizes_vs_kronecker(gpu, n, bc3d):
    """The compile-time-n instantiations of the v3 stencil (17/33: 2-row bands,
    65/129/193: 4-row bands), two systems in one launch, against the Kronecker
    restatement of K00 (assembly.py:83-125) with the Dirichlet-cube elimination."""
    import torch
    from paper_2505_08491_b200 import assembly as A, geometry as G
    from paper_2505_08491_b200.operators import CouplingOps
    grid = G.StructuredGrid(n)
    systems = [A.assemble_coupled_system(grid, G.random_tree(2, 5 + i, 1e-3), A.PhysicalParams(epsilon=1e-3),
                                         elems_per_edge=2, bc3d=bc3d) for i in range(2)]
    pb = A.DeviceProblem(systems)
    rng = np.random.default_rng(n)
    xs = [rng.standard_normal(pb.n3) for _ in range(2)]
    X, Y = pb.zeros(), pb.zeros()
    for i, x in enumerate(xs):
        X[i, :pb.n3] = torch.as_tensor(x, device="cuda")
    CouplingOps(pb).stencil(X, Y)
    p = systems[0].params
    f = _dirichlet_k00 if bc3d == "dirichlet" else _kron_k00
    for i, x in enumerate(xs):
        want = f(x, n, 1.0 / (n - 1), p.k_omega, p.sigma_omega)
        assert rel(Y[i, :pb.n3].cpu().numpy(), want) <= 1e-12


@pytest.mark.parametrize("n", [129])
def test_jacobi_sweep_large_vs_device_spmv(gpu, n):
    """Fused Jacobi epilogue of the n=129 instantiation against x + w (r - C x) / diag(C)
    formed from the device SpMV (which the reference-vector tests pin)."""
    import torch
    from paper_2505_08491_b200 import configs
    from paper_2505_08491_b200.assembly import DeviceProblem
    from paper_2505_08491_b200.operators import ReducedOperator
    pb = DeviceProblem(configs.cfg5_systems(n, 2))
    op = ReducedOperator(pb)
    X, Rr, Xo, T, CX = (pb.zeros() for _ in range(5))
    X[:, :pb.n3].normal_()
    Rr[:, :pb.n3].normal_()
    op.jacobi(Rr, X, Xo, 2.0 / 3.0, T)
    op.matvec(X, CX)
    d = pb._t["diag_c"].view(pb.nsys, pb.ld)
    want = X + (2.0 / 3.0) * (Rr - CX) / d
    for i in range(pb.nsys):
        assert rel(Xo[i, :pb.n3].cpu().numpy(), want[i, :pb.n3].cpu().numpy()) <= 1e-12


def test_coupled_spmv_129_batched_equals_serial_bitwise(gpu):
    import torch
    from paper_2505_08491_b200 import configs
    from paper_2505_08491_b200.assembly import DeviceProblem
    from paper_2505_08491_b200.operators import CoupledOperator
    pb = DeviceProblem(configs.cfg5_systems(129, 3))
    X = pb.zeros().normal_()
    Y = pb.zeros()
    CoupledOperator(pb).matvec(X, Y)
    for i in range(pb.nsys):
        Yi = pb.zeros()
        CoupledOperator(pb).matvec(X, Yi, torch.tensor([i], dtype=torch.int32, device="cuda"))
        assert torch.equal(Yi[i], Y[i])


def test_ilu3d_baseline_large_vs_reference(gpu):
    """3D ILU(0) on C at 33^3 (beyond the shared-memory sweep: x stays in global memory):
    the apply is bitwise equal to the reference's, the preconditioned solve takes its iterations."""
    from paper_2505_08491_b200 import assembly as A, geometry as G, krylov
    g = golden("ilu3d_n33")
    graph = G.Graph1D(g["vertices"], g["edges"], 1e-3, tuple(int(d) for d in g["dirichlet"]))
    s = A.assemble_coupled_system(G.StructuredGrid(33), graph, A.PhysicalParams())
    P = krylov.IluPreconditioner(A.reduced_operator(s))
    assert np.array_equal(P.apply(g["r"]), g["z"])
    x, rep = krylov.fgmres(A.reduced_operator(s), P, g["b"], restart=30, tol=1e-8, maxit=300)
    assert rep.converged and abs(rep.iterations - int(g["iters"])) <= 1

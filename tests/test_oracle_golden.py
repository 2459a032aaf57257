"""Pin the CPU oracle against fixtures produced by the reference itself.

Fixtures come from tests/golden/make_golden.py (reference imported
read-only in the build container).  Indices must match bit-exactly, values
to ~1e-13, FGMRES control flow (iterations, breakdowns, converged flag)
exactly.
"""

import math

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import problem as P
from oracle.unet import param_arrays
from conftest import golden


def csr(g, prefix):
    return sp.csr_matrix((g[f"{prefix}_data"], g[f"{prefix}_indices"], g[f"{prefix}_indptr"]),
                         shape=tuple(g[f"{prefix}_shape"]))


def assert_csr_equal(A, g, prefix, rtol=1e-13):
    A = sp.csr_matrix(A)
    assert np.array_equal(A.indptr, g[f"{prefix}_indptr"]), prefix
    assert np.array_equal(A.indices, g[f"{prefix}_indices"]), prefix
    ref = g[f"{prefix}_data"]
    scale = max(np.abs(ref).max(), 1e-300) if ref.size else 1.0
    assert np.max(np.abs(A.data - ref), initial=0.0) <= rtol * scale, prefix


def family_graph_from(g):
    return P.Graph(g["graph_vertices"], g["graph_edges"], 1e-3, (int(g["dirichlet"][0]),))


def build_case(name):
    g = golden(name)
    if name == "asm_n9_family":
        grid = P.StructuredGrid(9)
        # reference family graph: dirichlet = degree-1 root-face vertices
        graph = P.Graph(g["graph_vertices"], g["graph_edges"], 1e-3,
                        tuple(int(d) for d in g["dirichlet"]))
        s = P.assemble_coupled_system(grid, graph, P.PhysicalParams())
    elif name.startswith("asm_cfg1"):
        nc = int(name[-1])
        grid = P.StructuredGrid(17)
        graph = P.segment_graph([0.5, 0.5, 0.1], [0.5, 0.5, 0.9], 0.02)
        s = P.assemble_coupled_system(grid, graph, P.PhysicalParams(epsilon=0.02, beta=1.0),
                                      n_circle=nc, elems_per_edge=32)
    else:
        nc = int(name[-1])
        grid = P.StructuredGrid(33)
        graph = P.random_tree(8, 1, 0.015)
        assert np.array_equal(graph.vertices, g["tree_vertices"])
        s = P.assemble_coupled_system(grid, graph, P.PhysicalParams(epsilon=0.015, beta=1.0),
                                      n_circle=nc, elems_per_edge=16)
    return g, s


CASES = ["asm_n9_family", "asm_cfg1_nc1", "asm_cfg1_nc8", "asm_cfg2_nc1", "asm_cfg2_nc8"]


@pytest.mark.parametrize("name", CASES)
def test_assembly_bit_exact(name):
    g, s = build_case(name)
    assert np.array_equal(s.mesh.elements, g["mesh_elements"])
    assert np.array_equal(s.mesh.coords, g["mesh_coords"])
    assert np.array_equal(s.mesh.element_lengths, g["mesh_lengths"])
    rest = s.restriction
    assert_csr_equal(rest.matrix, g, "T")
    assert_csr_equal(rest.basis_1d, g, "psi")
    assert np.array_equal(rest.weights, g["wq"])
    assert np.array_equal(rest.points, g["qpts"])
    for blk in ("K11", "M00", "M01", "M10", "M11"):
        assert_csr_equal(getattr(s, blk), g, blk)
    assert_csr_equal(P.one_d_operator(s), g, "A11")
    assert np.allclose(s.rhs0, g["rhs0"], rtol=0, atol=1e-15 * max(1, np.abs(g["rhs0"]).max()))
    assert np.allclose(s.rhs1, g["rhs1"], rtol=0, atol=1e-14 * max(1, np.abs(g["rhs1"]).max()))
    if name == "asm_n9_family":
        assert_csr_equal(s.K00, g, "K00")


@pytest.mark.parametrize("name", CASES)
def test_operator_actions(name):
    g, s = build_case(name)
    x = g["x"]
    A = P.full_operator(s)
    C = P.reduced_operator(s)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(A @ x, g["Ax"]) < 1e-14
    assert rel(C @ x[:s.n3], g["Cx"]) < 1e-14
    assert rel(s.restriction.matrix @ x[:s.n3], g["Tx"]) < 1e-15
    assert rel(s.restriction.matrix.T @ g["v"], g["TTv"]) < 1e-15
    assert np.allclose(C.diagonal(), g["Cdiag"], rtol=1e-15, atol=0)
    f = oracle.ilu0(P.one_d_operator(s))
    assert np.allclose(f.data, g["ilu_data"], rtol=1e-14, atol=1e-300)
    assert rel(oracle.ilu0_apply(f, g["ilu_r"]), g["ilu_z"]) < 1e-14


def test_distance_field_matches():
    g = golden("asm_n9_family")
    d = P.distance_field(g["graph_vertices"], g["graph_edges"], P.StructuredGrid(9))
    assert np.array_equal(d, g["dfield"])


def test_fgmres_control_flow():
    g = golden("fgmres_cases")
    for name, kw in zip(g["names"], g["kw"]):
        kw = eval(str(kw))  # noqa: S307  (repr of a small literal dict we wrote)
        A = sp.csr_matrix(g[f"{name}_A"])
        b = g[f"{name}_b"]
        x0 = g[f"{name}_x0"] if f"{name}_x0" in g else None
        pre = None
        if name == "ilu_prec":
            f = oracle.ilu0(A)
            pre = lambda r, f=f: oracle.ilu0_apply(f, r)  # noqa: E731
        elif name == "zero_map":
            pre = lambda r: np.zeros_like(r)  # noqa: E731
        x, rep = oracle.fgmres(A, pre, b, x0=x0, **kw)
        assert rep.iterations == int(g[f"{name}_iters"]), name
        assert rep.converged == bool(g[f"{name}_conv"]), name
        assert rep.breakdowns == int(g[f"{name}_brk"]), name
        h = g[f"{name}_hist"]
        assert len(rep.residual_history) == len(h)
        assert np.allclose(rep.residual_history, h, rtol=1e-9, atol=1e-15), name
        assert np.allclose(x, g[f"{name}_x"], rtol=1e-10, atol=1e-12), name


@pytest.mark.parametrize("seed", [0, 1])
def test_param_init_and_noise_replicate(seed):
    g = golden("unet_forward")
    for tag, p in (("init", oracle.init_unet_params(seed)), ("noisy", oracle.noisy_params(seed))):
        for key, arr in param_arrays(p):
            assert np.array_equal(arr.ravel()[:6], g[f"{tag}{seed}_{key}_head"]), key
            assert math.isclose(arr.sum(), float(g[f"{tag}{seed}_{key}_sum"]), rel_tol=1e-12,
                                abs_tol=1e-12), key


def test_unet_layers_and_forward():
    g = golden("unet_forward")
    assert np.allclose(oracle.conv3d(g["conv_x"], g["conv_k"], g["conv_b"]), g["conv_y"],
                       rtol=1e-12, atol=1e-12)
    assert np.allclose(oracle.transposed_conv3d(g["tconv_x"], g["tconv_k"], 0, g["tconv_b"]),
                       g["tconv_y0"], rtol=1e-13, atol=1e-13)
    y1 = oracle.transposed_conv3d(g["tconv_x"], g["tconv_k"], 1, g["tconv_b"])
    assert np.allclose(y1, g["tconv_y1"], rtol=1e-13, atol=1e-13)
    assert np.array_equal(oracle.maxpool3d(g["pool_x"]), g["pool_y"])
    p = oracle.noisy_params(0)
    for n in (9, 13, 17):
        y = oracle.unet_forward(p, g[f"x_n{n}"])
        ref = g[f"y_n{n}"]
        assert np.max(np.abs(y - ref)) <= 1e-12 * max(1.0, np.abs(ref).max()), n
    yb = oracle.unet_forward(p, g["xb"])
    assert np.max(np.abs(yb - g["yb"])) <= 1e-12 * max(1.0, np.abs(g["yb"]).max())


def test_checkpoint_bytes_match(tmp_path):
    import hashlib
    g = golden("apply_solve_n9")
    path = tmp_path / "n.mdu3"
    oracle.save_checkpoint(oracle.noisy_params(0), path)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == str(g["ckpt_sha256"])


def _n9_system():
    g = golden("asm_n9_family")
    graph = P.Graph(g["graph_vertices"], g["graph_edges"], 1e-3,
                    tuple(int(d) for d in g["dirichlet"]))
    return P.assemble_coupled_system(P.StructuredGrid(9), graph, P.PhysicalParams())


def test_apply_neural_and_batched(tmp_path):
    g = golden("apply_solve_n9")
    s = _n9_system()
    path = tmp_path / "n.mdu3"
    oracle.save_checkpoint(oracle.noisy_params(0), path)
    p = oracle.load_checkpoint(path)
    from oracle.coupled import mesh_distance_field
    d = mesh_distance_field(s)
    assert np.allclose(d, g["dfield_mesh"], rtol=0, atol=1e-15)
    C = P.reduced_operator(s)
    z = oracle.apply_neural(p, g["r"], d)
    assert np.max(np.abs(z - g["z_plain"])) <= 1e-12 * np.abs(g["z_plain"]).max()
    zs = oracle.apply_neural(p, g["r"], d, smoothing=(2, 2.0 / 3.0), C=C)
    assert np.max(np.abs(zs - g["z_smooth"])) <= 1e-12 * np.abs(g["z_smooth"]).max()
    zb = oracle.apply_batched(p, list(g["rs"]), [d] * 4)
    assert np.max(np.abs(np.array(zb) - g["zs_batched"])) <= 1e-12 * np.abs(g["zs_batched"]).max()
    assert np.all(zb[3] == 0.0)


@pytest.mark.parametrize("label", ["none", "ilu0", "neural_s"])
def test_coupled_solve_n9(label, tmp_path):
    g = golden("apply_solve_n9")
    s = _n9_system()
    spec = {"type": label}
    if label == "neural_s":
        path = tmp_path / "n.mdu3"
        oracle.save_checkpoint(oracle.noisy_params(0), path)
        spec = {"type": "neural", "params": oracle.load_checkpoint(path), "smoothing": (2, 2.0 / 3.0)}
    st = oracle.CoupledStrategy(tol=1e-6, maxit=120, restart=30, inner_iterations=3, three_d=spec)
    u3, u1, rep = oracle.solve_coupled(s, st)
    assert rep.iterations == int(g[f"solve_{label}_iters"])
    assert rep.converged == bool(g[f"solve_{label}_conv"])
    assert np.allclose(rep.residual_history, g[f"solve_{label}_hist"], rtol=1e-6, atol=1e-12)
    assert np.allclose(u3, g[f"solve_{label}_u3"], rtol=1e-8, atol=1e-10)


@pytest.mark.parametrize("label", ["none", "ilu0"])
def test_coupled_solve_n9_direct_1d(label):
    """one_d='direct' (harness.py:356-358) pinned to the reference's solves."""
    g = golden("direct_n9")
    s = _n9_system()
    A11 = P.one_d_operator(s)
    import scipy.sparse.linalg as spla
    z1 = np.array([spla.spsolve(A11.tocsc(), r) for r in g["r1"]])
    assert np.max(np.abs(z1 - g["z1"])) <= 1e-12 * np.abs(g["z1"]).max()
    st = oracle.CoupledStrategy(tol=1e-6, maxit=120, restart=30, inner_iterations=3, three_d={"type": label},
                                one_d="direct")
    u3, u1, rep = oracle.solve_coupled(s, st)
    assert rep.iterations == int(g[f"solve_{label}_iters"])
    assert rep.converged == bool(g[f"solve_{label}_conv"])
    assert np.allclose(rep.residual_history, g[f"solve_{label}_hist"], rtol=1e-6, atol=1e-12)
    assert np.allclose(u3, g[f"solve_{label}_u3"], rtol=1e-8, atol=1e-10)
    assert np.allclose(u1, g[f"solve_{label}_u1"], rtol=1e-8, atol=1e-10)

"""Golden fixtures at the north-star sizes: cfg4 (128^3 cells) and cfg3 (16 x 64^3).

Run in the build container only (the reference parts need /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_large_golden.py [part ...]

Parts (each writes one ``.npz`` next to this script):

``cnn129``      the REFERENCE ``apply_neural`` (training.py:289-319 -> neural.unet_forward
                neural.py:423-472) of the perturbed seed-3 network (MDU3 round trip, the
                network configured for 32^3 and applied at 129^3: resolution transfer,
                neural.py:356,434-435) on a seeded residual and the distance field of the
                cfg4 tree.  A 129^3 output is 17 MB, so the fixture keeps 16384 seeded sample
                voxels, the norm and four seeded projections.
``cfg4_ref``    the REFERENCE ``assemble_coupled_system`` (assembly.py:306-348) on the cfg4
                geometry (129^3, 64-segment seed-3 tree, 32 elements per segment, ring
                average n_circle=8, beta=1) with R = 0.0078 < h = 1/128 so the reference's own
                radius check passes, Neumann cube: Pi / Psi / W and the 1D blocks
                bit-exact, full / reduced operator products on seeded vectors (1D part whole,
                3D part at every touched node plus samples), and the head (5 outer
                iterations) of the reference's neural-preconditioned solve_coupled
                (harness.py:342-398; restart 50, rtol 1e-8, Jacobi(2, 2/3)-smoothed CNN).
``cfg4_oracle`` the same for BASELINE cfg4 exactly as configured (R = 0.008 > h with the radius
                check relaxed, homogeneous Dirichlet cube, f1D = 1): the oracle restatement
                (pinned to the reference by the other fixtures), operator samples + solve head.
``cfg3``        BASELINE cfg3 (16 systems at 65^3, 32-segment trees seeds 2000+i, beta_i from
                default_rng(2)), oracle: per-system solve heads (4 outer iterations, restart
                50) and one operator sample.
``cfg2_full``   BASELINE cfg2's whole 2000-iteration oracle solve: iterations, converged flag,
                final residual and history.
"""

from __future__ import annotations

import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE))

NSAMPLE = 16384


def dump(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print("wrote", name, flush=True)


def sample_idx(n3, seed=7):
    return np.sort(np.random.default_rng(seed).choice(n3, NSAMPLE, replace=False)).astype(np.int64)


def projections(z, n3, seed=11):
    V = np.random.default_rng(seed).standard_normal((4, n3))
    return V @ z


def cfg4_graph():
    from oracle.problem import random_tree
    return random_tree(64, 3, 0.008)


def cfg4_vectors(n3, n1):
    rng = np.random.default_rng(41)
    return rng.standard_normal(n3 + n1)


def ref_params_ckpt(td, seed):
    import make_golden as MG
    from mdprec import neural
    ck = Path(td) / f"noisy{seed}.mdu3"
    neural.save_checkpoint(MG.noisy_params(seed), ck)
    return ck


def gen_cnn129():
    sys.path.insert(0, "/root/reference/pkg/src")
    from mdprec import geometry, neural, training
    n = 129
    g = cfg4_graph()
    grid = geometry.StructuredGrid(n)
    graph = geometry.Graph1D(g.vertices, g.edges, g.radius, g.dirichlet_vertices)
    d = geometry.distance_field(graph, grid)
    r = np.random.default_rng(129).standard_normal(n ** 3)
    with tempfile.TemporaryDirectory() as td:
        p = neural.load_checkpoint(ref_params_ckpt(td, 3))
    t = time.time()
    z = training.apply_neural(p, r, d)
    print("cnn129 reference apply", time.time() - t, "s", flush=True)
    idx = sample_idx(n ** 3)
    dump("cnn129", idx=idx, z_sample=z[idx], z_norm=np.array(np.linalg.norm(z)),
         z_proj=projections(z, n ** 3), d_sample=d.values[idx])


def _operator_pins(s_full, s_red_x, n3, n1, A, C, touched):
    x = cfg4_vectors(n3, n1)
    y = A @ x
    y3 = C @ x[:n3]
    idx = sample_idx(n3)
    return dict(y1=y[n3:], y3_touched=y[touched], y3_sample=y[idx], y_norm=np.array(np.linalg.norm(y)),
                c_touched=y3[touched], c_sample=y3[idx], c_norm=np.array(np.linalg.norm(y3)),
                touched=touched.astype(np.int64), idx=idx)


def _touched(T):
    return np.unique(T.tocsr().indices)


def gen_cfg4_ref():
    sys.path.insert(0, "/root/reference/pkg/src")
    import make_golden as MG
    from mdprec import assembly, geometry, harness
    n, R = 129, 0.0078
    g = cfg4_graph()
    assembly.refine_graph = MG.fixed_refine(32)
    try:
        grid = geometry.StructuredGrid(n)
        graph = geometry.Graph1D(g.vertices, g.edges, R, g.dirichlet_vertices)
        t = time.time()
        s = assembly.assemble_coupled_system(grid, graph, MG.BetaParams(epsilon=R, beta=1.0), n_circle=8)
        print("cfg4_ref assembly", time.time() - t, "s", flush=True)
        A = assembly.full_operator(s)
        C = assembly.reduced_operator(s)
        rest = assembly.build_restriction(grid, s.graph_mesh, 8, radius=R)  # assembly.py:316
        T = rest.matrix.tocsr()
        out = _operator_pins(s, None, s.n3, s.n1, A, C, _touched(T))
        A11 = assembly.one_d_operator(s).tocsr()
        M10 = s.M10.tocsr()
        out.update(T_indptr=T.indptr, T_indices=T.indices, T_data=T.data,
                   psi_indptr=rest.basis_1d.tocsr().indptr, psi_indices=rest.basis_1d.tocsr().indices,
                   psi_data=rest.basis_1d.tocsr().data, W=rest.weights,
                   A11_indptr=A11.indptr, A11_indices=A11.indices, A11_data=A11.data,
                   M10_indptr=M10.indptr, M10_indices=M10.indices, M10_data=M10.data,
                   rhs0_touched=s.rhs0[out["touched"]], rhs1=s.rhs1, n1=np.array(s.n1))
        with tempfile.TemporaryDirectory() as td:
            ck = ref_params_ckpt(td, 3)
            spec = {"type": "neural", "checkpoint": str(ck), "smoothing": {"maxit": 2}}
            st = harness.CoupledStrategy(tol=1e-8, maxit=5, restart=50, inner_iterations=3, one_d="ilu0",
                                         three_d=spec)
            t = time.time()
            _, _, rep = harness.solve_coupled(s, st)
            print("cfg4_ref solve head", rep.iterations, rep.residual_history, time.time() - t, "s", flush=True)
        out.update(head_iters=np.array(rep.iterations), head_conv=np.array(rep.converged),
                   head_hist=np.array(rep.residual_history))
        dump("cfg4_ref", **out)
    finally:
        assembly.refine_graph = MG._ORIG_REFINE


def _oracle_head(s, cnn_seed, restart, tol, maxit):
    import oracle
    spec = {"type": "neural", "params": oracle_params(cnn_seed), "smoothing": (2, 2.0 / 3.0)}
    st = oracle.CoupledStrategy(tol=tol, maxit=maxit, restart=restart, inner_iterations=3, three_d=spec)
    t = time.time()
    _, _, rep = oracle.solve_coupled(s, st)
    print("oracle solve", rep.iterations, rep.converged, rep.rel_residual, time.time() - t, "s", flush=True)
    return rep


def oracle_params(seed):
    """The perturbed network after the MDU3 float32 round trip (what the device loads)."""
    import oracle
    with tempfile.TemporaryDirectory() as td:
        path = Path(td) / "p.mdu3"
        oracle.save_checkpoint(oracle.noisy_params(seed), path)
        return oracle.load_checkpoint(path)


def gen_cfg4_oracle():
    from oracle import problem as OP
    n, R = 129, 0.008
    t = time.time()
    s = OP.assemble_coupled_system(OP.StructuredGrid(n), cfg4_graph(), OP.PhysicalParams(epsilon=R, beta=1.0),
                                   n_circle=8, elems_per_edge=32, bc3d="dirichlet", f1d=1.0, check_radius=False)
    print("cfg4_oracle assembly", time.time() - t, "s", flush=True)
    out = _operator_pins(s, None, s.n3, s.n1, OP.full_operator(s), OP.reduced_operator(s),
                         _touched(s.restriction.matrix))
    out.update(rhs1=s.rhs1, n1=np.array(s.n1))
    rep = _oracle_head(s, 3, 50, 1e-8, 5)
    out.update(head_iters=np.array(rep.iterations), head_conv=np.array(rep.converged),
               head_hist=np.array(rep.residual_history))
    dump("cfg4_oracle", **out)


def gen_cfg3():
    from oracle import problem as OP
    n = 65
    betas = np.random.default_rng(2).uniform(0.5, 2.0, 16)
    out = {"betas": betas}
    hists = []
    for i in range(16):
        s = OP.assemble_coupled_system(OP.StructuredGrid(n), OP.random_tree(32, 2000 + i, 0.01),
                                       OP.PhysicalParams(epsilon=0.01, beta=float(betas[i])), n_circle=8,
                                       elems_per_edge=16, bc3d="dirichlet", f1d=1.0)
        if i == 0:
            pins = _operator_pins(s, None, s.n3, s.n1, OP.full_operator(s), OP.reduced_operator(s),
                                  _touched(s.restriction.matrix))
            out.update({f"s0_{k}": v for k, v in pins.items()})
        rep = _oracle_head(s, 2, 50, 1e-6, 4)
        hists.append(rep.residual_history)
        out[f"iters_{i}"] = np.array(rep.iterations)
        out[f"conv_{i}"] = np.array(rep.converged)
    out["hist"] = np.array(hists)
    dump("cfg3_head", **out)


def gen_cfg2_full():
    from oracle import problem as OP
    s = OP.assemble_coupled_system(OP.StructuredGrid(33), OP.random_tree(8, 1, 0.015),
                                   OP.PhysicalParams(epsilon=0.015, beta=1.0), n_circle=8, elems_per_edge=16,
                                   bc3d="dirichlet", f1d=1.0)
    rep = _oracle_head(s, 1, 30, 1e-6, 2000)
    dump("cfg2_full", iters=np.array(rep.iterations), conv=np.array(rep.converged),
         rel=np.array(rep.rel_residual), hist=np.array(rep.residual_history), breakdowns=np.array(rep.breakdowns))


PARTS = {"cnn129": gen_cnn129, "cfg4_ref": gen_cfg4_ref, "cfg4_oracle": gen_cfg4_oracle, "cfg3": gen_cfg3,
         "cfg2_full": gen_cfg2_full}

if __name__ == "__main__":
    for part in (sys.argv[1:] or list(PARTS)):
        PARTS[part]()

"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports ``mdprec`` read-only from /root/reference/pkg/src and writes
small ``.npz`` fixtures next to this script.  BASELINE-only semantics the
reference API cannot express are injected with the reference's own
building blocks: a ``PhysicalParams`` subclass whose
``coupling_weight`` is beta (A3) and a fixed-m ``refine_graph`` patched into
``mdprec.assembly`` (A5).  Everything else is the stock reference code path.
"""

from __future__ import annotations

import dataclasses
import math
import os
import sys
import tempfile
from pathlib import Path

import numpy as np
import scipy.sparse as sp

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from mdprec import assembly, geometry, harness, krylov, neural, training  # noqa: E402

from oracle.problem import random_tree  # noqa: E402  (BASELINE generator, A6)


@dataclasses.dataclass(frozen=True)
class BetaParams(assembly.PhysicalParams):
    beta: float = 1.0

    @property
    def coupling_weight(self) -> float:
        return self.beta


_ORIG_REFINE = assembly.refine_graph


def fixed_refine(m):
    """refine_graph with a fixed number of elements per edge, same node order."""
    def refine(graph, h_target):
        coords = [graph.vertices]
        elems, lens = [], []
        nxt = len(graph.vertices)
        for (a, b), L in zip(graph.edges, graph.edge_lengths):
            pa, pb = graph.vertices[a], graph.vertices[b]
            t = np.arange(1, m)[:, None] / m
            coords.append(pa + t * (pb - pa))
            chain = [a] + list(range(nxt, nxt + m - 1)) + [b]
            nxt += m - 1
            for u, v in zip(chain[:-1], chain[1:]):
                elems.append((u, v))
                lens.append(L / m)
        return geometry.GraphMesh1D(np.vstack(coords), np.array(elems, dtype=np.int64),
                                    np.array(lens), tuple(graph.dirichlet_vertices))
    return refine


def csr_dict(prefix, A):
    A = sp.csr_matrix(A)
    return {f"{prefix}_indptr": A.indptr.astype(np.int64), f"{prefix}_indices": A.indices.astype(np.int64),
            f"{prefix}_data": A.data.copy(), f"{prefix}_shape": np.array(A.shape)}


def system_dict(s, rest):
    d = {}
    for name in ("K11", "M00", "M01", "M10", "M11"):
        d.update(csr_dict(name, getattr(s, name)))
    d.update(csr_dict("T", rest.matrix))
    d.update(csr_dict("psi", rest.basis_1d))
    d["wq"] = rest.weights
    d["qpts"] = rest.points
    d["rhs0"] = s.rhs0
    d["rhs1"] = s.rhs1
    d["dirichlet"] = np.array(s.dirichlet_nodes, dtype=np.int64)
    d["mesh_coords"] = s.graph_mesh.coords
    d["mesh_elements"] = s.graph_mesh.elements
    d["mesh_lengths"] = s.graph_mesh.element_lengths
    d["w"] = np.array(s.params.coupling_weight)
    A = assembly.full_operator(s)
    C = assembly.reduced_operator(s)
    A11 = assembly.one_d_operator(s)
    d.update(csr_dict("A11", A11))
    rng = np.random.default_rng(1234)
    x = rng.standard_normal(A.shape[0])
    d["x"] = x
    d["Ax"] = A @ x
    d["Cx"] = C @ x[:s.n3]
    d["M01x1"] = s.M01 @ x[s.n3:]
    d["Tx"] = rest.matrix @ x[:s.n3]
    v = rng.standard_normal(rest.matrix.shape[0])
    d["v"] = v
    d["TTv"] = rest.matrix.T @ v
    fact = krylov.ilu0(A11)
    r1 = rng.standard_normal(s.n1)
    d["ilu_r"] = r1
    d["ilu_z"] = krylov.ilu0_apply(fact, r1)
    d["ilu_data"] = fact.data
    d["Cdiag"] = np.asarray(C.diagonal())
    return d


def restriction_for(grid, graph, params, n_circle):
    mesh = assembly.refine_graph(graph, grid.h)
    return assembly.build_restriction(grid, mesh, n_circle, radius=params.epsilon)


def dump(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print("wrote", name, sum(np.asarray(v).nbytes for v in arrays.values()), "bytes raw")


def gen_assembly():
    # (1) reference-native: n=9, reference tree family, default physics
    grid = geometry.StructuredGrid(9)
    g = geometry.generate_graph(geometry.GraphFamilySpec(n_branches=5), 3)
    params = assembly.PhysicalParams()
    s = assembly.assemble_coupled_system(grid, g, params)
    d = system_dict(s, restriction_for(grid, g, params, 1))
    d.update(csr_dict("K00", s.K00))
    d["dfield"] = geometry.distance_field(g, grid).values
    d["graph_vertices"] = g.vertices
    d["graph_edges"] = g.edges
    dump("asm_n9_family", **d)

    # (2) cfg1 semantics under reference blocks: n=17 segment, m=32, R=0.02, beta=1
    assembly.refine_graph = fixed_refine(32)
    try:
        for nc in (1, 8):
            grid = geometry.StructuredGrid(17)
            g = geometry.Graph1D(np.array([[0.5, 0.5, 0.1], [0.5, 0.5, 0.9]]), np.array([[0, 1]]),
                                 0.02, (0,))
            params = BetaParams(epsilon=0.02, beta=1.0)
            s = assembly.assemble_coupled_system(grid, g, params, n_circle=nc)
            d = system_dict(s, restriction_for(grid, g, params, nc))
            dump(f"asm_cfg1_nc{nc}", **d)
    finally:
        assembly.refine_graph = _ORIG_REFINE

    # (3) cfg2 semantics: n=33, 8-segment BASELINE tree seed 1, m=16, R=0.015, beta=1
    assembly.refine_graph = fixed_refine(16)
    try:
        for nc in (1, 8):
            grid = geometry.StructuredGrid(33)
            t = random_tree(8, 1, 0.015)
            g = geometry.Graph1D(t.vertices, t.edges, 0.015, (0,))
            params = BetaParams(epsilon=0.015, beta=1.0)
            s = assembly.assemble_coupled_system(grid, g, params, n_circle=nc)
            d = system_dict(s, restriction_for(grid, g, params, nc))
            d["tree_vertices"] = t.vertices
            d["tree_edges"] = t.edges
            dump(f"asm_cfg2_nc{nc}", **d)
    finally:
        assembly.refine_graph = _ORIG_REFINE


def random_spd(n, seed, shift=None):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    return sp.csr_matrix(A @ A.T + (shift if shift is not None else n) * np.eye(n))


def gen_fgmres():
    cases = {}
    specs = [
        ("identity", sp.identity(40, format="csr"), np.linspace(1, 2, 40), None, dict()),
        ("spd_mgs", random_spd(80, 5, shift=10), np.random.default_rng(6).standard_normal(80), None,
         dict(restart=30, tol=1e-12, maxit=30)),
        ("restart5", random_spd(120, 9, shift=1.0), np.random.default_rng(10).standard_normal(120), "x0",
         dict(restart=5, tol=1e-8, maxit=5000)),
        ("maxit8", random_spd(100, 12, shift=0.5), np.random.default_rng(13).standard_normal(100), None,
         dict(restart=5, tol=1e-14, maxit=8)),
        ("ilu_prec", random_spd(60, 7), np.random.default_rng(8).standard_normal(60), "ilu",
         dict(tol=1e-9)),
        ("breakdown_I", sp.identity(10, format="csr"), np.ones(10), None, dict(tol=1e-12)),
        ("zero_map", random_spd(30, 2), np.ones(30), "zero", dict(restart=5, maxit=12)),
    ]
    out = {}
    for name, A, b, extra, kw in specs:
        x0 = None
        pre = None
        if extra == "x0":
            x0 = np.random.default_rng(11).standard_normal(A.shape[0])
            out[f"{name}_x0"] = x0
        elif extra == "ilu":
            pre = krylov.IluPreconditioner(A)
        elif extra == "zero":
            pre = lambda r: np.zeros_like(r)  # noqa: E731
        x, rep = krylov.fgmres(A, pre, b, x0=x0, **kw)
        out[f"{name}_A"] = A.toarray()
        out[f"{name}_b"] = b
        out[f"{name}_x"] = x
        out[f"{name}_iters"] = np.array(rep.iterations)
        out[f"{name}_conv"] = np.array(rep.converged)
        out[f"{name}_hist"] = np.array(rep.residual_history)
        out[f"{name}_brk"] = np.array(rep.breakdowns)
        cases[name] = kw
    out["names"] = np.array(list(cases))
    out["kw"] = np.array([repr(cases[k]) for k in cases])
    dump("fgmres_cases", **out)


def noisy_params(seed=0, scale=0.05):
    params = neural.init_unet_params(seed)
    rng = np.random.default_rng(seed + 999)
    for key, arr in params.arrays():
        params.set_array(key, arr + scale * rng.standard_normal(arr.shape))
    return params


def gen_unet():
    out = {}
    for seed in (0, 1):
        p = neural.init_unet_params(seed)
        q = noisy_params(seed)
        for key, arr in p.arrays():
            out[f"init{seed}_{key}_sum"] = np.array(arr.sum())
            out[f"init{seed}_{key}_head"] = arr.ravel()[:6].copy()
        for key, arr in q.arrays():
            out[f"noisy{seed}_{key}_sum"] = np.array(arr.sum())
            out[f"noisy{seed}_{key}_head"] = arr.ravel()[:6].copy()
    q = noisy_params(0)
    rng = np.random.default_rng(77)
    for n in (9, 13, 17):
        x = rng.standard_normal((2, n, n, n))
        x[1] = np.abs(x[1]) * 0.3
        out[f"x_n{n}"] = x
        out[f"y_n{n}"] = neural.unet_forward(q, x)
    xb = rng.standard_normal((3, 2, 9, 9, 9))
    out["xb"] = xb
    out["yb"] = neural.unet_forward(q, xb)
    # layer-level pins
    xc = rng.standard_normal((1, 5, 11, 11, 11))
    kc = rng.standard_normal((4, 5, 3, 3, 3))
    bc = rng.standard_normal(4)
    out["conv_x"], out["conv_k"], out["conv_b"] = xc, kc, bc
    out["conv_y"] = neural.conv3d(xc, kc, bc)
    xt = rng.standard_normal((1, 3, 5, 5, 5))
    kt = rng.standard_normal((3, 2, 2, 2, 2))
    bt = rng.standard_normal(2)
    out["tconv_x"], out["tconv_k"], out["tconv_b"] = xt, kt, bt
    out["tconv_y0"] = neural.transposed_conv3d(xt, kt, output_padding=0, bias=bt)
    out["tconv_y1"] = neural.transposed_conv3d(xt, kt, output_padding=1, bias=bt)
    xp = rng.standard_normal((1, 3, 7, 9, 8))
    out["pool_x"] = xp
    out["pool_y"] = neural.maxpool3d(xp)[0]
    dump("unet_forward", **out)


def gen_apply_and_solve():
    # reference apply path and coupled solve on the reference n=9 family graph,
    # weights f32-rounded through an MDU3 checkpoint exactly as build_preconditioner loads them
    grid = geometry.StructuredGrid(9)
    g = geometry.generate_graph(geometry.GraphFamilySpec(n_branches=5), 3)
    params = assembly.PhysicalParams()
    s = assembly.assemble_coupled_system(grid, g, params)
    C = assembly.reduced_operator(s)
    out = {}
    with tempfile.TemporaryDirectory() as td:
        ck = Path(td) / "noisy0.mdu3"
        neural.save_checkpoint(noisy_params(0), ck)
        import hashlib
        out["ckpt_sha256"] = np.array(hashlib.sha256(ck.read_bytes()).hexdigest())
        pr = neural.load_checkpoint(ck)
        dfield = harness._dfield_from_system(s)
        out["dfield_mesh"] = dfield.values
        rng = np.random.default_rng(5)
        r = rng.standard_normal(grid.num_nodes)
        out["r"] = r
        out["z_plain"] = training.apply_neural(pr, r, dfield)
        out["z_smooth"] = training.apply_neural(pr, r, dfield, smoothing=(2, 2.0 / 3.0), C=C)
        rs = [rng.standard_normal(grid.num_nodes) for _ in range(3)] + [np.zeros(grid.num_nodes)]
        out["rs"] = np.array(rs)
        out["zs_batched"] = np.array(training.apply_batched(pr, rs, [dfield] * 4))
        for label, spec in (("none", {"type": "none"}), ("ilu0", {"type": "ilu0"}),
                            ("neural_s", {"type": "neural", "checkpoint": str(ck),
                                          "smoothing": {"maxit": 2}})):
            st = harness.CoupledStrategy(tol=1e-6, maxit=120, restart=30, inner_iterations=3,
                                         one_d="ilu0", three_d=spec)
            u3, u1, rep = harness.solve_coupled(s, st)
            out[f"solve_{label}_iters"] = np.array(rep.iterations)
            out[f"solve_{label}_conv"] = np.array(rep.converged)
            out[f"solve_{label}_hist"] = np.array(rep.residual_history)
            out[f"solve_{label}_u3"] = u3
            out[f"solve_{label}_u1"] = u1
            print(label, rep.iterations, rep.converged, rep.rel_residual)
    dump("apply_solve_n9", **out)


def gen_cfg1_solve():
    # config 1 under reference blocks (Neumann, m=32, R=0.02, beta=1, n_circle 8),
    # noisy seed-0 CNN via MDU3, Jacobi(2, 2/3) smoothing -- SURVEY P13
    assembly.refine_graph = fixed_refine(32)
    try:
        grid = geometry.StructuredGrid(17)
        g = geometry.Graph1D(np.array([[0.5, 0.5, 0.1], [0.5, 0.5, 0.9]]), np.array([[0, 1]]),
                             0.02, (0,))
        params = BetaParams(epsilon=0.02, beta=1.0)
        s = assembly.assemble_coupled_system(grid, g, params, n_circle=8)
        out = {}
        with tempfile.TemporaryDirectory() as td:
            ck = Path(td) / "noisy0.mdu3"
            neural.save_checkpoint(noisy_params(0), ck)
            for label, spec in (("neural_s", {"type": "neural", "checkpoint": str(ck),
                                              "smoothing": {"maxit": 2}}),
                                ("none", {"type": "none"})):
                st = harness.CoupledStrategy(tol=1e-6, maxit=300, restart=30, inner_iterations=3,
                                             one_d="ilu0", three_d=spec)
                u3, u1, rep = harness.solve_coupled(s, st)
                out[f"{label}_iters"] = np.array(rep.iterations)
                out[f"{label}_conv"] = np.array(rep.converged)
                out[f"{label}_hist"] = np.array(rep.residual_history)
                out[f"{label}_u3"] = u3
                out[f"{label}_u1"] = u1
                print("cfg1", label, rep.iterations, rep.converged, rep.rel_residual, rep.wall_time)
        dump("solve_cfg1", **out)
    finally:
        assembly.refine_graph = _ORIG_REFINE


def gen_direct():
    # one_d="direct" (harness.py:356-358: splu of A11) on the reference n=9 family graph:
    # the exact 1D solve of seeded vectors and two coupled solves with it
    import scipy.sparse.linalg as spla
    grid = geometry.StructuredGrid(9)
    g = geometry.generate_graph(geometry.GraphFamilySpec(n_branches=5), 3)
    s = assembly.assemble_coupled_system(grid, g, assembly.PhysicalParams())
    A11 = assembly.one_d_operator(s)
    rng = np.random.default_rng(11)
    r1 = rng.standard_normal((3, s.n1))
    lu = spla.splu(A11.tocsc())
    out = {"r1": r1, "z1": np.array([lu.solve(r) for r in r1])}
    for label, spec in (("none", {"type": "none"}), ("ilu0", {"type": "ilu0"})):
        st = harness.CoupledStrategy(tol=1e-6, maxit=120, restart=30, inner_iterations=3,
                                     one_d="direct", three_d=spec)
        u3, u1, rep = harness.solve_coupled(s, st)
        out[f"solve_{label}_iters"] = np.array(rep.iterations)
        out[f"solve_{label}_conv"] = np.array(rep.converged)
        out[f"solve_{label}_hist"] = np.array(rep.residual_history)
        out[f"solve_{label}_u3"] = u3
        out[f"solve_{label}_u1"] = u1
        print("direct", label, rep.iterations, rep.converged, rep.rel_residual)
    dump("direct_n9", **out)


def gen_formats():
    # interchange files written by the reference (geometry.py:306-363, training.py:361-393)
    grid = geometry.StructuredGrid(9)
    g = geometry.generate_graph(geometry.GraphFamilySpec(n_branches=5), 3)
    d = geometry.distance_field(g, grid)
    rng = np.random.default_rng(21)
    vecs = rng.standard_normal((3, grid.num_nodes))
    vecs /= np.linalg.norm(vecs, axis=1, keepdims=True)  # samples live on the unit sphere
    tags = ["physics", "krylov", "random"]
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        geometry.save_graph(g, td / "g.json")
        geometry.save_distance_field(d, td / "d.bin")
        training._write_samples(td / "s.bin", [training.TrainingSample(v, t, 0) for v, t in zip(vecs, tags)])
        out = {name: np.frombuffer((td / name).read_bytes(), dtype=np.uint8).copy()
               for name in ("g.json", "d.bin", "s.bin")}
    dump("formats_n9", graph_json=out["g.json"], mdf1=out["d.bin"], mds1=out["s.bin"], vecs=vecs,
         tags=np.array(tags), dvalues=d.values, vertices=g.vertices, edges=g.edges,
         radius=np.array(g.radius), dirichlet=np.array(g.dirichlet_vertices))


def gen_gmg():
    # geometric multigrid baseline (krylov.py:302-387) on reduced operators of two coupled systems
    out = {}
    cases = [("n9", geometry.StructuredGrid(9), geometry.generate_graph(geometry.GraphFamilySpec(n_branches=5), 3),
              assembly.PhysicalParams(), 3)]
    try:
        g17 = geometry.Graph1D(np.array([[0.5, 0.5, 0.1], [0.5, 0.5, 0.9]]), np.array([[0, 1]]), 0.02, (0,))
        cases.append(("n17", geometry.StructuredGrid(17), g17, BetaParams(epsilon=0.02, beta=1.0), 4))
        for tag, grid, g, params, levels in cases:
            # cfg1 geometry: 32 elements on the segment (fixed refinement); n9: the reference refinement
            assembly.refine_graph = fixed_refine(32) if tag == "n17" else _ORIG_REFINE
            s = assembly.assemble_coupled_system(grid, g, params, n_circle=8 if tag == "n17" else 1)
            C = assembly.reduced_operator(s).tocsr()
            hier = krylov.gmg_build(grid, C, levels)
            rng = np.random.default_rng(31)
            r = rng.standard_normal(grid.num_nodes)
            out[f"{tag}_r"] = r
            out[f"{tag}_vcycle"] = krylov.gmg_vcycle(hier, r)
            out[f"{tag}_vcycle_22"] = krylov.gmg_vcycle(hier, r, n_pre=2, n_post=2)
            out[f"{tag}_apply3"] = krylov.GmgPreconditioner(hier, cycles=3).apply(r)
            b = rng.standard_normal(grid.num_nodes)
            out[f"{tag}_b"] = b
            x, rep = krylov.fgmres(C, krylov.GmgPreconditioner(hier, cycles=2), b, restart=20, tol=1e-8, maxit=200)
            out[f"{tag}_iters"] = np.array(rep.iterations)
            out[f"{tag}_hist"] = np.array(rep.residual_history)
            out[f"{tag}_x"] = x
            out[f"{tag}_coarse_nnz"] = np.array([M.nnz for M in hier.matrices])
            if tag == "n9":  # coupled solve with the gmg inner preconditioner (harness.py:218-221, 377-387)
                st = harness.CoupledStrategy(tol=1e-6, maxit=60, restart=30, inner_iterations=3, one_d="ilu0",
                                             three_d={"type": "gmg", "cycles": 2, "levels": levels})
                u3, u1, crep = harness.solve_coupled(s, st)
                out["coupled_iters"] = np.array(crep.iterations)
                out["coupled_conv"] = np.array(crep.converged)
                out["coupled_hist"] = np.array(crep.residual_history)
                out["coupled_u3"] = u3
                print("gmg coupled", crep.iterations, crep.converged)
            print("gmg", tag, rep.iterations, rep.converged, [M.shape[0] for M in hier.matrices])
    finally:
        assembly.refine_graph = _ORIG_REFINE
    dump("gmg", **out)


def gen_ilu3d():
    # the 3D ILU(0) baseline on a reduced operator too large for the shared-memory sweep (33^3)
    grid = geometry.StructuredGrid(33)
    g = geometry.generate_graph(geometry.GraphFamilySpec(n_branches=5), 3)
    s = assembly.assemble_coupled_system(grid, g, assembly.PhysicalParams())
    C = assembly.reduced_operator(s).tocsr()
    f = krylov.ilu0(C)
    rng = np.random.default_rng(41)
    r = rng.standard_normal(grid.num_nodes)
    b = rng.standard_normal(grid.num_nodes)
    x, rep = krylov.fgmres(C, krylov.IluPreconditioner(C), b, restart=30, tol=1e-8, maxit=300)
    print("ilu3d", rep.iterations, rep.converged)
    dump("ilu3d_n33", r=r, z=krylov.ilu0_apply(f, r), b=b, iters=np.array(rep.iterations),
         hist=np.array(rep.residual_history), vertices=g.vertices, edges=g.edges,
         dirichlet=np.array(g.dirichlet_vertices))


def gen_training():
    # dataset build + FP64 training (training.py:124-287) on the reference tests' small dataset
    # (tests/test_training.py:31-40): 5 family graphs at n = 9, random augmentation
    grid, params = geometry.StructuredGrid(9), assembly.PhysicalParams()
    graphs = [geometry.generate_graph(geometry.GraphFamilySpec(n_branches=3 + 4 * i), 50 + i) for i in range(5)]
    ds = training.build_dataset(grid, graphs, params, training.AugmentationSpec("random", 4), val_fraction=0.2, seed=0)
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for i, g in enumerate(graphs):
            geometry.save_graph(g, Path(td) / "g.json")
            out[f"graph{i}"] = np.frombuffer((Path(td) / "g.json").read_bytes(), dtype=np.uint8).copy()
    out["samples"] = np.stack([np.stack([s.vector for s in r.samples]) for r in ds.records])
    out["tags"] = np.array([[s.tag for s in r.samples] for r in ds.records])
    out["train_indices"], out["val_indices"] = np.array(ds.train_indices), np.array(ds.val_indices)
    alpha = training.compute_alpha(ds)
    out["alpha"] = np.array(alpha)
    out["risk_init1"] = np.array(training.risk(neural.init_unet_params(1), ds, ds.train_samples(), alpha))
    s0 = assembly.assemble_coupled_system(grid, graphs[0], params)
    b0 = training.generate_rhs(s0)
    out["rhs0"] = b0
    out["krylov0"] = np.stack(training.augment_krylov(assembly.reduced_operator(s0), b0, 4, 5))
    dk = training.build_dataset(grid, graphs[:2], params, training.AugmentationSpec("krylov", 3, 2), val_fraction=0.5,
                                seed=4)
    out["krylov_samples"] = np.stack([np.stack([s.vector for s in r.samples]) for r in dk.records])
    p, hist = training.train(ds, training.TrainConfig(epochs=2, seed=0))
    out["history"] = np.array(hist)
    for key, arr in p.arrays():
        out[f"sum:{key}"] = np.array([arr.sum(), (arr * arr).sum()])
    for key in ("head2.kernel", "head2.bias", "head1.bias", "enc1a.bias", "dec1.bias"):
        out[f"p:{key}"] = dict(p.arrays())[key]
    print("training history", hist)
    dump("training_n9", **out)


def gen_exact():
    # exact baselines: ExactPreconditioner (krylov.py:54-61), three_d="direct" and one_d="schur"
    # (harness.py:356-375) on the reference tests' single-segment system (tests/test_harness.py:26-30,
    # 176-187, 207-219) and the n = 9 family system
    import scipy.sparse.linalg as spla
    grid = geometry.StructuredGrid(9)
    out = {}

    def seg(eps):
        g = geometry.Graph1D(np.array([[0.31, 0.42, 0.11], [0.58, 0.63, 0.87]]), np.array([[0, 1]]), eps, (0,))
        return assembly.assemble_coupled_system(grid, g, assembly.PhysicalParams(epsilon=eps))

    s = seg(1e-3)
    C = assembly.reduced_operator(s)
    w = s.params.coupling_weight
    lu_c0 = spla.splu(C.tocsc())
    coupling = np.column_stack([lu_c0.solve(col) for col in (w * s.M01).toarray().T])
    out["seg_schur"] = assembly.one_d_operator(s).toarray() - (w * s.M10).toarray() @ coupling
    for label, one_d in (("schur", "schur"), ("direct", "direct")):
        st = harness.CoupledStrategy(tol=1e-12, maxit=50, one_d=one_d, three_d="direct")
        u3, u1, rep = harness.solve_coupled(s, st)
        out[f"seg_{label}_iters"] = np.array(rep.iterations)
        out[f"seg_{label}_hist"] = np.array(rep.residual_history)
        out[f"seg_{label}_u3"], out[f"seg_{label}_u1"] = u3, u1
        print("exact seg", label, rep.iterations, rep.rel_residual)
    for eps in (1e-6, 1e-9):
        u3, _, rep = harness.solve_coupled(seg(eps), harness.CoupledStrategy(tol=1e-12, maxit=50, one_d="direct",
                                                                              three_d="direct"))
        out[f"vanish_{eps:g}_norm"] = np.array(np.linalg.norm(u3))
        out[f"vanish_{eps:g}_iters"] = np.array(rep.iterations)
    g = geometry.generate_graph(geometry.GraphFamilySpec(n_branches=5), 3)
    f = assembly.assemble_coupled_system(grid, g, assembly.PhysicalParams())
    Cf = assembly.reduced_operator(f)
    r = np.random.default_rng(5).standard_normal((2, f.n3))
    out["fam_r"], out["fam_z"] = r, np.array([krylov.ExactPreconditioner(Cf).apply(v) for v in r])
    st = harness.CoupledStrategy(tol=1e-8, maxit=60, restart=30, inner_iterations=3, one_d="ilu0",
                                 three_d={"type": "exact"})
    u3, u1, rep = harness.solve_coupled(f, st)
    out["fam_inner_exact_iters"] = np.array(rep.iterations)
    out["fam_inner_exact_hist"] = np.array(rep.residual_history)
    out["fam_inner_exact_u3"], out["fam_inner_exact_u1"] = u3, u1
    print("exact fam inner", rep.iterations, rep.rel_residual)
    dump("exact_n9", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["assembly", "fgmres", "unet", "apply", "cfg1", "direct", "formats", "gmg", "ilu3d", "training", "exact"]
    if "assembly" in which:
        gen_assembly()
    if "fgmres" in which:
        gen_fgmres()
    if "unet" in which:
        gen_unet()
    if "apply" in which:
        gen_apply_and_solve()
    if "cfg1" in which:
        gen_cfg1_solve()
    if "direct" in which:
        gen_direct()
    if "formats" in which:
        gen_formats()
    if "gmg" in which:
        gen_gmg()
    if "ilu3d" in which:
        gen_ilu3d()
    if "training" in which:
        gen_training()
    if "exact" in which:
        gen_exact()

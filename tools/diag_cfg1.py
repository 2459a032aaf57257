"""Diagnostic: cfg1 (reference semantics) coupled solve with the TF32 and FP32 CNN paths vs the reference golden."""
import sys, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import golden
from paper_2505_08491_b200 import assembly as A, geometry as G, harness, neural
g = golden("solve_cfg1")
graph = G.Graph1D([[0.5, 0.5, 0.1], [0.5, 0.5, 0.9]], [[0, 1]], 0.02, (0,))
s = A.assemble_coupled_system(G.StructuredGrid(17), graph, A.PhysicalParams(epsilon=0.02, beta=1.0), n_circle=8, elems_per_edge=32)
import tempfile, os
d = tempfile.mkdtemp(); pth = os.path.join(d, "p.mdu3")
neural.save_checkpoint(neural.perturbed_params(0), pth)
p = neural.load_checkpoint(pth)
ref = g["neural_s_hist"]
print("ref iters", int(g["neural_s_iters"]), "hist[:8]", np.array2string(ref[:8], precision=6))
for path in (1, 0):
    spec = {"type": "neural", "params": p, "smoothing": {"maxit": 2}, "path": path}
    st = harness.CoupledStrategy(tol=1e-6, maxit=400, restart=30, inner_iterations=3, three_d=spec)
    u3, u1, rep = harness.solve_coupled(s, st)
    h = np.array(rep.residual_history)
    k = min(len(h), len(ref)) - 1
    print(f"path {path}: iters {rep.iterations} conv {rep.converged} rel {rep.rel_residual:.3e}")
    print("  hist[:8]", np.array2string(h[:8], precision=6))
    for j in (5, 10, 30, 60, 100, 150, 200, 260):
        if j < k:
            print(f"  it {j}: ours {h[j]:.4e} ref {ref[j]:.4e} ratio {h[j]/ref[j]:.4f}")
    print("  u3 rel diff", np.linalg.norm(u3 - g["neural_s_u3"]) / np.linalg.norm(g["neural_s_u3"]))

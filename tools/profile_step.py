"""One short cfg-N coupled solve for launch-list profiling (ncu)."""
import argparse, sys
sys.path.insert(0, ".")
import torch
from paper_2505_08491_b200 import configs, harness, neural

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--maxit", type=int, default=4)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
wl = configs.CONFIGS[a.workload]()
params = neural.perturbed_params(wl.cnn_seed)
spec = {"type": "neural", "params": params, "smoothing": {"maxit": 2, "omega": 2.0 / 3.0}}
st = harness.CoupledStrategy(tol=wl.tol, maxit=a.maxit, restart=wl.restart, inner_iterations=3, three_d=spec)
solver = harness.CoupledSolver(wl.systems, st)
for _ in range(a.reps):
    r = solver.solve()
torch.cuda.synchronize()
print("iters", [r[i].iterations for i in r])

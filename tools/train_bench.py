"""Time dataset construction and FP64 training on the GPU at the SURVEY P8 setting
(20 graphs at 17^3, eps = 0.02, beta = 1, random augmentation x4, 15 epochs, batch 5).

    python tools/train_bench.py [--n 17] [--graphs 20] [--epochs 15] [--out f.json]
Graphs are the seeded BASELINE random trees (radius 0.02); cost per sample does
not depend on the geometry."""
import argparse, json, sys, time
sys.path.insert(0, ".")
import torch
from paper_2505_08491_b200 import assembly as A, geometry as G, training as T

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=17)
ap.add_argument("--graphs", type=int, default=20)
ap.add_argument("--epochs", type=int, default=15)
ap.add_argument("--out", default="")
a = ap.parse_args()
grid = G.StructuredGrid(a.n)
params = A.PhysicalParams(epsilon=0.02, beta=1.0)
graphs = [G.random_tree(8, 100 + i, 0.02) for i in range(a.graphs)]
torch.cuda.synchronize()
t0 = time.perf_counter()
ds = T.build_dataset(grid, graphs, params, T.AugmentationSpec("random", 4), val_fraction=0.2, seed=0)
torch.cuda.synchronize()
t1 = time.perf_counter()
T.train(ds, T.TrainConfig(epochs=1, seed=0))  # warm-up (cuDNN plans, allocator)
torch.cuda.synchronize()
t2 = time.perf_counter()
p, hist = T.train(ds, T.TrainConfig(epochs=a.epochs, seed=0))
torch.cuda.synchronize()
t3 = time.perf_counter()
line = {"n": a.n, "graphs": a.graphs, "epochs": a.epochs, "train_samples": len(ds.train_samples()),
        "dataset_s": t1 - t0, "train_s": t3 - t2, "s_per_epoch": (t3 - t2) / a.epochs,
        "loss_first": hist[0], "loss_last": hist[-1], "device": torch.cuda.get_device_name(0)}
print(json.dumps(line))
if a.out:
    open(a.out, "w").write(json.dumps(line, indent=1) + "\n")

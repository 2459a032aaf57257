"""Build-container only (imports the reference read-only): time the reference's
CPU build_dataset + train on the same graphs and settings as tools/train_bench.py.

    python tools/train_ref_cpu.py [--n 17] [--graphs 20] [--epochs 2]"""
import argparse, dataclasses, json, os, sys, time
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ".")
from mdprec import assembly, geometry, training  # noqa: E402
from paper_2505_08491_b200 import geometry as G  # noqa: E402  (BASELINE seeded trees)


@dataclasses.dataclass(frozen=True)
class BetaParams(assembly.PhysicalParams):
    beta: float = 1.0

    @property
    def coupling_weight(self):
        return self.beta


ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=17)
ap.add_argument("--graphs", type=int, default=20)
ap.add_argument("--epochs", type=int, default=2)
a = ap.parse_args()
grid = geometry.StructuredGrid(a.n)
graphs = []
for i in range(a.graphs):
    g = G.random_tree(8, 100 + i, 0.02)
    graphs.append(geometry.Graph1D(g.vertices, g.edges, g.radius, tuple(g.dirichlet_vertices)))
t0 = time.perf_counter()
ds = training.build_dataset(grid, graphs, BetaParams(epsilon=0.02), training.AugmentationSpec("random", 4),
                            val_fraction=0.2, seed=0)
t1 = time.perf_counter()
p, hist = training.train(ds, training.TrainConfig(epochs=a.epochs, seed=0))
t2 = time.perf_counter()
print(json.dumps({"n": a.n, "graphs": a.graphs, "epochs": a.epochs, "dataset_s": t1 - t0, "train_s": t2 - t1,
                  "s_per_epoch": (t2 - t1) / a.epochs, "history": hist, "cpu_threads": os.cpu_count()}))

"""Paper Table 9 on the B200 (harness.run_batch_bench, harness.py:524-561): serial vs
batched CNN preconditioner passes at 21^3 for batch sizes 1/10/50/100.

    python tools/batch_bench.py [--out profiles/r01_batch_bench_21.json]

Same protocol as the reference: wall-clock around the public host-vector calls
(training.apply_neural per residual vs one training.apply_batched), outputs must
agree to 1e-12 (ours are bitwise equal).  Residuals: seeded unit vectors, distance
fields of seeded random trees (synthetic; the paper's graph pool is not shipped).
Also reported: device time of the batched forward alone (CUDA events).
The paper's numbers (V100, input (B, 2, 21^3)):
batched 1.5 / 4.1 / 13.5 / 25.5 ms, serial 1.5 / 11.8 / 58.2 / 114.9 ms.
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2505_08491_b200 import geometry as G, neural, training

PAPER = {1: (1.5, 1.5), 10: (11.8, 4.1), 50: (58.2, 13.5), 100: (114.9, 25.5)}  # (serial, batched) ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=21)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    grid = G.StructuredGrid(a.n)
    params = neural.perturbed_params(0)
    rng = np.random.default_rng(9)
    pool = []
    for i in range(16):
        r = rng.standard_normal(grid.num_nodes)
        pool.append((r / np.linalg.norm(r), G.distance_field(G.random_tree(8, 100 + i, 0.02), grid)))
    rows = []
    for B in (1, 10, 50, 100):
        rs = [pool[i % len(pool)][0] for i in range(B)]
        ds = [pool[i % len(pool)][1] for i in range(B)]
        training.apply_batched(params, rs, ds)  # warm (weights upload, workspace)
        [training.apply_neural(params, r, d) for r, d in zip(rs[:2], ds[:2])]
        torch.cuda.synchronize()
        ts, tb = [], []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            serial = [training.apply_neural(params, r, d) for r, d in zip(rs, ds)]
            ts.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            batched = training.apply_batched(params, rs, ds)
            tb.append(time.perf_counter() - t0)
        dev = max(float(np.max(np.abs(x - y))) for x, y in zip(serial, batched))
        assert dev <= 1e-12, dev
        # device time of the batched forward alone
        net = neural.device_net(params)
        n3 = grid.num_nodes
        R = torch.as_tensor(np.array(rs), device="cuda")
        D = torch.as_tensor(np.array([d.values for d in ds]), device="cuda")
        rn = torch.ones(B, dtype=torch.float64, device="cuda")
        Z = torch.empty_like(R)
        net.apply(a.n, R, n3, rn, D, n3, Z, n3, nb=B)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            net.apply(a.n, R, n3, rn, D, n3, Z, n3, nb=B)
        e.record()
        e.synchronize()
        row = {"batch": B, "time_serial_ms": 1e3 * float(np.median(ts)), "time_batched_ms": 1e3 * float(np.median(tb)),
               "speedup": float(np.median(ts) / np.median(tb)), "max_deviation": dev,
               "device_batched_forward_ms": s.elapsed_time(e) / 20,
               "paper_v100_serial_ms": PAPER[B][0], "paper_v100_batched_ms": PAPER[B][1]}
        row["vs_paper_batched"] = row["paper_v100_batched_ms"] / row["time_batched_ms"]
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        open(a.out, "w").write(json.dumps({"n": a.n, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()

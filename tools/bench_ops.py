"""BASELINE config 5: operator microbenchmark sweep (no solve).

Grids n in {33, 65, 129, 193} x batch {1, 8, 64} of seeded 32-segment trees.
Timed separately (CUDA events, L2 flushed -- written, then read back -- before
every timed rep): the K00 stencil alone, the coupled block SpMV, Pi gather, Pi^T scatter (pull), 30-vector Arnoldi
orthogonalisation, and the CNN preconditioner forward.  Algorithmic bytes /
FLOPs per SURVEY.md section 8d; peaks from MEASURED_PEAKS.json (HBM; TF32 = bf16 / 2, the
cuBLAS TF32 GEMM rate of the same run is recorded beside it).  The stencil and the coupled SpMV
are also timed streamed over rotating vector pairs; the gather / scatter rows carry the
launch + event floor of the timing method (a 1-element kernel).

    python tools/bench_ops.py [--sizes 33,65,129,193] [--batches 1,8,64] [--out f.json]
                              [--cpu-sizes 33,65,129] [--cpu-cnn-max 65]

--cpu-sizes: also time the CPU oracle (the reference path restated in
numpy/scipy, same seeded batch-1 system) per operator on the host cores:
full_operator @ x, T @ x3, T^T v, a 30-vector MGS step (krylov.py:138-140)
and the U-Net forward (n <= --cpu-cnn-max).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_08491_b200 import _ext, configs, neural  # noqa: E402


def timed(fn, reps, flush):
    """Cold-L2 median device time; host enqueue hidden behind a GPU sleep (bench.device_ms)."""
    return bench.device_ms(fn, reps, flush=flush, hide_us=2000)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="33,65,129,193")
    ap.add_argument("--batches", default="1,8,64")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--mem-gb", type=float, default=120.0)
    ap.add_argument("--out", default="")
    ap.add_argument("--cpu-sizes", default="")
    ap.add_argument("--cpu-cnn-max", type=int, default=65)
    a = ap.parse_args()
    lib = _ext.lib()
    pk = bench.peaks()
    cublas_tf32 = bench.measure_tf32_peak()
    tf32 = pk["bf16_tflops"] / 2  # kind::tf32 = half the dense bf16 rate (MEASURED_PEAKS); cuBLAS TF32 is a note
    flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")
    one = torch.zeros(1, device="cuda")
    floor_ms = bench.device_ms(lambda: one.add_(1.0), 10, flush=flush, hide_us=2000)  # launch + event floor
    from paper_2505_08491_b200.assembly import DeviceProblem
    from paper_2505_08491_b200.operators import CoupledOperator, CouplingOps
    rows = []
    net = neural.DeviceUNet(neural.perturbed_params(4))
    for n in [int(x) for x in a.sizes.split(",")]:
        for nb in [int(x) for x in a.batches.split(",")]:
            n3 = n ** 3
            # memory guard: vectors + CNN workspace
            est = nb * (n3 * 8 * 40 + lib.mdp_unet_workspace_bytes(n, 1, 0))
            if est > a.mem_gb * 1e9:
                rows.append({"n": n, "batch": nb, "skipped": f"needs ~{est / 1e9:.0f} GB"})
                continue
            t0 = time.time()
            systems = configs.cfg5_systems(n, nb)
            prob = DeviceProblem(systems)
            A = CoupledOperator(prob)
            ops = CouplingOps(prob)
            X = prob.zeros().normal_()
            Y = prob.zeros()
            N = [n3 + int(x) for x in prob.n1]
            Q = prob.Qtot
            U = int(prob._t["u_start"][-1].item())
            r = {"n": n, "batch": nb, "Q_total": Q, "setup_s": round(time.time() - t0, 2)}
            ms = timed(lambda: ops.stencil(X, Y), a.reps, flush)
            byt = 16 * n3 * nb
            r["stencil"] = {"ms": ms, "GBps": byt / (ms * 1e-3) / 1e9, "frac_hbm": byt / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                            "frac_hbm_spec_8tbs": byt / (ms * 1e-3) / 8e12, "bytes": byt,
                            "kernel": "stencil3_kernel (K00 alone)"}
            ms = timed(lambda: A.matvec(X, Y), a.reps, flush)
            byt = sum(16 * x for x in N) + 40 * Q
            r["spmv"] = {"ms": ms, "GBps": byt / (ms * 1e-3) / 1e9, "frac_hbm": byt / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                         "frac_hbm_spec_8tbs": byt / (ms * 1e-3) / 8e12, "bytes": byt}
            # the same launches streamed over rotating vector pairs (> 2x L2 in total), back to back
            nset = min(16, max(2, int(-(-2.5 * 126e6 // byt))))
            if nset * 2 * nb * prob.ld * 8 < 40e9:
                XS = [prob.zeros().normal_() for _ in range(nset)]
                YS = [prob.zeros() for _ in range(nset)]
                for key, fn in (("stencil", ops.stencil), ("spmv", A.matvec)):
                    sms = bench.device_ms_stream([(lambda X_=X_, Y_=Y_, fn=fn: fn(X_, Y_)) for X_, Y_ in zip(XS, YS)], 3)
                    r[key]["stream_ms"] = sms
                    r[key]["stream_frac_hbm"] = r[key]["bytes"] / (sms * 1e-3) / 1e9 / pk["hbm_gbs"]
                del XS, YS
            S = torch.zeros(max(Q, 1), dtype=torch.float64, device="cuda")
            ms = timed(lambda: ops.gather(X, None, S), a.reps, flush)
            byt = 112 * Q
            r["pi_gather"] = {"ms": ms, "GBps": byt / (ms * 1e-3) / 1e9, "bytes": byt, "launch_floor_ms": floor_ms}
            ms = timed(lambda: ops.scatter(S, 1.0, Y), a.reps, flush)
            byt = 48 * Q + 16 * U
            r["pi_scatter"] = {"ms": ms, "GBps": byt / (ms * 1e-3) / 1e9, "bytes": byt, "launch_floor_ms": floor_ms}
            # Arnoldi: 30 basis vectors (k = 30), orthogonalise w against all of them
            k = 30
            nmax = max(N)
            if nb * (k + 2) * prob.ld * 8 < 60e9:
                V = torch.randn((nb, k + 1, prob.ld), dtype=torch.float64, device="cuda")
                W = torch.randn((nb, prob.ld), dtype=torch.float64, device="cuda")
                H = torch.zeros((nb, k + 2), dtype=torch.float64, device="cuda")
                nv = torch.full((nb,), k, dtype=torch.int32, device="cuda")
                work = torch.zeros(lib.mdp_arnoldi_work_bytes(nb, k, nmax) // 8 + 1, dtype=torch.float64,
                                   device="cuda")

                gram = torch.zeros((nb, k + 1, k + 1), dtype=torch.float64, device="cuda")
                byt = (2 * k + 3) * nmax * 8 * nb
                for tag, gr, note in (("arnoldi30", gram, "one-pass MGS: V read 2x"),
                                      ("arnoldi30_cgs2", None, "CGS2: V read 3x")):
                    def arn():
                        _ext.check(lib.mdp_arnoldi(nb, None, V.data_ptr(), (k + 1) * prob.ld, prob.ld, nv.data_ptr(),
                                                   k, W.data_ptr(), prob.ld, nmax, H.data_ptr(), None, 0,
                                                   _ext.ptr(gr), work.data_ptr(), _ext.stream()))
                    ms = timed(arn, a.reps, flush)
                    r[tag] = {"ms": ms, "GBps": byt / (ms * 1e-3) / 1e9,
                              "frac_hbm": byt / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], "bytes": byt,
                              "note": note + "; bytes = survey formula (2k+3) N 8"}
                del V, W
            # CNN forward (pack -> U-Net -> rescale), batch nb
            D = torch.rand((nb, n3), dtype=torch.float64, device="cuda")
            R = X
            rn = torch.ones(nb, dtype=torch.float64, device="cuda")
            Z = prob.zeros()
            ms = timed(lambda: net.apply(n, R, prob.ld, rn, D, n3, Z, prob.ld, nb=nb), max(3, a.reps // 2), flush)
            fl = nb * neural_flops(n)
            r["cnn_forward"] = {"ms": ms, "TFLOPs": fl / (ms * 1e-3) / 1e12, "frac_tf32": fl / (ms * 1e-3) / 1e12 / tf32,
                                "flops": fl}
            rows.append(r)
            print(json.dumps(r), flush=True)
            del prob, A, ops, X, Y, S, D, Z, R
            torch.cuda.empty_cache()
    cpu = [cpu_row(int(n), a.cpu_cnn_max) for n in a.cpu_sizes.split(",") if n]
    out = {"peaks": pk, "tf32_peak_used": tf32, "cublas_tf32_tflops_this_run": cublas_tf32, "launch_floor_ms": floor_ms,
           "rows": rows, "cpu_oracle": cpu}
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1))


def cpu_row(n: int, cnn_max: int) -> dict:
    """The CPU oracle's per-operator times for the batch-1 cfg5 system at n (median of reps)."""
    import os
    import statistics
    import oracle
    from oracle import problem as OP

    def t(fn, reps):
        fn()  # warm (first calls pay allocation / BLAS start-up)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts) * 1e3

    R = min(0.005, 0.9 / (n - 1))
    t0 = time.perf_counter()
    o = OP.assemble_coupled_system(OP.StructuredGrid(n), OP.random_tree(32, 4000, R),
                                   OP.PhysicalParams(epsilon=R, beta=1.0), n_circle=8, elems_per_edge=16,
                                   bc3d="dirichlet", f1d=1.0)
    A = OP.full_operator(o)
    T = o.restriction.matrix
    rng = np.random.default_rng(n)
    x = rng.standard_normal(A.shape[0])
    v = rng.standard_normal(T.shape[0])
    V = rng.standard_normal((30, A.shape[0]))

    def mgs():  # krylov.py:138-140 for one Arnoldi step against 30 basis vectors
        w = x.copy()
        for i in range(30):
            h = float(w @ V[i])
            w -= h * V[i]
        return np.linalg.norm(w)

    row = {"n": n, "cores": len(os.sched_getaffinity(0)), "assembly_s": round(time.perf_counter() - t0, 2),
           "spmv_ms": t(lambda: A @ x, 5), "pi_gather_ms": t(lambda: T @ x[:o.n3], 5),
           "pi_scatter_ms": t(lambda: T.T @ v, 5), "mgs30_ms": t(mgs, 3)}
    if n <= cnn_max:
        xin = rng.standard_normal((1, 2, n, n, n))
        p = oracle.noisy_params(4)
        row["cnn_forward_ms"] = t(lambda: oracle.unet_forward(p, xin), 1)
    print(json.dumps({"cpu_oracle": row}), flush=True)
    return row


def neural_flops(n: int) -> float:
    m, q = n // 2, n // 4
    f = 0.0
    for name, op, cin, cout, ks, _ in neural.ARCHITECTURE:
        if op == "tconv":
            out = m ** 3 if name == "up2" else n ** 3  # survey convention: 2 * voxels_out * Cin * Cout
            f += 2.0 * out * cin * cout
        else:
            vox = {"enc3": m ** 3, "dec2": m ** 3, "bottleneck": q ** 3}.get(name, n ** 3)
            f += 2.0 * vox * cin * cout * ks ** 3
    return f


if __name__ == "__main__":
    main()

"""Benchmark of the neural-preconditioned coupled FGMRES solve on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg4]

A step is one full coupled solve (outer FGMRES(restart) with the ILU(0) 1D
block and the 3-step inner FGMRES on C preconditioned by the Jacobi(2,2/3)-
wrapped TF32 U-Net) of the workload's systems, inputs resident in HBM.
N > 1 (torchrun): every rank solves its own replica of the workload (the
path has no exchange step: replicas only); value is
the total solves/s over all ranks, timed on the device, max over ranks.

Extras on the one JSON line: roofline of the dominant kernel (the tcgen05
conv layer with the largest share), the coupled-SpMV HBM roofline, the
end-to-end drop-in API number (host buffers, copies inside the timed
region), the CPU oracle baseline, clocks sampled during the timed region,
and the number of our kernels launched.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "preconditioned FGMRES solves/sec + applies/sec at 1 B200; % HBM/tensor roofline"
# the e2e leg (drop-in API from host buffers) repeats the solve; at cfg4 a solve is
# ~15 s, so it is timed over at most this many steps
E2E_MAX_STEPS = 5


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while running."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def flush_l2(buf):
    buf.add_(1.0)  # 256 MiB write > 126 MB L2


def flush_l2_clean(buf):
    """Write-flush, then read the buffer back: L2 holds clean lines only, so no
    write-back of the flush's dirty lines lands inside a timed kernel."""
    buf.add_(1.0)
    buf.sum()


def device_ms(fn, reps=20, flush=None, hide_us=None):
    """Median device time (ms) of fn() over reps, CUDA events on the current stream.

    A GPU sleep queued ahead of each timed call keeps the device busy while the
    host enqueues fn (ctypes marshalling takes longer than a small kernel), so
    the events bracket device work only.  flush: L2-flush buffer written before
    every rep (cold-cache timing), else back-to-back warm reps.
    """
    import torch
    fn()
    torch.cuda.synchronize()
    cycles = int((hide_us or 400) * 2000)  # ~2 GHz
    ts = []
    if flush is None:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(cycles * reps)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        e.synchronize()
        return s.elapsed_time(e) / reps
    for _ in range(reps):
        flush_l2_clean(flush)
        torch.cuda._sleep(cycles)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def device_ms_stream(fns, reps=5):
    """Per-call device time (ms) of len(fns) calls on DIFFERENT buffers issued back to back
    (reps rounds inside one event pair).  The buffers together exceed 2x L2, so every call
    streams from HBM without an L2 flush and without a launch + event round trip per call:
    the in-solve condition (kernels follow each other in a CUDA graph)."""
    import torch
    for f in fns:
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(400 * 2000 * max(1, len(fns) * reps // 8)))
    s.record()
    for _ in range(reps):
        for f in fns:
            f()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / (reps * len(fns))


def spmv_stream_and_floors(prob, A, flush, nbytes):
    """Context for the single-launch coupled SpMV number at small byte counts: (1) the same launch
    streamed over rotating vector pairs (> 2x L2 in total), (2) a device copy of the same bytes timed
    exactly like the single launch (the practical ceiling of that method), (3) a 1-element kernel timed
    the same way (launch + event floor)."""
    import torch
    l2 = 126e6
    nset = max(2, int(-(-2.5 * l2 // max(nbytes, 1))))
    nset = min(nset, 64)
    XS = [prob.zeros().normal_() for _ in range(nset)]
    YS = [prob.zeros() for _ in range(nset)]
    ms = device_ms_stream([(lambda X=X, Y=Y: A.matvec(X, Y)) for X, Y in zip(XS, YS)])
    n = prob.zeros().numel()
    src, dst = torch.randn(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")
    copy_ms = device_ms(lambda: dst.copy_(src), 10, flush=flush)
    one = torch.zeros(1, device="cuda")
    floor_ms = device_ms(lambda: one.add_(1.0), 10, flush=flush)
    del XS, YS, src, dst
    return {"stream_ms": ms, "stream_GBps": nbytes / (ms * 1e-3) / 1e9, "stream_sets": nset,
            "copy_same_bytes_ms": copy_ms, "copy_same_bytes_GBps": 16 * n / (copy_ms * 1e-3) / 1e9,
            "launch_floor_ms": floor_ms,
            "context_note": "stream: rotating vector pairs (> 2x L2 in total) back to back in one event pair; copy / floor: "
                    "torch copy of the same vectors and a 1-element kernel timed like the single launch"}


def measure_tf32_peak():
    """cuBLAS TF32 GEMM 8192^3, best of 5 (the tensor-core denominator for kind::tf32)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(8192, 8192, device="cuda")
    b = torch.randn(8192, 8192, device="cuda")
    for _ in range(2):
        a @ b
    best = 0.0
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        e.synchronize()
        best = max(best, 2 * 8192 ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
    torch.backends.cuda.matmul.allow_tf32 = False
    del a, b
    return best


def conv_layer_times(n, reps=20):
    """Average device time of each tcgen05 conv layer of the forward at size n."""
    import numpy as np
    import torch
    from paper_2505_08491_b200 import _ext, neural
    lib = _ext.lib()
    m, q = n // 2, n // 4
    layers = [("enc1b", n, 16, 32, 0), ("enc2", n, 32, 64, 1), ("enc3", m, 64, 128, 1),
              ("bottleneck", q, 128, 128, 0), ("dec2", m, 128, 64, 0), ("dec1", n, 64, 32, 0)]
    out = {}
    rng = np.random.default_rng(0)
    for name, S, cin, cout, pool in layers:
        X = torch.as_tensor(rng.standard_normal(cin * S ** 3).astype(np.float32), device="cuda")
        W = torch.as_tensor(neural.pack_conv(rng.standard_normal((cout, cin, 3, 3, 3)) * 0.05, 0).ravel(),
                            device="cuda")
        So = S // 2 if pool else S
        Y = torch.empty(cout * So ** 3, dtype=torch.float32, device="cuda")
        scr = torch.zeros(max(lib.mdp_conv3_scratch_bytes(1, S, cin, cout), 16), dtype=torch.uint8, device="cuda")
        st = _ext.stream()

        def run():
            _ext.check(lib.mdp_conv3_layer(0, 1, S, cin, cout, X.data_ptr(), cin // 4, 0, W.data_ptr(), None, 1,
                                           Y.data_ptr(), cout // 4, 0, pool, scr.data_ptr(), scr.numel(), st))
        ms = device_ms(run, reps)
        flops = 2.0 * S ** 3 * cin * cout * 27
        out[name] = {"ms": ms, "flops": flops, "tflops": flops / (ms * 1e-3) / 1e12, "S": S}
    return out


def target_128(tf32_peak, hbm_peak, layers=None):
    """The north star's target configuration (BASELINE cfg4, 128^3 cells = 129^3
    nodes): conv layers vs the TF32 tensor peak, the CNN forward, and the
    coupled SpMV (L2 flushed before every rep) vs the HBM peak."""
    import torch
    from paper_2505_08491_b200 import configs, neural
    from paper_2505_08491_b200.operators import CoupledOperator
    from paper_2505_08491_b200.assembly import DeviceProblem
    n = 129
    layers = layers or conv_layer_times(n, reps=5)
    dom = max(layers, key=lambda k: layers[k]["ms"])
    stack_ms = sum(v["ms"] for v in layers.values())
    stack_fl = sum(v["flops"] for v in layers.values())
    net = neural.DeviceUNet(neural.perturbed_params(3))
    R = torch.randn((1, n ** 3), dtype=torch.float64, device="cuda")
    D = torch.rand((1, n ** 3), dtype=torch.float64, device="cuda")
    rn = torch.ones(1, dtype=torch.float64, device="cuda")
    Z = torch.empty_like(R)
    fwd_ms = device_ms(lambda: net.apply(n, R, n ** 3, rn, D, n ** 3, Z, n ** 3, nb=1), 5)
    fwd_fl = neural_forward_flops(n)
    del R, D, Z
    wl = configs.cfg4()
    prob = DeviceProblem(wl.systems)
    A = CoupledOperator(prob)
    X = prob.zeros().normal_()
    Y = prob.zeros()
    flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")
    sp_ms = device_ms(lambda: A.matvec(X, Y), 10, flush=flush)
    sp_bytes = sum(16 * (prob.n3 + int(n1)) for n1 in prob.n1) + 40 * prob.Qtot
    sp_ctx = spmv_stream_and_floors(prob, A, flush, sp_bytes)
    del prob, A, X, Y
    # the multi-query setting at 128^3 (8 seeded 32-segment trees, BASELINE cfg5 shapes):
    # the K00 stencil alone (16 B per node) and the whole coupled SpMV
    from paper_2505_08491_b200.operators import CouplingOps
    pb = DeviceProblem(configs.cfg5_systems(n, 8))
    A8, ops8 = CoupledOperator(pb), CouplingOps(pb)
    X8, Y8 = pb.zeros().normal_(), pb.zeros()
    st8_ms = device_ms(lambda: ops8.stencil(X8, Y8), 10, flush=flush)
    sp8_ms = device_ms(lambda: A8.matvec(X8, Y8), 10, flush=flush)
    st8_bytes = 16 * pb.n3 * pb.nsys
    sp8_bytes = sum(16 * (pb.n3 + int(n1)) for n1 in pb.n1) + 40 * pb.Qtot
    del pb, A8, ops8, X8, Y8
    out = {
        "config": "cfg4: 128^3 cells (129^3 nodes), 64-segment tree, 32 elements/segment",
        "conv_dominant": {"bound": "tensor", "kernel": f"conv3_tc_kernel ({dom})", "ms": layers[dom]["ms"],
                          "achieved": layers[dom]["tflops"], "peak": tf32_peak, "unit": "TFLOP/s",
                          "frac": layers[dom]["tflops"] / tf32_peak},
        "conv_stack": {"ms": stack_ms, "achieved": stack_fl / (stack_ms * 1e-3) / 1e12,
                       "frac": stack_fl / (stack_ms * 1e-3) / 1e12 / tf32_peak, "unit": "TFLOP/s",
                       "layers": {k: round(v["tflops"], 1) for k, v in layers.items()}},
        "cnn_forward": {"ms": fwd_ms, "achieved": fwd_fl / (fwd_ms * 1e-3) / 1e12,
                        "frac": fwd_fl / (fwd_ms * 1e-3) / 1e12 / tf32_peak, "unit": "TFLOP/s",
                        "note": "pack + 9 conv/tconv layers + heads; flops per SURVEY.md 8d"},
        "spmv": {"bound": "hbm", "ms": sp_ms, "bytes": sp_bytes, "achieved": sp_bytes / (sp_ms * 1e-3) / 1e9,
                 "peak": hbm_peak, "unit": "GB/s", "frac": sp_bytes / (sp_ms * 1e-3) / 1e9 / hbm_peak,
                 "frac_of_8tbs_spec": sp_bytes / (sp_ms * 1e-3) / 8e12,
                 "note": "one system; L2 flushed (write, then read back) before every rep",
                 "stream_frac": sp_ctx["stream_GBps"] / hbm_peak, **sp_ctx},
        "stencil_x8": {"bound": "hbm", "kernel": "stencil3_kernel (K00, 8 systems)", "ms": st8_ms,
                       "bytes": st8_bytes, "achieved": st8_bytes / (st8_ms * 1e-3) / 1e9, "peak": hbm_peak,
                       "unit": "GB/s", "frac": st8_bytes / (st8_ms * 1e-3) / 1e9 / hbm_peak,
                       "frac_of_8tbs_spec": st8_bytes / (st8_ms * 1e-3) / 8e12},
        "spmv_x8": {"bound": "hbm", "kernel": "coupled SpMV (stencil + Pi gather, Pi^T pull + 1D rows), 8 systems",
                    "ms": sp8_ms, "bytes": sp8_bytes, "achieved": sp8_bytes / (sp8_ms * 1e-3) / 1e9,
                    "peak": hbm_peak, "unit": "GB/s", "frac": sp8_bytes / (sp8_ms * 1e-3) / 1e9 / hbm_peak,
                    "frac_of_8tbs_spec": sp8_bytes / (sp8_ms * 1e-3) / 8e12},
    }
    del flush, net
    torch.cuda.empty_cache()
    return out


def neural_forward_flops(n):
    from paper_2505_08491_b200 import neural
    m, q = n // 2, n // 4
    f = 0.0
    for name, op, cin, cout, ks, _ in neural.ARCHITECTURE:
        if op == "tconv":
            f += 2.0 * (m ** 3 if name == "up2" else n ** 3) * cin * cout
        else:
            vox = {"enc3": m ** 3, "dec2": m ** 3, "bottleneck": q ** 3}.get(name, n ** 3)
            f += 2.0 * vox * cin * cout * ks ** 3
    return f


def ncu_traffic(key):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of a
    kernel from the committed ncu --set full summary (profiles/traffic.json,
    written by tools/ncu_summary.py --traffic), or None."""
    path = Path(__file__).resolve().parent / "profiles" / "traffic.json"
    try:
        return json.loads(path.read_text()).get(key)
    except (OSError, ValueError):
        return None


def spmv_roofline(solver, reps=20):
    """Coupled SpMV: algorithmic bytes 16 (N3 + N1) + 40 Q per system,
    L2 flushed (write, then read back) before every rep."""
    import torch
    p = solver.prob
    X = p.zeros().normal_()
    Y = p.zeros()
    flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")
    ms = device_ms(lambda: solver.A.matvec(X, Y), reps, flush=flush)
    nbytes = sum(16 * (p.n3 + int(n1)) for n1 in p.n1) + 40 * p.Qtot
    ctx = spmv_stream_and_floors(p, solver.A, flush, nbytes)
    del flush
    return ms, nbytes, ctx


def config_dict(name, wl):
    """The workload description printed identically by both arms."""
    return {"workload": name, **wl.meta, "systems_per_gpu": len(wl.systems), "restart": wl.restart,
            "rtol": wl.tol, "maxit": wl.maxit, "inner_iterations": wl.inner_iterations,
            "smoothing": list(wl.smoothing), "l2": "flushed between timed steps (256 MiB write)"}


# z-planes of the CNN slab the operator-model CPU sample runs the oracle forward on
# (op2 = 0 / op1 = 1 like the full 65^3 / 129^3 grids; cost scales with the voxel count)
SLAB_Z = 9


def oracle_sampler(name, wl):
    """CPU oracle timing of the workload (test infrastructure as the timed baseline).

    Returns (sample(), describe(times)): ``sample()`` runs one bounded piece
    of the oracle solve and returns (seconds measured, extrapolated seconds
    per outer FGMRES iteration of ONE system).

    * cfg1 / cfg2: two outer iterations of the oracle coupled solve
      (oracle.solve_coupled, the restatement of harness.py:342-398).
    * cfg3 / cfg4 (65^3 / 129^3: one oracle CNN forward alone takes 4 / 40 s):
      the per-operator model of one outer iteration: 3
      smoothed CNN applies (1 forward + 5 C-SpMVs each), 6 more C-SpMVs of
      the 3-step inner FGMRES, the A-SpMV plus its share of the per-cycle
      residual SpMVs, and one MGS step over the cycle-average number of basis
      vectors.  The forward is timed on a 9-plane z-slab of the grid and
      scaled by the voxel ratio; the SpMVs and the MGS step run at full size.
    """
    import numpy as np
    import oracle
    from oracle import problem as OP
    osys = oracle_system(name)
    params = oracle.noisy_params(wl.cnn_seed)
    sm = wl.smoothing
    if name in ("cfg1", "cfg2"):
        spec = {"type": "neural", "params": params, "smoothing": sm}
        it = 2

        def sample():
            st = oracle.CoupledStrategy(tol=wl.tol, maxit=it, restart=wl.restart,
                                        inner_iterations=wl.inner_iterations, three_d=spec)
            t0 = time.perf_counter()
            oracle.solve_coupled(osys, st)
            dt = time.perf_counter() - t0
            return dt, dt / it

        return sample, lambda: f"{it} outer iterations of the oracle coupled solve per sample"
    A = OP.full_operator(osys)
    C = OP.reduced_operator(osys)
    n, n3 = osys.grid.n, osys.n3
    N = A.shape[0]
    rng = np.random.default_rng(0)
    x = rng.standard_normal(N)
    x3 = x[:n3].copy()
    slab = rng.standard_normal((2, SLAB_Z, n, n))
    kavg = (wl.restart + 1) // 2
    V = rng.standard_normal((kavg, N))
    m = wl.inner_iterations
    n_c = m * (sm[0] * 2 + 1) + 2 * m   # smoothing SpMVs of m applies + the inner FGMRES SpMVs
    n_a = 1 + 2.0 / wl.restart

    def sample():
        t0 = time.perf_counter()
        oracle.unet_forward(params, slab)
        t_cnn = (time.perf_counter() - t0) * n / SLAB_Z
        t1 = time.perf_counter()
        C @ x3
        t_c = time.perf_counter() - t1
        t2 = time.perf_counter()
        w = A @ x
        t_a = time.perf_counter() - t2
        t3 = time.perf_counter()
        for i in range(kavg):  # krylov.py:138-140
            h = w @ V[i]
            w -= h * V[i]
        np.linalg.norm(w)
        t_mgs = time.perf_counter() - t3
        dt = time.perf_counter() - t0
        return dt, m * t_cnn + n_c * t_c + n_a * t_a + t_mgs

    return sample, lambda: (f"per-operator model of one outer iteration: oracle U-Net forward on a {SLAB_Z}x{n}x{n} "
                            f"slab scaled by {n}/{SLAB_Z} (x{m} applies), {n_c} C-SpMVs, {n_a:.2f} A-SpMVs, "
                            f"one MGS step over {kavg} vectors, all at {n}^3")


def run_reference(args):
    """CPU arm: the oracle restatement of the reference path on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2505_08491_b200 import configs
    wl = configs.CONFIGS[args.workload]()
    if args.maxit:
        wl.maxit = args.maxit
    sample, describe = oracle_sampler(args.workload, wl)
    times, per_iter = [], []
    for step in range(args.warmup + args.steps):
        dt, pit = sample()
        if step >= args.warmup:
            times.append(dt)
            per_iter.append(pit)
    pit = statistics.median(per_iter)
    full = wl.maxit
    value = len(wl.systems) / (pit * full * len(wl.systems))
    cores = len(os.sched_getaffinity(0))
    desc = f"{describe()}; extrapolated to {full} outer iterations per system"
    line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": config_dict(args.workload, wl), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": "port", "sample": desc,
                             "s_per_outer_iteration": pit},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


DATA = "synthetic (seeded BASELINE graphs, perturbed random-init CNN)"


def oracle_system(name):
    """The workload's first system built by the oracle from the same seeded graph."""
    from oracle import problem as OP
    if name == "cfg1":
        g = OP.segment_graph([0.5, 0.5, 0.1], [0.5, 0.5, 0.9], 0.02)
        return OP.assemble_coupled_system(OP.StructuredGrid(17), g, OP.PhysicalParams(epsilon=0.02, beta=1.0),
                                          n_circle=8, elems_per_edge=32, bc3d="dirichlet", f1d=1.0)
    if name == "cfg2":
        g = OP.random_tree(8, 1, 0.015)
        return OP.assemble_coupled_system(OP.StructuredGrid(33), g, OP.PhysicalParams(epsilon=0.015, beta=1.0),
                                          n_circle=8, elems_per_edge=16, bc3d="dirichlet", f1d=1.0)
    if name == "cfg3":
        import numpy as np
        beta = float(np.random.default_rng(2).uniform(0.5, 2.0, 16)[0])
        return OP.assemble_coupled_system(OP.StructuredGrid(65), OP.random_tree(32, 2000, 0.01),
                                          OP.PhysicalParams(epsilon=0.01, beta=beta), n_circle=8,
                                          elems_per_edge=16, bc3d="dirichlet", f1d=1.0)
    if name == "cfg4":
        return OP.assemble_coupled_system(OP.StructuredGrid(129), OP.random_tree(64, 3, 0.008),
                                          OP.PhysicalParams(epsilon=0.008, beta=1.0), n_circle=8,
                                          elems_per_edge=32, bc3d="dirichlet", f1d=1.0, check_radius=False)
    raise ValueError(f"no oracle builder for {name}")


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2505_08491_b200 import _ext, configs, harness, neural
    from paper_2505_08491_b200.replicas import aggregate_throughput

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _ext.lib()
    wl = configs.CONFIGS[args.workload]()
    if args.maxit:
        wl.maxit = args.maxit
    params = neural.perturbed_params(wl.cnn_seed)
    spec = {"type": "neural", "params": params, "smoothing": {"maxit": wl.smoothing[0], "omega": wl.smoothing[1]}}
    strat = harness.CoupledStrategy(tol=wl.tol, maxit=wl.maxit, restart=wl.restart,
                                    inner_iterations=wl.inner_iterations, three_d=spec)
    solver = harness.CoupledSolver(wl.systems, strat)
    flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    reps = None
    for _ in range(args.warmup):
        reps = solver.solve()
    iters = [reps[i].iterations for i in range(len(wl.systems))]
    conv = [reps[i].converged for i in range(len(wl.systems))]
    rel = [reps[i].rel_residual for i in range(len(wl.systems))]

    ms_steps = []
    l0 = lib.mdp_launch_count() + solver.outer.replayed_kernels
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush_l2(flush)
            barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            reps = solver.solve()
            e.record()
            e.synchronize()
            ms_steps.append(s.elapsed_time(e))
    launches = lib.mdp_launch_count() + solver.outer.replayed_kernels - l0
    # whole job: all ranks' solves / the slowest rank's device time (replicas, no data-path collective)
    value, t_max, _ = aggregate_throughput(sum(ms_steps), len(wl.systems) * args.steps, device="cuda")

    # -- preconditioner applies/s (smoothed CNN apply, batched over the workload systems)
    P = solver.inner
    p = solver.prob
    V = p.zeros().normal_()
    Z = p.zeros()
    sel = torch.arange(p.nsys, dtype=torch.int32, device="cuda")
    idx = list(range(p.nsys))
    for _ in range(3):
        P.apply_device(V, Z, sel, idx)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    na = 20
    s.record()
    for _ in range(na):
        P.apply_device(V, Z, sel, idx)
    e.record()
    e.synchronize()
    applies_per_s = na * p.nsys / (s.elapsed_time(e) * 1e-3)

    # -- e2e through the drop-in API with host buffers, on every rank (replicas), whole-job
    #    solves/s = all ranks' solves / the slowest rank's wall time
    e2e_n = min(args.steps, E2E_MAX_STEPS)
    e2e_ms, h2d, d2h = e2e_steps(wl, strat, e2e_n)
    e2e_value, _, _ = aggregate_throughput(e2e_ms * e2e_n, len(wl.systems) * e2e_n, device="cuda")

    out = None
    if rank == 0:
        pk = peaks()
        # -- dominant kernel roofline: tcgen05 conv layers at the workload size
        n = p.n
        layers = conv_layer_times(n)
        per_fwd = {k: v["ms"] for k, v in layers.items()}
        dom = max(per_fwd, key=per_fwd.get)
        # tensor denominator: kind::tf32 runs at half the dense bf16 rate; the measured bf16
        # burst peak (the layer is timed alone) / 2.  cuBLAS TF32 is reported beside it.
        tf32 = pk["bf16_tflops"] / 2
        cublas_tf32 = measure_tf32_peak()
        L = layers[dom]
        spmv_ms, spmv_bytes, spmv_ctx = spmv_roofline(solver)
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 system / tf32 CNN", "data": DATA,
            "config": config_dict(args.workload, wl),
            "iterations": iters, "converged": conv, "rel_residual": rel,
            "applies_per_s": applies_per_s,
            "roofline": {"bound": "tensor", "kernel": f"conv3_tc_kernel ({dom}, S={L['S']})",
                         "achieved": L["tflops"], "peak": tf32, "unit": "TFLOP/s",
                         "frac": L["tflops"] / tf32,
                         "traffic": (ncu_traffic(f"conv3_tc_kernel {dom} S={L['S']}") or {}).get("dram_bytes"),
                         "peak_note": f"MEASURED_PEAKS bf16_tflops/2 ({pk['source']}); cuBLAS TF32 8192^3 "
                                      f"in this run: {cublas_tf32:.1f} TF/s",
                         "frac_of_cublas_tf32": L["tflops"] / cublas_tf32},
            "conv_layers": layers,
            "roofline_spmv": {"bound": "hbm", "kernel": "coupled SpMV (stencil+Pi)",
                              "achieved": spmv_bytes / (spmv_ms * 1e-3) / 1e9, "peak": pk["hbm_gbs"],
                              "unit": "GB/s", "frac": spmv_bytes / (spmv_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                              "frac_of_8tbs_spec": spmv_bytes / (spmv_ms * 1e-3) / 8e12,
                              "note": "single launch; L2 flushed (write, then read back) before every rep",
                              "stream_frac": spmv_ctx["stream_GBps"] / pk["hbm_gbs"], **spmv_ctx},
            "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": h2d * world,
                    "d2h_bytes_per_step": d2h * world, "steps": e2e_n},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
        }
        if not args.no_target:
            line["target_128"] = target_128(tf32, pk["hbm_gbs"], layers if n == 129 else None)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.workload, wl, iters)
        out = line
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


def e2e_steps(wl, strat, steps):
    """Drop-in API: harness.solve_coupled(system(s), strategy) from host objects, host results."""
    import torch
    from paper_2505_08491_b200 import harness
    systems = wl.systems if len(wl.systems) > 1 else wl.systems[0]
    harness.solve_coupled(systems, strat)  # warm caches (weights upload is cached per params object)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        res = harness.solve_coupled(systems, strat)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    n = sum(s.n3 + s.n1 for s in wl.systems)
    from paper_2505_08491_b200.assembly import DeviceProblem
    desc_bytes = sum(t.numel() * t.element_size() for t in DeviceProblem(wl.systems)._t.values())
    h2d = desc_bytes + 8 * n + 8 * sum(s.n3 for s in wl.systems)
    d2h = 8 * n
    return ms, h2d, d2h


def cpu_baseline(name, wl, gpu_iters, samples=3):
    """The oracle on the host cores, a bounded sample of the same workload (see oracle_sampler)."""
    sample, describe = oracle_sampler(name, wl)
    sample()  # warm (numba-free numpy, but first-touch allocations)
    res = [sample() for _ in range(samples)]
    pit = statistics.median(r[1] for r in res)
    full = max(gpu_iters)
    return {"value": 1.0 / (pit * full), "unit": "solves/s", "cores": len(os.sched_getaffinity(0)),
            "kind": "port", "s_per_outer_iteration": pit,
            "sample": f"{describe()}; {samples} samples ({sum(r[0] for r in res):.1f} s), extrapolated to the "
                      f"{full} outer iterations per system of the GPU solve"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--maxit", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-target", action="store_true", help="skip the 128^3 target-config rooflines")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

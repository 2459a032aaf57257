"""Warm in-situ kernel breakdown of one coupled solve (torch.profiler / CUPTI).

Unlike an ncu launch list (serialised, cold cache), this records the kernels
as they run inside the solve's CUDA graphs, so busy-time vs span shows the
launch-gap overhead per outer iteration.

    python tools/step_breakdown.py [--workload cfg2] [--maxit 60] [--out f.json]
"""
import argparse, collections, json, sys
sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2505_08491_b200 import configs, harness, neural

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--maxit", type=int, default=60)
ap.add_argument("--out", default="")
a = ap.parse_args()
wl = configs.CONFIGS[a.workload]()
params = neural.perturbed_params(wl.cnn_seed)
spec = {"type": "neural", "params": params, "smoothing": {"maxit": wl.smoothing[0], "omega": wl.smoothing[1]}}
st = harness.CoupledStrategy(tol=wl.tol, maxit=a.maxit, restart=wl.restart, inner_iterations=3, three_d=spec)
solver = harness.CoupledSolver(wl.systems, st)
for _ in range(2):
    solver.solve()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); r = solver.solve(); e.record(); e.synchronize()
plain_ms = s.elapsed_time(e)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    solver.solve()
    torch.cuda.synchronize()
evs = [ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
kern = [ev for ev in evs if "memcpy" not in ev.name.lower() and "memset" not in ev.name.lower()]
t0 = min(ev.time_range.start for ev in evs)
t1 = max(ev.time_range.end for ev in evs)
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in kern:
    k = ev.name.split("(")[0][:60]
    agg[k][0] += 1
    agg[k][1] += ev.time_range.elapsed_us()
busy = sum(v[1] for v in agg.values())
iters = r[0].iterations
out = {"workload": a.workload, "outer_iterations": iters, "plain_ms": plain_ms, "span_us": t1 - t0,
       "kernel_busy_us": busy, "busy_frac": busy / (t1 - t0), "kernels": len(kern),
       "kernels_per_outer_iteration": len(kern) / max(iters, 1),
       "by_kernel": {k: {"n": v[0], "us": v[1], "avg_us": v[1] / v[0], "share": v[1] / busy}
                     for k, v in sorted(agg.items(), key=lambda x: -x[1][1])}}
print(json.dumps({k: v for k, v in out.items() if k != "by_kernel"}))
for k, v in list(out["by_kernel"].items())[:30]:
    print(f"{v['us']:10.1f} us {100 * v['share']:5.1f}%  n={v['n']:6d} avg={v['avg_us']:7.2f}  {k}")
if a.out:
    open(a.out, "w").write(json.dumps(out, indent=1))

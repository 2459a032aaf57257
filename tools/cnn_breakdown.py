"""Warm kernel breakdown of one CNN preconditioner forward (torch.profiler / CUPTI).

    python tools/cnn_breakdown.py [--n 129] [--nb 1] [--out f.json]
"""
import argparse, collections, json, sys
sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile
import bench
from paper_2505_08491_b200 import neural

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=129)
ap.add_argument("--nb", type=int, default=1)
ap.add_argument("--out", default="")
ap.add_argument("--lib", default="", help="A/B: load this build of the library instead")
a = ap.parse_args()
if a.lib:
    from pathlib import Path
    from paper_2505_08491_b200 import _ext
    _ext.load_library(Path(a.lib))
n, nb = a.n, a.nb
net = neural.DeviceUNet(neural.perturbed_params(3))
R = torch.randn((nb, n ** 3), dtype=torch.float64, device="cuda")
D = torch.rand((nb, n ** 3), dtype=torch.float64, device="cuda")
rn = torch.ones(nb, dtype=torch.float64, device="cuda")
Z = torch.empty_like(R)
fwd = lambda: net.apply(n, R, n ** 3, rn, D, n ** 3, Z, n ** 3, nb=nb)  # noqa: E731
ms = bench.device_ms(fwd, 5)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        fwd()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name.split("(")[0][:60]
        agg[k][0] += 1
        agg[k][1] += ev.time_range.elapsed_us() / 3
fl = nb * bench.neural_forward_flops(n)
out = {"n": n, "nb": nb, "forward_ms": ms, "tflops": fl / (ms * 1e-3) / 1e12,
       "kernels_us_per_forward": {k: round(v[1], 1) for k, v in sorted(agg.items(), key=lambda x: -x[1][1])}}
print(json.dumps({k: v for k, v in out.items() if k != "kernels_us_per_forward"}))
print(json.dumps(out["kernels_us_per_forward"]))
if a.out:
    open(a.out, "w").write(json.dumps(out, indent=1))

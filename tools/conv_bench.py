"""Per-layer tcgen05 conv timings at several sizes (CUDA events, warm)."""
import sys
sys.path.insert(0, ".")
import bench

for n in [int(a) for a in sys.argv[1:]] or [33, 65, 129]:
    L = bench.conv_layer_times(n, reps=10)
    tot = sum(v["ms"] for v in L.values())
    fl = sum(v["flops"] for v in L.values())
    print(f"n={n}: conv total {tot*1e3:8.1f} us  {fl/(tot*1e-3)/1e12:6.1f} TF/s  | " +
          "  ".join(f"{k}:{v['ms']*1e3:.1f}us/{v['tflops']:.0f}TF" for k, v in L.items()), flush=True)

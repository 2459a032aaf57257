"""Per-step clock64 trace of one stencil3 block: python tools/stencil_trace.py n nb"""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2505_08491_b200 import _ext, configs
from paper_2505_08491_b200.assembly import DeviceProblem
from paper_2505_08491_b200.operators import CouplingOps
n, nb = int(sys.argv[1]), int(sys.argv[2])
lib = _ext.lib()
lib.mdp_debug_trace.argtypes = [ctypes.c_int, ctypes.c_void_p]
p = DeviceProblem(configs.cfg5_systems(n, nb))
ops = CouplingOps(p)
X = p.zeros().normal_(); Y = p.zeros()
ops.stencil(X, Y); torch.cuda.synchronize()
lib.mdp_debug_trace(1, None)
buf = torch.empty(64 * 2 ** 20, device="cuda"); buf.add_(1); float(buf.sum())
ops.stencil(X, Y); torch.cuda.synchronize()
out = np.zeros((8, 512), dtype=np.int64)
lib.mdp_debug_trace(0, out.ctypes.data)
t0 = out[out > 0].min()
for w in (0, 1, 7):
    a = out[w].reshape(-1, 2)
    m = a[:, 0] > 0
    a = a[m] - t0
    print(f"warp {w}: steps {len(a)}")
    print("  start   ", a[:40, 0].tolist())
    print("  waited  ", (a[:40, 1] - a[:40, 0]).tolist())

"""Run one tcgen05 conv layer a few times (for ncu)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2505_08491_b200 import _ext, neural
S, cin, cout, pool = (int(a) for a in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
lib = _ext.lib()
rng = np.random.default_rng(0)
X = torch.as_tensor(rng.standard_normal(cin * S ** 3).astype(np.float32), device="cuda")
W = torch.as_tensor(neural.pack_conv(rng.standard_normal((cout, cin, 3, 3, 3)) * 0.05, 0).ravel(), device="cuda")
So = S // 2 if pool else S
Y = torch.empty(cout * So ** 3, dtype=torch.float32, device="cuda")
scr = torch.zeros(max(lib.mdp_conv3_scratch_bytes(1, S, cin, cout), 16), dtype=torch.uint8, device="cuda")
for _ in range(reps):
    _ext.check(lib.mdp_conv3_layer(0, 1, S, cin, cout, X.data_ptr(), cin // 4, 0, W.data_ptr(), None, 1,
                                   Y.data_ptr(), cout // 4, 0, pool, scr.data_ptr(), scr.numel(), _ext.stream()))
torch.cuda.synchronize()
print("ok")

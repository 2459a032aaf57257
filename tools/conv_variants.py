"""Time one conv layer under MDP_DEBUG_CONV variants (each in a fresh process)."""
import os, subprocess, sys
cfgs = [("dec1", "129 64 32 0"), ("enc3", "64 64 128 1")]
code = r'''
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2505_08491_b200 import _ext, neural
S, cin, cout, pool = (int(a) for a in sys.argv[1:5])
lib = _ext.lib(); rng = np.random.default_rng(0)
X = torch.as_tensor(rng.standard_normal(cin * S ** 3).astype(np.float32), device="cuda")
W = torch.as_tensor(neural.pack_conv(rng.standard_normal((cout, cin, 3, 3, 3)) * 0.05, 0).ravel(), device="cuda")
So = S // 2 if pool else S
Y = torch.empty(cout * So ** 3, dtype=torch.float32, device="cuda")
scr = torch.zeros(max(lib.mdp_conv3_scratch_bytes(1, S, cin, cout), 16), dtype=torch.uint8, device="cuda")
f = lambda: _ext.check(lib.mdp_conv3_layer(0, 1, S, cin, cout, X.data_ptr(), cin // 4, 0, W.data_ptr(), None, 1, Y.data_ptr(), cout // 4, 0, pool, scr.data_ptr(), scr.numel(), _ext.stream()))
f(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): f()
e.record(); e.synchronize()
print(f"{s.elapsed_time(e) / 10 * 1e3:.1f}")
'''
for name, args in cfgs:
    res = []
    for dbg in (15, 15 + 16 + 32, 15 + 16 + 32 + 64, 8 + 16 + 32 + 64, 8 + 16 + 32):
        env = dict(os.environ, MDP_DEBUG_CONV=str(dbg))
        out = subprocess.run([sys.executable, "-c", code, *args.split()], env=env, capture_output=True, text=True)
        res.append(f"dbg{dbg}={out.stdout.strip() or out.stderr.strip()[-80:]}")
    print(name, " ".join(res), flush=True)

"""clock64 trace of CTA 0 of one tcgen05 conv launch inside a CNN forward (needs a -DCONV_TRACE build):

    tools/build_ab.sh unet_tc paper_2505_08491_b200/csrc/unet_tc.cu /tmp/libtrace.so -DCONV_TRACE
    python tools/conv_trace.py /tmp/libtrace.so 129 <cin> <cout>      (enc1a on tensor cores: cin 4, cout 16)
"""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2505_08491_b200 import _ext
lib = _ext.load_library(Path(sys.argv[1]))
n, cin, cout = (int(a) for a in sys.argv[2:5])
from paper_2505_08491_b200 import neural
net = neural.DeviceUNet(neural.perturbed_params(3))
R = torch.randn((1, n ** 3), dtype=torch.float64, device="cuda")
D = torch.rand((1, n ** 3), dtype=torch.float64, device="cuda")
rn = torch.ones(1, dtype=torch.float64, device="cuda")
Z = torch.empty_like(R)
for _ in range(3):
    net.apply(n, R, n ** 3, rn, D, n ** 3, Z, n ** 3, nb=1)
torch.cuda.synchronize()
lib.mdp_conv_trace_select(cin, cout)
net.apply(n, R, n ** 3, rn, D, n ** 3, Z, n ** 3, nb=1)
torch.cuda.synchronize()
buf = np.zeros(16 + 6 * 48 * 4, dtype=np.int64)
lib.mdp_conv_trace_read(buf.ctypes.data_as(C.POINTER(C.c_longlong)))
t0, t1 = buf[0], buf[1]
ev = buf[16:].reshape(6, 48, 4)
print(f"layer cin={cin} cout={cout} n={n}: CTA 0 ran {t1 - t0} cycles")
print("tile | A-issue | mma: tmem-free  halo-ready  committed | epi0: full  done | epi1: full  done")
for i in range(48):
    if ev[1, i, 0] == 0:
        break
    r = lambda v: int(v - t0) if v else -1
    print(f"{i:4d} | {r(ev[0,i,0]):7d} | {r(ev[1,i,0]):9d} {r(ev[1,i,1]):10d} {r(ev[1,i,2]):10d} | "
          f"{r(ev[2,i,0]):8d} {r(ev[2,i,1]):8d} | {r(ev[3,i,0]):8d} {r(ev[3,i,1]):8d}")

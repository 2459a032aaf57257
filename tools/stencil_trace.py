"""Trace of three stencil3 blocks (first / middle / last slot) of the coupled SpMV of one system
(needs a -DST3_TRACE build of operators.cu):

    tools/build_ab.sh operators paper_2505_08491_b200/csrc/operators.cu abl/libst3trace.so -DST3_TRACE
    python tools/stencil_trace.py abl/libst3trace.so [cfg4|NxB]
"""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2505_08491_b200 import _ext
lib = _ext.load_library(Path(sys.argv[1]))
from paper_2505_08491_b200 import configs
from paper_2505_08491_b200.assembly import DeviceProblem
from paper_2505_08491_b200.operators import CoupledOperator
case = sys.argv[2] if len(sys.argv) > 2 else "cfg4"
if case.startswith("cfg"):
    systems = configs.CONFIGS[case]().systems
else:
    n, nb = (int(v) for v in case.split("x"))
    systems = configs.cfg5_systems(n, nb)
p = DeviceProblem(systems)
A = CoupledOperator(p)
XS = [p.zeros().normal_() for _ in range(10)]
YS = [p.zeros() for _ in range(10)]
for X, Y in zip(XS, YS):
    A.matvec(X, Y)
torch.cuda.synchronize()
for X, Y in zip(XS, YS):   # streamed: the trace keeps the last launch
    A.matvec(X, Y)
torch.cuda.synchronize()
buf = np.zeros(3 * 64, dtype=np.int64)
lib.mdp_st3_trace_read(buf.ctypes.data_as(C.POINTER(C.c_longlong)))
ev = buf.reshape(3, 64)
g0 = ev[:, 0].min()
for w, name in enumerate(("first slot", "middle slot", "last slot")):
    e = ev[w]
    print(f"{name}: entry at +{e[0] - g0} ns (globaltimer), block life {e[3] - e[0]} ns; setup {e[1] - e[2]} cycles")
    steps = [(int(e[4 + 2 * k] - e[2]), int(e[5 + 2 * k] - e[2])) for k in range(24) if e[4 + 2 * k]]
    print("   step: (full seen, done) cycles since entry:", steps)

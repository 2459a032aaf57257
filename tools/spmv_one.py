"""Coupled (or reduced) SpMV on cfg5-style systems (for ncu): python tools/spmv_one.py n nb reps [coupled]
(n = 0: the single BASELINE cfg4 system, 129^3 with the 64-segment tree)"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2505_08491_b200 import configs
from paper_2505_08491_b200.assembly import DeviceProblem
from paper_2505_08491_b200.operators import CoupledOperator, ReducedOperator
n, nb, reps = (int(a) for a in sys.argv[1:4])
coupled = len(sys.argv) > 4 and sys.argv[4] == "coupled"
p = DeviceProblem(configs.cfg4().systems if n == 0 else configs.cfg5_systems(n, nb))
C = CoupledOperator(p) if coupled else ReducedOperator(p)
X = p.zeros().normal_(); Y = p.zeros()
for _ in range(reps):
    C.matvec(X, Y)
torch.cuda.synchronize()
print("ok")

"""K00 stencil only on cfg5-style systems (for ncu): python tools/stencil_one.py n nb reps"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2505_08491_b200 import configs
from paper_2505_08491_b200.assembly import DeviceProblem
from paper_2505_08491_b200.operators import CouplingOps
n, nb, reps = (int(a) for a in sys.argv[1:4])
p = DeviceProblem(configs.cfg5_systems(n, nb))
ops = CouplingOps(p)
X = p.zeros().normal_(); Y = p.zeros()
for _ in range(reps):
    ops.stencil(X, Y)
torch.cuda.synchronize()
print("ok")

"""One CNN preconditioner forward at size n (for ncu): python tools/cnn_one.py n nb reps"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2505_08491_b200 import neural
n, nb, reps = (int(a) for a in sys.argv[1:4])
net = neural.DeviceUNet(neural.perturbed_params(1))
R = torch.randn((nb, n ** 3), dtype=torch.float64, device="cuda")
D = torch.rand((nb, n ** 3), dtype=torch.float64, device="cuda")
rn = torch.ones(nb, dtype=torch.float64, device="cuda")
Z = torch.empty_like(R)
for _ in range(reps):
    net.apply(n, R, n ** 3, rn, D, n ** 3, Z, n ** 3, nb=nb)
torch.cuda.synchronize()
print("ok")

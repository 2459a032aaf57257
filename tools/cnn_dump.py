"""Dump CNN forwards (seeded inputs) for bitwise A/B between library builds or env knobs:
python tools/cnn_dump.py out.pt  -> {(n, nb): Z}; compare two dumps with --cmp a.pt b.pt"""
import sys
sys.path.insert(0, ".")
import torch
if sys.argv[1] == "--cmp":
    a, b = torch.load(sys.argv[2]), torch.load(sys.argv[3])
    bad = [k for k in a if not torch.equal(a[k], b[k])]
    print("bitwise equal" if not bad else f"DIFFER: {bad}")
    sys.exit(1 if bad else 0)
from paper_2505_08491_b200 import neural
net = neural.DeviceUNet(neural.perturbed_params(1))
out = {}
g = torch.Generator(device="cuda").manual_seed(0)
for n, nb in ((33, 1), (33, 4), (65, 1), (65, 3), (129, 1), (49, 2)):
    R = torch.randn((nb, n ** 3), dtype=torch.float64, device="cuda", generator=g)
    D = torch.rand((nb, n ** 3), dtype=torch.float64, device="cuda", generator=g)
    rn = torch.ones(nb, dtype=torch.float64, device="cuda")
    Z = torch.empty_like(R)
    net.apply(n, R, n ** 3, rn, D, n ** 3, Z, n ** 3, nb=nb)
    out[(n, nb)] = Z.cpu()
torch.save(out, sys.argv[1])
print("ok", {k: float(v.abs().sum()) for k, v in out.items()})

"""A/B timing of mdp_arnoldi between the current library and another build.

    python tools/arnoldi_ab.py tools/ab/libold.so [more.so ...]
"""
import ctypes as C
import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2505_08491_b200 import _ext


def load(path):
    lib = C.CDLL(path)
    for name, (res, args) in _ext._SIGS.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


libs = {"cur": _ext.lib()}
for path in sys.argv[1:]:
    libs[path.rsplit("/", 1)[-1].replace(".so", "")] = load(path)
flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")
for n, nb, k in [(36000, 1, 30), (36000, 1, 4), (2146689, 1, 30), (2146689, 8, 30), (7189057, 1, 30), (274625, 16, 50)]:
    ld = (n + 31) // 32 * 32
    V = torch.randn((nb, k + 1, ld), dtype=torch.float64, device="cuda")
    W = torch.randn((nb, ld), dtype=torch.float64, device="cuda")
    H = torch.zeros((nb, k + 2), dtype=torch.float64, device="cuda")
    nv = torch.full((nb,), k, dtype=torch.int32, device="cuda")
    row = {"n": n, "nsel": nb, "k": k}
    for tag, lib in libs.items():
        work = torch.zeros(lib.mdp_arnoldi_work_bytes(nb, k, n) // 8 + 1, dtype=torch.float64, device="cuda")

        def arn():
            _ext.check(lib.mdp_arnoldi(nb, None, V.data_ptr(), (k + 1) * ld, ld, nv.data_ptr(), k, W.data_ptr(), ld, n,
                                       H.data_ptr(), None, 0, work.data_ptr(), _ext.stream()))
        ms = bench.device_ms(arn, 5, flush=flush, hide_us=3000)
        row[tag + "_us"] = round(ms * 1e3, 1)
        row[tag + "_GBps"] = round((3 * k + 3) * n * 8 * nb / (ms * 1e-3) / 1e9)
    print(row, flush=True)
    del V, W, H
    torch.cuda.empty_cache()

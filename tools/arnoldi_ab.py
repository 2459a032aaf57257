"""A/B timing of the Arnoldi step: one-pass MGS (Gram rows, V read twice, 3 launches)
vs CGS2 (V read three times, 4 launches), cold L2.

    python tools/arnoldi_ab.py
"""
import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2505_08491_b200 import _ext

lib = _ext.lib()
flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")
for n, nb, k in [(36000, 1, 30), (36000, 1, 3), (2146689, 1, 30), (2146689, 1, 50), (2146689, 1, 3), (2146689, 8, 30),
                 (7189057, 1, 30), (274625, 16, 50), (274625, 16, 3)]:
    ld = (n + 31) // 32 * 32
    V = torch.randn((nb, k + 1, ld), dtype=torch.float64, device="cuda")
    W = torch.randn((nb, ld), dtype=torch.float64, device="cuda")
    H = torch.zeros((nb, k + 2), dtype=torch.float64, device="cuda")
    nv = torch.full((nb,), k, dtype=torch.int32, device="cuda")
    gram = torch.zeros((nb, k + 1, k + 1), dtype=torch.float64, device="cuda")
    work = torch.zeros(lib.mdp_arnoldi_work_bytes(nb, k, n) // 8 + 1, dtype=torch.float64, device="cuda")
    row = {"n": n, "nsel": nb, "k": k, "survey_bytes": (2 * k + 3) * n * 8 * nb}
    for tag, gr, moved in (("mgs1", gram, 2 * k + 6), ("cgs2", None, 3 * k + 8)):
        def arn():
            _ext.check(lib.mdp_arnoldi(nb, None, V.data_ptr(), (k + 1) * ld, ld, nv.data_ptr(), k, W.data_ptr(), ld, n,
                                       H.data_ptr(), None, 0, _ext.ptr(gr), work.data_ptr(), _ext.stream()))
        ms = bench.device_ms(arn, 5, flush=flush, hide_us=3000)
        row[tag + "_us"] = round(ms * 1e3, 1)
        row[tag + "_survey_GBps"] = round(row["survey_bytes"] / (ms * 1e-3) / 1e9)
        row[tag + "_moved_GBps"] = round(moved * n * 8 * nb / (ms * 1e-3) / 1e9)
    print(row, flush=True)
    del V, W, H
    torch.cuda.empty_cache()

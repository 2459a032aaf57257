"""A/B of the coupled SpMV paths: two-launch (MDP_SPMV_V=3) vs single-launch (4).

    python tools/spmv_ab.py [--cases cfg4,cfg2,129x1,129x8] [--variants "V=3;V=4;V=4,PERSM=3"]

One subprocess per variant (selectors are read once per process).  Cold L2 before
every rep (256 MiB written, then read back).  Bytes per SURVEY.md 8d: coupled
16 (N3 + N1) + 40 Q per system, reduced 16 N3 + 40 Q, Jacobi sweep 24 N3 + 40 Q
(x, r read, out written; diag(C) read: +8 N3 -> 32 N3).
"""
import argparse
import json
import os
import subprocess
import sys

sys.path.insert(0, ".")


def child(cases):
    import torch
    from paper_2505_08491_b200 import configs
    from paper_2505_08491_b200.assembly import DeviceProblem
    from paper_2505_08491_b200.operators import CoupledOperator, CouplingOps, ReducedOperator
    buf = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")

    def timed(fn, reps=9):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            buf.add_(1.0)
            float(buf.sum())
            torch.cuda._sleep(2_000_000)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        return ts[len(ts) // 2]

    out = []
    for c in cases:
        if c.startswith("cfg"):
            systems = configs.CONFIGS[c]().systems
        else:
            n, nb = (int(v) for v in c.split("x"))
            systems = configs.cfg5_systems(n, nb)
        p = DeviceProblem(systems)
        A, C = CoupledOperator(p), ReducedOperator(p)
        X, Y, R, T = p.zeros().normal_(), p.zeros(), p.zeros().normal_(), p.zeros()
        ops = CouplingOps(p)
        ts = timed(lambda: ops.stencil(X, Y))
        tc = timed(lambda: A.matvec(X, Y))
        tr = timed(lambda: C.matvec(X, Y))
        tj = timed(lambda: C.jacobi(R, X, Y, 2.0 / 3.0, T))
        tcp = timed(lambda: Y.copy_(X))
        bc = sum(16 * (p.n3 + int(n1)) for n1 in p.n1) + 40 * p.Qtot
        br = 16 * p.n3 * p.nsys + 40 * p.Qtot
        bj = 32 * p.n3 * p.nsys + 40 * p.Qtot
        out.append({"case": c, "stencil_us": round(ts * 1e3, 2), "stencil_GBps": round(16 * p.n3 * p.nsys / ts / 1e6, 1),
                    "coupled_us": round(tc * 1e3, 2), "coupled_GBps": round(bc / tc / 1e6, 1),
                    "reduced_us": round(tr * 1e3, 2), "reduced_GBps": round(br / tr / 1e6, 1),
                    "jacobi_us": round(tj * 1e3, 2), "jacobi_GBps": round(bj / tj / 1e6, 1),
                    "copy_us": round(tcp * 1e3, 2), "copy_GBps": round(2 * 8 * X.numel() / tcp / 1e6, 1)})
        del p, A, C, X, Y, R, T
        torch.cuda.empty_cache()
    print("RESULT " + json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg4,cfg2,129x1,129x8,65x16,193x1")
    ap.add_argument("--variants", default="V=3;V=4")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    cases = a.cases.split(",")
    if a.child:
        child(cases)
        return
    for var in a.variants.split(";"):
        env = dict(os.environ)
        for kv in var.split(","):
            k, v = kv.split("=")
            env[{"V": "MDP_SPMV_V", "SV": "MDP_STENCIL_V", "NODES": "MDP_ITEM_NODES", "ROWS": "MDP_ITEM_ROWS",
                 "LAST": "MDP_FUSED_LAST"}.get(k, k)] = v
        r = subprocess.run([sys.executable, __file__, "--child", "--cases", a.cases], env=env, capture_output=True,
                           text=True)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
        if not lines:
            print(f"{var}: failed\n{r.stderr[-3000:]}")
            continue
        for row in json.loads(lines[0][7:]):
            print(json.dumps({"variant": var, **row}), flush=True)


if __name__ == "__main__":
    main()

"""A/B of the stencil kernels (MDP_STENCIL_V=1 / 2): K00 alone and the coupled SpMV.

    python tools/stencil_ab.py [--versions 1,2] [--cases 33x1,129x1,129x8,193x8] [--env K=V,...]

One subprocess per version (the selector is read once per process).  Cold
L2 before every rep: a 256 MiB buffer is written and then read back, so no
dirty lines from the flush are written back inside the timed region.
Bytes: K00 alone 16 N3 per system; coupled 16 (N3 + N1) + 40 Q.
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
    from paper_2505_08491_b200.operators import CoupledOperator, CouplingOps
    buf = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")

    def timed(fn, reps=9):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            buf.add_(1.0)
            float(buf.sum())  # read back: L2 now holds clean lines only
            torch.cuda._sleep(2_000_000)  # ~1 ms: host enqueue hidden
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        return ts[len(ts) // 2]

    out = []
    for n, nb in cases:
        p = DeviceProblem(configs.cfg5_systems(n, nb))
        A, ops = CoupledOperator(p), CouplingOps(p)
        X, Y = p.zeros().normal_(), p.zeros()
        t_st = timed(lambda: ops.stencil(X, Y))
        t_c = timed(lambda: A.matvec(X, Y))
        t_cp = timed(lambda: Y.copy_(X))
        t_g = timed(lambda: ops.gather(X, None, p.s_work))
        t_s = timed(lambda: ops.scatter(p.s_work, 1.0, Y))
        b_st = 16 * p.n3 * nb
        b_c = sum(16 * (p.n3 + int(n1)) for n1 in p.n1) + 40 * p.Qtot
        out.append({"n": n, "nb": nb, "stencil_us": round(t_st * 1e3, 2), "stencil_GBps": round(b_st / t_st / 1e6, 1),
                    "coupled_us": round(t_c * 1e3, 2), "coupled_GBps": round(b_c / t_c / 1e6, 1),
                    "copy_GBps": round(2 * X.numel() * 8 / t_cp / 1e6, 1), "gather_us": round(t_g * 1e3, 2),
                    "pull_us": round(t_s * 1e3, 2)})
        del p, A, ops, X, Y
        torch.cuda.empty_cache()
    print("RESULT " + json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--versions", default="1,3")
    ap.add_argument("--cases", default="33x1,65x8,129x1,129x8,193x8")
    ap.add_argument("--env", default="")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    cases = [tuple(int(v) for v in c.split("x")) for c in a.cases.split(",")]
    if a.child:
        child(cases)
        return
    extra = dict(kv.split("=") for kv in a.env.split(",") if kv)
    for v in a.versions.split(","):
        env = dict(os.environ, MDP_STENCIL_V=v, **extra)
        r = subprocess.run([sys.executable, __file__, "--child", "--cases", a.cases], env=env, capture_output=True,
                           text=True)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
        if not lines:
            print(f"v{v}: failed\n{r.stderr[-2000:]}")
            continue
        for row in json.loads(lines[0][7:]):
            print(json.dumps({"v": v, **extra, **row}))


if __name__ == "__main__":
    main()

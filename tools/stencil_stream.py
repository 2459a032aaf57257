"""Streamed (rotating vector pairs > 2x L2, back to back) timing of the K00 stencil, the coupled SpMV and
the Jacobi sweep under launch-shape variants (one subprocess per variant; env selectors are read once).

    python tools/stencil_stream.py [--cases cfg4,129x8,65x16,cfg2] [--variants "base;MDP_STENCIL_RY=2;MDP_STENCIL_ZCHUNK=17"]
"""
import argparse, json, os, subprocess, sys
sys.path.insert(0, ".")


def child(cases, lib):
    import torch
    import bench
    from paper_2505_08491_b200 import _ext, configs
    if lib:
        from pathlib import Path
        _ext.load_library(Path(lib))
    from paper_2505_08491_b200.assembly import DeviceProblem
    from paper_2505_08491_b200.operators import CoupledOperator, CouplingOps, ReducedOperator
    out = []
    for c in cases:
        if c.startswith("cfg"):
            systems = configs.CONFIGS[c]().systems
        else:
            n, nb = (int(v) for v in c.split("x"))
            systems = configs.cfg5_systems(n, nb)
        p = DeviceProblem(systems)
        A, C, ops = CoupledOperator(p), ReducedOperator(p), CouplingOps(p)
        nbytes = sum(16 * (p.n3 + int(n1)) for n1 in p.n1) + 40 * p.Qtot
        nset = min(64, max(2, int(-(-2.5 * 126e6 // nbytes))))
        XS = [p.zeros().normal_() for _ in range(nset)]
        YS = [p.zeros() for _ in range(nset)]
        R, T = p.zeros().normal_(), p.zeros()
        ts = bench.device_ms_stream([(lambda X=X, Y=Y: ops.stencil(X, Y)) for X, Y in zip(XS, YS)])
        tc = bench.device_ms_stream([(lambda X=X, Y=Y: A.matvec(X, Y)) for X, Y in zip(XS, YS)])
        tj = bench.device_ms_stream([(lambda X=X, Y=Y: C.jacobi(R, X, Y, 2.0 / 3.0, T)) for X, Y in zip(XS, YS)])
        hb = bench.peaks()["hbm_gbs"]
        out.append({"case": c, "stencil_us": round(ts * 1e3, 2), "stencil_frac": round(16 * p.n3 * p.nsys / ts / 1e6 / hb, 3),
                    "coupled_us": round(tc * 1e3, 2), "coupled_frac": round(nbytes / tc / 1e6 / hb, 3),
                    "jacobi_us": round(tj * 1e3, 2), "jacobi_frac": round((32 * p.n3 * p.nsys + 40 * p.Qtot) / tj / 1e6 / hb, 3)})
        del p, A, C, ops, XS, YS, R, T
        torch.cuda.empty_cache()
    print("RESULT " + json.dumps(out))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg4,129x8,65x16,cfg2")
    ap.add_argument("--variants", default="base")
    ap.add_argument("--lib", default="")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.cases.split(","), a.lib)
        sys.exit(0)
    for var in a.variants.split(";"):
        env = dict(os.environ)
        lib = a.lib
        if var != "base":
            for kv in var.split(","):
                k, v = kv.split("=")
                if k == "LIB":
                    lib = v
                else:
                    env[k] = v
        r = subprocess.run([sys.executable, __file__, "--child", "--cases", a.cases, "--lib", lib], env=env,
                           capture_output=True, text=True)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
        if not lines:
            print(f"{var}: failed\n{r.stderr[-2000:]}")
            continue
        for row in json.loads(lines[0][7:]):
            print(json.dumps({"variant": var, **row}), flush=True)

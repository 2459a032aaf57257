"""z-chunk sweep of the stencil / coupled SpMV (cold L2, device time).

    python tools/stencil_sweep.py [--lib path.so] [--tag name]
Runs one subprocess per MDP_STENCIL_ZCHUNK value (read once per process).
"""
import argparse, json, os, subprocess, sys
sys.path.insert(0, ".")

CASES = [(33, 1), (129, 1), (129, 8), (193, 8)]


def child(lib_path):
    import torch
    import bench
    from paper_2505_08491_b200 import _ext, configs
    if lib_path:
        _ext.LIB_PATH = __import__("pathlib").Path(lib_path)
        _ext.load_library(_ext.LIB_PATH)
    from paper_2505_08491_b200.assembly import DeviceProblem
    from paper_2505_08491_b200.operators import CoupledOperator, ReducedOperator
    flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")
    out = []
    for n, nb in CASES:
        p = DeviceProblem(configs.cfg5_systems(n, nb))
        A, C = CoupledOperator(p), ReducedOperator(p)
        X, Y = p.zeros().normal_(), p.zeros()
        ms_c = bench.device_ms(lambda: A.matvec(X, Y), 7, flush=flush, hide_us=2000)
        ms_r = bench.device_ms(lambda: C.matvec(X, Y), 7, flush=flush, hide_us=2000)
        byt = sum(16 * (p.n3 + int(n1)) for n1 in p.n1) + 40 * p.Qtot
        out.append({"n": n, "nb": nb, "coupled_us": round(ms_c * 1e3, 1), "reduced_us": round(ms_r * 1e3, 1),
                    "coupled_frac": round(byt / (ms_c * 1e-3) / 1e9 / bench.peaks()["hbm_gbs"], 3)})
        del p, A, C, X, Y
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--z", default="0,4,8,12,16,24,32")
    a = ap.parse_args()
    if a.child:
        child(a.lib)
        sys.exit(0)
    for z in [int(v) for v in a.z.split(",")]:
        env = dict(os.environ)
        if z:
            env["MDP_STENCIL_ZCHUNK"] = str(z)
        r = subprocess.run([sys.executable, __file__, "--child", "--lib", a.lib], env=env, capture_output=True,
                           text=True, timeout=600)
        rows = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]
        print(json.dumps({"zchunk": z or "auto", "rows": rows}), flush=True)

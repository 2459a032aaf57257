"""Is the cfg1-geometry 'none' solve (reference: 272 iterations) sensitive to summation order?

CPU experiment on the ORACLE restatement (FP64 throughout, MGS exactly as
krylov.py:138-140).  Variants change nothing but floating-point rounding:

  blas      w @ V[i] through BLAS ddot (the reference's own expression)
  pairwise  np.sum(w * V[i]) (numpy pairwise summation)
  fsum      math.fsum(w * V[i]) (correctly rounded dot of the rounded products)
  rhs+eps   blas, right-hand side scaled by (1 + 2^-52 * m), m = 1..4
  cgs2      classical Gram-Schmidt applied twice (this package's device order), BLAS

Each prints the iteration count of solve_coupled(cfg1 geometry, three_d=none,
restart 30, rtol 1e-6).  Writes profiles/r02_sensitivity_cfg1.json.
"""
import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
from oracle import problem as OP, solver as OS, coupled as OC  # noqa: E402


def make_fgmres(dot, orth="mgs"):
    def fgmres(apply_A, precond, b, restart=20, tol=1e-6, maxit=1000, x0=None):
        A = OS._as_apply(apply_A)
        P = precond
        b = np.asarray(b, dtype=float)
        n = b.shape[0]
        x = np.zeros(n)
        r = b - A(x)
        r0 = np.linalg.norm(r)
        if r0 == 0.0:
            return x, OS.SolveReport(0, True, [0.0], 0.0, 0.0, 0.0)
        hist, its, brk, conv = [1.0], 0, 0, False
        V = np.empty((restart + 1, n))
        Z = np.empty((restart, n))
        while not conv and its < maxit:
            beta = np.linalg.norm(r)
            if beta / r0 <= tol:
                conv = True
                break
            V[0] = r / beta
            H = np.zeros((restart + 1, restart))
            cs, sn, g = np.zeros(restart), np.zeros(restart), np.zeros(restart + 1)
            g[0] = beta
            j = 0
            while j < restart and its < maxit:
                Z[j] = V[j] if P is None else P(V[j])
                w = A(Z[j])
                if orth == "mgs":
                    for i in range(j + 1):
                        H[i, j] = dot(w, V[i])
                        w -= H[i, j] * V[i]
                else:
                    h1 = np.array([dot(w, V[i]) for i in range(j + 1)])
                    for i in range(j + 1):
                        w -= h1[i] * V[i]
                    h2 = np.array([dot(w, V[i]) for i in range(j + 1)])
                    for i in range(j + 1):
                        w -= h2[i] * V[i]
                    H[:j + 1, j] = h1 + h2
                hn = np.linalg.norm(w)
                for i in range(j):
                    t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                    H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                    H[i, j] = t
                den = np.hypot(H[j, j], hn)
                if den < OS.BREAKDOWN_TOL:
                    its += 1
                    hist.append(hist[-1])
                    brk += 1
                    break
                cs[j], sn[j] = H[j, j] / den, hn / den
                H[j, j] = den
                g[j + 1] = -sn[j] * g[j]
                g[j] = cs[j] * g[j]
                its += 1
                est = abs(g[j + 1]) / r0
                hist.append(est)
                j += 1
                if hn < OS.BREAKDOWN_TOL:
                    brk += 1
                    break
                V[j] = w / hn
                if est <= tol:
                    break
            if j > 0:
                y = np.zeros(j)
                for i in range(j - 1, -1, -1):
                    y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:j]) / H[i, i]
                x = x + Z[:j].T @ y
            r = b - A(x)
            if np.linalg.norm(r) / r0 <= tol:
                conv = True
        rel = float(np.linalg.norm(b - A(x)) / r0)
        hist.append(rel)
        return x, OS.SolveReport(its, conv, hist, rel, 0.0, 0.0, brk)
    return fgmres


def system():
    return OP.assemble_coupled_system(OP.StructuredGrid(17), OP.segment_graph([0.5, 0.5, 0.1], [0.5, 0.5, 0.9], 0.02),
                                      OP.PhysicalParams(epsilon=0.02, beta=1.0), n_circle=8, elems_per_edge=32)


def run(fg, scale=1.0, neural=False):
    s = system()
    if scale != 1.0:
        import dataclasses
        s = dataclasses.replace(s, rhs0=s.rhs0 * scale, rhs1=s.rhs1 * scale)
    OC.fgmres = fg
    spec = {"type": "none"}
    if neural:  # the reference tests' perturbed seed-0 network, Jacobi(2, 2/3)-smoothed, FP64
        spec = {"type": "neural", "params": oracle.noisy_params(0), "smoothing": (2, 2.0 / 3.0)}
    st = OC.CoupledStrategy(tol=1e-6, maxit=600 if neural else 300, restart=30, inner_iterations=3, three_d=spec)
    _, _, rep = OC.solve_coupled(s, st)
    return {"iterations": rep.iterations, "converged": bool(rep.converged), "rel": rep.rel_residual}


if __name__ == "__main__":
    blas = lambda a, b: a @ b  # noqa: E731
    out = {"blas": run(make_fgmres(blas)),
           "pairwise": run(make_fgmres(lambda a, b: np.sum(a * b))),
           "fsum": run(make_fgmres(lambda a, b: math.fsum(a * b))),
           "cgs2": run(make_fgmres(blas, "cgs2"))}
    for m in range(1, 5):
        out[f"rhs*(1+{m}ulp)"] = run(make_fgmres(blas), 1.0 + m * 2.0 ** -52)
    if "--neural" in sys.argv:
        out["neural_s blas (maxit 600)"] = run(make_fgmres(blas), neural=True)
        out["neural_s pairwise (maxit 600)"] = run(make_fgmres(lambda a, b: np.sum(a * b)), neural=True)
        out["neural_s rhs*(1+1ulp) (maxit 600)"] = run(make_fgmres(blas), 1.0 + 2.0 ** -52, neural=True)
    for k, v in out.items():
        print(k, v, flush=True)
    (ROOT / "profiles" / "r02_sensitivity_cfg1.json").write_text(json.dumps(out, indent=1))

"""Oracle Krylov pieces: FGMRES (MGS), ILU(0), weighted Jacobi.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

BREAKDOWN_TOL = 1e-14   # krylov.py:28


@dataclass
class SolveReport:
    """krylov.py:31-41."""

    iterations: int
    converged: bool
    residual_history: list
    rel_residual: float
    wall_time: float
    time_per_iter: float
    breakdowns: int = 0


def _as_apply(op):
    if callable(op) and not sp.issparse(op):
        return op
    return lambda v: op @ v


def fgmres(apply_A, precond, b, restart: int = 20, tol: float = 1e-6, maxit: int = 1000,
           x0=None):
    """Flexible GMRES(restart), right preconditioning, MGS (krylov.py:88-182).

    Control flow per SURVEY.md Appendix C: breakdown attempts count as
    iterations, convergence only from the true residual at cycle
    boundaries, tolerance relative to ||r0||.
    """
    if restart < 1:
        raise ValueError("restart must be at least 1")
    if tol <= 0:
        raise ValueError("tol must be positive")
    A = _as_apply(apply_A)
    P = precond
    b = np.asarray(b, dtype=float)
    n = b.shape[0]
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=float)
    t0 = time.perf_counter()
    r = b - A(x)
    r0 = np.linalg.norm(r)
    if r0 == 0.0:
        return x, SolveReport(0, True, [0.0], 0.0, time.perf_counter() - t0, 0.0)
    hist = [1.0]
    its = 0
    brk = 0
    conv = False
    V = np.empty((restart + 1, n))
    Z = np.empty((restart, n))
    while not conv and its < maxit:
        beta = np.linalg.norm(r)
        if beta / r0 <= tol:
            conv = True
            break
        V[0] = r / beta
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        j = 0
        while j < restart and its < maxit:
            Z[j] = V[j] if P is None else P(V[j])
            w = A(Z[j])
            for i in range(j + 1):
                H[i, j] = w @ V[i]
                w -= H[i, j] * V[i]
            hn = np.linalg.norm(w)
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], hn)
            if den < BREAKDOWN_TOL:
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
            if hn < BREAKDOWN_TOL:
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
    wall = time.perf_counter() - t0
    return x, SolveReport(its, conv, hist, rel, wall, wall / its if its else 0.0, brk)


@dataclass(frozen=True)
class IluFactor:
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray
    diag_pos: np.ndarray
    L: sp.csr_matrix
    U: sp.csr_matrix


def ilu0(A) -> IluFactor:
    """ILU(0) on the sorted CSR pattern of A (krylov.py:188-216, 247-267)."""
    A = sp.csr_matrix(A).copy()
    A.sort_indices()
    n = A.shape[0]
    ip, ix = A.indptr, A.indices
    dpos = np.full(n, -1, dtype=np.int64)
    for i in range(n):
        row = ix[ip[i]:ip[i + 1]]
        k = np.searchsorted(row, i)
        if k < len(row) and row[k] == i:
            dpos[i] = ip[i] + k
    if np.any(dpos < 0):
        raise ValueError(f"zero pivot: row {int(np.nonzero(dpos < 0)[0][0])} has no diagonal entry")
    a = A.data.astype(float).copy()
    for i in range(n):
        p = ip[i]
        while p < ip[i + 1] and ix[p] < i:
            k = ix[p]
            piv = a[dpos[k]]
            if abs(piv) < BREAKDOWN_TOL:
                raise ValueError(f"zero pivot in row {k} during ILU(0)")
            lik = a[p] / piv
            a[p] = lik
            pk, pi = dpos[k] + 1, p + 1
            while pk < ip[k + 1] and pi < ip[i + 1]:
                if ix[pk] == ix[pi]:
                    a[pi] -= lik * a[pk]
                    pk += 1
                    pi += 1
                elif ix[pk] < ix[pi]:
                    pk += 1
                else:
                    pi += 1
            p += 1
        if abs(a[dpos[i]]) < BREAKDOWN_TOL:
            raise ValueError(f"zero pivot in row {i} during ILU(0)")
    F = sp.csr_matrix((a, ix.copy(), ip.copy()), shape=A.shape)
    L = sp.tril(F, k=-1, format="csr") + sp.identity(n, format="csr")
    U = sp.triu(F, k=0, format="csr")
    return IluFactor(ip.copy(), ix.copy(), a, dpos, L.tocsr(), U.tocsr())


def ilu0_apply(f: IluFactor, r: np.ndarray) -> np.ndarray:
    """Unit-lower forward then upper backward sweep (krylov.py:219-233, 270-276)."""
    n = len(f.diag_pos)
    ip, ix, a, dp = f.indptr, f.indices, f.data, f.diag_pos
    x = np.empty(n)
    for i in range(n):
        s = r[i]
        for p in range(ip[i], dp[i]):
            s -= a[p] * x[ix[p]]
        x[i] = s
    for i in range(n - 1, -1, -1):
        s = x[i]
        for p in range(dp[i] + 1, ip[i + 1]):
            s -= a[p] * x[ix[p]]
        x[i] = s / a[dp[i]]
    return x


def jacobi_smooth(A, r, x0, maxit: int, omega: float = 2.0 / 3.0):
    """x <- x + omega (r - A x) / diag(A) (krylov.py:290-299)."""
    d = np.asarray(A.diagonal())
    if np.any(d == 0.0):
        raise ValueError("Jacobi relaxation needs a nonzero diagonal")
    x = np.array(x0, dtype=float)
    for _ in range(maxit):
        x = x + omega * (r - A @ x) / d
    return x

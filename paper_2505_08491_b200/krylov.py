"""Flexible GMRES on the device, batched over independent systems.

Reproduces ``mdprec.krylov.fgmres`` (krylov.py:88-182) control flow
literally: breakdown attempts count as iterations,
an Arnoldi breakdown (hypot(H_jj, h_next) < 1e-14) ends the cycle without
advancing j, a lucky breakdown (h_next < 1e-14) ends it after, the Givens
estimate only ends a cycle early, and convergence is declared solely from
the true residual ||b - A x|| / ||r0|| at cycle boundaries.

The vectors (V, Z, x, r, w) live in HBM as [nsys][k][ld] float64; the
orthogonalisation is the fused CGS2 kernel (mdp_arnoldi); the small
Hessenberg / Givens / back-substitution work runs on the host from one
device->host read of the new Hessenberg column per Arnoldi step for all
systems at once.  Each system keeps its own j, cycle, iteration count and
convergence state, so a batched solve reproduces every system's serial
solve (multi-query setting, paper section 5.7).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _ext

BREAKDOWN_TOL = 1e-14  # krylov.py:28


@dataclass
class SolveReport:
    """Outcome of one preconditioned solve (krylov.py:31-41)."""

    iterations: int
    converged: bool
    residual_history: list
    rel_residual: float
    wall_time: float
    time_per_iter: float
    breakdowns: int = 0


class Preconditioner:
    """Apply contract ``z = P(r)`` (krylov.py:44-51).

    Device preconditioners additionally implement ``apply_device(V, Z,
    sel)`` on ``(nsys, ld)`` float64 storages.
    """

    def apply(self, r):
        raise NotImplementedError

    def __call__(self, r):
        return self.apply(r)


# Dense device factorizations behind the exact baselines are limited to this many
# bytes per matrix (n = 33: C is 35937^2 doubles = 10.3 GB; 65^3 would need 600 GB).
EXACT_MAX_BYTES = 48 << 30


class ExactPreconditioner(Preconditioner):
    """Direct solve, the reference's 'perfect' preconditioner (krylov.py:54-61), on
    the device: C is symmetric positive definite (Neumann with a reaction term, or
    symmetric Dirichlet elimination), so it is factored once as a dense Cholesky
    product in HBM (cuSOLVER through torch.linalg) and every apply is two
    triangular solves.  Grids whose dense matrix exceeds EXACT_MAX_BYTES raise."""

    def __init__(self, A, device="cuda"):
        import torch
        if hasattr(A, "prob") and hasattr(A, "matvec"):
            from .assembly import host_reduced_operator
            A = host_reduced_operator(A.prob.systems[0])
        A = sp.coo_matrix(A)
        n = A.shape[0]
        if A.shape[0] != A.shape[1]:
            raise ValueError("exact solve needs a square matrix")
        if n * n * 8 > EXACT_MAX_BYTES:
            raise ValueError(f"dense exact solve of a {n}x{n} matrix exceeds {EXACT_MAX_BYTES >> 30} GiB")
        D = torch.zeros((n, n), dtype=torch.float64, device=device)
        D.index_put_((torch.as_tensor(A.row, device=device), torch.as_tensor(A.col, device=device)),
                     torch.as_tensor(A.data, device=device), accumulate=True)
        self.L, info = torch.linalg.cholesky_ex(D)
        del D
        if int(info) != 0:
            raise ValueError("exact solve: matrix is not positive definite")
        self.n = n

    def solve_device(self, B):
        """X = A^-1 B for a device (n,) or (n, k) tensor."""
        import torch
        vec = B.dim() == 1
        X = torch.cholesky_solve(B[:, None] if vec else B, self.L)
        return X[:, 0] if vec else X

    def apply(self, r):
        import torch
        r = np.asarray(r, dtype=float)
        if r.shape != (self.n,):
            raise ValueError("right-hand side length mismatch")
        return self.solve_device(torch.as_tensor(r, device=self.L.device)).cpu().numpy()

    def apply_device(self, V, Z, sel, idx=None):
        for s in (sel.cpu().tolist() if idx is None else idx):
            Z[s, :self.n] = self.solve_device(V[s, :self.n])


def spmv(A, x):
    """CSR / device-operator product with a dimension check (krylov.py:64-69)."""
    x = np.asarray(x)
    if A.shape[1] != x.shape[0]:
        raise ValueError(f"dimension mismatch: {A.shape} @ {x.shape}")
    return A @ x


def _gram_storage(nsys, k, f):
    """Strictly lower Gram rows V_m . V_c of a cycle's basis, [nsys][k+1][k+1]: the
    Arnoldi step then is modified Gram-Schmidt (krylov.py:138-140) from one pass of
    dot products (include/mdp_b200.h, mdp_arnoldi).  MDP_ORTH=cgs2 selects the
    two-pass classical variant (A/B timing only)."""
    import os
    import torch
    if os.environ.get("MDP_ORTH", "mgs") == "cgs2":
        return None
    return torch.zeros((nsys, k + 1, k + 1), **f)


class _State:
    __slots__ = ("j", "iters", "brk", "conv", "r0", "hist", "H", "cs", "sn", "g", "done", "rel", "beta",
                 "t0", "wall")

    def __init__(self, k):
        self.j = 0
        self.iters = 0
        self.brk = 0
        self.conv = False
        self.done = False
        self.r0 = 0.0
        self.hist = [1.0]
        # Hessenberg columns (rotated) and Givens state as Python floats: the
        # per-step host work runs while the device idles, and float ops are
        # the same IEEE double ops as numpy scalars (krylov.py:142-157)
        self.H = []
        self.cs = [0.0] * k
        self.sn = [0.0] * k
        self.g = [0.0] * (k + 1)
        self.rel = 0.0
        self.beta = 0.0


class FgmresEngine:
    """Workspace + driver for batched right-preconditioned FGMRES(k).

    ``A(X, Y, sel)`` and ``P(V, Z, sel, idx)`` act on (nsys, ld) float64
    CUDA storages for the systems listed in the int32 CUDA tensor ``sel``
    (``idx``: the same list on the host).
    ``n`` is the active vector length (entries beyond it stay zero).
    """

    def __init__(self, nsys: int, n: int, ld: int, restart: int, device="cuda"):
        import torch
        if restart < 1:
            raise ValueError("restart must be at least 1")
        self.lib = _ext.lib()
        self.nsys, self.n, self.ld, self.k = nsys, n, ld, restart
        f = dict(dtype=torch.float64, device=device)
        self.V = torch.zeros((nsys, restart + 1, ld), **f)
        self.Z = torch.zeros((nsys, restart, ld), **f)
        self.x = torch.zeros((nsys, ld), **f)
        self.r = torch.zeros((nsys, ld), **f)
        self.w = torch.zeros((nsys, ld), **f)
        self.vcur = torch.zeros((nsys, ld), **f)
        self.zcur = torch.zeros((nsys, ld), **f)
        self.tmp = torch.zeros((nsys, ld), **f)
        # Hessenberg columns [nsys][k+2] followed by one flag per system (graph
        # steps); two parities so a speculative step can run while the host
        # reads the previous one
        self._hb = []
        for _ in range(2):
            hb = torch.zeros(nsys * (restart + 2) + nsys, **f)
            self._hb.append((hb, hb[:nsys * (restart + 2)].view(nsys, restart + 2), hb[nsys * (restart + 2):]))
        self._use_parity(0)
        self._par = 0
        self._graphs = {}
        self.speculative = True      # enqueue step j+1 before reading step j (graph path)
        self.spec_discarded = 0      # speculative steps thrown away (cycle ends / exact redo)
        self.replayed_kernels = 0  # our kernels executed through graph replays
        self.rn = torch.zeros(nsys, **f)
        self.ybuf = torch.zeros((nsys, restart), **f)
        self.betad = torch.zeros(nsys, **f)
        wb = self.lib.mdp_arnoldi_work_bytes(nsys, restart, n)
        self.work = torch.zeros(wb // 8 + 1, **f)  # reduction tickets must start at zero
        self.gram = _gram_storage(nsys, restart, f)
        pin = dict(pin_memory=True)
        self.h_host = torch.zeros(nsys * (restart + 2) + nsys, dtype=torch.float64, **pin)
        self.rn_host = torch.zeros(nsys, dtype=torch.float64, **pin)
        self.y_host = torch.zeros((nsys, restart), dtype=torch.float64, **pin)
        self.beta_host = torch.zeros(nsys, dtype=torch.float64, **pin)
        # one pinned staging slot + device copy per upload purpose: a slot is
        # rewritten only after a stream synchronisation since its last copy
        self._regions = {}
        for name in ("all", "start", "arn0", "js0", "nv0", "arn1", "js1", "nv1", "end", "cnt", "res", "redo", "rjs",
                     "rnv"):
            self._regions[name] = (torch.zeros(nsys, dtype=torch.int32, pin_memory=True),
                                   torch.zeros(nsys, dtype=torch.int32, device=device))

    # -- small helpers -------------------------------------------------------------
    def _use_parity(self, par):
        self.hbuf, self.hcol, self.pflag = self._hb[par]
    def _upload(self, name, values):
        """Small int32 list -> device through its dedicated pinned slot."""
        import torch
        host, dev = self._regions[name]
        m = len(values)
        host[:m] = torch.as_tensor(np.asarray(values, dtype=np.int32))
        dev[:m].copy_(host[:m], non_blocking=True)
        return dev[:m]

    def _step(self, A, P, sel, jd, nv, ma, idx):
        """Z[j] = P(V[j]); w = A Z[j]; CGS2 projections; V[j+1] = w/||w|| (krylov.py:136-141, 165)."""
        k = self.k
        if P is None:
            _ext.check(self.lib.mdp_copy_vec(ma, sel.data_ptr(), self.vcur.data_ptr(), self.ld,
                                             self.zcur.data_ptr(), self.ld, None, 0, self.n, _ext.stream()))
        else:
            P(self.vcur, self.zcur, sel, idx)
        _ext.check(self.lib.mdp_copy_vec(ma, sel.data_ptr(), self.zcur.data_ptr(), self.ld,
                                         self.Z.data_ptr(), k * self.ld, jd.data_ptr(), self.ld, self.n,
                                         _ext.stream()))
        A(self.zcur, self.w, sel)
        _ext.check(self.lib.mdp_arnoldi(ma, sel.data_ptr(), self.V.data_ptr(), (k + 1) * self.ld, self.ld,
                                        nv.data_ptr(), k, self.w.data_ptr(), self.ld, self.n,
                                        self.hcol.data_ptr(), self.vcur.data_ptr(), self.ld,
                                        _ext.ptr(self.gram), self.work.data_ptr(), _ext.stream()))

    def _capture(self, A, Pg, sel, jd, nv, ma, idx):
        """CUDA graph of one Arnoldi step with a graph-safe preconditioner.

        Pg(V, Z, sel, idx, flag) must not allocate or synchronise and
        writes a nonzero flag for any system it could not handle exactly.
        """
        import torch

        def P(V, Z, sel_, idx_):
            Pg(V, Z, sel_, idx_, self.pflag)

        # eager warm-up (first-use setup outside capture), then restore vcur = V[j]
        self._step(A, P, sel, jd, nv, ma, idx)
        self._gather_slot(sel, jd, ma)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        l0 = self.lib.mdp_launch_count()
        with torch.cuda.graph(g):
            self._step(A, P, sel, jd, nv, ma, idx)
        return g, self.lib.mdp_launch_count() - l0

    def _gather_slot(self, sel, jd, m):
        """vcur_s = V[s, j_s] for the listed systems."""
        k = self.k
        _ext.check(self.lib.mdp_copy_slot(m, sel.data_ptr(), self.V.data_ptr(), (k + 1) * self.ld, jd.data_ptr(),
                                          self.ld, self.vcur.data_ptr(), self.ld, self.n, _ext.stream()))

    def _read_h(self, m, with_flags=False, then=None):
        """Hessenberg columns (+ flags) of the current parity to the host.

        ``then()`` is enqueued after the copies and before the wait, which
        covers only the work up to the copies (a speculative step keeps the
        device busy meanwhile)."""
        import torch
        kk = self.k + 2
        nf = self.nsys * kk
        self.h_host[:m * kk].copy_(self.hbuf[:m * kk], non_blocking=True)
        if with_flags:
            self.h_host[nf:nf + m].copy_(self.pflag[:m], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        if then is not None:
            then()
        ev.synchronize()
        h = self.h_host[:m * kk].numpy().reshape(m, kk)
        f = self.h_host[nf:nf + m].numpy() if with_flags else None
        return h, f

    def _graph(self, A, Pg, arn, par, js):
        """(graph, launches) of one Arnoldi step for the active set ``arn`` with
        the parity-``par`` buffers; uploads this step's j values."""
        key = (tuple(arn), par)
        sel = self._upload(f"arn{par}", arn)
        jd = self._upload(f"js{par}", js)
        nv = self._upload(f"nv{par}", [j + 1 for j in js])
        g = self._graphs.get(key)
        if g is None:
            self._use_parity(par)
            g = self._capture(A, Pg, sel, jd, nv, len(arn), list(arn))
            self._graphs[key] = g
        return g, sel, jd

    def _sync_read(self, dev, host, m):
        import torch
        host[:m].copy_(dev[:m], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return host[:m].numpy()

    def _residual(self, A, b, sel, m):
        """r = b - A x for the selected systems; returns ||r|| on the host."""
        A(self.x, self.tmp, sel)
        _ext.check(self.lib.mdp_residual(m, sel.data_ptr(), b.data_ptr(), self.tmp.data_ptr(),
                                         self.r.data_ptr(), self.ld, self.n, self.rn.data_ptr(),
                                         self.work.data_ptr(), _ext.stream()))
        return self._sync_read(self.rn, self.rn_host, m).copy()

    # -- the solve -----------------------------------------------------------------
    def solve(self, A, P, b, tol: float = 1e-6, maxit: int = 1000, x0=None, systems=None,
              final_residual: bool = True, Pg=None):
        """Solve A x = b for the listed systems (default all); returns reports.

        ``b`` is an (nsys, ld) storage; ``x0`` an optional storage.  The
        solution is left in ``self.x``.  ``final_residual=False`` skips the
        last cycle's true-residual computation when no further cycle can
        follow (inner solves whose report is discarded, harness.py:385-387);
        the returned x is unaffected.  ``Pg``: optional graph-safe variant
        of ``P`` (see ``_capture``); the Arnoldi step then runs as one CUDA
        graph per set of active systems, falling back to ``P`` for flagged
        systems.
        """
        import torch
        if tol <= 0:
            raise ValueError("tol must be positive")
        systems = list(range(self.nsys)) if systems is None else list(systems)
        k = self.k
        t_start = time.perf_counter()
        st = {s: _State(k) for s in systems}
        sel_all = self._upload("all", systems)
        m = len(systems)
        if x0 is None:
            # r = b - A(0) = b exactly; skip the SpMV of a zero vector
            self.x.index_fill_(0, sel_all.long(), 0.0)
            self.r.index_copy_(0, sel_all.long(), b.index_select(0, sel_all.long()))
            _ext.check(self.lib.mdp_norms(m, sel_all.data_ptr(), self.r.data_ptr(), self.ld, self.n,
                                          self.rn.data_ptr(), self.work.data_ptr(), _ext.stream()))
            rn = self._sync_read(self.rn, self.rn_host, m).copy()
        else:
            self.x.index_copy_(0, sel_all.long(), x0.index_select(0, sel_all.long()))
            rn = self._residual(A, b, sel_all, m)
        starting = []
        for i, s in enumerate(systems):
            S = st[s]
            S.r0 = float(rn[i])
            S.beta = S.r0
            if S.r0 == 0.0:
                S.done, S.conv, S.hist, S.rel = True, True, [0.0], 0.0
            else:
                starting.append(s)
        arn = []          # systems currently inside a cycle
        spec = None       # (systems, js, parity) of a speculatively enqueued Arnoldi step
        stale = False     # vcur advanced by a discarded speculative step
        while True:
            # ---- cycle starts (krylov.py:123-134)
            if starting:
                go = []
                for s in starting:
                    S = st[s]
                    if S.iters >= maxit:
                        self._finish(S)
                        continue
                    if S.beta / S.r0 <= tol:
                        S.conv = True
                        self._finish(S)
                        continue
                    go.append(s)
                    S.H = []
                    S.cs = [0.0] * k
                    S.sn = [0.0] * k
                    S.g = [0.0] * (k + 1)
                    S.g[0] = S.beta
                    S.j = 0
                if go:
                    sel = self._upload("start", go)
                    self.beta_host[:len(go)] = torch.as_tensor(np.array([st[s].beta for s in go], dtype=np.float64))
                    self.betad[:len(go)].copy_(self.beta_host[:len(go)], non_blocking=True)
                    # V[0] = r / beta (exact division) and the current vector
                    V0 = self.V[:, 0, :]
                    _ext.check(self.lib.mdp_scale(len(go), sel.data_ptr(), self.r.data_ptr(), self.ld, None,
                                                  self.betad.data_ptr(), V0.data_ptr(), (k + 1) * self.ld,
                                                  self.n, _ext.stream()))
                    _ext.check(self.lib.mdp_copy_vec(len(go), sel.data_ptr(), V0.data_ptr(), (k + 1) * self.ld,
                                                     self.vcur.data_ptr(), self.ld, None, 0, self.n,
                                                     _ext.stream()))
                    arn.extend(go)
                starting = []
            if not arn:
                break
            arn.sort()
            # ---- one Arnoldi step for every system inside a cycle (krylov.py:135-167)
            js = [st[s].j for s in arn]
            ma = len(arn)
            if Pg is not None:
                if spec is not None and spec[0] == tuple(arn) and spec[1] == js:
                    par = spec[2]  # this step is already enqueued (speculatively)
                else:
                    # the parity not used by the last enqueued step (its uploads are done)
                    par = self._par = self._par ^ 1
                    g, sel, jd = self._graph(A, Pg, arn, par, js)
                    if spec is not None or stale:
                        # a discarded speculative step advanced vcur: restore V[j]
                        self._gather_slot(sel, jd, ma)
                        self.spec_discarded += 1
                    self._use_parity(par)
                    g[0].replay()
                    self.replayed_kernels += g[1]
                spec, stale = None, False
                self._use_parity(par)
                # speculate: enqueue step j+1 for the same systems (a cycle end or
                # an exact redo below discards it); only with a captured graph
                nxt = None
                if self.speculative and all(st[s].j + 1 < k and st[s].iters + 1 < maxit for s in arn) \
                        and (tuple(arn), par ^ 1) in self._graphs:
                    def nxt(arn=arn, q=par ^ 1, js1=[j + 1 for j in js]):
                        nonlocal spec
                        g1 = self._graph(A, Pg, arn, q, js1)[0]
                        g1[0].replay()
                        self.replayed_kernels += g1[1]
                        self._par = q
                        spec = (tuple(arn), js1, q)
                hb = self._read_h(ma, with_flags=True, then=nxt)
                self._use_parity(par)
                redo = [s for i, s in enumerate(arn) if hb[1][i] != 0.0]
                if redo:
                    if spec is not None:
                        # the speculative step used the flagged systems' inexact step j:
                        # discard it (stream order keeps it ahead of the redo below)
                        spec, stale = None, True
                    # exact host-driven path for systems whose graph step hit a flagged case
                    rsel = self._upload("redo", redo)
                    rj = self._upload("rjs", [st[s].j for s in redo])
                    rnv = self._upload("rnv", [st[s].j + 1 for s in redo])
                    # the graph overwrote vcur with V[j+1]; restore V[j] for the redo
                    self._gather_slot(rsel, rj, len(redo))
                    self._step(A, P, rsel, rj, rnv, len(redo), redo)
                    hr = self._read_h(len(redo))[0]
                    pos = {s: i for i, s in enumerate(arn)}
                    hc = hb[0].copy()
                    for i, s in enumerate(redo):
                        hc[pos[s]] = hr[i]
                else:
                    hc = hb[0]
            else:
                sel = self._upload("arn0", arn)
                jd = self._upload("js0", js)
                nv = self._upload("nv0", [j + 1 for j in js])
                self._step(A, P, sel, jd, nv, ma, arn)
                hc = self._read_h(ma)[0]
            ending = []
            for i, s in enumerate(arn):
                S = st[s]
                j = S.j
                cs, sn, g = S.cs, S.sn, S.g
                col = hc[i, :j + 1].tolist()
                h_next = float(hc[i, k + 1])
                for ii in range(j):
                    a, c = col[ii], col[ii + 1]
                    col[ii + 1] = -sn[ii] * a + cs[ii] * c
                    col[ii] = cs[ii] * a + sn[ii] * c
                denom = float(np.hypot(col[j], h_next))
                if denom < BREAKDOWN_TOL:
                    S.iters += 1
                    S.hist.append(S.hist[-1])
                    S.brk += 1
                    ending.append(s)
                    continue
                cs[j], sn[j] = col[j] / denom, h_next / denom
                col[j] = denom
                S.H.append(col)
                g[j + 1] = -sn[j] * g[j]
                g[j] = cs[j] * g[j]
                S.iters += 1
                est = abs(g[j + 1]) / S.r0
                S.hist.append(est)
                S.j = j + 1
                if h_next < BREAKDOWN_TOL:
                    S.brk += 1
                    ending.append(s)
                elif est <= tol or S.j >= k or S.iters >= maxit:
                    ending.append(s)
            if ending:
                arn = [s for s in arn if s not in set(ending)]
                self._end_cycles(A, b, st, ending, tol, maxit, final_residual)
                starting = [s for s in ending if not st[s].done]
        wall = time.perf_counter() - t_start
        reports = {}
        for s in systems:
            S = st[s]
            reports[s] = SolveReport(S.iters, S.conv, S.hist, S.rel, wall, wall / S.iters if S.iters else 0.0,
                                     S.brk)
        return reports

    def _finish(self, S):
        # krylov.py:177-181: rel = ||b - A x|| / r0 (x unchanged since the last residual)
        S.rel = float(S.beta / S.r0)
        S.hist.append(S.rel)
        S.done = True

    def _end_cycles(self, A, b, st, ending, tol, maxit, final_residual):
        """x += Z[:j] y, r = b - A x, convergence test (krylov.py:168-175)."""
        import torch
        upd = [s for s in ending if st[s].j > 0]
        if upd:
            ys = np.zeros((len(upd), self.k))
            for i, s in enumerate(upd):
                S = st[s]
                j = S.j
                Hm = np.zeros((j, j))  # upper triangle of the rotated Hessenberg (krylov.py:168-171)
                for c in range(j):
                    Hm[:c + 1, c] = S.H[c][:c + 1]
                g = np.asarray(S.g)
                y = np.zeros(j)
                for ii in range(j - 1, -1, -1):
                    y[ii] = (g[ii] - Hm[ii, ii + 1:j] @ y[ii + 1:j]) / Hm[ii, ii]
                ys[i, :j] = y
            sel = self._upload("end", upd)
            cnt = self._upload("cnt", [st[s].j for s in upd])
            self.y_host[:len(upd)] = torch.as_tensor(ys)
            self.ybuf[:len(upd)].copy_(self.y_host[:len(upd)], non_blocking=True)
            _ext.check(self.lib.mdp_basis_update(len(upd), sel.data_ptr(), self.x.data_ptr(), self.ld,
                                                 self.Z.data_ptr(), self.k * self.ld, self.ld, cnt.data_ptr(),
                                                 self.ybuf.data_ptr(), self.k, self.n, _ext.stream()))
        # systems whose x changed need a new true residual; a breakdown at j=0
        # leaves x (hence r) unchanged bitwise, so the previous norm stands
        need = []
        for s in ending:
            S = st[s]
            if S.j == 0:
                continue
            if not final_residual and S.iters >= maxit:
                S.done = True
                S.rel = float("nan")
                continue
            need.append(s)
        if need:
            sel = self._upload("res", need)
            rn = self._residual(A, b, sel, len(need))
            for i, s in enumerate(need):
                st[s].beta = float(rn[i])
        for s in ending:
            S = st[s]
            if S.done:
                continue
            if S.beta / S.r0 <= tol:
                S.conv = True
            if S.conv or S.iters >= maxit:
                self._finish(S)


class FixedStepFgmres:
    """FGMRES with restart = maxit = m and tol = 1e-300, entirely on the device.

    This is the inner 3D solve of the block preconditioner
    (harness.py:385-387): with a tolerance of 1e-300 its control flow is
    static -- exactly m Arnoldi steps, then x = Z y -- unless an Arnoldi
    breakdown occurs or the right-hand side is zero.  The Givens rotations
    and the back substitution run in tiny device kernels (mdp_givens_step,
    mdp_backsub) so the whole solve can be captured in a CUDA graph; any
    system that hits a breakdown / zero rhs raises its flag and must be
    re-solved by the host-driven ``FgmresEngine`` (which reproduces
    krylov.fgmres branch by branch).
    """

    def __init__(self, nsys: int, n: int, ld: int, m: int, device="cuda"):
        import torch
        self.lib = _ext.lib()
        self.nsys, self.n, self.ld, self.k = nsys, n, ld, m
        f = dict(dtype=torch.float64, device=device)
        self.V = torch.zeros((nsys, m + 1, ld), **f)
        self.Z = torch.zeros((m, nsys, ld), **f)  # slot-major: P writes Z[j] (an (nsys, ld) storage) in place
        self.x = torch.zeros((nsys, ld), **f)
        self.w = torch.zeros((nsys, ld), **f)
        self.vcur = torch.zeros((nsys, ld), **f)
        self.hcol = torch.zeros((nsys, m + 2), **f)
        self.H = torch.zeros((nsys, m + 1, m), **f)
        self.cs = torch.zeros((nsys, m), **f)
        self.sn = torch.zeros((nsys, m), **f)
        self.g = torch.zeros((nsys, m + 1), **f)
        self.y = torch.zeros((nsys, m), **f)
        self.beta = torch.zeros(nsys, **f)
        self.flag = torch.zeros(nsys, **f)
        self.nvs = [torch.full((nsys,), j + 1, dtype=torch.int32, device=device) for j in range(m)]
        self.cnt = torch.full((nsys,), m, dtype=torch.int32, device=device)
        wb = self.lib.mdp_arnoldi_work_bytes(nsys, m, n)
        self.work = torch.zeros(wb // 8 + 1, **f)  # reduction tickets must start at zero
        self.gram = _gram_storage(nsys, m, f)

    def run(self, A, P, b, sel, idx, out=None, pre=None):
        """Enqueue the solve of A x = b for the selected systems (no host sync).

        ``out``: optional (nsys, ld) storage that receives x directly (else self.x).
        The start, each Arnoldi step's Givens update and the end are fused
        launches (mdp_fixed_start / mdp_arnoldi_givens / mdp_fixed_finish) with
        the arithmetic of the separate kernels.  ``pre``: optional (out, omega,
        diag) from ``P.first_sweep_spec()``: the kernels writing each apply's
        input also write its first Jacobi sweep, and P skips it."""
        L, st = self.lib, _ext.stream()
        m, k, ld, n = int(sel.numel()), self.k, self.ld, self.n
        sp_ = sel.data_ptr()
        jo, om, dg = (pre[0].data_ptr(), float(pre[1]), pre[2].data_ptr()) if pre is not None else (None, 0.0, None)
        _ext.check(L.mdp_norms(m, sp_, b.data_ptr(), ld, n, self.beta.data_ptr(), self.work.data_ptr(), st))
        V0 = self.V[:, 0, :]
        _ext.check(L.mdp_fixed_start(m, sp_, k, b.data_ptr(), ld, self.beta.data_ptr(), V0.data_ptr(), (k + 1) * ld,
                                     self.vcur.data_ptr(), ld, n, self.H.data_ptr(), self.cs.data_ptr(),
                                     self.sn.data_ptr(), self.g.data_ptr(), self.flag.data_ptr(), jo, om, dg, st))
        for j in range(k):
            Zj = self.Z[j]
            if P is None:
                _ext.check(L.mdp_copy_vec(m, sp_, self.vcur.data_ptr(), ld, Zj.data_ptr(), ld, None, 0, n, st))
            elif pre is not None:
                P(self.vcur, Zj, sel, idx, presmoothed=True)
            else:
                P(self.vcur, Zj, sel, idx)
            A(Zj, self.w, sel)
            _ext.check(L.mdp_arnoldi_givens(m, sp_, self.V.data_ptr(), (k + 1) * ld, ld, self.nvs[j].data_ptr(), k,
                                            self.w.data_ptr(), ld, n, self.hcol.data_ptr(), self.vcur.data_ptr(), ld,
                                            _ext.ptr(self.gram), self.work.data_ptr(), j, self.H.data_ptr(),
                                            self.cs.data_ptr(),
                                            self.sn.data_ptr(), self.g.data_ptr(), self.flag.data_ptr(),
                                            jo if j + 1 < k else None, om, dg, st))
        x = self.x if out is None else out
        _ext.check(L.mdp_fixed_finish(m, sp_, k, k, self.Z.data_ptr(), ld, self.nsys * ld, x.data_ptr(), ld, n,
                                      self.H.data_ptr(), self.g.data_ptr(), self.flag.data_ptr(), st))


# ---------------------------------------------------------------------------
# drop-in host-vector entry point

class _HostCallableOperator:
    """A host callable ``v -> A v`` behind the device-operator interface (one
    host round trip per product), so ``fgmres`` accepts any callable as the
    reference does (krylov.py:72-75)."""

    def __init__(self, fn, n: int, device="cuda"):
        from .operators import _CsrProblem
        self.fn, self.shape = fn, (n, n)
        self.prob = _CsrProblem(n, device)

    def matvec(self, X, Y, sel=None):
        import torch
        if sel is not None and int(sel.numel()) == 0:
            return
        n = self.shape[0]
        y = np.asarray(self.fn(X[0, :n].cpu().numpy()), dtype=float)
        if y.shape != (n,):
            raise ValueError(f"operator returned shape {y.shape}, expected ({n},)")
        Y[0, :n] = torch.as_tensor(y, device=Y.device)


def _device_operator(op, n: int):
    """The operator argument of ``fgmres`` as a device operator (krylov.py:72-75):
    this package's device operators pass through, sparse / dense matrices are
    uploaded as a device CSR operator (``operators.CsrOperator``), any other
    callable is applied on the host."""
    from .operators import CsrOperator
    if hasattr(op, "matvec") and hasattr(op, "prob"):
        return op
    if sp.issparse(op) or isinstance(op, np.ndarray):
        if op.shape[1] != n:
            raise ValueError(f"dimension mismatch: {op.shape} @ ({n},)")
        return CsrOperator(sp.csr_matrix(op))
    if callable(op):
        return _HostCallableOperator(op, n)
    raise TypeError("operator must be a sparse matrix, a device operator or a callable")


def fgmres(apply_A, precond, b, restart: int = 20, tol: float = 1e-6, maxit: int = 1000, x0=None):
    """Drop-in ``krylov.fgmres`` (krylov.py:88-182) on the device.

    ``apply_A`` is a device operator of this package (``full_operator`` /
    ``reduced_operator``), a scipy sparse or dense matrix (uploaded as a
    device CSR operator) or any host callable (applied through a host round
    trip), as in the reference (krylov.py:72-75); ``precond`` is None, a
    device preconditioner of this package, or any callable / Preconditioner
    on host vectors (then applied through a host round trip).  Returns
    ``(x, SolveReport)`` with host numpy x.
    """
    import torch
    if restart < 1:
        raise ValueError("restart must be at least 1")
    if tol <= 0:
        raise ValueError("tol must be positive")
    if precond is not None and not (isinstance(precond, Preconditioner) or callable(precond)):
        raise TypeError("preconditioner must be None, callable, or Preconditioner")
    b = np.asarray(b, dtype=float)
    n = b.shape[0]
    apply_A = _device_operator(apply_A, n)
    prob = apply_A.prob
    if n != apply_A.shape[0]:
        raise ValueError(f"dimension mismatch: {apply_A.shape} @ {b.shape}")
    eng = FgmresEngine(1, n, prob.ld, restart)
    B = prob.zeros()
    B[0, :n] = torch.as_tensor(b, device=prob.device)
    X0 = None
    if x0 is not None:
        X0 = prob.zeros()
        X0[0, :n] = torch.as_tensor(np.asarray(x0, dtype=float), device=prob.device)
    P = None
    if precond is not None:
        if hasattr(precond, "apply_device"):
            P = precond.apply_device
        else:
            fn = precond.apply if isinstance(precond, Preconditioner) else precond

            def P(V, Z, sel, idx, fn=fn):
                z = np.asarray(fn(V[0, :n].cpu().numpy()), dtype=float)
                Z[0, :n] = torch.as_tensor(z, device=prob.device)

    rep = eng.solve(apply_A.matvec, P, B, tol=tol, maxit=maxit, x0=X0)[0]
    return eng.x[0, :n].cpu().numpy(), rep


# ---------------------------------------------------------------------------
# ILU(0) of the 1D block

class IluFactorization:
    """Host ILU(0) factor (krylov.py:236-267) + device level schedule."""

    def __init__(self, A):
        A = sp.csr_matrix(A).copy()
        A.sort_indices()
        if A.shape[0] != A.shape[1]:
            raise ValueError("ILU(0) needs a square matrix")
        n = A.shape[0]
        ip = A.indptr.astype(np.int64)
        ix = A.indices.astype(np.int64)
        dpos = np.full(n, -1, dtype=np.int64)
        for i in range(n):
            row = ix[ip[i]:ip[i + 1]]
            h = np.searchsorted(row, i)
            if h < len(row) and row[h] == i:
                dpos[i] = ip[i] + h
        miss = np.nonzero(dpos < 0)[0]
        if len(miss):
            raise ValueError(f"zero pivot: row {miss[0]} has no diagonal entry")
        data = A.data.astype(float).copy()
        lib = _ext.load_library()
        bad = lib.mdp_ilu0_factor_host(n, ip.ctypes.data, ix.ctypes.data, data.ctypes.data, dpos.ctypes.data)
        if bad >= 0:
            raise ValueError(f"zero pivot in row {bad} during ILU(0)")
        self.indptr, self.indices, self.data, self.diag_pos, self.shape = ip, ix, data, dpos, A.shape
        pf = np.zeros(n, dtype=np.int32)
        pb = np.zeros(n, dtype=np.int32)
        lf = np.zeros(n + 1, dtype=np.int32)
        lb = np.zeros(n + 1, dtype=np.int32)
        nf = np.zeros(1, dtype=np.int32)
        nb = np.zeros(1, dtype=np.int32)
        lib.mdp_ilu0_levels_host(n, ip.ctypes.data, ix.ctypes.data, dpos.ctypes.data, pf.ctypes.data,
                                 lf.ctypes.data, nf.ctypes.data, pb.ctypes.data, lb.ctypes.data, nb.ctypes.data)
        self.perm_f, self.lev_f, self.nlev_f = pf, lf, int(nf[0])
        self.perm_b, self.lev_b, self.nlev_b = pb, lb, int(nb[0])


def ilu0(A) -> IluFactorization:
    return IluFactorization(A)


def tree_elimination_order(A) -> np.ndarray:
    """Leaf-first (perfect) elimination order of a matrix whose graph is a forest.

    The 1D block A11 = K11 + w M11 of a tree-shaped vessel graph (eliminated
    Dirichlet rows decoupled) is tree-structured, so LU in this order creates
    no fill: ILU(0) of P A P^T is then the exact factorisation.  Raises
    ValueError when the graph has a cycle.
    """
    A = sp.csr_matrix(A)
    n = A.shape[0]
    G = (abs(A) + abs(A.T)).tocsr()
    G.setdiag(0)
    G.eliminate_zeros()
    deg = np.diff(G.indptr).astype(np.int64)
    queued = deg <= 1
    queue = list(np.nonzero(queued)[0])
    done = np.zeros(n, dtype=bool)
    order = []
    head = 0
    while head < len(queue):
        v = int(queue[head])
        head += 1
        done[v] = True
        order.append(v)
        for u in G.indices[G.indptr[v]:G.indptr[v + 1]]:
            if not done[u]:
                deg[u] -= 1
                if deg[u] <= 1 and not queued[u]:
                    queued[u] = True
                    queue.append(u)
    if len(order) != n:
        raise ValueError("one_d='direct' needs a tree-structured 1D block (the graph has a cycle)")
    return np.asarray(order, dtype=np.int32)


class DirectFactorization(IluFactorization):
    """Exact LU of a tree-structured 1D block: ILU(0) of P A P^T in a leaf-first
    order (no fill, so no dropped terms).  Device sweeps apply
    z = P^T (LU)^-1 P r; replaces splu(A11).solve (harness.py:356-358)."""

    def __init__(self, A):
        A = sp.csr_matrix(A)
        perm = tree_elimination_order(A)
        B = A[perm][:, perm].tocsr()
        B.sort_indices()
        super().__init__(B)
        self.perm = perm


def direct_1d(A) -> DirectFactorization:
    return DirectFactorization(A)


class DeviceIlu:
    """Batched device sweeps of per-system ILU(0) factors (``mdp_ilu``)."""

    def __init__(self, factors, device="cuda"):
        import torch
        nsys = len(factors)
        rows = [f.shape[0] for f in factors]
        stride = max(rows) + 1
        row_start = np.concatenate([[0], np.cumsum(rows)]).astype(np.int32)
        nnz = [len(f.data) for f in factors]
        nz_start = np.concatenate([[0], np.cumsum(nnz)])
        ptr = np.concatenate([f.indptr[:-1] + nz_start[i] for i, f in enumerate(factors)] + [[nz_start[-1]]])
        col = np.concatenate([f.indices for f in factors])
        val = np.concatenate([f.data for f in factors])
        diag = np.concatenate([f.diag_pos + nz_start[i] for i, f in enumerate(factors)])
        lev_f = np.zeros((nsys, stride), dtype=np.int32)
        lev_b = np.zeros((nsys, stride), dtype=np.int32)
        for i, f in enumerate(factors):
            lev_f[i, :f.nlev_f + 1] = f.lev_f[:f.nlev_f + 1]
            lev_b[i, :f.nlev_b + 1] = f.lev_b[:f.nlev_b + 1]
        perms = [getattr(f, "perm", None) for f in factors]
        T = lambda a, dt=torch.int32: torch.as_tensor(np.ascontiguousarray(a).ravel(), dtype=dt, device=device)  # noqa: E731
        self._t = dict(row_start=T(row_start), ptr=T(ptr), col=T(col), val=T(val, torch.float64), diag=T(diag),
                       lev_f=T(lev_f), perm_f=T(np.concatenate([f.perm_f for f in factors])),
                       lev_b=T(lev_b), perm_b=T(np.concatenate([f.perm_b for f in factors])),
                       nlev_f=T([f.nlev_f for f in factors]), nlev_b=T([f.nlev_b for f in factors]))
        if any(pm is not None for pm in perms):
            self._t["perm"] = T(np.concatenate([np.arange(r, dtype=np.int32) if pm is None else pm
                                                for pm, r in zip(perms, rows)]))
        d = _ext.MdpIlu()
        d.nsys, d.lev_stride = nsys, stride
        d.max_rows, d.max_nnz = max(rows), max(nnz)
        for key, t in self._t.items():
            setattr(d, key, t.data_ptr())
        self.desc = d
        self.lib = _ext.lib()

    def apply(self, R, Z, ld, sel=None, nsys=None):
        cnt = int(sel.numel()) if sel is not None else int(nsys)
        _ext.check(self.lib.mdp_ilu0_apply(self.desc, cnt, None if sel is None else sel.data_ptr(),
                                           R.data_ptr(), Z.data_ptr(), ld, _ext.stream()))


def ilu0_apply(fact: IluFactorization, r):
    """Host-vector drop-in for krylov.ilu0_apply (krylov.py:270-276), run on the device
    (a DirectFactorization gives the exact solve of one_d='direct')."""
    import torch
    r = np.asarray(r, dtype=float)
    if r.shape != (fact.shape[0],):
        raise ValueError("right-hand side length mismatch")
    dev = DeviceIlu([fact])
    R = torch.as_tensor(r, device="cuda").reshape(1, -1)
    Z = torch.zeros_like(R)
    dev.apply(R, Z, R.shape[1], nsys=1)
    return Z[0].cpu().numpy()


class IluPreconditioner(Preconditioner):
    """ILU(0) preconditioner (krylov.py:279-283): host factor, device sweeps (x in shared
    memory for small factors, in global memory for the 3D baseline on C)."""

    def __init__(self, A):
        if hasattr(A, "prob") and hasattr(A, "matvec"):  # this package's device reduced_operator
            from .assembly import host_reduced_operator
            A = host_reduced_operator(A.prob.systems[0])
        self.fact = ilu0(A)
        self._dev = None

    def apply(self, r):
        return ilu0_apply(self.fact, r)

    def apply_device(self, V, Z, sel, idx=None):
        """Z_s = ILU(V_s) for the listed systems of (nsys, ld) storages (one factor shared)."""
        if self._dev is None:
            self._dev = DeviceIlu([self.fact])
        for s in (sel.cpu().tolist() if idx is None else idx):
            self._dev.apply(V[s:s + 1], Z[s:s + 1], V.shape[1], nsys=1)


# ---------------------------------------------------------------------------
# smoothing and geometric multigrid (krylov.py:286-387): the baseline the
# paper compares the neural preconditioner against ("AMG(m)").  The hierarchy
# is the reference's own Galerkin construction on the host (scipy products,
# identical matrices); the V-cycles run on the device (csrc/gmg.cu).

def jacobi_smooth(A, r, x0, maxit: int, omega: float = 2.0 / 3.0):
    """``maxit`` weighted-Jacobi sweeps on A x = r from x0, host CSR (krylov.py:289-299)."""
    diag = np.asarray(A.diagonal())
    if np.any(diag == 0.0):
        raise ValueError("Jacobi relaxation needs a nonzero diagonal")
    x = np.array(x0, dtype=float)
    for _ in range(maxit):
        x = x + omega * (r - A @ x) / diag
    return x


def prolongation_3d(n_coarse: int) -> sp.csr_matrix:
    """Trilinear interpolation from an ``n_coarse`` grid to ``2n-1`` points (krylov.py:302-314)."""
    nf = 2 * n_coarse - 1
    rows, cols, vals = [], [], []
    for i in range(nf):
        if i % 2 == 0:
            rows.append(i), cols.append(i // 2), vals.append(1.0)
        else:
            rows += [i, i]
            cols += [i // 2, i // 2 + 1]
            vals += [0.5, 0.5]
    P1 = sp.csr_matrix((vals, (rows, cols)), shape=(nf, n_coarse))
    return sp.kron(sp.kron(P1, P1), P1).tocsr()  # x index fastest


class _DevCsr:
    """int32 / float64 CSR arrays of one matrix on the device."""

    def __init__(self, A, device="cuda"):
        import torch
        A = sp.csr_matrix(A)
        A.sort_indices()
        self.n = A.shape[0]
        self.ptr = torch.as_tensor(A.indptr.astype(np.int32), device=device)
        self.col = torch.as_tensor(A.indices.astype(np.int32), device=device)
        self.val = torch.as_tensor(A.data.astype(np.float64), device=device)

    def args(self):
        return self.n, self.ptr.data_ptr(), self.col.data_ptr(), self.val.data_ptr()


@dataclass
class GmgHierarchy:
    """krylov.py:317-322 plus the device copy of every level."""

    matrices: list          # fine to coarse (host CSR)
    prolongs: list          # prolongs[l]: level l+1 -> level l
    coarse_lu: object
    grid_sizes: list
    device: object = None   # _GmgDevice


# largest coarsest level the device V-cycle inverts densely (17^3 = 4913 unknowns: 190 MB)
GMG_MAX_COARSE = 4913


class _GmgDevice:
    def __init__(self, hier: GmgHierarchy):
        import torch
        self.lib = _ext.lib()
        self.A = [_DevCsr(M) for M in hier.matrices]
        self.d = [torch.as_tensor(np.asarray(M.diagonal(), dtype=np.float64), device="cuda") for M in hier.matrices]
        self.P = [_DevCsr(P) for P in hier.prolongs]
        self.PT = [_DevCsr(P.T.tocsr()) for P in hier.prolongs]
        # the coarsest solve (splu in the reference) as a dense inverse: the level has 27-125 unknowns
        # with the default level count (gmg_build rejects coarsest levels above GMG_MAX_COARSE)
        Mc = hier.matrices[-1].toarray()
        self.Minv = torch.as_tensor(np.linalg.inv(Mc).ravel(), device="cuda")
        f = dict(dtype=torch.float64, device="cuda")
        sizes = [M.shape[0] for M in hier.matrices]
        self.r = [torch.zeros(s, **f) for s in sizes]      # right-hand side per level
        self.z = [torch.zeros(s, **f) for s in sizes]      # solution per level
        self.t = [torch.zeros(s, **f) for s in sizes]      # sweep / residual scratch per level
        self.acc = torch.zeros(sizes[0], **f)
        self.res0 = torch.zeros(sizes[0], **f)

    def _copy(self, src, dst):
        _ext.check(self.lib.mdp_copy_vec(1, None, src.data_ptr(), 0, dst.data_ptr(), 0, None, 0, src.numel(),
                                         _ext.stream()))

    def _sweeps(self, l, r, z, k, omega, from_zero):
        """k Jacobi sweeps on level l (jacobi_smooth, krylov.py:289-299); the result lands in z,
        which holds the start vector unless from_zero."""
        L, st = self.lib, _ext.stream()
        n, pp, cc, vv = self.A[l].args()
        if k == 0:
            if from_zero:
                _ext.check(L.mdp_fill(1, None, z.data_ptr(), 0, n, 0.0, st))
            return
        # ping-pong between z and the level scratch so that the last sweep writes z
        bufs = (z, self.t[l]) if (from_zero and k % 2 == 1) else (self.t[l], z)
        cur = None if from_zero else z
        if not from_zero and k % 2 == 1:
            self._copy(z, self.t[l])  # odd count from a start vector: start from the scratch copy
            cur, bufs = self.t[l], (z, self.t[l])
        for it in range(k):
            dst = bufs[it % 2]
            _ext.check(L.mdp_csr_jacobi(n, pp, cc, vv, self.d[l].data_ptr(), r.data_ptr(),
                                        None if cur is None else cur.data_ptr(), dst.data_ptr(), float(omega), st))
            cur = dst

    def vcycle(self, l, r, z, n_pre, n_post, omega=2.0 / 3.0):
        """z = V(r) on level l (krylov.py:343-356)."""
        L, st = self.lib, _ext.stream()
        if l == len(self.A) - 1:
            _ext.check(L.mdp_dense_matvec(self.A[l].n, self.Minv.data_ptr(), r.data_ptr(), z.data_ptr(), st))
            return
        self._sweeps(l, r, z, n_pre, omega, from_zero=True)
        n, pp, cc, vv = self.A[l].args()
        _ext.check(L.mdp_csr_residual(n, pp, cc, vv, r.data_ptr(), z.data_ptr(), self.t[l].data_ptr(), st))
        nc, qp, qc, qv = self.PT[l].args()
        _ext.check(L.mdp_csr_spmv(nc, qp, qc, qv, self.t[l].data_ptr(), self.r[l + 1].data_ptr(), 0, st))
        self.vcycle(l + 1, self.r[l + 1], self.z[l + 1], n_pre, n_post, omega)
        nf, fp, fc, fv = self.P[l].args()
        _ext.check(L.mdp_csr_spmv(nf, fp, fc, fv, self.z[l + 1].data_ptr(), z.data_ptr(), 1, st))
        self._sweeps(l, r, z, n_post, omega, from_zero=False)

    def apply(self, r, z, cycles, n_pre, n_post):
        """z = GmgPreconditioner.apply(r) (krylov.py:373-387) on device vectors of the fine size."""
        L, st = self.lib, _ext.stream()
        self.vcycle(0, r, z, n_pre, n_post)
        n, pp, cc, vv = self.A[0].args()
        for _ in range(cycles - 1):
            _ext.check(L.mdp_csr_residual(n, pp, cc, vv, r.data_ptr(), z.data_ptr(), self.res0.data_ptr(), st))
            self.vcycle(0, self.res0, self.acc, n_pre, n_post)
            # z = z + V(r - A z)  (krylov.py:385-386)
            _ext.check(L.mdp_axpby(1, None, 1.0, self.acc.data_ptr(), 1.0, z.data_ptr(), 0, n, st))


def gmg_build(grid, fine_operator, levels: int) -> GmgHierarchy:
    """Galerkin hierarchy below a fine operator (krylov.py:325-340), same checks and messages.

    ``fine_operator``: a sparse matrix, a callable grid -> matrix, or this
    package's device ``reduced_operator`` (assembled on the host here)."""
    if levels < 1:
        raise ValueError("levels must be at least 1")
    if hasattr(fine_operator, "prob") and hasattr(fine_operator, "matvec"):  # device reduced_operator
        from .assembly import host_reduced_operator
        A0 = host_reduced_operator(fine_operator.prob.systems[0])
    elif callable(fine_operator) and not sp.issparse(fine_operator):
        A0 = fine_operator(grid)
    else:
        A0 = fine_operator
    if A0.shape != (grid.num_nodes, grid.num_nodes):
        raise ValueError("fine operator shape does not match the grid")
    mats = [sp.csr_matrix(A0)]
    prolongs = []
    sizes = [grid.n]
    n = grid.n
    for _ in range(levels - 1):
        if (n - 1) % 2 != 0 or (n - 1) // 2 + 1 < 3:
            raise ValueError(f"grid with {n} points per edge is not coarsenable")
        nc = (n - 1) // 2 + 1
        P = prolongation_3d(nc)
        mats.append((P.T @ mats[-1] @ P).tocsr())
        prolongs.append(P)
        sizes.append(nc)
        n = nc
    # the device V-cycle inverts the coarsest level densely: a hierarchy that stops
    # coarsening early is rejected rather than densified (levels=1 at 33^3 would be
    # a 35937^2 inverse)
    if mats[-1].shape[0] > GMG_MAX_COARSE:
        raise ValueError(f"coarsest GMG level has {mats[-1].shape[0]} unknowns (> {GMG_MAX_COARSE}); "
                         f"use more levels so the dense coarse solve stays small")
    import scipy.sparse.linalg as spla
    coarse_lu = spla.splu(sp.csc_matrix(mats[-1]))
    hier = GmgHierarchy(mats, prolongs, coarse_lu, sizes)
    hier.device = _GmgDevice(hier)
    return hier


def gmg_vcycle(hierarchy: GmgHierarchy, r, n_pre: int = 1, n_post: int = 1):
    """One V-cycle for A z = r with damped-Jacobi smoothing (krylov.py:343-356), on the device."""
    import torch
    r = np.asarray(r, dtype=float)
    dev = hierarchy.device
    R = torch.as_tensor(r, device="cuda")
    Z = torch.zeros_like(R)
    dev.vcycle(0, R, Z, n_pre, n_post)
    return Z.cpu().numpy()


class GmgPreconditioner(Preconditioner):
    """Fixed number of V-cycles per application, the AMG(m) analogue (krylov.py:359-387)."""

    def __init__(self, hierarchy: GmgHierarchy, cycles: int = 1, n_pre: int = 1, n_post: int = 1):
        if cycles < 1:
            raise ValueError("cycles must be at least 1")
        self.hierarchy = hierarchy
        self.cycles = cycles
        self.n_pre = n_pre
        self.n_post = n_post

    def apply(self, r):
        import torch
        R = torch.as_tensor(np.asarray(r, dtype=float), device="cuda")
        Z = torch.zeros_like(R)
        self.hierarchy.device.apply(R, Z, self.cycles, self.n_pre, self.n_post)
        return Z.cpu().numpy()

    def apply_device(self, V, Z, sel, idx=None):
        """Z_s[:n] = P(V_s[:n]) for the (single) listed system of an (nsys, ld) storage."""
        if idx is None:
            idx = sel.cpu().tolist()
        n = self.hierarchy.matrices[0].shape[0]
        for s in idx:
            self.hierarchy.device.apply(V[s, :n], Z[s, :n], self.cycles, self.n_pre, self.n_post)

"""Device operators over a ``DeviceProblem`` batch (all float64, matrix-free).

``CoupledOperator`` replaces ``full_operator(s)`` (assembly.py:370-374) and
``ReducedOperator`` replaces ``reduced_operator(s)`` (assembly.py:351-353).
Both accept host vectors (``A @ x`` with a numpy array, like the scipy CSR
they replace, via krylov.spmv's contract krylov.py:64-69) or device
storages ``(nsys, ld)`` through ``matvec(X, Y, sel)``.
"""

from __future__ import annotations

import numpy as np

from . import _ext


def sel_args(sel, nsys):
    """(count, device pointer) for a selection tensor or None (= all)."""
    if sel is None:
        return nsys, None
    return int(sel.numel()), sel.data_ptr()


class _DeviceOp:
    def __init__(self, prob):
        self.prob = prob
        self.lib = _ext.lib()

    @property
    def nsys(self):
        return self.prob.nsys

    def __call__(self, x):
        return self @ x

    def _host_apply(self, x, length):
        import torch
        x = np.asarray(x, dtype=float)
        if self.prob.nsys != 1:
            raise ValueError("host-vector application needs a single-system operator")
        if x.shape != (length,):
            raise ValueError(f"dimension mismatch: ({length}, {length}) @ {x.shape}")
        X = self.prob.zeros()
        X[0, :length] = torch.as_tensor(x, device=self.prob.device)
        Y = self.prob.zeros()
        self.matvec(X, Y)
        return Y[0, :length].cpu().numpy()


class CoupledOperator(_DeviceOp):
    """y = [K00 + w M00, w M01; w M10, K11 + w M11] x."""

    @property
    def shape(self):
        n = self.prob.n3 + int(self.prob.n1[0])
        return (n, n)

    def matvec(self, X, Y, sel=None):
        cnt, sp = sel_args(sel, self.prob.nsys)
        _ext.check(self.lib.mdp_coupled_spmv(self.prob.desc, cnt, sp, X.data_ptr(), Y.data_ptr(),
                                             self.prob.s_work.data_ptr(), _ext.stream()))

    def __matmul__(self, x):
        return self._host_apply(x, self.shape[0])


class ReducedOperator(_DeviceOp):
    """y3 = (K00 + w M00) x3 (1D part of the storage ignored)."""

    @property
    def shape(self):
        return (self.prob.n3, self.prob.n3)

    def matvec(self, X, Y, sel=None):
        cnt, sp = sel_args(sel, self.prob.nsys)
        _ext.check(self.lib.mdp_reduced_spmv(self.prob.desc, cnt, sp, X.data_ptr(), Y.data_ptr(),
                                             self.prob.s_work.data_ptr(), _ext.stream()))

    def jacobi(self, R, X, Xout, omega, tmp, sel=None):
        """Xout = X + omega (R - C X) / diag(C); X None means zero (krylov.py:290-299)."""
        cnt, sp = sel_args(sel, self.prob.nsys)
        _ext.check(self.lib.mdp_jacobi_sweep(self.prob.desc, cnt, sp, R.data_ptr(),
                                             None if X is None else X.data_ptr(), Xout.data_ptr(),
                                             float(omega), tmp.data_ptr(), self.prob.s_work.data_ptr(),
                                             _ext.stream()))

    def diagonal(self):
        return self.prob._t["diag_c"][0, :self.prob.n3].cpu().numpy()

    def __matmul__(self, x):
        return self._host_apply(x, self.prob.n3)


class CouplingOps:
    """The Pi gather / Pi^T pull pieces used by the block preconditioner."""

    def __init__(self, prob):
        self.prob = prob
        self.lib = _ext.lib()

    def minus_w_m01(self, Z, Y, sel=None, copy_from=None):
        """Y3 += -w M01 z1 = w T^T W Psi D z1 (the harness.py:391 coupling term, sign folded).

        ``copy_from``: first set Y3 = copy_from3 (same launch as the gather)."""
        cnt, sp = sel_args(sel, self.prob.nsys)
        p = self.prob
        n3 = p.n3
        if copy_from is None:
            _ext.check(self.lib.mdp_pi_gather(p.desc, cnt, sp, None, Z.data_ptr() + 8 * n3, p.ld,
                                              p.s_work.data_ptr(), _ext.stream()))
        else:
            _ext.check(self.lib.mdp_pi_gather_copy(p.desc, cnt, sp, None, Z.data_ptr() + 8 * n3, p.ld,
                                                   p.s_work.data_ptr(), copy_from.data_ptr(), Y.data_ptr(), n3,
                                                   _ext.stream()))
        # s = -W Psi D z1  ->  T^T s * (-w) adds +w T^T W Psi D z1
        _ext.check(self.lib.mdp_pi_scatter(p.desc, cnt, sp, p.s_work.data_ptr(), -1.0, Y.data_ptr(),
                                           p.ld, _ext.stream()))

    def gather(self, X3, X1, S, sel=None):
        cnt, sp = sel_args(sel, self.prob.nsys)
        _ext.check(self.lib.mdp_pi_gather(self.prob.desc, cnt, sp, None if X3 is None else X3.data_ptr(),
                                          None if X1 is None else X1.data_ptr(), self.prob.ld,
                                          S.data_ptr(), _ext.stream()))

    def scatter(self, S, alpha, Y3, sel=None):
        cnt, sp = sel_args(sel, self.prob.nsys)
        _ext.check(self.lib.mdp_pi_scatter(self.prob.desc, cnt, sp, S.data_ptr(), float(alpha),
                                           Y3.data_ptr(), self.prob.ld, _ext.stream()))

    def stencil(self, X, Y, sel=None):
        cnt, sp = sel_args(sel, self.prob.nsys)
        _ext.check(self.lib.mdp_stencil_apply(self.prob.desc, cnt, sp, X.data_ptr(), self.prob.ld,
                                              Y.data_ptr(), self.prob.ld, _ext.stream()))


class _CsrProblem:
    """Single-system storage descriptor for CsrOperator (what FgmresEngine needs)."""

    def __init__(self, n: int, device):
        self.n, self.nsys, self.device = n, 1, device
        self.ld = (n + 31) // 32 * 32

    def zeros(self):
        import torch
        return torch.zeros((1, self.ld), dtype=torch.float64, device=self.device)


class CsrOperator:
    """A general sparse matrix (e.g. the 1D block A11) as a device operator,
    y = A x one row per thread in CSR order (``mdp_csr_spmv``, csrc/gmg.cu),
    so ``krylov.fgmres`` can solve with it (training.generate_rhs)."""

    def __init__(self, A, device="cuda"):
        import scipy.sparse as sp
        import torch
        A = sp.csr_matrix(A)
        if A.shape[0] != A.shape[1]:
            raise ValueError("CsrOperator needs a square matrix")
        self.shape = A.shape
        self.host = A
        self.ptr = torch.as_tensor(A.indptr.astype(np.int32), device=device)
        self.col = torch.as_tensor(A.indices.astype(np.int32), device=device)
        self.val = torch.as_tensor(A.data.astype(np.float64), device=device)
        self.prob = _CsrProblem(A.shape[0], device)
        self.lib = _ext.lib()

    def matvec(self, X, Y, sel=None):
        if sel is not None and int(sel.numel()) == 0:
            return
        _ext.check(self.lib.mdp_csr_spmv(self.shape[0], self.ptr.data_ptr(), self.col.data_ptr(),
                                         self.val.data_ptr(), X.data_ptr(), Y.data_ptr(), 0, _ext.stream()))

    def __matmul__(self, x):
        import torch
        x = np.asarray(x, dtype=float)
        if x.shape != (self.shape[0],):
            raise ValueError(f"dimension mismatch: {self.shape} @ {x.shape}")
        X, Y = self.prob.zeros(), self.prob.zeros()
        X[0, :self.shape[0]] = torch.as_tensor(x, device=self.prob.device)
        self.matvec(X, Y)
        return Y[0, :self.shape[0]].cpu().numpy()

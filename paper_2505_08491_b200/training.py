"""Preconditioner apply path: ``apply_neural``, ``apply_batched``,
``NeuralPreconditioner`` (training.py:287-355), on the device.

z = ||r|| U([r/||r|| | d]) with r = 0 -> 0; with ``smoothing=(maxit, omega)``
the correction is wrapped in weighted-Jacobi pre/post sweeps on C
(training.py:304-311, krylov.py:290-299), each sweep one fused
reduced-SpMV + update on the device.
"""

from __future__ import annotations

import numpy as np

from . import _ext
from .geometry import DistanceField
from .krylov import Preconditioner
from .neural import PATH_TCGEN05, device_net


class BatchedNeural:
    """Neural (+ optional Jacobi) preconditioner over a DeviceProblem batch.

    ``apply_device(V, Z, sel, idx)``: Z_s = P_s(V_s) for the listed systems;
    V, Z are (nsys, ld) float64 storages, only the 3D part is used.
    """

    def __init__(self, net, dists, n: int, ld: int, nsys: int, C=None, smoothing=None,
                 zero_distance: bool = False):
        import torch
        self.net, self.n, self.ld, self.nsys = net, n, ld, nsys
        self.n3 = n ** 3
        self.C = C
        self.smoothing = smoothing
        if smoothing is not None and C is None:
            raise ValueError("smoothing needs the reduced operator")
        dev = "cuda"
        self.D = torch.zeros((nsys, self.n3), dtype=torch.float64, device=dev)
        if not zero_distance:
            self.D.copy_(dists)
        f = dict(dtype=torch.float64, device=dev)
        self.rn = torch.zeros(nsys, **f)
        self.lib = _ext.lib()
        self.work = torch.zeros(self.lib.mdp_arnoldi_work_bytes(nsys, 1, self.n3) // 8 + 1, **f)
        if smoothing is not None:
            self.t1 = torch.zeros((nsys, ld), **f)
            self.t2 = torch.zeros((nsys, ld), **f)
            self.rr = torch.zeros((nsys, ld), **f)
            self.tmp = torch.zeros((nsys, ld), **f)
        self.lib = _ext.lib()

    def _net(self, R, Z, sel, m):
        # ||r|| per system, then the fused pack -> U-Net -> rescale (float64 out)
        _ext.check(self.lib.mdp_norms(m, sel.data_ptr(), R.data_ptr(), self.ld, self.n3, self.rn.data_ptr(),
                                      self.work.data_ptr(), _ext.stream()))
        self.net.apply(self.n, R, self.ld, self.rn, self.D, self.n3, Z, self.ld, sel=sel)

    def first_sweep_spec(self):
        """(out, omega, diag) of the first Jacobi sweep from zero, (omega r) / diag(C), which
        the producer of r may write itself (then call apply_device(..., presmoothed=True))."""
        if self.smoothing is None or self.smoothing[0] < 1:
            return None
        return self.t1, self.smoothing[1], self.C.prob._t["diag_c"]

    def apply_device(self, V, Z, sel, idx=None, presmoothed=False):
        m = int(sel.numel())
        if self.smoothing is None:
            self._net(V, Z, sel, m)
            return
        maxit, omega = self.smoothing
        C = self.C
        # z = S_J(C, r, 0): first sweep from zero needs no SpMV (already in t1 when presmoothed)
        cur = None
        bufs = [self.t1, self.t2]
        start = 0
        if presmoothed and maxit >= 1:
            cur, start = self.t1, 1
        for it in range(start, maxit):
            out = bufs[it % 2]
            C.jacobi(V, cur, out, omega, self.tmp, sel)
            cur = out
        if cur is None:
            Z.index_fill_(0, sel.long(), 0.0)
            cur = Z
        # rr = r - C z and ||rr||, then zn = U(rr)
        C.matvec(cur, self.tmp, sel)
        _ext.check(self.lib.mdp_residual(m, sel.data_ptr(), V.data_ptr(), self.tmp.data_ptr(), self.rr.data_ptr(),
                                         self.ld, self.n3, self.rn.data_ptr(), self.work.data_ptr(),
                                         _ext.stream()))
        # z = z + U(rr) (accumulated by the fused head epilogue), then maxit post sweeps from z
        self.net.apply(self.n, self.rr, self.ld, self.rn, self.D, self.n3, cur, self.ld, sel=sel, accumulate=True)
        src = cur
        for it in range(maxit):
            out = Z if it == maxit - 1 else (self.t2 if src is self.t1 else self.t1)
            C.jacobi(V, src, out, omega, self.tmp, sel)
            src = out
        if maxit == 0 and cur is not Z:
            Z.index_copy_(0, sel.long(), cur.index_select(0, sel.long()))


def _single_problem(C):
    if C is None:
        return None
    if not hasattr(C, "jacobi"):
        raise TypeError("C must be this package's reduced_operator (device)")
    return C


def _row_stride(n3: int) -> int:
    """Row stride of standalone (batch, n^3) device buffers: a multiple of 32
    elements, as DeviceProblem.ld (the Krylov kernels load 16-byte pairs)."""
    return (n3 + 31) // 32 * 32


def apply_neural(params, r, dfield: DistanceField, smoothing=None, C=None, zero_distance: bool = False,
                 path: int = PATH_TCGEN05):
    """One preconditioner application z ~ C^-1 r (training.py:290-319)."""
    import torch
    r = np.asarray(r, dtype=float)
    if r.shape != (dfield.grid.num_nodes,):
        raise ValueError("residual length must match the grid")
    if smoothing is not None and C is None:
        raise ValueError("smoothing needs the reduced operator")
    C = _single_problem(C)
    n = dfield.grid.n
    n3 = n ** 3
    ld = C.prob.ld if C is not None else _row_stride(n3)
    P = BatchedNeural(device_net(params, path), torch.as_tensor(dfield.values, device="cuda")[None], n, ld, 1,
                      C=C, smoothing=smoothing, zero_distance=zero_distance)
    V = torch.zeros((1, ld), dtype=torch.float64, device="cuda")
    V[0, :n3] = torch.as_tensor(r, device="cuda")
    Z = torch.zeros_like(V)
    sel = torch.zeros(1, dtype=torch.int32, device="cuda")
    P.apply_device(V, Z, sel, [0])
    return Z[0, :n3].cpu().numpy()


def apply_batched(params, residuals: list, dfields: list, path: int = PATH_TCGEN05) -> list:
    """Batched network pass over (r, dfield) pairs of one size (training.py:322-338)."""
    import torch
    if len(residuals) != len(dfields):
        raise ValueError("need one distance field per residual")
    sizes = {d.grid.n for d in dfields}
    if len(sizes) != 1:
        raise ValueError("batched application needs a single spatial size")
    n = sizes.pop()
    n3 = n ** 3
    b = len(residuals)
    ld = _row_stride(n3)
    R = torch.zeros((b, ld), dtype=torch.float64, device="cuda")
    R[:, :n3] = torch.as_tensor(np.stack([np.asarray(r, dtype=float) for r in residuals]), device="cuda")
    D = torch.as_tensor(np.stack([d.values for d in dfields]), device="cuda")
    P = BatchedNeural(device_net(params, path), D, n, ld, b)
    Z = torch.zeros_like(R)
    sel = torch.arange(b, dtype=torch.int32, device="cuda")
    P.apply_device(R, Z, sel, list(range(b)))
    Zh = Z[:, :n3].cpu().numpy()
    return [Zh[i].copy() for i in range(b)]


class NeuralPreconditioner(Preconditioner):
    """Stateless apply wrapper binding weights to one graph (training.py:341-355)."""

    def __init__(self, params, dfield: DistanceField, smoothing=None, C=None, zero_distance: bool = False,
                 path: int = PATH_TCGEN05):
        import torch
        self.params = params
        self.dfield = dfield
        self.smoothing = smoothing
        self.C = _single_problem(C)
        self.zero_distance = zero_distance
        n = dfield.grid.n
        ld = self.C.prob.ld if self.C is not None else _row_stride(n ** 3)
        if smoothing is not None and self.C is None:
            raise ValueError("smoothing needs the reduced operator")
        self._dev = BatchedNeural(device_net(params, path), torch.as_tensor(dfield.values, device="cuda")[None],
                                  n, ld, 1, C=self.C, smoothing=smoothing, zero_distance=zero_distance)

    def apply_device(self, V, Z, sel, idx=None):
        self._dev.apply_device(V, Z, sel, idx)

    def apply(self, r):
        return apply_neural(self.params, r, self.dfield, self.smoothing, self.C, self.zero_distance)


# ---------------------------------------------------------------------------
# MDS1 sample files of the dataset directory format (training.py:361-393):
# magic, u32 count, then per sample u32 tag code + n_h little-endian f64

_SAMPLES_MAGIC = b"MDS1"
SAMPLE_TAGS = {"physics": 0, "krylov": 1, "random": 2}
_TAG_NAMES = {v: k for k, v in SAMPLE_TAGS.items()}


def write_samples(path, vectors, tags) -> None:
    """Write (vector, tag) samples; tags in SAMPLE_TAGS."""
    import struct
    if len(vectors) != len(tags):
        raise ValueError("one tag per sample vector")
    with open(path, "wb") as fh:
        fh.write(_SAMPLES_MAGIC)
        fh.write(struct.pack("<I", len(vectors)))
        for v, t in zip(vectors, tags):
            fh.write(struct.pack("<I", SAMPLE_TAGS[t]))
            fh.write(np.asarray(v, dtype="<f8").tobytes())


def read_samples(path) -> tuple:
    """(vectors [count][n_h], tags) of an MDS1 file; ValueError on a bad magic or truncation."""
    import struct
    with open(path, "rb") as fh:
        raw = fh.read()
    if raw[:4] != _SAMPLES_MAGIC:
        raise ValueError(f"bad samples magic {raw[:4]!r}")
    (count,) = struct.unpack_from("<I", raw, 4)
    if count == 0:
        return np.zeros((0, 0)), []
    body = len(raw) - 8
    if body % count:
        raise ValueError("truncated samples file")
    n_h = (body // count - 4) // 8
    vecs, tags, off = [], [], 8
    for _ in range(count):
        (code,) = struct.unpack_from("<I", raw, off)
        off += 4
        vecs.append(np.frombuffer(raw, dtype="<f8", count=n_h, offset=off).astype(float))
        off += 8 * n_h
        tags.append(_TAG_NAMES[code])
    return np.array(vecs), tags

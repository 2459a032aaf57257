"""Preconditioner apply path: ``apply_neural``, ``apply_batched``,
``NeuralPreconditioner`` (training.py:287-355), on the device.

z = ||r|| U([r/||r|| | d]) with r = 0 -> 0; with ``smoothing=(maxit, omega)``
the correction is wrapped in weighted-Jacobi pre/post sweeps on C
(training.py:304-311, krylov.py:290-299), each sweep one fused
reduced-SpMV + update on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

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


# ---------------------------------------------------------------------------
# Dataset construction and training (training.py:36-287, neural.py:475-556),
# on the GPU.  The reference trains in FP64 on the CPU; here the U-Net runs in
# FP64 on the device (PyTorch's CUDA convolutions: tcgen05 has no FP64 MMA and
# training is offline), the loss operator C is this package's device stencil
# operator and Adam is evaluated elementwise in the reference's order.  RNG use
# (initial weights, epoch permutations, random augmentation) is the reference's
# numpy stream, so runs follow the reference step for step.

class SolveError(RuntimeError):
    """training.py:36-37."""


class TrainingDivergedError(RuntimeError):
    """Raised when the loss turns non-finite; carries the batch id (training.py:40-45)."""

    def __init__(self, batch_id: int):
        super().__init__(f"non-finite loss in batch {batch_id}")
        self.batch_id = batch_id


@dataclass(frozen=True)
class TrainingSample:
    """Unit vector + tag + owning graph (training.py:51-65)."""

    vector: np.ndarray
    tag: str
    graph_index: int

    def __post_init__(self):
        norm = np.linalg.norm(self.vector)
        if abs(norm - 1.0) > 1e-12:
            raise ValueError(f"sample vectors live on the unit sphere (norm was {norm})")
        if self.tag not in SAMPLE_TAGS:
            raise ValueError(f"unknown sample tag {self.tag!r}")


@dataclass
class GraphRecord:
    """Graph, distance field, device reduced operator C and samples (training.py:68-75)."""

    graph: object
    dfield: DistanceField
    operator: object
    samples: list


@dataclass(frozen=True)
class AugmentationSpec:
    """none | krylov(count, shift) | random(count) (training.py:78-88)."""

    mode: str = "random"
    count: int = 4
    shift: int = 5

    def __post_init__(self):
        if self.mode not in ("none", "krylov", "random"):
            raise ValueError(f"unknown augmentation mode {self.mode!r}")


@dataclass
class Dataset:
    """training.py:91-106."""

    grid: object
    params: object
    records: list
    train_indices: tuple
    val_indices: tuple
    augmentation: AugmentationSpec

    def train_samples(self):
        return [(i, s) for i in self.train_indices for s in self.records[i].samples]

    def val_samples(self):
        return [(i, s) for i in self.val_indices for s in self.records[i].samples]


@dataclass
class TrainConfig:
    """training.py:109-121."""

    epochs: int
    batch_size: int = 5
    learning_rate: float = 1e-3
    lr_decay: float = 0.97
    alpha: float | None = None
    augmentation: AugmentationSpec = field(default_factory=AugmentationSpec)
    seed: int = 0

    def __post_init__(self):
        if self.alpha is not None and self.alpha <= 0:
            raise ValueError("alpha must be positive")


def generate_rhs(system, tol: float = 1e-4) -> np.ndarray:
    """Physics forcing C-side: solve the 1D block with ILU(0)-FGMRES(20) to ``tol`` on the
    device, then couple (training.py:124-136)."""
    from .assembly import one_d_operator, reduced_rhs
    from .krylov import IluPreconditioner, fgmres
    from .operators import CsrOperator
    A11 = one_d_operator(system)
    x1, report = fgmres(CsrOperator(A11), IluPreconditioner(A11), system.rhs1, restart=20, tol=tol, maxit=500)
    if not report.converged:
        raise SolveError(f"1D solve stalled at residual {report.rel_residual}")
    return reduced_rhs(system, x1)


def augment_krylov(C, b, p: int = 4, p_prime: int = 5) -> list:
    """Krylov vectors q_{p'} .. q_{p'+p-1} of span(b, Cb, ...) by MGS with a second sweep
    (training.py:139-160); C is this package's device operator, the basis lives on the GPU."""
    import warnings
    import torch
    b = np.asarray(b, dtype=float)
    norm_b = np.linalg.norm(b)
    if norm_b == 0:
        raise ValueError("augmentation needs a nonzero seed vector")
    n = b.shape[0]
    X, Y = C.prob.zeros(), C.prob.zeros()
    basis = [torch.as_tensor(b / norm_b, device=X.device)]
    for _ in range(p_prime + p - 1):
        X[0, :n] = basis[-1]
        C.matvec(X, Y)
        w = Y[0, :n].clone()
        for _ in range(2):
            for q in basis:
                w -= torch.dot(w, q) * q
        norm_w = float(torch.linalg.vector_norm(w))
        if norm_w < 1e-12:
            warnings.warn(f"Krylov space exhausted after {len(basis)} vectors")
            break
        basis.append(w / norm_w)
    return [q.cpu().numpy() for q in basis[p_prime:p_prime + p]]


def augment_random(n: int, m: int, seed: int) -> list:
    """m uniform unit vectors (normalised normals), the reference's numpy stream (training.py:163-170)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(m):
        v = rng.standard_normal(n)
        out.append(v / np.linalg.norm(v))
    return out


def _unit(v):
    return v / np.linalg.norm(v)


def build_graph_record(grid, graph, params, augmentation: AugmentationSpec, graph_index: int, seed: int,
                       rhs_tol: float = 1e-4) -> GraphRecord:
    """training.py:177-192."""
    from .assembly import assemble_coupled_system, reduced_operator
    from .geometry import distance_field
    system = assemble_coupled_system(grid, graph, params)
    C = reduced_operator(system)
    dfield = distance_field(graph, grid)
    b = generate_rhs(system, rhs_tol)
    samples = [TrainingSample(_unit(b), "physics", graph_index)]
    if augmentation.mode == "krylov":
        vecs = augment_krylov(C, b, augmentation.count, augmentation.shift)
        samples += [TrainingSample(v, "krylov", graph_index) for v in vecs]
    elif augmentation.mode == "random":
        vecs = augment_random(grid.num_nodes, augmentation.count, seed)
        samples += [TrainingSample(v, "random", graph_index) for v in vecs]
    return GraphRecord(graph, dfield, C, samples)


def build_dataset(grid, graphs: list, params, augmentation: AugmentationSpec = AugmentationSpec(),
                  val_fraction: float = 0.2, seed: int = 0, rhs_tol: float = 1e-4) -> Dataset:
    """One record per graph; the trailing fraction validates (training.py:195-206)."""
    records = [build_graph_record(grid, g, params, augmentation, i, seed=seed * 100_003 + i, rhs_tol=rhs_tol)
               for i, g in enumerate(graphs)]
    n_val = int(round(val_fraction * len(graphs)))
    n_train = len(graphs) - n_val
    return Dataset(grid, params, records, tuple(range(n_train)), tuple(range(n_train, len(graphs))), augmentation)


def compute_alpha(dataset: Dataset) -> float:
    """Mean over training graphs of ||diag(C)||_2 / sqrt(N_h) (training.py:209-214)."""
    n_h = dataset.grid.num_nodes
    vals = [np.linalg.norm(dataset.records[i].operator.diagonal()) / np.sqrt(n_h) for i in dataset.train_indices]
    return float(np.mean(vals))


class _Fp64UNet:
    """The U-Net of neural.py:423-472 in FP64 on the device, differentiable (its
    reverse pass is unet_backward's, neural.py:475-516: ReLU masks by the forward
    output, max-pool routes to the window maximum, concat splits)."""

    def __init__(self, params, device="cuda"):
        import torch
        from .neural import ARCHITECTURE
        self.keys = [k for k, _ in params.arrays()]
        self.t = {k: torch.tensor(a, dtype=torch.float64, device=device) for k, a in params.arrays()}
        self.kind = {name: op for name, op, *_ in ARCHITECTURE}

    def leaves(self):
        return [self.t[k] for k in self.keys]

    def to_params(self):
        from .neural import UNetParams, ARCHITECTURE
        blocks = {}
        for name, *_, has_bias in ARCHITECTURE:
            blocks[name] = {"kernel": self.t[f"{name}.kernel"].detach().cpu().numpy(),
                            "bias": self.t[f"{name}.bias"].detach().cpu().numpy() if has_bias else None}
        return UNetParams(blocks)

    def forward(self, x):
        import torch
        import torch.nn.functional as F

        def step(name, inp, op=0):
            k, b = self.t[f"{name}.kernel"], self.t.get(f"{name}.bias")
            if self.kind[name] == "tconv":
                out = F.conv_transpose3d(inp, k, b, stride=2, output_padding=op)
            else:
                out = F.conv3d(inp, k, b, padding=(k.shape[-1] - 1) // 2)
            return out if name == "head2" else F.relu(out)

        a1 = step("enc1a", x)
        skip1 = step("enc1b", a1)
        skip2 = F.max_pool3d(step("enc2", skip1), 2)
        p2 = F.max_pool3d(step("enc3", skip2), 2)
        bott = step("bottleneck", p2)
        u2 = step("up2", bott, skip2.shape[2] - 2 * bott.shape[2])
        d2 = step("dec2", torch.cat([u2, skip2], 1))
        u1 = step("up1", d2, skip1.shape[2] - 2 * d2.shape[2])
        d1 = step("dec1", torch.cat([u1, skip1], 1))
        return step("head2", step("head1", d1))


def _inputs(dataset: Dataset, chosen, device="cuda"):
    import torch
    n = dataset.grid.n
    xs = np.stack([np.stack([s.vector.reshape(n, n, n), dataset.records[ri].dfield.values.reshape(n, n, n)])
                   for ri, s in chosen])
    return torch.as_tensor(xs, device=device)


class _LossOps:
    """resid = s - C u / alpha and C^T resid per sample through each record's device C
    (symmetric: C^T = C)."""

    def __init__(self, dataset: Dataset):
        self.ds = dataset
        self.buf = {}

    def apply_c(self, ri, v):
        C = self.ds.records[ri].operator
        if ri not in self.buf:
            self.buf[ri] = (C.prob.zeros(), C.prob.zeros())
        X, Y = self.buf[ri]
        n = v.numel()
        X[0, :n] = v
        C.matvec(X, Y)
        return Y[0, :n].clone()


def _fwd_mode():
    import torch
    return torch.backends.cudnn.flags(enabled=True, benchmark=False, deterministic=True)


def risk(params, dataset: Dataset, pairs: list, alpha: float, _net=None) -> float:
    """Mean squared residual mismatch over (record, sample) pairs (training.py:224-233)."""
    import torch
    if not pairs:
        raise ZeroDivisionError("risk over an empty sample list")
    net = _net or _Fp64UNet(params)
    ops = _LossOps(dataset)
    total = torch.zeros((), dtype=torch.float64, device="cuda")
    with torch.no_grad(), _fwd_mode():
        for start in range(0, len(pairs), 16):
            chosen = pairs[start:start + 16]
            us = net.forward(_inputs(dataset, chosen))
            for k, (ri, s) in enumerate(chosen):
                v = torch.as_tensor(s.vector, device="cuda")
                resid = v - ops.apply_c(ri, us[k, 0].reshape(-1)) / alpha
                total += torch.dot(resid, resid)
    return float(total) / len(pairs)


def train(dataset: Dataset, config: TrainConfig) -> tuple:
    """Adam on the empirical risk, on the GPU (training.py:236-284); returns (params, history)
    with one (mean train loss, validation risk) pair per epoch."""
    import torch
    from .neural import init_unet_params
    alpha = config.alpha if config.alpha is not None else compute_alpha(dataset)
    params = init_unet_params(config.seed)
    if config.epochs == 0:
        return params, []
    net = _Fp64UNet(params)
    leaves = net.leaves()
    m = [torch.zeros_like(t) for t in leaves]
    v = [torch.zeros_like(t) for t in leaves]
    beta1, beta2, eps = 0.9, 0.999, 1e-8
    step = 0
    ops = _LossOps(dataset)
    rng = np.random.default_rng(config.seed)
    train_pairs = dataset.train_samples()
    val_pairs = dataset.val_samples()
    history = []
    batch_id = 0
    for epoch in range(config.epochs):
        lr = config.learning_rate * config.lr_decay ** epoch
        order = rng.permutation(len(train_pairs))
        epoch_loss = 0.0
        for start in range(0, len(order), config.batch_size):
            chosen = [train_pairs[i] for i in order[start:start + config.batch_size]]
            for t in leaves:
                t.requires_grad_(True)
            with _fwd_mode():
                us = net.forward(_inputs(dataset, chosen))
                grad_out = torch.empty_like(us)
                loss = torch.zeros((), dtype=torch.float64, device="cuda")
                with torch.no_grad():
                    for k, (ri, s) in enumerate(chosen):
                        sv = torch.as_tensor(s.vector, device="cuda")
                        resid = sv - ops.apply_c(ri, us[k, 0].reshape(-1)) / alpha
                        loss += torch.dot(resid, resid)
                        grad_out[k, 0] = (-(2.0 / (alpha * len(chosen))) * ops.apply_c(ri, resid)).reshape(
                            us.shape[2:])
                batch_loss = float(loss)
                if not np.isfinite(batch_loss):
                    raise TrainingDivergedError(batch_id)
                epoch_loss += batch_loss
                grads = torch.autograd.grad(us, leaves, grad_out)
            # bias-corrected Adam (neural.py:539-556), same operation order
            step += 1
            with torch.no_grad():
                for i, (p, g) in enumerate(zip(leaves, grads)):
                    m[i] = beta1 * m[i] + (1 - beta1) * g
                    v[i] = beta2 * v[i] + (1 - beta2) * g * g
                    m_hat = m[i] / (1 - beta1 ** step)
                    v_hat = v[i] / (1 - beta2 ** step)
                    leaves[i] = (p - lr * m_hat / (torch.sqrt(v_hat) + eps)).detach()
                for key, t in zip(net.keys, leaves):
                    net.t[key] = t
            batch_id += 1
        val_loss = risk(None, dataset, val_pairs, alpha, _net=net) if val_pairs else float("nan")
        history.append((epoch_loss / len(train_pairs), val_loss))
    return net.to_params(), history


def save_dataset(dataset: Dataset, outdir) -> None:
    """Dataset directory: meta.json + per-graph graph JSON, MDF1 distance field, MDS1 samples
    (training.py:399-425)."""
    import json
    from pathlib import Path
    from .geometry import save_distance_field, save_graph
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    p = dataset.params
    meta = {
        "n": dataset.grid.n,
        "params": {"k_omega": p.k_omega, "sigma_omega": p.sigma_omega, "k_lambda": p.k_lambda,
                   "epsilon": p.epsilon},
        "n_graphs": len(dataset.records),
        "train_indices": list(dataset.train_indices),
        "val_indices": list(dataset.val_indices),
        "augmentation": {"mode": dataset.augmentation.mode, "count": dataset.augmentation.count,
                         "shift": dataset.augmentation.shift},
    }
    with open(outdir / "meta.json", "w") as fh:
        json.dump(meta, fh, indent=1)
    for i, rec in enumerate(dataset.records):
        save_graph(rec.graph, outdir / f"graph_{i:04d}.json")
        save_distance_field(rec.dfield, outdir / f"dfield_{i:04d}.bin")
        write_samples(outdir / f"samples_{i:04d}.bin", [s.vector for s in rec.samples],
                      [s.tag for s in rec.samples])


def load_dataset(path) -> Dataset:
    """Load records and re-assemble each graph's (device) reduced operator (training.py:428-447)."""
    import json
    from pathlib import Path
    from .assembly import PhysicalParams, assemble_coupled_system, reduced_operator
    from .geometry import StructuredGrid, load_distance_field, load_graph
    path = Path(path)
    with open(path / "meta.json") as fh:
        meta = json.load(fh)
    grid = StructuredGrid(meta["n"])
    params = PhysicalParams(**meta["params"])
    records = []
    for i in range(meta["n_graphs"]):
        graph = load_graph(path / f"graph_{i:04d}.json")
        dfield = load_distance_field(path / f"dfield_{i:04d}.bin")
        vecs, tags = read_samples(path / f"samples_{i:04d}.bin")
        samples = [TrainingSample(v, t, i) for v, t in zip(vecs, tags)]
        records.append(GraphRecord(graph, dfield, reduced_operator(assemble_coupled_system(grid, graph, params)),
                                   samples))
    return Dataset(grid, params, records, tuple(meta["train_indices"]), tuple(meta["val_indices"]),
                   AugmentationSpec(**meta["augmentation"]))

"""Oracle U-Net forward and preconditioner apply, float64 numpy.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates ``mdprec.neural`` (conv as z-slab im2col + BLAS GEMM, stride-2
transposed conv, floor max-pool, ReLU, concat) and ``mdprec.training``'s
apply path.  Tensor layout (batch, channel, z, y, x) so a flat grid vector
reshapes losslessly (neural.py:10-13).
"""

from __future__ import annotations

import struct

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

from .solver import jacobi_smooth

# name, op, c_in, c_out, kernel, bias (neural.py:342-354)
ARCHITECTURE = (
    ("enc1a", "conv", 2, 16, 3, True),
    ("enc1b", "conv", 16, 32, 3, True),
    ("enc2", "conv", 32, 64, 3, False),
    ("enc3", "conv", 64, 128, 3, False),
    ("bottleneck", "conv", 128, 128, 3, False),
    ("up2", "tconv", 128, 64, 2, False),
    ("dec2", "conv", 128, 64, 3, True),
    ("up1", "tconv", 64, 32, 2, True),
    ("dec1", "conv", 64, 32, 3, True),
    ("head1", "conv", 32, 16, 1, True),
    ("head2", "conv", 16, 1, 1, True),
)
MIN_INPUT_SIZE = 8
RESIDUAL_CHANNEL_GAIN = 16.0
_SLAB_BYTES = 64 * 2 ** 20


def init_unet_params(seed: int = 0) -> dict:
    """Fan-in uniform kernels, zero biases; x16 residual channel, zero head2 (neural.py:391-415)."""
    rng = np.random.default_rng(seed)
    p = {}
    for name, op, cin, cout, ks, has_b in ARCHITECTURE:
        lim = np.sqrt(6.0 / (cin * ks ** 3))
        shape = (cin, cout, ks, ks, ks) if op == "tconv" else (cout, cin, ks, ks, ks)
        p[name] = {"kernel": rng.uniform(-lim, lim, size=shape),
                   "bias": np.zeros(cout) if has_b else None}
    p["enc1a"]["kernel"][:, 0] *= RESIDUAL_CHANNEL_GAIN
    p["head2"]["kernel"][...] = 0.0
    return p


def param_arrays(p: dict):
    """(key, array) in architecture order, kernel before bias (neural.py:365-372)."""
    out = []
    for name, *_, has_b in ARCHITECTURE:
        out.append((f"{name}.kernel", p[name]["kernel"]))
        if has_b:
            out.append((f"{name}.bias", p[name]["bias"]))
    return out


def noisy_params(seed: int = 0, scale: float = 0.05) -> dict:
    """Reference-blessed generic network (tests/test_training.py:232-238)."""
    p = init_unet_params(seed)
    rng = np.random.default_rng(seed + 999)
    for key, arr in param_arrays(p):
        name, part = key.split(".")
        p[name][part] = arr + scale * rng.standard_normal(arr.shape)
    return p


def conv3d(x: np.ndarray, k: np.ndarray, bias=None) -> np.ndarray:
    """Same-padding cross-correlation, z-slab im2col + GEMM (neural.py:110-154)."""
    b, cin, n1, n2, n3 = x.shape
    cout, _, ks = k.shape[:3]
    if ks == 1:
        y = np.einsum("oc,bcs->bos", k.reshape(cout, cin),
                      x.reshape(b, cin, -1)).reshape(b, cout, n1, n2, n3)
    else:
        pad = (ks - 1) // 2
        xp = np.pad(x, ((0, 0), (0, 0)) + ((pad, pad),) * 3)
        W = k.reshape(cout, cin * ks ** 3)
        y = np.empty((b, cout, n1, n2, n3))
        per_plane = n2 * n3 * cin * ks ** 3 * 8
        step = max(1, _SLAB_BYTES // per_plane)
        for bi in range(b):
            for z0 in range(0, n1, step):
                z1 = min(z0 + step, n1)
                win = sliding_window_view(xp[bi, :, z0:z1 + ks - 1], (ks, ks, ks), axis=(1, 2, 3))
                # win: (cin, mz, n2, n3, kz, ky, kx) -> rows (cin,kz,ky,kx), cols voxels
                cols = np.ascontiguousarray(win.transpose(0, 4, 5, 6, 1, 2, 3)).reshape(
                    cin * ks ** 3, -1)
                y[bi, :, z0:z1] = (W @ cols).reshape(cout, z1 - z0, n2, n3)
    if bias is not None:
        y += bias[None, :, None, None, None]
    return y


def transposed_conv3d(x: np.ndarray, k: np.ndarray, output_padding: int, bias=None) -> np.ndarray:
    """Kernel 2 stride 2, size 2n+op; the op plane keeps the bias only (neural.py:215-246)."""
    b, cin, n1, n2, n3 = x.shape
    cout = k.shape[1]
    op = output_padding
    y = np.zeros((b, cout, 2 * n1 + op, 2 * n2 + op, 2 * n3 + op))
    for a in range(2):
        for c in range(2):
            for d in range(2):
                t = np.tensordot(x, k[:, :, a, c, d], axes=([1], [0]))
                y[:, :, a:a + 2 * n1:2, c:c + 2 * n2:2, d:d + 2 * n3:2] = t.transpose(0, 4, 1, 2, 3)
    if bias is not None:
        y += bias[None, :, None, None, None]
    return y


def maxpool3d(x: np.ndarray) -> np.ndarray:
    """2x2x2 max, floor on odd sizes (neural.py:275-290)."""
    b, c, n1, n2, n3 = x.shape
    m1, m2, m3 = n1 // 2, n2 // 2, n3 // 2
    t = x[:, :, :2 * m1, :2 * m2, :2 * m3].reshape(b, c, m1, 2, m2, 2, m3, 2)
    return t.max(axis=(3, 5, 7))


def relu(x):
    return np.maximum(x, 0.0)


def unet_forward(p: dict, x: np.ndarray) -> np.ndarray:
    """Three-level U-Net forward graph (neural.py:423-472)."""
    squeeze = x.ndim == 4
    xb = x[None] if squeeze else x
    if xb.shape[1] != 2:
        raise ValueError("the preconditioner expects exactly 2 input channels")
    if min(xb.shape[2:]) < MIN_INPUT_SIZE:
        raise ValueError(f"spatial size must be at least {MIN_INPUT_SIZE}")

    def conv(name, t, act=True):
        y = conv3d(t, p[name]["kernel"], p[name]["bias"])
        return relu(y) if act else y

    def up(name, t, op):
        return relu(transposed_conv3d(t, p[name]["kernel"], op, p[name]["bias"]))

    a1 = conv("enc1a", xb)
    skip1 = conv("enc1b", a1)
    skip2 = maxpool3d(conv("enc2", skip1))
    p2 = maxpool3d(conv("enc3", skip2))
    bott = conv("bottleneck", p2)
    u2 = up("up2", bott, skip2.shape[2] - 2 * bott.shape[2])
    d2 = conv("dec2", np.concatenate([u2, skip2], axis=1))
    u1 = up("up1", d2, skip1.shape[2] - 2 * d2.shape[2])
    d1 = conv("dec1", np.concatenate([u1, skip1], axis=1))
    h1 = conv("head1", d1)
    y = conv("head2", h1, act=False)
    return y[0] if squeeze else y


def forward_flops(n: int) -> float:
    """Algorithmic FLOPs of one forward at size n."""
    m, q = n // 2, n // 4
    vol = {"enc1a": n ** 3, "enc1b": n ** 3, "enc2": n ** 3, "enc3": m ** 3,
           "bottleneck": q ** 3, "dec2": m ** 3, "dec1": n ** 3, "head1": n ** 3,
           "head2": n ** 3}
    f = 0.0
    for name, op, cin, cout, ks, _ in ARCHITECTURE:
        if op == "tconv":
            out = (2 * q + (m - 2 * q)) ** 3 if name == "up2" else (2 * m + (n - 2 * m)) ** 3
            f += 2.0 * out * cin * cout
        else:
            f += 2.0 * vol[name] * cin * cout * ks ** 3
    return f


# ---------------------------------------------------------------------------
# apply (training.py:290-355)

def apply_neural(p: dict, r: np.ndarray, dvals: np.ndarray, smoothing=None, C=None,
                 zero_distance: bool = False) -> np.ndarray:
    """z = ||r|| U([r/||r|| | d]), optional Jacobi wrap (training.py:290-319)."""
    r = np.asarray(r, dtype=float)
    if r.shape != dvals.shape:
        raise ValueError("residual length must match the grid")
    if smoothing is not None:
        if C is None:
            raise ValueError("smoothing needs the reduced operator")
        maxit, omega = smoothing
        z = jacobi_smooth(C, r, np.zeros_like(r), maxit, omega)
        z = z + apply_neural(p, r - C @ z, dvals, zero_distance=zero_distance)
        return jacobi_smooth(C, r, z, maxit, omega)
    nr = np.linalg.norm(r)
    if nr == 0.0:
        return np.zeros_like(r)
    n = round(len(r) ** (1 / 3))
    d = np.zeros_like(dvals) if zero_distance else dvals
    x = np.stack([(r / nr).reshape(n, n, n), d.reshape(n, n, n)])
    return nr * unet_forward(p, x).reshape(-1)


def apply_batched(p: dict, residuals: list, dfields: list) -> list:
    """One batched forward, per-item norms (zero norm divides by 1) (training.py:322-338)."""
    if len(residuals) != len(dfields):
        raise ValueError("need one distance field per residual")
    n = round(len(dfields[0]) ** (1 / 3))
    norms = [np.linalg.norm(np.asarray(r, dtype=float)) for r in residuals]
    xs = np.stack([np.stack([(np.asarray(r, dtype=float) / (nr if nr else 1.0)).reshape(n, n, n),
                             d.reshape(n, n, n)]) for r, nr, d in zip(residuals, norms, dfields)])
    out = unet_forward(p, xs)
    return [nr * out[i, 0].reshape(-1) for i, nr in enumerate(norms)]


# ---------------------------------------------------------------------------
# MDU3 checkpoint (neural.py:562-632)

_MAGIC = b"MDU3"
_KIND_CONV, _KIND_BIAS, _KIND_TCONV = 0, 1, 2


def save_checkpoint(p: dict, path) -> None:
    ents = []
    for name, op, *_, has_b in ARCHITECTURE:
        ents.append((_KIND_TCONV if op == "tconv" else _KIND_CONV, p[name]["kernel"]))
        if has_b:
            ents.append((_KIND_BIAS, p[name]["bias"]))
    with open(path, "wb") as fh:
        fh.write(_MAGIC + struct.pack("<II", 1, len(ents)))
        for kind, arr in ents:
            fh.write(struct.pack("<BB", kind, arr.ndim) + struct.pack(f"<{arr.ndim}I", *arr.shape))
            fh.write(arr.astype("<f4").tobytes())


def load_checkpoint(path) -> dict:
    raw = open(path, "rb").read()
    if raw[:4] != _MAGIC:
        raise ValueError("bad checkpoint magic")
    ver, cnt = struct.unpack_from("<II", raw, 4)
    if ver != 1:
        raise ValueError(f"unsupported checkpoint version {ver}")
    off, arrs = 12, []
    for _ in range(cnt):
        kind, nd = struct.unpack_from("<BB", raw, off)
        off += 2
        shape = struct.unpack_from(f"<{nd}I", raw, off)
        off += 4 * nd
        c = int(np.prod(shape))
        if off + 4 * c > len(raw):
            raise ValueError("truncated checkpoint")
        arrs.append((kind, np.frombuffer(raw, "<f4", c, off).astype(float).reshape(shape)))
        off += 4 * c
    p, i = {}, 0
    for name, op, cin, cout, ks, has_b in ARCHITECTURE:
        kind, k = arrs[i]
        i += 1
        bias = None
        if has_b:
            bias = arrs[i][1]
            i += 1
        p[name] = {"kernel": k, "bias": bias}
    return p

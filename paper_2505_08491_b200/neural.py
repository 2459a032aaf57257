"""U-Net weights and the device forward pass.

Mirrors the hot-path surface of ``mdprec.neural``: ``ARCHITECTURE``
(neural.py:342-354), ``UNetParams``, ``init_unet_params`` (same RNG order, so
seeds give the reference's weights), MDU3 ``save_checkpoint`` /
``load_checkpoint`` (neural.py:562-632) and ``unet_forward``
(neural.py:423-472), which here runs on the GPU.

Weights are uploaded once as float32 in kernel-specific packed layouts:

  path 0 (tcgen05 TF32, product):  3^3 conv [chunk][tap][quad][Cout][4],
      chunk = 16 input channels, values rounded to TF32;
  path 1 (CUDA-core FP32, check):  3^3 conv [Cout/16][Cin][27][16];
  both: enc1a [16][2][27], tconv [Cout/16][Cin][8][16], head1 [16][32],
      head2 [16].
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from . import _ext

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

PATH_TCGEN05 = 0
PATH_CUDA_CORE = 1


@dataclass
class UNetParams:
    """Weights keyed by block name (neural.py:359-385)."""

    blocks: dict = field(default_factory=dict)

    def arrays(self):
        out = []
        for name, *_, has_bias in ARCHITECTURE:
            out.append((f"{name}.kernel", self.blocks[name]["kernel"]))
            if has_bias:
                out.append((f"{name}.bias", self.blocks[name]["bias"]))
        return out

    def num_params(self) -> int:
        return sum(a.size for _, a in self.arrays())

    def copy(self) -> "UNetParams":
        return UNetParams({k: {"kernel": v["kernel"].copy(),
                               "bias": None if v["bias"] is None else v["bias"].copy()}
                           for k, v in self.blocks.items()})

    def set_array(self, key: str, value) -> None:
        name, part = key.split(".")
        self.blocks[name][part] = value


def init_unet_params(seed: int = 0) -> UNetParams:
    """Fan-in uniform init, x16 residual channel, zero head2 (neural.py:391-415)."""
    rng = np.random.default_rng(seed)
    blocks = {}
    for name, op, cin, cout, ks, has_bias in ARCHITECTURE:
        bound = np.sqrt(6.0 / (cin * ks ** 3))
        shape = (cin, cout, ks, ks, ks) if op == "tconv" else (cout, cin, ks, ks, ks)
        blocks[name] = {"kernel": rng.uniform(-bound, bound, size=shape),
                        "bias": np.zeros(cout) if has_bias else None}
    blocks["enc1a"]["kernel"][:, 0] *= RESIDUAL_CHANNEL_GAIN
    blocks["head2"]["kernel"][...] = 0.0
    return UNetParams(blocks)


def perturbed_params(seed: int = 0, scale: float = 0.05) -> UNetParams:
    """The reference tests' generic random network: init + scale*N(0,1) from seed+999
    (tests/test_training.py:232-238)."""
    p = init_unet_params(seed)
    rng = np.random.default_rng(seed + 999)
    for key, arr in p.arrays():
        p.set_array(key, arr + scale * rng.standard_normal(arr.shape))
    return p


_MAGIC = b"MDU3"
_KIND = {"conv.kernel": 0, "bias": 1, "tconv.kernel": 2}


def save_checkpoint(params: UNetParams, path) -> None:
    """MDU3: magic, u32 version 1, u32 count, entries (u8 kind, u8 ndim, u32 dims, f32 LE)."""
    entries = []
    for name, op, *_, has_bias in ARCHITECTURE:
        entries.append((_KIND["tconv.kernel" if op == "tconv" else "conv.kernel"], params.blocks[name]["kernel"]))
        if has_bias:
            entries.append((_KIND["bias"], params.blocks[name]["bias"]))
    with open(path, "wb") as fh:
        fh.write(_MAGIC + struct.pack("<II", 1, len(entries)))
        for kind, arr in entries:
            fh.write(struct.pack("<BB", kind, arr.ndim) + struct.pack(f"<{arr.ndim}I", *arr.shape))
            fh.write(np.asarray(arr).astype("<f4").tobytes())


def load_checkpoint(path) -> UNetParams:
    """Read and validate an MDU3 checkpoint (neural.py:585-632)."""
    raw = open(path, "rb").read()
    if raw[:4] != _MAGIC:
        raise ValueError(f"bad checkpoint magic {raw[:4]!r}")
    version, count = struct.unpack_from("<II", raw, 4)
    if version != 1:
        raise ValueError(f"unsupported checkpoint version {version}")
    pos, arrays = 12, []
    for _ in range(count):
        if pos + 2 > len(raw):
            raise ValueError("truncated checkpoint")
        kind, nd = struct.unpack_from("<BB", raw, pos)
        pos += 2
        shape = struct.unpack_from(f"<{nd}I", raw, pos)
        pos += 4 * nd
        c = int(np.prod(shape))
        if pos + 4 * c > len(raw):
            raise ValueError("truncated checkpoint")
        arrays.append((kind, np.frombuffer(raw, "<f4", c, pos).astype(float).reshape(shape)))
        pos += 4 * c
    blocks, i = {}, 0
    for name, op, cin, cout, ks, has_bias in ARCHITECTURE:
        if i >= len(arrays):
            raise ValueError("checkpoint has too few layers")
        kind, k = arrays[i]
        i += 1
        want = (cin, cout, ks, ks, ks) if op == "tconv" else (cout, cin, ks, ks, ks)
        if kind != _KIND["tconv.kernel" if op == "tconv" else "conv.kernel"] or k.shape != want:
            raise ValueError(f"layer {name}: unexpected kind/shape in checkpoint")
        b = None
        if has_bias:
            kb, b = arrays[i]
            i += 1
            if kb != _KIND["bias"] or b.shape != (cout,):
                raise ValueError(f"layer {name}: unexpected bias in checkpoint")
        blocks[name] = {"kernel": k, "bias": b}
    if i != len(arrays):
        raise ValueError("checkpoint has extra layers")
    return UNetParams(blocks)


def tf32_round(a: np.ndarray) -> np.ndarray:
    """Round float32 values to TF32 (10-bit mantissa), nearest-even."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)


def pack_conv(kernel: np.ndarray, path: int) -> np.ndarray:
    """(Cout, Cin, 3, 3, 3) -> packed float32 for the given conv path."""
    cout, cin = kernel.shape[:2]
    k = np.asarray(kernel, dtype=np.float32).reshape(cout, cin, 27)
    if path == PATH_CUDA_CORE:
        return np.ascontiguousarray(k.reshape(cout // 16, 16, cin, 27).transpose(0, 2, 3, 1))
    cqc = 4  # 16-channel chunks (unet_tc.cu)
    nch = cin // (4 * cqc)
    if cout <= 64:  # z-tap fold (unet_tc.cu issue_stage_fold): [chunk][dydx][quad][dz][cout][4]
        p = k.reshape(cout, nch, cqc, 4, 3, 9).transpose(1, 5, 2, 4, 0, 3)
        # followed by the same pack of the filter with dy and dz exchanged: the row-remainder launch
        # of odd grids runs the kernel on a (x, z, y) view of the activations (unet_tc.cu tc_conv3)
        kp = np.asarray(kernel, dtype=np.float32).transpose(0, 1, 3, 2, 4).reshape(cout, cin, 27)
        pp = kp.reshape(cout, nch, cqc, 4, 3, 9).transpose(1, 5, 2, 4, 0, 3)
        return tf32_round(np.concatenate([np.ascontiguousarray(p).ravel(), np.ascontiguousarray(pp).ravel()]))
    else:
        p = k.reshape(cout, nch, cqc, 4, 27).transpose(1, 4, 2, 0, 3)  # [chunk][tap][quad][cout][4]
    return tf32_round(np.ascontiguousarray(p))


def pack_tconv(kernel: np.ndarray, path: int = 1) -> np.ndarray:
    """(Cin, Cout, 2, 2, 2) -> path 1 (CUDA cores): [Cout/16][Cin][8][16];
    path 0 (tcgen05): [tap][quad][Cout][4], TF32-rounded (tap = 4a + 2b + c)."""
    cin, cout = kernel.shape[:2]
    if path == PATH_CUDA_CORE:
        k = np.asarray(kernel, dtype=np.float32).reshape(cin, cout // 16, 16, 8)
        return np.ascontiguousarray(k.transpose(1, 0, 3, 2))
    k = np.asarray(kernel, dtype=np.float32).reshape(cin // 4, 4, cout, 8)
    return tf32_round(np.ascontiguousarray(k.transpose(3, 0, 2, 1)))


class DeviceUNet:
    """Packed float32 weights on the device + the ``mdp_unet`` descriptor."""

    def __init__(self, params: UNetParams, path: int = PATH_TCGEN05, device="cuda"):
        import torch
        self.lib = _ext.lib()
        self.path = path
        self.device = device
        self.params = params
        self._t = []
        d = _ext.MdpUnet()
        d.path = path
        for i, (name, op, cin, cout, ks, has_bias) in enumerate(ARCHITECTURE):
            k = params.blocks[name]["kernel"]
            if name == "enc1a":
                w = np.asarray(k, dtype=np.float32).reshape(16, 2, 27)
            elif op == "tconv":
                w = pack_tconv(k, path)
            elif ks == 1:
                w = np.asarray(k, dtype=np.float32).reshape(cout, cin)
            else:
                w = pack_conv(k, path)
            wt = torch.as_tensor(np.ascontiguousarray(w).ravel(), device=device)
            self._t.append(wt)
            d.w[i] = wt.data_ptr()
            if has_bias:
                bt = torch.as_tensor(np.asarray(params.blocks[name]["bias"], dtype=np.float32), device=device)
                self._t.append(bt)
                d.b[i] = bt.data_ptr()
            else:
                d.b[i] = None
        self.desc = d
        self._ws = None
        self._old = []

    def workspace(self, n: int, nb: int):
        """Grow-only activation workspace (a captured CUDA graph may hold the
        current buffer, so it is never freed while this object lives)."""
        import torch
        nbytes = self.lib.mdp_unet_workspace_bytes(n, nb, self.path)
        if self._ws is None or self._ws.numel() < nbytes:
            if self._ws is not None:
                self._old.append(self._ws)
            self._ws = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        return self._ws

    def apply(self, n: int, R, ld: int, rnorm, D, ldd: int, Z, ldz: int, sel=None, nb=None,
              accumulate: bool = False):
        """Z_s = rnorm_i * U([R_s / rnorm_i | D_s]) for the selected systems
        (Z_s += ... with accumulate)."""
        nb = int(sel.numel()) if sel is not None else int(nb)
        if n < MIN_INPUT_SIZE:
            raise ValueError(f"spatial size must be at least {MIN_INPUT_SIZE}")
        ws = self.workspace(n, nb)
        self.desc.n = n
        self.desc.accumulate = int(accumulate)
        _ext.check(self.lib.mdp_unet_apply(self.desc, nb, None if sel is None else sel.data_ptr(),
                                           R.data_ptr(), ld, rnorm.data_ptr(), D.data_ptr(), ldd, Z.data_ptr(),
                                           ldz, ws.data_ptr(), ws.numel(), _ext.stream()))


_DEVICE_NETS = {}


def device_net(params: UNetParams, path: int = PATH_TCGEN05) -> DeviceUNet:
    key = (id(params), path)
    net = _DEVICE_NETS.get(key)
    if net is None or net.params is not params:
        net = DeviceUNet(params, path)
        _DEVICE_NETS[key] = net
    return net


def unet_forward(params: UNetParams, x: np.ndarray, path: int = PATH_TCGEN05) -> np.ndarray:
    """Device forward (neural.py:423-472): (2,n,n,n) or (B,2,n,n,n) -> (1|B,1,n,n,n)."""
    import torch
    x = np.asarray(x, dtype=float)
    squeeze = x.ndim == 4
    if x.ndim not in (4, 5):
        raise ValueError(f"expected a 4D or 5D tensor, got shape {x.shape}")
    xb = x[None] if squeeze else x
    if xb.shape[1] != 2:
        raise ValueError("the preconditioner expects exactly 2 input channels")
    if min(xb.shape[2:]) < MIN_INPUT_SIZE:
        raise ValueError(f"spatial size must be at least {MIN_INPUT_SIZE}")
    b, _, n = xb.shape[:3]
    n3 = n ** 3
    R = torch.as_tensor(np.ascontiguousarray(xb[:, 0].reshape(b, n3)), device="cuda")
    D = torch.as_tensor(np.ascontiguousarray(xb[:, 1].reshape(b, n3)), device="cuda")
    ones = torch.ones(b, dtype=torch.float64, device="cuda")
    Z = torch.empty((b, n3), dtype=torch.float64, device="cuda")
    device_net(params, path).apply(n, R, n3, ones, D, n3, Z, n3, nb=b)
    y = Z.cpu().numpy().reshape(b, 1, n, n, n)
    return y[0] if squeeze else y

"""ctypes binding of the C ABI in ``include/mdp_b200.h`` (libmdp_b200.so).

There is no fallback: if the library is missing or no CUDA device is
visible, every device operation raises ``RuntimeError``.  Device memory
is owned by torch; the library receives raw pointers and the current
torch CUDA stream.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("MDP_LIB_PATH", "")  # A/B timing of alternative builds only
                or Path(__file__).resolve().parent / "lib" / "libmdp_b200.so")

_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_f64 = C.c_double


class MdpProblem(C.Structure):
    _fields_ = [("n", _i32), ("nsys", _i32), ("bc3d", _i32), ("pad0", _i32), ("ld", _i64),
                ("h", _f64), ("k_omega", _f64), ("sigma_omega", _f64),
                ("wc", _vp), ("n1", _vp), ("q_start", _vp), ("t_ptr", _vp), ("t_col", _vp),
                ("t_val", _vp), ("psi_col", _vp), ("psi_val", _vp), ("wq", _vp),
                ("u_start", _vp), ("u_node", _vp), ("u_ptr", _vp), ("u_q", _vp), ("u_val", _vp),
                ("r1_start", _vp), ("k_ptr", _vp), ("k_col", _vp), ("k_val", _vp),
                ("p_ptr", _vp), ("p_q", _vp), ("p_val", _vp), ("diag_c", _vp),
                ("qmax", _i32), ("umax", _i32), ("r1max", _i32), ("pad1", _i32),
                ("ell_q", _vp), ("ell_val", _vp), ("ell_w", _i32), ("pad2", _i32)]


class MdpIlu(C.Structure):
    _fields_ = [("nsys", _i32), ("lev_stride", _i32), ("row_start", _vp), ("ptr", _vp),
                ("col", _vp), ("val", _vp), ("diag", _vp), ("lev_f", _vp), ("perm_f", _vp),
                ("lev_b", _vp), ("perm_b", _vp), ("nlev_f", _vp), ("nlev_b", _vp),
                ("max_rows", _i32), ("max_nnz", _i32), ("perm", _vp)]


class MdpUnet(C.Structure):
    _fields_ = [("n", _i32), ("path", _i32), ("w", _vp * 11), ("b", _vp * 11), ("accumulate", _i32),
                ("reserved", _i32)]


_SIGS = {
    "mdp_coupled_spmv": (_i32, [C.POINTER(MdpProblem), _i32, _vp, _vp, _vp, _vp, _vp]),
    "mdp_reduced_spmv": (_i32, [C.POINTER(MdpProblem), _i32, _vp, _vp, _vp, _vp, _vp]),
    "mdp_stencil_apply": (_i32, [C.POINTER(MdpProblem), _i32, _vp, _vp, _i64, _vp, _i64, _vp]),
    "mdp_pi_gather": (_i32, [C.POINTER(MdpProblem), _i32, _vp, _vp, _vp, _i64, _vp, _vp]),
    "mdp_pi_gather_copy": (_i32, [C.POINTER(MdpProblem), _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp]),
    "mdp_pi_scatter": (_i32, [C.POINTER(MdpProblem), _i32, _vp, _vp, _f64, _vp, _i64, _vp]),
    "mdp_jacobi_sweep": (_i32, [C.POINTER(MdpProblem), _i32, _vp, _vp, _vp, _vp, _f64, _vp, _vp, _vp]),
    "mdp_csr_jacobi": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f64, _vp]),
    "mdp_csr_residual": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mdp_csr_spmv": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "mdp_dense_matvec": (_i32, [_i32, _vp, _vp, _vp, _vp]),
    "mdp_distance_field": (_i32, [_i32, _vp, _i32, _vp, _vp]),
    "mdp_ilu0_factor_host": (_i64, [_i64, _vp, _vp, _vp, _vp]),
    "mdp_ilu0_levels_host": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mdp_ilu0_apply": (_i32, [C.POINTER(MdpIlu), _i32, _vp, _vp, _vp, _i64, _vp]),
    "mdp_arnoldi_work_bytes": (C.c_size_t, [_i32, _i32, _i64]),
    "mdp_arnoldi": (_i32, [_i32, _vp, _vp, _i64, _i64, _vp, _i32, _vp, _i64, _i64, _vp, _vp, _i64,
                           _vp, _vp, _vp]),
    "mdp_norms": (_i32, [_i32, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "mdp_scale": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _vp]),
    "mdp_basis_update": (_i32, [_i32, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _i32, _i64, _vp]),
    "mdp_residual": (_i32, [_i32, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "mdp_axpby": (_i32, [_i32, _vp, _f64, _vp, _f64, _vp, _i64, _i64, _vp]),
    "mdp_copy_vec": (_i32, [_i32, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp]),
    "mdp_fixed_init": (_i32, [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mdp_fixed_start": (_i32, [_i32, _vp, _i32, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
                               _vp, _f64, _vp, _vp]),
    "mdp_arnoldi_givens": (_i32, [_i32, _vp, _vp, _i64, _i64, _vp, _i32, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i32,
                                  _vp, _vp, _vp, _vp, _vp, _vp, _f64, _vp, _vp]),
    "mdp_fixed_finish": (_i32, [_i32, _vp, _i32, _i32, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "mdp_givens_step": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mdp_backsub": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "mdp_fill": (_i32, [_i32, _vp, _vp, _i64, _i64, _f64, _vp]),
    "mdp_copy_slot": (_i32, [_i32, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp]),
    "mdp_unet_workspace_bytes": (C.c_size_t, [_i32, _i32, _i32]),
    "mdp_unet_apply": (_i32, [C.POINTER(MdpUnet), _i32, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _i64,
                              _vp, C.c_size_t, _vp]),
    "mdp_conv3_layer": (_i32, [_i32, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _i32, _vp,
                               _i32, _i32, _i32, _vp, C.c_size_t, _vp]),
    "mdp_conv3_scratch_bytes": (C.c_size_t, [_i32, _i32, _i32, _i32]),
    "mdp_last_error": (C.c_char_p, []),
    "mdp_version": (_i32, []),
    "mdp_launch_count": (C.c_longlong, []),
    "mdp_device_sm_count": (_i32, []),
}

EXPORTED = tuple(_SIGS)

_LIB = None


def load_library(path: Path = LIB_PATH):
    """Load the shared library and declare every exported symbol (no GPU needed)."""
    global _LIB
    if _LIB is None:
        if not path.exists():
            raise RuntimeError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def lib():
    """The library, after checking that a CUDA device is present."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2505_08491_b200 needs a CUDA device (sm_100a); none is visible")
    return load_library()


def check(rc: int) -> None:
    if rc != 0:
        msg = _LIB.mdp_last_error().decode() if _LIB is not None else "library not loaded"
        if rc == 1001:
            raise ValueError(msg)
        raise RuntimeError(f"mdp_b200 error {rc}: {msg}")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def loaded_path() -> str | None:
    return str(LIB_PATH) if _LIB is not None else None


os.environ.setdefault("CUDA_MODULE_LOADING", "LAZY")

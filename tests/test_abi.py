"""C-ABI library: loads without a GPU, exports every symbol the header declares."""

import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2505_08491_b200 import _ext

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "mdp_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mdp_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_ext.EXPORTED)


def test_library_exports_all_symbols():
    lib = _ext.load_library()
    for name in header_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_ext.LIB_PATH)], capture_output=True, text=True).stdout
    for name in header_symbols():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_ext.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_ilu_matches_oracle_bitwise():
    # host-side native ILU(0) factor (no GPU): bitwise against the oracle restatement
    import scipy.sparse as sp
    import oracle
    from paper_2505_08491_b200.krylov import ilu0
    from conftest import golden
    g = golden("asm_cfg2_nc8")
    A = sp.csr_matrix((g["A11_data"], g["A11_indices"], g["A11_indptr"]), shape=tuple(g["A11_shape"]))
    f = ilu0(A)
    assert np.array_equal(f.data, g["ilu_data"])
    assert np.array_equal(f.data, oracle.ilu0(A).data)
    # level schedule is a valid topological order of the sweeps
    pos = np.empty(len(f.perm_f), dtype=int)
    lev = np.empty(len(f.perm_f), dtype=int)
    for L in range(f.nlev_f):
        for r in f.perm_f[f.lev_f[L]:f.lev_f[L + 1]]:
            lev[r] = L
    for i in range(A.shape[0]):
        for p in range(f.indptr[i], f.diag_pos[i]):
            assert lev[f.indices[p]] < lev[i]


def test_zero_pivot_names_row():
    import scipy.sparse as sp
    from paper_2505_08491_b200.krylov import ilu0
    with pytest.raises(ValueError, match="row 1"):
        ilu0(sp.csr_matrix(np.array([[1.0, 1.0], [1.0, 1.0]])))
    A = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]]))
    A.eliminate_zeros()
    with pytest.raises(ValueError, match="diagonal"):
        ilu0(A)


def test_checkpoint_roundtrip_and_init_match_reference(tmp_path):
    import hashlib
    from paper_2505_08491_b200 import neural
    from conftest import golden
    g = golden("apply_solve_n9")
    path = tmp_path / "p.mdu3"
    neural.save_checkpoint(neural.perturbed_params(0), path)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == str(g["ckpt_sha256"])
    p = neural.load_checkpoint(path)
    assert p.num_params() == 1092657
    with pytest.raises(ValueError, match="magic"):
        bad = tmp_path / "bad"
        bad.write_bytes(b"XXXX" + path.read_bytes()[4:])
        neural.load_checkpoint(bad)
    with pytest.raises(ValueError, match="truncated"):
        bad = tmp_path / "trunc"
        bad.write_bytes(path.read_bytes()[:5000])
        neural.load_checkpoint(bad)


def test_weight_packing_layouts():
    from paper_2505_08491_b200 import neural
    rng = np.random.default_rng(0)
    k = rng.standard_normal((64, 32, 3, 3, 3)).astype(np.float32)
    p1 = neural.pack_conv(k, neural.PATH_CUDA_CORE).reshape(4, 32, 27, 16)
    assert p1[1, 5, 13, 7] == k[16 + 7, 5].ravel()[13]
    k128 = rng.standard_normal((128, 32, 3, 3, 3)).astype(np.float32)  # Cout = 128: [chunk][tap][quad][cout][4]
    p0 = neural.pack_conv(k128, neural.PATH_TCGEN05).reshape(2, 27, 4, 128, 4)
    assert abs(p0[1, 13, 2, 40, 3] - k128[40, 16 + 2 * 4 + 3].ravel()[13]) <= 2e-3 * abs(k128[40, 27].ravel()[13])
    # Cout <= 64: z-tap fold layout, followed by the same pack of the dy <-> dz exchanged filter
    p64 = neural.pack_conv(k, neural.PATH_TCGEN05).reshape(2, 2, 9, 4, 3, 64, 4)
    assert abs(p64[0, 1, 4, 2, 1, 40, 3] - k[40, 16 + 2 * 4 + 3, 1, 1, 1]) <= 2e-3 * abs(k[40, 27, 1, 1, 1])
    k32 = rng.standard_normal((32, 64, 3, 3, 3)).astype(np.float32)  # Cout = 32: z-tap fold layout
    pf = neural.pack_conv(k32, neural.PATH_TCGEN05).reshape(2, 4, 9, 4, 3, 32, 4)  # [copy][chunk][dydx][quad][dz][cout][4]
    assert abs(pf[0, 2, 7, 1, 2, 30, 3] - k32[30, 2 * 16 + 1 * 4 + 3, 2, 2, 1]) <= 1e-3 * abs(k32[30, 39, 2, 2, 1])
    # permuted copy: unit 7 = (line offset 2, dx 1), plane offset 0 -> physical (dz, dy, dx) = (2, 0, 1)
    assert abs(pf[1, 2, 7, 1, 0, 30, 3] - k32[30, 39, 2, 0, 1]) <= 1e-3 * abs(k32[30, 39, 2, 0, 1])
    t = rng.standard_normal((64, 32, 2, 2, 2)).astype(np.float32)
    pt = neural.pack_tconv(t).reshape(2, 64, 8, 16)
    assert pt[1, 10, 5, 3] == t[10, 16 + 3].ravel()[5]
    p0 = neural.pack_tconv(t, neural.PATH_TCGEN05).reshape(8, 16, 32, 4)  # [tap][quad][cout][4]
    assert abs(p0[5, 3, 17, 2] - t[3 * 4 + 2, 17].ravel()[5]) <= 1e-3 * abs(t[14, 17].ravel()[5])


_CTYPE = {"int32_t": "c_int", "int64_t": "c_long", "double": "c_double", "float": "c_float", "size_t": "c_ulong"}


def header_struct(name):
    """(field, ctype-name) pairs of ``typedef struct name {...}`` in the header."""
    text = (ROOT / "include" / "mdp_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    body = re.search(rf"typedef struct {name}\s*\{{(.*?)\}}\s*{name}\s*;", text, flags=re.S).group(1)
    out = []
    for decl in body.split(";"):
        decl = " ".join(decl.split())
        if not decl:
            continue
        m = re.match(r"(const )?(\w+)(\*?) (.*)", decl)
        _, base, ptr, names = m.groups()
        for nm in names.split(","):
            nm = nm.strip()
            arr = re.match(r"(\*?)(\w+)\[(\d+)\]", nm)
            star = ptr or nm.startswith("*")
            nm = nm.lstrip("*")
            if arr:
                out.append((arr.group(2), "ptr", int(arr.group(3))))
            else:
                out.append((nm, "ptr" if star else _CTYPE[base], 1))
    return out


def _binding_fields(struct):
    import ctypes as C
    out = []
    for nm, ty in struct._fields_:
        if issubclass(ty, C.Array):
            out.append((nm, "ptr" if ty._type_ is C.c_void_p else ty._type_.__name__, ty._length_))
        else:
            out.append((nm, "ptr" if ty is C.c_void_p else ty.__name__, 1))
    return out


@pytest.mark.parametrize("cname,pyname", [("mdp_problem", "MdpProblem"), ("mdp_ilu", "MdpIlu"),
                                          ("mdp_unet", "MdpUnet")])
def test_struct_layout_header_vs_binding(cname, pyname):
    """Every descriptor struct of the header and its ctypes mirror agree field by field
    (a shorter ctypes struct would make the C side read past its end)."""
    assert header_struct(cname) == _binding_fields(getattr(_ext, pyname))


def test_integration_doc_struct_matches_binding():
    """The MdpProblem snippet in INTEGRATION.md is the full struct, not an abridged prefix."""
    text = (ROOT / "INTEGRATION.md").read_text()
    snippet = re.search(r"class MdpProblem\(C\.Structure\):.*?_fields_ = \[(.*?)\]\n", text, flags=re.S).group(1)
    names = re.findall(r'\("(\w+)"', snippet)
    assert names == [nm for nm, _ in _ext.MdpProblem._fields_]

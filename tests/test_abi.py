"""CPU-only checks of the C ABI: the library loads, exports every symbol include/asot.h declares,
and its host-side logic (argument checks, tile enumeration) behaves.  No compute calls."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "asot.h")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(asot_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2310_16123_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib.load()


def test_exports_every_header_symbol(lib):
    from paper_2310_16123_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in asot.h but not exported"
    assert set(syms) == set(_lib.EXPORTED), "binding signature table out of sync with asot.h"
    assert lib.asot_abi_version() == 1


def header_param_types():
    """{function: [C parameter types]} parsed from include/asot.h (comments stripped)."""
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    out = {}
    for m in re.finditer(r"\b(asot_[a-z0-9_]+)\s*\(([^;{)]*)\)\s*;", src):
        params = [p.strip() for p in m.group(2).split(",") if p.strip() and p.strip() != "void"]
        out[m.group(1)] = params
    return out


def _ctype_for(decl: str):
    decl = " ".join(decl.split())
    if "*" in decl:
        return ctypes.c_void_p
    base = decl.rsplit(" ", 1)[0] if " " in decl else decl
    base = base.replace("const ", "")
    return {"int64_t": ctypes.c_int64, "int32_t": ctypes.c_int32, "float": ctypes.c_float,
            "size_t": ctypes.c_size_t, "asot_precision": ctypes.c_int32, "uint32_t": ctypes.c_uint32,
            "double": ctypes.c_double}[base]


def test_binding_signatures_match_header():
    """Every ctypes signature in _lib has the header's parameter count and scalar types (a
    mismatch would silently shift arguments)."""
    from paper_2310_16123_b200 import _lib
    hdr = header_param_types()
    for name, (_, args) in _lib._SIGS.items():
        assert name in hdr, name
        params = hdr[name]
        assert len(args) == len(params), f"{name}: binding {len(args)} args, header {len(params)}"
        for a, decl in zip(args, params):
            want = _ctype_for(decl)
            if want is ctypes.c_void_p:
                assert a is ctypes.c_void_p or (hasattr(a, "_type_") and isinstance(a._type_, type)), (name, decl)
            else:
                assert a is want or (ctypes.sizeof(a) == ctypes.sizeof(want) and
                                     (a is ctypes.c_float) == (want is ctypes.c_float) and
                                     (a is ctypes.c_double) == (want is ctypes.c_double)), (name, decl, a)


def test_num_tiles_and_enumeration(lib):
    import paper_2310_16123_b200 as asot
    for n in (1, 2, 15, 16, 17, 33, 64, 100, 1000):
        nb = (n + 15) // 16
        assert asot.num_tiles(n) == nb * (nb + 1)
        i, j, v = asot.tile_pairs(n)
        got = sorted(zip(i[v].tolist(), j[v].tolist()))
        want = [(a, b) for a in range(n) for b in range(a + 1, n)]
        assert got == want                      # every unordered pair exactly once (Def. 1)
        assert np.all(i[v] < j[v])
    # sub-ranges concatenate to the whole
    n = 100
    nt = asot.num_tiles(n)
    parts = [asot.tile_pairs(n, a, b) for a, b in ((0, 7), (7, 30), (30, nt))]
    i_all, j_all, v_all = asot.tile_pairs(n)
    np.testing.assert_array_equal(np.concatenate([p[0] for p in parts]), i_all)
    np.testing.assert_array_equal(np.concatenate([p[2] for p in parts]), v_all)


def test_host_argument_errors(lib):
    # invalid arguments are rejected synchronously without touching any device pointer
    rc = lib.asot_pairwise_sinkhorn(None, 10, 16, None, 1.0, 0.05, 10, 1, None, None, 5, None, None,
                                    None, 0, None)
    assert rc == 1
    assert b"null" in lib.asot_last_error()
    fake = 0x1000
    rc = lib.asot_pairwise_sinkhorn(fake, 10, 16, fake, 1.0, 0.0, 10, 1, fake, fake, 5, fake, fake,
                                    fake, 0, None)
    assert rc == 1 and b"eps" in lib.asot_last_error()
    rc = lib.asot_pairwise_sinkhorn(fake, 10, 16, fake, 5.0, 0.05, 10, 1, fake, fake, 5, fake, fake,
                                    fake, 0, None)
    assert rc == 1 and b"80" in lib.asot_last_error()      # max(C)/eps guard (R#12)
    rc = lib.asot_pairwise_sinkhorn(fake, 10, 2048, fake, 1.0, 0.05, 10, 1, fake, fake, 5, fake,
                                    fake, fake, 0, None)
    assert rc == 5                                         # K > 1024 unsupported
    rc = lib.asot_pairwise_sinkhorn(fake, 10, 16, fake, 1.0, 0.05, 10, 1, fake, fake, 5, fake, fake,
                                    fake, 16, None)
    assert rc == 6                                         # workspace too small
    rc = lib.asot_pairwise_sinkhorn(fake, 10, 16, fake, 1.0, 0.05, 10, 1, None, None, 0, None, fake,
                                    None, 0, None)
    assert rc == 0                                         # empty pair list: nothing to do
    rc = lib.asot_distance_matrix(None, None, None, None, 10, 4, None, 16, fake, 1.0, 0.05, 10, 1,
                                  None, 0, 10**6, fake, None, None, None, fake, fake, 1 << 20, None)
    assert rc == 1 and b"tile range" in lib.asot_last_error()


def test_workspace_queries(lib):
    a = lib.asot_distance_matrix_workspace_bytes(1000, 35000, 128, 0)
    assert a >= 1000 * 128 * 4 + 35000 * 4 + 2 * 128 * 128 * 4
    b = lib.asot_distance_matrix_host_workspace_bytes(1000, 35000, 32, 128, 0)
    assert b >= a + 1000 * 1000 * 4


def test_product_path_has_no_oracle_or_cpu_fallback():
    """The product package never imports oracle/ and has no numpy/torch compute fallback."""
    pkg = os.path.join(ROOT, "paper_2310_16123_b200")
    for name in os.listdir(pkg):
        if name.endswith(".py"):
            src = open(os.path.join(pkg, name)).read()
            assert "oracle" not in src.replace("never imports oracle", ""), name
            assert "torch.exp" not in src and "np.exp" not in src and "matmul" not in src, name


def test_binding_rejects_malformed_pair_lists():
    """The binding validates pair lists and shapes before any device call: int64 index
    tensors (the ABI reads i32), unequal lengths, a cost of the wrong size, non-f32 histograms."""
    import torch
    import paper_2310_16123_b200 as asot
    H = torch.zeros(10, 16)
    C = torch.zeros(16, 16)
    i32 = torch.zeros(5, dtype=torch.int32)
    with pytest.raises(ValueError, match="int32"):
        asot.pairwise_sinkhorn(H, C, 0.05, 10, torch.zeros(5, dtype=torch.int64), i32)
    with pytest.raises(ValueError, match="entries"):
        asot.pairwise_sinkhorn(H, C, 0.05, 10, i32, torch.zeros(4, dtype=torch.int32))
    with pytest.raises(ValueError, match="cost"):
        asot.pairwise_sinkhorn(H, torch.zeros(15, 15), 0.05, 10, i32, i32)
    with pytest.raises(ValueError, match="float32"):
        asot.pairwise_sinkhorn(H.double(), C, 0.05, 10, i32, i32)
    with pytest.raises(ValueError, match="int32"):
        asot.exact_asot_pairs(H, C, i32.long(), i32)
    with pytest.raises(ValueError, match="cuda"):   # well-formed CPU tensors: no CPU path
        asot.pairwise_sinkhorn(H, C, 0.05, 10, i32, i32)

"""C-ABI checks that need no GPU: the library loads, exports every symbol declared in
include/turbo_ns.h, and rejects bad arguments before touching the device."""
import ctypes
import os
import re

import numpy as np

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "turbo_ns.h")


def declared_symbols():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:ns|nsx)_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["ns_orthogonalize", "ns_orthogonalize_batched", "nsx_gram", "nsx_precondition",
              "nsx_poly", "nsx_update", "ns_read_flags", "ns_workspace_size"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2512_04632_b200 import _lib
    for s in declared_symbols():
        assert hasattr(_lib.lib, s), s
    assert set(_lib.EXPORTS) == set(declared_symbols())
    assert _lib.lib.ns_abi_version() == 2


def test_invalid_arguments_rejected_on_host():
    from paper_2512_04632_b200._lib import NS_ERR_INVALID_VALUE, lib
    c = (ctypes.c_float * 12)(*([1.0] * 12))
    v = ctypes.c_void_p(0x1000)
    # iters out of range, NULL coeffs, bad precond, bad shape, NULL X
    assert lib.ns_orthogonalize(v, 8, 8, 1, 0, c, 2, 0, None) == NS_ERR_INVALID_VALUE
    assert lib.ns_orthogonalize(v, 8, 8, 1, 65, c, 2, 0, None) == NS_ERR_INVALID_VALUE
    assert lib.ns_orthogonalize(v, 8, 8, 1, 4, None, 2, 0, None) == NS_ERR_INVALID_VALUE
    assert lib.ns_orthogonalize(v, 8, 8, 1, 4, c, 7, 0, None) == NS_ERR_INVALID_VALUE
    assert lib.ns_orthogonalize(v, 0, 8, 1, 4, c, 2, 0, None) == NS_ERR_INVALID_VALUE
    assert lib.ns_orthogonalize(None, 8, 8, 1, 4, c, 2, 0, None) == NS_ERR_INVALID_VALUE
    assert lib.ns_orthogonalize(v, 8, 8, 0, 4, c, 2, 0, None) == NS_ERR_INVALID_VALUE
    bad = (ctypes.c_float * 12)(*([float("nan")] * 12))
    assert lib.ns_orthogonalize(v, 8, 8, 1, 4, bad, 2, 0, None) == NS_ERR_INVALID_VALUE
    assert lib.ns_last_error()


def test_call_limits_rejected_on_host():
    """Header limits checked before anything touches the device (tile words pack
    the job index in 20 bits): 2^20 matrices in one call, a matrix pointer not aligned to
    its element size, a dimension beyond 2^30."""
    import numpy as np
    from paper_2512_04632_b200._lib import NS_ERR_INVALID_VALUE, NS_ERR_NOT_SUPPORTED, lib
    c = (ctypes.c_float * 12)(*([1.0] * 12))
    cnt = 1 << 20
    ptrs = np.full(cnt, 0x1000, dtype=np.uint64)
    dims = np.full(cnt, 8, dtype=np.int64)
    X = ptrs.ctypes.data_as(ctypes.POINTER(ctypes.c_void_p))
    M = dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    assert lib.ns_orthogonalize_batched(X, None, M, M, cnt, 4, c, 2, 0, None) == NS_ERR_NOT_SUPPORTED
    assert b"2^20" in lib.ns_last_error()
    odd = ctypes.c_void_p(0x1001)
    assert lib.ns_orthogonalize(odd, 8, 8, 1, 4, c, 2, 0, None) == NS_ERR_NOT_SUPPORTED
    v = ctypes.c_void_p(0x1000)
    assert lib.ns_orthogonalize(v, (1 << 30) + 1, 8, 1, 4, c, 2, 0, None) == NS_ERR_INVALID_VALUE


def test_workspace_size_host_only():
    import paper_2512_04632_b200 as ns
    b = ns.workspace_size([(768, 768)])
    assert b >= 3 * 768 * 768 * 2 + 768 * 4


def test_product_coeffs_match_test_tables():
    from paper_2512_04632_b200 import coeffs as P
    from synth import coeffs as S
    assert P.MUON_PLUS_5 == S.MUON_PLUS_5 and P.MUON_CONST == S.MUON_CONST
    assert P.turbo(4) == S.turbo(4)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2512_04632_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b|ns_oracle|#include.*oracle", src, re.M), f


def test_workspace_size_groups_and_batch():
    """ns_workspace_size sizes a call as the planner runs it: a bf16 list mixing a TMA-
    unaligned shape (n = 49) with aligned ones is two plans, each with its own 1 KiB header;
    `batch` repeats every shape (the two-plan split was under-counted)."""
    import paper_2512_04632_b200 as ns
    a, u = (1024, 1024), (960, 49)
    assert ns.workspace_size([a, u]) == ns.workspace_size([a]) + ns.workspace_size([u])
    assert ns.workspace_size([a, a, a]) == ns.workspace_size([a], batch=3)
    assert ns.workspace_size([a, u], batch=2) == ns.workspace_size([a, a]) + ns.workspace_size([u, u])

"""ctypes loader for libturbons.so (the C ABI in include/turbo_ns.h).

There is no fallback: if the shared library is missing or fails to load, importing the
package raises, naming the build command.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libturbons.so")

NS_OK, NS_ERR_INVALID_VALUE, NS_ERR_NOT_SUPPORTED, NS_ERR_WORKSPACE, NS_ERR_CUDA = range(5)
PRECOND = {"none": 0, "frobenius": 1, "aol": 2}
DTYPE_BF16, DTYPE_FP32 = 0, 1
FLAG_ZERO_SCALE, FLAG_NONFINITE = 1, 2

EXPORTS = [
    "ns_orthogonalize", "ns_orthogonalize_batched", "ns_orthogonalize_cast", "ns_orthogonalize_peers", "ns_muon_step", "ns_muon_apply", "ns_workspace_size", "ns_set_workspace", "ns_read_flags",
    "ns_launch_count", "ns_set_path", "ns_status_string", "ns_last_error", "ns_abi_version",
    "ns_shutdown", "ns_profile_enable", "ns_profile_read", "nsx_epilogue_counters", "nsx_gram", "nsx_precondition", "nsx_poly", "nsx_update",
]


class NSError(RuntimeError):
    pass


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python paper_2512_04632_b200/build.py` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    c_i64, c_int, c_vp, c_float = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_float
    c_fp = ctypes.POINTER(ctypes.c_float)
    lib.ns_orthogonalize.argtypes = [c_vp, c_i64, c_i64, c_i64, c_int, c_fp, c_int, c_int, c_vp]
    lib.ns_orthogonalize_batched.argtypes = [
        ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
        c_i64, c_int, c_fp, c_int, c_int, c_vp]
    lib.ns_orthogonalize_cast.argtypes = [
        ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
        c_i64, c_int, c_fp, c_int, c_vp]
    lib.ns_orthogonalize_peers.argtypes = [
        ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_int, ctypes.POINTER(c_i64),
        ctypes.POINTER(c_i64), c_i64, c_int, c_fp, c_int, c_int, c_vp]
    lib.ns_muon_step.argtypes = [
        ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
        ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), c_i64, c_int, c_int, c_float, c_float, c_float, c_float,
        c_int, c_int, c_fp, c_int, c_vp]
    lib.ns_muon_apply.argtypes = [ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_i64),
                                  ctypes.POINTER(c_i64), c_i64, c_int, c_float, c_float, c_vp]
    lib.ns_workspace_size.argtypes = [ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), c_i64, c_i64, c_int,
                                      ctypes.POINTER(ctypes.c_size_t)]
    lib.ns_set_workspace.argtypes = [c_vp, ctypes.c_size_t, c_vp]
    lib.ns_read_flags.argtypes = [c_vp, ctypes.POINTER(ctypes.c_uint32)]
    lib.ns_launch_count.restype = ctypes.c_uint64
    lib.ns_launch_count.argtypes = []
    lib.ns_set_path.argtypes = [c_int]
    lib.ns_set_path.restype = c_int
    lib.ns_status_string.restype = ctypes.c_char_p
    lib.ns_status_string.argtypes = [c_int]
    lib.ns_last_error.restype = ctypes.c_char_p
    lib.ns_last_error.argtypes = []
    lib.ns_abi_version.restype = c_int
    lib.ns_shutdown.argtypes = []
    lib.ns_shutdown.restype = None
    lib.ns_profile_enable.argtypes = [c_int]
    lib.ns_profile_enable.restype = None
    lib.ns_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64), c_int]
    lib.nsx_epilogue_counters.argtypes = [ctypes.POINTER(ctypes.c_uint64), c_int]
    lib.nsx_gram.argtypes = [c_vp, c_i64, c_i64, c_vp, c_vp, c_int, c_vp]
    lib.nsx_precondition.argtypes = [c_vp, c_i64, c_int, c_vp, c_vp, c_int, c_vp]
    lib.nsx_poly.argtypes = [c_vp, c_i64, c_float, c_float, c_vp, c_vp, c_int, c_vp]
    lib.nsx_update.argtypes = [c_vp, c_i64, c_i64, c_vp, c_float, c_vp, c_vp, c_int, c_vp]
    for name in EXPORTS:
        if name not in ("ns_launch_count", "ns_set_path", "ns_status_string", "ns_last_error",
                        "ns_abi_version", "ns_shutdown", "ns_profile_enable"):
            getattr(lib, name).restype = c_int
    return lib


lib = _load()


def check(status: int, what: str) -> None:
    if status != NS_OK:
        msg = lib.ns_last_error().decode(errors="replace")
        name = lib.ns_status_string(status).decode()
        raise NSError(f"{what}: {name}: {msg}")

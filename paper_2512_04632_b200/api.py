"""Python binding of libturbons.so: argument marshalling only.

Every step of the path runs in the library's CUDA kernels; this module passes device
pointers, shapes, coefficients and the current CUDA stream through the C ABI
(include/turbo_ns.h).  PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import torch

from . import coeffs as _coeffs
from ._lib import DTYPE_BF16, DTYPE_FP32, PRECOND, check, lib

__all__ = [
    "orthogonalize", "orthogonalize_list", "workspace_size", "read_flags", "launch_count",
    "set_path", "set_workspace", "muon_apply", "shutdown", "profile_enable", "profile_read", "gram", "precondition", "poly", "update", "default_coeffs",
]


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return DTYPE_BF16
    if t.dtype == torch.float32:
        return DTYPE_FP32
    raise TypeError(f"unsupported dtype {t.dtype}; use bfloat16 or float32")


def _check_tensor(t: torch.Tensor, name: str = "tensor") -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (row-major)")


class _Nothing:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_NOTHING = _Nothing()


def _on_device(dev: torch.device):
    """torch.cuda.device(dev), skipped when dev is already current (a per-call host cost)."""
    return _NOTHING if dev.index == torch.cuda.current_device() else torch.cuda.device(dev)


def _stream(t: torch.Tensor | None = None) -> ctypes.c_void_p:
    dev = t.device if t is not None else None
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


_DEFAULT_COEFFS: dict = {}


def _coeff_array(iters: int, coeffs, precond: str):
    if coeffs is None:  # the default schedules are data: one ctypes array per (iters, precond)
        key = (iters, precond)
        arr = _DEFAULT_COEFFS.get(key)
        if arr is None:
            arr = _DEFAULT_COEFFS[key] = _coeff_array(iters, default_coeffs(iters, precond), precond)
        return arr
    flat = [float(v) for t in coeffs for v in t] if len(coeffs) and hasattr(coeffs[0], "__len__") \
        else [float(v) for v in coeffs]
    if len(flat) != 3 * iters:
        raise ValueError(f"need {iters} (a, b, c) triples, got {len(flat)} values")
    return (ctypes.c_float * len(flat))(*flat)


def default_coeffs(iters: int = 4, precond: str = "aol"):
    """Turbo-Muon: the last `iters` Muon+ triples; Muon+ for Frobenius."""
    return _coeffs.turbo(iters) if precond == "aol" else _coeffs.muon_plus(iters)


def orthogonalize(x: torch.Tensor, iters: int = 4, precond: str = "aol", coeffs=None) -> torch.Tensor:
    """In place: x (m x n, or batch x m x n) <- NS_iters(precond(x)).  Returns x."""
    _check_tensor(x, "x")
    if x.dim() == 2:
        batch, (m, n) = 1, x.shape
    elif x.dim() == 3:
        batch, m, n = x.shape
    else:
        raise ValueError("x must be 2-D or 3-D")
    if x.numel() == 0:
        return x
    c = _coeff_array(iters, coeffs, precond)
    with _on_device(x.device):
        st = lib.ns_orthogonalize(ctypes.c_void_p(x.data_ptr()), m, n, batch, iters, c,
                                  PRECOND[precond], _dtype_code(x), _stream(x))
    check(st, "ns_orthogonalize")
    return x


def _check_list(xs, out):
    dt = _dtype_code(xs[0])
    for i, t in enumerate(xs):
        _check_tensor(t, f"xs[{i}]")
        if t.dim() != 2 or _dtype_code(t) != dt or t.device != xs[0].device:
            raise ValueError("all matrices must be 2-D, same dtype, same device")
    if out is not None:
        out = list(out)
        if len(out) != len(xs):
            raise ValueError("out must match xs")
        for i, (o, t) in enumerate(zip(out, xs)):
            _check_tensor(o, f"out[{i}]")
            if o.shape != t.shape or o.dtype != t.dtype:
                raise ValueError("out[i] must match xs[i] in shape and dtype")
    return out


def orthogonalize_list(xs: Sequence[torch.Tensor], out: Sequence[torch.Tensor] | None = None,
                       iters: int = 4, precond: str = "aol", coeffs=None,
                       peer_ptrs: Sequence[Sequence[int]] | None = None,
                       compute: torch.dtype | None = None) -> list[torch.Tensor]:
    """Grouped call: one launch per NS step over all matrices.  In place unless `out`.

    peer_ptrs[i] = device addresses (ints) where matrix i's result is ALSO stored by the
    last iteration's epilogue (fused collective, ns_orthogonalize_peers).
    compute=torch.bfloat16 with fp32 matrices: mixed precision (ns_orthogonalize_cast) --
    cast to bf16 on the GPU, bf16 NS, results widened back to fp32."""
    xs = list(xs)
    if not xs:
        return []
    dt = _dtype_code(xs[0])
    out = _check_list(xs, out)
    cnt = len(xs)
    X = (ctypes.c_void_p * cnt)(*[t.data_ptr() for t in xs])
    O = (ctypes.c_void_p * cnt)(*[t.data_ptr() for t in out]) if out is not None else None
    M = (ctypes.c_int64 * cnt)(*[t.shape[0] for t in xs])
    N = (ctypes.c_int64 * cnt)(*[t.shape[1] for t in xs])
    c = _coeff_array(iters, coeffs, precond)
    mixed = compute is not None and compute != xs[0].dtype
    if mixed and (xs[0].dtype != torch.float32 or compute != torch.bfloat16 or peer_ptrs is not None):
        raise ValueError("mixed precision: fp32 matrices with compute=torch.bfloat16 (no peer stores)")
    with _on_device(xs[0].device):
        if mixed:
            st = lib.ns_orthogonalize_cast(X, O, M, N, cnt, iters, c, PRECOND[precond], _stream(xs[0]))
            check(st, "ns_orthogonalize_cast")
        elif peer_ptrs is None:
            st = lib.ns_orthogonalize_batched(X, O, M, N, cnt, iters, c, PRECOND[precond], dt,
                                              _stream(xs[0]))
            check(st, "ns_orthogonalize_batched")
        else:
            npeer = len(peer_ptrs[0]) if cnt else 0
            if any(len(p) != npeer for p in peer_ptrs) or len(peer_ptrs) != cnt:
                raise ValueError("peer_ptrs must list the same number of peers for every matrix")
            flat = [int(p) for ps in peer_ptrs for p in ps]
            Pp = (ctypes.c_void_p * max(1, len(flat)))(*flat) if flat else None
            st = lib.ns_orthogonalize_peers(X, O, Pp, npeer, M, N, cnt, iters, c, PRECOND[precond], dt,
                                            _stream(xs[0]))
            check(st, "ns_orthogonalize_peers")
    return out if out is not None else xs


class PreparedCall:
    """Argument arrays of one grouped call, built once and replayed (an optimizer's steady
    state calls with the same tensors every step).  `valid()` re-checks the data pointers."""

    def __init__(self, xs, out, iters: int = 4, precond: str = "aol", coeffs=None):
        _check_list(list(xs), out)
        self.xs, self.out = list(xs), list(out) if out is not None else None
        cnt = len(self.xs)
        self.ptrs = [t.data_ptr() for t in self.xs] + ([t.data_ptr() for t in self.out] if self.out else [])
        self.X = (ctypes.c_void_p * cnt)(*[t.data_ptr() for t in self.xs])
        self.O = (ctypes.c_void_p * cnt)(*[t.data_ptr() for t in self.out]) if self.out is not None else None
        self.M = (ctypes.c_int64 * cnt)(*[t.shape[0] for t in self.xs])
        self.N = (ctypes.c_int64 * cnt)(*[t.shape[1] for t in self.xs])
        self.c = _coeff_array(iters, coeffs, precond)
        self.cnt, self.iters, self.pc, self.dt = cnt, iters, PRECOND[precond], _dtype_code(self.xs[0])
        self.device = self.xs[0].device

    def valid(self) -> bool:
        ts = self.xs + (self.out or [])
        return all(t.data_ptr() == p for t, p in zip(ts, self.ptrs))

    def __call__(self):
        st = lib.ns_orthogonalize_batched(self.X, self.O, self.M, self.N, self.cnt, self.iters, self.c, self.pc,
                                          self.dt, ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        check(st, "ns_orthogonalize_batched")


def workspace_size(shapes: Sequence[tuple[int, int]], dtype=torch.bfloat16, batch: int = 1) -> int:
    """ns_workspace_size: bytes of workspace for `shapes`, each repeated `batch` times."""
    cnt = len(shapes)
    M = (ctypes.c_int64 * cnt)(*[s[0] for s in shapes])
    N = (ctypes.c_int64 * cnt)(*[s[1] for s in shapes])
    out = ctypes.c_size_t(0)
    check(lib.ns_workspace_size(M, N, cnt, int(batch), DTYPE_BF16 if dtype == torch.bfloat16 else DTYPE_FP32,
                                ctypes.byref(out)), "ns_workspace_size")
    return out.value


def muon_apply(weights: Sequence[torch.Tensor], updates: Sequence[torch.Tensor], lr: float,
               weight_decay: float = 0.0) -> None:
    """ns_muon_apply: W <- W (1 - lr wd) - lr max(1, m/n)^(1/2) U for each pair (W fp32 or
    bf16, U bf16 of the same shape); one launch on the current stream."""
    ws, us = list(weights), list(updates)
    if len(ws) != len(us) or not ws:
        raise ValueError("weights and updates must be non-empty lists of equal length")
    wdt = _dtype_code(ws[0])
    for w, u in zip(ws, us):
        _check_tensor(w, "weight")
        _check_tensor(u, "update")
        if w.dim() != 2 or w.shape != u.shape or u.dtype != torch.bfloat16 or _dtype_code(w) != wdt:
            raise ValueError("weights: 2-D, one dtype; updates: bf16, same shapes")
    cnt = len(ws)
    arr = lambda xs: (ctypes.c_void_p * cnt)(*[t.data_ptr() for t in xs])  # noqa: E731
    with torch.cuda.device(ws[0].device):
        check(lib.ns_muon_apply(arr(ws), arr(us), (ctypes.c_int64 * cnt)(*[w.shape[0] for w in ws]),
                                (ctypes.c_int64 * cnt)(*[w.shape[1] for w in ws]), cnt, wdt, float(lr),
                                float(weight_decay), _stream()), "ns_muon_apply")


def set_workspace(buf: torch.Tensor | None) -> None:
    """Caller-owned workspace (ns_set_workspace): plans built afterwards carve their
    workspace from `buf` (a contiguous CUDA tensor, 256-byte aligned); None returns to
    library-owned workspace.  Keep `buf` alive while it is set."""
    if buf is None:
        check(lib.ns_set_workspace(None, 0, _stream()), "ns_set_workspace")
        return
    _check_tensor(buf, "workspace")
    with torch.cuda.device(buf.device):
        check(lib.ns_set_workspace(ctypes.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size(), _stream(buf)),
              "ns_set_workspace")


def read_flags(device=None) -> int:
    """Synchronises; returns and clears NS_FLAG_* bits (1: zero scale, 2: non-finite)."""
    f = ctypes.c_uint32(0)
    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        check(lib.ns_read_flags(_stream(), ctypes.byref(f)), "ns_read_flags")
    return int(f.value)


def launch_count() -> int:
    return int(lib.ns_launch_count())


def set_path(path: int) -> int:
    """0 auto, 1 CUDA-core kernels, 2 tcgen05 1-CTA tiles, 4 per-step launches for every
    matrix (no cluster kernels), 5 every matrix that fits takes the FFMA cluster kernel, 7 every
    bf16 matrix with N <= 256 that fits takes the tcgen05 cluster kernel.  Returns the previous
    path, or -1 (and changes nothing) for any other value."""
    return int(lib.ns_set_path(int(path)))


KERNEL_KINDS = ("gram", "precondition", "poly", "update", "simt", "copy", "cluster_tc", "cluster")


def profile_enable(on: bool = True) -> None:
    """Bracket every library launch with CUDA events on its stream (measurement)."""
    lib.ns_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """Synchronise and return {kind: (total_ms, launches)}; clears the records."""
    ms = (ctypes.c_double * 8)()
    cnt = (ctypes.c_uint64 * 8)()
    check(lib.ns_profile_read(ms, cnt, 8), "ns_profile_read")
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_KINDS)}


def shutdown() -> None:
    lib.ns_shutdown()


# ---------------------------------------------------------------------- single steps
def _short(m: int, n: int) -> int:
    return min(m, n)


def partials_ld(N: int) -> int:
    """Slots per row of the AOL row-sum partials (nsx_gram): ceil(N/64) + ceil(N/32)."""
    return (N + 63) // 64 + (N + 31) // 32


def gram(x: torch.Tensor, partials: bool = False):
    """A = Xh^T Xh (N x N), Eq. 3 / Eq. 7.  partials=True: returns (A, part) with the AOL
    row-sum partials of the Gram epilogue (Eq. 8), fp32 [N, partials_ld(N)]."""
    _check_tensor(x, "x")
    m, n = x.shape
    N = _short(m, n)
    a = torch.empty((N, N), dtype=x.dtype, device=x.device)
    part = torch.zeros((N, partials_ld(N)), dtype=torch.float32, device=x.device) if partials else None
    with torch.cuda.device(x.device):
        check(lib.nsx_gram(ctypes.c_void_p(x.data_ptr()), m, n, ctypes.c_void_p(a.data_ptr()),
                           ctypes.c_void_p(part.data_ptr()) if partials else None, _dtype_code(x), _stream(x)),
              "nsx_gram")
    return (a, part) if partials else a


def precondition(a: torch.Tensor, precond: str = "aol", part: torch.Tensor | None = None) -> torch.Tensor:
    """In place a <- diag(s) a diag(s); returns s (fp32).  Eqs. 8-10, Alg. 2 l.4.  part: the
    Gram's AOL partials (gram(x, partials=True)) -- the production row-sum branches."""
    _check_tensor(a, "a")
    N = a.shape[0]
    s = torch.empty((N,), dtype=torch.float32, device=a.device)
    with torch.cuda.device(a.device):
        check(lib.nsx_precondition(ctypes.c_void_p(a.data_ptr()), N, PRECOND[precond],
                                   ctypes.c_void_p(part.data_ptr()) if part is not None else None,
                                   ctypes.c_void_p(s.data_ptr()), _dtype_code(a), _stream(a)),
              "nsx_precondition")
    return s


def poly(a: torch.Tensor, b: float, c: float, s: torch.Tensor | None = None) -> torch.Tensor:
    """B = (b A + c A A) diag(s), Eq. 4."""
    _check_tensor(a, "a")
    N = a.shape[0]
    out = torch.empty_like(a)
    sp = ctypes.c_void_p(s.data_ptr()) if s is not None else None
    with torch.cuda.device(a.device):
        check(lib.nsx_poly(ctypes.c_void_p(a.data_ptr()), N, float(b), float(c), sp,
                           ctypes.c_void_p(out.data_ptr()), _dtype_code(a), _stream(a)), "nsx_poly")
    return out


def update(x: torch.Tensor, bmat: torch.Tensor, a: float, s: torch.Tensor | None = None) -> torch.Tensor:
    """Out = a Xh diag(s) + Xh B^T in x's layout, Eq. 5 (iteration-1 scaling folded)."""
    _check_tensor(x, "x")
    _check_tensor(bmat, "B")
    m, n = x.shape
    out = torch.empty_like(x)
    sp = ctypes.c_void_p(s.data_ptr()) if s is not None else None
    with torch.cuda.device(x.device):
        check(lib.nsx_update(ctypes.c_void_p(x.data_ptr()), m, n, ctypes.c_void_p(bmat.data_ptr()),
                             float(a), sp, ctypes.c_void_p(out.data_ptr()), _dtype_code(x), _stream(x)),
              "nsx_update")
    return out

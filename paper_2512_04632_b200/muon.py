"""Turbo-Muon as a drop-in torch optimizer ("simple drop-in replacement").

Every >= 2-D parameter with a gradient is updated by one grouped `ns_muon_step` call per
parameter group: momentum + nesterov (fp32 state) -> bf16 staging -> AOL-preconditioned NS
(4 iterations, last four Muon+ triples) -> W -= lr * max(1, m/n)^(1/2) * update, all in the
library's CUDA kernels (3*iters + 3 launches per group).  Conv weights are viewed as
(out, in * kh * kw) matrices.  1-D parameters (biases, norms) are not Muon's job:
pass them to another optimizer.
"""
from __future__ import annotations

import ctypes

import torch

from . import coeffs as _coeffs
from ._lib import DTYPE_BF16, DTYPE_FP32, PRECOND, check, lib

__all__ = ["TurboMuon"]


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return DTYPE_BF16
    if t.dtype == torch.float32:
        return DTYPE_FP32
    raise TypeError(f"TurboMuon supports bf16 / fp32 parameters and gradients, got {t.dtype}")


class TurboMuon(torch.optim.Optimizer):
    def __init__(self, params, lr: float = 0.02, momentum: float = 0.95, nesterov: bool = True,
                 weight_decay: float = 0.0, iters: int = 4, precond: str = "aol", coeffs=None):
        if not 0.0 <= momentum < 1.0:
            raise ValueError("momentum must be in [0, 1)")
        defaults = dict(lr=lr, momentum=momentum, nesterov=nesterov, weight_decay=weight_decay,
                        iters=iters, precond=precond, coeffs=coeffs)
        super().__init__(params, defaults)

    @torch.no_grad()
    def step(self, closure=None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        for group in self.param_groups:
            ps = [p for p in group["params"] if p.grad is not None]
            if not ps:
                continue
            by_dtype: dict = {}
            for p in ps:
                if p.dim() < 2:
                    raise ValueError("TurboMuon updates matrices only; give 1-D parameters to another optimizer")
                if not (p.is_cuda and p.is_contiguous() and p.grad.is_contiguous()):
                    raise ValueError("parameters and gradients must be contiguous CUDA tensors")
                by_dtype.setdefault((p.dtype, p.grad.dtype, p.device), []).append(p)
            iters = group["iters"]
            cf = group["coeffs"]
            if cf is None:
                cf = _coeffs.turbo(iters) if group["precond"] == "aol" else _coeffs.muon_plus(iters)
            flat = [float(v) for t in cf for v in t]
            if len(flat) != 3 * iters:
                raise ValueError("coeffs must hold `iters` (a, b, c) triples")
            carr = (ctypes.c_float * len(flat))(*flat)
            for (pdt, gdt, dev), plist in by_dtype.items():
                W, G, M, U, ms, ns_ = [], [], [], [], [], []
                for p in plist:
                    st = self.state[p]
                    m, n = p.shape[0], p.numel() // p.shape[0]
                    if "momentum_buffer" not in st:
                        st["momentum_buffer"] = torch.zeros((m, n), dtype=torch.float32, device=dev)
                        st["ns_staging"] = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
                    W.append(p.data_ptr()); G.append(p.grad.data_ptr())
                    M.append(st["momentum_buffer"].data_ptr()); U.append(st["ns_staging"].data_ptr())
                    ms.append(m); ns_.append(n)
                cnt = len(plist)
                arr = lambda xs: (ctypes.c_void_p * cnt)(*xs)  # noqa: E731
                with torch.cuda.device(dev):
                    status = lib.ns_muon_step(
                        arr(W), arr(G), arr(M), arr(U), (ctypes.c_int64 * cnt)(*ms), (ctypes.c_int64 * cnt)(*ns_),
                        cnt, _dt(plist[0]), _dt(plist[0].grad), float(group["lr"]), float(group["momentum"]),
                        float(group["weight_decay"]), 1 if group["nesterov"] else 0, iters, carr,
                        PRECOND[group["precond"]], ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
                check(status, "ns_muon_step")
        return loss

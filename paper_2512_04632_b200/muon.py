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


def _coeff_carr(group):
    iters = group["iters"]
    cf = group["coeffs"]
    if cf is None:
        cf = _coeffs.turbo(iters) if group["precond"] == "aol" else _coeffs.muon_plus(iters)
    flat = [float(v) for t in cf for v in t]
    if len(flat) != 3 * iters:
        raise ValueError("coeffs must hold `iters` (a, b, c) triples")
    return (ctypes.c_float * len(flat))(*flat)


def _muon_step_call(W, G, M, U, ms, ns_, w_dt, g_dt, group, carr, dev, grad_scale: float = 1.0):
    """One grouped ns_muon_step over pointer lists (momentum -> NS -> update)."""
    cnt = len(W)
    arr = lambda xs: (ctypes.c_void_p * cnt)(*xs)  # noqa: E731
    with torch.cuda.device(dev):
        status = lib.ns_muon_step(
            arr(W), arr(G), arr(M), arr(U), (ctypes.c_int64 * cnt)(*ms), (ctypes.c_int64 * cnt)(*ns_),
            cnt, w_dt, g_dt, float(group["lr"]), float(group["momentum"]), float(group["weight_decay"]),
            float(grad_scale), 1 if group["nesterov"] else 0, group["iters"], carr, PRECOND[group["precond"]],
            ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    check(status, "ns_muon_step")

__all__ = ["TurboMuon", "DistributedTurboMuon"]


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
            carr = _coeff_carr(group)
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
                _muon_step_call(W, G, M, U, ms, ns_, _dt(plist[0]), _dt(plist[0].grad), group, carr, dev)
        return loss


class DistributedTurboMuon(torch.optim.Optimizer):
    """Data-parallel Turbo-Muon over a process group (the steps on either
    side of the path, with a reduce-scatter by ownership instead of a gradient all-reduce).
    Every rank holds the same parameter list and its LOCAL gradients; one step:

      1. reduce-scatter by matrix ownership (sum over ranks; LPT ownership on NS FLOPs, as in
         parallel.orthogonalize_sharded): each rank receives the summed gradient of only the
         matrices it owns (packed by one multi-tensor copy; the 1/world mean is applied inside
         the momentum kernel);
      2. the owner runs the fused Muon step (momentum -> NS -> update of its own weights), the
         orthogonalised update U landing in its segment of a packed bf16 buffer;
      3. one all-gather of U, then every rank applies the same update kernel (ns_muon_apply)
         to the matrices it does not own -- the weights stay bitwise identical on all ranks.

    Momentum state exists only on the owner (1/world of it per rank).  All parameters must
    share one dtype and one device; gradients one dtype."""

    def __init__(self, params, group=None, lr: float = 0.02, momentum: float = 0.95, nesterov: bool = True,
                 weight_decay: float = 0.0, iters: int = 4, precond: str = "aol", coeffs=None):
        if not 0.0 <= momentum < 1.0:
            raise ValueError("momentum must be in [0, 1)")
        defaults = dict(lr=lr, momentum=momentum, nesterov=nesterov, weight_decay=weight_decay,
                        iters=iters, precond=precond, coeffs=coeffs)
        super().__init__(params, defaults)
        self.pg = group
        self._ubuf = {}

    @torch.no_grad()
    def step(self, closure=None):
        import torch.distributed as dist

        from .api import muon_apply
        from .parallel import make_plan, reduce_scatter_owned, _gather
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        on = dist.is_initialized()
        world = dist.get_world_size(self.pg) if on else 1
        for gi, group in enumerate(self.param_groups):
            ps = [p for p in group["params"] if p.grad is not None]
            if not ps:
                continue
            for p in ps:
                if p.dim() < 2 or not (p.is_cuda and p.is_contiguous() and p.grad.is_contiguous()):
                    raise ValueError("contiguous CUDA matrices (>= 2-D) with gradients expected")
            dev = ps[0].device
            shapes = [(p.shape[0], p.numel() // p.shape[0]) for p in ps]
            iters = group["iters"]
            # summed (not averaged) gradients: the 1/world mean is folded into the momentum kernel
            mine, owned_g = reduce_scatter_owned([p.grad.view(s) for p, s in zip(ps, shapes)], self.pg, iters,
                                                 mean=False)
            plan = make_plan(shapes, world, iters, 1)
            key = (gi, tuple(shapes), world)
            if key not in self._ubuf:
                self._ubuf[key] = torch.empty(plan.total, dtype=torch.bfloat16, device=dev)
            ubuf = self._ubuf[key]
            uv = [ubuf[o:o + m * n].view(m, n) for o, (m, n) in zip(plan.offsets, shapes)]
            carr = _coeff_carr(group)
            if mine:
                W, G, M, U, ms, ns_ = [], [], [], [], [], []
                for i, g in zip(mine, owned_g):
                    p = ps[i]
                    st = self.state[p]
                    m, n = shapes[i]
                    if "momentum_buffer" not in st:
                        st["momentum_buffer"] = torch.zeros((m, n), dtype=torch.float32, device=dev)
                    W.append(p.data_ptr()); G.append(g.data_ptr())
                    M.append(st["momentum_buffer"].data_ptr()); U.append(uv[i].data_ptr())
                    ms.append(m); ns_.append(n)
                _muon_step_call(W, G, M, U, ms, ns_, _dt(ps[0]), _dt(owned_g[0]), group, carr, dev,
                                grad_scale=1.0 / world)
            if world > 1:
                _gather(ubuf, plan, 0, dist.get_rank(self.pg), self.pg)
                others = [i for i in range(len(ps)) if i not in set(mine)]
                if others:
                    muon_apply([ps[i].data.view(shapes[i]) for i in others], [uv[i] for i in others],
                               group["lr"], group["weight_decay"])
        return loss

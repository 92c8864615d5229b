"""Multi-GPU orthogonalisation of a Muon parameter set: whole-matrix ownership + all-gather.

Matrices are independent units (the paper orthogonalises every 2-D update separately,
P:L97, "batches of 32 matrices" P:L247), so the path shards by matrix: each rank runs the
grouped NS launch on the matrices it owns, writing straight into its segment of a packed
buffer, and one collective (NCCL all-gather over NVLink) gives every rank every result --
the exchange a data-parallel optimizer step needs.  No matrix is split across ranks
(splitting one would need a Gram all-reduce every step, the bottleneck P:L100/L313 name).

Ownership is LPT (longest-processing-time-first) on the algorithmic FLOPs of §8(a):
deterministic and identical on every rank (no communication to agree on it).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import torch
import torch.distributed as dist

__all__ = ["ns_flops", "lpt_owners", "ShardPlan", "make_plan", "orthogonalize_sharded"]

_ALIGN = 64  # elements; keeps every packed matrix 128-byte aligned in bf16


def ns_flops(m: int, n: int, iters: int = 4) -> int:
    """Algorithmic FLOPs of one NS call (symmetric products counted once):
    iters * (M N (N+1) [Gram] + N^2 (N+1) [A^2] + 2 M N^2 [X B])."""
    M, N = max(m, n), min(m, n)
    return iters * (M * N * (N + 1) + N * N * (N + 1) + 2 * M * N * N)


def lpt_owners(shapes: Sequence[tuple[int, int]], world: int, iters: int = 4) -> list[int]:
    """Sort by FLOPs (descending, ties by index); give each to the least-loaded rank."""
    order = sorted(range(len(shapes)), key=lambda i: (-ns_flops(*shapes[i], iters), i))
    load = [0] * world
    owner = [0] * len(shapes)
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[i] = r
        load[r] += ns_flops(*shapes[i], iters)
    return owner


@dataclass
class ShardPlan:
    world: int
    owners: list[int]
    offsets: list[int]       # element offset of matrix i inside the gathered buffer
    seg_elems: int           # elements per rank segment (equal for all ranks)
    load: list[int]          # FLOPs per rank

    def mine(self, rank: int) -> list[int]:
        return [i for i, r in enumerate(self.owners) if r == rank]


def make_plan(shapes: Sequence[tuple[int, int]], world: int, iters: int = 4) -> ShardPlan:
    owners = lpt_owners(shapes, world, iters)
    seg_fill = [0] * world
    local = [0] * len(shapes)
    for i, (m, n) in enumerate(shapes):
        r = owners[i]
        local[i] = seg_fill[r]
        seg_fill[r] += -(-(m * n) // _ALIGN) * _ALIGN
    seg = max(max(seg_fill), _ALIGN)
    offsets = [owners[i] * seg + local[i] for i in range(len(shapes))]
    load = [0] * world
    for i, s in enumerate(shapes):
        load[owners[i]] += ns_flops(*s, iters)
    return ShardPlan(world, owners, offsets, seg, load)


_BUFFERS: dict = {}


def _gather_buffer(key, numel, dtype, device) -> torch.Tensor:
    buf = _BUFFERS.get(key)
    if buf is None or buf.numel() != numel:
        buf = torch.empty(numel, dtype=dtype, device=device)
        _BUFFERS[key] = buf
    return buf


def orthogonalize_sharded(xs: Sequence[torch.Tensor], group=None, iters: int = 4,
                          precond: str = "aol", coeffs=None, inplace: bool = False,
                          compute: Callable | None = None) -> list[torch.Tensor]:
    """Every rank passes the same list (the post-all-reduce gradients / momenta).
    Returns the orthogonalised matrices (views into one gathered buffer); with
    inplace=True they are also copied back into `xs`.

    `compute(inputs, outputs)` runs NS on this rank's matrices; it defaults to the
    grouped CUDA call.  (The CPU multi-process tests inject a CPU function here.)
    """
    xs = list(xs)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    shapes = [tuple(t.shape) for t in xs]
    plan = make_plan(shapes, world, iters)
    dtype, device = xs[0].dtype, xs[0].device
    key = (tuple(shapes), world, dtype, str(device), id(group))
    buf = _gather_buffer(key, plan.seg_elems * world, dtype, device)
    views = [buf[o:o + m * n].view(m, n) for o, (m, n) in zip(plan.offsets, shapes)]
    mine = plan.mine(rank)
    if mine:
        ins = [xs[i] for i in mine]
        outs = [views[i] for i in mine]
        if compute is None:
            from .api import orthogonalize_list
            orthogonalize_list(ins, out=outs, iters=iters, precond=precond, coeffs=coeffs)
        else:
            compute(ins, outs)
    if world > 1:
        seg = buf[rank * plan.seg_elems:(rank + 1) * plan.seg_elems]
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(buf, seg, group=group)
        else:
            chunks = list(buf.split(plan.seg_elems))
            dist.all_gather(chunks, seg.clone(), group=group)
    if inplace:
        for t, v in zip(xs, views):
            t.copy_(v)
    return views

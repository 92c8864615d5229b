"""Multi-process (world_size 2 and 4, gloo, CPU) tests of the sharded path's host logic:
LPT ownership, packed-buffer layout, and that the gathered result on every rank equals the
single-process result bitwise.  The per-rank NS compute is injected (fp64 oracle on CPU);
on the GPU the same code calls the grouped CUDA launch and NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_04632_b200.parallel import lpt_owners, make_plan, ns_flops, orthogonalize_sharded
from synth import coeffs as C
from synth import inputs as I


def test_lpt_balance_gpt2_sets():
    for size in ("small", "medium", "large"):
        shapes = I.gpt2_shapes(size)
        for world in (2, 4, 8):
            plan = make_plan(shapes, world)
            assert max(plan.load) / (sum(plan.load) / world) == pytest.approx(1.0)
            assert plan.owners == lpt_owners(shapes, world)  # deterministic


def test_lpt_greedy_bound():
    """List-scheduling bound: max load <= mean load + largest job; and >= both."""
    rng = np.random.default_rng(0)
    shapes = [(int(rng.integers(8, 64)) * 8, int(rng.integers(8, 64)) * 8) for _ in range(37)]
    for world in (2, 3, 5):
        plan = make_plan(shapes, world)
        f = [ns_flops(m, n) for m, n in shapes]
        assert max(sum(f) / world, max(f)) <= max(plan.load) <= sum(f) / world + max(f)


def test_packed_layout():
    shapes = I.cifar_shapes() + I.gpt2_shapes("small")[:10]
    for world in (1, 2, 4):
        plan = make_plan(shapes, world)
        spans = sorted((o, o + m * n) for o, (m, n) in zip(plan.offsets, shapes))
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert a1 <= b0
        assert spans[-1][1] <= plan.seg_elems * world
        for i, o in enumerate(plan.offsets):
            r = plan.owners[i]
            assert r * plan.seg_elems <= o < (r + 1) * plan.seg_elems
            assert o % 64 == 0


def _oracle_compute(ins, outs):
    from oracle import ns_oracle as O
    for x, o in zip(ins, outs):
        y = O.newton_schulz(x.double().numpy(), C.turbo(4), "aol")
        o.copy_(torch.from_numpy(y).to(o.dtype))


def test_bucketed_layout():
    shapes = I.gpt2_shapes("small")
    for world in (1, 2, 4):
        for nb in (1, 3, 4):
            plan = make_plan(shapes, world, buckets=nb)
            spans = sorted((o, o + m * n) for o, (m, n) in zip(plan.offsets, shapes))
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 <= b0
            assert spans[-1][1] <= plan.total
            assert sorted(plan.mine(0) + [i for r in range(1, world) for i in plan.mine(r)]) == list(range(len(shapes)))
            for b, per_rank in enumerate(plan.buckets):  # each rank's matrices sit in its segment
                for r, mats in enumerate(per_rank):
                    lo = plan.bucket_base[b] + r * plan.bucket_seg[b]
                    for i in mats:
                        assert lo <= plan.offsets[i] and plan.offsets[i] + shapes[i][0] * shapes[i][1] <= lo + plan.bucket_seg[b]


def _worker(rank, world, port, shapes, q, buckets=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    xs = [torch.from_numpy(I.gaussian(m, n, seed=100 + i)) for i, (m, n) in enumerate(shapes)]
    outs = orthogonalize_sharded(xs, iters=4, compute=_oracle_compute, buckets=buckets)
    q.put((rank, [o.clone().numpy() for o in outs]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,buckets", [(2, 1), (4, 1), (2, 3)])
def test_sharded_gloo_matches_single(world, buckets):
    shapes = [(96, 64), (64, 160), (128, 128), (40, 24), (200, 56), (64, 64), (32, 96)]
    xs = [torch.from_numpy(I.gaussian(m, n, seed=100 + i)) for i, (m, n) in enumerate(shapes)]
    single = orthogonalize_sharded(xs, iters=4, compute=_oracle_compute)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shapes, q, buckets)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get() for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, outs in results:
        for a, b in zip(outs, single):
            assert np.array_equal(a, b.numpy())


def _rs_worker(rank, world, port, shapes, q, mean=True):
    from paper_2512_04632_b200.parallel import reduce_scatter_owned
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank-dependent local "gradients": g_r[i] = gaussian(i) * (r + 1)
    gs = [torch.from_numpy(I.gaussian(m, n, seed=300 + i, bf16=False)) * (rank + 1) for i, (m, n) in enumerate(shapes)]
    mine, views = reduce_scatter_owned(gs, mean=mean)
    q.put((rank, mine, [v.clone().numpy() for v in views]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mean", [(2, True), (4, True), (2, False)])
def test_reduce_scatter_owned_gloo(world, mean):
    """Each rank receives the cross-rank mean (or, for DistributedTurboMuon, which folds the
    1/world into its momentum kernel, the sum) of exactly the matrices it owns (LPT ownership
    identical to the sharded NS), and the owners partition the list."""
    shapes = [(96, 64), (64, 160), (128, 128), (40, 24), (200, 56), (64, 64), (32, 96)]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_rs_worker, args=(r, world, port, shapes, q, mean)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get() for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    owners = lpt_owners(shapes, world)
    seen = []
    mean_factor = sum(r + 1 for r in range(world)) / (world if mean else 1)
    for rank, mine, views in results:
        assert mine == [i for i in range(len(shapes)) if owners[i] == rank]
        seen += mine
        for i, v in zip(mine, views):
            ref = I.gaussian(*shapes[i], seed=300 + i, bf16=False) * mean_factor
            np.testing.assert_allclose(v, ref, rtol=1e-6, atol=1e-6)
    assert sorted(seen) == list(range(len(shapes)))

"""End-to-end parity of the CUDA path (through the C ABI) against the fp64 oracle (GPU).

Gates (BASELINE.json north_star): relative Frobenius difference <= 2e-2 in bf16 and
<= 1e-4 in fp32 mode; the GPU polar error no worse than the oracle's by more than 5%.
Both sides consume the same bf16-representable inputs from synth/ and the same
coefficient arrays.
"""
import numpy as np
import pytest
import torch

from oracle import ns_oracle as O
from synth import coeffs as C
from synth import inputs as I
from tests.helpers import oracle_run, polar_excess, relF, assert_parity, bf16_model_out

pytestmark = pytest.mark.gpu

ns = pytest.importorskip("paper_2512_04632_b200")

BF16_TOL = 2e-2
FP32_TOL = 1e-4
POLAR_SLACK = 1.05


def _run(x32: np.ndarray, coeffs, precond: str, dtype=torch.bfloat16) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x32, dtype=np.float32)).to(dtype).cuda()
    ns.orthogonalize(t, iters=len(coeffs), precond=precond, coeffs=coeffs)
    torch.cuda.synchronize()
    return t.float().cpu().numpy().astype(np.float64)


CASES = [
    # (m, n, dist) -- square, tall, wide, ragged tiles, CIFAR, GPT-2 shapes, unaligned (SIMT)
    (256, 256, "gaussian"),
    (768, 768, "gaussian"),
    (3072, 768, "gaussian"),
    (768, 3072, "gaussian"),
    (520, 136, "gaussian"),
    (64, 216, "gaussian"),
    (256, 2304, "lowrank"),
    (512, 512, "levy1.0"),
    (1000, 600, "levy1.5"),
    (100, 37, "gaussian"),
]


@pytest.fixture(params=[0, 4], ids=["auto", "per-step"])
def launch_mode(request):
    """0 auto (small matrices on the cluster kernel), 4 one tcgen05/SIMT launch per step for
    every matrix."""
    old = ns.set_path(request.param)
    yield request.param
    ns.set_path(old)


@pytest.mark.parametrize("m,n,dist", CASES)
def test_turbo_muon_aol4(m, n, dist, launch_mode):
    x = I.make_matrix(m, n, seed=I.matrix_seed(1, m + n), dist=dist)
    coeffs = C.turbo(4)
    out = _run(x, coeffs, "aol")
    ref = oracle_run(x, coeffs, "aol")
    model = bf16_model_out(x, coeffs, "aol") if dist.startswith("levy") else None
    assert_parity(out, ref, BF16_TOL, f"{m}x{n} {dist}", model=model)
    eg, eo = polar_excess(out, ref, x)
    assert eg <= POLAR_SLACK * eo, (eg, eo)


@pytest.mark.parametrize("m,n", [(768, 768), (3072, 768), (64, 576)])
def test_muon_plus_frobenius5(m, n, launch_mode):
    x = I.gaussian(m, n, seed=21)
    coeffs = C.muon_plus(5)
    out = _run(x, coeffs, "frobenius")
    ref = oracle_run(x, coeffs, "frobenius")
    assert_parity(out, ref, BF16_TOL)
    eg, eo = polar_excess(out, ref, x)
    assert eg <= POLAR_SLACK * eo, (eg, eo)


def test_precond_none_closed_form():
    """precond=none on a matrix with ||X||_2 < 1."""
    x = I.round_bf16(I.gaussian(384, 256, seed=22, bf16=False) / np.float32(40.0))
    coeffs = C.turbo(4)
    assert_parity(_run(x, coeffs, "none"), oracle_run(x, coeffs, "none"), BF16_TOL)


@pytest.mark.parametrize("m,n,dist", [(128, 128, "gaussian"), (128, 128, "levy1.5"), (96, 200, "gaussian")])
def test_fp32_exact_mode(m, n, dist):
    """Config 1: 128 x 128 fp32, relF <= 1e-4 vs the fp64 oracle."""
    x = I.make_matrix(m, n, seed=31, dist=dist, bf16=False)
    coeffs = C.turbo(4)
    out = _run(x, coeffs, "aol", dtype=torch.float32)
    ref = oracle_run(x, coeffs, "aol")
    assert_parity(out, ref, FP32_TOL)
    eg, eo = polar_excess(out, ref, x)
    assert eg <= POLAR_SLACK * eo


def test_batched_equals_single_bitwise(launch_mode):
    shapes = [(768, 768), (3072, 768), (768, 3072), (64, 216), (520, 136)]
    xs = [I.gaussian(m, n, seed=40 + i) for i, (m, n) in enumerate(shapes)]
    singles = [_run(x, C.turbo(4), "aol") for x in xs]
    ts = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in xs]
    outs = [torch.empty_like(t) for t in ts]
    ns.orthogonalize_list(ts, out=outs, iters=4)
    for o, s in zip(outs, singles):
        assert np.array_equal(o.float().cpu().numpy().astype(np.float64), s)
    # batch-strided entry point
    xb = np.stack([I.gaussian(256, 128, seed=50 + i) for i in range(3)])
    tb = torch.from_numpy(xb).to(torch.bfloat16).cuda()
    ns.orthogonalize(tb, iters=4)
    for i in range(3):
        assert np.array_equal(tb[i].float().cpu().numpy(), _run(xb[i], C.turbo(4), "aol").astype(np.float32))


def test_odd_iters_in_place_and_out_of_place():
    x = I.gaussian(512, 256, seed=60)
    coeffs = C.muon_plus(5)
    a = _run(x, coeffs, "aol")
    t = torch.from_numpy(x).to(torch.bfloat16).cuda()
    o = torch.empty_like(t)
    ns.orthogonalize_list([t], out=[o], iters=5, precond="aol", coeffs=coeffs)
    assert np.array_equal(o.float().cpu().numpy().astype(np.float64), a)
    assert np.array_equal(t.float().cpu().numpy(), x)  # input untouched


def test_scale_invariance_bitwise():
    """NS(AOL(4^k X)) == NS(AOL(X)) bitwise: exponent-exact scaling (reading R4)."""
    x = I.gaussian(768, 512, seed=61)
    a = _run(x, C.turbo(4), "aol")
    b = _run(x * np.float32(16.0), C.turbo(4), "aol")
    assert np.array_equal(a, b)


def test_transpose_symmetry():
    x = I.gaussian(1024, 384, seed=62)
    a = _run(x, C.turbo(4), "aol")
    b = _run(np.ascontiguousarray(x.T), C.turbo(4), "aol")
    assert relF(b.T, a) <= 1e-2


def test_singular_value_band_tall():
    """Tall Gaussian (aspect 4): sigma_min(X1) >= 0.05, so sigma(out) in [0.97, 1.04]."""
    x = I.gaussian(3072, 768, seed=63)
    out = _run(x, C.turbo(4), "aol")
    sv = np.linalg.svd(out, compute_uv=False)
    assert sv.min() >= 0.97 and sv.max() <= 1.04, (sv.min(), sv.max())


def test_descent_alignment_and_determinism():
    x = I.levy(512, 384, seed=64, alpha=1.0)
    a = _run(x, C.turbo(4), "aol")
    b = _run(x, C.turbo(4), "aol")
    assert np.array_equal(a, b)
    assert O.descent_alignment(x, a) > 0


def test_removed_paths_rejected():
    """Paths 3 (fused single launch) and 6 (multicast clusters) lost every A/B run and were
    removed: ns_set_path rejects them (-1) and leaves the current path unchanged."""
    old = ns.set_path(0)
    try:
        assert ns.set_path(3) == -1 and ns.set_path(6) == -1
        assert ns.set_path(0) == 0
    finally:
        ns.set_path(old)


def test_zero_column_flag():
    x = I.gaussian(256, 128, seed=65)
    x[:, 5] = 0
    ns.read_flags()
    out = _run(x, C.turbo(4), "aol")
    assert ns.read_flags() & 1
    assert np.all(np.isfinite(out)) and np.all(out[:, 5] == 0)
    assert_parity(out, oracle_run(x, C.turbo(4), "aol"), BF16_TOL)


def test_launch_count_grouped():
    """One launch per step over all matrices: 3T + 1 launches (path 0/4)."""
    shapes = [(768, 768)] * 4 + [(3072, 768), (768, 3072)]
    ts = [torch.from_numpy(I.gaussian(m, n, seed=70 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    ns.orthogonalize_list(ts, iters=4)  # builds the plan
    c0 = ns.launch_count()
    ns.orthogonalize_list(ts, iters=4)
    torch.cuda.synchronize()
    assert ns.launch_count() - c0 == 3 * 4 + 1


@pytest.mark.parametrize("n", [8192])
def test_full_size_properties(n):
    """8192^2 (BASELINE config 4): properties that hold at any size -- finite output,
    bitwise determinism, exact scale invariance, descent alignment, bounded spectrum."""
    x = I.gaussian(n, n, seed=80)
    t1 = torch.from_numpy(x).to(torch.bfloat16).cuda()
    t2 = (t1 * 4).contiguous()
    ns.orthogonalize(t1)
    ns.orthogonalize(t2)
    torch.cuda.synchronize()
    assert torch.isfinite(t1.float()).all()
    assert torch.equal(t1, t2)
    xf = torch.from_numpy(x).cuda()
    assert float((xf * t1.float()).sum()) > 0
    # spectral norm by power iteration (fp32): AOL keeps ||X1||_2 <= 1, so every output
    # singular value is at most max_{s in [0,1]} P(s) of the schedule (Eq. 2 acts per
    # singular value); allow 2% for bf16 rounding.
    grid = np.linspace(0.0, 1.0, 200001)
    for a, b, c in C.turbo(4):
        grid = a * grid + b * grid ** 3 + c * grid ** 5
    bound = 1.02 * grid.max()
    v = torch.randn(n, 1, device="cuda", generator=None)
    o = t1.float()
    for _ in range(30):
        v = o.T @ (o @ v)
        v = v / v.norm()
    assert float((o @ v).norm()) <= bound


def test_host_pipeline_matches_device_path():
    """orthogonalize_host (pinned host in/out, bucketed copy/compute overlap) returns the
    same bits as the device-resident grouped call."""
    from paper_2512_04632_b200.parallel import orthogonalize_host
    shapes = [(768, 768)] * 3 + [(3072, 768), (768, 3072), (64, 216)]
    xs = [I.gaussian(m, n, seed=110 + i) for i, (m, n) in enumerate(shapes)]
    host = [torch.from_numpy(x).to(torch.bfloat16).pin_memory() for x in xs]
    outs = orthogonalize_host(host, iters=4, buckets=3)
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        t = torch.from_numpy(x).to(torch.bfloat16).cuda()
        ns.orthogonalize(t, iters=4)
        assert torch.equal(o, t.cpu())


def test_sharded_nccl_world1():
    """The NCCL code path of the sharder (init, in-place all_gather_into_tensor, bucketed
    overlap on a comm stream) at world size 1 -- the only size one GPU can run."""
    import os
    import torch.distributed as dist
    from paper_2512_04632_b200.parallel import orthogonalize_sharded
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        shapes = [(1024, 1024)] * 4 + [(4096, 1024), (1024, 4096)]
        xs = [torch.from_numpy(I.gaussian(m, n, seed=120 + i)).to(torch.bfloat16).cuda()
              for i, (m, n) in enumerate(shapes)]
        outs = orthogonalize_sharded(xs, iters=4, buckets=3)
        torch.cuda.synchronize()
        for x, o in zip(xs, outs):
            t = x.clone()
            ns.orthogonalize(t, iters=4)
            assert torch.equal(o, t)
    finally:
        dist.destroy_process_group()


def test_fused_peer_stores_c_abi():
    """ns_orthogonalize_peers: the last iteration's epilogue writes every output tile to the
    extra destinations as well (here two local buffers standing in for peers' NVLink-mapped
    gather buffers, NaN-filled so that a missed tile shows): all copies are bitwise the regular
    result, and a peer copy of the ragged matrix matches the fp64 oracle on its own."""
    shapes = [(1024, 1024), (3072, 768), (768, 3072), (520, 136)]
    xs_np = [I.gaussian(m, n, seed=130 + i) for i, (m, n) in enumerate(shapes)]
    xs = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in xs_np]
    ref = [x.clone() for x in xs]
    ns.orthogonalize_list(ref, iters=4)
    outs = [torch.empty_like(x) for x in xs]
    peers = [[torch.full_like(x, float("nan")) for _ in range(2)] for x in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4, peer_ptrs=[[p.data_ptr() for p in ps] for ps in peers])
    torch.cuda.synchronize()
    for r, o, ps in zip(ref, outs, peers):
        assert torch.equal(o, r)
        for p in ps:
            assert torch.equal(p, r)
    peer = peers[3][1].float().cpu().numpy().astype(np.float64)
    assert_parity(peer, oracle_run(xs_np[3], C.turbo(4), "aol"), 2e-2, "peer copy 520x136")


def test_sharded_fused_collective_world1():
    """Symmetric-memory gather buffer + fused peer stores through the sharder (world 1)."""
    import os
    import torch.distributed as dist
    from paper_2512_04632_b200.parallel import orthogonalize_sharded
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29537"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        shapes = [(1024, 1024)] * 2 + [(4096, 1024), (1024, 4096)]
        xs = [torch.from_numpy(I.gaussian(m, n, seed=140 + i)).to(torch.bfloat16).cuda()
              for i, (m, n) in enumerate(shapes)]
        outs = orthogonalize_sharded(xs, iters=4, collective="fused")
        torch.cuda.synchronize()
        for x, o in zip(xs, outs):
            t = x.clone()
            ns.orthogonalize(t, iters=4)
            assert torch.equal(o, t)
    finally:
        dist.destroy_process_group()


def test_cuda_graph_capture_replay():
    """After the first (plan-building) call, a call only enqueues kernel launches: it can be
    captured in a CUDA graph and replayed, with bitwise-identical results."""
    shapes = [(768, 768), (3072, 768), (768, 3072)]
    xs = [torch.from_numpy(I.gaussian(m, n, seed=150 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    outs = [torch.empty_like(x) for x in xs]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ns.orthogonalize_list(xs, out=outs, iters=4)  # builds the plan (not capturable)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs]
    for o in outs:
        o.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ns.orthogonalize_list(xs, out=outs, iters=4)
    g.replay()
    torch.cuda.synchronize()
    for r, o in zip(ref, outs):
        assert torch.equal(r, o)


@pytest.mark.parametrize("m,n", [(8192, 8), (8, 8192), (4096, 1), (1, 4096), (8, 4096), (16, 24)])
def test_extreme_aspect_ratios(m, n):
    """Very thin / very wide matrices (N = 1 .. 8, M up to 8192) on whichever path they route
    to (cluster kernel, tcgen05 with TMA zero fill, SIMT): same gates as the other cases."""
    x = I.gaussian(m, n, seed=I.matrix_seed(9, m + n))
    out = _run(x, C.turbo(4), "aol")
    ref = oracle_run(x, C.turbo(4), "aol")
    assert np.all(np.isfinite(out))
    assert_parity(out, ref, BF16_TOL)


def test_many_matrices_one_call_bitwise():
    """300 matrices of mixed shapes in one grouped call (cluster kernel + tcgen05 step engine
    + SIMT for unaligned shapes, one plan): every result bitwise equal to its single call."""
    rng = np.random.default_rng(5)
    cand = [(64, 64), (128, 96), (256, 128), (512, 256), (200, 72), (40, 600), (768, 256), (100, 37), (264, 200)]
    shapes = [cand[i] for i in rng.integers(0, len(cand), size=300)]
    xs = [torch.from_numpy(I.gaussian(m, n, seed=1000 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    outs = [torch.empty_like(x) for x in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    for k in range(0, 300, 37):
        t = xs[k].clone()
        ns.orthogonalize(t, iters=4)
        torch.cuda.synchronize()
        assert torch.equal(t, outs[k]), (k, shapes[k])


@pytest.mark.parametrize("dtype,shapes,path", [
    (torch.float32, [(128, 128), (64, 216), (256, 64)], 0),          # FFMA cluster kernel + L2 exchange scratch
    (torch.bfloat16, [(1024, 128), (64, 576), (256, 2304)], 0),       # tcgen05 cluster kernel beside the step engine
    (torch.bfloat16, [(1024, 128), (64, 576), (256, 2304), (768, 256)], 7),  # every one on the tcgen05 cluster kernel
])
def test_exact_workspace_covers_cluster_kernels(dtype, shapes, path):
    """A caller workspace of exactly ns_workspace_size bytes is enough when matrices take the
    cluster-resident kernels (their Gram-partial / A-image and row-exchange scratch), and the
    results are bitwise those of library-owned workspace."""
    xs = [torch.from_numpy(I.gaussian(m, n, seed=700 + i, bf16=dtype == torch.bfloat16)).to(dtype).cuda()
          for i, (m, n) in enumerate(shapes)]
    old = ns.set_path(path)
    try:
        ref = [torch.empty_like(x) for x in xs]
        ns.orthogonalize_list(xs, out=ref, iters=4)
        buf = torch.empty(ns.workspace_size(shapes, dtype=dtype), dtype=torch.uint8, device="cuda")
        try:
            ns.set_workspace(buf)
            outs = [torch.empty_like(x) for x in xs]
            ns.orthogonalize_list(xs, out=outs, iters=4)
            torch.cuda.synchronize()
        finally:
            ns.set_workspace(None)
        for r, o in zip(ref, outs):
            assert torch.equal(r, o)
    finally:
        ns.set_path(old)


def test_caller_owned_workspace():
    """ns_set_workspace: plans carve their workspace from a caller buffer (results bitwise
    equal to library-owned workspace); a too-small buffer fails with NS_ERR_WORKSPACE."""
    shapes = [(768, 768), (3072, 768), (1024, 512)]
    xs = [torch.from_numpy(I.gaussian(m, n, seed=190 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    ref = [torch.empty_like(x) for x in xs]
    ns.orthogonalize_list(xs, out=ref, iters=4)
    need = ns.workspace_size(shapes)
    buf = torch.empty(need + 4096, dtype=torch.uint8, device="cuda")
    try:
        ns.set_workspace(buf)
        outs = [torch.empty_like(x) for x in xs]
        ns.orthogonalize_list(xs, out=outs, iters=4)
        torch.cuda.synchronize()
        for r, o in zip(ref, outs):
            assert torch.equal(r, o)
        small = torch.empty(4096, dtype=torch.uint8, device="cuda")
        ns.set_workspace(small)
        with pytest.raises(ns.NSError, match="NS_ERR_WORKSPACE"):
            ns.orthogonalize_list(xs, out=outs, iters=4)
    finally:
        ns.set_workspace(None)
    outs = [torch.empty_like(x) for x in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    for r, o in zip(ref, outs):
        assert torch.equal(r, o)


def test_gpt2_large_set_full_size_sampled():
    """BASELINE config 5's GPT-2-large hidden-matrix set (216 matrices, 1.4 GB) in one
    grouped call; one matrix of each shape checked against the oracle, all finite."""
    shapes = I.shape_set("gpt2-large")
    xs_np = {}
    pick = {}
    for i, s in enumerate(shapes):
        pick.setdefault(s, i)
    ts = []
    for i, (m, n) in enumerate(shapes):
        x = I.gaussian(m, n, seed=I.matrix_seed(6, i))
        if i in pick.values():
            xs_np[i] = x
        ts.append(torch.from_numpy(x).to(torch.bfloat16).cuda())
    ns.orthogonalize_list(ts, iters=4)
    torch.cuda.synchronize()
    assert all(bool(torch.isfinite(t.float()).all()) for t in ts)
    for i, x in xs_np.items():
        out = ts[i].float().cpu().numpy().astype(np.float64)
        assert_parity(out, oracle_run(x, C.turbo(4), "aol"), BF16_TOL)


@pytest.mark.parametrize("m,n", [(768, 256), (64, 216), (100, 37)])
def test_nonfinite_input_raises_flag(m, n):
    """A NaN / Inf in the input is not an error (reading R4: flags instead of a sync): the call
    completes on every path (tcgen05 step engine, cluster kernel, SIMT) and raises flag bit 1
    (NS_FLAG_NONFINITE)."""
    for bad in (np.nan, np.inf):
        x = I.gaussian(m, n, seed=77)
        x[3, 2] = bad
        ns.read_flags()
        t = torch.from_numpy(x).to(torch.bfloat16).cuda()
        ns.orthogonalize(t, iters=4)
        torch.cuda.synchronize()
        assert ns.read_flags() & 2
    # and the flags clear: a clean call afterwards raises nothing
    t = torch.from_numpy(I.gaussian(m, n, seed=78)).to(torch.bfloat16).cuda()
    ns.orthogonalize(t, iters=4)
    assert ns.read_flags() == 0


def test_fresh_buffers_every_call_do_not_accumulate_workspace():
    """A caller that passes new tensors every call gets a new plan each time; the plan cache
    evicts by workspace bytes, so device memory stays bounded (no OOM, results correct)."""
    shapes = [(4096, 1024)] * 8  # ~200 MB of workspace per plan
    keep = []  # keep every step's inputs alive: each call sees new pointers -> a new plan
    free0 = torch.cuda.mem_get_info()[0]
    c0 = ns.launch_count()
    for step in range(40):  # 40 plans x ~200 MB of workspace would be 8 GB without eviction
        xs = [torch.randn(m, n, device="cuda").bfloat16() for m, n in shapes]
        ns.orthogonalize_list(xs, iters=4)
        keep.append(xs)
    torch.cuda.synchronize()
    assert ns.launch_count() - c0 == 40 * 13
    inputs = 40 * sum(m * n * 2 for m, n in shapes)
    used = free0 - torch.cuda.mem_get_info()[0] - inputs
    assert used < 5 * 2 ** 30, used
    t = keep[-1][0].clone()
    ns.orthogonalize(t, iters=4)
    assert torch.equal(t, keep[-1][0]) is False and torch.isfinite(t.float()).all()


@pytest.mark.parametrize("m,n,dtype", [(300, 201, torch.bfloat16), (201, 300, torch.bfloat16),
                                       (256, 200, torch.float32), (520, 136, torch.float32)])
def test_simt_engine_paths(m, n, dtype):
    """Shapes the TMA engine cannot address (m or n not a multiple of 8) and fp32 matrices
    too big for the cluster kernel run on the CUDA-core step kernels: same gates."""
    bf16 = dtype == torch.bfloat16
    x = I.gaussian(m, n, seed=I.matrix_seed(11, m + n), bf16=bf16)
    out = _run(x, C.turbo(4), "aol", dtype=dtype)
    ref = oracle_run(x, C.turbo(4), "aol")
    assert_parity(out, ref, (BF16_TOL if bf16 else FP32_TOL))


@pytest.mark.parametrize("path", [1, 2])
def test_forced_paths_full_ns(path):
    """ns_set_path(1) (SIMT kernels for everything) and (2) (single-CTA 128x256 tcgen05
    tiles) run the whole iteration within the gates."""
    old = ns.set_path(path)
    try:
        for (m, n) in [(768, 256), (256, 768), (520, 136)]:
            x = I.gaussian(m, n, seed=I.matrix_seed(12, m + n))
            assert_parity(_run(x, C.turbo(4), "aol"), oracle_run(x, C.turbo(4), "aol"), BF16_TOL)
    finally:
        ns.set_path(old)


def test_bench_workload_full_size_sampled():
    """The bench workload itself: the GPT-2-medium set (144 matrices, 604 MB) with bench.py's
    seeded inputs, run the way bench.py times it at N = 1 (orthogonalize_sharded, one bucket);
    every output finite, a sample of matrices of each shape against the fp64 oracle, and the
    sharded results bitwise equal to one grouped call."""
    from paper_2512_04632_b200.parallel import orthogonalize_sharded

    shapes = I.shape_set("gpt2-medium")
    assert len(shapes) == 144
    rng = np.random.default_rng(2025)
    picks = set()
    for s in sorted(set(shapes)):
        idx = [i for i, t in enumerate(shapes) if t == s]
        picks.update(int(i) for i in rng.choice(idx, size=2, replace=False))
    xs_np = {}
    ts = []
    for i, (m, n) in enumerate(shapes):
        x = I.gaussian(m, n, seed=I.matrix_seed(5, i))  # bench.py make_inputs(shapes, 5)
        if i in picks:
            xs_np[i] = x
        ts.append(torch.from_numpy(x).to(torch.bfloat16).cuda())
    outs = orthogonalize_sharded(ts, None, iters=4, precond="aol", buckets=1)
    torch.cuda.synchronize()
    assert all(bool(torch.isfinite(o.float()).all()) for o in outs)
    grouped = [t.clone() for t in ts]
    ns.orthogonalize_list(grouped, iters=4)
    torch.cuda.synchronize()
    for i in sorted(picks):
        assert torch.equal(outs[i], grouped[i]), i
        out = outs[i].float().cpu().numpy().astype(np.float64)
        ref = oracle_run(xs_np[i], C.turbo(4), "aol")
        assert_parity(out, ref, BF16_TOL)
        eg, eo = polar_excess(out, ref, xs_np[i])
        assert eg <= POLAR_SLACK * eo, (i, shapes[i], eg, eo)


def test_internal_graph_replay_bitwise():
    """From a plan's second use on, the library replays its launch sequence as one CUDA
    graph: every replay equals the first (direct) call bitwise, the launch count per call is
    unchanged, and with per-launch profiling on (direct launches again) the result is the same."""
    shapes = [(256, 2304), (64, 216), (768, 768), (1024, 128)]
    xs = [torch.from_numpy(I.gaussian(m, n, seed=700 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    res, counts = [], []
    for _ in range(4):
        outs = [torch.full_like(x, float("nan")) for x in xs]
        c0 = ns.launch_count()
        ns.orthogonalize_list(xs, out=outs, iters=4)
        torch.cuda.synchronize()
        counts.append(ns.launch_count() - c0)
        res.append(outs)
    for r in res[1:]:
        for a, b in zip(res[0], r):
            assert torch.equal(a, b)
    assert len(set(counts)) == 1
    ns.profile_enable(True)
    try:
        outs = [torch.empty_like(x) for x in xs]
        ns.orthogonalize_list(xs, out=outs, iters=4)
        ns.profile_read()
    finally:
        ns.profile_enable(False)
    for a, b in zip(res[0], outs):
        assert torch.equal(a, b)


def test_narrow_tiles_bitwise_equal_wide_tiles():
    """Tile-starved plans use 128-wide tiles (api.cu choose_bn); TNS_BN=256 forces the
    256-wide ones.  Every output element is the same UMMA K-sequence and the AOL partials
    are per 64 columns either way: bitwise equal results, for AOL, Frobenius and split-K."""
    import os
    shapes = [(256, 2304), (768, 256), (520, 136), (2304, 256)]
    xs = [torch.from_numpy(I.gaussian(m, n, seed=800 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    res = {}
    for bn in ("128", "256"):
        os.environ["TNS_BN"] = bn
        try:
            ns.shutdown()
            for precond in ("aol", "frobenius"):
                outs = [torch.empty_like(x) for x in xs]
                ns.orthogonalize_list(xs, out=outs, iters=4, precond=precond)
                torch.cuda.synchronize()
                res[(bn, precond)] = outs
        finally:
            del os.environ["TNS_BN"]
            ns.shutdown()
    for precond in ("aol", "frobenius"):
        for a, b in zip(res[("128", precond)], res[("256", precond)]):
            assert torch.equal(a, b)


def test_unaligned_matrix_does_not_change_the_others():
    """A bf16 list with a matrix TMA cannot address (row pitch not a multiple of 16 bytes,
    short side > 128) runs that one on the CUDA-core kernels and the rest on tcgen05: every
    result bitwise equals its single call, and the aligned ones keep the tensor-core path."""
    shapes = [(768, 768), (300, 201), (1024, 256), (64, 216)]
    xs = [torch.from_numpy(I.gaussian(m, n, seed=900 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    singles = []
    for x in xs:
        t = x.clone()
        ns.orthogonalize(t, iters=4)
        singles.append(t)
    outs = [torch.empty_like(x) for x in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4)
    ns.profile_enable(True)
    try:
        ns.orthogonalize_list(xs, out=outs, iters=4)
        prof = ns.profile_read()
    finally:
        ns.profile_enable(False)
    assert prof["simt"][1] == 12 and prof["update"][1] == 4  # both engines ran (3T SIMT GEMMs)
    for o, s in zip(outs, singles):
        assert torch.equal(o, s)


def test_first_call_on_fresh_pointers_does_not_block_the_host():
    """§8(b): the plan build of a new problem list is stream-ordered (cudaMallocAsync,
    cudaMemsetAsync, cudaMemcpyAsync on the caller's stream): with ~0.3 s of GPU work queued
    ahead of it, the call returns long before that work finishes, and the result is right."""
    import time
    shapes = [(768, 768), (3072, 768), (1000, 64)]
    warm = [torch.from_numpy(I.gaussian(m, n, seed=300 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    ns.orthogonalize_list(warm, iters=4)  # device context set-up (once per process)
    xs = [torch.from_numpy(I.gaussian(m, n, seed=310 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    ref = [x.clone() for x in xs]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(6e8))  # ~0.3 s at 1.9 GHz on the current stream
    t0 = time.perf_counter()
    ns.orthogonalize_list(xs, iters=4)  # fresh pointers: builds a new plan
    host_ms = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    assert host_ms < 150, host_ms
    ns.orthogonalize_list(ref, iters=4)
    torch.cuda.synchronize()
    for a, b in zip(xs, ref):
        assert torch.equal(a, b)


def test_failed_second_plan_leaves_first_group_untouched():
    """A list mixing a TMA-unaligned bf16 matrix with aligned ones runs as two plans; both are
    built before either launches, so when the second does not fit a caller workspace sized
    for the first only, the call fails with NS_ERR_WORKSPACE and no matrix is modified
    (header contract)."""
    shapes = [(300, 301), (768, 768)]  # 301: TMA-unaligned, and N > 256 (no cluster kernel)
    xs = [torch.from_numpy(I.gaussian(m, n, seed=320 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    keep = [x.clone() for x in xs]
    need_first = ns.workspace_size([shapes[0]])
    buf = torch.empty(need_first, dtype=torch.uint8, device="cuda")
    try:
        ns.set_workspace(buf)
        with pytest.raises(ns.NSError, match="NS_ERR_WORKSPACE"):
            ns.orthogonalize_list(xs, iters=4)
        torch.cuda.synchronize()
        for a, b in zip(xs, keep):
            assert torch.equal(a, b)
        # exactly ns_workspace_size bytes is enough for the whole mixed list
        full = torch.empty(ns.workspace_size(shapes), dtype=torch.uint8, device="cuda")
        ns.set_workspace(full)
        outs = [torch.empty_like(x) for x in xs]
        ns.orthogonalize_list(xs, out=outs, iters=4)
        torch.cuda.synchronize()
    finally:
        ns.set_workspace(None)
    for x, o in zip(keep, outs):
        t = x.clone()
        ns.orthogonalize(t, iters=4)
        assert torch.equal(t, o)


def test_same_list_on_two_streams_is_ordered():
    """Thread-safety contract (turbo_ns.h): calls with the SAME problem list share its cached
    workspace; a call on another stream than the previous one waits for that call's last
    launch inside the library, so alternating streams with no caller-side events gives the
    results of one stream (both engines: step engine and tcgen05 cluster kernel)."""
    shapes = [(2048, 2048), (1024, 1024), (3072, 768), (1024, 128)]
    xs = [torch.from_numpy(I.gaussian(m, n, seed=950 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    outs = [torch.empty_like(x) for x in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4)
    ref = [o.clone() for o in outs]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    for i in range(8):
        with torch.cuda.stream(s1 if i % 2 == 0 else s2):
            ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)


def test_concurrent_streams_distinct_lists():
    """Thread-safety contract (turbo_ns.h): calls from several host threads, each on its own
    stream with its own problem list (step engine, tcgen05 cluster kernel and FFMA cluster
    kernel matrices mixed, so the internal side streams are shared), give bitwise the
    results of the same calls made one at a time."""
    import threading
    lists = [[(768, 768), (1024, 128), (64, 216)], [(3072, 768), (256, 2304)], [(512, 512), (64, 576), (128, 128)],
             [(2048, 256), (100, 37)]]
    inputs = [[torch.from_numpy(I.gaussian(m, n, seed=900 + 10 * j + i)).to(torch.bfloat16).cuda()
               for i, (m, n) in enumerate(shapes)] for j, shapes in enumerate(lists)]
    ref = []
    for xs in inputs:
        outs = [torch.empty_like(x) for x in xs]
        ns.orthogonalize_list(xs, out=outs, iters=4)
        ref.append(outs)
    torch.cuda.synchronize()
    results = [None] * len(lists)
    errors = []

    def worker(j):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                outs = [torch.empty_like(x) for x in inputs[j]]
                for _ in range(10):
                    ns.orthogonalize_list(inputs[j], out=outs, iters=4)
            s.synchronize()
            results[j] = outs
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(j,)) for j in range(len(lists))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for r, o in zip(ref, results):
        for a, b in zip(r, o):
            assert torch.equal(a, b)

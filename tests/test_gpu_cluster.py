"""Parity of the cluster-resident small-matrix kernel against the
fp64 oracle, through the C ABI (GPU).

Matrices with short side N <= 128 whose fp32 copy fits in shared memory run the whole NS
in ONE launch of an 8-CTA cluster (path 0).  The same gates as the step engine apply:
relF <= 2e-2 (bf16) / 1e-4 (fp32) against oracle/ns_oracle.py on the same inputs, polar
error within 5% of the oracle's.  Edge cases: 1 x 1, ragged N (not a multiple of 4 or of
the 8-CTA split), wide inputs, the largest eligible M, odd iteration counts in place, zero
columns, a zero matrix, mixing with step-engine matrices (side-stream fork/join, graph
capture).
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


@pytest.fixture(autouse=True)
def _cluster_whenever_it_fits():
    """Path 5: every matrix that fits takes the cluster kernel (path 0 routes bf16 matrices
    with M*N^2 > 2.2e6 to the step engine, measured faster there; see test_auto_routing)."""
    old = ns.set_path(5)
    yield
    ns.set_path(old)


def _run(x32, coeffs, precond, dtype=torch.bfloat16, path=5):
    t = torch.from_numpy(np.ascontiguousarray(x32, dtype=np.float32)).to(dtype).cuda()
    old = ns.set_path(path)
    try:
        c0 = ns.launch_count()
        ns.orthogonalize(t, iters=len(coeffs), precond=precond, coeffs=coeffs)
        torch.cuda.synchronize()
        launches = ns.launch_count() - c0
    finally:
        ns.set_path(old)
    return t.float().cpu().numpy().astype(np.float64), launches


SHAPES = [(128, 128), (64, 216), (216, 64), (64, 576), (100, 37), (37, 100), (5, 3), (1, 1), (160, 128),
          (632, 64), (1352, 32), (96, 200)]


@pytest.mark.parametrize("m,n", SHAPES)
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "fp32"])
def test_cluster_aol4(m, n, dtype):
    x = I.make_matrix(m, n, seed=I.matrix_seed(7, m * 1000 + n), dist="gaussian", bf16=(dtype == torch.bfloat16))
    out, launches = _run(x, C.turbo(4), "aol", dtype)
    assert launches == 1  # the whole NS in one cluster launch
    ref = oracle_run(x, C.turbo(4), "aol")
    assert_parity(out, ref, BF16_TOL if dtype == torch.bfloat16 else FP32_TOL, f"{m}x{n}")
    if min(m, n) > 1:
        eg, eo = polar_excess(out, ref, x)
        assert eg <= 1.05 * eo + (1e-6 if dtype == torch.float32 else 0.0), (eg, eo)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "fp32"])
@pytest.mark.parametrize("m,n", [(128, 128), (64, 576), (100, 37)])
@pytest.mark.parametrize("precond,coeffs", [("frobenius", C.muon_plus(5)), ("aol", C.muon_plus(5)),
                                            ("none", C.turbo(4))])
def test_cluster_preconds_and_odd_iters(m, n, precond, coeffs, dtype):
    """Every preconditioner and an odd iteration count, bf16 and fp32 (fp32: the row-wise
    X' = aX + b(XA) + c((XA)A) of reading R16 where it applies, 128^2 and 64x576)."""
    x = I.gaussian(m, n, seed=3, bf16=dtype == torch.bfloat16)
    if precond == "none":
        x = x / np.float32(4 * np.sqrt(max(m, n)))
        if dtype == torch.bfloat16:
            x = I.round_bf16(x)
    out, launches = _run(x, coeffs, precond, dtype)
    assert launches == 1
    assert_parity(out, oracle_run(x, coeffs, precond), BF16_TOL if dtype == torch.bfloat16 else FP32_TOL)


@pytest.mark.parametrize("dist", ["lowrank", "levy1.0", "levy1.5"])
def test_cluster_distributions(dist):
    x = I.make_matrix(64, 576, seed=11, dist=dist)
    out, _ = _run(x, C.turbo(4), "aol")
    ref = oracle_run(x, C.turbo(4), "aol")
    assert_parity(out, ref, BF16_TOL, dist, model=bf16_model_out(x, C.turbo(4), "aol"))


def test_cluster_matches_step_engine():
    """Cluster kernel (path 0) and the per-step tcgen05 engine (path 4) both meet the gate
    and agree with each other to bf16 rounding."""
    x = I.gaussian(128, 160, seed=12)
    a, la = _run(x, C.turbo(4), "aol", path=5)
    b, lb = _run(x, C.turbo(4), "aol", path=4)
    assert la == 1 and lb == 13
    ref = oracle_run(x, C.turbo(4), "aol")
    assert relF(a, ref) <= BF16_TOL and relF(b, ref) <= BF16_TOL
    assert relF(a, b) <= BF16_TOL


def test_cluster_eligibility_boundary():
    """N = 128 fp32 (the FFMA cluster kernel's own mode): M = 160 is the largest eligible height
    (227 KB of shared memory); 168 goes to the CUDA-core step kernels."""
    for m, want in [(160, 1), (168, 13)]:
        x = I.gaussian(m, 128, seed=13, bf16=False)
        out, launches = _run(x, C.turbo(4), "aol", torch.float32)
        assert launches == want, (m, launches)
        assert_parity(out, oracle_run(x, C.turbo(4), "aol"), FP32_TOL)


def test_cluster_determinism_and_scale_invariance_bitwise():
    x = I.gaussian(64, 216, seed=14)
    a, _ = _run(x, C.turbo(4), "aol")
    b, _ = _run(x, C.turbo(4), "aol")
    c, _ = _run(x * np.float32(16.0), C.turbo(4), "aol")
    assert np.array_equal(a, b)
    assert np.array_equal(a, c)
    assert O.descent_alignment(x, a) > 0


def test_cluster_transpose_symmetry():
    x = I.gaussian(200, 96, seed=15)
    a, _ = _run(x, C.turbo(4), "aol")
    b, _ = _run(np.ascontiguousarray(x.T), C.turbo(4), "aol")
    assert np.array_equal(a, b.T)  # same oriented problem, same kernel: bitwise


def test_cluster_zero_column_and_zero_matrix_flags():
    x = I.gaussian(128, 64, seed=16)
    x[:, 9] = 0
    ns.read_flags()
    out, _ = _run(x, C.turbo(4), "aol")
    assert ns.read_flags() & 1
    assert np.all(np.isfinite(out)) and np.all(out[:, 9] == 0)
    assert_parity(out, oracle_run(x, C.turbo(4), "aol"), BF16_TOL)
    z = np.zeros((32, 48), dtype=np.float32)
    out, _ = _run(z, C.muon_plus(5), "frobenius")
    assert ns.read_flags() & 1
    assert np.all(out == 0)


def test_cluster_in_place_and_out_of_place_odd():
    x = I.gaussian(64, 216, seed=17)
    coeffs = C.muon_plus(5)
    a, _ = _run(x, coeffs, "aol")
    t = torch.from_numpy(x).to(torch.bfloat16).cuda()
    o = torch.empty_like(t)
    ns.orthogonalize_list([t], out=[o], iters=5, precond="aol", coeffs=coeffs)
    torch.cuda.synchronize()
    assert np.array_equal(o.float().cpu().numpy().astype(np.float64), a)
    assert np.array_equal(t.float().cpu().numpy(), x)


def _mixed():
    shapes = [(768, 768), (64, 216), (3072, 768), (128, 128), (256, 2304), (64, 576)]
    return [torch.from_numpy(I.gaussian(m, n, seed=180 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]


def test_mixed_list_fork_join_bitwise():
    """Small matrices on the side stream, the rest through the step engine: one extra
    launch, results bitwise equal to each matrix alone."""
    xs = _mixed()
    singles = []
    for x in xs:
        t = x.clone()
        ns.orthogonalize(t, iters=4)
        singles.append(t)
    outs = [torch.empty_like(x) for x in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4)  # plan
    c0 = ns.launch_count()
    ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    assert ns.launch_count() - c0 == 13 + 1 + 4  # + the split-K Gram reductions of 256 x 2304
    for o, s in zip(outs, singles):
        assert torch.equal(o, s)


def test_mixed_list_graph_capture():
    xs = _mixed()
    outs = [torch.empty_like(x) for x in xs]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ns.orthogonalize_list(xs, out=outs, iters=4)
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


@pytest.mark.parametrize("precond,coeffs", [("frobenius", C.muon_plus(5)), ("aol", C.turbo(4))])
def test_cluster_repeated_calls_bitwise(precond, coeffs):
    """50 launches of the same problem give one bit pattern: guards the DSMEM exchange
    against races (the in-place rescale of A0 once raced with the outgoing bulk copies of
    this CTA's rows -- 1-ulp differences in a few percent of the runs with Frobenius)."""
    x = I.gaussian(128, 128, seed=3)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    ref = None
    for _ in range(50):
        o = torch.empty_like(xt)
        ns.orthogonalize_list([xt], out=[o], iters=len(coeffs), precond=precond, coeffs=coeffs)
        if ref is None:
            ref = o
        else:
            assert torch.equal(o, ref)
    torch.cuda.synchronize()


def test_cluster_size_groups_bitwise():
    """Small matrices that fit the 16-CTA layout and ones that only fit the 8-CTA layout run
    in separate cluster launches; every result is bitwise its single-call result."""
    shapes = [(160, 128), (128, 128), (64, 576), (632, 64)]
    xs = [torch.from_numpy(I.gaussian(m, n, seed=230 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    singles = []
    for x in xs:
        t = x.clone()
        ns.orthogonalize(t, iters=4)
        singles.append(t)
    outs = [torch.empty_like(x) for x in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4)
    c0 = ns.launch_count()
    ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    assert ns.launch_count() - c0 == 2
    for o, s in zip(outs, singles):
        assert torch.equal(o, s)


def test_auto_routing_by_cost():
    """Path 0: bf16 matrices with N <= 128 that TMA can address take the tcgen05 cluster kernel
    (one launch); fp32 ones that fit the FFMA cluster kernel take it (one launch); path 5 sends
    every matrix that fits to the FFMA kernel, path 4 everything to the step engine.  All routes
    meet the gate and agree to rounding."""
    cases = [(64, 216, torch.bfloat16, 1), (64, 576, torch.bfloat16, 1), (160, 128, torch.bfloat16, 1),
             (64, 576, torch.float32, 1), (128, 128, torch.bfloat16, 1)]
    for m, n, dt, want in cases:
        x = I.gaussian(m, n, seed=240, bf16=(dt == torch.bfloat16))
        a, la = _run(x, C.turbo(4), "aol", dt, path=0)
        b, lb = _run(x, C.turbo(4), "aol", dt, path=5)
        c, lc = _run(x, C.turbo(4), "aol", dt, path=4)
        assert la == want and lb == 1 and lc == 13, (m, n, dt, la, lb, lc)
        tol = BF16_TOL if dt == torch.bfloat16 else FP32_TOL
        ref = oracle_run(x, C.turbo(4), "aol")
        assert relF(a, ref) <= tol and relF(b, ref) <= tol and relF(c, ref) <= tol



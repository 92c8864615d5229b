"""Step-level parity of the CUDA path against the fp64 oracle (GPU).

Each step of the hot path is called through its C-ABI entry point (nsx_*), on seeded
synthetic inputs from synth/, and compared element by element with the oracle's
definition of that step (oracle/ns_oracle.py) on the same bf16 values.

Error model: bf16 operands are exact in fp32 products, accumulation is
fp32 (relative ~K*2^-24), and each stored output is rounded once to bf16 (relative
2^-9).  So every element must satisfy |gpu - ref| <= 2^-8 |ref| + tol_abs, with
tol_abs a small multiple of the fp32 accumulation error bound.
"""
import numpy as np
import pytest
import torch

from oracle import ns_oracle as O
from synth import inputs as I

pytestmark = pytest.mark.gpu

ns = pytest.importorskip("paper_2512_04632_b200")

# (m, n): tall, wide, square, ragged (partial 128/256 tiles), tiny, CIFAR-like
SHAPES = [(264, 200), (200, 264), (256, 256), (520, 136), (64, 216), (1024, 768), (72, 8), (8, 1000)]


def _bf(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).cuda()


def _np(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy().astype(np.float64)


def _assert_close(gpu, ref, absmag, rel=2.0 ** -8, k=1.0):
    """|gpu - ref| <= rel*|ref| + 1e-5 * k * absmag  elementwise."""
    err = np.abs(gpu - ref)
    bound = rel * np.abs(ref) + 1e-5 * k * absmag
    bad = err > bound
    assert not bad.any(), (f"{bad.sum()} / {bad.size} elements out of bound; "
                           f"max excess {(err - bound).max():.3e}; max err {err.max():.3e}")


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("path", [0, 1, 2])
def test_gram(shape, path):
    m, n = shape
    x = I.gaussian(m, n, seed=1)
    old = ns.set_path(path)
    try:
        a = _np(ns.gram(_bf(x)))
    finally:
        ns.set_path(old)
    y, _ = O.orient(x)
    ref = O.gram(y)
    # accumulation bound: sum_k |x_ki||x_kj| <= sqrt(A_ii A_jj)
    d = np.sqrt(np.diag(ref))
    _assert_close(a, ref, np.outer(d, d))


def test_gram_mirror_symmetric():
    """Off-diagonal 256-blocks are written twice from one accumulator: bitwise symmetric."""
    x = I.gaussian(300, 776, seed=2)
    a = _np(ns.gram(_bf(x)))
    idx = np.arange(a.shape[0]) // 256
    mask = idx[:, None] != idx[None, :]
    assert np.array_equal(a[mask], a.T[mask])


@pytest.mark.parametrize("N", [136, 256, 520, 768])
@pytest.mark.parametrize("precond", ["aol", "frobenius"])
def test_precondition(N, precond):
    x = I.gaussian(N + 64, N, seed=3)
    a0 = I.round_bf16(O.gram(x.astype(np.float64)))  # bf16 Gram built by the oracle, input to both
    at = _bf(a0)
    s = ns.precondition(at, precond).cpu().numpy().astype(np.float64)
    if precond == "aol":
        s_ref = O.aol_scaling(a0.astype(np.float64))
    else:
        s_ref = np.full(N, 1.0 / np.sqrt(np.trace(a0.astype(np.float64))))
    np.testing.assert_allclose(s, s_ref, rtol=3e-6)
    ref = O.rescale_gram(a0.astype(np.float64), s_ref)
    _assert_close(_np(at), ref, np.abs(ref).max(), k=0.1)


@pytest.mark.parametrize("N", [136, 256, 520, 768])
@pytest.mark.parametrize("scaled", [False, True])
@pytest.mark.parametrize("path", [0, 1, 2])
def test_poly(N, scaled, path):
    x = I.gaussian(N + 40, N, seed=4).astype(np.float64)
    y1, a1 = O.precondition(x, "aol")
    A = I.round_bf16(a1).astype(np.float64)
    b, c = -6.3029, 2.6377
    s = (0.5 + np.random.default_rng(5).random(N)).astype(np.float32)
    old = ns.set_path(path)
    try:
        B = _np(ns.poly(_bf(A), b, c, torch.from_numpy(s).cuda() if scaled else None))
    finally:
        ns.set_path(old)
    ref = b * A + c * (A @ A)
    if scaled:
        ref = ref * s.astype(np.float64)[None, :]
    mag = (np.abs(b) * np.abs(A) + np.abs(c) * (np.abs(A) @ np.abs(A)))
    _assert_close(B, ref, mag.max(), k=0.2)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("scaled", [False, True])
@pytest.mark.parametrize("path", [0, 1, 2])
def test_update(shape, scaled, path):
    m, n = shape
    N = min(m, n)
    x = I.gaussian(m, n, seed=6)
    g = np.random.default_rng(7)
    Bm = I.round_bf16(g.standard_normal((N, N)).astype(np.float32) / np.sqrt(N))
    s = (0.5 + g.random(N)).astype(np.float32)
    a = 3.9505
    old = ns.set_path(path)
    try:
        out = _np(ns.update(_bf(x), _bf(Bm), a, torch.from_numpy(s).cuda() if scaled else None))
    finally:
        ns.set_path(old)
    y, t = O.orient(x.astype(np.float64))
    sv = s.astype(np.float64) if scaled else np.ones(N)
    ref = a * y * sv[None, :] + y @ Bm.astype(np.float64).T  # Out = a Xh diag(s) + Xh B^T
    ref = O.unorient(ref, t)
    mag = np.abs(a) * np.abs(O.unorient(y, t)) * 2 + np.abs(O.unorient(np.abs(y) @ np.abs(Bm.T), t))
    _assert_close(out, ref, mag.max(), k=0.2)


# ------------------------------------------------------------ full-size sampled checks
@pytest.mark.parametrize("shape", [(8192, 8192), (3072, 768), (768, 3072), (4096, 1024)])
def test_full_size_sampled_steps(shape):
    """BASELINE sizes: sampled outputs of each step, computed one by one by fp64 dots."""
    m, n = shape
    x = I.gaussian(m, n, seed=10).astype(np.float64)
    xt = _bf(x)
    y, t = O.orient(x)
    N = y.shape[1]
    A = _np(ns.gram(xt))
    rng = np.random.default_rng(11)
    ii, jj = rng.integers(0, N, 256), rng.integers(0, N, 256)
    ref = np.einsum("ki,ki->i", y[:, ii], y[:, jj])
    scale = np.sqrt(np.einsum("ki,ki->i", y[:, ii], y[:, ii]) * np.einsum("ki,ki->i", y[:, jj], y[:, jj]))
    assert np.all(np.abs(A[ii, jj] - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-5 * scale)
    # poly on a synthetic symmetric input (bf16 values fed to both sides)
    g = np.random.default_rng(12)
    G = g.standard_normal((N, N)).astype(np.float32)
    Ab = I.round_bf16((G + G.T) / np.float32(2.0 * np.sqrt(N))).astype(np.float64)
    b, c = -3.1427, 1.2046
    B = _np(ns.poly(_bf(Ab), b, c))
    ref = b * Ab[ii, jj] + c * np.einsum("ik,ik->i", Ab[ii, :], Ab[jj, :])
    mag = np.abs(b * Ab[ii, jj]) + np.abs(c) * np.einsum("ik,ik->i", np.abs(Ab[ii, :]), np.abs(Ab[jj, :]))
    assert np.all(np.abs(B[ii, jj] - ref) <= 2.0 ** -8 * np.abs(ref) + 2e-6 * mag)
    # update with a synthetic B (not the GPU's poly output)
    Bs = I.round_bf16(g.standard_normal((N, N)).astype(np.float32) / np.float32(np.sqrt(N))).astype(np.float64)
    a = 2.8769
    out = _np(ns.update(xt, _bf(Bs), a))
    rr = rng.integers(0, y.shape[0], 256)
    cc = rng.integers(0, N, 256)
    refu = a * y[rr, cc] + np.einsum("ik,ik->i", y[rr, :], Bs[cc, :])
    magu = np.abs(a * y[rr, cc]) + np.einsum("ik,ik->i", np.abs(y[rr, :]), np.abs(Bs[cc, :]))
    got = out.T[rr, cc] if t else out[rr, cc]
    assert np.all(np.abs(got - refu) <= 2.0 ** -8 * np.abs(refu) + 2e-6 * magu)

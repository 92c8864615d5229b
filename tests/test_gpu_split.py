"""Split-K Gram of the step engine (GPU): in tile-starved calls, for N <= 256 and K = M >=
1024 the Gram XᵀX (Eq. 3 / Eq. 7) runs as S = ceil(nk / 8) independent k-range tiles whose
fp32 partials a reduction launch sums in a fixed order (api.cu choose_splits, simt.cu
split_reduce_kernel).

Gates: the same as the rest of the step engine against the fp64 oracle (relF <= 2e-2, polar
error within 5% of the oracle's); the split factor depends on the shape alone, so results
are bitwise the same across tile-starved calls and deterministic; a call that fills the GPU
does not split and equals the unsplit single call bitwise; the reduction reproduces the AOL
row sums (zero-column flag) and the non-finite flag; with the split disabled (TNS_NOSPLIT=1,
a measurement knob) the result moves only at rounding level.
"""
import os

import numpy as np
import pytest
import torch

from synth import coeffs as C
from synth import inputs as I
from tests.helpers import oracle_run, polar_excess, relF, assert_parity

pytestmark = pytest.mark.gpu

ns = pytest.importorskip("paper_2512_04632_b200")

BF16_TOL = 2e-2
POLAR_SLACK = 1.05

# (m, n): short side <= 256 with a long contraction; wide and tall orientations, ragged N,
# the 16-range cap, and the smallest K that splits (nk = 16 -> S = 2)
SPLIT_CASES = [(256, 2304), (2304, 256), (200, 4096), (128, 8192), (1024, 256), (256, 8192)]


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).cuda()


def _run(x, coeffs, precond="aol"):
    t = _t(x)
    c0 = ns.launch_count()
    ns.orthogonalize(t, iters=len(coeffs), precond=precond, coeffs=coeffs)
    torch.cuda.synchronize()
    return t.float().cpu().numpy().astype(np.float64), ns.launch_count() - c0


@pytest.mark.parametrize("m,n", SPLIT_CASES)
@pytest.mark.parametrize("precond", ["aol", "frobenius"])
def test_split_gram_parity(m, n, precond):
    x = I.gaussian(m, n, seed=m + 3 * n)
    coeffs = C.turbo(4) if precond == "aol" else C.muon_plus(5)
    out, _ = _run(x, coeffs, precond)
    ref = oracle_run(x, coeffs, precond)
    assert np.all(np.isfinite(out))
    assert_parity(out, ref, BF16_TOL)
    eg, eo = polar_excess(out, ref, x)
    assert eg <= POLAR_SLACK * eo, (eg, eo)


def test_split_adds_one_reduction_per_gram():
    """256 x 2304 (nk = 36 -> S = 5): 3T + 1 step launches + T reductions."""
    x = I.gaussian(256, 2304, seed=7)
    _run(x, C.turbo(4))  # plan
    _, launches = _run(x, C.turbo(4))
    assert launches == 3 * 4 + 1 + 4


def test_split_batch_invariant_and_deterministic():
    shapes = [(256, 2304), (64, 216), (768, 768), (200, 4096), (1024, 256)]
    xs = [I.gaussian(m, n, seed=300 + i) for i, (m, n) in enumerate(shapes)]
    singles = [_run(x, C.turbo(4))[0] for x in xs]
    ts = [_t(x) for x in xs]
    ns.orthogonalize_list(ts, iters=4)
    torch.cuda.synchronize()
    for t, s in zip(ts, singles):
        assert np.array_equal(t.float().cpu().numpy().astype(np.float64), s)
    again = _run(xs[0], C.turbo(4))[0]
    assert np.array_equal(again, singles[0])


def test_full_call_splits_shape_only():
    """64 x (256 x 2304) fills the GPU, and still splits (reading R11, round 2: the split-K
    choice depends on the shape alone): T reductions, and every result equals its single
    call bitwise -- the property the sharded path needs (a matrix's result must not depend
    on which rank's list it lands in)."""
    xs = [I.gaussian(256, 2304, seed=500 + i) for i in range(64)]
    ts = [_t(x) for x in xs]
    ns.orthogonalize_list(ts, iters=4)  # plan
    ts = [_t(x) for x in xs]
    c0 = ns.launch_count()
    ns.orthogonalize_list(ts, iters=4)
    torch.cuda.synchronize()
    assert ns.launch_count() - c0 == 3 * 4 + 1 + 4
    for i in (0, 31, 63):
        s, _ = _run(xs[i], C.turbo(4))
        assert np.array_equal(ts[i].float().cpu().numpy().astype(np.float64), s)


def test_split_vs_unsplit_rounding_level():
    x = I.gaussian(256, 2304, seed=11)
    a, la = _run(x, C.turbo(4))
    os.environ["TNS_NOSPLIT"] = "1"
    try:
        ns.shutdown()  # plans are rebuilt: the knob is read at plan build
        b, lb = _run(x, C.turbo(4))
    finally:
        del os.environ["TNS_NOSPLIT"]
        ns.shutdown()
    assert la == lb + 4
    assert relF(a, b) <= 1e-2
    ref = oracle_run(x, C.turbo(4), "aol")
    assert abs(relF(a, ref) - relF(b, ref)) <= 5e-3


def test_split_zero_column_and_nonfinite_flags():
    x = I.gaussian(2304, 256, seed=12)
    x[:, 17] = 0
    ns.read_flags()
    out, _ = _run(x, C.turbo(4))
    assert ns.read_flags() & 1  # AOL: zero row of A0 -> s = 0, flagged (from the reduction's sums)
    assert np.all(out[:, 17] == 0) and np.all(np.isfinite(out))
    assert_parity(out, oracle_run(x, C.turbo(4), "aol"), BF16_TOL)
    y = I.gaussian(256, 2304, seed=13)
    y[3, 5] = np.nan
    ns.read_flags()
    _run(y, C.turbo(4))
    assert ns.read_flags() & 2


def test_split_workspace_size_covers_plan():
    """ns_workspace_size accounts for the partials: a caller-owned buffer of exactly that
    size serves a split problem list."""
    shapes = [(256, 2304), (128, 8192)]
    need = ns.workspace_size(shapes)
    buf = torch.empty(need + 256, dtype=torch.uint8, device="cuda")
    xs = [_t(I.gaussian(m, n, seed=400 + i)) for i, (m, n) in enumerate(shapes)]
    ref = [t.clone() for t in xs]
    ns.orthogonalize_list(ref, iters=4)
    ns.set_workspace(buf)
    try:
        ns.orthogonalize_list(xs, iters=4)
        torch.cuda.synchronize()
    finally:
        ns.set_workspace(None)
    for a, b in zip(xs, ref):
        assert torch.equal(a, b)

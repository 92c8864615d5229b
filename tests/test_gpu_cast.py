"""Mixed precision (ns_orthogonalize_cast): fp32 caller matrices, bf16
compute.  Pin: the result is bitwise float(NS_bf16(bf16_rne(X))) -- the same NS the bf16 API
computes on the RNE-cast input -- for the step engine, the split-K path and the cluster
kernel, in place and out of place, odd and even iteration counts; and within the bf16 gate
of the fp64 oracle."""
import numpy as np
import pytest
import torch

from synth import coeffs as C
from synth import inputs as I
from tests.helpers import oracle_run, relF, assert_parity

pytestmark = pytest.mark.gpu

ns = pytest.importorskip("paper_2512_04632_b200")

SHAPES = [(768, 256), (256, 2304), (64, 216), (100, 37), (300, 201), (1024, 1024)]


def _inputs(seed):
    # fp32 values that are NOT bf16-representable, so the cast matters
    return [I.gaussian(m, n, seed=seed + i, bf16=False) for i, (m, n) in enumerate(SHAPES)]


@pytest.mark.parametrize("iters,precond", [(4, "aol"), (5, "frobenius")])
@pytest.mark.parametrize("inplace", [True, False])
def test_cast_equals_bf16_path_bitwise(iters, precond, inplace):
    coeffs = C.turbo(4) if precond == "aol" else C.muon_plus(5)
    xs = _inputs(900)
    f32 = [torch.from_numpy(x).cuda() for x in xs]
    ref = [t.to(torch.bfloat16) for t in f32]  # torch RNE cast
    ns.orthogonalize_list(ref, iters=iters, precond=precond, coeffs=coeffs)
    outs = None if inplace else [torch.full_like(t, float("nan")) for t in f32]
    got = ns.orthogonalize_list(f32, out=outs, iters=iters, precond=precond, coeffs=coeffs,
                                compute=torch.bfloat16)
    torch.cuda.synchronize()
    for g, r, x in zip(got, ref, xs):
        assert g.dtype == torch.float32
        assert torch.equal(g, r.float())
    if not inplace:  # inputs untouched
        for t, x in zip(f32, xs):
            assert np.array_equal(t.cpu().numpy(), x)


def test_cast_parity_with_oracle_and_repeat():
    xs = _inputs(950)
    f32 = [torch.from_numpy(x).cuda() for x in xs]
    outs = [torch.empty_like(t) for t in f32]
    for _ in range(3):  # plan, graph capture, graph replay
        ns.orthogonalize_list(f32, out=outs, iters=4, compute=torch.bfloat16)
    torch.cuda.synchronize()
    for o, x in zip(outs, xs):
        ref = oracle_run(I.round_bf16(x), C.turbo(4), "aol")
        assert_parity(o.cpu().numpy().astype(np.float64), ref, 2e-2)


def test_cast_rejects_bad_combinations():
    x = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        ns.orthogonalize_list([x], compute=torch.float16)

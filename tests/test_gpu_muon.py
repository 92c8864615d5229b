"""Muon optimizer step (ns_muon_step / TurboMuon) against the fp64 Muon-step oracle (GPU)."""
import numpy as np
import pytest
import torch

from oracle import muon_oracle as MO
from oracle import ns_oracle as O
from synth import coeffs as C
from synth import inputs as I
from tests.helpers import relF

pytestmark = pytest.mark.gpu
ns = pytest.importorskip("paper_2512_04632_b200")


@pytest.mark.parametrize("wdt", [torch.float32, torch.bfloat16])
def test_turbo_muon_two_steps_vs_oracle(wdt):
    # (100, 37): numel % 8 != 0 -> the element-wise fallback of the momentum/update kernels
    shapes = [(768, 768), (3072, 768), (768, 3072), (64, 576), (100, 37)]
    lr, beta, wd = 0.05, 0.9, 0.01
    ws = [I.gaussian(m, n, seed=200 + i, bf16=(wdt == torch.bfloat16)) for i, (m, n) in enumerate(shapes)]
    params = [torch.nn.Parameter(torch.from_numpy(w).to(wdt).cuda()) for w in ws]
    opt = ns.TurboMuon(params, lr=lr, momentum=beta, weight_decay=wd)
    W = [p.detach().double().cpu().numpy() for p in params]
    M = [np.zeros(s) for s in shapes]
    for step in range(2):
        W_prev = [w.copy() for w in W]
        grads = [I.gaussian(m, n, seed=300 + 10 * step + i) for i, (m, n) in enumerate(shapes)]
        for p, g in zip(params, grads):
            p.grad = torch.from_numpy(g).to(wdt).cuda()
        opt.step()
        torch.cuda.synchronize()
        for i, (p, g) in enumerate(zip(params, grads)):
            M[i], U = MO.muon_momentum(g.astype(np.float64), M[i], beta, nesterov=True)
            # the GPU orthogonalises bf16(U): feed the oracle the same rounding of U
            Ub = I.round_bf16(U.astype(np.float32)).astype(np.float64)
            Ot = O.newton_schulz(Ub, C.turbo(4), "aol")
            W[i] = W[i] * (1 - lr * wd) - lr * MO.muon_scale(*shapes[i]) * Ot
            st = opt.state[p]
            np.testing.assert_allclose(st["momentum_buffer"].cpu().numpy(), M[i], rtol=1e-5, atol=1e-6)
            got = p.detach().double().cpu().numpy()
            assert relF(got, W[i]) <= 1e-2
            # the applied update itself: (W_prev (1 - lr wd) - W_new) / (lr scale) vs NS(U)
            upd = (W_prev[i] * (1 - lr * wd) - got) / (lr * MO.muon_scale(*shapes[i]))
            if wdt == torch.float32:
                assert relF(upd, Ot) <= 2e-2
            W[i] = got  # continue from the GPU state (bf16 weights round every step)
        del grads


def test_muon_step_beta0_equals_plain_ns():
    """beta = 0, wd = 0: W1 = W - lr * scale * NS(G) exactly as the orthogonalize call."""
    m, n = 1024, 256
    w = torch.from_numpy(I.gaussian(m, n, seed=1, bf16=False)).cuda()
    g = torch.from_numpy(I.gaussian(m, n, seed=2)).cuda()  # bf16-representable fp32 values
    p = torch.nn.Parameter(w.clone())
    p.grad = g.clone()
    ns.TurboMuon([p], lr=0.1, momentum=0.0, weight_decay=0.0).step()
    o = g.to(torch.bfloat16)
    ns.orthogonalize(o, iters=4)
    exp = w - 0.1 * 2.0 * o.float()
    torch.cuda.synchronize()
    assert torch.allclose(p.detach(), exp, rtol=0, atol=1e-6)

"""Muon optimizer step (ns_muon_step / TurboMuon) against the fp64 Muon-step oracle (GPU)."""
import os

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


def test_muon_apply_matches_formula():
    """ns_muon_apply: W <- W (1 - lr wd) - lr max(1, m/n)^(1/2) U (fp32 weights, bf16 U)."""
    shapes = [(768, 256), (256, 768), (100, 37)]
    ws = [torch.from_numpy(I.gaussian(m, n, seed=400 + i, bf16=False)).cuda() for i, (m, n) in enumerate(shapes)]
    us = [torch.from_numpy(I.gaussian(m, n, seed=500 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    ref = [w.clone() * (1 - 0.1 * 0.01) - 0.1 * MO.muon_scale(*w.shape) * u.float() for w, u in zip(ws, us)]
    ns.muon_apply(ws, us, lr=0.1, weight_decay=0.01)
    torch.cuda.synchronize()
    for w, r in zip(ws, ref):
        assert torch.allclose(w, r, rtol=1e-6, atol=1e-7)


def test_distributed_turbo_muon_world1_equals_turbo_muon():
    """DistributedTurboMuon (reduce-scatter by ownership -> owner's fused step -> all-gather
    of U -> ns_muon_apply elsewhere) at NCCL world size 1 gives bitwise the TurboMuon result."""
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29541"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        shapes = [(768, 768), (3072, 768), (768, 3072), (64, 576)]
        ws = [I.gaussian(m, n, seed=600 + i, bf16=False) for i, (m, n) in enumerate(shapes)]
        pa = [torch.nn.Parameter(torch.from_numpy(w).cuda()) for w in ws]
        pb = [torch.nn.Parameter(torch.from_numpy(w).cuda()) for w in ws]
        oa = ns.TurboMuon(pa, lr=0.05, momentum=0.9, weight_decay=0.01)
        ob = ns.DistributedTurboMuon(pb, lr=0.05, momentum=0.9, weight_decay=0.01)
        for step in range(2):
            for i, (m, n) in enumerate(shapes):
                g = torch.from_numpy(I.gaussian(m, n, seed=700 + 10 * step + i)).cuda()
                pa[i].grad = g.clone()
                pb[i].grad = g.clone()
            oa.step()
            ob.step()
            torch.cuda.synchronize()
            for a, b in zip(pa, pb):
                assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


def test_turbo_muon_step_cuda_graph():
    """After the first (table-building) step, an optimizer step only enqueues launches: it
    can be captured in a CUDA graph and replayed with results bitwise equal to eager steps."""
    shapes = [(768, 768), (3072, 768), (64, 576)]
    ws = [I.gaussian(m, n, seed=800 + i, bf16=False) for i, (m, n) in enumerate(shapes)]
    gs = [torch.from_numpy(I.gaussian(m, n, seed=900 + i)).cuda() for i, (m, n) in enumerate(shapes)]
    pa = [torch.nn.Parameter(torch.from_numpy(w).cuda()) for w in ws]
    pb = [torch.nn.Parameter(torch.from_numpy(w).cuda()) for w in ws]
    for p, g in zip(pa + pb, gs + gs):
        p.grad = g.clone()
    oa = ns.TurboMuon(pa, lr=0.02, momentum=0.9)
    ob = ns.TurboMuon(pb, lr=0.02, momentum=0.9)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        oa.step()
        ob.step()  # builds tables and plans
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ob.step()
    for _ in range(3):
        oa.step()
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(pa, pb):
        assert torch.equal(a, b)


def test_grad_scale_folds_the_mean():
    """ns_muon_step's grad_scale (the data-parallel 1/world mean inside the momentum kernel):
    a step on G with grad_scale 1/4 is bitwise the step on G / 4 (exact power-of-two scale)."""
    from paper_2512_04632_b200.muon import _coeff_carr, _muon_step_call
    from paper_2512_04632_b200._lib import DTYPE_FP32
    m, n = 768, 512
    w0 = torch.from_numpy(I.gaussian(m, n, seed=7, bf16=False)).cuda()
    g = torch.from_numpy(I.gaussian(m, n, seed=8, bf16=False)).cuda()
    group = {"lr": 0.05, "momentum": 0.9, "weight_decay": 0.01, "nesterov": True, "iters": 4, "precond": "aol",
             "coeffs": None}
    outs = []
    for gg, scale in ((g, 0.25), (g / 4, 1.0)):
        w = w0.clone()
        mom = torch.full((m, n), 0.5, device="cuda")
        u = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
        _muon_step_call([w.data_ptr()], [gg.data_ptr()], [mom.data_ptr()], [u.data_ptr()], [m], [n], DTYPE_FP32,
                        DTYPE_FP32, group, _coeff_carr(group), w.device, grad_scale=scale)
        torch.cuda.synchronize()
        outs.append((w, mom))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])

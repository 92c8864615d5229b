"""Time one TurboMuon optimizer step (momentum + NS + update) on the GPT-2-medium hidden
matrices and its parts; the momentum/update kernels are HBM-bound (bytes per element below).

    python tools/muon_bench.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402


def ev(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


shapes = I.shape_set("gpt2-medium")
params = [torch.nn.Parameter(torch.randn(m, n, device="cuda") * 0.02) for m, n in shapes]
for p in params:
    p.grad = torch.randn_like(p).bfloat16().float()
opt = ns.TurboMuon(params, lr=0.02, momentum=0.95)
ms_step = ev(lambda: opt.step())
us = [opt.state[p]["ns_staging"] for p in params]
ms_ns = ev(lambda: ns.orthogonalize_list(us, iters=4))
numel = sum(m * n for m, n in shapes)
# momentum: read G (fp32 4 B) + M (4 B), write M (4 B) + U (bf16 2 B) = 14 B/elem;
# update: read W (4) + U (2), write W (4) = 10 B/elem
bytes_aux = numel * (14 + 10)
aux_ms = ms_step - ms_ns
print(json.dumps({"workload": "gpt2-medium", "params": numel, "ms_step": round(ms_step, 3), "ms_ns": round(ms_ns, 3),
                  "ms_momentum_plus_update": round(aux_ms, 3),
                  "gbs_momentum_plus_update": round(bytes_aux / (aux_ms * 1e-3) / 1e9, 1) if aux_ms > 0 else None}))

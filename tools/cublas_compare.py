"""Context comparator (bench/analysis only, never the product): cuBLAS (torch.bmm, bf16) on
the same GEMM shapes as one XB launch of the GPT-2-medium set -- 96 x (1024x1024 @ 1024x1024)
and 48 x (4096x1024 @ 1024x1024) -- against this library's XB launch on those shapes.

    python tools/cublas_compare.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402


def ev_time(fn, reps=20):
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


g = torch.Generator(device="cuda").manual_seed(0)
sq_x = torch.randn(96, 1024, 1024, device="cuda", generator=g).bfloat16()
sq_b = torch.randn(96, 1024, 1024, device="cuda", generator=g).bfloat16()
tl_x = torch.randn(48, 4096, 1024, device="cuda", generator=g).bfloat16()
tl_b = torch.randn(48, 1024, 1024, device="cuda", generator=g).bfloat16()
flops = 2 * (96 * 1024 ** 3 + 48 * 4096 * 1024 * 1024)
ms_cublas = ev_time(lambda: (torch.bmm(sq_x, sq_b), torch.bmm(tl_x, tl_b)))
# ours: per-launch XB time from the library's profile events on the real NS call
shapes = I.shape_set("gpt2-medium")
xs = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
outs = [torch.empty_like(t) for t in xs]
for _ in range(3):
    ns.orthogonalize_list(xs, out=outs, iters=4)
torch.cuda.synchronize()
ns.profile_enable(True)
for _ in range(10):
    ns.orthogonalize_list(xs, out=outs, iters=4)
torch.cuda.synchronize()
prof = ns.profile_read()
ns.profile_enable(False)
ms_xb = prof["update"][0] / prof["update"][1]
ms_gram = prof["gram"][0] / prof["gram"][1]
print(json.dumps({"xb_gemm_flops": flops, "cublas_bmm_ms": round(ms_cublas, 4),
                  "cublas_tflops": round(flops / ms_cublas / 1e9, 1), "ours_xb_ms": round(ms_xb, 4),
                  "ours_xb_tflops": round(flops / ms_xb / 1e9, 1), "ours_gram_ms": round(ms_gram, 4),
                  "note": "same dense FLOPs (2*M*N*N summed); cuBLAS computes plain products, ours includes the epilogue"}))

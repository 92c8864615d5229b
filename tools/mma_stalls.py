"""MMA-issuer stall breakdown (needs a TNS_MEASURE=1 build; TNS_DBG=64): per accumulator
tile, cycles the single MMA-issuing thread waited for a free TMEM accumulator (epilogue-
bound), waited for operands (feed-bound), and spent issuing.

    TNS_DBG=64 python tools/mma_stalls.py gpt2-medium
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from paper_2512_04632_b200._lib import lib  # noqa: E402
from synth import inputs as I  # noqa: E402

for w in sys.argv[1:] or ["gpt2-medium"]:
    shapes = I.shape_set(w)
    xs = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    outs = [torch.empty_like(t) for t in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    c = (ctypes.c_uint64 * 8)()
    lib.nsx_epilogue_counters(c, 1)
    for _ in range(5):
        ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    lib.nsx_epilogue_counters(c, 1)
    n = max(c[0], 1)
    tot = c[1] + c[2] + c[3]
    print(json.dumps({"workload": w, "tiles": c[0], "cycles_per_tile": {"wait_accumulator": round(c[1] / n),
                      "wait_operands": round(c[2] / n), "issue": round(c[3] / n)},
                      "share": {"epilogue_bound": round(c[1] / tot, 3), "feed_bound": round(c[2] / tot, 3),
                                "issuing": round(c[3] / tot, 3)}}))

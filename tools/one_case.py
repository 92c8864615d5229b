"""Run one small orthogonalisation a few times (for ncu launch lists of the small configs).

    python tools/one_case.py 64 216 [fp32] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
fp32 = len(sys.argv) > 3 and sys.argv[3] == "fp32"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
x = torch.from_numpy(I.gaussian(m, n, seed=0, bf16=not fp32)).cuda()
if not fp32:
    x = x.to(torch.bfloat16)
o = torch.empty_like(x)
dbg = int(os.environ.get("TNS_DBG", "0"))
if dbg & (8 | 16 | 128):
    import ctypes
    from paper_2512_04632_b200._lib import lib
    ns.orthogonalize_list([x], out=[o], iters=4)
    c = (ctypes.c_uint64 * 8)()
    lib.nsx_epilogue_counters(c, 1)
for _ in range(reps):
    ns.orthogonalize_list([x], out=[o], iters=4)
torch.cuda.synchronize()
print("ok", float(o.float().norm()))
if dbg & 128:
    lib.nsx_epilogue_counters(c, 1)
    names = ["load", "G0", "precond", "P0", "Xcomp0", "Xbcast0", "loop_end", "end"]
    print({names[i]: int(c[i]) for i in range(7)}, "launches", c[7])
elif dbg & 8:
    lib.nsx_epilogue_counters(c, 1)
    n = max(c[0], 1)
    names = ["warp_tiles", "wait_acc", "tmem_ld", "aux_wait", "math", "bulk_read_wait", "store_issue"]
    print({names[i]: (int(c[i]) if i == 0 else round(c[i] / n)) for i in range(7)})
elif dbg & 16:
    lib.nsx_epilogue_counters(c, 1)
    n = max(c[7], 1)
    names = ["setup", "pdl_wait", "first_tma_issued", "first_operands", "first_acc", "epi_done", "end"]
    print({names[i]: round(c[i] / n) for i in range(7)}, "launches", c[7])

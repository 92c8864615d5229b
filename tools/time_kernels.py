"""Per-kernel CUDA-event timing of one workload (library profiling hook).

    python tools/time_kernels.py --workload gpt2-medium --reps 10
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="gpt2-medium")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--iters", type=int, default=4)
a = ap.parse_args()
if os.environ.get("TNS_PATH"):
    ns.set_path(int(os.environ["TNS_PATH"]))
shapes = I.shape_set(a.workload)
xs = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
outs = [torch.empty_like(t) for t in xs]
for _ in range(3):
    ns.orthogonalize_list(xs, out=outs, iters=a.iters)
torch.cuda.synchronize()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
import time  # noqa: E402
from paper_2512_04632_b200.parallel import orthogonalize_sharded  # noqa: E402
orthogonalize_sharded(xs, iters=a.iters)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h0 = time.perf_counter()
for _ in range(a.reps):
    orthogonalize_sharded(xs, iters=a.iters)  # the bench's step (packed outputs)
host_us = (time.perf_counter() - h0) / a.reps * 1e6
e1.record()
torch.cuda.synchronize()
ms_sharded = e0.elapsed_time(e1) / a.reps
e0.record()
for _ in range(a.reps):
    ns.orthogonalize_list(xs, out=outs, iters=a.iters)
e1.record()
torch.cuda.synchronize()
ms_clean = e0.elapsed_time(e1) / a.reps
cs = ClockSampler(0)
cs.start()
ns.profile_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    ns.orthogonalize_list(xs, out=outs, iters=a.iters)
e1.record()
torch.cuda.synchronize()
prof = ns.profile_read()
clk = cs.stop()
print(json.dumps({"workload": a.workload, "dbg": os.environ.get("TNS_DBG", "0"), "path": os.environ.get("TNS_PATH", "0"), "sm_mhz": clk["sm_mhz"],
                  "reasons": clk["reasons"], "ms_per_call_no_events": round(ms_clean, 4),
                  "ms_sharded_step": round(ms_sharded, 4), "host_us_per_step": round(host_us, 1),
                  "ms_per_call": round(e0.elapsed_time(e1) / a.reps, 4),
                  "kernel_ms_per_call": {k: round(v[0] / a.reps, 4) for k, v in prof.items() if v[1]}}))
if int(os.environ.get("TNS_DBG", "0")) & 8:
    import ctypes
    from paper_2512_04632_b200._lib import lib
    c = (ctypes.c_uint64 * 8)()
    lib.nsx_epilogue_counters(c, 1)
    n = max(c[0], 1)
    names = ["tiles", "wait_acc", "tmem_ld", "aux_wait", "math", "stage_wait", "store_issue", "-"]
    print(json.dumps({"epilogue_cycles_per_warp_tile": {names[i]: round(c[i] / n, 1) for i in range(1, 7)},
                      "warp_tiles": c[0]}))

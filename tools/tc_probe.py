"""Latency of the cluster-resident tcgen05 kernel vs the step engine (graph replay of one
call, median of 3 x 50 replays): CIFAR set and single mid-size matrices, ns_set_path 0 (auto:
tcgen05 cluster kernel for N <= 256 bf16 that fits) vs 4 (step engine only) vs 7 (tcgen05
cluster kernel also for the FFMA kernel's small ones)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402


def replay_us(xs, outs):
    ns.orthogonalize_list(xs, out=outs, iters=4)
    ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ns.orthogonalize_list(xs, out=outs, iters=4)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 50 * 1e3)
    return statistics.median(ts)


cases = {"cifar": I.shape_set("cifar"), "256x2304": [(256, 2304)], "256x576": [(256, 576)],
         "768x256": [(768, 256)], "1024x128": [(1024, 128)], "64x576": [(64, 576)], "64x216": [(64, 216)],
         "128x128": [(128, 128)], "3072x192": [(3072, 192)], "gpt2-small-like 16x768x256": [(768, 256)] * 16,
         "batch 64x1024x128": [(1024, 128)] * 64, "batch 64x64x576": [(64, 576)] * 64,
         "batch 16x1024x128": [(1024, 128)] * 16}
if len(sys.argv) > 1:  # a subset by name prefix
    cases = {k: v for k, v in cases.items() if any(k.startswith(a) for a in sys.argv[1:])}
for name, shapes in cases.items():
    xs = [torch.randn(m, n, device="cuda").bfloat16() for m, n in shapes]
    outs = [torch.empty_like(x) for x in xs]
    row = [name]
    for path in (0, 4, 7):
        old = ns.set_path(path)
        try:
            ns.shutdown()
            c0 = ns.launch_count()
            ns.orthogonalize_list(xs, out=outs, iters=4)
            torch.cuda.synchronize()
            nl = ns.launch_count() - c0
            row.append(f"path{path} {replay_us(xs, outs):7.1f} us ({nl} launches)")
        finally:
            ns.set_path(old)
    print("  ".join(row), flush=True)

"""Graph-replay latency of the FFMA cluster kernel (fp32 exact mode and TMA-unaligned bf16
small matrices): one call per case, median of 3 x 50 replays."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
import statistics  # noqa: E402


def replay_us(xs, outs):
    for _ in range(2):
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


cases = [("128x128 fp32", (128, 128), torch.float32), ("64x216 fp32", (64, 216), torch.float32),
         ("256x64 fp32", (256, 64), torch.float32), ("64x27 bf16", (64, 27), torch.bfloat16),
         ("100x36 bf16", (100, 36), torch.bfloat16)]
for name, (m, n), dt in cases:
    xs = [torch.randn(m, n, device="cuda").to(dt)]
    outs = [torch.empty_like(xs[0])]
    c0 = ns.launch_count()
    ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    print(f"{name:14s} {replay_us(xs, outs):7.1f} us ({ns.launch_count() - c0} launches)", flush=True)

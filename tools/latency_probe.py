"""Latency breakdown of the small configs (CIFAR conv set, 128^2 fp32): one call timed
alone, back-to-back calls, CUDA-graph replay, per-kernel profile events, per library path.

    python tools/latency_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402


def case(name, xs, outs, path):
    ns.set_path(path)
    f = lambda: ns.orthogonalize_list(xs, out=outs, iters=4)  # noqa: E731
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    single = ts[len(ts) // 2] * 1e3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    for _ in range(100):
        f()
    e1.record()
    host = (time.perf_counter() - h0) / 100 * 1e6
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / 100 * 1e3
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(100):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / 100 * 1e3
    ns.profile_enable(True)
    for _ in range(20):
        f()
    torch.cuda.synchronize()
    prof = ns.profile_read()
    ns.profile_enable(False)
    print(json.dumps({"case": name, "path": path, "launches": ns.launch_count(), "us_single_call": round(single, 1),
                      "us_back_to_back": round(b2b, 1), "host_us_per_call": round(host, 1),
                      "us_graph_replay": round(graph, 1),
                      "kernel_us_per_call": {k: round(v[0] / 20 * 1e3, 1) for k, v in prof.items() if v[1]},
                      "kernel_launches_per_call": {k: v[1] / 20 for k, v in prof.items() if v[1]}}), flush=True)


shapes = I.shape_set("cifar")
xs = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
outs = [torch.empty_like(t) for t in xs]
for p in [int(v) for v in os.environ.get("PATHS", "0,3,4").split(",")]:
    case("cifar", xs, outs, p)
for shp in [(256, 2304), (64, 216)]:
    x = [torch.from_numpy(I.gaussian(*shp, seed=0)).to(torch.bfloat16).cuda()]
    case(f"{shp[0]}x{shp[1]}", x, [torch.empty_like(x[0])], 0)
x1 = [torch.from_numpy(I.gaussian(128, 128, seed=0, bf16=False)).cuda()]
case("fp32_128", x1, [torch.empty_like(x1[0])], 0)
ns.set_path(0)

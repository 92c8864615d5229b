"""Cost of small matrices riding along a big call: GPT-2-small set alone vs with 2 / 8 small
bf16 matrices (cluster kernel on the side stream), graph replay."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402


def graph_us(shapes):
    xs = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    outs = [torch.empty_like(x) for x in xs]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ns.orthogonalize_list(xs, out=outs, iters=4)
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / 20 * 1e3, 1)


base = I.shape_set(sys.argv[1] if len(sys.argv) > 1 else "gpt2-small")
for extra in ([], [(64, 216)] * 2, [(64, 216)] * 8, [(128, 128)] * 8):
    print(json.dumps({"extra": f"{len(extra)} x {extra[0] if extra else ''}", "us": graph_us(base + extra),
                      "alone_small_us": graph_us(extra) if extra else None}), flush=True)

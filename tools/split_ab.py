"""CUDA-graph replay time of one orthogonalize_list call, split-K Gram on/off (TNS_NOSPLIT),
interleaved, for a few tall short-side <= 256 problem lists."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402

CASES = {
    "cifar": I.shape_set("cifar"),
    "256x2304": [(256, 2304)],
    "256x8192": [(256, 8192)],
    "128x8192": [(128, 8192)],
    "256x16384": [(256, 16384)],
    "8x(256x4608)": [(256, 4608)] * 8,
    "64x(256x2304)": [(256, 2304)] * 64,
}


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
    for _ in range(5):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 50 * 1e3


for rep in range(2):
    for name, shapes in CASES.items():
        r = {}
        for v in ("0", "1"):
            os.environ["TNS_NOSPLIT"] = v
            ns.shutdown()
            r["split" if v == "0" else "nosplit"] = round(graph_us(shapes), 1)
        print(json.dumps({"case": name, **r}), flush=True)

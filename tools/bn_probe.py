"""Graph replay of a few mid-size problem lists with the tile width forced (TNS_BN=128/256
in the environment, one process per setting)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402

CASES = {"gpt2-small": I.shape_set("gpt2-small"), "2048^2": [(2048, 2048)], "1024^2x4": [(1024, 1024)] * 4,
         "4096x1024": [(4096, 1024)], "cifar": I.shape_set("cifar"), "768x768x8": [(768, 768)] * 8}
res = {"bn": os.environ.get("TNS_BN", "auto")}
for name, shapes in CASES.items():
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
    res[name] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
print(json.dumps(res), flush=True)

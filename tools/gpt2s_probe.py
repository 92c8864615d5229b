"""Median ms of one GPT-2-small grouped call (L2 flushed before each), as bench extras."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402

shapes = I.shape_set("gpt2-small")
xs = [torch.from_numpy(I.gaussian(m, n, seed=I.matrix_seed(2, i))).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
outs = [torch.empty_like(t) for t in xs]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3):
    ns.orthogonalize_list(xs, out=outs, iters=4)
ts = []
for _ in range(20):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ns.orthogonalize_list(xs, out=outs, iters=4)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(round(statistics.median(ts), 4))

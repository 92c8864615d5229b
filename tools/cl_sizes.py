"""Graph-replay time of the cluster-resident kernel for a few small shapes (A/B of the
cluster size with TNS_CL_CTAS=8 in a separate process)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402

res = {}
ns.set_path(int(os.environ.get("NS_PATH", "0")))
for (m, n, fp32) in [(64, 216, False), (64, 576, False), (128, 128, True), (128, 128, False), (96, 96, False), (32, 1000, False)]:
    x = torch.from_numpy(I.gaussian(m, n, seed=1, bf16=not fp32))
    x = (x if fp32 else x.to(torch.bfloat16)).cuda()
    o = torch.empty_like(x)
    for _ in range(3):
        ns.orthogonalize_list([x], out=[o], iters=4)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ns.orthogonalize_list([x], out=[o], iters=4)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        ns.orthogonalize_list([x], out=[o], iters=4)
    for _ in range(5):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(100):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res[f"{m}x{n}{'f32' if fp32 else ''}"] = round(e0.elapsed_time(e1) / 100 * 1e3, 1)
print(json.dumps({"ctas": os.environ.get("TNS_CL_CTAS", "auto"), "path": os.environ.get("NS_PATH", "0"), **res}))

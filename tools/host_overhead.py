"""Host-side cost of one library call (no GPU wait): 8 calls enqueued back to back after a
synchronize (few enough launches that the launch queue never fills), per call; for the
public list API and for a PreparedCall (argument arrays built once)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from paper_2512_04632_b200.api import PreparedCall  # noqa: E402
from synth import inputs as I  # noqa: E402

CASES = {"cifar": I.shape_set("cifar"), "256x2304": [(256, 2304)], "768x256": [(768, 256)],
         "gpt2-small": I.shape_set("gpt2-small")}
for name, shapes in CASES.items():
    xs = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    outs = [torch.empty_like(x) for x in xs]
    pc = PreparedCall(xs, outs, iters=4)
    res = {"case": name}
    for label, f in (("list_api", lambda: ns.orthogonalize_list(xs, out=outs, iters=4)), ("prepared", pc)):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(8):
                f()
            best = min(best, (time.perf_counter() - t0) / 8 * 1e6)
        res[label + "_host_us"] = round(best, 1)
    torch.cuda.synchronize()
    print(json.dumps(res), flush=True)

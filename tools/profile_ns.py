"""Small driver for ncu captures: `calls` Turbo-Muon calls on one synthetic workload.

    python tools/profile_ns.py --workload square8192 --calls 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="square8192")
ap.add_argument("--calls", type=int, default=2)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--precond", default="aol")
a = ap.parse_args()
shapes = I.shape_set(a.workload)
xs = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
outs = [torch.empty_like(t) for t in xs]
for _ in range(a.calls):
    ns.orthogonalize_list(xs, out=outs, iters=a.iters, precond=a.precond)
torch.cuda.synchronize()
print("ok", a.workload, len(shapes), "launches", ns.launch_count())

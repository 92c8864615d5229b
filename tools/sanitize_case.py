"""Small cases for compute-sanitizer: ragged shapes through every launch mode.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402

shapes = [(216, 64), (64, 576), (520, 136), (256, 256), (100, 37)]
for path in (0, 3, 1):
    ns.set_path(path)
    ts = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    ns.orthogonalize_list(ts, iters=4)
    ns.orthogonalize_list(ts[:2], iters=5, precond="frobenius")
    torch.cuda.synchronize()
ns.set_path(0)
x = torch.from_numpy(I.gaussian(128, 128, seed=9, bf16=False)).cuda()
ns.orthogonalize(x, iters=4)
torch.cuda.synchronize()
print("flags", ns.read_flags(), "ok")

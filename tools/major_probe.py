"""Gram / A^2 / update kernel time for tall vs wide inputs of the same shape (measurement only):
tall X (m >= n) feeds the Gram MN-major operands, wide X (m < n) K-major ones."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402

for name, shape, cnt in (("tall 4096x1024", (4096, 1024), 48), ("wide 1024x4096", (1024, 4096), 48),
                         ("tall 8192x2048", (8192, 2048), 8), ("wide 2048x8192", (2048, 8192), 8)):
    xs = [torch.randn(*shape, device="cuda").bfloat16() for _ in range(cnt)]
    outs = [torch.empty_like(x) for x in xs]
    for _ in range(3):
        ns.orthogonalize_list(xs, out=outs, iters=4)
    torch.cuda.synchronize()
    ns.profile_enable(True)
    for _ in range(10):
        ns.orthogonalize_list(xs, out=outs, iters=4)
    p = ns.profile_read()
    ns.profile_enable(False)
    print(name, {k: round(v[0] / 10, 4) for k, v in p.items() if v[1]}, flush=True)

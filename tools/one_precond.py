"""One 8192^2 AOL call after a warm-up (ncu target for the preconditioner launch)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
x = torch.randn(n, n, device="cuda").bfloat16()
ns.orthogonalize(x, iters=4)
ns.orthogonalize(x, iters=4)
torch.cuda.synchronize()

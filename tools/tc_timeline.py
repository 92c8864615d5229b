"""TNS_DBG=4096: per-phase cycle stamps of the tcgen05 cluster kernel (CTA 0), one call."""
import os
import sys

os.environ["TNS_DBG"] = "4096"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402

ns.set_path(7)  # every eligible matrix on the tcgen05 cluster kernel

for m, n in ((256, 2304), (2304, 256), (256, 576), (768, 256), (1024, 128)):
    x = torch.randn(m, n, device="cuda").bfloat16()
    for _ in range(3):
        ns.orthogonalize(x, iters=4)
    torch.cuda.synchronize()
    print(m, n, flush=True)

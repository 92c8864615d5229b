"""e2e (pinned host in -> NS -> pinned host out) time of orthogonalize_host vs bucket count.

    python tools/e2e_buckets.py 6 12 24
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_04632_b200.parallel import orthogonalize_host  # noqa: E402
from synth import inputs as I  # noqa: E402

shapes = I.shape_set("gpt2-medium")
host = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).pin_memory() for i, (m, n) in enumerate(shapes)]
for nb in [int(v) for v in sys.argv[1:]] or [6]:
    for _ in range(2):
        orthogonalize_host(host, iters=4, buckets=nb)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        orthogonalize_host(host, iters=4, buckets=nb)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    print(f"buckets {nb}: median {ts[2]:.2f} ms (min {ts[0]:.2f})", flush=True)

"""Preconditioner launch time and bandwidth on actual bytes (bench.precond_bytes) for the
8192^2 and GPT-2 workloads (per-launch CUDA events, mean over 20 calls)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_04632_b200 as ns  # noqa: E402
from synth import inputs as I  # noqa: E402

peaks = bench.load_peaks()
for name, shapes in (("8192sq", [(8192, 8192)]), ("gpt2-medium", I.shape_set("gpt2-medium")),
                     ("gpt2-small", I.shape_set("gpt2-small"))):
    xs = [torch.randn(m, n, device="cuda").bfloat16() for m, n in shapes]
    for _ in range(3):
        ns.orthogonalize_list(xs, iters=4)
    torch.cuda.synchronize()
    ns.profile_enable(True)
    for _ in range(20):
        ns.orthogonalize_list(xs, iters=4)
    prof = ns.profile_read()
    ns.profile_enable(False)
    ms = prof["precondition"][0] / prof["precondition"][1]
    by = sum(bench.precond_bytes(min(m, n)) for m, n in shapes)
    gbs = by / (ms * 1e-3) / 1e9
    print(f"{name}: precondition {ms * 1e3:.1f} us, {by / 1e6:.1f} MB actual -> {gbs:.0f} GB/s = "
          f"{gbs / peaks['hbm']:.3f} of HBM", flush=True)
    del xs
    torch.cuda.empty_cache()

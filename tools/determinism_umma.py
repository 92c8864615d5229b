"""Repeated grouped calls through the step engine (and its opt-in paths): count distinct
output bit patterns per matrix set (race detector for the tcgen05 engine).

    python tools/determinism_umma.py
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import coeffs as C  # noqa: E402
from synth import inputs as I  # noqa: E402

TALL = [(256, 8192), (2304, 256), (128, 8192)]  # split-K Gram + 128-wide tiles
for name, reps in (("gpt2-small", 30), ("cifar", 50), ("square2048", 30), ("tall", 40)):
    shapes = TALL if name == "tall" else I.shape_set(name)
    xs = [torch.from_numpy(I.gaussian(m, n, seed=i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    for path in (0, 3, 4, 6):
        for pc, cf in (("aol", C.turbo(4)), ("frobenius", C.muon_plus(5))):
            ns.set_path(path)
            outs = [torch.empty_like(x) for x in xs]
            seen = set()
            for _ in range(reps):
                ns.orthogonalize_list(xs, out=outs, iters=len(cf), precond=pc, coeffs=cf)
                h = hashlib.sha1()
                for o in outs:
                    h.update(o.view(torch.int16).cpu().numpy().tobytes())
                seen.add(h.hexdigest())
            print(name, "path", path, pc, "distinct", len(seen), flush=True)
ns.set_path(0)

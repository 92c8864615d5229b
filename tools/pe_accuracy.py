"""relF vs the fp64 oracle of Polar-Express schedules t = 1..9 on the tcgen05 path (a_k I
folded into B') and on the CUDA-core path (a_k X applied in the fp32 epilogue): does the
fold move the bf16 error?  1024 x 768 Gaussian, AOL and Frobenius."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from oracle import ns_oracle as O  # noqa: E402
from synth import inputs as I  # noqa: E402
from synth import polar_express as PE  # noqa: E402

for t in range(1, 10):
    cf = [tuple(map(float, c)) for c in PE.polar_express(t)]
    x = I.gaussian(1024, 768, seed=I.matrix_seed(14, t))
    row = [f"t={t} a1={cf[0][0]:.2f}"]
    for precond in ("aol", "frobenius"):
        ref = O.newton_schulz(x.astype(np.float64), cf, precond)
        for path in (0, 1):
            old = ns.set_path(path)
            g = torch.from_numpy(x).to(torch.bfloat16).cuda()
            ns.orthogonalize(g, iters=t, precond=precond, coeffs=cf)
            torch.cuda.synchronize()
            ns.set_path(old)
            out = g.float().cpu().numpy().astype(np.float64)
            row.append(f"{precond}/{'tc' if path == 0 else 'simt'} {np.linalg.norm(out - ref) / np.linalg.norm(ref):.4f}")
    print("  ".join(row), flush=True)

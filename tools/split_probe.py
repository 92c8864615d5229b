"""Parity numbers of one shape with and without the split-K Gram (TNS_NOSPLIT)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import coeffs as C  # noqa: E402
from synth import inputs as I  # noqa: E402
from tests.helpers import oracle_run, polar_excess, relF  # noqa: E402

m, n, precond = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
x = I.gaussian(m, n, seed=m + 3 * n)
coeffs = C.turbo(4) if precond == "aol" else C.muon_plus(5)
ref = oracle_run(x, coeffs, precond)
for v in ("0", "1"):
    os.environ["TNS_NOSPLIT"] = v
    ns.shutdown()
    t = torch.from_numpy(x).to(torch.bfloat16).cuda()
    ns.orthogonalize(t, iters=len(coeffs), precond=precond, coeffs=coeffs)
    out = t.float().cpu().numpy().astype(np.float64)
    eg, eo = polar_excess(out, ref, x)
    print(f"NOSPLIT={v} relF {relF(out, ref):.5f} polar gpu {eg:.5f} oracle {eo:.5f} ratio {eg / eo:.4f}")

"""Repeat small cluster-kernel calls and count distinct output bit patterns (race detector).

    python tools/determinism_probe.py
"""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2512_04632_b200 as ns
from synth import inputs as I, coeffs as C
for (m, n, dt, pc, cf) in [(128, 128, torch.bfloat16, "frobenius", C.muon_plus(5)), (128, 128, torch.bfloat16, "frobenius", C.turbo(4)),
                            (128, 128, torch.bfloat16, "aol", C.muon_plus(5)), (128, 128, torch.bfloat16, "none", C.muon_plus(5)),
                            (128, 128, torch.bfloat16, "frobenius", C.muon_plus(2)), (128, 128, torch.float32, "frobenius", C.muon_plus(5)),
                            (64, 216, torch.bfloat16, "frobenius", C.muon_plus(5)), (128, 128, torch.bfloat16, "aol", C.turbo(4)),
                            (632, 64, torch.bfloat16, "aol", C.turbo(4)), (100, 37, torch.bfloat16, "frobenius", C.muon_plus(5))]:
    x = I.gaussian(m, n, seed=3, bf16=(dt == torch.bfloat16))
    if pc == "none": x = x / np.float32(40)
    outs = set()
    xt = torch.from_numpy(x).to(dt).cuda()
    for rep in range(300):
        o = torch.empty_like(xt)
        ns.orthogonalize_list([xt], out=[o], iters=len(cf), precond=pc, coeffs=cf)
        torch.cuda.synchronize()
        outs.add(o.float().cpu().numpy().tobytes())
    print(m, n, dt, pc, len(cf), "distinct", len(outs), flush=True)

"""Randomized soak test (measurement / validation only): random shape lists through every
execution path, each matrix against the fp64 oracle (relF gate) and each grouped call bitwise
against single calls where routing is shape-only; repeated calls bitwise equal (races).

    python tools/soak.py --seed 1 --cases 200
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import coeffs as C  # noqa: E402
from synth import inputs as I  # noqa: E402
from tests.helpers import oracle_run, relF  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--cases", type=int, default=200)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
DIMS = [1, 8, 16, 32, 48, 64, 96, 128, 136, 192, 200, 256, 320, 512, 576, 768, 1024, 1152, 2304, 3072]
fails = 0
for case in range(a.cases):
    cnt = int(rng.integers(1, 6))
    shapes = [(int(rng.choice(DIMS)), int(rng.choice(DIMS))) for _ in range(cnt)]
    u = rng.random()
    dtype = torch.bfloat16 if u < 0.7 else torch.float32
    cast = 0.7 <= u < 0.85  # fp32 matrices, bf16 compute (ns_orthogonalize_cast)
    precond = ["aol", "frobenius", "none"][int(rng.integers(0, 3))]
    iters = int(rng.integers(1, 6))
    coeffs = C.turbo(iters) if precond == "aol" else C.muon_plus(iters)
    path = int(rng.choice([0, 4, 5, 7]))
    xs_np = []
    for i, (m, n) in enumerate(shapes):
        x = I.gaussian(m, n, seed=int(rng.integers(0, 1 << 30)), bf16=dtype == torch.bfloat16 or cast)
        if precond == "none":
            x = (x / np.float32(4 * np.sqrt(max(m, n)))).astype(np.float32)
            if dtype == torch.bfloat16 or cast:  # cast: bf16-exact values, so the oracle sees the GPU's input
                x = I.round_bf16(x)
        xs_np.append(x)
    old = ns.set_path(path)
    try:
        xs = [torch.from_numpy(x).to(dtype).cuda() for x in xs_np]
        grouped = [torch.empty_like(x) for x in xs]
        kw = dict(iters=iters, precond=precond, coeffs=coeffs, compute=torch.bfloat16 if cast else None)
        ns.orthogonalize_list(xs, out=grouped, **kw)
        again = [torch.empty_like(x) for x in xs]
        ns.orthogonalize_list(xs, out=again, **kw)  # graph replay
        singles = []
        for x in xs:
            o = torch.empty_like(x)
            ns.orthogonalize_list([x], out=[o], **kw)
            singles.append(o)
        torch.cuda.synchronize()
        flags = ns.read_flags()
    finally:
        ns.set_path(old)
    tol = 2e-2 if (dtype == torch.bfloat16 or cast) else 1e-4
    for i, (x, g, r, s1) in enumerate(zip(xs_np, grouped, again, singles)):
        msg = f"case {case} path {path} {dtype}{' cast' if cast else ''} {precond} T={iters} {shapes[i]} in {shapes}"
        if not torch.equal(g, r):
            print("REPEAT MISMATCH", msg, flush=True)
            fails += 1
        if path in (0, 5, 7) and not torch.equal(g, s1):
            print("BATCH MISMATCH", msg, flush=True)
            fails += 1
        if min(x.shape) <= 1:
            continue
        got = g.float().cpu().numpy().astype(np.float64)
        if not np.all(np.isfinite(got)):
            print("NONFINITE", msg, "flags", flags, flush=True)
            fails += 1
            continue
        ref = oracle_run(x, coeffs, precond)
        e = relF(got, ref)
        if e > tol:
            print(f"RELF {e:.3e} > {tol}", msg, flush=True)
            fails += 1
    if case % 50 == 49:
        print(f"{case + 1} cases, {fails} failures", flush=True)
print(f"done: {a.cases} cases, {fails} failures")

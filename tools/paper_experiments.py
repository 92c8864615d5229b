"""Reproduce the shape of the paper's accuracy/runtime figures on B200 with this library.

  * Fig. 1 / App. C: polar error vs time, Muon (constant triple, T=5,
    Frobenius), Muon+ (T=5, Frobenius), Turbo-Muon (AOL, T=4 and T=5), square n x n;
  * Fig. 3a: polar error vs number of iterations (Muon+ and Turbo truncations);
  * Fig. 2: polar error of the preconditioned X1 alone (AOL vs Frobenius);
  * App. B: the same on Levy alpha-stable inputs (alpha = 1, 1.5, 2);
  * --fig4: Fig. 4: eps_bias(AOL), eps_approx(NS_t, AOL) and the total polar
    error of Turbo-Muon vs the unpreconditioned-bias baseline for t = 1..9 with Polar-Express
    schedules recomputed for every t (synth/polar_express.py), and App. D:
    Muon+ / Turbo-Muon with their own schedules vs with Polar-Express ones on Levy inputs.

Times: CUDA events, median of 10 calls on one B200 (our kernels).  Polar errors:
||NS(X) - U V^T||_F / sqrt(n) with U V^T from torch.linalg.svd on the GPU (float64 for
n <= 2048, float32 above) -- an evaluation tool, not part of the product path.

    python tools/paper_experiments.py [--sizes 1024 2048 4096 8192] > profiles/r01_paper_figures.jsonl
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_04632_b200 as ns  # noqa: E402
from synth import coeffs as C  # noqa: E402
from synth import inputs as I  # noqa: E402
from synth import polar_express as PE  # noqa: E402

METHODS = {
    "muon_T5": (C.muon(5), "frobenius"),
    "muon_plus_T5": (C.muon_plus(5), "frobenius"),
    "turbo_T4": (C.turbo(4), "aol"),
    "turbo_T5": (C.turbo(5), "aol"),
}


def polar(x: torch.Tensor) -> torch.Tensor:
    dt = torch.float64 if max(x.shape) <= 2048 else torch.float32
    u, _, vh = torch.linalg.svd(x.to(dt), full_matrices=False)
    return (u @ vh).float()


def perr(y: torch.Tensor, q: torch.Tensor) -> float:
    return float((y.float() - q).norm() / (min(y.shape) ** 0.5))


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def aol64(x: torch.Tensor) -> torch.Tensor:
    """AOL(X) = X diag(s), s_i = (sum_j |X^T X|_ij)^(-1/2) in fp64 (evaluation only)."""
    y = x.double()
    s = (y.T @ y).abs().sum(1).rsqrt()
    return y * s[None, :]


def fig4(a):
    n, nb = a.fig4_n, a.fig4_batch
    xs = [torch.from_numpy(I.gaussian(n, n, seed=I.matrix_seed(12, i))).to(torch.bfloat16).cuda() for i in range(nb)]
    qs = [polar(x) for x in xs]
    q_aol = [polar(aol64(x)) for x in xs]
    bias = statistics.mean(perr(q1, q) for q1, q in zip(q_aol, qs))
    out = [torch.empty_like(x) for x in xs]
    for t in range(1, 10):
        cf = PE.polar_express(t)
        row = {"fig": "fig4", "n": n, "matrices": nb, "iters": t, "eps_bias": round(bias, 4)}
        ns.orthogonalize_list(xs, out=out, iters=t, precond="aol", coeffs=cf)
        row["turbo_pe_eps_approx"] = round(statistics.mean(perr(o, q) for o, q in zip(out, q_aol)), 4)
        row["turbo_pe_eps_polar"] = round(statistics.mean(perr(o, q) for o, q in zip(out, qs)), 4)
        ns.orthogonalize_list(xs, out=out, iters=t, precond="frobenius", coeffs=cf)
        row["frobenius_pe_eps_polar"] = round(statistics.mean(perr(o, q) for o, q in zip(out, qs)), 4)
        print(json.dumps(row), flush=True)
    del xs, qs, q_aol, out
    # App. D ablation: own schedules vs Polar-Express schedules on Levy inputs
    for alpha in (1.0, 1.5, 2.0):
        xs = [torch.from_numpy(I.levy(512, 512, seed=I.matrix_seed(13, i), alpha=alpha)).to(torch.bfloat16).cuda()
              for i in range(a.batch)]
        qs = [polar(x) for x in xs]
        out = [torch.empty_like(x) for x in xs]
        for t in range(1, 6):
            row = {"fig": "appD_pe_ablation", "alpha": alpha, "n": 512, "iters": t}
            for name, cf, pc in (("muon_plus", C.muon_plus(t), "frobenius"), ("muon_plus_pe", PE.polar_express(t), "frobenius"),
                                 ("turbo", C.turbo(t), "aol"), ("turbo_pe", PE.polar_express(t), "aol")):
                ns.orthogonalize_list(xs, out=out, iters=t, precond=pc, coeffs=cf)
                row[name] = round(statistics.mean(perr(o, q) for o, q in zip(out, qs)), 4)
            print(json.dumps(row), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[1024, 2048, 4096, 8192])
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--fig4", action="store_true", help="only Fig. 4 and the App. D Polar-Express ablation")
    ap.add_argument("--fig4-n", type=int, default=512)
    ap.add_argument("--fig4-batch", type=int, default=100)
    a = ap.parse_args()
    if a.fig4:
        fig4(a)
        return
    for n in a.sizes:
        nb = max(1, a.batch if n <= 2048 else a.batch // 2 if n <= 4096 else 1)
        xs = [torch.from_numpy(I.gaussian(n, n, seed=I.matrix_seed(4, i))).to(torch.bfloat16).cuda() for i in range(nb)]
        qs = [polar(x) for x in xs]
        out = [torch.empty_like(x) for x in xs]
        for name, (cf, pc) in METHODS.items():
            ms = timed(lambda: ns.orthogonalize_list([xs[0]], out=[out[0]], iters=len(cf), precond=pc, coeffs=cf))
            ns.orthogonalize_list(xs, out=out, iters=len(cf), precond=pc, coeffs=cf)
            e = statistics.mean(perr(o, q) for o, q in zip(out, qs))
            print(json.dumps({"fig": "pareto", "n": n, "method": name, "ms": round(ms, 3),
                              "polar_error": round(e, 4), "matrices": nb}), flush=True)
        # Fig. 3a: error vs iterations (truncated schedules)
        for t in range(1, 6):
            for name, cf, pc in (("muon_plus", C.muon_plus(t), "frobenius"), ("turbo", C.turbo(t), "aol")):
                ns.orthogonalize_list(xs, out=out, iters=t, precond=pc, coeffs=cf)
                e = statistics.mean(perr(o, q) for o, q in zip(out, qs))
                print(json.dumps({"fig": "iters", "n": n, "method": name, "iters": t,
                                  "polar_error": round(e, 4)}), flush=True)
        # Fig. 2: X1 alone (AOL vs Frobenius), one NS step with the identity polynomial
        ident = [(1.0, 0.0, 0.0)]
        for pc in ("aol", "frobenius"):
            ns.orthogonalize_list(xs, out=out, iters=1, precond=pc, coeffs=ident)
            e = statistics.mean(perr(o, q) for o, q in zip(out, qs))
            print(json.dumps({"fig": "precond_x1", "n": n, "precond": pc, "polar_error": round(e, 4)}), flush=True)
        del xs, qs, out
        torch.cuda.empty_cache()
    # App. B: Levy alpha-stable, 512 x 512 (the paper stops at 512 because SVD is unstable)
    for alpha in (1.0, 1.5, 2.0):
        xs = [torch.from_numpy(I.levy(512, 512, seed=I.matrix_seed(11, i), alpha=alpha)).to(torch.bfloat16).cuda()
              for i in range(a.batch)]
        qs = [polar(x) for x in xs]
        out = [torch.empty_like(x) for x in xs]
        for name, (cf, pc) in METHODS.items():
            ns.orthogonalize_list(xs, out=out, iters=len(cf), precond=pc, coeffs=cf)
            e = statistics.mean(perr(o, q) for o, q in zip(out, qs))
            print(json.dumps({"fig": "levy", "alpha": alpha, "n": 512, "method": name,
                              "polar_error": round(e, 4)}), flush=True)


if __name__ == "__main__":
    main()

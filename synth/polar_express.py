"""Polar-Express coefficient schedules (DATA for the NS iteration, like synth/coeffs.py).

PAPER.md uses them twice: Fig. 4 ("Since existing methods had coefficients computed
for only five iterations, we recomputed those using the method from [amsel2025polar]") and
App. D ("We recomputed the optimal coefficient for each number of iterations,
using default parameters (l = 10^-3, cushion = 0.024, and safety_factor = 2 x 10^-2)").
The paper prints no values and the construction is the cited external method, so this
module re-derives the tables from its definition (reading R14 in DESIGN.md):

  * step k works on an interval [l_k, u_k] that contains every singular value
    (l_1 = l, u_1 = 1);
  * p_k is the odd quintic p(x) = a x + b x^3 + c x^5 of minimal max |1 - p(x)| on
    [max(l_k, cushion * u_k), u_k] (Remez exchange: the error equioscillates at 4 points);
  * p_k is rescaled so that it is centred on 1 over the true interval:
    p_k <- 2 p_k / (p_k(l_k) + p_k(u_k));
  * next interval: l_{k+1} = p_k(l_k), u_{k+1} = 2 - l_{k+1};
  * safety factor: every polynomial but the last is evaluated at x / (1 + safety)
    (a / (1+s), b / (1+s)^3, c / (1+s)^5), so that round-off cannot push a singular value
    above the interval the next polynomial was designed for.

Pinned in tests/test_polar_express.py by the published default table of the cited method
(8 steps, l = 1e-3, before the safety factor; tests/golden/polar_express_default.json,
transcribed like the Muon+ table, reading R1), reproduced to ~1e-12, and by properties of
the definition (equioscillation, minimality against perturbations, the composed scalar
map's band).
"""
from __future__ import annotations

import numpy as np

CUSHION = 0.02407327424182761  # App. D "cushion = 0.024": the cited default, unrounded
SAFETY = 2e-2        # App. D
L_MIN = 1e-3         # App. D


def quintic(abc, x):
    a, b, c = abc
    x = np.asarray(x, dtype=np.float64)
    return a * x + b * x ** 3 + c * x ** 5


def optimal_quintic(lo: float, hi: float, iters: int = 100, tol: float = 1e-14):
    """argmin over odd quintics of max_{x in [lo, hi]} |1 - p(x)|, by Remez exchange.

    The optimum has 3 free coefficients, so the error 1 - p equioscillates at 4 points
    lo < x1 < x2 < hi with signs (+, -, +, -) (p is below 1 at lo, peaks above 1 at x1,
    dips below at x2, ends above at hi).  p(x) = x q(t), t = x^2, with q written in the
    centred variable tau = (t - t0) / h on [lo^2, hi^2] so that narrow intervals stay
    well conditioned.  For an interval narrower than 1e-4 (relative) the optimum is the
    limit quintic with p(1) = 1, p'(1) = p''(1) = 0, i.e. (15/8, -10/8, 3/8) (the Remez
    optimum there differs from it by < 1e-6 and its error is < 1e-12).
    Returns (a, b, c, E)."""
    if not 0 < lo < hi:
        raise ValueError("need 0 < lo < hi")
    if hi - lo < 1e-4 * hi:  # the optimum's error is < 1e-12 here: below fp64 resolution
        return 15.0 / 8.0, -10.0 / 8.0, 3.0 / 8.0, 0.0
    t0, h = (lo * lo + hi * hi) / 2.0, (hi * hi - lo * lo) / 2.0
    sgn = np.array([1.0, -1.0, 1.0, -1.0])

    def solve(xs):
        M = np.array([[x, x * (x * x - t0) / h, x * ((x * x - t0) / h) ** 2, sg] for x, sg in zip(xs, sgn)])
        return np.linalg.solve(M, np.ones(4))  # alpha, beta, gamma, E

    xs = [lo, np.sqrt(t0 - h / 2), np.sqrt(t0 + h / 2), hi]
    al = be = ga = E = 0.0
    for _ in range(iters):
        al, be, ga, E = solve(xs)
        # p'(x) = q(t) + 2 t q'(t) = [al + 2 be t0/h] + tau [3 be + 4 ga t0/h] + tau^2 [5 ga]
        c0, c1, c2 = al + 2 * be * t0 / h, 3 * be + 4 * ga * t0 / h, 5 * ga
        if abs(c2) < 1e-300:
            taus = [-c0 / c1] if abs(c1) > 1e-300 else []
        else:
            disc = c1 * c1 - 4 * c2 * c0
            taus = [] if disc < 0 else [(-c1 - np.sqrt(disc)) / (2 * c2), (-c1 + np.sqrt(disc)) / (2 * c2)]
        crit = sorted(np.sqrt(t0 + h * tau) for tau in taus if -1.0 < tau < 1.0)
        if len(crit) != 2:
            break
        new = [lo, crit[0], crit[1], hi]
        done = max(abs(p - q) for p, q in zip(new, xs)) <= tol * hi
        xs = new
        if done:
            break
    al, be, ga, E = solve(xs)
    a = al - be * t0 / h + ga * t0 * t0 / (h * h)
    b = be / h - 2.0 * ga * t0 / (h * h)
    c = ga / (h * h)
    return float(a), float(b), float(c), float(abs(E))


def polar_express(iters: int, l: float = L_MIN, cushion: float = CUSHION,
                  safety: float = SAFETY) -> list[tuple[float, float, float]]:
    """The greedy Polar-Express schedule of `iters` quintic steps (see module docstring)."""
    if iters < 1:
        raise ValueError("iters >= 1")
    lo, hi = float(l), 1.0
    raw = []
    for _ in range(iters):
        if hi - lo < 1e-4 * hi:  # interval ~[1, 1]: the limit quintic (error < 1e-12), p(1) = 1
            a, b, c = 15.0 / 8.0, -10.0 / 8.0, 3.0 / 8.0
        else:
            a, b, c, _ = optimal_quintic(max(lo, cushion * hi), hi)
            r = 2.0 / (quintic((a, b, c), lo) + quintic((a, b, c), hi))
            a, b, c = a * r, b * r, c * r
        raw.append((a, b, c))
        lo = min(float(quintic((a, b, c), lo)), 1.0)
        hi = 2.0 - lo
    f = 1.0 + safety
    out = [(a / f, b / f ** 3, c / f ** 5) for (a, b, c) in raw[:-1]] + [raw[-1]]
    return [(float(a), float(b), float(c)) for a, b, c in out]


def scalar_map(schedule, s):
    """The composed scalar map sigma -> p_T(...p_1(sigma)) (Eq. 2 acts per singular value)."""
    s = np.asarray(s, dtype=np.float64)
    for abc in schedule:
        s = quintic(abc, s)
    return s

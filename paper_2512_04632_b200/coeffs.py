"""Default Newton-Schulz coefficient schedules of the product API (data, not arithmetic).

PAPER.md prints no numeric triples (§3; App. D).  Muon+ uses the
"adaptive polynomial factors ... computed for five iterations" of the Dion implementation
(footnote L122); Turbo-Muon "inherit[s] the polynomial factors from Muon+" and keeps
"the n last" triples for fewer iterations.  Values transcribed from the cited
public implementations (reading R1).  The tests check that this table equals the
one in synth/coeffs.py that the oracle tests use.
"""
MUON_PLUS_5 = (
    (4.0848, -6.8946, 2.9270),
    (3.9505, -6.3029, 2.6377),
    (3.7418, -5.5913, 2.3037),
    (2.8769, -3.1427, 1.2046),
    (2.8366, -3.0525, 1.2012),
)
MUON_CONST = (3.4445, -4.7750, 2.0315)


def turbo(iters: int = 4):
    """Last `iters` Muon+ triples (App. D)."""
    if not 1 <= iters <= len(MUON_PLUS_5):
        raise ValueError("Turbo-Muon schedule supports 1..5 iterations; pass coeffs explicitly")
    return list(MUON_PLUS_5[len(MUON_PLUS_5) - iters:])


def muon_plus(iters: int = 5):
    return turbo(iters)


def muon(iters: int = 5):
    return [MUON_CONST] * iters


def polar_express(iters: int, l: float = 1e-3, cushion: float = 0.02407327424182761, safety: float = 2e-2):
    """Polar-Express schedule of `iters` odd quintics (the method PAPER.md cites as
    [amsel2025polar] for its recomputed schedules, Fig. 4 P:L383 and App. D, with the
    defaults stated there): per step the minimax odd quintic approximating 1 on
    [max(l_k, cushion u_k), u_k] (Remez), recentred on 1 over [l_k, u_k]; safety divides the
    input of every polynomial but the last by (1 + safety).  Host-side data generation (the
    same construction as synth/polar_express.py, checked equal by tests/test_abi.py)."""
    import numpy as np

    def quintic(abc, x):
        a, b, c = abc
        return a * x + b * x ** 3 + c * x ** 5

    def optimal(lo, hi):
        if hi - lo < 1e-4 * hi:
            return 15.0 / 8.0, -10.0 / 8.0, 3.0 / 8.0
        t0, h = (lo * lo + hi * hi) / 2.0, (hi * hi - lo * lo) / 2.0
        sgn = (1.0, -1.0, 1.0, -1.0)

        def solve(xs):
            M = np.array([[x, x * (x * x - t0) / h, x * ((x * x - t0) / h) ** 2, sg] for x, sg in zip(xs, sgn)])
            return np.linalg.solve(M, np.ones(4))

        xs = [lo, np.sqrt(t0 - h / 2), np.sqrt(t0 + h / 2), hi]
        for _ in range(100):
            al, be, ga, _ = solve(xs)
            c0, c1, c2 = al + 2 * be * t0 / h, 3 * be + 4 * ga * t0 / h, 5 * ga
            disc = c1 * c1 - 4 * c2 * c0
            if abs(c2) < 1e-300 or disc < 0:
                break
            taus = [(-c1 - np.sqrt(disc)) / (2 * c2), (-c1 + np.sqrt(disc)) / (2 * c2)]
            crit = sorted(np.sqrt(t0 + h * tau) for tau in taus if -1.0 < tau < 1.0)
            if len(crit) != 2:
                break
            new = [lo, crit[0], crit[1], hi]
            done = max(abs(p - q) for p, q in zip(new, xs)) <= 1e-14 * hi
            xs = new
            if done:
                break
        al, be, ga, _ = solve(xs)
        return (al - be * t0 / h + ga * t0 * t0 / (h * h), be / h - 2.0 * ga * t0 / (h * h), ga / (h * h))

    if iters < 1:
        raise ValueError("iters >= 1")
    lo, hi, raw = float(l), 1.0, []
    for _ in range(iters):
        if hi - lo < 1e-4 * hi:
            abc = (15.0 / 8.0, -10.0 / 8.0, 3.0 / 8.0)
        else:
            abc = optimal(max(lo, cushion * hi), hi)
            r = 2.0 / (quintic(abc, lo) + quintic(abc, hi))
            abc = tuple(v * r for v in abc)
        raw.append(abc)
        lo = min(float(quintic(abc, lo)), 1.0)
        hi = 2.0 - lo
    f = 1.0 + safety
    return [(a / f, b / f ** 3, c / f ** 5) for (a, b, c) in raw[:-1]] + [tuple(raw[-1])]

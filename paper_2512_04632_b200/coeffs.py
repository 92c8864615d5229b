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

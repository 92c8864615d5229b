"""Newton-Schulz coefficient schedules, as DATA (inputs to both the oracle and the kernels).

PAPER.md prints no numeric (a, b, c) triples.
It states where they come from:
  * Muon: "the original Newton-Schulz implementation ... with constant
    polynomial factor" -- the public Muon implementation cited in the footnote at L122.
  * Muon+ (PAPER.md L127): "adaptive polynomial factors from [cesista2025muonoptcoeffs],
    computed for five iterations" -- the Dion implementation cited at L122.
  * Turbo-Muon (App. D): "inherit the polynomial factors from Muon+"
    and, for fewer iterations, "retaining only the n last polynomial coefficients".
The values below are transcribed from those public implementations (DESIGN.md
reading R1).  Parity never depends on them: both sides receive the same array.
"""
from __future__ import annotations

# Muon+ / Dion five-step schedule (iteration k uses row k).
MUON_PLUS_5: tuple[tuple[float, float, float], ...] = (
    (4.0848, -6.8946, 2.9270),
    (3.9505, -6.3029, 2.6377),
    (3.7418, -5.5913, 2.3037),
    (2.8769, -3.1427, 1.2046),
    (2.8366, -3.0525, 1.2012),
)

# Original Muon constant triple.
MUON_CONST: tuple[float, float, float] = (3.4445, -4.7750, 2.0315)

# Classical (textbook) quintic Newton-Schulz for the polar factor: p(s) = s(15 - 10 s^2 + 3 s^4)/8.
# It fixes s = 1 with p'(1) = p''(1) = 0 and converges for 0 < s < sqrt(7/3) -- used only
# by the oracle pins (convergence to the SVD polar factor).
CLASSICAL_QUINTIC: tuple[float, float, float] = (15.0 / 8.0, -10.0 / 8.0, 3.0 / 8.0)


def truncate(schedule, keep_last: int) -> list[tuple[float, float, float]]:
    """App. D: keep the n LAST triples, order preserved."""
    schedule = list(schedule)
    if not 1 <= keep_last <= len(schedule):
        raise ValueError(f"keep_last={keep_last} outside [1, {len(schedule)}]")
    return schedule[len(schedule) - keep_last:]


def turbo(iters: int = 4) -> list[tuple[float, float, float]]:
    """Turbo-Muon schedule: last `iters` triples of the Muon+ table (default 4)."""
    return truncate(MUON_PLUS_5, iters)


def muon_plus(iters: int = 5) -> list[tuple[float, float, float]]:
    return truncate(MUON_PLUS_5, iters)


def muon(iters: int = 5) -> list[tuple[float, float, float]]:
    return [MUON_CONST] * iters


def flat(schedule) -> list[float]:
    """[(a1,b1,c1),(a2,...)] -> [a1,b1,c1,a2,...] (the C-ABI coefficient layout)."""
    return [float(v) for t in schedule for v in t]

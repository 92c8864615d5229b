"""Pins for the Polar-Express schedule generator (synth/polar_express.py; reading R14) and
for the Fig. 4 decomposition it feeds (CPU, fp64)."""
import json
import os

import numpy as np
import pytest

from oracle import ns_oracle as O
from synth import inputs as I
from synth import polar_express as PE

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "polar_express_default.json")))


def test_reproduces_published_default_table():
    """The greedy minimax chain with the cited defaults reproduces the published table."""
    got = PE.polar_express(len(GOLD["steps"]), l=GOLD["l"], cushion=GOLD["cushion"], safety=0.0)
    for k, (g, w) in enumerate(zip(got, GOLD["steps"])):
        np.testing.assert_allclose(g, w, rtol=1e-9, atol=1e-9, err_msg=f"step {k + 1}")


@pytest.mark.parametrize("lo,hi", [(1e-3, 1.0), (0.024, 1.0), (0.3, 1.0), (0.9, 1.1), (0.5, 1.5)])
def test_optimal_quintic_equioscillates_and_is_minimal(lo, hi):
    a, b, c, E = PE.optimal_quintic(lo, hi)
    g = np.linspace(lo, hi, 100001)
    err = 1.0 - PE.quintic((a, b, c), g)
    assert abs(np.abs(err).max() - E) <= 1e-9 * max(E, 1e-12) + 1e-15
    # alternation: endpoints carry +E and -E
    assert err[0] == pytest.approx(E, rel=1e-8) and err[-1] == pytest.approx(-E, rel=1e-8)
    # interior local extrema of the error: exactly one minimum (-E, the peak of p) followed
    # by one maximum (+E, the dip)
    i = np.arange(1, len(g) - 1)
    mins = i[(err[i] < err[i - 1]) & (err[i] <= err[i + 1])]
    maxs = i[(err[i] > err[i - 1]) & (err[i] >= err[i + 1])]
    assert len(mins) == 1 and len(maxs) == 1, (mins, maxs)
    assert err[mins[0]] == pytest.approx(-E, rel=1e-6) and err[maxs[0]] == pytest.approx(E, rel=1e-6)
    assert mins[0] < maxs[0]
    # no nearby odd quintic does better (Chebyshev alternation theorem, checked numerically)
    rng = np.random.default_rng(0)
    for _ in range(50):
        d = rng.normal(size=3) * 1e-3 * np.array([abs(a), abs(b), abs(c)])
        assert np.abs(1.0 - PE.quintic((a + d[0], b + d[1], c + d[2]), g)).max() >= E * (1 - 1e-9)


def test_limit_quintic_for_vanishing_interval():
    """As the interval shrinks to {1} the optimum tends to the classical quintic
    (p(1) = 1, p'(1) = p''(1) = 0)."""
    a, b, c, E = PE.optimal_quintic(1 - 1e-3, 1 + 1e-3)
    np.testing.assert_allclose((a, b, c), (15 / 8, -10 / 8, 3 / 8), atol=1e-5)
    assert E < 1e-9


def test_composed_map_band_shrinks():
    """The composed scalar map of the raw chain maps [l, 1] into [1 - E_T, 1 + E_T] with
    E_T strictly decreasing (until fp64 resolution)."""
    g = np.geomspace(1e-3, 1.0, 200001)
    prev = np.inf
    for T in range(1, 8):
        out = PE.scalar_map(PE.polar_express(T, safety=0.0), g)
        e = np.abs(out - 1.0).max()
        assert e < prev or e < 1e-9
        prev = e
    assert prev < 1e-5


def test_safety_factor_structure():
    raw = PE.polar_express(5, safety=0.0)
    saf = PE.polar_express(5, safety=0.02)
    for (a, b, c), (a2, b2, c2) in zip(raw[:-1], saf[:-1]):
        np.testing.assert_allclose((a2, b2, c2), (a / 1.02, b / 1.02 ** 3, c / 1.02 ** 5), rtol=1e-15)
    assert saf[-1] == raw[-1]


def test_fig4_decomposition_properties():
    """Fig. 4 on a small fp64 case: eps_approx(t) of NS_t o AOL with Polar-
    Express schedules falls towards 0 as t grows, eps_bias does not depend on t, and the
    triangle inequality eps_polar <= eps_bias + eps_approx holds at every t."""
    x = I.gaussian(48, 48, seed=3).astype(np.float64)
    q = O.polar_exact(x)
    bias = O.bias_error(x)
    assert 0.0 < bias < 1.0
    prev = np.inf
    for t in range(1, 9):
        sched = PE.polar_express(t)
        ap = O.approx_error(x, sched)
        pol = O.polar_error(O.newton_schulz(x, sched, "aol"), q)
        assert pol <= bias + ap + 1e-12
        assert ap < prev + 1e-12
        prev = ap
    assert prev < 1e-3

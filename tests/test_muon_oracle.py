"""Pins for the Muon-step oracle (CPU)."""
import numpy as np
import pytest

from oracle import muon_oracle as MO
from oracle import ns_oracle as O
from synth import coeffs as C
from synth import inputs as I


def test_beta0_is_plain_orthogonalised_step():
    """beta = 0: M = G, U = G, W1 = W - lr * scale * NS(G)."""
    g = I.gaussian(48, 16, seed=1).astype(np.float64)
    w = I.gaussian(48, 16, seed=2).astype(np.float64)
    W1, M1, Ot = MO.muon_step(w, g, np.zeros_like(g), lr=0.1, beta=0.0, wd=0.0, nesterov=True, coeffs=C.turbo(4))
    np.testing.assert_array_equal(M1, g)
    np.testing.assert_allclose(W1, w - 0.1 * np.sqrt(3.0) * O.newton_schulz(g, C.turbo(4), "aol"), atol=1e-14)


def test_momentum_constant_gradient_closed_form():
    """Constant G: M_t = (1 - beta^t) G (lerp form); nesterov U_t = (1 - beta^(t+1)) G."""
    g = I.gaussian(8, 8, seed=3).astype(np.float64)
    M = np.zeros_like(g)
    beta = 0.9
    for t in range(1, 6):
        M, U = MO.muon_momentum(g, M, beta, nesterov=True)
        np.testing.assert_allclose(M, (1 - beta ** t) * g, atol=1e-14)
        np.testing.assert_allclose(U, (1 - beta ** (t + 1)) * g, atol=1e-14)
    M2, U2 = MO.muon_momentum(g, np.zeros_like(g), beta, nesterov=False)
    np.testing.assert_array_equal(U2, M2)


def test_weight_decay_and_scale():
    w = I.gaussian(64, 16, seed=4).astype(np.float64)
    g = np.zeros_like(w)
    W1, _, Ot = MO.muon_step(w, g, np.zeros_like(w), lr=0.5, beta=0.0, wd=0.2, nesterov=False, coeffs=C.turbo(4))
    np.testing.assert_allclose(W1, w * 0.9, atol=1e-15)  # NS(0) = 0 (reading R4)
    assert MO.muon_scale(64, 16) == 2.0 and MO.muon_scale(16, 64) == 1.0


@pytest.mark.parametrize("shape", [(40, 24), (24, 40)])
def test_update_is_descent_direction(shape):
    """<G, O> > 0 for the orthogonalised update (App. A.1), so -lr*O decreases <G, W>."""
    g = I.gaussian(*shape, seed=5).astype(np.float64)
    _, _, Ot = MO.muon_step(np.zeros(shape), g, np.zeros(shape), lr=1.0, beta=0.0, wd=0.0, nesterov=True,
                            coeffs=C.turbo(4))
    assert float(np.sum(g * Ot)) > 0

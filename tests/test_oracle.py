"""Pins for the fp64 oracle (CPU only).  The oracle is checked against things other
than itself: LAPACK SVD (textbook convergence), closed forms built from an explicit
SVD, hand-computed worked examples (tests/golden/worked_examples.json), invariants
the paper states, and its qualitative claims.

Which plausible mistake each pin catches:
  * dropped c*A^2 or b*A term, wrong sign, wrong coefficient order -> closed-form
    spectral test (test_closed_form_unpreconditioned) and the 1x1/diagonal examples;
  * X B vs B X (transposed operand) -> closed form with U != V on square inputs;
  * AOL row- vs column-scaling, 1/r vs 1/sqrt(r), missing |.| -> worked examples and
    test_aol_orthonormal_columns_exact;
  * Gram reuse wrong (A1 != (X0 s)^T (X0 s)) -> test_gram_reuse_identity and the
    textbook-convergence test (the iteration converges to polar(AOL(X)) only if A1 is
    the Gram of X1);
  * orientation bugs for m < n -> test_transpose_symmetry + wide closed forms.
"""
import json
import os

import numpy as np
import pytest

from oracle import ns_oracle as O
from synth import coeffs as C
from synth import inputs as I

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def scalar_poly_chain(sig, coeffs):
    """p_T o ... o p_1 applied to scalars: p(s) = a s + b s^3 + c s^5 (Eq. 2)."""
    s = np.array(sig, dtype=np.float64)
    for a, b, c in coeffs:
        s = a * s + b * s ** 3 + c * s ** 5
    return s


# ----------------------------------------------------------------- worked examples
def test_worked_aol_scaling():
    for ex in GOLD["aol_scaling"]:
        np.testing.assert_allclose(O.aol_scaling(np.array(ex["a0"])), ex["s"], rtol=0, atol=1e-15)


def test_worked_aol_precondition():
    for ex in GOLD["aol_precondition"]:
        y1, a1 = O.precondition(np.array(ex["x"]), "aol")
        np.testing.assert_allclose(y1, ex["x1"], atol=1e-15)
        np.testing.assert_allclose(a1, np.array(ex["x1"]).T @ np.array(ex["x1"]), atol=1e-14)


def test_worked_rescale_gram():
    for ex in GOLD["rescale_gram"]:
        np.testing.assert_allclose(O.rescale_gram(np.array(ex["a0"]), np.array(ex["s"])), ex["a1"])


def test_worked_ns_step():
    for ex in GOLD["ns_step"]:
        a, b, c = ex["abc"]
        np.testing.assert_allclose(O.ns_step(np.array(ex["x"]), a, b, c), ex["out"], atol=1e-15)


def test_worked_metrics():
    for ex in GOLD["frobenius_scaling"]:
        assert O.frobenius_scaling(np.array(ex["x"])) == pytest.approx(ex["s"], abs=1e-15)
    for ex in GOLD["ortho_error"]:
        assert O.ortho_error(np.array(ex["x"])) == pytest.approx(ex["value"], abs=1e-12)
    for ex in GOLD["polar_error"]:
        assert O.polar_error(np.array(ex["approx"]), np.array(ex["q"])) == pytest.approx(ex["value"])
    ex = GOLD["matmul_count"][0]
    assert O.matmul_count(ex["turbo_iters"]) == ex["turbo"]
    assert O.matmul_count(ex["muon_plus_iters"]) == ex["muon_plus"]
    assert O.matmul_count(4) / O.matmul_count(5) == pytest.approx(ex["ratio"])


def test_coefficient_truncation():
    # App. D: Turbo keeps the n LAST Muon+ triples.
    assert C.turbo(4) == list(C.MUON_PLUS_5[1:])
    assert C.turbo(5) == list(C.MUON_PLUS_5)
    assert C.turbo(1) == [C.MUON_PLUS_5[-1]]
    with pytest.raises(ValueError):
        C.truncate(C.MUON_PLUS_5, 6)


# ----------------------------------------------------------------- textbook / LAPACK
@pytest.mark.parametrize("shape", [(40, 12), (12, 40), (24, 24)])
def test_textbook_convergence_to_svd_polar(shape):
    """Classical quintic x 60 converges to the LAPACK polar factor of the preconditioned
    matrix (pins the iteration mechanics, the Gram reuse and the orientation)."""
    m, n = shape
    x = I.gaussian(m, n, seed=11).astype(np.float64)
    if m == n:  # keep square inputs well conditioned so 60 steps converge to 1e-12
        x = x + 6.0 * np.eye(n)
    sched = [C.CLASSICAL_QUINTIC] * 60
    # Frobenius scaling does not change the polar factor.
    out_f = O.newton_schulz(x, sched, "frobenius")
    np.testing.assert_allclose(out_f, O.polar_exact(x), atol=1e-12)
    # AOL converges to PolarFactor(AOL(X)) = PolarFactor(X diag(s)) (short side).
    y, t = O.orient(x)
    s = O.aol_scaling(y.T @ y)
    q_aol = O.polar_exact(y * s[None, :])
    out_a = O.newton_schulz(x, sched, "aol")
    np.testing.assert_allclose(out_a, q_aol.T if t else q_aol, atol=1e-12)


# ----------------------------------------------------------------- closed forms
@pytest.mark.parametrize("shape", [(30, 30), (50, 20), (20, 50)])
@pytest.mark.parametrize("sched", ["turbo4", "muonplus5", "muon5"])
def test_closed_form_unpreconditioned(shape, sched):
    """X = U diag(sigma) V^T, precond=none: NS_T(X) = U diag(p_T o..o p_1(sigma)) V^T
    (Eq. 2 maps singular values; Eqs. 3-5 preserve singular vectors)."""
    m, n = shape
    k = min(m, n)
    g = np.random.default_rng(3)
    U = np.linalg.qr(g.standard_normal((m, k)))[0]
    V = np.linalg.qr(g.standard_normal((n, k)))[0]
    sig = np.linspace(0.03, 0.9, k)
    x = (U * sig) @ V.T
    coeffs = {"turbo4": C.turbo(4), "muonplus5": C.muon_plus(5), "muon5": C.muon(5)}[sched]
    expect = (U * scalar_poly_chain(sig, coeffs)) @ V.T
    np.testing.assert_allclose(O.newton_schulz(x, coeffs, "none"), expect, atol=2e-14)


@pytest.mark.parametrize("shape", [(64, 16), (16, 64), (32, 32)])
def test_aol_orthonormal_columns_exact(shape):
    """X = Q diag(c) with orthonormal Q: A0 = diag(c^2), s = 1/c, AOL(X) = Q exactly,
    so NS_T(AOL(X)) = P(1) Q with P = p_T o..o p_1 (Eqs. 6-9, Alg. 2)."""
    m, n = shape
    M, N = max(m, n), min(m, n)
    Q = I.orthonormal(M, N, seed=5)
    c = np.linspace(0.2, 7.0, N)
    x = Q * c[None, :]
    if m < n:
        x, Q = x.T, Q.T
    p1 = scalar_poly_chain([1.0], C.turbo(4))[0]
    assert p1 == pytest.approx(0.9941459109, abs=1e-9)  # value of the shipped table at s=1
    np.testing.assert_allclose(O.newton_schulz(x, C.turbo(4), "aol"), p1 * Q, atol=1e-13)
    # Frobenius on the same input does NOT reach Q in 4 steps (conditioning kept).
    assert np.linalg.norm(O.newton_schulz(x, C.turbo(4), "frobenius") - p1 * Q) > 1e-2


def test_aol_constant_rowsum_closed_form():
    """X = Q (alpha I + beta J)^{1/2}: the Gram has constant row sums alpha + n beta, so
    AOL is the scalar 1/sqrt(alpha + n beta) and the output is
    Q V diag(P(sqrt(lambda)/sqrt(alpha+n beta))) V^T."""
    n, m, alpha, beta = 12, 30, 0.7, 0.3
    Q = I.orthonormal(m, n, seed=9)
    G = alpha * np.eye(n) + beta * np.ones((n, n))
    lam, V = np.linalg.eigh(G)
    R = (V * np.sqrt(lam)) @ V.T
    x = Q @ R
    coeffs = C.turbo(4)
    P = scalar_poly_chain(np.sqrt(lam) / np.sqrt(alpha + n * beta), coeffs)
    np.testing.assert_allclose(O.newton_schulz(x, coeffs, "aol"), Q @ ((V * P) @ V.T), atol=1e-13)


def test_rank_one_and_column_vector():
    """n x 1: AOL gives x/||x|| (Gram is the scalar ||x||^2) and output P(1) x/||x||."""
    x = I.gaussian(37, 1, seed=2).astype(np.float64)
    p1 = scalar_poly_chain([1.0], C.turbo(4))[0]
    np.testing.assert_allclose(O.newton_schulz(x, C.turbo(4), "aol"), p1 * x / np.linalg.norm(x), atol=1e-14)
    np.testing.assert_allclose(O.newton_schulz(np.array([[-2.5]]), C.turbo(4), "aol"), [[-p1]], atol=1e-15)


def test_zero_column_reading_R4():
    """Reading R4: a zero column of X gives s_i = 0 and a zero output column, no NaN."""
    x = I.gaussian(20, 6, seed=4).astype(np.float64)
    x[:, 2] = 0.0
    out = O.newton_schulz(x, C.turbo(4), "aol")
    assert np.all(np.isfinite(out)) and np.all(out[:, 2] == 0)
    assert np.all(O.newton_schulz(np.zeros((5, 3)), C.turbo(4), "frobenius") == 0)


# ----------------------------------------------------------------- invariants
@pytest.mark.parametrize("dist", ["gaussian", "levy1.0", "levy1.5", "lowrank", "rank1"])
def test_aol_spectral_bound(dist):
    """||X diag(s)||_2 <= 1 (Gershgorin argument, App. A.3)."""
    for seed in range(5):
        if dist == "rank1":
            g = np.random.default_rng(seed)
            x = np.outer(g.standard_normal(40), g.standard_normal(17))
        else:
            x = I.make_matrix(40, 17, seed, dist).astype(np.float64)
        y1, _ = O.precondition(x, "aol")
        assert np.linalg.norm(y1, 2) <= 1.0 + 1e-12


def test_gram_reuse_identity():
    """diag(s) A0 diag(s) == (X0 diag s)^T (X0 diag s)  (Alg. 2 l.4)."""
    x = I.gaussian(70, 33, seed=8).astype(np.float64)
    y1, a1 = O.precondition(x, "aol")
    np.testing.assert_allclose(a1, y1.T @ y1, rtol=1e-13, atol=1e-15)


def test_scale_invariance_and_transpose_symmetry():
    x = I.gaussian(48, 20, seed=12).astype(np.float64)
    coeffs = C.turbo(4)
    base = O.newton_schulz(x, coeffs, "aol")
    np.testing.assert_allclose(O.newton_schulz(7.3 * x, coeffs, "aol"), base, atol=1e-13)
    np.testing.assert_allclose(O.newton_schulz(x.T, coeffs, "aol"), base.T, atol=0)
    np.testing.assert_allclose(O.newton_schulz(x.T, coeffs, "frobenius"),
                               O.newton_schulz(x, coeffs, "frobenius").T, atol=0)


@pytest.mark.parametrize("dist", ["gaussian", "levy1.0", "lowrank"])
def test_descent_alignment_positive(dist):
    """<G, NS(AOL(G))> > 0 and <G, PolarFactor(G S)> > 0 (Lemma, App. A.1)."""
    for seed in range(6):
        g = I.make_matrix(24, 40, seed, dist).astype(np.float64)
        assert O.descent_alignment(g, O.newton_schulz(g, C.turbo(4), "aol")) > 0
        y, t = O.orient(g)
        s = O.aol_scaling(y.T @ y)
        q = O.polar_exact(y * s[None, :])
        assert O.descent_alignment(y, q) > 0


def test_singular_value_band():
    """When sigma(X1) lies in [lo, hi] the output's singular values lie in
    P([lo, hi]) (Eq. 2 acts per singular value)."""
    x = I.gaussian(1024, 256, seed=21).astype(np.float64)
    y1, _ = O.precondition(x, "aol")
    sv = np.linalg.svd(y1, compute_uv=False)
    grid = np.linspace(sv.min(), sv.max(), 20001)
    P = scalar_poly_chain(grid, C.turbo(4))
    out_sv = np.linalg.svd(O.newton_schulz(x, C.turbo(4), "aol"), compute_uv=False)
    assert out_sv.min() >= P.min() - 1e-9 and out_sv.max() <= P.max() + 1e-9
    assert sv.min() > 0.05 and 0.97 < out_sv.min() and out_sv.max() < 1.04


def test_triangle_inequality_bias_approx():
    """eps_polar <= eps_bias + eps_approx (§6)."""
    x = I.gaussian(64, 64, seed=13).astype(np.float64)
    out = O.newton_schulz(x, C.turbo(4), "aol")
    ep = O.polar_error(out, O.polar_exact(x))
    assert ep <= O.bias_error(x) + O.approx_error(x, C.turbo(4)) + 1e-12


# ----------------------------------------------------------------- paper's qualitative claims
def test_fig2_aol_beats_frobenius_on_x1():
    """Fig. 2: AOL's X1 is closer to the polar factor than Frobenius's."""
    for seed in range(3):
        x = I.gaussian(256, 256, seed=100 + seed).astype(np.float64)
        q = O.polar_exact(x)
        ya, _ = O.precondition(x, "aol")
        yf, _ = O.precondition(x, "frobenius")
        assert O.polar_error(ya, q) < O.polar_error(yf, q)


@pytest.mark.slow
def test_fig3a_turbo4_vs_muonplus5_large():
    """Fig. 3a: Turbo@4 reaches a lower polar error than Muon+@5 for
    large matrices (SPEC acceptance #4 uses a 5% slack)."""
    errs_t, errs_m = [], []
    for seed in range(3):
        x = I.gaussian(1024, 1024, seed=200 + seed).astype(np.float64)
        q = O.polar_exact(x)
        errs_t.append(O.polar_error(O.turbo_muon(x, C.turbo(4)), q))
        errs_m.append(O.polar_error(O.muon_plus(x, C.muon_plus(5)), q))
    assert np.mean(errs_t) <= np.mean(errs_m)


def test_app_b_levy_turbo4_vs_muonplus5():
    """App. B: on Levy alpha=1 inputs Turbo@4 beats Muon+@5."""
    x = I.levy(256, 256, seed=7, alpha=1.0).astype(np.float64)
    q = O.polar_exact(x)
    assert (O.polar_error(O.turbo_muon(x, C.turbo(4)), q)
            < O.polar_error(O.muon_plus(x, C.muon_plus(5)), q))


# ----------------------------------------------------------------- polar factor via the Gram
@pytest.mark.parametrize("shape", [(5, 5), (9, 4), (4, 9), (300, 300), (700, 200)])
def test_polar_exact_gram_equals_svd_route(shape):
    """X (X^T X)^(-1/2) from LAPACK syevd == U V^T from LAPACK gesdd (two different library
    routines for the same definition)."""
    x = I.gaussian(*shape, seed=11, bf16=False).astype(np.float64)
    np.testing.assert_allclose(O.polar_exact_gram(x), O.polar_exact(x), atol=1e-9)


def test_polar_exact_gram_2x2_rotation():
    """Closed form: the polar factor of a 2 x 2 matrix with positive determinant is the
    rotation [[a+d, b-c], [c-b, a+d]] / sqrt((a+d)^2 + (c-b)^2)."""
    a, b, c, d = 1.0, 1.0, 0.0, 1.0
    r = np.hypot(a + d, c - b)
    q = np.array([[a + d, b - c], [c - b, a + d]]) / r
    np.testing.assert_allclose(O.polar_exact_gram(np.array([[a, b], [c, d]])), q, atol=1e-15)
    with pytest.raises(ValueError):
        O.polar_exact_gram(np.array([[1.0, 2.0], [2.0, 4.0]]))


# ----------------------------------------------------------------- eps_bias (§6)
def test_bias_error_hand_computed_2x2():
    """X = [[1, 1], [0, 1]]: A0 = X^T X = [[1, 1], [1, 2]], row sums of |A0| (2, 3), so
    s = (2^-1/2, 3^-1/2) (Eq. 8) and X1 = X diag(s).  Both polar factors are rotations
    (closed form above): Q = R(theta), theta = -atan(1/2); Q_aol = R(phi),
    phi = -atan(3^-1/2 / (2^-1/2 + 3^-1/2)).  ||R(t) - R(p)||_F = 2 sqrt(2) |sin((t - p)/2)|,
    so eps_bias = ||Q - Q_aol||_F / sqrt(2) = 2 |sin((theta - phi) / 2)| = 0.04122...
    A wrong scaling (1/r instead of 1/sqrt(r), rows instead of columns, no |.|) or a wrong
    normalisation (sqrt(n)) changes the value."""
    x = np.array([[1.0, 1.0], [0.0, 1.0]])
    theta = -np.arctan(0.5)
    phi = -np.arctan((1 / np.sqrt(3)) / (1 / np.sqrt(2) + 1 / np.sqrt(3)))
    want = 2 * abs(np.sin((theta - phi) / 2))
    assert want == pytest.approx(0.0412152, abs=1e-6)
    assert O.bias_error(x) == pytest.approx(want, rel=1e-12)


def test_bias_error_exact_zero_cases():
    """AOL changes nothing when s is constant: orthonormal columns (A0 = I, s = 1) and a
    Gram with constant absolute row sums (s = c 1; a scalar does not move the polar
    factor) -- eps_bias = 0 up to rounding; a generic matrix has eps_bias > 0."""
    q = I.orthonormal(40, 12, seed=3)
    assert O.bias_error(q) == pytest.approx(0.0, abs=1e-12)
    # X = Q diag(d) with the columns of Q orthonormal: A0 = diag(d^2); constant row sums iff
    # |d| constant -> take d = 3 (a multiple of an orthonormal frame)
    assert O.bias_error(3.0 * q) == pytest.approx(0.0, abs=1e-12)
    # circulant-like Gram with constant |row| sums: X^T X = [[2, 1], [1, 2]] (row sums 3, 3)
    l = np.linalg.cholesky(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert O.bias_error(l.T) == pytest.approx(0.0, abs=1e-12)
    assert O.bias_error(I.gaussian(30, 10, seed=4, bf16=False).astype(np.float64)) > 1e-3

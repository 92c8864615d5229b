"""fp64 CPU ORACLE for AOL-preconditioned Newton-Schulz (arxiv 2512.04632, "Turbo-Muon").

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import or execute this
module.  The product path (`paper_2512_04632_b200/`) never imports it, and this
module never imports the product path: they share no code.  Inputs come from
`synth/` (input construction only).

Plain, slow, obviously-correct numpy float64, following the paper step by step in
its own order and notation.  Citations are PAPER.md line numbers (P:Lnnn).
No blocking, fusion or reordering beyond what the cited equations state.
Library primitives used as steps: `@` (BLAS dgemm), `numpy.linalg.svd` (LAPACK).

Readings of the paper that this file takes (listed again in DESIGN.md §2):
  R2  non-square inputs: work on the short side; if m < n the iteration runs on X^T
      and the result is transposed back ("all results generalize to the
      non-square case").  Square inputs use X^T X and column scaling
      (the paper's literal form, Eq. 6, "applied column-wise" P:L198).
  R3  "A1 = s^T A0 s" (Alg. 2 l.4) is diag(s) A0 diag(s) elementwise
      ("elementwise multiplication"); "X1 = X0 s" is X0 diag(s).
  R4  a zero row-sum of A0 (zero column of X) gives s_i = 0 (no epsilon, Eq. 7
      has none); a zero matrix under Frobenius scaling is returned unchanged.
  R10 polar error of an m x n matrix is normalised by sqrt(min(m, n)) (P:L92 uses
      sqrt(n) for square).

Parity pins: every function here is pinned by `tests/test_oracle.py` against closed
forms, LAPACK, worked examples or invariants (see that file's docstring); no
function is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "orient", "unorient", "gram", "aol_scaling", "frobenius_scaling", "rescale_gram",
    "precondition", "ns_step", "newton_schulz", "muon", "muon_plus", "turbo_muon",
    "polar_exact", "polar_exact_gram", "polar_error", "ortho_error", "descent_alignment",
    "bias_error", "approx_error", "matmul_count",
]

PRECONDS = ("none", "frobenius", "aol")


def _f64(x) -> np.ndarray:
    return np.array(x, dtype=np.float64, copy=True)


# --------------------------------------------------------------------------- orientation
def orient(x: np.ndarray) -> tuple[np.ndarray, bool]:
    """Reading R2: return (Y, transposed) with Y of shape (M, N), N = min(m, n)."""
    x = _f64(x)
    if x.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    if x.shape[0] >= x.shape[1]:
        return x, False
    return x.T.copy(), True


def unorient(y: np.ndarray, transposed: bool) -> np.ndarray:
    return y.T.copy() if transposed else y


# --------------------------------------------------------------------------- Eq. 3 / Eq. 7
def gram(y: np.ndarray) -> np.ndarray:
    """A = Y^T Y  (Eq. 3; Eq. 7 'matmul' P:L205)."""
    return y.T @ y


def aol_scaling(a0: np.ndarray) -> np.ndarray:
    """s_i = 1 / sqrt(sum_j |A0_ij|)  (Eq. 8; Alg. 2 l.2).

    Reading R4: s_i = 0 where the row sum is exactly 0.
    """
    r = np.abs(a0).sum(axis=1)
    s = np.zeros_like(r)
    pos = r > 0
    s[pos] = 1.0 / np.sqrt(r[pos])
    return s


def frobenius_scaling(y: np.ndarray) -> float:
    """s = 1 / sqrt(sum_ij Y_ij^2) = 1/||Y||_F  (Eq. 10; Alg. 1 l.1).

    Reading R4: 0 for the zero matrix.
    """
    f = np.sqrt(np.sum(y * y))
    return 0.0 if f == 0 else 1.0 / f


def rescale_gram(a0: np.ndarray, s: np.ndarray) -> np.ndarray:
    """A1 = s^T A0 s read as A1_ij = s_i A0_ij s_j  (Alg. 2 l.4; R3)."""
    return s[:, None] * a0 * s[None, :]


# --------------------------------------------------------------------------- preconditioners
def precondition(y: np.ndarray, precond: str):
    """Return (Y1, A1) where A1 is the cached Gram of Y1 for AOL (Alg. 2), else None.

    aol       : A0 = Y0^T Y0 (Eq. 7); s (Eq. 8); Y1 = Y0 diag(s) (Eq. 9);
                A1 = diag(s) A0 diag(s) (Alg. 2 l.4) -- no second matmul.
    frobenius : s = 1/||Y0||_F (Eq. 10); Y1 = Y0 s (Eq. 11).  No cached Gram: Alg. 1
                l.3 recomputes A1 = Y1^T Y1.
    none      : Y1 = Y0 (caller guarantees ||Y0||_2 <= 1).
    """
    if precond == "aol":
        a0 = gram(y)                       # Eq. 7
        s = aol_scaling(a0)                # Eq. 8
        y1 = y * s[None, :]                # Eq. 9, X1 = X0 s (column-wise)
        a1 = rescale_gram(a0, s)           # Alg. 2 l.4
        return y1, a1
    if precond == "frobenius":
        s = frobenius_scaling(y)           # Eq. 10
        return y * s, None                 # Eq. 11
    if precond == "none":
        return y.copy(), None
    raise ValueError(f"precond must be one of {PRECONDS}")


# --------------------------------------------------------------------------- Eqs. 3-5
def ns_step(y: np.ndarray, a: float, b: float, c: float, gram_in: np.ndarray | None = None):
    """One quintic Newton-Schulz step in the paper's three-step form:

        A_k = X_k^T X_k            (Eq. 3)   -- or the cached Gram (Alg. 2)
        B_k = b A_k + c A_k A_k    (Eq. 4)
        X_{k+1} = a X_k + X_k B_k  (Eq. 5)
    """
    A = gram(y) if gram_in is None else gram_in
    B = b * A + c * (A @ A)
    return a * y + y @ B


def newton_schulz(x: np.ndarray, coeffs, precond: str = "aol") -> np.ndarray:
    """NS_T(precond(X)) for T = len(coeffs) triples (a_k, b_k, c_k), k = 1..T.

    Alg. 1 for 'frobenius' / 'none', Alg. 2 for 'aol':
    the AOL Gram is reused as iteration 1's A (Alg. 2 l.4-6); "Next iteration of NS
    (no rescaling)" (Alg. 1/2 last line) for k >= 2.
    """
    coeffs = [tuple(map(float, t)) for t in coeffs]
    if len(coeffs) < 1:
        raise ValueError("need at least one (a, b, c) triple")
    y, transposed = orient(x)
    y, a_cached = precondition(y, precond)
    for k, (a, b, c) in enumerate(coeffs):
        y = ns_step(y, a, b, c, gram_in=a_cached if k == 0 else None)
    return unorient(y, transposed)


def muon(x, coeffs):
    """Muon / Muon+ (Frobenius preconditioning, Alg. 1)."""
    return newton_schulz(x, coeffs, "frobenius")


muon_plus = muon


def turbo_muon(x, coeffs):
    """Turbo-Muon (AOL preconditioning with Gram reuse, Alg. 2)."""
    return newton_schulz(x, coeffs, "aol")


def matmul_count(iters: int) -> int:
    """Matrix products per call: 3 per iteration for every pipeline (Eqs. 3-5); for
    AOL the preconditioner's matmul is absorbed into iteration 1."""
    return 3 * int(iters)


# --------------------------------------------------------------------------- metrics (§3, §6)
def polar_exact(x: np.ndarray) -> np.ndarray:
    """PolarFactor(X) = U V^T from the (thin) SVD X = U Sigma V^T."""
    u, _, vt = np.linalg.svd(_f64(x), full_matrices=False)
    return u @ vt


def polar_exact_gram(x: np.ndarray) -> np.ndarray:
    """PolarFactor(X) = X (X^T X)^(-1/2) for X of full rank (X = Q P with P the
    symmetric PSD square root of X^T X), on the short side (R2), through the symmetric
    eigendecomposition X^T X = V diag(w) V^T (LAPACK syevd): the same factor as U V^T of
    polar_exact at about a third of an SVD's cost -- for the full-size (8192^2) GPU tests.
    Raises for a rank-deficient X (w_min <= 0), where the factor is not unique."""
    y, t = orient(x)
    w, v = np.linalg.eigh(y.T @ y)
    if w.min() <= 0:
        raise ValueError("rank-deficient matrix: the polar factor is not unique")
    q = y @ ((v / np.sqrt(w)[None, :]) @ v.T)
    return unorient(q, t)


def polar_error(approx: np.ndarray, q: np.ndarray) -> float:
    """||NS_t(X) - Q||_F / sqrt(n); sqrt(min(m, n)) for rectangular (R10)."""
    approx = _f64(approx)
    n = min(approx.shape)
    return float(np.linalg.norm(approx - _f64(q)) / np.sqrt(n))


def ortho_error(x: np.ndarray) -> float:
    """||X^T X - I||_F, on the short side."""
    y, _ = orient(x)
    return float(np.linalg.norm(y.T @ y - np.eye(y.shape[1])))


def descent_alignment(g: np.ndarray, update: np.ndarray) -> float:
    """<G, update>_F = tr(G^T update)  (App. A.1 lemma)."""
    return float(np.sum(_f64(g) * _f64(update)))


def bias_error(x: np.ndarray) -> float:
    """eps_bias = ||Q - Q_aol||_F / sqrt(n), Q_aol = PolarFactor(AOL(X))  (§6)."""
    y, t = orient(x)
    y1, _ = precondition(y, "aol")
    return polar_error(polar_exact(y), polar_exact(y1))


def approx_error(x: np.ndarray, coeffs) -> float:
    """eps_approx = ||Q_aol - NS_t(AOL(X))||_F / sqrt(n)  (§6)."""
    y, t = orient(x)
    y1, _ = precondition(y, "aol")
    out, _ = orient(newton_schulz(x, coeffs, "aol"))
    return polar_error(out, polar_exact(y1))

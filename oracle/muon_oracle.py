"""fp64 CPU ORACLE for one Muon / Turbo-Muon optimizer step (TEST INFRASTRUCTURE ONLY; same
rules as ns_oracle.py: only tests/, smoke() and bench.py's CPU legs may use it).

The paper uses Muon as a drop-in: "momentum -> orthogonalize -> update" with the NS step
replaced.  It does not print the momentum / scaling formulas; reading
R13 takes those of the public Muon implementation the paper cites (footnote
P:L122):
    M_t = beta M_{t-1} + (1 - beta) G_t                       (momentum, "lerp" form)
    U_t = (1 - beta) G_t + beta M_t   if nesterov else M_t
    O_t = NS_T(precond(U_t))                                 (this paper: AOL, T = 4)
    W_t = W_{t-1} (1 - lr wd) - lr * max(1, m/n)^(1/2) * O_t  (m x n weight)
Pinned in tests/test_muon_oracle.py (closed forms for beta = 0, constant gradients, and
weight decay alone).
"""
from __future__ import annotations

import numpy as np

from .ns_oracle import newton_schulz


def muon_momentum(G, M, beta: float, nesterov: bool = True):
    G = np.asarray(G, dtype=np.float64)
    M1 = beta * np.asarray(M, dtype=np.float64) + (1.0 - beta) * G
    U = (1.0 - beta) * G + beta * M1 if nesterov else M1
    return M1, U


def muon_scale(m: int, n: int) -> float:
    return max(1.0, m / n) ** 0.5


def muon_step(W, G, M, lr: float, beta: float, wd: float, nesterov: bool, coeffs, precond: str = "aol"):
    """Returns (W_new, M_new, O) in float64."""
    W = np.asarray(W, dtype=np.float64)
    M1, U = muon_momentum(G, M, beta, nesterov)
    O = newton_schulz(U, coeffs, precond)
    W1 = W * (1.0 - lr * wd) - lr * muon_scale(*W.shape) * O
    return W1, M1, O

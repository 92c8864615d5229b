"""Shared test helpers (test side only)."""
from __future__ import annotations

import numpy as np

from oracle import ns_oracle as O


def relF(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def to_np(t) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def oracle_run(x32: np.ndarray, coeffs, precond: str) -> np.ndarray:
    return O.newton_schulz(x32.astype(np.float64), coeffs, precond)


def polar_excess(gpu_out, oracle_out, x) -> tuple[float, float]:
    q = O.polar_exact(np.asarray(x, dtype=np.float64))
    return O.polar_error(gpu_out, q), O.polar_error(oracle_out, q)

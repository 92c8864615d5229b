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


def assert_parity(out, ref, tol: float, what: str = "") -> dict:
    """End-to-end gate of a CUDA result against the fp64 oracle, element by element.

    * global relative Frobenius difference <= tol (BASELINE north_star: 2e-2 bf16, 1e-4 fp32);
    * the same gate per row and per column (lines of >= 64 elements; shorter lines 2 tol), so
      a corrupted strip -- a ragged edge tile, one wrong row block -- cannot hide in the
      global norm;
    * every element: |out - ref| <= tol * rms(ref) * sqrt(2 ln(numel) + 8).  Error model: each
      output element carries the sum of many independent bf16 roundings (stored X, A, B,
      fp32 accumulation), i.e. an approximately Gaussian error of standard deviation
      relF * rms(ref); the gate's relF bound `tol` as that deviation and the Gaussian maximum
      over numel samples (sqrt(2 ln numel), plus margin) bound the worst element.
    Returns the measured values."""
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert out.shape == ref.shape, (out.shape, ref.shape)
    assert np.all(np.isfinite(out)), f"{what}: non-finite output"
    d = out - ref
    g = float(np.linalg.norm(d) / max(np.linalg.norm(ref), 1e-300))
    assert g <= tol, f"{what}: relF {g:.3e} > {tol}"
    res = {"relF": g}
    for axis, name in ((1, "row"), (0, "col")):
        ln = ref.shape[axis]
        rn = np.linalg.norm(ref, axis=axis)
        dn = np.linalg.norm(d, axis=axis)
        ok = rn > 0
        worst = float((dn[ok] / rn[ok]).max()) if ok.any() else 0.0
        lim = tol if ln >= 64 else 2 * tol
        assert worst <= lim, f"{what}: worst {name} relF {worst:.3e} > {lim}"
        assert np.all(dn[~ok] == 0), f"{what}: {name} with zero reference is not zero"
        res[name] = worst
    rms = float(np.sqrt(np.mean(ref * ref)))
    bound = tol * rms * np.sqrt(2 * np.log(max(ref.size, 2)) + 8)
    mx = float(np.abs(d).max())
    assert mx <= bound, f"{what}: max |diff| {mx:.3e} > {bound:.3e}"
    res["max_abs"], res["max_abs_bound"] = mx, float(bound)
    return res

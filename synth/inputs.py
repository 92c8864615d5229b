"""Seeded, synthetic gradient-like matrices with the shapes of the paper's workloads.

Input recipe (stated in DESIGN.md §3):
  * gaussian      -- i.i.d. N(0,1); the paper's main distribution ("sampled from a
                     normal distribution", §4.2 and Fig. 2 caption L135).
  * lowrank_noise -- N(0,1) + U diag(geomspace(snr,1,r)*(sqrt m + sqrt n)) V^T with U, V
                     orthonormal (QR of Gaussians): gradient-like spectrum with a few
                     dominant directions.
  * levy          -- symmetric alpha-stable (beta = 0), the paper's heavy-tailed stress
                     family (App. B, alpha in {1, 1.5, 2}).  Drawn with
                     the Chambers-Mallows-Stuck construction.
Every matrix is rounded to bf16 (round-to-nearest-even) ONCE here, returned as
float32 holding bf16-representable values, so that the CUDA path (bf16 storage)
and the fp64 oracle consume bit-identical inputs.

Nothing in this module computes any step of the method.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "round_bf16", "gaussian", "lowrank_noise", "levy", "orthonormal",
    "make_matrix", "matrix_seed",
    "gpt2_shapes", "cifar_shapes", "square_shapes", "shape_set",
]


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round float values to the nearest bf16 (ties to even); return float32 array.

    bf16 keeps the top 16 bits of an IEEE float32.  Non-finite values pass through.
    """
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    bad = ~np.isfinite(f)
    if bad.any():
        out = out.copy()
        out[bad] = f[bad]
    return out


def _rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(int(seed)))


def gaussian(m: int, n: int, seed: int, bf16: bool = True) -> np.ndarray:
    x = _rng(seed).standard_normal((m, n))
    x = x.astype(np.float32)
    return round_bf16(x) if bf16 else x


def orthonormal(m: int, n: int, seed: int) -> np.ndarray:
    """m x n (m >= n) matrix with orthonormal columns, fp64 (QR of a Gaussian)."""
    assert m >= n
    g = _rng(seed).standard_normal((m, n))
    q, r = np.linalg.qr(g)
    return q * np.sign(np.diag(r))[None, :]


def lowrank_noise(m: int, n: int, seed: int, r: int = 16, snr: float = 10.0,
                  bf16: bool = True) -> np.ndarray:
    g = _rng(seed)
    noise = g.standard_normal((m, n))
    r = min(r, m, n)
    u, _ = np.linalg.qr(g.standard_normal((m, r)))
    v, _ = np.linalg.qr(g.standard_normal((n, r)))
    sig = np.geomspace(snr, 1.0, r) * (np.sqrt(m) + np.sqrt(n))
    x = (noise + (u * sig[None, :]) @ v.T).astype(np.float32)
    return round_bf16(x) if bf16 else x


def levy(m: int, n: int, seed: int, alpha: float = 1.5, beta: float = 0.0,
         bf16: bool = True) -> np.ndarray:
    """Symmetric alpha-stable samples (Chambers-Mallows-Stuck), unit scale.

    Only beta = 0 is used by the paper (App. B: "We set beta=0").
    """
    if beta != 0.0:
        raise ValueError("only beta=0 (symmetric) is supported, as in PAPER.md L654")
    g = _rng(seed)
    v = g.uniform(-np.pi / 2, np.pi / 2, size=(m, n))
    w = g.exponential(1.0, size=(m, n))
    if alpha == 1.0:
        x = np.tan(v)
    else:
        x = (np.sin(alpha * v) / np.cos(v) ** (1.0 / alpha)
             * (np.cos((1.0 - alpha) * v) / w) ** ((1.0 - alpha) / alpha))
    x = x.astype(np.float32)
    return round_bf16(x) if bf16 else x


def make_matrix(m: int, n: int, seed: int, dist: str = "gaussian", bf16: bool = True,
                **kw) -> np.ndarray:
    if dist == "gaussian":
        return gaussian(m, n, seed, bf16=bf16)
    if dist == "lowrank":
        return lowrank_noise(m, n, seed, bf16=bf16, **kw)
    if dist.startswith("levy"):
        alpha = kw.pop("alpha", None)
        if alpha is None:
            alpha = float(dist[4:]) if len(dist) > 4 else 1.5
        return levy(m, n, seed, alpha=alpha, bf16=bf16)
    raise ValueError(f"unknown distribution {dist!r}")


def matrix_seed(config: int, index: int, base: int = 0) -> int:
    """Deterministic per-(config, matrix index) seed."""
    return (base * 1_000_003 + config * 10_007 + index) & 0x7FFFFFFF


# ---------------------------------------------------------------------------
# Workload shape lists (SURVEY.md §8 shape table; BASELINE.json configs)
# ---------------------------------------------------------------------------

def gpt2_shapes(size: str = "small") -> list[tuple[int, int]]:
    """Hidden-matrix Muon parameter set of a GPT-2 model.

    Per layer: q, k, v, o projections (d x d), MLP fc (4d x d stored out x in) and
    MLP proj (d x 4d).  small: d=768, 12 layers (72 matrices); medium: d=1024,
    24 layers (144); large: d=1280, 36 layers (216).
    """
    d, layers = {"small": (768, 12), "medium": (1024, 24), "large": (1280, 36)}[size]
    shapes: list[tuple[int, int]] = []
    for _ in range(layers):
        shapes += [(d, d)] * 4
        shapes.append((4 * d, d))
        shapes.append((d, 4 * d))
    return shapes


def cifar_shapes() -> list[tuple[int, int]]:
    """CIFAR-10 airbench conv weights reshaped to (out, in*3*3)."""
    return [(64, 216), (64, 576), (256, 576), (256, 2304), (256, 2304), (256, 2304)]


def square_shapes() -> list[int]:
    return [1024, 2048, 4096, 8192]


def shape_set(name: str) -> list[tuple[int, int]]:
    if name in ("gpt2-small", "gpt2_small"):
        return gpt2_shapes("small")
    if name in ("gpt2-medium", "gpt2_medium"):
        return gpt2_shapes("medium")
    if name in ("gpt2-large", "gpt2_large"):
        return gpt2_shapes("large")
    if name == "cifar":
        return cifar_shapes()
    if name.startswith("square"):
        n = int(name[6:])
        return [(n, n)]
    raise ValueError(name)

"""Kaiser-Bessel interpolation kernel and its deapodization (oracle, float64).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The paper names only "a GPU-accelerated NUFFT library" (§III-D, §V);
it fixes no kernel.  The reading adopted (SURVEY.md §8(c) readings #1, #6, #7, #8, DESIGN.md
"Readings"): Kaiser-Bessel kernel of width W on a sigma-times oversampled grid with the Beatty
(2005) shape parameter, open support, phi(0) = 1, and analytic (continuous-FT) deapodization by
default, discrete deapodization selectable.
"""
from __future__ import annotations

import numpy as np


def kb_beta(W: int, sigma: float) -> float:
    """beta = pi * sqrt((W/sigma)^2 (sigma - 1/2)^2 - 0.8)."""
    return float(np.pi * np.sqrt((W / sigma) ** 2 * (sigma - 0.5) ** 2 - 0.8))


def kb_kernel(u, W: int, beta: float) -> np.ndarray:
    """phi(u) = I0(beta sqrt(1 - (2u/W)^2)) / I0(beta) for |u| < W/2, else 0 (open support).

    SURVEY.md §8(c)(ii) step 2; reading #6 (a tap at distance exactly W/2 has weight 0) and #7
    (normalised so phi(0) = 1).
    """
    u = np.asarray(u, dtype=np.float64)
    out = np.zeros_like(u)
    inside = np.abs(u) < W / 2.0
    t = 1.0 - (2.0 * u[inside] / W) ** 2
    out[inside] = np.i0(beta * np.sqrt(t)) / np.i0(beta)
    return out


def kb_deapod_analytic(n, G: int, W: int, beta: float) -> np.ndarray:
    """psi(n) = W sinh(sqrt(beta^2 - (pi W n/G)^2)) / sqrt(beta^2 - (pi W n/G)^2) / I0(beta).

    The continuous Fourier transform of phi at frequency n/G.  When
    the radicand is negative the sinh(z)/z becomes sin(z)/z with z = sqrt(-radicand).
    """
    n = np.asarray(n, dtype=np.float64)
    rad = beta ** 2 - (np.pi * W * n / G) ** 2
    out = np.empty_like(n)
    pos = rad > 0
    z = np.sqrt(rad[pos])
    out[pos] = np.sinh(z) / z
    zn = np.sqrt(-rad[~pos])
    with np.errstate(invalid="ignore", divide="ignore"):
        out[~pos] = np.where(zn > 0, np.sin(zn) / np.where(zn > 0, zn, 1.0), 1.0)
    return W * out / np.i0(beta)


def kb_deapod_discrete(n, G: int, W: int, beta: float) -> np.ndarray:
    """psi_d(n) = sum_{d in Z, |d| < W/2} phi(d) cos(2 pi d n / G).

    The DFT of the sampled kernel; makes on-grid (Cartesian) sampling exact (reading #8, #9).
    """
    n = np.asarray(n, dtype=np.float64)
    dmax = int(np.ceil(W / 2.0))
    d = np.arange(-dmax, dmax + 1, dtype=np.float64)
    w = kb_kernel(d, W, beta)
    return (w[None, :] * np.cos(2 * np.pi * np.outer(n, d) / G)).sum(1).reshape(n.shape)


def deapod(n, G: int, W: int, beta: float, mode: str = "analytic") -> np.ndarray:
    if mode == "analytic":
        return kb_deapod_analytic(n, G, W, beta)
    if mode == "discrete":
        return kb_deapod_discrete(n, G, W, beta)
    raise ValueError(f"unknown deapodization mode {mode!r}")

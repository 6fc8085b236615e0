"""Density compensation: Pipe-Menon iteration (oracle).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).  The density-compensated initialisation
X^0 = A^H (w . b) of Algorithm 1 ("X^0 = A* b", with the optional diagonal
weighting of SPEC.md:315) needs per-sample weights w.  The paper does not say how they are
obtained; reading 23: the Pipe-Menon fixed-point iteration on the same gridding
interpolation matrix Phi (Phi_{j,m} = phi(u_jx - m_x) phi(u_jy - m_y), the taps of the forward
gridding, ``oracle.nufft.taps``):

    w^(0) = 1,   w^(t+1)_j = w^(t)_j / (Phi Phi^T w^(t))_j,

i.e. spread w onto the sigma*N grid (Phi^T) and interpolate back (Phi), written out below with
``numpy.bincount`` and a gather.  The fixed point satisfies Phi Phi^T w = 1.
"""
from __future__ import annotations

import numpy as np

from .nufft import GridParams, taps


def phi_phit(w, k, gp: GridParams) -> np.ndarray:
    """(Phi Phi^T w)_j: spread w to the G x G grid with the gridding taps, then interpolate back."""
    G = gp.G
    mx, my, wx, wy = taps(k, gp)
    flat = ((my % G)[:, :, None] * G + (mx % G)[:, None, :]).reshape(len(k), -1)   # [M][W*W]
    wt = (wy[:, :, None] * wx[:, None, :]).reshape(len(k), -1)                      # [M][W*W]
    grid = np.bincount(flat.ravel(), weights=(wt * np.asarray(w, np.float64)[:, None]).ravel(), minlength=G * G)
    return (wt * grid[flat]).sum(1)


def pipe_menon(k, N: int, W: int, n_iter: int = 20, sigma: float = 2.0) -> np.ndarray:
    """Density-compensation weights [M] of one interleaf k [M][2] after n_iter iterations."""
    gp = GridParams(N, W, sigma)
    w = np.ones(len(k), dtype=np.float64)
    for _ in range(n_iter):
        w = w / phi_phit(w, k, gp)
    return w


def dcf(traj, N: int, W: int, n_iter: int = 20, sigma: float = 2.0) -> np.ndarray:
    """Weights [R][M] for every interleaf of traj [R][M][2]."""
    return np.stack([pipe_menon(traj[r], N, W, n_iter, sigma) for r in range(traj.shape[0])])

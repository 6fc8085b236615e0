"""Float64 oracle of the manifold-structured regularisation of MS-LLR (Eqs. 7-11).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).  SURVEY.md §8(f) f2 (with ``oracle.llr``).

  w_ij = exp(-||Q_i(M) - Q_j(M)||_F^2 / sigma^2),  i != j,  w_ii = 0          (Eq. 8)
  L = D - W,  D_ii = sum_j w_ij                                               (Eqs. 10-11)
  J_MS(X) = Tr(Q(X) L Q(X)^H)                                                 (Eq. 9)
  gradient term of Eq. 15: lambda_1 Q^*(Q(X) L)

Q(X) is the Casorati matrix whose column j is the vectorised patch j (patches as in
``oracle.llr``: p x p, stride s, corners 0, s, ... and N - p, ordered row-major by corner).
Readings (after SPEC.md:387, 415-420): the parameter maps M = (T1, T2, PD) are
standardised per channel (zero mean, unit std) over the foreground PD > 0.1 max PD before the
distances; sigma^2 = the median of the nonzero pairwise squared distances (i < j); the penalty is
the trace form, which equals (1/2) sum over ordered pairs i != j of w_ij ||Q_i - Q_j||^2.
"""
from __future__ import annotations

import numpy as np

from .llr import patch_corners


def patches(N: int, p: int = 11, s: int = 5):
    c = patch_corners(N, p, s)
    return [(y, x) for y in c for x in c]


def casorati_all(X: np.ndarray, P, p: int) -> np.ndarray:
    """Q(X): [C*p*p][n] for X [C][N][N] (channel-major, then row-major inside the patch)."""
    return np.stack([np.asarray(X)[:, y:y + p, x:x + p].reshape(-1) for (y, x) in P], axis=1)


def scatter_adjoint(Qm: np.ndarray, shape, P, p: int) -> np.ndarray:
    """Q^*: sums the columns back onto their patches (overlaps add)."""
    out = np.zeros(shape, dtype=np.result_type(Qm, np.float64))
    C = shape[0]
    for j, (y, x) in enumerate(P):
        out[:, y:y + p, x:x + p] += Qm[:, j].reshape(C, p, p)
    return out


def standardise(maps: np.ndarray) -> np.ndarray:
    """maps [3][N][N] = (T1, T2, PD): per-channel zero mean / unit std over PD > 0.1 max PD."""
    maps = np.asarray(maps, np.float64)
    pd = maps[2]
    fg = pd > 0.1 * pd.max() if pd.max() > 0 else np.ones_like(pd, bool)
    out = np.empty_like(maps)
    for c in range(maps.shape[0]):
        v = maps[c][fg]
        sd = v.std()
        out[c] = (maps[c] - v.mean()) / (sd if sd > 0 else 1.0)
    return out


def weights(maps: np.ndarray, N: int, p: int = 11, s: int = 5, sigma2: float | None = None, raw: bool = False):
    """(W [n][n], sigma^2) from the parameter maps (Eq. 8).  The distances use the standardised
    maps (reading 26); raw=True: the printed form, Euclidean distances of the raw (T1, T2, PD)
    patches."""
    P = patches(N, p, s)
    V = casorati_all(np.asarray(maps, np.float64) if raw else standardise(maps), P, p)   # [3 p^2][n]
    sq = np.sum(V * V, axis=0)
    d2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * (V.T @ V), 0.0)
    n = d2.shape[0]
    iu = np.triu_indices(n, 1)
    nz = d2[iu][d2[iu] > 0]
    if sigma2 is None:
        sigma2 = float(np.median(nz)) if nz.size else 1.0
    W = np.exp(-d2 / sigma2)
    np.fill_diagonal(W, 0.0)
    return W, sigma2


def laplacian(W: np.ndarray) -> np.ndarray:
    return np.diag(W.sum(axis=1)) - W


def penalty(X: np.ndarray, Lap: np.ndarray, N: int, p: int = 11, s: int = 5) -> float:
    Qm = casorati_all(X, patches(N, p, s), p)
    return float(np.real(np.trace(Qm @ Lap @ np.conj(Qm).T)))


def gradient(X: np.ndarray, Lap: np.ndarray, N: int, p: int = 11, s: int = 5) -> np.ndarray:
    """Q^*(Q(X) L) for X [L][N][N] (the manifold term of Eq. 15 without lambda_1)."""
    P = patches(N, p, s)
    return scatter_adjoint(casorati_all(X, P, p) @ Lap, np.shape(X), P, p)

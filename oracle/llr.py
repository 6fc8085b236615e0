"""Float64 oracle of the locally-low-rank (LLR) outer step of Algorithm 1.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).  SURVEY.md §8(f) f2, restricted to the
paper's LLR ablation ("using only locally low-rank constraints", lambda_1 = 0, no
manifold term).  Written from the paper, step by step:

  basis d (Eq. 17): an orthonormal basis of the fingerprint subspace,
      "approximated by the precomputed dictionary D": the leading right singular vectors of D
      keeping a fraction `energy` of ||D||_F^2 (reading 24).
  P_S(X) = X d^dagger d (Eq. 17) on every voxel's time series (rows of d orthonormal).
  Z = P_S(X - mu [A^*(A X - b)])                       (Eq. 15 with lambda_1 = 0)
  P_q = SVT_{1/beta}(Q_q(Z)) = sum max(sigma - 1/beta, 0) u v^H        (Eq. 20)
  X+ = argmin (1/2mu)||X - Z||^2 + (lambda_2 beta / 2) sum_q ||P_q - Q_q(X)||^2
     = (Z + gamma Q^*(P)) / (1 + gamma c),  gamma = mu lambda_2 beta, c(v) = #patches covering v
                                                       (Eq. 21; reading 25: with overlapping
                                                        patches the minimiser divides by 1 + gamma c)
Patches: p x p = 11 x 11 voxels, stride s = 5 (reading 19), top-left corners
0, s, 2s, ... and N - p (so every voxel is covered), no wrap.  Q_q(X) is the p^2 x L Casorati
matrix of a patch (rows = voxels in row-major order inside the patch, columns = frames).
"""
from __future__ import annotations

import numpy as np


def basis(D: np.ndarray, energy: float = 0.9999, max_rank: int = 64) -> np.ndarray:
    """[r][L] orthonormal rows: leading right singular vectors of D [K][L] (complex)."""
    _, s, vh = np.linalg.svd(np.asarray(D, np.complex128), full_matrices=False)
    e = np.cumsum(s ** 2) / np.sum(s ** 2)
    r = min(int(np.searchsorted(e, energy) + 1), max_rank, len(s))
    return vh[:r]


def project(X: np.ndarray, d: np.ndarray) -> np.ndarray:
    """P_S(X) = X d^dagger d for X [L][N][N] frame-major (voxel time series are the columns)."""
    L = X.shape[0]
    Xv = np.asarray(X, np.complex128).reshape(L, -1).T             # [V][L]
    return ((Xv @ np.conj(d).T) @ d).T.reshape(X.shape)


def patch_corners(N: int, p: int = 11, s: int = 5) -> np.ndarray:
    c = list(range(0, N - p + 1, s))
    if c[-1] != N - p:
        c.append(N - p)
    return np.asarray(c)


def casorati(X: np.ndarray, y0: int, x0: int, p: int) -> np.ndarray:
    """Q_q(X): [p*p][L], rows = voxels (y0+i, x0+j) in row-major order."""
    L = X.shape[0]
    return np.asarray(X[:, y0:y0 + p, x0:x0 + p]).reshape(L, p * p).T


def svt(C: np.ndarray, tau: float) -> np.ndarray:
    """Singular value thresholding (Eq. 20): U max(S - tau, 0) V^H."""
    u, s, vh = np.linalg.svd(C, full_matrices=False)
    return (u * np.maximum(s - tau, 0.0)) @ vh


def llr_prox(Z: np.ndarray, tau: float, gamma: float, p: int = 11, s: int = 5, literal: bool = False):
    """Eqs. (20)-(21): P_q = SVT_tau(Q_q(Z)) for all patches, then
    X = (Z + gamma Q^*(P)) / (1 + gamma c) (reading 25: c(v) = number of patches covering v, the
    exact minimiser with overlapping patches).  literal=True: the printed scalar form
    X = (Z + gamma Q^*(P)) / (1 + gamma) of Eq. (23) (exact only when the
    patches do not overlap).  Returns (X, nuclear norm sum of Q_q(Z))."""
    L, N, _ = Z.shape
    acc = np.zeros(Z.shape, dtype=np.complex128)
    cnt = np.zeros((N, N))
    nuc = 0.0
    cs = patch_corners(N, p, s)
    for y0 in cs:
        for x0 in cs:
            C = casorati(Z, y0, x0, p)
            nuc += np.linalg.svd(C, compute_uv=False).sum()
            P = svt(C, tau)
            acc[:, y0:y0 + p, x0:x0 + p] += P.T.reshape(L, p, p)
            cnt[y0:y0 + p, x0:x0 + p] += 1.0
    den = (1.0 + gamma) * np.ones_like(cnt) if literal else (1.0 + gamma * cnt)
    return (np.asarray(Z, np.complex128) + gamma * acc) / den[None], nuc


def llr_step(X, rhs, normal, d, mu: float, lam2: float, beta: float, p: int = 11, s: int = 5,
             lam1: float = 0.0, lap=None, literal: bool = False):
    """One iteration of Algorithm 1: Eq. (15) -> Eq. (20) -> Eq. (21).  normal(v) = A^H A v;
    rhs = A^H b; lam1, lap: the manifold term lam1 Q^*(Q(X) L) of Eq. (15) (``oracle.manifold``),
    omitted when lam1 = 0 (the LLR ablation).  Returns (X+, Z)."""
    G = normal(X) - rhs
    if lam1:
        from .manifold import gradient
        G = G + lam1 * gradient(np.asarray(X, np.complex128), lap, X.shape[1], p, s)
    Z = project(np.asarray(X, np.complex128) - mu * G, d)
    Xn, _ = llr_prox(Z, 1.0 / beta, mu * lam2 * beta, p, s, literal=literal)
    return Xn, Z

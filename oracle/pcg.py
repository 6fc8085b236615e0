"""Preconditioned CG for the data-consistency solve, with a circulant image-space preconditioner
(SURVEY.md §8(f) f4 "preconditioned CG"; float64, oracle).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The system is the one of ``oracle.cg`` -- (A^H A + mu I) x = rhs (BASELINE.json north_star; the
normal operator 𝒜*𝒜 of PAPER.md:217 Eq. (15)).  Preconditioning with any Hermitian positive
definite M leaves its solution unchanged; only the iterates differ.  Textbook PCG:

    r0 = rhs - H x0;  z0 = M^-1 r0;  p0 = z0;  rho0 = <r0, z0>
    for k < n_iter:
        q = H p;  alpha = rho_k / Re<p, q>;  x += alpha p;  r -= alpha q
        if tol > 0 and ||r|| / ||r0|| < tol: stop
        z = M^-1 r;  rho_{k+1} = Re<r, z>;  p = z + (rho_{k+1} / rho_k) p

The preconditioner (reading 28): per frame, M = C + gamma I with C T. Chan's optimal
circulant approximation of that frame's exact normal operator A^H A (the circulant closest in
Frobenius norm).  Its eigenvalues are the Rayleigh quotients of A^H A at the Fourier vectors,

    lambda_m = f_m^H A^H A f_m = ||A f_m||^2,   f_m[n] = exp(+i 2 pi m . n / N) / N,

m and n centred in [-N/2, N/2)^2; with A's rows (1/N) exp(-i 2 pi k_j . n) this is the closed form

    lambda_m = N^-4 sum_j F(kx_j - mx/N) F(ky_j - my/N),   F(t) = sin^2(pi N t) / sin^2(pi t)

(the Fejer kernel, F(0) = N^2).  C >= 0 because every lambda_m is a Rayleigh quotient of a PSD
operator, so M is HPD for gamma > 0.  Applying M^-1 is a 2D DFT, a division, an inverse DFT:
M^-1 v = sum_m f_m (f_m^H v) / (lambda_m + gamma).  With coil maps the circulant of the
single-coil operator is scaled by the mean coil power (1/N^2) sum_n sum_c |S_c[n]|^2 (1 for the
sum-of-squares-normalised maps of the configs) -- a choice of preconditioner, not of solution.
gamma = mu + shift * mean(lambda) (shift = 30 by default: the undersampled spiral leaves most
lambda_m near 0, and dividing those by mu alone would steer the iterates into the null space of A;
measured in DESIGN.md).
"""
from __future__ import annotations

import numpy as np

from .cg import vdot


def fejer(t, N: int):
    """F(t) = |sum_{n=-N/2}^{N/2-1} exp(-i 2 pi t n)|^2 = sin^2(pi N t) / sin^2(pi t), F(integer) = N^2."""
    t = np.asarray(t, dtype=np.float64)
    s = np.sin(np.pi * t)
    small = np.abs(s) < 1e-12
    return np.where(small, float(N) * N, (np.sin(np.pi * N * t) / np.where(small, 1.0, s)) ** 2)


def circulant_eigs(k, N: int) -> np.ndarray:
    """lambda[my + N/2][mx + N/2] = ||A f_m||^2 for the points k [M][2] (kx, ky) of one frame."""
    k = np.asarray(k, dtype=np.float64)
    m = np.arange(N) - N // 2
    Fx = fejer(k[:, 0:1] - m[None, :] / N, N)      # [M][N] over mx
    Fy = fejer(k[:, 1:2] - m[None, :] / N, N)      # [M][N] over my
    return (Fy.T @ Fx) / float(N) ** 4               # one library step: sum over the points j


def shift_gamma(lam: np.ndarray, mu: float, shift: float) -> float:
    """gamma = mu + shift * mean(lambda) over all frames' eigenvalues."""
    return float(mu + shift * np.mean(lam))


def coil_power(coils, N: int) -> float:
    if coils is None:
        return 1.0
    c = np.asarray(coils, dtype=np.complex128)
    return float(np.sum(np.abs(c) ** 2) / (N * N))


def precond_apply(v, lam_frames, gamma: float, scale: float = 1.0) -> np.ndarray:
    """M^-1 v per frame: sum_m f_m (f_m^H v_l) / (scale lambda_l[m] + gamma), v [L][N][N].

    f_m^H v = (1/N) sum_n v[n] exp(-i 2 pi m . n / N) with centred m, n (ifftshift/fftshift put
    index N/2 at position 0); lam_frames [L][N][N] indexed [my + N/2][mx + N/2]."""
    v = np.asarray(v, dtype=np.complex128)
    out = np.empty_like(v)
    for l in range(v.shape[0]):
        c = np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(v[l]), norm="ortho"))   # f_m^H v
        c = c / (scale * lam_frames[l] + gamma)
        out[l] = np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(c), norm="ortho"))  # sum_m f_m c_m
    return out


def pcg(H, Minv, rhs, x0, n_iter: int, tol: float = 0.0, dot=vdot):
    """Returns (x, history) with history[k] = ||r_k|| (the true residual norm), len = iterations + 1."""
    x = np.array(x0, dtype=np.complex128, copy=True)
    r = np.asarray(rhs, dtype=np.complex128) - H(x)
    z = Minv(r)
    p = z.copy()
    rho = dot(r, z).real
    rr0 = dot(r, r).real
    hist = [np.sqrt(rr0)]
    if rr0 == 0.0:
        return x, hist
    for _ in range(n_iter):
        q = H(p)
        pq = dot(p, q).real
        if not pq > 0.0:
            raise FloatingPointError("PCG breakdown: Re<p, Hp> <= 0")
        alpha = rho / pq
        x += alpha * p
        r -= alpha * q
        rr = dot(r, r).real
        hist.append(np.sqrt(rr))
        if tol > 0.0 and np.sqrt(rr / rr0) < tol:
            break
        z = Minv(r)
        rho_new = dot(r, z).real
        p = z + (rho_new / rho) * p
        rho = rho_new
    return x, hist


def preconditioned_krylov_projection(Hmat, Mi_mat, rhs, x0, n: int):
    """n-step PCG iterate as a Galerkin projection: x_n = x0 + V (V^H H V)^{-1} V^H r0 with V an
    orthonormal basis of K_n(M^-1 H, M^-1 r0) (Arnoldi, full re-orthogonalisation).  PCG's n-th
    iterate minimises the H-norm of the error over exactly that space.  Dense, tiny pins only."""
    Hmat = np.asarray(Hmat, dtype=np.complex128)
    Mi_mat = np.asarray(Mi_mat, dtype=np.complex128)
    r0 = np.asarray(rhs, dtype=np.complex128) - Hmat @ x0
    V = np.zeros((len(r0), n), dtype=np.complex128)
    v = Mi_mat @ r0
    for i in range(n):
        v = v / np.linalg.norm(v)
        for _ in range(2):
            v = v - V[:, :i] @ (V[:, :i].conj().T @ v)
        V[:, i] = v / np.linalg.norm(v)
        v = Mi_mat @ (Hmat @ V[:, i])
    T = V.conj().T @ Hmat @ V
    return x0 + V @ np.linalg.solve(T, V.conj().T @ r0)

"""Seeded synthetic workloads (BASELINE.json ``configs``; SURVEY.md §8(d) "Synthetic inputs").

The paper's own data (phantom maps, FA/TR waveforms, dictionary, in-vivo raw k-space,
PAPER.md:314, 384, 429) is not available, so these seeded generators stand in for it, with the
shapes and structure of BASELINE.json's five configs.  Nothing here implements the method: no
Kaiser-Bessel kernel, no FFT, no gridding.  Both the float64 oracle and the CUDA path consume the
arrays returned here (trajectories are produced in float64 and STORED as float32; both sides read
the stored float32 values, SURVEY.md §8(c) reading #10).

Seeding: every stream is ``numpy.random.default_rng([seed, stream, *index])`` so that any frame
subset (a rank's shard) can be generated without generating the others:
    stream 0: i.i.d. Gaussian images, per frame l
    stream 1: ellipse geometry + per-component amplitudes (rank-5 phantoms)
    stream 2: temporal curves u_r(l)
    stream 3: coil phases
    stream 4: measurement noise, per frame l
"""
from __future__ import annotations

import dataclasses
from typing import Iterable, Sequence

import numpy as np

__all__ = [
    "Config", "CONFIGS", "get_config", "spiral_trajectory", "cartesian_trajectory",
    "random_trajectory", "frame_interleaf", "iid_images", "rank5_factors", "rank5_images",
    "images", "coil_maps", "unit_noise", "random_kspace",
]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    N: int            # image side
    L: int            # frames
    M: int            # nonuniform points per frame (one interleaf)
    C: int            # coils (1 => no coil maps, S = 1)
    R: int            # distinct interleaves; frame l uses interleaf l mod R
    W: int            # Kaiser-Bessel width
    sigma: float      # oversampling
    turns: float      # spiral turns
    p: float          # spiral exponent k = 0.5 tau^p e^{i 2 pi turns tau}
    image_kind: str   # "iid" | "rank5"
    noise: float      # relative noise level (0.01 => 1% of RMS |y_clean|)
    mu: float         # Tikhonov shift of the CG solve
    cg_iters: int     # CG iterations of the config's run
    seed: int         # master seed (= config index)

    @property
    def G(self) -> int:
        return int(round(self.sigma * self.N))


# BASELINE.json configs[0..4] (SURVEY.md §8(a) "Sizes at BJ configs", §8(d) table).
CONFIGS = {
    "pr1": Config("pr1", 32, 8, 256, 1, 8, 6, 2.0, 4, 1.5, "iid", 0.0, 0.01, 5, 1),
    "cfg2": Config("cfg2", 128, 200, 1024, 1, 24, 6, 2.0, 16, 1.5, "rank5", 0.0, 0.01, 10, 2),
    "mrf": Config("mrf", 256, 1000, 2048, 1, 48, 6, 2.0, 24, 1.5, "rank5", 0.0, 0.01, 10, 3),
    "sense": Config("sense", 256, 1000, 2048, 8, 48, 6, 2.0, 24, 1.5, "rank5", 0.01, 0.01, 10, 4),
    "stress": Config("stress", 256, 2000, 4096, 16, 96, 8, 2.0, 24, 4.0, "iid", 0.0, 0.01, 10, 5),
}


def get_config(name: str, **overrides) -> Config:
    return dataclasses.replace(CONFIGS[name], **overrides)


# ----------------------------------------------------------------------------- trajectories
def spiral_trajectory(M: int, R: int, turns: float, p: float) -> np.ndarray:
    """Variable-density spiral interleaves, float32 [R][M][2] = (kx, ky) in cycles/pixel.

    k(tau) = 0.5 tau^p exp(i 2 pi turns tau), tau_m = m/(M-1) (BASELINE.json configs[0];
    SURVEY.md §8(c) reading #10), interleaf r rotated by exp(i 2 pi r / R).
    """
    tau = np.arange(M, dtype=np.float64) / max(M - 1, 1)
    k = 0.5 * tau ** p * np.exp(2j * np.pi * turns * tau)
    rot = np.exp(2j * np.pi * np.arange(R, dtype=np.float64) / R)
    kr = rot[:, None] * k[None, :]
    out = np.empty((R, M, 2), dtype=np.float32)
    out[..., 0] = kr.real
    out[..., 1] = kr.imag
    return out


def cartesian_trajectory(N: int) -> np.ndarray:
    """Full Cartesian grid k = (m_x, m_y)/N, m in [-N/2, N/2): float32 [1][N*N][2], x fastest."""
    m = (np.arange(N) - N // 2) / N
    ky, kx = np.meshgrid(m, m, indexing="ij")
    out = np.empty((1, N * N, 2), dtype=np.float32)
    out[0, :, 0] = kx.ravel()
    out[0, :, 1] = ky.ravel()
    return out


def random_trajectory(M: int, R: int, seed: int) -> np.ndarray:
    """Uniform random k in [-0.5, 0.5)^2, float32 [R][M][2]."""
    rng = np.random.default_rng([seed, 7])
    return (rng.random((R, M, 2)) - 0.5).astype(np.float32)


def frame_interleaf(frames: Iterable[int], R: int) -> np.ndarray:
    """Frame l uses interleaf l mod R (BASELINE.json configs[2])."""
    return np.asarray([int(l) % R for l in frames], dtype=np.int32)


# ----------------------------------------------------------------------------- images
def iid_images(N: int, frames: Sequence[int], seed: int) -> np.ndarray:
    """i.i.d. N(0,1) real and imaginary parts, complex64 [len(frames)][N][N]."""
    out = np.empty((len(frames), N, N), dtype=np.complex64)
    for i, l in enumerate(frames):
        rng = np.random.default_rng([seed, 0, int(l)])
        v = rng.standard_normal((2, N, N), dtype=np.float32)
        out[i].real = v[0]
        out[i].imag = v[1]
    return out


def rank5_factors(N: int, L: int, seed: int, rank: int = 5, n_ellipses: int = 6, n_sines: int = 8):
    """Spatial components s_r (complex128 [rank][N][N]) and temporal curves u_r (complex128 [L][rank]).

    s_r = sum_e a_{r,e} 1[x in ellipse e]: 6 shared ellipses (centres U[-0.3,0.3]^2, semi-axes
    U[0.05,0.35], angle U[0,pi)), amplitudes a ~ CN(0,1).  u_r(l) = sum_q b_q exp(i(2 pi f_q l/L +
    phi_q)), f ~ U[0,4), b ~ U[0.5,1], phi ~ U[0,2pi), then ||u_r||_2 = 1.
    """
    rng = np.random.default_rng([seed, 1])
    cen = rng.uniform(-0.3, 0.3, (n_ellipses, 2))
    ax = rng.uniform(0.05, 0.35, (n_ellipses, 2))
    ang = rng.uniform(0.0, np.pi, n_ellipses)
    amp = (rng.standard_normal((rank, n_ellipses)) + 1j * rng.standard_normal((rank, n_ellipses))) / np.sqrt(2)
    pos = (np.arange(N) - N // 2) / N
    yy, xx = np.meshgrid(pos, pos, indexing="ij")
    S = np.zeros((rank, N, N), dtype=np.complex128)
    for e in range(n_ellipses):
        dx, dy = xx - cen[e, 0], yy - cen[e, 1]
        c, s = np.cos(ang[e]), np.sin(ang[e])
        xr, yr = dx * c + dy * s, -dx * s + dy * c
        inside = (xr / ax[e, 0]) ** 2 + (yr / ax[e, 1]) ** 2 <= 1.0
        S += amp[:, e, None, None] * inside[None]
    rng2 = np.random.default_rng([seed, 2])
    l = np.arange(L, dtype=np.float64)
    U = np.zeros((L, rank), dtype=np.complex128)
    for r in range(rank):
        f = rng2.uniform(0.0, 4.0, n_sines)
        b = rng2.uniform(0.5, 1.0, n_sines)
        ph = rng2.uniform(0.0, 2 * np.pi, n_sines)
        u = (b[None, :] * np.exp(1j * (2 * np.pi * f[None, :] * l[:, None] / L + ph[None, :]))).sum(1)
        U[:, r] = u / np.linalg.norm(u)
    return S, U


def rank5_images(N: int, L: int, frames: Sequence[int], seed: int) -> np.ndarray:
    """X_l = sum_r s_r u_r(l), complex64 [len(frames)][N][N]."""
    S, U = rank5_factors(N, L, seed)
    Uf = U[np.asarray(list(frames), dtype=np.int64)]
    return np.einsum("lr,rij->lij", Uf, S).astype(np.complex64)


def images(cfg: Config, frames: Sequence[int] | None = None) -> np.ndarray:
    frames = range(cfg.L) if frames is None else frames
    frames = list(frames)
    if cfg.image_kind == "iid":
        return iid_images(cfg.N, frames, cfg.seed)
    return rank5_images(cfg.N, cfg.L, frames, cfg.seed)


# ----------------------------------------------------------------------------- coils / noise
def coil_maps(N: int, C: int, seed: int) -> np.ndarray | None:
    """Gaussian-blob sensitivities, complex64 [C][N][N], unit sum-of-squares.

    Centre 0.6 (cos 2 pi c/C, sin 2 pi c/C) in FOV units, width 0.4 FOV, phase U[0, 2 pi).
    C == 1 returns None (single coil, S = 1; reading #12).
    """
    if C == 1:
        return None
    rng = np.random.default_rng([seed, 3])
    phase = rng.uniform(0.0, 2 * np.pi, C)
    pos = (np.arange(N) - N // 2) / N
    yy, xx = np.meshgrid(pos, pos, indexing="ij")
    S = np.empty((C, N, N), dtype=np.complex128)
    for c in range(C):
        cx, cy = 0.6 * np.cos(2 * np.pi * c / C), 0.6 * np.sin(2 * np.pi * c / C)
        S[c] = np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * 0.4 ** 2)) * np.exp(1j * phase[c])
    S /= np.sqrt((np.abs(S) ** 2).sum(0, keepdims=True))
    return S.astype(np.complex64)


def unit_noise(C: int, M: int, frames: Sequence[int], seed: int) -> np.ndarray:
    """Complex Gaussian, unit complex variance (1/sqrt2 per component), complex64 [F][C][M]."""
    out = np.empty((len(frames), C, M), dtype=np.complex64)
    for i, l in enumerate(frames):
        rng = np.random.default_rng([seed, 4, int(l)])
        v = rng.standard_normal((2, C, M), dtype=np.float32) / np.float32(np.sqrt(2.0))
        out[i].real = v[0]
        out[i].imag = v[1]
    return out


def random_kspace(C: int, M: int, frames: Sequence[int], seed: int) -> np.ndarray:
    """i.i.d. complex k-space samples (adjoint-test inputs), complex64 [F][C][M]."""
    out = np.empty((len(frames), C, M), dtype=np.complex64)
    for i, l in enumerate(frames):
        rng = np.random.default_rng([seed, 5, int(l)])
        v = rng.standard_normal((2, C, M), dtype=np.float32)
        out[i].real = v[0]
        out[i].imag = v[1]
    return out

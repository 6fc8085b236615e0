"""Seeded synthetic MRF dictionary and voxel fingerprints for dictionary matching.

No arithmetic of the matching method lives here: only the parameter grid, a pulse schedule, a
closed-form stand-in for the Bloch response B(eta, theta) of PAPER.md:69-74 (Eq. 3), and voxel
fingerprints built from it.  The paper's dictionary is simulated with the Bloch equation and
its FA/TR schedule is not published; EPG/Bloch simulation is out of scope
(DESIGN.md §11), so a smooth surrogate signal model stands in.  The matching operator does not
depend on where the atoms come from.

  * ``t1t2_grid``: the paper's discretisation: T1 in [100, 2000] ms step 20 and
    [2300, 5000] ms step 300; T2 in [20, 100] step 5, [110, 200] step 10, [300, 1900] step 200;
    pairs with T1 < T2 omitted -> 3336 atoms.
  * ``surrogate_dictionary``: d_l(T1, T2) = sin(a_l) (1 - 2 exp(-t_l / T1)) exp(-s_l / T2)
    exp(i phi_l T2 / 1000), with a smooth random flip-angle train a_l, cumulative time t_l,
    a T2-weighting schedule s_l and a phase schedule phi_l (seeded).  Proton density 1 per atom
    (PAPER.md:74), so atom norms differ.
  * ``voxel_fingerprints``: x_v = rho_v d_{k_v} + noise for seeded atom indices k_v and PD rho_v.
"""
from __future__ import annotations

import numpy as np


def t1t2_grid() -> np.ndarray:
    """[K][2] float64 (T1, T2) in ms, T1-major, the paper's grid."""
    t1 = np.concatenate([np.arange(100, 2001, 20), np.arange(2300, 5001, 300)]).astype(np.float64)
    t2 = np.concatenate([np.arange(20, 101, 5), np.arange(110, 201, 10), np.arange(300, 1901, 200)]).astype(np.float64)
    pairs = [(a, b) for a in t1 for b in t2 if not a < b]
    return np.asarray(pairs, dtype=np.float64)


def pulse_schedule(L: int, seed: int = 11):
    """Smooth random flip angles (rad), cumulative time t_l (ms), T2-weighting s_l (ms), phase phi_l."""
    rng = np.random.default_rng([seed, 0])
    l = np.arange(L, dtype=np.float64)
    n_seg = max(1, L // 200)
    amp = rng.uniform(10.0, 70.0, size=n_seg)
    fa_deg = 5.0 + np.concatenate([a * np.abs(np.sin(np.pi * np.arange(200) / 200.0)) for a in amp])[:L]
    if fa_deg.size < L:
        fa_deg = np.pad(fa_deg, (0, L - fa_deg.size), constant_values=5.0)
    tr = 12.0 + 3.0 * np.sin(2 * np.pi * l / 250.0) + rng.uniform(0.0, 1.0, size=L)
    t = np.cumsum(tr)
    s = 20.0 + 80.0 * (0.5 + 0.5 * np.sin(2 * np.pi * l / 170.0 + rng.uniform(0, 2 * np.pi)))
    phi = 2 * np.pi * (0.5 + 0.5 * np.cos(2 * np.pi * l / 310.0 + rng.uniform(0, 2 * np.pi)))
    return np.deg2rad(fa_deg), t, s, phi


def surrogate_dictionary(L: int, grid: np.ndarray | None = None, seed: int = 11) -> np.ndarray:
    """[K][L] complex128 atoms for the (T1, T2) grid (closed-form stand-in for Eq. 3)."""
    grid = t1t2_grid() if grid is None else grid
    a, t, s, phi = pulse_schedule(L, seed)
    T1 = grid[:, 0:1]
    T2 = grid[:, 1:2]
    mag = np.sin(a)[None, :] * (1.0 - 2.0 * np.exp(-t[None, :] / T1)) * np.exp(-s[None, :] / T2)
    return mag * np.exp(1j * phi[None, :] * (T2 / 1000.0))


def voxel_fingerprints(D: np.ndarray, V: int, seed: int = 12, noise: float = 0.0):
    """x_v = rho_v d_{k_v} + noise: returns (X [V][L] complex128, k [V], rho [V])."""
    rng = np.random.default_rng([seed, 1])
    K, L = D.shape
    k = rng.integers(0, K, size=V)
    rho = rng.uniform(0.2, 2.0, size=V)
    X = rho[:, None] * D[k]
    if noise:
        sc = noise * np.sqrt(np.mean(np.abs(X) ** 2))
        X = X + sc * (rng.standard_normal(X.shape) + 1j * rng.standard_normal(X.shape)) / np.sqrt(2)
    return X, k, rho


def parameter_maps(N: int, seed: int = 3) -> np.ndarray:
    """(T1 [ms], T2 [ms], PD) maps [3][N][N]: seeded ellipses of tissue values on a zero background
    (the input of the manifold weights, Eq. 8, in place of Phi_D's estimates)."""
    rng = np.random.default_rng([seed, 2])
    yy, xx = np.mgrid[0:N, 0:N] / N - 0.5
    maps = np.zeros((3, N, N))
    for _ in range(7):
        cy, cx = rng.uniform(-0.3, 0.3, 2)
        ay, ax = rng.uniform(0.05, 0.3, 2)
        th = rng.uniform(0, np.pi)
        u = ((xx - cx) * np.cos(th) + (yy - cy) * np.sin(th)) / ax
        v = (-(xx - cx) * np.sin(th) + (yy - cy) * np.cos(th)) / ay
        m = u * u + v * v <= 1.0
        t2 = rng.uniform(20, 300)
        maps[0][m] = rng.uniform(max(300.0, t2), 3000)
        maps[1][m] = t2
        maps[2][m] = rng.uniform(0.3, 1.0)
    return maps

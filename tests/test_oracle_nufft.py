"""Pins for oracle/nufft.py (SURVEY.md §8(c) "What pins each part").

Each test ties the oracle to something other than itself: a brute-force NUDFT, numpy.fft on a
Cartesian trajectory, closed forms, the adjoint identity, Hermitian/PSD structure, A^H A = I.
"""
import numpy as np
import pytest

import synth
from oracle import nufft as on


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.fixture(scope="module")
def pr1():
    cfg = synth.get_config("pr1")
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    x = synth.images(cfg)
    return cfg, traj, x


# ------------------------------------------------------------------ the NUDFT itself
def test_nudft_cartesian_equals_numpy_fft():
    """k on the Cartesian grid: the direct sum equals fftshift(fft2(ifftshift(x), ortho))."""
    N = 16
    rng = np.random.default_rng(0)
    x = crandn(rng, N, N)
    k = synth.cartesian_trajectory(N)[0]
    y = on.nudft_forward_frame(x, None, k)[0]
    ref = np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x), norm="ortho")).ravel()
    assert rel(y, ref) < 1e-13
    xa = on.nudft_adjoint_frame(y[None], None, k, N)
    ref_a = np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(ref.reshape(N, N)), norm="ortho"))
    assert rel(xa, ref_a) < 1e-13
    assert rel(xa, x) < 1e-13


def test_nudft_delta_closed_form():
    """x = delta at n0 => y_j = exp(-i 2 pi k_j . n0) / N (sign + centering)."""
    N = 16
    n0 = (3, -5)                    # (n_x, n_y)
    x = np.zeros((N, N), complex)
    x[n0[1] + N // 2, n0[0] + N // 2] = 1.0
    k = synth.random_trajectory(50, 1, 3)[0].astype(np.float64)
    y = on.nudft_forward_frame(x, None, k)[0]
    ref = np.exp(-2j * np.pi * (k[:, 0] * n0[0] + k[:, 1] * n0[1])) / N
    assert np.max(np.abs(y - ref)) < 1e-14


def test_nudft_wrap_half():
    """k = +1/2 and -1/2 are the same sample for integer n (reading #4)."""
    N = 16
    rng = np.random.default_rng(1)
    x = crandn(rng, N, N)
    k1 = np.array([[0.5, 0.1], [0.2, 0.5], [0.5, 0.5]])
    k2 = np.array([[-0.5, 0.1], [0.2, -0.5], [-0.5, -0.5]])
    assert rel(on.nudft_forward_frame(x, None, k1), on.nudft_forward_frame(x, None, k2)) < 1e-12


def test_nudft_adjoint_identity():
    N, C = 12, 3
    rng = np.random.default_rng(2)
    S = crandn(rng, C, N, N)
    x = crandn(rng, N, N)
    k = synth.random_trajectory(40, 1, 4)[0]
    y = crandn(rng, C, 40)
    lhs = np.vdot(on.nudft_forward_frame(x, S, k), y)
    rhs = np.vdot(x, on.nudft_adjoint_frame(y, S, k, N))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


# ------------------------------------------------------------------ gridding vs the definition
def test_gridding_vs_nudft_pr1(pr1):
    """PR1 tiny spiral (32^2, M=256, L=8), W=6, sigma=2: rel L2 <= 1e-4 (BASELINE north_star)."""
    cfg, traj, x = pr1
    y = on.forward(x, traj, None, cfg.W)
    y_ref = on.nudft_forward(x, traj, None)
    e = rel(y, y_ref)
    assert e < 1e-4 and e < 2e-5, e           # survey measured 6.7e-6
    yr = synth.random_kspace(1, cfg.M, range(cfg.L), 11)
    xa = on.adjoint(yr, traj, None, cfg.N, cfg.W)
    xa_ref = on.nudft_adjoint(yr, traj, None, cfg.N)
    assert rel(xa, xa_ref) < 2e-5


def test_gridding_vs_nudft_random_points_coils():
    """16x16 image, 200 random coordinates, < 1e-4 vs the direct DFT; with coils."""
    N, M, C = 16, 200, 3
    rng = np.random.default_rng(5)
    S = crandn(rng, C, N, N)
    x = crandn(rng, 2, N, N)
    traj = synth.random_trajectory(M, 2, 6)
    y = on.forward(x, traj, S, 6)
    assert rel(y, on.nudft_forward(x, traj, S)) < 1e-4
    yr = crandn(rng, 2, C, M)
    assert rel(on.adjoint(yr, traj, S, N, 6), on.nudft_adjoint(yr, traj, S, N)) < 1e-4


def test_width_monotone(pr1):
    """error(W=4) > error(W=6) > error(W=8)."""
    cfg, traj, x = pr1
    y_ref = on.nudft_forward(x[:2], traj, None)
    errs = [rel(on.forward(x[:2], traj, None, W), y_ref) for W in (4, 6, 8)]
    assert errs[0] > errs[1] > errs[2], errs
    assert errs[2] < 1e-6


def test_gridding_adjoint_identity(pr1):
    cfg, traj, x = pr1
    rng = np.random.default_rng(7)
    y = crandn(rng, cfg.L, 1, cfg.M)
    lhs = np.vdot(on.forward(x, traj, None, cfg.W), y)
    rhs = np.vdot(x, on.adjoint(y, traj, None, cfg.N, cfg.W))
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(on.forward(x, traj, None, cfg.W)) * np.linalg.norm(y)


def test_gridding_adjoint_identity_coils_w8():
    N, C, M = 32, 4, 300
    rng = np.random.default_rng(8)
    S = crandn(rng, C, N, N)
    traj = synth.spiral_trajectory(M, 3, 4, 4.0)
    x = crandn(rng, 3, N, N)
    y = crandn(rng, 3, C, M)
    Ax = on.forward(x, traj, S, 8)
    lhs = np.vdot(Ax, y)
    rhs = np.vdot(x, on.adjoint(y, traj, S, N, 8))
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(Ax) * np.linalg.norm(y)


def test_cartesian_equals_fft_discrete_and_analytic():
    """Reading #9: Cartesian k equals fft2 ortho; <= 1e-12 discrete deapod, <= 1e-4 analytic."""
    N = 32
    rng = np.random.default_rng(9)
    x = crandn(rng, 1, N, N)
    traj = synth.cartesian_trajectory(N)
    ref = np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x[0]), norm="ortho")).ravel()
    yd = on.forward(x, traj, None, 6, deapod_mode="discrete")[0, 0]
    ya = on.forward(x, traj, None, 6, deapod_mode="analytic")[0, 0]
    assert rel(yd, ref) < 1e-12
    assert rel(ya, ref) < 1e-4
    # adjoint of the Cartesian data is the inverse FFT
    xd = on.adjoint(ref[None, None], traj, None, N, 6, deapod_mode="discrete")[0]
    assert rel(xd, x[0]) < 1e-12


def test_single_dc_sample_constant_image():
    """One sample at k = 0 => adjoint is the constant image y conj(S)/N."""
    N = 16
    traj = np.zeros((1, 1, 2), np.float32)
    y = np.array([[[2.0 - 1.0j]]])
    xd = on.adjoint(y, traj, None, N, 6, deapod_mode="discrete")[0]
    assert np.max(np.abs(xd - y[0, 0, 0] / N)) < 1e-14
    xa = on.adjoint(y, traj, None, N, 6, deapod_mode="analytic")[0]
    assert np.max(np.abs(xa - y[0, 0, 0] / N)) / abs(y[0, 0, 0] / N) < 1e-4
    rng = np.random.default_rng(10)
    S = crandn(rng, 2, N, N)
    xs = on.adjoint(np.array([[[1.5 + 0.5j], [0.25 - 1j]]]), traj, S, N, 6, deapod_mode="discrete")[0]
    assert np.max(np.abs(xs - (np.conj(S[0]) * (1.5 + 0.5j) + np.conj(S[1]) * (0.25 - 1j)) / N)) < 1e-13


def test_zero_in_zero_out(pr1):
    cfg, traj, _ = pr1
    assert not np.any(on.forward(np.zeros((2, cfg.N, cfg.N), complex), traj, None, cfg.W))
    assert not np.any(on.adjoint(np.zeros((2, 1, cfg.M), complex), traj, None, cfg.N, cfg.W))


def test_normal_hermitian_psd(pr1):
    cfg, traj, x = pr1
    rng = np.random.default_rng(12)
    z = crandn(rng, cfg.L, cfg.N, cfg.N)
    Nx = on.normal(x, traj, None, cfg.W)
    Nz = on.normal(z, traj, None, cfg.W)
    a, b = np.vdot(x, Nz), np.vdot(Nx, z)
    assert abs(a - b) <= 1e-12 * abs(a)
    q = np.vdot(x, Nx)
    Ax = on.forward(x, traj, None, cfg.W)
    assert abs(q.imag) <= 1e-12 * abs(q.real)
    assert abs(q.real - np.vdot(Ax, Ax).real) <= 1e-12 * q.real
    assert q.real > 0
    mu = 0.01
    assert rel(on.normal(x, traj, None, cfg.W, mu=mu), Nx + mu * x.astype(np.complex128)) < 1e-14


def test_normal_identity_full_cartesian_sos_coils():
    """Full Cartesian + unit-SoS coils + discrete deapod => A^H A = I exactly."""
    N = 16
    rng = np.random.default_rng(13)
    S = crandn(rng, 4, N, N)
    S /= np.sqrt((np.abs(S) ** 2).sum(0, keepdims=True))
    x = crandn(rng, 2, N, N)
    traj = synth.cartesian_trajectory(N)
    out = on.normal(x, traj, S, 6, deapod_mode="discrete", frame_interleaf=[0, 0])
    assert rel(out, x) < 1e-12


def test_frame_shard_consistency(pr1):
    """Forward on frames [3, 8) with frame_offset=3 equals the same rows of the full forward."""
    cfg, traj, x = pr1
    full = on.forward(x, traj, None, cfg.W)
    part = on.forward(x[3:], traj, None, cfg.W, frame_offset=3)
    assert np.array_equal(full[3:], part)
    il = synth.frame_interleaf(range(3, 8), cfg.R)
    part2 = on.forward(x[3:], traj, None, cfg.W, frame_interleaf=il)
    assert np.array_equal(full[3:], part2)


def test_stages_consistent(pr1):
    """The exposed intermediates compose to y (row FFT then column FFT = fft2; taps gather)."""
    cfg, traj, x = pr1
    gp = on.GridParams(cfg.N, cfg.W)
    y, st = on.grid_forward_frame(x[0], None, traj[0], gp, stages=True)
    g, half, X = st["g"][0], st["half"][0], st["X"][0]
    full_from_half = np.zeros_like(X)
    full_from_half[gp.idx, :] = half
    assert rel(np.fft.fft(full_from_half, axis=0), X) < 1e-13
    assert rel(np.fft.fft2(g), X) < 1e-13

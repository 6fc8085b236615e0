"""Pins for oracle/pcg.py (preconditioned CG; reading 28).

The circulant eigenvalues are checked against their definition -- Rayleigh quotients of the
exact (NUDFT) normal operator at the Fourier vectors -- by brute force; M^-1 against a dense solve
with the explicitly assembled circulant; Chan's Frobenius optimality by perturbation; PCG against
the preconditioned Krylov (Galerkin) projection, the dense solve, and plain CG for M = I.
"""
import numpy as np
import pytest

import synth
from oracle import cg as ocg
from oracle import nufft as on
from oracle import pcg as opc


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def fourier_vectors(N):
    """f_m[n] = exp(+i 2 pi m . n / N) / N over centred m, n; columns ordered [my][mx] like lambda."""
    n = np.arange(N) - N // 2
    ny, nx = np.meshgrid(n, n, indexing="ij")
    F = np.empty((N * N, N * N), dtype=np.complex128)
    for a, my in enumerate(n):
        for b, mx in enumerate(n):
            F[:, a * N + b] = (np.exp(2j * np.pi * (mx * nx + my * ny) / N) / N).ravel()
    return F


@pytest.fixture(scope="module")
def tiny():
    """8x8 images, one frame of an asymmetric spiral (axis swaps show), dense exact normal."""
    N, M, mu = 8, 37, 0.01
    traj = synth.spiral_trajectory(M, 3, 2, 1.5)[1:2]          # a rotated interleaf
    eye = np.eye(N * N, dtype=complex)
    A = np.stack([on.nudft_forward(eye[i].reshape(1, N, N), traj, None).ravel() for i in range(N * N)], axis=1)
    T = A.conj().T @ A                                          # exact A^H A (Toeplitz)
    return N, traj, T, mu


def test_fejer_closed_form():
    N = 8
    t = np.array([0.0, 1.0, -2.0, 0.013, -0.37, 0.5])
    brute = np.abs(np.exp(-2j * np.pi * t[:, None] * (np.arange(N) - N // 2)[None, :]).sum(1)) ** 2
    assert np.allclose(opc.fejer(t, N), brute, rtol=1e-12, atol=1e-9)


def test_eigenvalues_are_rayleigh_quotients_of_the_exact_normal(tiny):
    N, traj, T, mu = tiny
    F = fourier_vectors(N)
    rq = np.real(np.einsum("im,ij,jm->m", F.conj(), T, F)).reshape(N, N)
    lam = opc.circulant_eigs(traj[0], N)
    assert np.allclose(lam, rq, rtol=1e-11, atol=1e-14)
    assert lam.min() >= 0.0


def test_chan_circulant_is_frobenius_optimal(tiny):
    """C = F diag(lambda) F^H is the circulant closest to A^H A: perturbing its eigenvalues only
    increases ||C - T||_F."""
    N, traj, T, mu = tiny
    F = fourier_vectors(N)
    lam = opc.circulant_eigs(traj[0], N).ravel()
    base = np.linalg.norm(F @ np.diag(lam) @ F.conj().T - T)
    rng = np.random.default_rng(4)
    for _ in range(5):
        lp = lam + 1e-3 * rng.standard_normal(lam.shape)
        assert np.linalg.norm(F @ np.diag(lp) @ F.conj().T - T) > base


def test_precond_apply_equals_dense_solve(tiny):
    N, traj, T, mu = tiny
    F = fourier_vectors(N)
    lam = opc.circulant_eigs(traj[0], N)
    gamma, scale = 0.37, 1.3
    Mmat = F @ np.diag(scale * lam.ravel() + gamma) @ F.conj().T
    v = crandn(np.random.default_rng(5), 1, N, N)
    got = opc.precond_apply(v, lam[None], gamma, scale)
    assert np.linalg.norm(got.ravel() - np.linalg.solve(Mmat, v.ravel())) <= 1e-12 * np.linalg.norm(got)


@pytest.mark.parametrize("n", [1, 3, 5])
def test_pcg_iterate_equals_preconditioned_krylov_projection(tiny, n):
    N, traj, T, mu = tiny
    H = T + mu * np.eye(N * N)
    lam = opc.circulant_eigs(traj[0], N)
    g = opc.shift_gamma(lam, mu, 3.0)
    F = fourier_vectors(N)
    Mi = F @ np.diag(1.0 / (lam.ravel() + g)) @ F.conj().T
    rng = np.random.default_rng(6)
    rhs, x0 = crandn(rng, 1, N, N), 0.1 * crandn(rng, 1, N, N)
    Hf = lambda v: (H @ v.ravel()).reshape(v.shape)
    x, _ = opc.pcg(Hf, lambda v: opc.precond_apply(v, lam[None], g), rhs, x0, n)
    ref = opc.preconditioned_krylov_projection(H, Mi, rhs.ravel(), x0.ravel(), n)
    assert np.linalg.norm(x.ravel() - ref) <= 1e-10 * np.linalg.norm(ref)


def test_pcg_converges_to_the_unpreconditioned_solution(tiny):
    N, traj, T, mu = tiny
    H = T + mu * np.eye(N * N)
    lam = opc.circulant_eigs(traj[0], N)
    g = opc.shift_gamma(lam, mu, 30.0)
    rhs = crandn(np.random.default_rng(7), 1, N, N)
    Hf = lambda v: (H @ v.ravel()).reshape(v.shape)
    x, hist = opc.pcg(Hf, lambda v: opc.precond_apply(v, lam[None], g), rhs, np.zeros_like(rhs), 500, tol=1e-13)
    assert np.linalg.norm(x.ravel() - np.linalg.solve(H, rhs.ravel())) <= 1e-10 * np.linalg.norm(x)
    assert hist[-1] / hist[0] < 1e-13


def test_pcg_with_identity_is_cg():
    cfg = synth.get_config("pr1")
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    x = synth.images(cfg)[:2]
    H = lambda v: on.normal(v, traj, None, cfg.W, mu=cfg.mu)
    rhs = on.adjoint(on.forward(x, traj, None, cfg.W), traj, None, cfg.N, cfg.W)
    a, ha = opc.pcg(H, lambda v: v.copy(), rhs, np.zeros_like(rhs), 5)
    b, hb = ocg.cg(H, rhs, np.zeros_like(rhs), 5)
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
    assert np.allclose(ha, hb, rtol=1e-12, atol=0)


def test_pcg_tol_stops_on_the_true_residual(tiny):
    N, traj, T, mu = tiny
    H = T + mu * np.eye(N * N)
    lam = opc.circulant_eigs(traj[0], N)
    g = opc.shift_gamma(lam, mu, 30.0)
    rhs = crandn(np.random.default_rng(8), 1, N, N)
    Hf = lambda v: (H @ v.ravel()).reshape(v.shape)
    x, hist = opc.pcg(Hf, lambda v: opc.precond_apply(v, lam[None], g), rhs, np.zeros_like(rhs), 200, tol=1e-4)
    assert hist[-1] / hist[0] < 1e-4 and all(h / hist[0] >= 1e-4 for h in hist[:-1])
    assert np.isclose(hist[-1], np.linalg.norm(rhs.ravel() - H @ x.ravel()), rtol=1e-6)

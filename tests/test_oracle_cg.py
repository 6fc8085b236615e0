"""Pins for oracle/cg.py: CG = Krylov projection, converged CG = dense solve, A^H A = I case."""
import numpy as np
import pytest

import synth
from oracle import nufft as on
from oracle import cg as ocg


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.fixture(scope="module")
def tiny():
    """8x8 image, 1 frame, M=40 spiral points, W=6: dense 64x64 H = A^H A + mu I."""
    N, M, W, mu = 8, 40, 6, 0.01
    traj = synth.spiral_trajectory(M, 1, 2, 1.5)
    def H(v):
        return on.normal(v.reshape(1, N, N), traj, None, W, mu=mu).reshape(v.shape)
    eye = np.eye(N * N, dtype=complex)
    Hmat = np.stack([H(eye[i].reshape(1, N, N)).ravel() for i in range(N * N)], axis=1)
    rng = np.random.default_rng(0)
    rhs = crandn(rng, 1, N, N)
    return N, H, Hmat, rhs, mu


def test_dense_h_hermitian_pd(tiny):
    N, H, Hmat, rhs, mu = tiny
    assert np.max(np.abs(Hmat - Hmat.conj().T)) < 1e-12 * np.max(np.abs(Hmat))
    ev = np.linalg.eigvalsh(0.5 * (Hmat + Hmat.conj().T))
    assert ev.min() >= mu * (1 - 1e-9)


@pytest.mark.parametrize("n", [1, 3, 5])
def test_cg_iterate_equals_krylov_projection(tiny, n):
    N, H, Hmat, rhs, mu = tiny
    rng = np.random.default_rng(1)
    x0 = crandn(rng, 1, N, N) * 0.1
    x_cg, _ = ocg.cg(H, rhs, x0, n)
    x_kr = ocg.krylov_projection(Hmat, rhs.ravel(), x0.ravel(), n)
    assert np.linalg.norm(x_cg.ravel() - x_kr) <= 1e-10 * np.linalg.norm(x_kr)


def test_cg_converges_to_dense_solve(tiny):
    N, H, Hmat, rhs, mu = tiny
    x_cg, hist = ocg.cg(H, rhs, np.zeros_like(rhs), 300, tol=1e-14)
    x_ref = np.linalg.solve(Hmat, rhs.ravel())
    assert np.linalg.norm(x_cg.ravel() - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
    assert hist[-1] / hist[0] < 1e-13


def test_cg_tol_stops_early(tiny):
    N, H, Hmat, rhs, mu = tiny
    _, hist_full = ocg.cg(H, rhs, np.zeros_like(rhs), 40)
    _, hist_tol = ocg.cg(H, rhs, np.zeros_like(rhs), 40, tol=1e-3)
    assert len(hist_tol) < len(hist_full)
    assert hist_tol[-1] / hist_tol[0] < 1e-3
    assert all(h / hist_tol[0] >= 1e-3 for h in hist_tol[:-1])


def test_cg_identity_case_one_iteration():
    """A^H A = I (full Cartesian, SoS coils, discrete deapod) => x1 = rhs / (1 + mu)."""
    N, mu = 16, 0.01
    rng = np.random.default_rng(2)
    S = crandn(rng, 3, N, N)
    S /= np.sqrt((np.abs(S) ** 2).sum(0, keepdims=True))
    traj = synth.cartesian_trajectory(N)
    H = lambda v: on.normal(v, traj, S, 6, mu=mu, deapod_mode="discrete", frame_interleaf=[0, 0])
    rhs = crandn(rng, 2, N, N)
    x1, hist = ocg.cg(H, rhs, np.zeros_like(rhs), 1)
    assert np.linalg.norm(x1 - rhs / (1 + mu)) <= 1e-12 * np.linalg.norm(rhs)
    assert hist[1] <= 1e-12 * hist[0]


def test_cg_zero_rhs_returns_x0(tiny):
    N, H, Hmat, rhs, mu = tiny
    x, hist = ocg.cg(H, np.zeros_like(rhs), np.zeros_like(rhs), 5)
    assert not np.any(x) and len(hist) == 1


def test_cg_pr1_monotone_energy_error():
    """On PR1, the H-norm of the error to the solution decreases monotonically (CG optimality)."""
    cfg = synth.get_config("pr1")
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    x = synth.images(cfg)[:1]
    y = on.forward(x, traj, None, cfg.W)
    H = lambda v: on.normal(v, traj, None, cfg.W, mu=cfg.mu)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, None, cfg.N, cfg.W), None, cfg.mu)
    x_star, _ = ocg.cg(H, rhs, np.zeros_like(rhs), 400, tol=1e-13)
    errs = []
    for n in range(1, 8):
        xn, _ = ocg.cg(H, rhs, np.zeros_like(rhs), n)
        e = xn - x_star
        errs.append(np.vdot(e, H(e)).real)
    assert all(b < a for a, b in zip(errs, errs[1:])), errs

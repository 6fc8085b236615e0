"""GPU parity of the LLR outer step (SURVEY.md §8(f) f2 with lambda_1 = 0) against the oracle.

PAPER.md:217-264 Eqs. (15), (17), (20), (21); readings 24, 25.  The library computes the
subspace basis by subspace iteration and runs the patch SVT in subspace coordinates; the oracle
uses a full SVD of the dictionary and of every p^2 x L patch Casorati matrix in the time domain.
"""
import numpy as np
import pytest
import torch

import synth
import synth.dictionary as sd
from oracle import llr as ol
from oracle import nufft as on

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def binding():
    from paper_2310_05647_b200 import binding as b
    return b


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def projector(d):
    d = np.asarray(d, np.complex128)
    return np.conj(d).T @ d


def test_basis_matches_the_svd(binding):
    D = sd.surrogate_dictionary(200)
    dic = binding.Dictionary(D)
    dg = dic.basis(0.9999, 32)
    do = ol.basis(D, 0.9999, 32)
    assert dg.shape == do.shape
    assert np.allclose(dg @ np.conj(dg).T, np.eye(dg.shape[0]), atol=1e-5)
    assert rel(projector(dg), projector(do)) <= 1e-5
    dic.close()


@pytest.mark.parametrize("N,L,p,s", [(64, 100, 11, 5), (32, 60, 7, 3)])
def test_llr_step_against_the_oracle(binding, N, L, p, s):
    D = sd.surrogate_dictionary(L)
    M, R, W = 512, 10, 6
    traj = synth.spiral_trajectory(M, R, 8, 1.5)
    x_true = synth.rank5_images(N, L, range(L), 7)
    y = on.forward(x_true, traj, None, W)
    rhs = on.adjoint(y, traj, None, N, W)                 # A^H b; X^0 = A^H b (Algorithm 1)
    mu, lam2, beta = 1.0, 0.1, 0.2
    d_o = ol.basis(D, 0.9999, 32)
    normal = lambda v: on.normal(v, traj, None, W)
    X_ref, Z_ref = ol.llr_step(rhs, rhs, normal, d_o, mu, lam2, beta, p, s)
    _, nuc_ref = ol.llr_prox(Z_ref, 1.0 / beta, mu * lam2 * beta, p, s)

    dic = binding.Dictionary(D)
    dic.basis(0.9999, 32)
    op = binding.LLR(dic, N, p, s)
    pl = binding.Plan(N, traj, L, W=W)
    xd = torch.from_numpy(rhs.astype(np.complex64)).cuda()
    x_next, nuc, _ = op.step(pl, xd, xd, mu, lam2, beta)
    torch.cuda.synchronize()
    assert rel(x_next.cpu().numpy(), X_ref) <= 1e-4
    assert abs(nuc - nuc_ref) / nuc_ref <= 1e-4
    # the thresholding is active: some but not all singular values survive
    assert 0.0 < rel(X_ref, Z_ref) < 1.0
    x_alias, _, _ = op.step(pl, xd, xd, mu, lam2, beta, x_out=xd.clone())
    torch.cuda.synchronize()
    pl.close()
    op.close()
    dic.close()


def test_invalid_llr_calls(binding):
    D = sd.surrogate_dictionary(20)
    dic = binding.Dictionary(D)
    with pytest.raises(binding.MrfError):
        binding.LLR(dic, 32)                                   # no basis yet
    dic.basis()
    op = binding.LLR(dic, 32)
    pl = binding.Plan(64, synth.spiral_trajectory(128, 2, 4, 1.5), 20)   # N differs
    x = torch.zeros((20, 32, 32), dtype=torch.complex64, device="cuda")
    with pytest.raises(Exception):
        op.step(pl, x, x)
    pl.close()
    op.close()
    dic.close()


def test_llr_step_full_mrf_size_window(binding):
    """The MRF size (256 x 256 x 1000 frames, 2500 patches, the 3336-atom dictionary): the oracle
    computes Z for all frames (A^H A is per frame but global in space) and the exact patch SVTs of
    the 49 patches that cover a 21 x 21 window; the library's X+ must match there."""
    import os
    cfg = synth.get_config("mrf")
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    D = sd.surrogate_dictionary(cfg.L)
    x0 = synth.images(cfg)
    workers = max(1, len(os.sched_getaffinity(0)))
    y = on.forward(x0, traj, None, cfg.W, workers=workers)
    rhs = on.adjoint(y, traj, None, cfg.N, cfg.W, workers=workers)
    mu, lam2, beta, p, s = 1.0, 0.1, 0.2, 11, 5
    # library
    dic = binding.Dictionary(D)
    dic.basis(0.9999, 32)
    op = binding.LLR(dic, cfg.N, p, s)
    pl = binding.Plan(cfg.N, traj, cfg.L, W=cfg.W)
    xd = torch.from_numpy(rhs.astype(np.complex64)).cuda()
    xg, _, _ = op.step(pl, xd, xd, mu, lam2, beta)
    lo, hi = 120, 141
    xg_w = xg[:, lo:hi, lo:hi].cpu().numpy()
    pl.close()
    op.close()
    dic.close()
    # oracle: Z everywhere, then the covering patches' SVTs and the update on the window
    d_o = ol.basis(D, 0.9999, 32)
    Z = ol.project(rhs - mu * (on.normal(rhs, traj, None, cfg.W, workers=workers) - rhs), d_o)
    gamma = mu * lam2 * beta
    acc = np.zeros((cfg.L, hi - lo, hi - lo), np.complex128)
    cnt = np.zeros((hi - lo, hi - lo))
    cs = ol.patch_corners(cfg.N, p, s)
    near = [c for c in cs if c + p > lo and c < hi]
    for y0 in near:
        for x0_ in near:
            P = ol.svt(ol.casorati(Z, y0, x0_, p), 1.0 / beta).T.reshape(cfg.L, p, p)
            ys, xs = slice(max(y0, lo), min(y0 + p, hi)), slice(max(x0_, lo), min(x0_ + p, hi))
            acc[:, ys.start - lo:ys.stop - lo, xs.start - lo:xs.stop - lo] += \
                P[:, ys.start - y0:ys.stop - y0, xs.start - x0_:xs.stop - x0_]
            cnt[ys.start - lo:ys.stop - lo, xs.start - lo:xs.stop - lo] += 1
    X_ref = (Z[:, lo:hi, lo:hi] + gamma * acc) / (1.0 + gamma * cnt)[None]
    assert rel(xg_w, X_ref) <= 1e-4


def test_manifold_term_against_the_oracle(binding):
    """MS-LLR step with the manifold term (lambda_1 > 0): the Laplacian from parameter maps
    (sigma^2 by the median rule, degrees), the step and the trace penalty vs the oracle."""
    from oracle import manifold as omf
    N, L, p, s = 64, 100, 11, 5
    D = sd.surrogate_dictionary(L)
    traj = synth.spiral_trajectory(512, 10, 8, 1.5)
    x_true = synth.rank5_images(N, L, range(L), 7)
    rhs = on.adjoint(on.forward(x_true, traj, None, 6), traj, None, N, 6)
    maps = sd.parameter_maps(N, 3)                             # (T1, T2, PD) [3][N][N]
    W, s2 = omf.weights(maps, N, p, s)
    Lap = omf.laplacian(W)
    lam1 = 0.1 * float(Lap.max()) / 50.0
    mu, lam2, beta = 1.0, 0.1, 0.2
    d_o = ol.basis(D, 0.9999, 32)
    X_ref, _ = ol.llr_step(rhs, rhs, lambda v: on.normal(v, traj, None, 6), d_o, mu, lam2, beta, p, s,
                           lam1=lam1, lap=Lap)
    pen_ref = omf.penalty(ol.project(rhs, d_o), Lap, N, p, s)

    dic = binding.Dictionary(D)
    dic.basis(0.9999, 32)
    op = binding.LLR(dic, N, p, s)
    params = torch.from_numpy(np.ascontiguousarray(np.stack([maps[0].ravel(), maps[1].ravel()], 1))).float().cuda()
    pd = torch.from_numpy(np.ascontiguousarray(maps[2].ravel())).float().cuda()
    s2g, mdeg = op.laplacian(params, pd)
    assert abs(s2g - s2) / s2 <= 1e-5
    assert abs(mdeg - Lap.max()) / Lap.max() <= 1e-4
    pl = binding.Plan(N, traj, L, W=6)
    xd = torch.from_numpy(rhs.astype(np.complex64)).cuda()
    xg, _, pen = op.step(pl, xd, xd, mu, lam2, beta, lam1=lam1, penalty=True)
    torch.cuda.synchronize()
    assert rel(xg.cpu().numpy(), X_ref) <= 1e-4
    assert abs(pen - pen_ref) / abs(pen_ref) <= 1e-4
    # the manifold term matters here: the lambda_1 = 0 step differs
    x0, _, _ = op.step(pl, xd, xd, mu, lam2, beta)
    assert rel(x0.cpu().numpy(), X_ref) > 1e-3
    pl.close()
    op.close()
    dic.close()


def _oracle_basis_problem(N=32, L=60, seed=11):
    D = sd.surrogate_dictionary(L)
    d_o = ol.basis(D, 0.9999, 32)                               # float64 SVD basis (the oracle's)
    traj = synth.spiral_trajectory(512, 10, 8, 1.5)
    return D, d_o, traj


def test_subspace_normal_against_the_nudft(binding):
    """mrf_llr_subspace_normal on a Toeplitz plan with the ORACLE's basis (mrf_llr_create_basis):
    the coefficients of P_S A^H A (u d) against the plain-definition operator (NUDFT) in float64."""
    N, L = 32, 60
    D, d_o, traj = _oracle_basis_problem(N, L)
    r = d_o.shape[0]
    rng = np.random.default_rng([31, 1])
    u = (rng.standard_normal((r, N, N)) + 1j * rng.standard_normal((r, N, N))).astype(np.complex64)
    op = binding.LLR.from_basis(d_o, N, 7, 3)
    pl = binding.Plan(N, traj, L, W=6, normal="toeplitz")
    z = op.subspace_normal(pl, torch.from_numpy(u).cuda())
    torch.cuda.synchronize()
    X = np.einsum("il,iyx->lyx", d_o.astype(np.complex64).astype(np.complex128), u.astype(np.complex128))
    n = on.nudft_adjoint(on.nudft_forward(X, traj, None), traj, None, N)
    z_ref = np.einsum("il,lyx->iyx", np.conj(d_o.astype(np.complex64).astype(np.complex128)), n)
    assert rel(z.cpu().numpy(), z_ref) <= 1e-5
    with pytest.raises(binding.MrfError):
        op.subspace_normal(binding.Plan(N, traj, L, W=6), torch.from_numpy(u).cuda())   # gridding plan
    pl.close(), op.close()


def test_llr_step_with_the_oracle_basis(binding):
    """The LLR step with the oracle's basis (no basis difference between the two sides)."""
    N, L, p, s = 32, 60, 7, 3
    D, d_o, traj = _oracle_basis_problem(N, L)
    x_true = synth.rank5_images(N, L, range(L), 7)
    rhs = on.adjoint(on.forward(x_true, traj, None, 6), traj, None, N, 6)
    mu, lam2, beta = 0.02, 0.1, 0.2
    X_ref, _ = ol.llr_step(rhs, rhs, lambda v: on.normal(v, traj, None, 6), d_o.astype(np.complex64).astype(np.complex128),
                           mu, lam2, beta, p, s)
    op = binding.LLR.from_basis(d_o, N, p, s)
    pl = binding.Plan(N, traj, L, W=6)
    xd = torch.from_numpy(rhs.astype(np.complex64)).cuda()
    xg, _, _ = op.step(pl, xd, xd, mu, lam2, beta)
    torch.cuda.synchronize()
    assert rel(xg.cpu().numpy(), X_ref) <= 1e-5
    with pytest.raises(binding.MrfError):
        binding.LLR.from_basis(np.zeros((0, L), np.complex64), N)
    pl.close(), op.close()

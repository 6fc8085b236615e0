"""Pins of the Algorithm-1 oracle (oracle/msllr.py): closed forms of the cost
terms, the stop rule, projected-gradient descent when both regularisers are off, and the maps
output.  Small sizes (N = 16, L = 12, 5 x 5 patches, stride 2)."""
import numpy as np

import synth
from oracle import llr as ol
from oracle import manifold as om
from oracle import msllr as oms
from oracle import nufft as on

N, L, P, S, W = 16, 12, 5, 2, 6


def _setup(seed=0):
    rng = np.random.default_rng(seed)
    traj = synth.spiral_trajectory(96, 4, 4, 1.5)
    t = rng.standard_normal((3, L)) + 1j * rng.standard_normal((3, L))
    amps = rng.standard_normal((3, N, N)) + 1j * rng.standard_normal((3, N, N))
    X = np.einsum("kl,kyx->lyx", t, amps)                          # rank-3 time series
    return rng, traj, X, t


def test_cost_closed_forms():
    rng, traj, X, _ = _setup()
    A = lambda Y: on.forward(Y, traj, None, W)
    b = A(X)
    # data term: 1/2 ||A X - b||^2 = 0 at the generating image, and = 1/2 ||A E||^2 for X + E
    c, (data, trace, nuc) = oms.cost(X, b, A, 0.0, 0.0, None, P, S)
    assert data < 1e-20 and trace == 0.0 and c == data
    E = 1e-2 * (rng.standard_normal(X.shape) + 1j * rng.standard_normal(X.shape))
    _, (data2, _, _) = oms.cost(X + E, b, A, 0.0, 0.0, None, P, S)
    assert np.isclose(data2, 0.5 * np.sum(np.abs(A(E)) ** 2), rtol=1e-9)
    # nuclear term of a separable image X[l, y, x] = a[y, x] t[l]: every patch Casorati matrix is
    # rank one, ||Q_q||_* = ||a_q||_2 ||t||_2
    a = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
    tt = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    Xs = tt[:, None, None] * a[None]
    _, (_, _, nuc) = oms.cost(Xs, A(Xs), A, 0.0, 1.0, None, P, S)
    cs = ol.patch_corners(N, P, S)
    ref = sum(np.linalg.norm(a[y:y + P, x:x + P]) for y in cs for x in cs) * np.linalg.norm(tt)
    assert np.isclose(nuc, ref, rtol=1e-10)
    # trace term: identical patches (spatially constant image) -> 0 (rows of L sum to zero); weights
    # and the total combine linearly
    maps = np.stack([rng.uniform(500, 2000, (N, N)), rng.uniform(20, 200, (N, N)), rng.uniform(0.2, 1, (N, N))])
    lap = om.laplacian(om.weights(maps, N, P, S)[0])
    Xc = np.broadcast_to(tt[:, None, None], (L, N, N)).copy()
    _, (_, tr0, _) = oms.cost(Xc, A(Xc), A, 1.0, 0.0, lap, P, S)
    assert abs(tr0) < 1e-9 * np.sum(np.abs(Xc) ** 2) * lap.max()
    c3, (d3, t3, n3) = oms.cost(X + E, b, A, 0.3, 0.7, lap, P, S)
    assert t3 > 0 and np.isclose(c3, d3 + 0.3 * t3 + 0.7 * n3, rtol=1e-12)


def test_stop_rule_and_projected_gradient():
    rng, traj, X, t = _setup(1)
    b = on.forward(X, traj, None, W)
    # basis of the true temporal subspace (rank 3): P_S keeps X
    d = np.linalg.qr(t.conj().T)[0].conj().T                       # [3][L] orthonormal rows
    assert np.allclose(ol.project(X, d), X, atol=1e-10)
    D = np.concatenate([t, rng.standard_normal((5, L)) + 1j * rng.standard_normal((5, L))])
    lut = np.stack([np.arange(8) * 100.0 + 500, np.arange(8) * 10.0 + 50], 1)
    # lambda_1 = lambda_2 = 0: X^n = P_S(X^{n-1} - mu A^*(A X^{n-1} - b)), projected Landweber; with
    # mu below 1 / lambda_max(A^H A) the data term decreases monotonically
    lmax = 60.0
    out = oms.solve(b, traj, D, lut, d, 1.0 / lmax, 0.0, 0.0, 1.0, 6, tol=0.0, W=W, N=N, p=P, s=S)
    assert out["iters"] == 6 and len(out["cost"]) == 6
    assert all(c1 < c0 for c0, c1 in zip(out["cost"], out["cost"][1:]))
    # one step by hand from X^0 = A^* b
    rhs = on.adjoint(b, traj, None, N, W)
    X1 = ol.project(rhs - (1.0 / lmax) * (on.normal(rhs, traj, None, W) - rhs), d)
    one = oms.solve(b, traj, D, lut, d, 1.0 / lmax, 0.0, 0.0, 1.0, 1, tol=0.0, W=W, N=N, p=P, s=S)
    assert np.allclose(one["x"], X1, rtol=0, atol=1e-12 * np.abs(X1).max())
    # the stop rule: a huge tolerance stops at n = 2 (the first n with a cost(n-1))
    st = oms.solve(b, traj, D, lut, d, 1.0 / lmax, 0.0, 0.0, 1.0, 6, tol=1e9, W=W, N=N, p=P, s=S)
    assert st["iters"] == 2 and np.allclose(st["cost"], out["cost"][:2])
    # the maps output is Phi_D of the returned X
    k, _, rho, _ = __import__("oracle").match.match(out["x"].reshape(L, -1).T, D, lut)
    assert np.array_equal(out["k"], k) and np.allclose(out["rho"], rho)


def test_manifold_loop_uses_the_current_maps():
    """lambda_1 > 0: lambda_1 = lambda_1^0 max(L) with L from Phi_D of the current iterate."""
    rng, traj, X, t = _setup(2)
    b = on.forward(X, traj, None, W)
    d = np.linalg.qr(t.conj().T)[0].conj().T
    D = np.concatenate([t, rng.standard_normal((5, L)) + 1j * rng.standard_normal((5, L))])
    lut = np.stack([np.arange(8) * 100.0 + 500, np.arange(8) * 10.0 + 50], 1)
    out = oms.solve(b, traj, D, lut, d, 0.01, 1e-3, 0.05, 0.5, 2, tol=0.0, W=W, N=N, p=P, s=S)
    _, m = oms.maps_of(oms.solve(b, traj, D, lut, d, 0.01, 1e-3, 0.05, 0.5, 1, tol=0.0, W=W, N=N, p=P, s=S)["x"], D, lut)
    lap = om.laplacian(om.weights(m, N, P, S)[0])
    assert np.isclose(out["lambda1"], 1e-3 * lap.max(), rtol=1e-12)


def test_nudft_operator_mode_agrees_with_gridding_to_the_nufft_error():
    """op="nudft" runs the same loop on the plain-definition operator: one LLR iteration differs
    from the gridding loop by about the gridding error (~1e-5 at W = 6)."""
    rng, traj, X, t = _setup(3)
    b = on.nudft_forward(X, traj, None)
    d = np.linalg.qr(t.conj().T)[0].conj().T
    D = np.concatenate([t, rng.standard_normal((5, L)) + 1j * rng.standard_normal((5, L))])
    lut = np.stack([np.arange(8) * 100.0 + 500, np.arange(8) * 10.0 + 50], 1)
    a = oms.solve(b, traj, D, lut, d, 0.01, 0.0, 0.05, 0.5, 2, tol=0.0, W=W, N=N, p=P, s=S, op="nudft")
    g = oms.solve(b, traj, D, lut, d, 0.01, 0.0, 0.05, 0.5, 2, tol=0.0, W=W, N=N, p=P, s=S, op="grid")
    e = np.linalg.norm(a["x"] - g["x"]) / np.linalg.norm(a["x"])
    assert 1e-9 < e < 1e-4
    assert np.allclose(a["cost"], g["cost"], rtol=1e-3)

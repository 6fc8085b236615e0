"""Pins of the manifold-regularisation oracle (Eqs. 7-11)."""
import numpy as np

from oracle import manifold as om


def test_laplacian_of_the_papers_three_node_example():
    # SPEC.md:399 (Eq. 11 with w12 = 1, w13 = 2, w23 = 3)
    W = np.array([[0, 1, 2], [1, 0, 3], [2, 3, 0]], float)
    assert np.array_equal(om.laplacian(W), np.array([[3, -1, -2], [-1, 4, -3], [-2, -3, 5]], float))


def test_laplacian_rows_sum_to_zero_and_psd():
    rng = np.random.default_rng(1)
    A = rng.uniform(0, 1, (50, 50))
    W = np.triu(A, 1) + np.triu(A, 1).T
    Lp = om.laplacian(W)
    assert np.allclose(Lp.sum(1), 0, atol=1e-12)
    assert np.linalg.eigvalsh(Lp).min() >= -1e-10


def test_weights_brute_force_and_identities():
    rng = np.random.default_rng(2)
    N, p, s = 14, 5, 3
    maps = np.stack([rng.uniform(500, 2000, (N, N)), rng.uniform(20, 200, (N, N)), rng.uniform(0.1, 1, (N, N))])
    W, sig2 = om.weights(maps, N, p, s)
    P = om.patches(N, p, s)
    Mz = om.standardise(maps)
    n = len(P)
    d2 = np.zeros((n, n))
    for i, (yi, xi) in enumerate(P):        # explicit double loop over patch pairs
        for j, (yj, xj) in enumerate(P):
            d2[i, j] = np.sum((Mz[:, yi:yi + p, xi:xi + p] - Mz[:, yj:yj + p, xj:xj + p]) ** 2)
    nz = d2[np.triu_indices(n, 1)]
    assert np.isclose(sig2, np.median(nz[nz > 0]), rtol=1e-12)
    Wb = np.exp(-d2 / sig2)
    np.fill_diagonal(Wb, 0)
    assert np.allclose(W, Wb, rtol=1e-10, atol=1e-14)
    assert np.allclose(W, W.T) and np.all(np.diag(W) == 0) and W.max() <= 1
    # identical patches -> w = 1; distance^2 = sigma^2 -> exp(-1)
    W2, _ = om.weights(np.ones((3, N, N)), N, p, s, sigma2=1.0)
    assert np.allclose(W2[~np.eye(n, dtype=bool)], 1.0)


def test_standardise_over_foreground():
    rng = np.random.default_rng(3)
    maps = np.stack([rng.uniform(100, 3000, (8, 8)), rng.uniform(10, 300, (8, 8)), rng.uniform(0, 1, (8, 8))])
    z = om.standardise(maps)
    fg = maps[2] > 0.1 * maps[2].max()
    assert np.allclose(z[:, fg].mean(1), 0, atol=1e-12) and np.allclose(z[:, fg].std(1), 1, atol=1e-12)


def test_scatter_is_the_adjoint_and_counts_coverage():
    rng = np.random.default_rng(4)
    N, p, s, L = 12, 5, 3, 4
    P = om.patches(N, p, s)
    X = rng.standard_normal((L, N, N)) + 1j * rng.standard_normal((L, N, N))
    Qm = rng.standard_normal((L * p * p, len(P))) + 1j * rng.standard_normal((L * p * p, len(P)))
    lhs = np.vdot(om.casorati_all(X, P, p), Qm)
    rhs = np.vdot(X, om.scatter_adjoint(Qm, X.shape, P, p))
    assert np.isclose(lhs, rhs, rtol=1e-12)
    cov = om.scatter_adjoint(np.ones((p * p, len(P))), (1, N, N), P, p)[0]
    assert cov.min() >= 1


def test_trace_form_equals_half_the_ordered_pair_sum():
    rng = np.random.default_rng(5)
    N, p, s, L = 8, 3, 2, 4
    X = rng.standard_normal((L, N, N)) + 1j * rng.standard_normal((L, N, N))
    maps = np.stack([rng.uniform(500, 2000, (N, N)), rng.uniform(20, 200, (N, N)), rng.uniform(0.1, 1, (N, N))])
    W, _ = om.weights(maps, N, p, s)
    Lp = om.laplacian(W)
    P = om.patches(N, p, s)
    Qm = om.casorati_all(X, P, p)
    pair = sum(W[i, j] * np.linalg.norm(Qm[:, i] - Qm[:, j]) ** 2 for i in range(len(P)) for j in range(len(P)) if i != j)
    assert np.isclose(om.penalty(X, Lp, N, p, s), 0.5 * pair, rtol=1e-10)
    # constant data -> zero penalty; quadratic in X
    assert abs(om.penalty(np.ones((L, N, N)), Lp, N, p, s)) < 1e-9
    assert np.isclose(om.penalty(2 * X, Lp, N, p, s), 4 * om.penalty(X, Lp, N, p, s), rtol=1e-12)
    # the gradient is the derivative of the penalty: d/dt J(X + tE) at 0 = 2 Re <grad, E>
    E = rng.standard_normal(X.shape) + 1j * rng.standard_normal(X.shape)
    t = 1e-6
    num = (om.penalty(X + t * E, Lp, N, p, s) - om.penalty(X - t * E, Lp, N, p, s)) / (2 * t)
    assert np.isclose(num, 2 * np.real(np.vdot(om.gradient(X, Lp, N, p, s), E)), rtol=1e-6)


def test_raw_map_weights_printed_eq8():
    """Eq. (8) on the raw maps (reading 26 standardises them first): the weights
    equal an explicit loop over patch pairs of the raw (T1, T2, PD) values with the same median
    bandwidth, and equal the standardised weights when the maps are already standardised."""
    import synth.dictionary as sd
    N, p, s = 16, 5, 3
    maps = sd.parameter_maps(N)
    W, s2 = om.weights(maps, N, p, s, raw=True)
    P = om.patches(N, p, s)
    vec = [np.concatenate([maps[c][y0:y0 + p, x0:x0 + p].ravel() for c in range(3)]) for (y0, x0) in P]
    n = len(vec)
    d2 = np.array([[np.sum((vec[i] - vec[j]) ** 2) for j in range(n)] for i in range(n)])
    nz = d2[np.triu_indices(n, 1)]
    nz = nz[nz > 0]
    assert np.isclose(s2, np.median(nz), rtol=1e-12)
    ref = np.exp(-d2 / s2)
    np.fill_diagonal(ref, 0.0)
    assert np.allclose(W, ref, rtol=1e-12, atol=1e-15)
    st = om.standardise(maps)
    Ws, _ = om.weights(st, N, p, s, raw=True)
    Wr, _ = om.weights(maps, N, p, s, raw=False)
    assert np.allclose(Ws, Wr, atol=1e-12)

"""Pins of the LLR outer-step oracle (Eqs. (15), (17), (20), (21))."""
import numpy as np

from oracle import llr


def rand_c(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_basis_recovers_a_known_subspace():
    rng = np.random.default_rng(1)
    L = 40
    V, _ = np.linalg.qr(rand_c(rng, L, 3))          # orthonormal columns
    V = V.T                                          # [3][L] orthonormal rows
    D = rand_c(rng, 200, 3) @ V                      # exact rank 3
    d = llr.basis(D, energy=0.9999)
    assert d.shape == (3, L)
    assert np.allclose(d @ np.conj(d).T, np.eye(3), atol=1e-12)
    assert np.allclose(V @ np.conj(d).T @ d, V, atol=1e-12)   # span(V) = span(d)


def test_projection_is_the_orthogonal_projector():
    rng = np.random.default_rng(2)
    L, N = 30, 8
    d = np.linalg.qr(rand_c(rng, L, 4))[0].T
    X = rand_c(rng, L, N, N)
    P1 = llr.project(X, d)
    assert np.allclose(llr.project(P1, d), P1, atol=1e-12)                     # idempotent
    R = (X - P1).reshape(L, -1)
    assert np.allclose(np.conj(d) @ R, 0, atol=1e-12)                          # residual orthogonal
    # a voxel whose time series is a basis row is unchanged
    X2 = np.zeros((L, N, N), np.complex128)
    X2[:, 3, 5] = d[2]
    assert np.allclose(llr.project(X2, d), X2, atol=1e-12)


def test_patch_corners_cover_the_image():
    assert list(llr.patch_corners(256))[:3] == [0, 5, 10] and llr.patch_corners(256)[-1] == 245
    assert len(llr.patch_corners(256)) == 50
    assert list(llr.patch_corners(32)) == [0, 5, 10, 15, 20, 21]


def test_svt_closed_forms():
    rng = np.random.default_rng(3)
    # diagonal: soft threshold of the diagonal magnitudes
    Dg = np.diag([5.0, 2.0, 0.5, 0.0]).astype(np.complex128)
    assert np.allclose(llr.svt(Dg, 1.0), np.diag([4.0, 1.0, 0.0, 0.0]), atol=1e-12)
    # rank one: (sigma - tau)_+ u v^H
    u = rand_c(rng, 9)
    u /= np.linalg.norm(u)
    v = rand_c(rng, 20)
    v /= np.linalg.norm(v)
    C = 3.0 * np.outer(u, np.conj(v))
    assert np.allclose(llr.svt(C, 1.0), 2.0 * np.outer(u, np.conj(v)), atol=1e-12)
    assert np.allclose(llr.svt(C, 3.5), 0.0, atol=1e-12)
    C = rand_c(rng, 9, 20)
    assert np.allclose(llr.svt(C, 0.0), C, atol=1e-12)


def test_svt_is_the_nuclear_norm_prox():
    # SVT_tau(C) = argmin_P tau ||P||_* + 1/2 ||P - C||_F^2: no random perturbation does better
    rng = np.random.default_rng(4)
    C = rand_c(rng, 7, 12)
    tau = 1.3
    obj = lambda P: tau * np.linalg.svd(P, compute_uv=False).sum() + 0.5 * np.linalg.norm(P - C) ** 2
    P0 = llr.svt(C, tau)
    f0 = obj(P0)
    for _ in range(50):
        assert obj(P0 + 1e-3 * rand_c(rng, 7, 12)) >= f0 - 1e-12


def test_prox_update_is_the_minimiser_with_overlaps():
    # X+ minimises 1/2||X - Z||^2 + gamma/2 sum_q ||P_q - Q_q(X)||^2 (gradient zero), and reduces
    # to the identity for gamma = 0 and for tau = 0 (P_q = Q_q(Z))
    rng = np.random.default_rng(5)
    L, N, p, s, tau, gamma = 6, 21, 11, 5, 0.7, 0.35
    Z = rand_c(rng, L, N, N)
    X, _ = llr.llr_prox(Z, tau, gamma, p, s)
    grad = X - Z
    for y0 in llr.patch_corners(N, p, s):
        for x0 in llr.patch_corners(N, p, s):
            P = llr.svt(llr.casorati(Z, y0, x0, p), tau)
            Rq = llr.casorati(X, y0, x0, p) - P
            grad[:, y0:y0 + p, x0:x0 + p] += gamma * Rq.T.reshape(L, p, p)
    assert np.allclose(grad, 0, atol=1e-12)
    assert np.allclose(llr.llr_prox(Z, tau, 0.0, p, s)[0], Z, atol=1e-12)
    assert np.allclose(llr.llr_prox(Z, 0.0, gamma, p, s)[0], Z, atol=1e-12)


def test_step_without_regularisation_is_the_projected_gradient():
    rng = np.random.default_rng(6)
    L, N = 12, 16
    d = np.linalg.qr(rand_c(rng, L, 3))[0].T
    X, rhs = rand_c(rng, L, N, N), rand_c(rng, L, N, N)
    normal = lambda v: 0.5 * v
    Xn, Z = llr.llr_step(X, rhs, normal, d, mu=1.0, lam2=0.0, beta=0.2)
    assert np.allclose(Z, llr.project(X - (0.5 * X - rhs), d), atol=1e-12)
    assert np.allclose(Xn, Z, atol=1e-12)


def test_literal_eq23_update():
    """The printed Eq. (23) update X = (Z + g Q*(P)) / (1 + g): equal to the
    overlap-exact reading 25 when the patches do not overlap (stride = patch size: every voxel is
    covered once), and on an overlapping tiling equal to the formula written out by hand for a
    voxel covered by several patches."""
    rng = np.random.default_rng(9)
    L, N, p = 6, 8, 4
    Z = rand_c(rng, L, N, N)
    g = 0.7
    a, _ = llr.llr_prox(Z, 0.3, g, p, p, literal=True)
    b, _ = llr.llr_prox(Z, 0.3, g, p, p, literal=False)
    assert np.allclose(a, b, rtol=0, atol=1e-12)
    # overlapping (stride 2): voxel (3, 3) lies in the patches with corners {0, 2} x {0, 2}
    lit, _ = llr.llr_prox(Z, 0.3, g, p, 2, literal=True)
    exact, _ = llr.llr_prox(Z, 0.3, g, p, 2, literal=False)
    acc = np.zeros(L, complex)
    for y0 in (0, 2):
        for x0 in (0, 2):
            P = llr.svt(llr.casorati(Z, y0, x0, p), 0.3)
            acc += P[(3 - y0) * p + (3 - x0)]
    assert np.allclose(lit[:, 3, 3], (Z[:, 3, 3] + g * acc) / (1 + g), atol=1e-12)
    assert np.allclose(exact[:, 3, 3], (Z[:, 3, 3] + g * acc) / (1 + 4 * g), atol=1e-12)
    assert not np.allclose(lit, exact)

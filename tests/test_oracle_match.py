"""Pins of the dictionary-matching oracle (Eq. (5))."""
import numpy as np
import pytest

import synth.dictionary as sd
from oracle import match as om


def test_grid_is_the_papers_3336_atoms():
    # "... results in a dictionary with the size of 3336 x L"
    g = sd.t1t2_grid()
    assert g.shape == (3336, 2)
    assert np.all(g[:, 0] >= g[:, 1])
    assert g[:, 0].min() == 100 and g[:, 0].max() == 5000
    assert g[:, 1].min() == 20 and g[:, 1].max() == 1900


def brute(X, D, p=1):
    """Eq. (5) with explicit loops (no matrix product, no numpy argmax)."""
    V, L = X.shape
    K = D.shape[0]
    ks, rhos = [], []
    for v in range(V):
        best, bk, bc = -1.0, 0, 0j
        for k in range(K):
            c = 0j
            n2 = 0.0
            for l in range(L):
                c += D[k, l].conjugate() * X[v, l]
                n2 += abs(D[k, l]) ** 2
            s = abs(c) / (n2 ** 0.5 if p == 1 else n2)
            if s > best:          # strict: ties keep the lowest index
                best, bk, bc = s, k, c / n2
        ks.append(bk)
        rhos.append(max(bc.real, 0.0))
    return np.array(ks), np.array(rhos)


def test_matches_brute_force_loops():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((6, 9)) + 1j * rng.standard_normal((6, 9))
    D = rng.standard_normal((7, 9)) + 1j * rng.standard_normal((7, 9))
    for p in (1, 2):
        k, _, rho, _ = om.match(X, D, p=p)
        kb, rb = brute(X, D, p)
        assert np.array_equal(k, kb)
        assert np.allclose(rho, rb, rtol=1e-12, atol=1e-14)


def test_scaled_unit_atom_is_recovered():
    # equal-norm atoms: Eq. (5) is the normalised correlation, maximal (Cauchy-Schwarz) at the atom
    D = sd.surrogate_dictionary(64)[::37]
    D = D / np.linalg.norm(D, axis=1)[:, None]
    lut = np.arange(D.shape[0] * 2, dtype=np.float64).reshape(-1, 2)
    k0 = np.array([0, 5, 17, D.shape[0] - 1])
    X = 2.5 * D[k0]
    k, eta, rho, _ = om.match(X, D, lut)
    assert np.array_equal(k, k0)
    assert np.allclose(rho, 2.5, rtol=1e-12)
    assert np.array_equal(eta, lut[k0])


def test_negative_atom_clamps_pd_and_zero_voxel_takes_index_0():
    D = sd.surrogate_dictionary(32)[::100]
    D = D / np.linalg.norm(D, axis=1)[:, None]
    X = np.stack([-D[3], np.zeros(32, np.complex128)])
    k, _, rho, _ = om.match(X, D)
    assert k[0] == 3 and rho[0] == 0.0
    assert k[1] == 0 and rho[1] == 0.0


def test_denominator_reading():
    # d_1 = 0.5 d_0 and x = d_0.  Printed Eq. (5) (p = 2): scores 1 and 2 -> picks d_1, the
    # half-norm copy.  Reading 21 (p = 1): scores ||d_0|| for both -> tie -> lowest index d_0.
    # rho = Re<d_k, x>/||d_k||^2 in both cases.
    d = np.exp(1j * np.linspace(0, 3, 16))
    D = np.stack([d, 0.5 * d])
    k, _, rho, score = om.match(d[None, :], D, p=2)
    assert k[0] == 1 and np.allclose(score[0], [1.0, 2.0]) and np.isclose(rho[0], 2.0)
    k, _, rho, score = om.match(d[None, :], D, p=1)
    assert k[0] == 0 and np.allclose(score[0], [4.0, 4.0]) and np.isclose(rho[0], 1.0)


def test_scaled_atoms_of_the_pd1_dictionary_are_recovered():
    # atoms with PD 1 (different norms): p = 1 returns the generating atom, p = 2 does not
    D = sd.surrogate_dictionary(200)
    X, k0, rho0 = sd.voxel_fingerprints(D, 40)
    k, _, rho, _ = om.match(X, D, p=1)
    assert np.mean(k == k0) >= 0.95          # exact up to near-duplicate atoms
    assert np.allclose(rho[k == k0], rho0[k == k0], rtol=1e-10)
    k2, _, _, _ = om.match(X, D, p=2)
    assert np.mean(k2 == k0) < 0.5


def test_length_mismatch_is_rejected():
    with pytest.raises(ValueError):
        om.match(np.zeros((2, 5), np.complex128), np.ones((3, 4), np.complex128))


def test_noisy_fingerprints_recover_the_atom_neighbourhood():
    # with 1 % noise the matched (T1, T2) stay at or next to the true atom on the paper's grid
    D = sd.surrogate_dictionary(200)
    X, k0, rho0 = sd.voxel_fingerprints(D, 40, noise=0.01)
    g = sd.t1t2_grid()
    k, eta, rho, _ = om.match(X, D, g)
    rel = np.abs(eta - g[k0]) / g[k0]
    assert np.median(rel) < 0.05
    assert np.all(rho >= 0)

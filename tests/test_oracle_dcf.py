"""Pins of the density-compensation oracle (Pipe-Menon, reading 23)."""
import numpy as np

import synth
from oracle import dcf as od
from oracle.kb import kb_kernel
from oracle.nufft import GridParams


def brute_phi_phit(w, k, N, W):
    """(Phi Phi^T w)_j = sum_i w_i sum_m phi(u_j - m) phi(u_i - m), m over the wrapped grid, with
    explicit loops over point pairs and over the shared grid cells (no bincount, no tap arrays)."""
    gp = GridParams(N, W)
    G = gp.G
    u = G * np.asarray(k, np.float64)

    def cells(uj):   # the W x W grid cells of a point with their weights, as a dict
        out = {}
        m0 = np.floor(uj - W / 2.0).astype(int) + 1
        for ty in range(W):
            for tx in range(W):
                my, mx = m0[1] + ty, m0[0] + tx
                out[(my % G, mx % G)] = out.get((my % G, mx % G), 0.0) + \
                    float(kb_kernel(uj[1] - my, W, gp.beta) * kb_kernel(uj[0] - mx, W, gp.beta))
        return out

    C = [cells(uj) for uj in u]
    res = np.zeros(len(k))
    for j in range(len(k)):
        for i in range(len(k)):
            res[j] += w[i] * sum(v * C[i].get(m, 0.0) for m, v in C[j].items())
    return res


def test_phi_phit_matches_brute_force():
    rng = np.random.default_rng(4)
    k = rng.uniform(-0.5, 0.5, size=(40, 2))
    k[:5] = [[0.5, 0.5], [-0.5, 0.0], [0.49, -0.5], [0.0, 0.0], [0.01, 0.02]]   # wrap + centre
    w = rng.uniform(0.5, 2.0, size=40)
    gp = GridParams(16, 6)
    assert np.allclose(od.phi_phit(w, k, gp), brute_phi_phit(w, k, 16, 6), rtol=1e-12)


def test_cartesian_weights_are_constant_fixed_point():
    # points on the N-grid (every second cell of the sigma = 2 grid): Phi Phi^T 1 is the same
    # constant c at every point (shift invariance), so w = 1/c after one iteration and stays there
    N, W = 16, 6
    k = synth.cartesian_trajectory(N)[0].astype(np.float64)
    gp = GridParams(N, W)
    c = od.phi_phit(np.ones(len(k)), k, gp)
    assert np.allclose(c, c[0], rtol=1e-12)
    w1 = od.pipe_menon(k, N, W, n_iter=1)
    w5 = od.pipe_menon(k, N, W, n_iter=5)
    assert np.allclose(w1, 1.0 / c[0], rtol=1e-12) and np.allclose(w5, w1, rtol=1e-12)


def test_converges_to_the_fixed_point_on_the_spiral():
    cfg = synth.get_config("pr1")
    k = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)[0].astype(np.float64)
    gp = GridParams(cfg.N, cfg.W)
    # Pipe-Menon approaches Phi Phi^T w = 1 in the mean and then stalls (RMS ~1 %): pin the
    # decrease of the RMS residual and its level, and positivity
    res = []
    for n in (1, 4, 16):
        w = od.pipe_menon(k, cfg.N, cfg.W, n_iter=n)
        res.append(np.sqrt(np.mean((od.phi_phit(w, k, gp) - 1.0) ** 2)))
        assert np.all(w > 0)
    assert res[0] > res[1] > res[2] and res[2] < 0.01


def test_radial_weights_grow_with_radius():
    # radial spokes: sample density ~ 1/|k|, so the weights grow ~ |k| away from the centre
    M, S = 64, 32
    r = (np.arange(M) - M / 2 + 0.5) / M
    ang = np.pi * np.arange(S) / S
    k = np.stack([np.outer(np.cos(ang), r).ravel(), np.outer(np.sin(ang), r).ravel()], axis=1)
    w = od.pipe_menon(k, 32, 6, n_iter=30)
    kr = np.linalg.norm(k, axis=1)
    mid = (kr > 0.1) & (kr < 0.4)
    ratio = w[mid] / kr[mid]
    assert np.std(ratio) / np.mean(ratio) < 0.15
    assert w[kr > 0.3].mean() > 2.5 * w[(kr > 0.05) & (kr < 0.12)].mean()

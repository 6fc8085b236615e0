"""Pins for oracle/kb.py: the Kaiser-Bessel kernel and its deapodization (SURVEY.md §8(c) pins)."""
import os

import numpy as np
import pytest
from scipy import integrate

from oracle.kb import kb_beta, kb_kernel, kb_deapod_analytic, kb_deapod_discrete

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_i0_matches_textbook_table():
    """np.i0 (the Bessel routine the kernel uses) vs Abramowitz & Stegun Table 9.8 values."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "i0_table.txt")) if l.strip() and not l.startswith("#")]
    for xs, vs in rows:
        x, v = float(xs), float(vs)
        assert abs(np.i0(x) - v) <= 1e-9 * max(1.0, abs(v)), (x, np.i0(x), v)


def test_i0_series_definition():
    """I0(x) = sum_k (x^2/4)^k / (k!)^2 (closed form) at the kernel's largest argument beta(W=8)."""
    import math
    for x in (kb_beta(6, 2.0), kb_beta(8, 2.0), 0.3):
        s = sum((x * x / 4.0) ** k / math.factorial(k) ** 2 for k in range(80))
        assert abs(np.i0(x) - s) <= 1e-13 * s


@pytest.mark.parametrize("W", [4, 6, 8])
def test_kernel_shape(W):
    beta = kb_beta(W, 2.0)
    assert kb_kernel(0.0, W, beta) == 1.0                        # reading #7: phi(0) = 1
    u = np.linspace(-W / 2 + 1e-9, W / 2 - 1e-9, 101)
    assert np.array_equal(kb_kernel(u, W, beta), kb_kernel(-u, W, beta))   # even
    assert np.all(kb_kernel(u, W, beta) > 0)
    assert kb_kernel(W / 2.0, W, beta) == 0.0                    # reading #6: open support
    assert kb_kernel(-W / 2.0, W, beta) == 0.0
    assert kb_kernel(W / 2.0 + 0.3, W, beta) == 0.0
    # monotone decreasing in |u|
    up = np.linspace(0, W / 2 - 1e-6, 200)
    assert np.all(np.diff(kb_kernel(up, W, beta)) < 0)


def test_beta_positive_and_increasing():
    b = [kb_beta(W, 2.0) for W in (4, 6, 8)]
    assert 0 < b[0] < b[1] < b[2]


@pytest.mark.parametrize("W", [4, 6, 8])
def test_analytic_deapod_is_kernel_fourier_transform(W):
    """psi(n) = int phi(u) cos(2 pi u n / G) du (numerical quadrature, independent of the closed form)."""
    G, beta = 64, kb_beta(W, 2.0)
    n = np.arange(-16, 16)
    psi = kb_deapod_analytic(n, G, W, beta)
    for ni, p in zip(n, psi):
        q, _ = integrate.quad(lambda u: kb_kernel(u, W, beta) * np.cos(2 * np.pi * u * ni / G),
                              -W / 2, W / 2, epsabs=0, epsrel=1e-13, limit=200)
        assert abs(p - q) <= 1e-12 * abs(q), (ni, p, q)


def test_analytic_deapod_sin_branch():
    """Beyond the sinh/sin switch point the closed form must still equal the quadrature."""
    W, G = 6, 16
    beta = kb_beta(W, 2.0)
    n0 = beta * G / (np.pi * W)            # radicand zero
    for ni in (np.floor(n0) + 1, np.floor(n0) + 3):
        q, _ = integrate.quad(lambda u: kb_kernel(u, W, beta) * np.cos(2 * np.pi * u * ni / G), -W / 2, W / 2,
                              epsabs=1e-15, epsrel=1e-12, limit=200)
        p = kb_deapod_analytic(np.array([ni]), G, W, beta)[0]
        assert abs(p - q) <= 1e-10 * max(abs(q), 1e-3)


def test_discrete_deapod_is_sampled_kernel_dft():
    """psi_d(n) equals the G-point DFT of the kernel sampled at integers (numpy.fft)."""
    W, G = 6, 64
    beta = kb_beta(W, 2.0)
    d = np.arange(G)
    dd = np.where(d < G // 2, d, d - G)
    h = kb_kernel(dd.astype(float), W, beta)
    ref = np.fft.fft(h).real
    n = np.arange(-G // 2, G // 2)
    assert np.allclose(kb_deapod_discrete(n, G, W, beta), ref[n % G], rtol=0, atol=1e-13)

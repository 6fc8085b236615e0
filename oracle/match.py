"""Float64 oracle of the dictionary-matching operator Phi_D (Eqs. (4)-(5)).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).  Written from the paper:

    k      = argmax_k |<d_k, x>| / ||d_k||_2^p        (ties: the lowest index)
    eta    = LUT[k]
    rho    = max{ Re<d_k, x> / ||d_k||_2^2 , 0 }

with <d, x> = sum_l conj(d_l) x_l.  Eq. (5) prints p = 2 while the atoms carry
proton density 1 and therefore different norms; with p = 2 the argmax prefers
low-norm atoms and does not return "the best matching entry" (a scaled atom x = rho d_k is not
matched to d_k; tests/test_oracle_match.py shows it).  Reading 21: p = 1, the
normalised correlation of the standard MRF template match, which recovers scaled atoms by
Cauchy-Schwarz; for atoms of equal norm both readings coincide.  rho keeps the printed ||d||^2.
A matrix product is the one library step.
"""
from __future__ import annotations

import numpy as np


def correlations(X: np.ndarray, D: np.ndarray) -> np.ndarray:
    """c[v, k] = <d_k, x_v> = sum_l conj(D[k, l]) X[v, l]  ([V][K] complex128)."""
    return np.asarray(X, np.complex128) @ np.conj(np.asarray(D, np.complex128)).T


def match(X: np.ndarray, D: np.ndarray, lut: np.ndarray | None = None, p: int = 1):
    """Phi_D (Eq. 5): returns (k [V] int64, eta [V][P] or None, rho [V] float64, score [V][K])."""
    X = np.atleast_2d(np.asarray(X, np.complex128))
    D = np.asarray(D, np.complex128)
    if X.shape[1] != D.shape[1]:
        raise ValueError("temporal length of the data and the atoms differ")
    c = correlations(X, D)
    n2 = np.sum(np.abs(D) ** 2, axis=1)
    score = np.abs(c) / (np.sqrt(n2) if p == 1 else n2)[None, :]
    k = np.argmax(score, axis=1)                      # first maximum = lowest index
    ck = c[np.arange(X.shape[0]), k]
    rho = np.maximum(ck.real / n2[k], 0.0)
    eta = None if lut is None else np.asarray(lut)[k]
    return k, eta, rho, score

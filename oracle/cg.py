"""Conjugate gradient on (A^H A + mu I) x = A^H y + mu z (oracle, float64).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The paper's data term is 1/2 ||A X - b||_F^2 (Eq. (12), Alg. 1) and its
gradient A*(A X - b) (Eq. (15)); BASELINE.json's north_star asks for the exact
data-consistency (proximal) form of the same term, a CG solve of (A^H A + mu I) x = b.  The
iteration below is SURVEY.md §8(c)(ii) step 7, i.e. textbook CG (Hestenes-Stiefel) written out:

    rhs = A^H y + mu z;  r0 = rhs - H x0;  p0 = r0;  rho0 = <r0, r0>
    for k < n_iter:
        q = H p;  alpha = rho_k / Re<p, q>;  x += alpha p;  r -= alpha q;  rho_{k+1} = <r, r>
        if tol > 0 and sqrt(rho_{k+1}/rho0) < tol: stop
        p = r + (rho_{k+1}/rho_k) p

with <a, b> = sum over ALL frames (and all ranks) of conj(a) b (reading #16).  ``dot`` may be
replaced by a distributed inner product (tests use torch.distributed/gloo).
"""
from __future__ import annotations

import numpy as np


def vdot(a, b) -> complex:
    return complex(np.vdot(np.asarray(a).ravel(), np.asarray(b).ravel()))


def cg(H, rhs, x0, n_iter: int, tol: float = 0.0, dot=vdot):
    """Returns (x, history) with history[k] = sqrt(rho_k) (residual norm), len = iterations + 1."""
    x = np.array(x0, dtype=np.complex128, copy=True)
    r = np.asarray(rhs, dtype=np.complex128) - H(x)
    p = r.copy()
    rho = dot(r, r).real
    rho0 = rho
    hist = [np.sqrt(rho)]
    if rho0 == 0.0:
        return x, hist
    for _ in range(n_iter):
        q = H(p)
        pq = dot(p, q).real
        if not pq > 0.0:
            raise FloatingPointError("CG breakdown: Re<p, Hp> <= 0")
        alpha = rho / pq
        x += alpha * p
        r -= alpha * q
        rho_new = dot(r, r).real
        hist.append(np.sqrt(rho_new))
        if tol > 0.0 and np.sqrt(rho_new / rho0) < tol:
            break
        p = r + (rho_new / rho) * p
        rho = rho_new
    return x, hist


def dc_rhs(adjoint_y, z, mu):
    """rhs = A^H y + mu z (z = None => 0), SURVEY.md §8(a) row a8."""
    rhs = np.asarray(adjoint_y, dtype=np.complex128)
    if z is not None:
        rhs = rhs + mu * np.asarray(z, dtype=np.complex128)
    return rhs


def krylov_projection(Hmat, rhs, x0, n: int):
    """n-step CG iterate as a Galerkin projection: x_n = x0 + V (V^H H V)^{-1} V^H r0.

    V spans the Krylov space K_n(H, r0), built by Arnoldi with full re-orthogonalisation (not raw
    matrix powers).  For Hermitian positive definite H, CG's n-th iterate equals this projection
    (the defining property of CG).  Dense, float64; for tiny pins only.
    """
    Hmat = np.asarray(Hmat, dtype=np.complex128)
    r0 = np.asarray(rhs, dtype=np.complex128) - Hmat @ x0
    V = np.zeros((len(r0), n), dtype=np.complex128)
    v = r0 / np.linalg.norm(r0)
    for i in range(n):
        for _ in range(2):
            v = v - V[:, :i] @ (V[:, :i].conj().T @ v)
        V[:, i] = v / np.linalg.norm(v)
        v = Hmat @ V[:, i]
    T = V.conj().T @ Hmat @ V
    return x0 + V @ np.linalg.solve(T, V.conj().T @ r0)

"""Float64 oracle of Algorithm 1 of the paper: the MS-LLR reconstruction loop.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).  SURVEY.md §8(f) f2 ("Eq. 23 update, cost and
stop rule").  Written from the pseudocode, line by line:

    X^0 = A^* b,  M^0 = Phi_D(X^0),  L^0
    for n = 1 .. N_max:
        Z^n (Eq. 15), P^n (Eq. 20), X^n (Eq. 21)
        cost(n) = 1/2 ||A X - b||_F^2 + lambda_1 Tr(Q(X) L Q(X)^H)
                  + lambda_2 sum_i ||Q_{q_i}(X)||_*
        if cost(n-1)/cost(n) - 1 < 1e-5: break
        M^{n+1} = Phi_D(X^n);  L^{n+1} (Eq. 11);  lambda_1^{n+1} = lambda_1^0 max(L^{n+1})
                                                                              
    output X^, M^ = Phi_D(X^)

Readings: 27 -- the stop test starts at n = 2 (cost(0) is not defined by the
pseudocode); lambda_1 = 0 skips the maps inside the loop (the LLR-only reconstruction);
Phi_D = ``oracle.match`` (reading 21), the maps of the Laplacian are (T1, T2, PD) (reading 26);
the step uses the lambda_1 and L in force at iteration n, and so does cost(n).
"""
from __future__ import annotations

import numpy as np

from . import llr as ol
from . import manifold as om
from . import match as omatch
from . import nufft as on


def cost(X, b, A, lam1: float, lam2: float, lap=None, p: int = 11, s: int = 5):
    """cost(n) of Algorithm 1 at X [L][N][N]: returns (total, (data, manifold trace, nuclear sum)).
    A(X) -> k-space [L][C][M]; lap: the Laplacian (None -> the trace term is 0)."""
    X = np.asarray(X, np.complex128)
    L, N, _ = X.shape
    r = A(X) - np.asarray(b, np.complex128)
    data = 0.5 * float(np.sum(np.abs(r) ** 2))
    trace = 0.0 if lap is None else om.penalty(X, lap, N, p, s)
    nuc = 0.0
    cs = ol.patch_corners(N, p, s)
    for y0 in cs:
        for x0 in cs:
            nuc += float(np.linalg.svd(ol.casorati(X, y0, x0, p), compute_uv=False).sum())
    return data + lam1 * trace + lam2 * nuc, (data, trace, nuc)


def maps_of(X, D, lut, match_p: int = 1):
    """Phi_D(X) for X [L][N][N]: (k [V], eta [V][P], rho [V]) and the map stack (T1, T2, PD) [3][N][N].
    match_p = 2: Eq. (5)'s printed ||d||^2 denominator (reading 21 uses ||d||)."""
    L, N, _ = X.shape
    k, eta, rho, _ = omatch.match(np.asarray(X).reshape(L, -1).T, D, lut, p=match_p)
    m = np.stack([eta[:, 0].reshape(N, N), eta[:, 1].reshape(N, N), rho.reshape(N, N)])
    return (k, eta, rho), m


def solve(b, traj, D, lut, d, mu: float, lam1_0: float, lam2: float, beta: float, max_iter: int,
          tol: float = 1e-5, W: int = 6, N: int | None = None, p: int = 11, s: int = 5,
          sigma2: float | None = None, workers: int = 1, op: str = "grid", coils=None, literal_update: bool = False,
          raw_maps: bool = False, match_p: int = 1):
    """Algorithm 1.  b [L][C][M] k-space, traj [R][M][2], D [K][L] atoms, lut [K][2] (T1, T2),
    d [r][L] the basis of P_S, coils [C][N][N] or None (A = F_u C).  op = "grid":
    A is the KB gridding NUFFT; op = "nudft": A is the plain definition (the direct non-uniform DFT).
    The printed-form switches (readings 21, 25, 26): literal_update -> Eq. (21)'s scalar
    1 + mu lambda2 beta denominator; raw_maps -> Eq. (8) on the raw maps; match_p = 2 -> Eq. (5)'s
    ||d||^2 denominator in Phi_D.  Returns dict(x, k, eta, rho, iters, cost, lambda1)."""
    b = np.asarray(b, np.complex128)
    S = coils
    if op == "nudft":
        A = lambda X: on.nudft_forward(X, traj, S)
        normal = lambda X: on.nudft_adjoint(on.nudft_forward(X, traj, S), traj, S, N)
        rhs = on.nudft_adjoint(b, traj, S, N)
    else:
        A = lambda X: on.forward(X, traj, S, W, workers=workers)
        normal = lambda X: on.normal(X, traj, S, W, workers=workers)
        rhs = on.adjoint(b, traj, S, N, W, workers=workers)           # A^* b
    X = rhs.copy()                                                     # X^0
    lam1, lap = 0.0, None

    def update_maps(X):
        nonlocal lam1, lap
        _, m = maps_of(X, D, lut, match_p)
        Wm, _ = om.weights(m, N, p, s, sigma2, raw=raw_maps)
        lap = om.laplacian(Wm)
        lam1 = lam1_0 * float(lap.max())                              # lambda_1^0 max(L)

    if lam1_0 > 0:
        update_maps(X)                                                 # M^0, L^0
    costs, prev, it = [], 0.0, 0
    for n in range(1, max_iter + 1):
        X, _ = ol.llr_step(X, rhs, normal, d, mu, lam2, beta, p, s, lam1=lam1, lap=lap, literal=literal_update)
        c, _ = cost(X, b, A, lam1, lam2, lap, p, s)
        costs.append(c)
        it = n
        if n >= 2 and tol > 0 and prev / c - 1.0 < tol:
            break
        prev = c
        if lam1_0 > 0 and n < max_iter:
            update_maps(X)
    (k, eta, rho), _ = maps_of(X, D, lut, match_p)
    return {"x": X, "k": k, "eta": eta, "rho": rho, "iters": it, "cost": costs, "lambda1": lam1}

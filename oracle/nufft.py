"""Multi-frame, multi-coil non-Cartesian acquisition operator A = F_u C and its adjoint (oracle).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Conventions (SURVEY.md §8(c) readings #2-#7):
  * image x_l[iy, ix], centred indices n = (n_x, n_y) = (ix - N/2, iy - N/2), x fastest;
  * k in cycles/pixel, |k| <= 1/2 (k = +1/2 and -1/2 are the same sample);
  * forward exponent e^{-i 2 pi k.n}, adjoint e^{+i 2 pi k.n};
  * orthonormal scale s = 1/N, so a full Cartesian A is unitary;
  * frame l samples interleaf ``frame_interleaf[l]`` of ``traj`` [R][M][2];
  * coils [C][N][N] or None (S = 1).

Shapes: x [L][N][N] complex, y [L][C][M] complex.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.fft as sfft

from .kb import kb_beta, kb_kernel, deapod


def _coils(S, N):
    if S is None:
        return np.ones((1, N, N), dtype=np.complex128)
    return np.asarray(S, dtype=np.complex128)


def _centred(N):
    return np.arange(N, dtype=np.float64) - N // 2


# ============================================================================ (i) the definition
def nudft_forward_frame(x, S, k) -> np.ndarray:
    """y[c, j] = (1/N) sum_n S_c[n] x[n] exp(-i 2 pi (kx_j n_x + ky_j n_y)).

    PAPER.md:56-60 (Eq. (1) ``data_ac``: b = A X, A = F_u C, per coil and frame) with the
    conventions above; SPEC.md:274 (coil multiply -> transform -> sample).  Direct sum.
    """
    x = np.asarray(x, dtype=np.complex128)
    N = x.shape[0]
    k = np.asarray(k, dtype=np.float64)
    n = _centred(N)
    ny, nx = np.meshgrid(n, n, indexing="ij")
    E = np.exp(-2j * np.pi * (k[:, 0, None] * nx.ravel()[None, :] + k[:, 1, None] * ny.ravel()[None, :]))
    Sx = (_coils(S, N) * x[None]).reshape(-1, N * N)
    return (Sx @ E.T) / N


def nudft_adjoint_frame(y, S, k, N: int) -> np.ndarray:
    """x[n] = (1/N) sum_c conj(S_c[n]) sum_j y[c, j] exp(+i 2 pi (kx_j n_x + ky_j n_y)).

    The exact adjoint A* of ``nudft_forward_frame``.  Direct sum.
    """
    y = np.asarray(y, dtype=np.complex128)
    k = np.asarray(k, dtype=np.float64)
    n = _centred(N)
    ny, nx = np.meshgrid(n, n, indexing="ij")
    E = np.exp(+2j * np.pi * (nx.ravel()[:, None] * k[None, :, 0] + ny.ravel()[:, None] * k[None, :, 1]))
    per_coil = (E @ y.T).T.reshape(-1, N, N)          # [C][N][N]
    return (np.conj(_coils(S, N)) * per_coil).sum(0) / N


# ============================================================================ (ii) gridding NUFFT
class GridParams:
    """Per-transform constants of SURVEY.md §8(c)(ii) steps 1-3 (beta, psi, wrapped indices)."""

    def __init__(self, N: int, W: int, sigma: float = 2.0, deapod_mode: str = "analytic"):
        G = sigma * N
        if abs(G - round(G)) > 1e-9:
            raise ValueError("sigma*N must be an integer")
        self.N, self.W, self.sigma, self.G = N, W, sigma, int(round(G))
        self.beta = kb_beta(W, sigma)
        n = _centred(N)
        self.psi = deapod(n, self.G, W, self.beta, deapod_mode)   # [N], psi(n) for n = -N/2..N/2-1
        self.idx = (n.astype(np.int64)) % self.G                  # grid index of image index (wrap)


def taps(k, gp: GridParams):
    """Tap indices and weights of each point (reading #6).

    u = G k; m0 = floor(u - W/2) + 1; taps m = m0..m0+W-1 along each axis; weight phi(u - m).
    Returns (m_x, m_y) int64 [M][W] (not yet wrapped) and (w_x, w_y) float64 [M][W].
    """
    k = np.asarray(k, dtype=np.float64)
    u = gp.G * k                                   # [M][2]
    m0 = np.floor(u - gp.W / 2.0).astype(np.int64) + 1
    t = np.arange(gp.W, dtype=np.int64)
    mx = m0[:, 0, None] + t[None, :]
    my = m0[:, 1, None] + t[None, :]
    wx = kb_kernel(u[:, 0, None] - mx, gp.W, gp.beta)
    wy = kb_kernel(u[:, 1, None] - my, gp.W, gp.beta)
    return mx, my, wx, wy


def grid_forward_frame(x, S, k, gp: GridParams, stages: bool = False):
    """Gridding forward A for one frame, all coils.

    4.1 g[(n_y mod G), (n_x mod G)] = S_c[n] x[n] / (psi(n_x) psi(n_y) N), zero elsewhere;
    4.2 X = DFT_{GxG}(g), e^{-i 2 pi m n / G}, unnormalised;
    4.3 y_j = sum_{t_y, t_x} phi(u_y - m_y) phi(u_x - m_x) X[m_y mod G, m_x mod G].
    With ``stages`` also returns the intermediates (padded grid, row-FFT half grid, full grid).
    """
    x = np.asarray(x, dtype=np.complex128)
    N, G = gp.N, gp.G
    Sm = _coils(S, N)
    C = Sm.shape[0]
    mx, my, wx, wy = taps(k, gp)
    mxw, myw = mx % G, my % G
    scale = 1.0 / (gp.psi[:, None] * gp.psi[None, :] * N)
    y = np.empty((C, len(k)), dtype=np.complex128)
    st = {"g": [], "half": [], "X": []}
    for c in range(C):
        g = np.zeros((G, G), dtype=np.complex128)
        g[np.ix_(gp.idx, gp.idx)] = Sm[c] * x * scale                       # 4.1
        X = sfft.fft2(g, workers=1)                                           # 4.2
        vals = X[myw[:, :, None], mxw[:, None, :]]                            # [M][Wy][Wx]
        y[c] = (wy[:, :, None] * wx[:, None, :] * vals).sum((1, 2))           # 4.3
        if stages:
            st["g"].append(g)
            st["half"].append(sfft.fft(g[gp.idx, :], axis=1, workers=1))       # rows n_y, all G cols
            st["X"].append(X)
    if stages:
        return y, {key: np.stack(v) for key, v in st.items()}
    return y


def grid_adjoint_frame(y, S, k, gp: GridParams, stages: bool = False):
    """Gridding adjoint A^H for one frame: the exact transpose of ``grid_forward_frame``.

    SURVEY.md §8(c)(ii) step 5: 5.1 spread y with the same taps and weights; 5.2 unnormalised
    inverse DFT (e^{+i}); 5.3 crop at the same wrapped indices; 5.4 divide by psi psi N, multiply
    by conj(S_c) and sum over coils.  The spread uses ``numpy.bincount`` (sequential, deterministic;
    SPEC.md:320).
    """
    y = np.asarray(y, dtype=np.complex128)
    N, G = gp.N, gp.G
    Sm = _coils(S, N)
    C = Sm.shape[0]
    mx, my, wx, wy = taps(k, gp)
    flat = ((my % G)[:, :, None] * G + (mx % G)[:, None, :]).ravel()      # [M*Wy*Wx]
    w = (wy[:, :, None] * wx[:, None, :])                                  # [M][Wy][Wx]
    scale = 1.0 / (gp.psi[:, None] * gp.psi[None, :] * N)
    out = np.zeros((N, N), dtype=np.complex128)
    st = {"spread": [], "img": []}
    for c in range(C):
        contrib = (w * y[c][:, None, None]).ravel()
        Gs = (np.bincount(flat, weights=contrib.real, minlength=G * G)
              + 1j * np.bincount(flat, weights=contrib.imag, minlength=G * G)).reshape(G, G)   # 5.1
        img = sfft.ifft2(Gs, norm="forward", workers=1)                   # 5.2: sum e^{+i}, no 1/G^2
        crop = img[np.ix_(gp.idx, gp.idx)]                                # 5.3
        out += np.conj(Sm[c]) * crop * scale                              # 5.4
        if stages:
            st["spread"].append(Gs)
            st["img"].append(img)
    if stages:
        return out, {key: np.stack(v) for key, v in st.items()}
    return out


# ============================================================================ multi-frame operators
def _frames(n_frames, fn, workers):
    if workers <= 1:
        return [fn(l) for l in range(n_frames)]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(fn, range(n_frames)))


def _interleaf(traj, frame_interleaf, L, frame_offset=0):
    R = traj.shape[0]
    if frame_interleaf is None:
        return np.asarray([(frame_offset + l) % R for l in range(L)])
    return np.asarray(frame_interleaf)


def forward(x, traj, coils, W, sigma=2.0, frame_interleaf=None, deapod_mode="analytic",
            frame_offset=0, workers=1) -> np.ndarray:
    """A over all frames: x [L][N][N] -> y [L][C][M] (frame l uses interleaf frame_interleaf[l])."""
    x = np.asarray(x)
    L, N = x.shape[0], x.shape[1]
    gp = GridParams(N, W, sigma, deapod_mode)
    il = _interleaf(traj, frame_interleaf, L, frame_offset)
    return np.stack(_frames(L, lambda l: grid_forward_frame(x[l], coils, traj[il[l]], gp), workers))


def adjoint(y, traj, coils, N, W, sigma=2.0, frame_interleaf=None, deapod_mode="analytic",
            frame_offset=0, workers=1) -> np.ndarray:
    """A^H over all frames: y [L][C][M] -> x [L][N][N]."""
    y = np.asarray(y)
    L = y.shape[0]
    gp = GridParams(N, W, sigma, deapod_mode)
    il = _interleaf(traj, frame_interleaf, L, frame_offset)
    return np.stack(_frames(L, lambda l: grid_adjoint_frame(y[l], coils, traj[il[l]], gp), workers))


def normal(x, traj, coils, W, mu=0.0, sigma=2.0, frame_interleaf=None, deapod_mode="analytic",
           frame_offset=0, workers=1) -> np.ndarray:
    """(A^H A + mu I) x, frame by frame (PAPER.md:217 A*(A X))."""
    x = np.asarray(x)
    L, N = x.shape[0], x.shape[1]
    gp = GridParams(N, W, sigma, deapod_mode)
    il = _interleaf(traj, frame_interleaf, L, frame_offset)

    def one(l):
        xl = np.asarray(x[l], dtype=np.complex128)
        return grid_adjoint_frame(grid_forward_frame(xl, coils, traj[il[l]], gp), coils, traj[il[l]], gp) + mu * xl

    return np.stack(_frames(L, one, workers))


def nudft_forward(x, traj, coils, frame_interleaf=None, frame_offset=0) -> np.ndarray:
    x = np.asarray(x)
    il = _interleaf(traj, frame_interleaf, x.shape[0], frame_offset)
    return np.stack([nudft_forward_frame(x[l], coils, traj[il[l]]) for l in range(x.shape[0])])


def nudft_adjoint(y, traj, coils, N, frame_interleaf=None, frame_offset=0) -> np.ndarray:
    y = np.asarray(y)
    il = _interleaf(traj, frame_interleaf, y.shape[0], frame_offset)
    return np.stack([nudft_adjoint_frame(y[l], coils, traj[il[l]], N) for l in range(y.shape[0])])

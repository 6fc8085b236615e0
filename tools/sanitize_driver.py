"""Small invocations of every kernel family of libmrfnufft.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; SURVEY.md §5 race detection).

  compute-sanitizer --tool racecheck python tools/sanitize_driver.py [all|ops|cg|dict|llr]

Sizes are small (pr1: 32^2, cfg2-shaped 64^2 with several batches and both lanes, a stress-like
spiral with reduction slices) so the instrumented run finishes in minutes; each call is synced.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2310_05647_b200 import binding as mrf  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def ops():
    # pr1 (G = 64), a 64^2 multi-batch plan (G = 128, two lanes), a 128^2 stress-like spiral
    # (G = 256, cells with > 128 spread entries -> reduction slices) with 4 coils
    # plus the MRF shape (G = 512), G = 1024 and the W extremes 2 and 16
    cases = [("pr1", {}, None, 0), ("cfg2", dict(N=64, L=24), None, 8),
             ("stress", dict(N=128, L=6, C=4), 4, 3), ("mrf", dict(L=8), None, 4),
             ("cfg2", dict(N=512, L=2), None, 0), ("pr1", dict(W=2), None, 0), ("pr1", dict(W=16), None, 0)]
    for name, over, C, bf in cases:
        cfg = synth.get_config(name, **over)
        traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
        coils = synth.coil_maps(cfg.N, cfg.C, cfg.seed)
        x = dev(synth.images(cfg, list(range(cfg.L))))
        for normal in ("gridding", "toeplitz"):
            pl = mrf.Plan(cfg.N, traj, cfg.L, coils=coils, W=cfg.W, batch_frames=bf, normal=normal,
                          dcf=(normal == "gridding"))
            y = pl.forward(x)
            pl.adjoint(y)
            pl.normal(x, mu=cfg.mu)
            if normal == "gridding":
                pl.adjoint_dcf(y)
            pl.dc_cg(y, mu=cfg.mu, n_iter=3, zero_init=True)
            pl.dc_cg(y, mu=cfg.mu, n_iter=2, tol=1e-3)
            torch.cuda.synchronize()
            pl.close()
        print(f"ops {name} N={cfg.N} W={cfg.W}: ok", flush=True)


def dictionary():
    import synth.dictionary as sd
    grid = sd.t1t2_grid()[::23]
    for L in (40, 300):
        D = sd.surrogate_dictionary(L, grid)
        X, _, _ = sd.voxel_fingerprints(D, 700)
        dic = mrf.Dictionary(D, grid)
        dic.match(dev(X.T.astype(np.complex64)))
        d = dic.basis(0.9999, 32)
        u = dev((X @ d.conj().T).T.astype(np.complex64))
        dic.match_coef(u)
        torch.cuda.synchronize()
        dic.close()
    print("dict: ok", flush=True)


def llr():
    import synth.dictionary as sd
    N, L = 32, 40
    grid = sd.t1t2_grid()[::97]
    D = sd.surrogate_dictionary(L, grid)
    traj = synth.spiral_trajectory(512, 10, 8, 1.5)
    x = dev(synth.rank5_images(N, L, range(L), 7).astype(np.complex64))
    dic = mrf.Dictionary(D, grid)
    dic.basis(0.9999, 32)
    op = mrf.LLR(dic, N, 7, 3)
    for normal in ("gridding", "toeplitz"):
        pl = mrf.Plan(N, traj, L, W=6, normal=normal)
        b = pl.forward(x)
        for lam1 in (0.0, 1e-3):
            op.solve(dic, pl, b, mu=0.02, lam1=lam1, lam2=0.05, beta=0.5, max_iter=3, tol=0.0)
        torch.cuda.synchronize()
        pl.close()
    op.close(), dic.close()
    print("llr: ok", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    torch.cuda.set_device(0)
    if which in ("all", "ops"):
        ops()
    if which in ("all", "dict"):
        dictionary()
    if which in ("all", "llr"):
        llr()

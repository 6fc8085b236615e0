"""Time the MS-LLR outer step (mrf_llr_step) at the MRF size: 256 x 256 x 1000 frames, 2500
patches, with lambda_1 = 0 (LLR ablation) and with the manifold term (Laplacian from maps)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import synth.dictionary as sd  # noqa: E402
from paper_2310_05647_b200 import binding  # noqa: E402

cfg = synth.get_config("mrf")
traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
pl = binding.Plan(cfg.N, traj, cfg.L, W=cfg.W)
dic = binding.Dictionary(sd.surrogate_dictionary(cfg.L))
d = dic.basis(0.9999, 32)
op = binding.LLR(dic, cfg.N)
x = torch.from_numpy(synth.images(cfg)).cuda()
rhs = pl.adjoint(pl.forward(x))
xo = torch.empty_like(x)
maps = sd.parameter_maps(cfg.N, 3)
params = torch.from_numpy(np.ascontiguousarray(np.stack([maps[0].ravel(), maps[1].ravel()], 1))).float().cuda()
pdm = torch.from_numpy(np.ascontiguousarray(maps[2].ravel())).float().cuda()
op.laplacian(params, pdm)
torch.cuda.synchronize()
t0 = time.perf_counter()
s2, mdeg = op.laplacian(params, pdm)
torch.cuda.synchronize()
print(f"laplacian: {1e3 * (time.perf_counter() - t0):.1f} ms (sigma2 {s2:.3f}, max degree {mdeg:.1f})")


def timed(lam1):
    for _ in range(3):
        op.step(pl, rhs, rhs, x_out=xo, nuclear=False, lam1=lam1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        op.step(pl, rhs, rhs, x_out=xo, nuclear=False, lam1=lam1)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 5


print(f"llr step (lambda1 = 0): {timed(0.0):.3f} ms; ms-llr step (lambda1 > 0): {timed(0.1 * mdeg / 100):.3f} ms "
      f"(rank {d.shape[0]})")

# Algorithm 1 end to end (mrf_msllr_solve): per-iteration time = (T(5) - T(1)) / 4, where one
# iteration = step + cost + Phi_D + Laplacian update (lambda1 > 0)
lut = sd.t1t2_grid().astype(np.float32)
dic2 = binding.Dictionary(sd.surrogate_dictionary(cfg.L), lut)
dic2.basis(0.9999, 32)
op2 = binding.LLR(dic2, cfg.N)
b = pl.forward(x)
c, terms = op.cost(pl, xo, b, lam1=0.1, lam2=0.1)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    op.cost(pl, xo, b, lam1=0.1, lam2=0.1)
torch.cuda.synchronize()
print(f"cost: {1e3 * (time.perf_counter() - t0) / 5:.3f} ms (terms {terms})")


plt = binding.Plan(cfg.N, traj, cfg.L, W=cfg.W, normal="toeplitz")


def solve_ms(n, lam1, plan=None):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = op2.solve(dic2, plan or pl, b, mu=0.018, lam1=lam1, lam2=0.05, beta=0.5, max_iter=n, tol=0.0)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


solve_ms(1, 1e-3)
solve_ms(2, 1e-3, plt)
for plan, name in ((pl, "gridding plan"), (plt, "toeplitz plan (basis coordinates)")):
    for lam1 in (0.0, 1e-7):
        per = []
        for _ in range(2):
            t1, _ = solve_ms(1, lam1, plan)
            t11, out = solve_ms(11, lam1, plan)
            per.append((t11 - t1) / 10)
        print(f"msllr solve {name} lambda1_0={lam1}: {1e3 * min(per):.2f} ms per Algorithm-1 iteration "
              f"(T(1) = {1e3 * t1:.1f} ms, cost {['%.4g' % c for c in out['cost'][:4]]} ...)")

"""One MS-LLR solve in basis coordinates (Toeplitz plan, MRF size) bracketed by cudaProfilerStart /
Stop, for `ncu --profile-from-start off` launch lists: python tools/sub_profile.py [iters] [lam1_0]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import synth.dictionary as sd  # noqa: E402
from paper_2310_05647_b200 import binding  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 6
lam1 = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-7
cfg = synth.get_config("mrf")
traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
plt = binding.Plan(cfg.N, traj, cfg.L, W=cfg.W, normal="toeplitz")
dic = binding.Dictionary(sd.surrogate_dictionary(cfg.L), sd.t1t2_grid().astype(np.float32))
dic.basis(0.9999, 32)
op = binding.LLR(dic, cfg.N)
b = plt.forward(torch.from_numpy(synth.images(cfg)).cuda())
op.solve(dic, plt, b, mu=0.018, lam1=lam1, lam2=0.05, beta=0.5, max_iter=2, tol=0.0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
op.solve(dic, plt, b, mu=0.018, lam1=lam1, lam2=0.05, beta=0.5, max_iter=iters, tol=0.0)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"solve({iters}): {1e3 * (time.perf_counter() - t0):.2f} ms wall")

"""Small driver for ncu / compute-sanitizer: runs the operators of one workload a few times.

  python tools/prof_ops.py --workload mrf --frames 96 --reps 2 [--cg 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2310_05647_b200 import binding  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="mrf")
ap.add_argument("--frames", type=int, default=96)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--cg", type=int, default=0)
ap.add_argument("--ops", default="fwd,adj,normal")
a = ap.parse_args()
cfg = synth.get_config(a.workload)
L = min(a.frames, cfg.L)
traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
coils = synth.coil_maps(cfg.N, cfg.C, cfg.seed)
x = torch.from_numpy(synth.images(cfg, range(L))).cuda()
pl = binding.Plan(cfg.N, traj, L, coils=coils, W=cfg.W)
y = pl.forward(x)
for _ in range(a.reps):
    if "fwd" in a.ops:
        pl.forward(x, y=y)
    if "adj" in a.ops:
        pl.adjoint(y)
    if "normal" in a.ops:
        pl.normal(x, mu=0.01)
if a.cg:
    pl.dc_cg(y, mu=0.01, n_iter=a.cg)
torch.cuda.synchronize()
pl.close()
print("ok", L)

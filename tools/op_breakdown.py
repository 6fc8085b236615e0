"""Per-kernel-class device time of one operator (CUDA events inside the library).

  python tools/op_breakdown.py --workload mrf --normal toeplitz --op normal --reps 5
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
ap.add_argument("--normal", default="gridding")
ap.add_argument("--op", default="normal")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--frames", type=int, default=0)
ap.add_argument("--bf", type=int, default=0)
a = ap.parse_args()
cfg = synth.get_config(a.workload)
L = a.frames or cfg.L
traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
coils = synth.coil_maps(cfg.N, cfg.C, cfg.seed)
pl = binding.Plan(cfg.N, traj, L, coils=coils, W=cfg.W, normal=a.normal, batch_frames=a.bf)
x = torch.randn(pl.x_shape, dtype=torch.complex64, device="cuda")
out = torch.empty_like(x)
y = torch.randn(pl.y_shape, dtype=torch.complex64, device="cuda")
op = {"normal": lambda: pl.normal(x, mu=0.01, out=out), "forward": lambda: pl.forward(x, y=y),
      "adjoint": lambda: pl.adjoint(y, x=out), "cg": lambda: pl.dc_cg(y, mu=0.01, n_iter=10, x=out)}[a.op]
for _ in range(2):
    op()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.reps):
    op()
e.record()
torch.cuda.synchronize()
wall = s.elapsed_time(e) / a.reps
pl.profile(True)
for _ in range(a.reps):
    op()
torch.cuda.synchronize()
parts = {k: pl.profile_query(k) for k in binding.KERNEL_CLASSES}
pl.profile(False)
print(f"{a.workload} {a.normal} {a.op}: wall {wall:.3f} ms/op;",
      ", ".join(f"{k} {v[0] / a.reps:.3f} ms ({v[1] // a.reps} launches)" for k, v in parts.items() if v[1]))
pl.close()

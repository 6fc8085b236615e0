"""Time the LLR outer step (mrf_llr_step) at the MRF size: 256 x 256 x 1000 frames, 2500 patches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
for _ in range(3):
    op.step(pl, rhs, rhs, x_out=xo, nuclear=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    op.step(pl, rhs, rhs, x_out=xo, nuclear=False)
e.record()
torch.cuda.synchronize()
print(f"llr step: {s.elapsed_time(e) / 5:.3f} ms (rank {d.shape[0]})")

"""A/B timing of the MRF normal operator and the 10-iteration CG step for the library named by
MRF_LIB_PATH (default: the in-tree build); prints one line."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2310_05647_b200 import binding  # noqa: E402

cfg = synth.get_config("mrf")
traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
pl = binding.Plan(cfg.N, traj, cfg.L, W=cfg.W)
x = torch.from_numpy(synth.images(cfg, list(range(cfg.L)))).cuda()
y = pl.forward(x)
out = torch.empty_like(x)
xs = torch.empty_like(x)


def t(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


n = t(lambda: pl.normal(x, mu=cfg.mu, out=out), 20)
f = t(lambda: pl.forward(x, y=y), 20)
ad = t(lambda: pl.adjoint(y, x=out), 20)
st = t(lambda: pl.dc_cg(y, mu=cfg.mu, n_iter=10, x=xs, zero_init=True), 10)
print(f"{os.path.basename(os.environ.get('MRF_LIB_PATH', 'libmrfnufft.so'))}: normal {n:.3f} fwd {f:.3f} adj {ad:.3f} "
      f"cg-step {st:.2f} ms")

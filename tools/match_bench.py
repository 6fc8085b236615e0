"""Time mrf_dict_match on the MRF-sized problem (65536 voxels x 3336 atoms x 1000 frames) for
several voxel populations: noisy fingerprints, the rank-5 phantom series, the CG solution of the
bench workload, and white noise; prints ms, the filter GEMM share and the full-scan (overflow)
voxel count.  Optional: --ncu runs one match per population (for ncu --launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import synth.dictionary as sd  # noqa: E402
from paper_2310_05647_b200 import binding  # noqa: E402

L, V = 1000, 65536
g = sd.t1t2_grid()
D = sd.surrogate_dictionary(L, g)
dic = binding.Dictionary(D, g)
print("filter (Rf, beta, residual):", dic.filter_info())
cfg = synth.get_config("mrf")
pops = {}
X, _, _ = sd.voxel_fingerprints(D, V, noise=0.01)
pops["fingerprints"] = torch.from_numpy(np.ascontiguousarray(X.T.astype(np.complex64))).cuda()
del X
pops["rank5 phantom"] = torch.from_numpy(synth.images(cfg, list(range(L))).reshape(L, -1)).cuda()
traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
pl = binding.Plan(cfg.N, traj, L, W=cfg.W)
y = pl.forward(pops["rank5 phantom"].view(L, cfg.N, cfg.N))
xs, _ = pl.dc_cg(y, mu=cfg.mu, n_iter=10, zero_init=True)
pops["CG solution"] = xs.view(L, -1).clone()
pl.close()
pops["white noise"] = torch.randn(L, V, dtype=torch.complex64, device="cuda")
for name, x in pops.items():
    for _ in range(2):
        dic.match(x)
    torch.cuda.synchronize()
    ov = dic.overflow()
    dic.profile(True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    s.record()
    for _ in range(reps):
        dic.match(x)
    e.record()
    torch.cuda.synchronize()
    gm, gn = dic.profile_query()
    dic.profile(False)
    ms = s.elapsed_time(e) / reps
    print(f"{name:15s}: {ms:7.3f} ms per match, filter GEMMs {gm / max(gn, 1):.3f} ms, full-scan voxels {ov}")
dic.close()

"""Bitwise comparison of k_adj_cols' two-threads-per-transform variant (MRF_ADJ_T2=1) with the default,
on the MRF shape (adjoint, normal, CG) and a stress-like multi-coil plan; then timings."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2310_05647_b200 import binding

def plan(cfgname, L, t2, **kw):
    os.environ["MRF_ADJ_T2"] = "1" if t2 else "0"
    cfg = synth.get_config(cfgname)
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    coils = synth.coil_maps(cfg.N, cfg.C, 5) if cfg.C > 1 else None
    return cfg, binding.Plan(cfg.N, traj, L, W=cfg.W, coils=coils, **kw)

for name, L in (("mrf", 300), ("stress", 24), ("sense", 40)):
    outs = []
    for t2 in (0, 1):
        cfg, pl = plan(name, L, t2)
        g = torch.Generator(device="cpu").manual_seed(1)
        x = torch.view_as_complex(torch.randn(L, cfg.N, cfg.N, 2, generator=g)).cuda()
        y = pl.forward(x)
        a = pl.adjoint(y)
        n = pl.normal(x, mu=0.01)
        xs, _ = pl.dc_cg(y, mu=0.01, n_iter=4)
        outs.append((a.cpu(), n.cpu(), xs.cpu()))
        pl.close()
    same = [bool(torch.equal(torch.view_as_real(u), torch.view_as_real(v))) for u, v in zip(*outs)]
    print(name, "adjoint/normal/cg bitwise equal:", same, flush=True)
    assert all(same)

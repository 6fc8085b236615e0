"""One rank of a frame-sharded run of the library (launched by tests/test_gpu_multirank.py).

Every rank builds a plan over its contiguous frame block (paper_2310_05647_b200.sharding, the
block-diagonal operator of PAPER.md:60) and routes the plan's rank reductions through a gloo
all-reduce (mrf_plan_set_host_allreduce), so several ranks can share one GPU -- NCCL cannot
place two ranks on one device.  Rank 0 also runs the unsharded solve on one plan.  Results go to
``<out>/rank<k>.npz``; the test compares them.

  RANK=k WORLD_SIZE=n MASTER_ADDR=127.0.0.1 MASTER_PORT=p python tests/multirank_worker.py MODE OUT
  MODE: cg-<config>  (mrf_dc_cg, 10 iterations from x0 = 0, MRF_CG_ZERO_INIT)
        msllr        (mrf_msllr_solve, lambda_1 = 0, on mrf_llr_create_shard operators)
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2310_05647_b200 import binding  # noqa: E402
from paper_2310_05647_b200.sharding import frame_shard  # noqa: E402


def gloo_sum(buf: np.ndarray) -> None:
    dist.all_reduce(torch.from_numpy(buf), op=dist.ReduceOp.SUM)


def run_cg(name: str, rank: int, world: int, out: str) -> None:
    cfg = synth.get_config(name)
    L = min(cfg.L, 240)                     # enough frames for several batches per shard
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    coils = synth.coil_maps(cfg.N, cfg.C, cfg.seed)
    off, Ll = frame_shard(L, world, rank)
    res = {}
    x_sh = torch.from_numpy(synth.images(cfg, list(range(off, off + Ll)))).cuda()
    pl = binding.Plan(cfg.N, traj, Ll, coils=coils, W=cfg.W, frame_offset=off, batch_frames=32)
    pl.set_host_allreduce(gloo_sum)
    y = pl.forward(x_sh)
    x, info = pl.dc_cg(y, mu=cfg.mu, n_iter=cfg.cg_iters, zero_init=True)
    res["x"] = x.cpu().numpy()
    res["history"] = np.array(info["history"])
    res["alpha"] = np.array(info["alpha"])
    res["beta"] = np.array(info["beta"])
    pl.close()
    if rank == 0:                           # the unsharded solve on one plan (no reduction)
        xa = torch.from_numpy(synth.images(cfg, list(range(L)))).cuda()
        pa = binding.Plan(cfg.N, traj, L, coils=coils, W=cfg.W, batch_frames=32)
        ya = pa.forward(xa)
        x1, i1 = pa.dc_cg(ya, mu=cfg.mu, n_iter=cfg.cg_iters, zero_init=True)
        res["x_full"] = x1.cpu().numpy()
        res["history_full"] = np.array(i1["history"])
        res["alpha_full"] = np.array(i1["alpha"])
        pa.close()
    np.savez(os.path.join(out, f"rank{rank}.npz"), offset=off, **res)


def run_msllr(rank: int, world: int, out: str) -> None:
    import synth.dictionary as sd
    from oracle import nufft as on       # test infrastructure: the shared k-space b
    N, L, P, S, W = 32, 60, 7, 3, 6
    grid = sd.t1t2_grid()[::80]
    D = sd.surrogate_dictionary(L, grid)
    x_true = synth.rank5_images(N, L, range(L), 11)
    traj = synth.spiral_trajectory(512, 10, 8, 1.5)
    b = on.forward(x_true, traj, None, W).astype(np.complex64)
    off, Ll = frame_shard(L, world, rank)
    dic = binding.Dictionary(D, grid.astype(np.float32))
    dic.basis(0.9999, 32)
    kw = dict(mu=0.02, lam1=0.0, lam2=0.05, beta=0.5, max_iter=4, tol=0.0)
    op = binding.LLR.shard(dic, off, Ll, N, P, S)
    pl = binding.Plan(N, traj, Ll, W=W, frame_offset=off)
    pl.set_host_allreduce(gloo_sum)
    r = op.solve(dic, pl, torch.from_numpy(b[off:off + Ll]).cuda(), **kw)
    res = {"x": r["x"].cpu().numpy(), "index": r["index"].cpu().numpy(), "cost": np.array(r["cost"])}
    for o in (op, pl):
        o.close()
    if rank == 0:
        one, pa = binding.LLR(dic, N, P, S), binding.Plan(N, traj, L, W=W)
        r1 = one.solve(dic, pa, torch.from_numpy(b).cuda(), **kw)
        res.update(x_full=r1["x"].cpu().numpy(), index_full=r1["index"].cpu().numpy(), cost_full=np.array(r1["cost"]))
        one.close(), pa.close()
    dic.close()
    np.savez(os.path.join(out, f"rank{rank}.npz"), offset=off, **res)


def main() -> int:
    mode, out = sys.argv[1], sys.argv[2]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_DEVICE", "0")))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if mode.startswith("cg-"):
            run_cg(mode[3:], rank, world, out)
        elif mode == "msllr":
            run_msllr(rank, world, out)
        else:
            raise SystemExit(f"unknown mode {mode}")
        dist.barrier()
    finally:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

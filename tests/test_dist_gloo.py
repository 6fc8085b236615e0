"""World-size-2 gloo tests of the frame-sharded path.

The operator is block-diagonal over frames, so forward/adjoint/normal shard with no
communication; the CG solve needs the two global inner products per iteration.  These tests run
the oracle CG with ``torch.distributed`` all-reduce of the inner products (the same exchange the
CUDA path does with NCCL) and compare with the unsharded solve, and check the rank partition
helper that bench.py and the binding use.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2310_05647_b200.sharding import frame_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import nufft as on, cg as ocg
    cfg = synth.get_config("pr1")
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    off, cnt = frame_shard(cfg.L, world, rank)
    frames = range(off, off + cnt)
    x_true = synth.images(cfg, frames)
    y = on.forward(x_true, traj, None, cfg.W, frame_offset=off)

    def gdot(a, b):
        t = torch.tensor([complex(np.vdot(a.ravel(), b.ravel())).real,
                          complex(np.vdot(a.ravel(), b.ravel())).imag], dtype=torch.float64)
        dist.all_reduce(t)
        return complex(t[0].item(), t[1].item())

    H = lambda v: on.normal(v, traj, None, cfg.W, mu=cfg.mu, frame_offset=off)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, None, cfg.N, cfg.W, frame_offset=off), None, cfg.mu)
    x, hist = ocg.cg(H, rhs, np.zeros_like(rhs), cfg.cg_iters, dot=gdot)
    out_q.put((rank, off, x, hist))
    dist.barrier()
    dist.destroy_process_group()


def test_frame_shard_partition():
    for L in (1, 7, 8, 1000, 2000):
        for world in (1, 2, 3, 4, 8):
            parts = [frame_shard(L, world, r) for r in range(world)]
            assert parts[0][0] == 0
            for (o1, c1), (o2, _) in zip(parts, parts[1:]):
                assert o1 + c1 == o2
            assert sum(c for _, c in parts) == L
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1


def test_sharded_cg_equals_unsharded_gloo():
    from oracle import nufft as on, cg as ocg
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    x_sh = np.concatenate([r[2] for r in res])
    assert np.allclose(res[0][3], res[1][3], rtol=1e-13, atol=0)    # both ranks see the same scalars

    cfg = synth.get_config("pr1")
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    x_true = synth.images(cfg)
    y = on.forward(x_true, traj, None, cfg.W)
    H = lambda v: on.normal(v, traj, None, cfg.W, mu=cfg.mu)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, None, cfg.N, cfg.W), None, cfg.mu)
    x_ref, hist_ref = ocg.cg(H, rhs, np.zeros_like(rhs), cfg.cg_iters)
    assert np.linalg.norm(x_sh - x_ref) <= 1e-12 * np.linalg.norm(x_ref)
    assert np.allclose(res[0][3], hist_ref, rtol=1e-12, atol=0)

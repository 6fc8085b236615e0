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


# ------------------------------------------------------- frame-sharded LLR step
_LN, _LL, _LP, _LS = 16, 12, 5, 2     # N, L, patch, stride of the small LLR case


def _llr_case():
    from oracle import llr as ol
    rng = np.random.default_rng(41)
    traj = synth.spiral_trajectory(96, 4, 4, 1.5)
    t = rng.standard_normal((3, _LL)) + 1j * rng.standard_normal((3, _LL))
    amps = rng.standard_normal((3, _LN, _LN)) + 1j * rng.standard_normal((3, _LN, _LN))
    X = np.einsum("kl,kyx->lyx", t, amps) + 0.1 * (rng.standard_normal((_LL, _LN, _LN)) + 0j)
    rhs = rng.standard_normal((_LL, _LN, _LN)) + 1j * rng.standard_normal((_LL, _LN, _LN))
    D = np.concatenate([t, rng.standard_normal((6, _LL)) + 1j * rng.standard_normal((6, _LL))])
    d = ol.basis(D, 0.9999, 8)
    return traj, X, rhs, d


def _llr_worker(rank, world, port, out_q):
    """The decomposition mrf_llr_create_shard implements: each rank forms the projected gradient
    on its own frames, the coefficient partials Y_rank = Z_rank d_rank^dagger are all-reduced (the
    only exchange), every rank runs the patch SVT on the full Y (SVT(Q_q(Y d)) = SVT(Y_q) d for
    orthonormal rows of d), and expands the update on its own frames."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import llr as ol, nufft as on
    traj, X, rhs, d = _llr_case()
    off, cnt = frame_shard(_LL, world, rank)
    Xl, rl, dl = X[off:off + cnt], rhs[off:off + cnt], d[:, off:off + cnt]
    mu, lam2, beta = 0.02, 0.3, 0.5
    Z = Xl - mu * (on.normal(Xl, traj, None, 6, frame_offset=off) - rl)
    Yp = Z.reshape(cnt, -1).T @ np.conj(dl).T                           # [V][r] partial
    t = torch.from_numpy(np.stack([Yp.real, Yp.imag]))
    dist.all_reduce(t)
    Y = t[0].numpy() + 1j * t[1].numpy()
    Yi = Y.reshape(_LN, _LN, -1)
    acc = np.zeros_like(Yi)
    cnt_p = np.zeros((_LN, _LN))
    gamma = mu * lam2 * beta
    for y0 in ol.patch_corners(_LN, _LP, _LS):
        for x0 in ol.patch_corners(_LN, _LP, _LS):
            Yq = Yi[y0:y0 + _LP, x0:x0 + _LP].reshape(_LP * _LP, -1)
            acc[y0:y0 + _LP, x0:x0 + _LP] += ol.svt(Yq, 1.0 / beta).reshape(_LP, _LP, -1)
            cnt_p[y0:y0 + _LP, x0:x0 + _LP] += 1.0
    Xc = (Yi + gamma * acc) / (1.0 + gamma * cnt_p)[..., None]
    out_q.put((rank, np.einsum("yxr,rl->lyx", Xc, dl)))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_llr_step_equals_unsharded_gloo():
    from oracle import llr as ol, nufft as on
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_llr_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    x_sh = np.concatenate([r[1] for r in res])
    traj, X, rhs, d = _llr_case()
    ref, _ = ol.llr_step(X, rhs, lambda v: on.normal(v, traj, None, 6), d, 0.02, 0.3, 0.5, _LP, _LS)
    assert np.linalg.norm(x_sh - ref) <= 1e-10 * np.linalg.norm(ref)

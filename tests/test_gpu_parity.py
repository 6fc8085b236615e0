"""GPU parity: the sm_100a path through the C-ABI vs the float64 oracle, element by element.

Tolerances (BASELINE.json north_star): relative L2 <= 1e-5 per operator,
<= 1e-4 on the CG solution; adjoint identity of the fp32 path <= 1e-6 normalised.
All inputs come from ``synth`` (seeded); every expected value comes from ``oracle``.
"""
import os

import numpy as np
import pytest
import torch

import synth
from oracle import nufft as on
from oracle import cg as ocg

pytestmark = pytest.mark.gpu

OP_TOL = 1e-5
CG_TOL = 1e-4
WORKERS = max(1, min(8, len(os.sched_getaffinity(0))))


@pytest.fixture(scope="module")
def mrf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_05647_b200 import binding
    return binding


def rel(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def setup(name, frames=None, **over):
    cfg = synth.get_config(name, **over)
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    coils = synth.coil_maps(cfg.N, cfg.C, cfg.seed)
    frames = list(range(cfg.L)) if frames is None else list(frames)
    x = synth.images(cfg, frames)
    return cfg, traj, coils, frames, x


def plan_for(mrf, cfg, traj, coils, frames, **kw):
    fil = synth.frame_interleaf(frames, cfg.R)
    return mrf.Plan(cfg.N, traj, len(frames), coils=coils, W=cfg.W, frame_interleaf=fil, **kw)


# ------------------------------------------------------------------------ operators
@pytest.mark.parametrize("name", ["pr1", "cfg2"])
def test_operators_vs_oracle(mrf, name):
    cfg, traj, coils, frames, x = setup(name)
    fil = synth.frame_interleaf(frames, cfg.R)
    pl = plan_for(mrf, cfg, traj, coils, frames)
    y_gpu = host(pl.forward(dev(x)))
    y_ref = on.forward(x, traj, coils, cfg.W, frame_interleaf=fil, workers=WORKERS)
    assert rel(y_gpu, y_ref) <= OP_TOL
    yr = synth.random_kspace(cfg.C, cfg.M, frames, cfg.seed)
    xa_gpu = host(pl.adjoint(dev(yr)))
    xa_ref = on.adjoint(yr, traj, coils, cfg.N, cfg.W, frame_interleaf=fil, workers=WORKERS)
    assert rel(xa_gpu, xa_ref) <= OP_TOL
    xn_gpu = host(pl.normal(dev(x), mu=cfg.mu))
    xn_ref = on.normal(x, traj, coils, cfg.W, mu=cfg.mu, frame_interleaf=fil, workers=WORKERS)
    assert rel(xn_gpu, xn_ref) <= OP_TOL


def test_operators_sense_coils_subset(mrf):
    """SENSE (8 coils, Gaussian-blob maps) on a frame subset that spans two batches."""
    cfg, traj, coils, frames, x = setup("sense", frames=range(40, 52))
    fil = synth.frame_interleaf(frames, cfg.R)
    pl = plan_for(mrf, cfg, traj, coils, frames, batch_frames=5)
    y_gpu = host(pl.forward(dev(x)))
    y_ref = on.forward(x, traj, coils, cfg.W, frame_interleaf=fil, workers=WORKERS)
    assert rel(y_gpu, y_ref) <= OP_TOL
    xa_gpu = host(pl.adjoint(dev(y_ref.astype(np.complex64))))
    xa_ref = on.adjoint(y_ref.astype(np.complex64), traj, coils, cfg.N, cfg.W, frame_interleaf=fil, workers=WORKERS)
    assert rel(xa_gpu, xa_ref) <= OP_TOL
    xn_gpu = host(pl.normal(dev(x), mu=cfg.mu))
    xn_ref = on.normal(x, traj, coils, cfg.W, mu=cfg.mu, frame_interleaf=fil, workers=WORKERS)
    assert rel(xn_gpu, xn_ref) <= OP_TOL


def test_operators_stress_subset(mrf):
    """Stress spiral (p = 4, W = 8, 16 coils, M = 4096) on 3 frames: worst spreading contention."""
    cfg, traj, coils, frames, x = setup("stress", frames=[0, 37, 1999])
    fil = synth.frame_interleaf(frames, cfg.R)
    pl = plan_for(mrf, cfg, traj, coils, frames)
    y_gpu = host(pl.forward(dev(x)))
    y_ref = on.forward(x, traj, coils, cfg.W, frame_interleaf=fil, workers=WORKERS)
    assert rel(y_gpu, y_ref) <= OP_TOL
    xa_gpu = host(pl.adjoint(dev(y_ref.astype(np.complex64))))
    xa_ref = on.adjoint(y_ref.astype(np.complex64), traj, coils, cfg.N, cfg.W, frame_interleaf=fil, workers=WORKERS)
    assert rel(xa_gpu, xa_ref) <= OP_TOL


def test_normal_stress_subset(mrf):
    """The stress normal operator A^H A + mu I (16 coils, W = 8, 280 points in the DC cell:
    reduction slices in the spread) on 3 frames, two of them in one batch, vs the oracle."""
    cfg, traj, coils, frames, x = setup("stress", frames=[5, 6, 1500])
    fil = synth.frame_interleaf(frames, cfg.R)
    pl = plan_for(mrf, cfg, traj, coils, frames, batch_frames=2)
    xn_gpu = host(pl.normal(dev(x), mu=cfg.mu))
    xn_ref = on.normal(x, traj, coils, cfg.W, mu=cfg.mu, frame_interleaf=fil, workers=WORKERS)
    assert rel(xn_gpu, xn_ref) <= OP_TOL
    for i in range(len(frames)):   # and frame by frame (no frame hides behind another's norm)
        assert rel(xn_gpu[i], xn_ref[i]) <= OP_TOL


def test_full_mrf_launch_config_sampled_frames(mrf):
    """MRF-shaped config at full size (L = 1000, the bench launch configuration): sampled frames
    of forward / normal vs the oracle computed frame by frame."""
    cfg = synth.get_config("mrf")
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    x = synth.images(cfg)
    pl = mrf.Plan(cfg.N, traj, cfg.L, W=cfg.W)
    xd = dev(x)
    y = pl.forward(xd)
    xn = pl.normal(xd, mu=cfg.mu)
    sample = [0, 1, 47, 48, 499, 998, 999]
    y_s = host(y[sample])
    xn_s = host(xn[sample])
    y_ref = on.forward(x[sample], traj, None, cfg.W, frame_interleaf=[l % cfg.R for l in sample], workers=WORKERS)
    xn_ref = on.normal(x[sample], traj, None, cfg.W, mu=cfg.mu, frame_interleaf=[l % cfg.R for l in sample],
                       workers=WORKERS)
    for i in range(len(sample)):
        assert rel(y_s[i], y_ref[i]) <= OP_TOL
        assert rel(xn_s[i], xn_ref[i]) <= OP_TOL


def test_full_mrf_cg_against_the_oracle(mrf):
    """The bench step at full size: mrf_dc_cg from x0 = 0 over all 1000 MRF frames, 10 iterations,
    against the float64 oracle's CG over all frames (threaded over the host cores), element by
    element.  The exported step lengths are checked against the residual history
    (beta_k = rho_{k+1} / rho_k)."""
    cfg = synth.get_config("mrf")
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    y = synth.random_kspace(1, cfg.M, range(cfg.L), cfg.seed)
    pl = mrf.Plan(cfg.N, traj, cfg.L, W=cfg.W)
    xg, info = pl.dc_cg(dev(y), mu=cfg.mu, n_iter=cfg.cg_iters, zero_init=True)
    xg = host(xg)
    pl.close()
    a, b, h = np.array(info["alpha"]), np.array(info["beta"]), np.array(info["history"])
    assert info["iters"] == cfg.cg_iters and np.all(a > 0) and np.all(b > 0)
    assert np.allclose(b, (h[1:] / h[:-1]) ** 2, rtol=1e-10)
    workers = max(1, len(os.sched_getaffinity(0)))
    H = lambda v: on.normal(v, traj, None, cfg.W, mu=cfg.mu, workers=workers)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, None, cfg.N, cfg.W, workers=workers), None, cfg.mu)
    x_ref, h_ref = ocg.cg(H, rhs, np.zeros_like(rhs), cfg.cg_iters)
    assert rel(xg, x_ref) <= CG_TOL
    assert np.allclose(h, h_ref, rtol=1e-3, atol=0)


@pytest.mark.parametrize("N,W", [(32, 2), (32, 16), (64, 6), (128, 8), (512, 6)])
def test_grid_sizes_and_widths(mrf, N, W):
    """Every supported G (64..1024) and the extreme widths W = 2 and W = 16 (max)."""
    L, M, R = 3, 700, 2
    traj = synth.spiral_trajectory(M, R, 5, 1.5)
    rng_frames = range(L)
    x = synth.iid_images(N, rng_frames, 99)
    pl = mrf.Plan(N, traj, L, W=W)
    y_gpu = host(pl.forward(dev(x)))
    y_ref = on.forward(x, traj, None, W)
    assert rel(y_gpu, y_ref) <= OP_TOL
    yr = synth.random_kspace(1, M, rng_frames, 98)
    assert rel(host(pl.adjoint(dev(yr))), on.adjoint(yr, traj, None, N, W)) <= OP_TOL


def test_edges_wrap_dc_single_point(mrf):
    """Points exactly at k = +-0.5 (wrap) and at DC, M = 1, L = 1."""
    N = 32
    traj = np.array([[[0.5, 0.5]], [[-0.5, 0.25]], [[0.0, 0.0]], [[0.5, -0.5]]], np.float32)
    for r in range(4):
        x = synth.iid_images(N, [r], 5)
        pl = mrf.Plan(N, traj[r:r + 1], 1, W=6)
        y_gpu = host(pl.forward(dev(x)))
        y_ref = on.forward(x, traj[r:r + 1], None, 6)
        assert rel(y_gpu, y_ref) <= OP_TOL
        yv = np.array([[[1.0 - 2.0j]]], np.complex64)
        assert rel(host(pl.adjoint(dev(yv))), on.adjoint(yv, traj[r:r + 1], None, N, 6)) <= OP_TOL


def test_cartesian_discrete_equals_fft(mrf):
    """Full Cartesian trajectory with discrete deapodisation: the GPU forward equals the FFT."""
    N = 32
    traj = synth.cartesian_trajectory(N)
    x = synth.iid_images(N, [0, 1], 17)
    pl = mrf.Plan(N, traj, 2, W=6, deapod="discrete")
    y_gpu = host(pl.forward(dev(x)))
    ref = np.stack([np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x[i].astype(np.complex128)), norm="ortho")).ravel()
                    for i in range(2)])[:, None, :]
    assert rel(y_gpu, ref) <= OP_TOL
    assert rel(host(pl.normal(dev(x))), x) <= OP_TOL      # A^H A = I


def test_zero_in_zero_out(mrf):
    cfg, traj, coils, frames, _ = setup("pr1")
    pl = plan_for(mrf, cfg, traj, coils, frames)
    z = torch.zeros(pl.x_shape, dtype=torch.complex64, device="cuda")
    assert not torch.any(pl.forward(z)).item()
    assert not torch.any(pl.adjoint(torch.zeros(pl.y_shape, dtype=torch.complex64, device="cuda"))).item()


def test_adjoint_identity_fp32(mrf):
    cfg, traj, coils, frames, x = setup("sense", frames=range(3))
    pl = plan_for(mrf, cfg, traj, coils, frames)
    yr = synth.random_kspace(cfg.C, cfg.M, frames, 3)
    Ax = host(pl.forward(dev(x))).astype(np.complex128)
    AHy = host(pl.adjoint(dev(yr))).astype(np.complex128)
    lhs, rhs = np.vdot(Ax, yr), np.vdot(x.astype(np.complex128), AHy)
    assert abs(lhs - rhs) <= 1e-6 * np.linalg.norm(Ax) * np.linalg.norm(yr)


def test_host_pointer_path_matches_device(mrf):
    cfg, traj, coils, frames, x = setup("pr1")
    pl = plan_for(mrf, cfg, traj, coils, frames)
    y_dev = host(pl.forward(dev(x)))
    y_host = pl.forward(torch.from_numpy(x)).numpy()
    assert np.array_equal(y_dev, y_host)
    xp = torch.from_numpy(x).pin_memory()
    y_pin = pl.forward(xp).numpy()
    assert np.array_equal(y_dev, y_pin)


def test_forward_deterministic(mrf):
    cfg, traj, coils, frames, x = setup("cfg2", frames=range(30))
    pl = plan_for(mrf, cfg, traj, coils, frames)
    xd = dev(x)
    a, b = host(pl.forward(xd)), host(pl.forward(xd))
    assert np.array_equal(a, b)
    yr = dev(synth.random_kspace(1, cfg.M, frames, 1))
    u, v = host(pl.adjoint(yr)), host(pl.adjoint(yr))
    assert np.array_equal(u, v)          # output-stationary spread: bit-deterministic


def test_batching_invariance(mrf):
    """Results do not depend on the frame-batch size (ragged last batch included)."""
    cfg, traj, coils, frames, x = setup("pr1")
    outs = []
    for bf in (1, 3, 8):
        pl = plan_for(mrf, cfg, traj, coils, frames, batch_frames=bf)
        outs.append(host(pl.normal(dev(x), mu=0.01)))
    assert rel(outs[0], outs[2]) <= 1e-6 and rel(outs[1], outs[2]) <= 1e-6


# ------------------------------------------------------------------------ CG
def _cg_case(mrf, name, frames=None, n_iter=None, **over):
    cfg, traj, coils, frames, x = setup(name, frames=frames, **over)
    fil = synth.frame_interleaf(frames, cfg.R)
    y = on.forward(x, traj, coils, cfg.W, frame_interleaf=fil, workers=WORKERS)
    if cfg.noise > 0:
        sig = cfg.noise * np.sqrt(np.mean(np.abs(y) ** 2))
        y = y + sig * synth.unit_noise(cfg.C, cfg.M, frames, cfg.seed)
    y = y.astype(np.complex64)
    n_iter = cfg.cg_iters if n_iter is None else n_iter
    H = lambda v: on.normal(v, traj, coils, cfg.W, mu=cfg.mu, frame_interleaf=fil, workers=WORKERS)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, coils, cfg.N, cfg.W, frame_interleaf=fil, workers=WORKERS), None, cfg.mu)
    x_ref, h_ref = ocg.cg(H, rhs, np.zeros_like(rhs), n_iter)
    pl = plan_for(mrf, cfg, traj, coils, frames)
    xg, info = pl.dc_cg(dev(y), mu=cfg.mu, n_iter=n_iter)
    xg = host(xg)
    assert info["iters"] == n_iter
    assert rel(xg, x_ref) <= CG_TOL
    assert np.allclose(info["history"], h_ref, rtol=1e-3, atol=0)
    return rel(xg, x_ref)


def test_cg_pr1(mrf):
    _cg_case(mrf, "pr1")


def test_cg_cfg2(mrf):
    _cg_case(mrf, "cfg2")


def test_cg_sense_subset(mrf):
    _cg_case(mrf, "sense", frames=range(10))


def test_cg_sense_multi_batch(mrf):
    """SENSE CG (8 coils, 1 % noise, 10 iterations) over 16 frames in 4-frame batches on both
    lanes, frames 40..55 (16 distinct interleaves), vs the oracle's CG."""
    cfg, traj, coils, frames, x = setup("sense", frames=range(40, 56))
    fil = synth.frame_interleaf(frames, cfg.R)
    y = on.forward(x, traj, coils, cfg.W, frame_interleaf=fil, workers=WORKERS)
    y = (y + cfg.noise * np.sqrt(np.mean(np.abs(y) ** 2)) * synth.unit_noise(cfg.C, cfg.M, frames, cfg.seed)).astype(np.complex64)
    H = lambda v: on.normal(v, traj, coils, cfg.W, mu=cfg.mu, frame_interleaf=fil, workers=WORKERS)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, coils, cfg.N, cfg.W, frame_interleaf=fil, workers=WORKERS), None, cfg.mu)
    x_ref, h_ref = ocg.cg(H, rhs, np.zeros_like(rhs), cfg.cg_iters)
    pl = plan_for(mrf, cfg, traj, coils, frames, batch_frames=4)
    xg, info = pl.dc_cg(dev(y), mu=cfg.mu, n_iter=cfg.cg_iters, zero_init=True)
    assert rel(host(xg), x_ref) <= CG_TOL
    assert np.allclose(info["history"], h_ref, rtol=1e-3, atol=0)


def test_cg_x0_z(mrf):
    """Non-zero x0 and z (rhs = A^H y + mu z), mu = 0.05, 5 iterations vs the oracle."""
    cfg, traj, coils, frames, x = setup("pr1")
    y = on.forward(x, traj, None, cfg.W).astype(np.complex64)
    rng = np.random.default_rng(3)
    x0 = (0.1 * (rng.standard_normal(x.shape) + 1j * rng.standard_normal(x.shape))).astype(np.complex64)
    z = (rng.standard_normal(x.shape) + 1j * rng.standard_normal(x.shape)).astype(np.complex64)
    mu = 0.05
    H = lambda v: on.normal(v, traj, None, cfg.W, mu=mu)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, None, cfg.N, cfg.W), z, mu)
    x_ref, h_ref = ocg.cg(H, rhs, x0, 5)
    pl = plan_for(mrf, cfg, traj, None, frames)
    xg, info = pl.dc_cg(dev(y), x0=dev(x0), z=dev(z), mu=mu, n_iter=5)
    assert rel(host(xg), x_ref) <= CG_TOL
    assert np.allclose(info["history"], h_ref, rtol=1e-4, atol=0)


def test_cg_tol_stop(mrf):
    """tol > 0 stops at the oracle's iteration; long fp32 CG runs drift from the float64 iterates
    (about 1e-2 after 20-30 iterations at kappa ~ 1e3, reproduced by perturbing the oracle's
    operator at fp32 level), so the stopped solution is checked by its
    residual instead of element-wise."""
    cfg, traj, coils, frames, x = setup("pr1")
    y = on.forward(x, traj, None, cfg.W).astype(np.complex64)
    mu = 0.05
    H = lambda v: on.normal(v, traj, None, cfg.W, mu=mu)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, None, cfg.N, cfg.W), None, mu)
    x_ref, h_ref = ocg.cg(H, rhs, np.zeros_like(rhs), 40, tol=1e-2)
    pl = plan_for(mrf, cfg, traj, None, frames)
    xg, info = pl.dc_cg(dev(y), mu=mu, n_iter=40, tol=1e-2)
    assert abs(info["iters"] - (len(h_ref) - 1)) <= 1
    assert info["rel_resid"] < 1e-2
    r = rhs - H(host(xg).astype(np.complex128))
    assert np.linalg.norm(r) / np.linalg.norm(rhs) < 1.5e-2
    assert rel(host(xg), x_ref) <= 5e-2


def test_cg_zero_rhs(mrf):
    cfg, traj, coils, frames, x = setup("pr1")
    pl = plan_for(mrf, cfg, traj, None, frames)
    xg, info = pl.dc_cg(torch.zeros(pl.y_shape, dtype=torch.complex64, device="cuda"), mu=0.01, n_iter=4)
    assert info["iters"] == 0
    assert not torch.any(xg).item()


def test_cg_host_pointers(mrf):
    cfg, traj, coils, frames, x = setup("pr1")
    pl = plan_for(mrf, cfg, traj, None, frames)
    y = on.forward(x, traj, None, cfg.W).astype(np.complex64)
    xd, _ = pl.dc_cg(dev(y), mu=0.01, n_iter=5)
    xh, _ = pl.dc_cg(torch.from_numpy(y), mu=0.01, n_iter=5)
    assert rel(xh.numpy(), host(xd)) <= 1e-6


def test_invalid_calls(mrf):
    cfg, traj, coils, frames, x = setup("pr1")
    pl = plan_for(mrf, cfg, traj, None, frames)
    xd = dev(x)
    with pytest.raises(mrf.MrfError) as e:
        pl.normal(xd, mu=-1.0)
    assert e.value.status == 1
    import ctypes
    assert mrf.lib.mrf_normal(pl._h, ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(xd.data_ptr()),
                              ctypes.c_float(0.0), None) == 1     # aliasing
    with pytest.raises(mrf.MrfError):
        pl.dc_cg(dev(np.zeros(pl.y_shape, np.complex64)), n_iter=-1)
    with pytest.raises(mrf.MrfError):   # host and device pointers mixed
        pl.forward(xd, torch.zeros(pl.y_shape, dtype=torch.complex64))


# ------------------------------------------------------------------------ NCCL path, graphs
def test_cg_with_nccl_communicator_single_rank(mrf):
    """mrf_dc_cg through a 1-rank NCCL communicator (the all-reduce calls of the multi-GPU path
    run; with one rank the result must equal the communicator-free solve)."""
    import ctypes
    cfg, traj, coils, frames, x = setup("pr1")
    y = on.forward(x, traj, None, cfg.W).astype(np.complex64)
    buf = (ctypes.c_ubyte * 128)()
    assert mrf.lib.mrf_nccl_get_unique_id(ctypes.cast(buf, ctypes.c_void_p)) == 0, mrf.lib.mrf_last_error()
    comm = ctypes.c_void_p()
    assert mrf.lib.mrf_nccl_comm_init(ctypes.byref(comm), 1, ctypes.cast(buf, ctypes.c_void_p), 0, 0) == 0, \
        mrf.lib.mrf_last_error()
    try:
        pl_c = plan_for(mrf, cfg, traj, None, frames, nccl_comm=comm.value)
        pl_0 = plan_for(mrf, cfg, traj, None, frames)
        xc, ic = pl_c.dc_cg(dev(y), mu=cfg.mu, n_iter=cfg.cg_iters)
        x0, i0 = pl_0.dc_cg(dev(y), mu=cfg.mu, n_iter=cfg.cg_iters)
        assert np.array_equal(host(xc), host(x0))
        assert ic["history"] == i0["history"]
        pl_c.close()
    finally:
        mrf.nccl_comm_destroy(comm.value)


def test_operators_graph_capturable(mrf):
    """forward / adjoint / normal on device pointers allocate nothing and sync nothing, so a CUDA
    graph of them replays to the same result (multi-batch plan: the fork/join lanes are captured)."""
    cfg, traj, coils, frames, x = setup("cfg2", frames=range(40))
    pl = plan_for(mrf, cfg, traj, coils, frames, batch_frames=8)
    xd = dev(x)
    y = torch.empty(pl.y_shape, dtype=torch.complex64, device="cuda")
    xn = torch.empty(pl.x_shape, dtype=torch.complex64, device="cuda")
    ref_y = host(pl.forward(xd)).copy()
    ref_n = host(pl.normal(xd, mu=0.01)).copy()
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        pl.forward(xd, y=y)          # warm-up on the capture stream
        pl.normal(xd, mu=0.01, out=xn)
        with torch.cuda.graph(g, stream=s):
            pl.forward(xd, y=y)
            pl.normal(xd, mu=0.01, out=xn)
    y.zero_()
    xn.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(host(y), ref_y)
    assert rel(host(xn), ref_n) <= 1e-6


@pytest.mark.parametrize("coil_cfg", ["cfg2", "sense"])
def test_cg_graph_replay_equals_direct_launches(mrf, coil_cfg):
    """A tol = 0 mrf_dc_cg is captured once into a CUDA graph and replayed: the replay (also after
    the inputs' contents change behind the same pointers) equals the directly launched solve
    (per-kernel profiling forces direct launches) bit for bit, history included."""
    over = {"N": 64, "M": 700, "R": 4} if coil_cfg == "sense" else {}
    cfg, traj, coils, frames, x = setup(coil_cfg, frames=range(24), **over)
    pl = plan_for(mrf, cfg, traj, coils, frames, batch_frames=8)
    y = pl.forward(dev(x))
    xg = torch.empty(pl.x_shape, dtype=torch.complex64, device="cuda")
    for _ in range(2):                                            # capture, then replay
        _, ig = pl.dc_cg(y, mu=cfg.mu, n_iter=6, x=xg, zero_init=True)
    pl.profile(True)
    xd, idr = pl.dc_cg(y, mu=cfg.mu, n_iter=6, zero_init=True)
    pl.profile(False)
    assert torch.equal(xg, xd) and ig["history"] == idr["history"] and ig["alpha"] == idr["alpha"]
    y.mul_(0.5)                                                   # new contents, same pointers
    pl.dc_cg(y, mu=cfg.mu, n_iter=6, x=xg, zero_init=True)
    pl.profile(True)
    xd2, _ = pl.dc_cg(y, mu=cfg.mu, n_iter=6, zero_init=True)
    pl.profile(False)
    assert torch.equal(xg, xd2) and rel(host(xd2), 0.5 * host(xd)) <= 1e-6
    pl.close()


# ------------------------------------------------------------------------ Toeplitz normal (f1)
def _nudft_normal(x, traj, coils, fil, mu):
    """The plain definition A^H A x + mu x with the direct NUDFT (oracle layer (i))."""
    y = on.nudft_forward(x, traj, coils, frame_interleaf=fil)
    return on.nudft_adjoint(y, traj, coils, x.shape[1], frame_interleaf=fil) + mu * x.astype(np.complex128)


@pytest.mark.parametrize("name,frames,over", [
    ("pr1", None, {}),
    ("cfg2", [0, 5, 23, 199], {}),
    ("sense", [0, 3], {"N": 64, "M": 700, "R": 4}),
    ("stress", [0, 1], {"N": 64, "M": 1024, "R": 4, "C": 4}),
])
def test_toeplitz_normal_vs_nudft(mrf, name, frames, over):
    """MRF_NORMAL_TOEPLITZ: the exact (NUDFT) normal operator up to fp32 rounding."""
    cfg, traj, coils, frames, x = setup(name, frames=frames, **over)
    fil = synth.frame_interleaf(frames, cfg.R)
    pl = plan_for(mrf, cfg, traj, coils, frames, normal="toeplitz")
    got = host(pl.normal(dev(x), mu=cfg.mu))
    ref = _nudft_normal(x, traj, coils, fil, cfg.mu)
    assert rel(got, ref) <= OP_TOL
    # the gridding normal differs from the exact one by the NUFFT error only
    grid = on.normal(x, traj, coils, cfg.W, mu=cfg.mu, frame_interleaf=fil)
    assert rel(grid, ref) <= 1e-4


def test_toeplitz_cg_pr1(mrf):
    """CG with the Toeplitz normal vs the oracle CG with the exact normal (rhs from A^H y)."""
    cfg, traj, coils, frames, x = setup("pr1")
    y = on.forward(x, traj, None, cfg.W).astype(np.complex64)
    H = lambda v: _nudft_normal(v, traj, None, synth.frame_interleaf(frames, cfg.R), cfg.mu)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, None, cfg.N, cfg.W), None, cfg.mu)
    x_ref, h_ref = ocg.cg(H, rhs, np.zeros_like(rhs), cfg.cg_iters)
    pl = plan_for(mrf, cfg, traj, None, frames, normal="toeplitz")
    xg, info = pl.dc_cg(dev(y), mu=cfg.mu, n_iter=cfg.cg_iters)
    assert rel(host(xg), x_ref) <= CG_TOL
    assert np.allclose(info["history"], h_ref, rtol=1e-3, atol=0)


@pytest.mark.parametrize("N,M,L,bf", [(32, 300, 5, 2), (64, 500, 3, 0), (512, 64, 1, 0)])
def test_toeplitz_sizes_and_batches(mrf, N, M, L, bf):
    """Toeplitz normal for G = 64, 128, 1024, with ragged frame batches."""
    traj = synth.spiral_trajectory(M, 2, 4, 1.5)
    frames = list(range(L))
    x = synth.iid_images(N, frames, 31)
    fil = synth.frame_interleaf(frames, 2)
    pl = mrf.Plan(N, traj, L, W=6, frame_interleaf=fil, normal="toeplitz", batch_frames=bf)
    got = host(pl.normal(dev(x), mu=0.02))
    ref = _nudft_normal(x, traj, None, fil, 0.02)
    assert rel(got, ref) <= OP_TOL


# ------------------------------------------------------------------ density compensation (f4)
def test_dcf_weights_and_weighted_adjoint(mrf):
    from oracle import dcf as odcf
    binding = mrf
    for name, over in (("pr1", {}), ("cfg2", {"L": 6})):
        cfg = synth.get_config(name, **over)
        traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
        pl = binding.Plan(cfg.N, traj, cfg.L, W=cfg.W, dcf=True)
        w = pl.dcf_weights()
        w_ref = odcf.dcf(traj.astype(np.float64), cfg.N, cfg.W, n_iter=20)
        assert np.max(np.abs(w - w_ref) / w_ref) < 1e-5
        y = synth.random_kspace(1, cfg.M, range(cfg.L), cfg.seed)
        il = np.arange(cfg.L) % cfg.R
        yw = y.astype(np.complex128) * w_ref[il][:, None, :]
        x_ref = on.adjoint(yw, traj, None, cfg.N, cfg.W)
        x = pl.adjoint_dcf(torch.from_numpy(y.astype(np.complex64)).cuda())
        assert rel(x.cpu().numpy(), x_ref) <= OP_TOL
        xh = pl.adjoint_dcf(torch.from_numpy(y.astype(np.complex64)))          # host-pointer path
        assert rel(xh.numpy(), x_ref) <= OP_TOL
        pl.close()
    pl = binding.Plan(32, synth.spiral_trajectory(256, 8, 4, 1.5), 2)
    with pytest.raises(binding.MrfError):
        pl.adjoint_dcf(torch.zeros(pl.y_shape, dtype=torch.complex64, device="cuda"))
    pl.close()


def test_cg_zero_init_matches_zeroed_x0(mrf):
    """mrf_dc_cg_ex(MRF_CG_ZERO_INIT): no normal operator for r0 = rhs, x output only; the same
    iterates as mrf_dc_cg from a zeroed x (H 0 = 0 exactly), on the device and the host path."""
    cfg, traj, coils, frames, x = setup("pr1")
    y = on.forward(x, traj, None, cfg.W).astype(np.complex64)
    pl = mrf.Plan(cfg.N, traj, cfg.L, W=cfg.W)
    xa, ia = pl.dc_cg(dev(y), mu=cfg.mu, n_iter=cfg.cg_iters)
    xb, ib = pl.dc_cg(dev(y), mu=cfg.mu, n_iter=cfg.cg_iters, zero_init=True)
    xh, ih = pl.dc_cg(torch.from_numpy(y), mu=cfg.mu, n_iter=cfg.cg_iters, zero_init=True)
    pl.close()
    a, b = host(xa), host(xb)
    assert np.array_equal(a, b) and np.array_equal(a, xh.numpy())
    assert ia["history"] == ib["history"] == ih["history"]


def test_cg_async_host_pipeline(mrf):
    """MRF_CG_ASYNC_HOST: a pipelined stream of host-buffer solves (result copies on the plan's
    copy stream, two device slots) gives exactly the synchronous host path's results, and a
    device-pointer call with the flag is rejected."""
    cfg, traj, coils, frames, x = setup("pr1")
    rng = np.random.default_rng(5)
    ys = [on.forward(x * (1.0 + 0.5 * k), traj, None, cfg.W).astype(np.complex64) for k in range(3)]
    pl = mrf.Plan(cfg.N, traj, cfg.L, W=cfg.W)
    ref = [pl.dc_cg(torch.from_numpy(y), mu=cfg.mu, n_iter=cfg.cg_iters, zero_init=True)[0].numpy() for y in ys]
    yh = [torch.from_numpy(y).pin_memory() for y in ys]
    xh = [torch.full(pl.x_shape, complex(rng.standard_normal()), dtype=torch.complex64).pin_memory() for _ in ys]
    for k in range(3):
        pl.dc_cg(yh[k], mu=cfg.mu, n_iter=cfg.cg_iters, x=xh[k], zero_init=True, async_host=True)
    pl.wait()
    for k in range(3):
        assert np.array_equal(xh[k].numpy(), ref[k])
    with pytest.raises(mrf.MrfError):
        pl.dc_cg(dev(ys[0]), mu=cfg.mu, n_iter=2, zero_init=True, async_host=True)
    pl.close()


# ------------------------------------------------------------------------ stage-wise parity
@pytest.mark.parametrize("name,over", [("pr1", {}), ("sense", {"N": 64, "M": 700, "R": 4})])
def test_stagewise_half_grids(mrf, name, over):
    """Stage-wise parity: the half grid between the row and the column pass, against
    the oracle's own stages (oracle.nufft grid_*_frame(stages=True)).  Forward: the row FFT of the
    deapodised, coil-weighted, zero-padded image (image row iy, all G columns); adjoint: the spread
    grid after the column inverse DFT at the N kept rows."""
    cfg, traj, coils, frames, x = setup(name, frames=range(3), **over)
    fil = synth.frame_interleaf(frames, cfg.R)
    L, N, G, C = len(frames), cfg.N, cfg.G, cfg.C
    pl = plan_for(mrf, cfg, traj, coils, frames, batch_frames=L)
    gp = on.GridParams(N, cfg.W)
    pl.forward(dev(x))
    Hf = pl.debug_halfgrid(L).reshape(L * C, G // 16, N, 16).transpose(0, 2, 1, 3).reshape(L, C, N, G)
    yr = synth.random_kspace(C, cfg.M, frames, cfg.seed).astype(np.complex64)
    pl.adjoint(dev(yr))
    Ha = pl.debug_halfgrid(L).reshape(L, C, N, G)
    for l in range(L):
        k = traj[fil[l]]
        _, st = on.grid_forward_frame(x[l], coils, k, gp, stages=True)
        assert rel(Hf[l], st["half"]) <= OP_TOL
        _, sa = on.grid_adjoint_frame(yr[l], coils, k, gp, stages=True)
        col = np.fft.ifft(sa["spread"], axis=1, norm="forward")[:, gp.idx, :]   # columns only, kept rows
        assert rel(Ha[l], col) <= OP_TOL
    pl.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name,normal", [("cfg2", "gridding"), ("cfg2", "toeplitz"), ("sense", "gridding")])
def test_split_phase_cg_matches_textbook_cg(mrf, monkeypatch, name, normal):
    """The split-phase CG (alpha = rho / (<p, A^H A p> + mu ||p||^2) with <p, A^H A p> = ||A p||^2 on
    gridding plans and sum_k T(k) |FFT(pad p)|^2 (Parseval) on Toeplitz plans, r advanced inside the
    adjoint row pass; reading 30) against the textbook loop (alpha = rho / Re<p, q>,
    separate r update; MRF_CG_SPLIT=0) on the same plan inputs: the two are the same iteration in
    exact arithmetic, so their iterates agree to fp32 rounding."""
    cfg, traj, coils, frames, x = setup(name, frames=range(40 if name == "cfg2" else 12))
    y = host(plan_for(mrf, cfg, traj, coils, frames).forward(dev(x)))
    out = {}
    for split in ("1", "0"):
        monkeypatch.setenv("MRF_CG_SPLIT", split)
        pl = plan_for(mrf, cfg, traj, coils, frames, normal=normal)
        xs, info = pl.dc_cg(dev(y), mu=cfg.mu, n_iter=8)
        out[split] = (host(xs), np.asarray(info["history"]))
        pl.close()
    assert rel(out["1"][0], out["0"][0]) < 1e-5
    assert np.allclose(out["1"][1], out["0"][1], rtol=1e-5, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mrf", "stress"])
def test_two_thread_stage2_variant_is_bitwise_identical(mrf, monkeypatch, name):
    """k_adj_cols<G = 512> has a 16-warp variant (two threads per stage-2 transform, the lane pair
    exchanging its half-combined radix-4 values by shuffle; an option, MRF_ADJ_T2=1).  It performs the same floating-point operations in the same order per
    output as the 8-warp kernel, so adjoint, normal operator and CG must agree bit for bit."""
    over = dict(frames=range(3)) if name == "stress" else dict(frames=range(40))
    cfg, traj, coils, frames, x = setup(name, **over)
    yr = synth.random_kspace(cfg.C, cfg.M, frames, cfg.seed)
    out = {}
    for t2 in ("0", "1"):
        monkeypatch.setenv("MRF_ADJ_T2", t2)
        pl = plan_for(mrf, cfg, traj, coils, frames, batch_frames=max(1, len(frames) // 3))
        xs, _ = pl.dc_cg(dev(yr), mu=cfg.mu, n_iter=3)
        out[t2] = (host(pl.adjoint(dev(yr))), host(pl.normal(dev(x), mu=cfg.mu)), host(xs))
        pl.close()
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg2", "stress"])
def test_dynamic_item_handout_is_bitwise_identical(mrf, monkeypatch, name):
    """k_adj_cols hands its items out dynamically on plans whose spread chunks overflow the
    staging buffer (MRF_ADJ_DYN overrides the plan's choice).  Every item is computed the same
    whichever CTA takes it, so the adjoint and the normal operator must agree bit for bit between
    the static round-robin and the dynamic hand-out, on several batches and both lanes."""
    over = dict(frames=range(3)) if name == "stress" else dict(frames=range(60))
    cfg, traj, coils, frames, x = setup(name, **over)
    yr = synth.random_kspace(cfg.C, cfg.M, frames, cfg.seed)
    out = {}
    for dyn in ("0", "1"):
        monkeypatch.setenv("MRF_ADJ_DYN", dyn)
        pl = plan_for(mrf, cfg, traj, coils, frames, batch_frames=max(1, len(frames) // 3))
        out[dyn] = (host(pl.adjoint(dev(yr))), host(pl.normal(dev(x), mu=cfg.mu)))
        pl.close()
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][1], out["1"][1])

"""GPU parity of Algorithm 1 (mrf_msllr_solve, mrf_llr_cost) against the float64 oracle
(oracle/msllr.py).

Inputs are synthetic and seeded: a coarse (T1, T2) grid of surrogate atoms (synth.dictionary),
tissue maps with every voxel in some tissue (so Phi_D has no noise-driven background voxels),
x_true[l, v] = pd_v d_{k_v}[l] and b = A x_true from the oracle's gridding NUFFT.  The GPU and the
oracle each run the whole loop from b (basis, X^0, maps, Laplacian, steps, costs, stop rule).
The loop's maps feed back into the iteration when lambda_1 > 0 (through the Laplacian), so that
case uses one tissue with piecewise-constant PD, where Phi_D's atom is unambiguous; the final maps
must equal the oracle's except valid near-ties (within TIE_REL of the best score).
"""
import numpy as np
import pytest
import torch

import synth
import synth.dictionary as sd
from oracle import llr as ol
from oracle import msllr as oms
from oracle import nufft as on

pytestmark = pytest.mark.gpu

N, L, P, S, W = 32, 60, 7, 3, 6


@pytest.fixture(scope="module")
def binding():
    from paper_2310_05647_b200 import binding as b
    return b


def make_problem(tissues: int):
    grid = sd.t1t2_grid()[::80]                                   # coarse: well-separated atoms
    D = sd.surrogate_dictionary(L, grid)
    lut = grid.astype(np.float32)
    rng = np.random.default_rng([27, tissues])
    yy, xx = np.mgrid[0:N, 0:N] / N - 0.5
    kmap = np.full((N, N), rng.integers(len(grid)))
    pdm = np.full((N, N), 0.4)
    for _ in range(4):                                            # ellipses on a tissue background
        cy, cx = rng.uniform(-0.25, 0.25, 2)
        a, c = rng.uniform(0.1, 0.3, 2)
        m = ((yy - cy) / a) ** 2 + ((xx - cx) / c) ** 2 <= 1.0
        if tissues > 1:
            kmap[m] = rng.integers(len(grid))
        pdm[m] = rng.uniform(0.5, 1.0)
    x_true = (pdm.reshape(-1)[:, None] * D[kmap.reshape(-1)]).T.reshape(L, N, N)
    traj = synth.spiral_trajectory(512, 10, 8, 1.5)
    b = on.forward(x_true, traj, None, W)
    # mu below 1 / lambda_max(A^H A) (power iteration on one frame of the oracle's normal operator)
    v = rng.standard_normal((1, N, N)) + 0j
    for _ in range(30):
        v = on.normal(v, traj, None, W)
        lam = np.linalg.norm(v)
        v /= lam
    d = ol.basis(D, 0.9999, 32)
    return {"D": D, "lut": lut, "traj": traj, "b": b, "mu": 0.9 / lam, "d": d}


@pytest.fixture(scope="module")
def problem():
    """Four tissues: boundary voxels are mixtures, so Phi_D may resolve near-ties either way."""
    return make_problem(4)


@pytest.fixture(scope="module")
def problem1():
    """One tissue with piecewise-constant PD: the maps that feed the Laplacian back into the loop
    carry no tissue-boundary mixtures."""
    return make_problem(1)


def _gpu(binding, pr):
    dic = binding.Dictionary(pr["D"], pr["lut"])
    dic.basis(0.9999, 32)
    op = binding.LLR(dic, N, P, S)
    pl = binding.Plan(N, pr["traj"], L, W=W)
    b = torch.from_numpy(pr["b"].astype(np.complex64)).cuda()
    return dic, op, pl, b


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


# Phi_D is exact (tests/test_gpu_match.py); the GPU and oracle iterates differ by ~1e-6 (fp32), so a
# voxel whose best and second-best scores on the oracle's x lie closer than that may flip
TIE_REL = 1e-5


@pytest.mark.parametrize("lam1,iters,which", [(0.0, 3, "problem"), (2e-3, 2, "problem1"), (2e-3, 4, "problem1")])
def test_solve_against_the_oracle(binding, request, lam1, iters, which):
    pr = request.getfixturevalue(which)
    lam2, beta = 0.05, 0.5
    ref = oms.solve(pr["b"], pr["traj"], pr["D"], pr["lut"], pr["d"], pr["mu"], lam1, lam2, beta, iters, tol=0.0,
                    W=W, N=N, p=P, s=S)
    dic, op, pl, b = _gpu(binding, pr)
    out = op.solve(dic, pl, b, mu=pr["mu"], lam1=lam1, lam2=lam2, beta=beta, max_iter=iters, tol=0.0)
    torch.cuda.synchronize()
    assert out["iters"] == ref["iters"] == iters
    assert _rel(out["x"].cpu().numpy(), ref["x"]) <= 1e-4
    assert np.allclose(out["cost"], ref["cost"], rtol=1e-4, atol=0)
    # final maps M^ = Phi_D(X^): the oracle's atom wherever its best score is clear of the second
    # by TIE_REL, else a valid near-tie (within TIE_REL of the best)
    k = out["index"].cpu().numpy()
    _, _, _, score = __import__("oracle").match.match(ref["x"].reshape(L, -1).T, pr["D"], pr["lut"])
    srt = np.sort(score, axis=1)
    clear = (srt[:, -1] - srt[:, -2]) > TIE_REL * srt[:, -1]
    assert np.array_equal(k[clear], ref["k"][clear])
    assert np.all(score[np.arange(k.size), k] >= (1 - TIE_REL) * srt[:, -1])
    same = k == ref["k"]
    # pd follows x, which is compared in the global relative norm: tolerance relative to max pd
    assert np.max(np.abs(out["pd"].cpu().numpy()[same] - ref["rho"][same])) <= 1e-4 * ref["rho"].max()
    assert np.array_equal(out["params"].cpu().numpy()[same], ref["eta"][same])
    if lam1:
        assert abs(out["lambda1"] - ref["lambda1"]) <= 1e-4 * ref["lambda1"]
    pl.close(), op.close(), dic.close()


def test_cost_terms_against_the_oracle(binding, problem1):
    """mrf_llr_cost at a step iterate (in the subspace, where it equals the paper's cost)."""
    pr = problem1
    dic, op, pl, b = _gpu(binding, pr)
    out = op.solve(dic, pl, b, mu=pr["mu"], lam1=0.0, lam2=0.05, beta=0.5, max_iter=1, tol=0.0)
    x = out["x"]
    params = out["params"][:, :2].contiguous()
    op.laplacian(params, out["pd"])
    c, terms = op.cost(pl, x, b, lam1=0.3, lam2=0.7)
    torch.cuda.synchronize()
    # oracle at the GPU iterate is not allowed (no oracle input from the CUDA path): run the
    # oracle's own one-step solve and its own maps, then compare the cost of its iterate
    ref = oms.solve(pr["b"], pr["traj"], pr["D"], pr["lut"], pr["d"], pr["mu"], 0.0, 0.05, 0.5, 1, tol=0.0,
                    W=W, N=N, p=P, s=S)
    from oracle import manifold as omf
    _, m = oms.maps_of(ref["x"], pr["D"], pr["lut"])
    lap = omf.laplacian(omf.weights(m, N, P, S)[0])
    A = lambda X: on.forward(X, pr["traj"], None, W)
    c_ref, t_ref = oms.cost(ref["x"], pr["b"], A, 0.3, 0.7, lap, P, S)
    for g, o in zip(terms, t_ref):
        assert abs(g - o) <= 1e-4 * abs(o), (terms, t_ref)
    assert abs(c - c_ref) <= 1e-4 * c_ref
    pl.close(), op.close(), dic.close()


def test_stop_rule(binding, problem):
    pr = problem
    dic, op, pl, b = _gpu(binding, pr)
    out = op.solve(dic, pl, b, mu=pr["mu"], lam1=0.0, lam2=0.05, beta=0.5, max_iter=6, tol=1e9)
    assert out["iters"] == 2 and len(out["cost"]) == 2
    with pytest.raises(binding.MrfError):        # lambda1 > 0 needs a (T1, T2) LUT
        dnl = binding.Dictionary(pr["D"])
        dnl.basis()
        op2 = binding.LLR(dnl, N, P, S)
        op2.solve(dnl, pl, b, mu=pr["mu"], lam1=1e-3, max_iter=1)
    pl.close(), op.close(), dic.close()


@pytest.mark.parametrize("lam1,iters,which", [(0.0, 4, "problem"), (2e-3, 2, "problem1")])
def test_basis_coordinate_loop_on_a_toeplitz_plan(binding, request, lam1, iters, which):
    """On a MRF_NORMAL_TOEPLITZ plan mrf_msllr_solve runs iterations n >= 2 in basis coordinates
    (subspace normal P_S A^H A from the PSF spectra, the cost by the inner-product identity): the
    operator is the exact NUDFT normal, so the oracle runs its loop with op="nudft"."""
    pr = request.getfixturevalue(which)
    lam2, beta = 0.05, 0.5
    ref = oms.solve(pr["b"], pr["traj"], pr["D"], pr["lut"], pr["d"], pr["mu"], lam1, lam2, beta, iters, tol=0.0,
                    W=W, N=N, p=P, s=S, op="nudft")
    dic = binding.Dictionary(pr["D"], pr["lut"])
    dic.basis(0.9999, 32)
    op = binding.LLR(dic, N, P, S)
    pl = binding.Plan(N, pr["traj"], L, W=W, normal="toeplitz")
    b = torch.from_numpy(pr["b"].astype(np.complex64)).cuda()
    out = op.solve(dic, pl, b, mu=pr["mu"], lam1=lam1, lam2=lam2, beta=beta, max_iter=iters, tol=0.0)
    torch.cuda.synchronize()
    assert out["iters"] == iters
    assert _rel(out["x"].cpu().numpy(), ref["x"]) <= 1e-4
    assert np.allclose(out["cost"], ref["cost"], rtol=1e-4, atol=0)
    if lam1:
        assert abs(out["lambda1"] - ref["lambda1"]) <= 1e-4 * ref["lambda1"]
    pl.close(), op.close(), dic.close()


@pytest.mark.parametrize("normal,opn", [("gridding", "grid"), ("toeplitz", "nudft")])
def test_multicoil_loop(binding, problem, normal, opn):
    """Algorithm 1 with C = 3 coil sensitivities (A = F_u C, SENSE-like; SURVEY.md §8(c) #13 maps):
    LLR-only, 3 iterations, on a gridding and on a Toeplitz (basis-coordinate) plan."""
    pr = problem
    coils = synth.coil_maps(N, 3, 5)
    D = pr["D"]                                   # the fixture's dictionary; data re-simulated with coils
    rng = np.random.default_rng([27, 9])
    k = rng.integers(D.shape[0], size=N * N)
    x_true = (rng.uniform(0.4, 1.0, N * N)[:, None] * D[k]).T.reshape(L, N, N)
    b = on.forward(x_true, pr["traj"], coils, W)
    ref = oms.solve(b, pr["traj"], D, pr["lut"], pr["d"], pr["mu"], 0.0, 0.05, 0.5, 3, tol=0.0, W=W, N=N, p=P, s=S,
                    op=opn, coils=coils)
    dic = binding.Dictionary(D, pr["lut"])
    dic.basis(0.9999, 32)
    op = binding.LLR(dic, N, P, S)
    pl = binding.Plan(N, pr["traj"], L, W=W, coils=coils, normal=normal)
    bd = torch.from_numpy(b.astype(np.complex64)).cuda()
    out = op.solve(dic, pl, bd, mu=pr["mu"], lam1=0.0, lam2=0.05, beta=0.5, max_iter=3, tol=0.0)
    torch.cuda.synchronize()
    assert _rel(out["x"].cpu().numpy(), ref["x"]) <= 1e-4
    assert np.allclose(out["cost"], ref["cost"], rtol=1e-4, atol=0)
    pl.close(), op.close(), dic.close()


def test_solve_edge_cases(binding, problem):
    """max_iter = 0 returns X^0 = A^H b and Phi_D(X^0); a dictionary whose basis changed after the
    LLR operator was created falls back to frame-domain matching and stays correct; match_coef
    without a basis is rejected."""
    pr = problem
    dic, op, pl, b = _gpu(binding, pr)
    out0 = op.solve(dic, pl, b, mu=pr["mu"], lam1=0.0, max_iter=0)
    assert out0["iters"] == 0 and out0["cost"] == []
    x0 = pl.adjoint(b)
    torch.cuda.synchronize()
    assert torch.equal(out0["x"], x0)
    i0, _, _ = dic.match(x0.view(L, -1))
    assert torch.equal(out0["index"], i0)
    # basis recomputed with another rank after the operator was created: the operator keeps its
    # own basis; Phi_D inside the loop then runs on frames (same answer as the coefficient path)
    ref = op.solve(dic, pl, b, mu=pr["mu"], lam1=0.0, lam2=0.05, beta=0.5, max_iter=2, tol=0.0)
    dic.basis(0.99, 4)
    alt = op.solve(dic, pl, b, mu=pr["mu"], lam1=0.0, lam2=0.05, beta=0.5, max_iter=2, tol=0.0)
    torch.cuda.synchronize()
    assert _rel(alt["x"].cpu().numpy(), ref["x"].cpu().numpy()) <= 1e-6
    assert np.allclose(alt["cost"], ref["cost"], rtol=1e-6)
    assert (alt["index"] == ref["index"]).float().mean().item() > 0.99
    pl.close(), op.close(), dic.close()
    d2 = binding.Dictionary(pr["D"], pr["lut"])
    with pytest.raises(binding.MrfError):
        d2.match_coef(torch.zeros((4, 16), dtype=torch.complex64, device="cuda"))
    d2.close()


def test_stop_rule_in_basis_coordinates(binding, problem):
    pr = problem
    dic = binding.Dictionary(pr["D"], pr["lut"])
    dic.basis(0.9999, 32)
    op = binding.LLR(dic, N, P, S)
    pl = binding.Plan(N, pr["traj"], L, W=W, normal="toeplitz")
    b = torch.from_numpy(pr["b"].astype(np.complex64)).cuda()
    full = op.solve(dic, pl, b, mu=pr["mu"], lam1=0.0, lam2=0.05, beta=0.5, max_iter=8, tol=0.0)
    c = full["cost"]
    # a tolerance between two successive relative decreases stops exactly after the first of them
    rel = [c[n - 1] / c[n] - 1.0 for n in range(1, len(c))]
    n_stop = next(n for n in range(1, len(rel)) if rel[n] < rel[n - 1])   # first n where the decrease slows
    tol = 0.5 * (rel[n_stop] + rel[n_stop - 1])
    early = [n for n in range(1, len(c)) if rel[n - 1] < tol]
    out = op.solve(dic, pl, b, mu=pr["mu"], lam1=0.0, lam2=0.05, beta=0.5, max_iter=8, tol=tol)
    assert out["iters"] == early[0] + 1
    assert np.allclose(out["cost"], c[:out["iters"]], rtol=1e-6)
    pl.close(), op.close(), dic.close()


def test_basis_coordinate_loop_at_the_mrf_size(binding):
    """Full MRF size (256^2, 1000 frames, the 3336-atom dictionary, 2500 patches): three MS-LLR
    iterations in basis coordinates (Toeplitz plan) against the frame-domain loop on a gridding plan
    (both parity-tested against the oracle at small sizes above).  They differ by the gridding
    error of the gridding plan's A^H A (~1e-5), not by the reformulation."""
    cfg = synth.get_config("mrf")
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    grid = sd.t1t2_grid()
    dic = binding.Dictionary(sd.surrogate_dictionary(cfg.L, grid), grid.astype(np.float32))
    dic.basis(0.9999, 32)
    op = binding.LLR(dic, cfg.N)
    pg = binding.Plan(cfg.N, traj, cfg.L, W=cfg.W)
    pt = binding.Plan(cfg.N, traj, cfg.L, W=cfg.W, normal="toeplitz")
    b = pg.forward(torch.from_numpy(synth.images(cfg)).cuda())
    kw = dict(mu=0.018, lam1=1e-7, lam2=0.1, beta=0.2, max_iter=3, tol=0.0)
    og = op.solve(dic, pg, b, **kw)
    ot = op.solve(dic, pt, b, **kw)
    torch.cuda.synchronize()
    assert _rel(ot["x"].cpu().numpy(), og["x"].cpu().numpy()) <= 1e-4
    assert np.allclose(ot["cost"], og["cost"], rtol=1e-4)
    assert (ot["index"] == og["index"]).float().mean().item() > 0.999
    pg.close(), pt.close(), op.close(), dic.close()


@pytest.mark.parametrize("normal", ["gridding", "toeplitz"])
def test_solve_without_cost_monitoring(binding, problem1, normal):
    """tol <= 0 and no cost output: cost(n) is skipped, the iterates are unchanged."""
    pr = problem1
    dic = binding.Dictionary(pr["D"], pr["lut"])
    dic.basis(0.9999, 32)
    op = binding.LLR(dic, N, P, S)
    pl = binding.Plan(N, pr["traj"], L, W=W, normal=normal)
    b = torch.from_numpy(pr["b"].astype(np.complex64)).cuda()
    kw = dict(mu=pr["mu"], lam1=2e-3, lam2=0.05, beta=0.5, max_iter=3, tol=0.0)
    a = op.solve(dic, pl, b, **kw)
    c = op.solve(dic, pl, b, costs=False, **kw)
    torch.cuda.synchronize()
    assert c["cost"] == [] and c["iters"] == 3
    assert _rel(c["x"].cpu().numpy(), a["x"].cpu().numpy()) <= 1e-6
    assert torch.equal(c["index"], a["index"])
    pl.close(), op.close(), dic.close()


# ------------------------------------------------------------------ frame sharding
def _comm1(binding):
    import ctypes
    buf = (ctypes.c_ubyte * 128)()
    assert binding.lib.mrf_nccl_get_unique_id(ctypes.cast(buf, ctypes.c_void_p)) == 0, binding.lib.mrf_last_error()
    comm = ctypes.c_void_p()
    assert binding.lib.mrf_nccl_comm_init(ctypes.byref(comm), 1, ctypes.cast(buf, ctypes.c_void_p), 0,
                                          torch.cuda.current_device()) == 0, binding.lib.mrf_last_error()
    return comm.value


def test_shard_takes_its_columns_of_the_basis(binding, problem):
    """mrf_llr_create_shard(dict, f0, Ll) on a plan over frames [f0, f0 + Ll) (frame_offset = f0)
    is the operator of the basis columns [f0, f0 + Ll): bit-identical to mrf_llr_create_basis with
    that slice (no communicator: the coefficients are this shard's partial sums)."""
    pr = problem
    dic = binding.Dictionary(pr["D"], pr["lut"])
    d = dic.basis(0.9999, 32)
    f0, Ll = 21, 25
    sh = binding.LLR.shard(dic, f0, Ll, N, P, S)
    ref = binding.LLR.from_basis(d[:, f0:f0 + Ll], N, P, S)
    pl = binding.Plan(N, pr["traj"], Ll, W=W, frame_offset=f0)
    rng = np.random.default_rng(5)
    x = torch.from_numpy((rng.standard_normal((Ll, N, N)) + 1j * rng.standard_normal((Ll, N, N))).astype(np.complex64)).cuda()
    rhs = torch.from_numpy((rng.standard_normal((Ll, N, N)) + 1j * rng.standard_normal((Ll, N, N))).astype(np.complex64)).cuda()
    a, na, _ = sh.step(pl, x, rhs, mu=pr["mu"], lam2=0.05, beta=0.5)
    b, nb, _ = ref.step(pl, x, rhs, mu=pr["mu"], lam2=0.05, beta=0.5)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and na == nb
    # the full range is the unsharded operator
    full, one = binding.LLR.shard(dic, 0, L, N, P, S), binding.LLR(dic, N, P, S)
    pl2 = binding.Plan(N, pr["traj"], L, W=W)
    xb = torch.from_numpy(on.adjoint(pr["b"], pr["traj"], None, N, W).astype(np.complex64)).cuda()
    assert torch.equal(full.step(pl2, xb, xb, mu=pr["mu"])[0], one.step(pl2, xb, xb, mu=pr["mu"])[0])
    with pytest.raises(binding.MrfError):
        binding.LLR.shard(dic, 50, 20, N, P, S)                  # frames beyond L
    for o in (sh, ref, full, one, pl, pl2, dic):
        o.close()


def test_sharded_solve_through_a_single_rank_communicator(binding, problem):
    """Algorithm 1 (lambda_1 = 0) on a frame-sharded operator whose plan carries a 1-rank NCCL
    communicator: the coefficient and data-term all-reduces run, and with one rank the result is
    the unsharded solve's, bit for bit.  Unsupported sharded modes fail loudly."""
    pr = problem
    comm = _comm1(binding)
    try:
        dic = binding.Dictionary(pr["D"], pr["lut"])
        dic.basis(0.9999, 32)
        b = torch.from_numpy(pr["b"].astype(np.complex64)).cuda()
        kw = dict(mu=pr["mu"], lam1=0.0, lam2=0.05, beta=0.5, max_iter=3, tol=0.0)
        sh, pl_c = binding.LLR.shard(dic, 0, L, N, P, S), binding.Plan(N, pr["traj"], L, W=W, nccl_comm=comm)
        one, pl = binding.LLR(dic, N, P, S), binding.Plan(N, pr["traj"], L, W=W)
        a = sh.solve(dic, pl_c, b, **kw)
        c = one.solve(dic, pl, b, **kw)
        torch.cuda.synchronize()
        assert torch.equal(a["x"], c["x"]) and torch.equal(a["index"], c["index"])
        assert a["cost"] == c["cost"] and a["iters"] == 3
        with pytest.raises(binding.MrfError):                     # Phi_D of X^0 needs every rank's frames
            sh.solve(dic, pl_c, b, **{**kw, "lam1": 2e-3})
        pl_t = binding.Plan(N, pr["traj"], L, W=W, normal="toeplitz", nccl_comm=comm)
        with pytest.raises(binding.MrfError):                     # basis coordinates are not frame-sharded
            sh.solve(dic, pl_t, b, **kw)
        for o in (sh, pl_c, one, pl, pl_t, dic):
            o.close()
    finally:
        binding.nccl_comm_destroy(comm)


def test_printed_form_switches_against_the_oracle(binding, problem1):
    """Algorithm 1 with every printed-form switch on (mrf_llr_set_options): Eq. (23)'s scalar
    denominator, Eq. (8) on raw maps, Eq. (5)'s ||d||^2 in Phi_D -- against the oracle's loop with
    literal_update, raw_maps, match_p = 2; and the switched loop differs from the default one."""
    pr = problem1
    lam1, lam2, beta, iters = 2e-3, 0.05, 0.5, 2
    ref = oms.solve(pr["b"], pr["traj"], pr["D"], pr["lut"], pr["d"], pr["mu"], lam1, lam2, beta, iters, tol=0.0,
                    W=W, N=N, p=P, s=S, literal_update=True, raw_maps=True, match_p=2)
    dic, op, pl, b = _gpu(binding, pr)
    op.set_options(literal_eq23=True, raw_maps=True, match_norm2=True)
    out = op.solve(dic, pl, b, mu=pr["mu"], lam1=lam1, lam2=lam2, beta=beta, max_iter=iters, tol=0.0)
    torch.cuda.synchronize()
    assert _rel(out["x"].cpu().numpy(), ref["x"]) <= 1e-4
    assert np.allclose(out["cost"], ref["cost"], rtol=1e-4, atol=0)
    assert abs(out["lambda1"] - ref["lambda1"]) <= 1e-4 * ref["lambda1"]
    op.set_options()
    dflt = op.solve(dic, pl, b, mu=pr["mu"], lam1=lam1, lam2=lam2, beta=beta, max_iter=iters, tol=0.0)
    assert _rel(dflt["x"].cpu().numpy(), ref["x"]) > 1e-3
    assert binding.lib.mrf_llr_set_options(op._h, 8) == 1          # unknown option: MRF_EINVAL
    pl.close(), op.close(), dic.close()

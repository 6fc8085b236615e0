#!/usr/bin/env python
"""Benchmark of the MS-LLR data-consistency hot path on B200 (one JSON line on rank 0).

A step is one full data-consistency solve ``mrf_dc_cg`` (rhs = A^H y, r0 = rhs - H x0, then
n_iter = 10 CG iterations of H = A^H A + mu I, mu = 0.01) over ALL L frames of the MRF-shaped
workload (BASELINE.json configs[2]: 256 x 256, L = 1000, M = 2048, W = 6, sigma = 2, single
coil), i.e. every row of SURVEY.md §8(a).  ``value`` is NUFFT non-uniform point-passes per second:
each forward or adjoint over the L frames processes L*C*M points, and one step does 1 adjoint +
(n_iter + 1) normal operators = (2 n_iter + 3) passes.  ``ms_per_AHA`` is the time of one normal
operator over L frames, timed separately.  Frames are sharded contiguously over ranks (strong
scaling, fixed L); the CG inner products are all-reduced with NCCL.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload mrf|sense|stress|cfg2]
  python bench.py --impl reference ...    # the float64 CPU oracle on a bounded frame sample
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "NUFFT fwd+adj nonuniform pts/s and ms per A^H A (L frames); HBM GB/s vs peak"
UNIT = "pts/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="mrf", choices=list(synth.CONFIGS))
    ap.add_argument("--cg-iters", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-toeplitz", action="store_true")
    ap.add_argument("--no-match", action="store_true", help="skip the dictionary-matching (Phi_D) measurement")
    ap.add_argument("--no-llr", action="store_true", help="skip the LLR outer-step measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pcg", action="store_true", help="skip the preconditioned-CG measurement")
    ap.add_argument("--no-fft-stages", action="store_true", help="skip the per-stage comparison with cuFFT")
    ap.add_argument("--pcg-tol", type=float, default=1e-3)
    ap.add_argument("--flush-l2", default="auto", choices=["auto", "on", "off"],
                    help="flush L2 between timed steps (auto: when the working set is < 4x L2)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU work of the oracle sample")
    ap.add_argument("--batch-frames", type=int, default=0)
    return ap.parse_args()


def passes_per_step(n_iter: int, zero_init: bool = True) -> int:
    """NUFFT point-passes of one CG step: 1 adjoint (rhs) + the normals (fwd + adj each).  From
    x0 = 0 with mrf_dc_cg_ex(MRF_CG_ZERO_INIT) the library applies n_iter normals; the oracle's
    textbook CG also applies one to x0 (n_iter + 1), and its reference line counts that work."""
    return 2 * n_iter + (1 if zero_init else 3)


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names[1:], parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------ helpers
def ncu_traffic(kernel_class):
    """DRAM bytes per launch of one kernel class from the committed `ncu --set full` capture
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return dict(t["kernels"][kernel_class], source=t.get("source", "profiles/ncu_traffic.json"))
    except (OSError, KeyError, ValueError):
        return None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def fp32_peak_tflops(sm_count: int, mhz: float) -> float:
    """FP32 CUDA-core peak: SMs x 128 FMA lanes x 2 flop x clock."""
    return sm_count * 128 * 2 * mhz * 1e6 / 1e12


def kernel_flops(cfg, cls: str, frames: int) -> float:
    """Algorithmic FP32 flops of one kernel class over `frames` frames:
    FFT 5 n log2 n per length-n transform, N row transforms + G column transforms per (l, c);
    interp / spread 4 W^2 M per (l, c); deapod/coil (2 + 6C) N^2 per frame."""
    N, G, C, M, W = cfg.N, cfg.G, cfg.C, cfg.M, cfg.W
    f1 = 5.0 * G * math.log2(G)
    if cls in ("fwd_rows", "adj_rows"):
        return frames * (C * N * f1 + (2 + 6 * C) * N * N)
    if cls in ("fwd_cols", "adj_cols"):
        return frames * C * (G * f1 + 4 * W * W * M)
    return 0.0


def step_bytes(cfg, L: int, n_iter: int) -> float:
    """Compulsory HBM bytes of one dc_cg step from x0 = 0 (SURVEY.md §8(d) "Algorithmic bytes"):
    adjoint L(8N^2 + 8CM); each of the n_iter normals L 16 N^2; CG init (x = 0, r = rhs, p = r)
    3 image passes; each CG iteration 8 image passes beyond its normal (the minimum)."""
    N, C, M = cfg.N, cfg.C, cfg.M
    img = 8.0 * N * N * L
    return L * (8.0 * N * N + 8.0 * C * M) + n_iter * 2 * img + 3 * img + n_iter * 8 * img


def cpu_model():
    """The host CPU model (lscpu "Model name", else /proc/cpuinfo)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def make_inputs(cfg, frames, device, torch):
    """Images and k-space for this rank's frames (seeded; generated on the host, then copied)."""
    x = synth.images(cfg, frames)
    coils = synth.coil_maps(cfg.N, cfg.C, cfg.seed)
    return torch.from_numpy(x).to(device), coils


# ------------------------------------------------------------------------------------ oracle arm
def oracle_sample(cfg, n_iter: int, target_s: float, nf=None):
    """Time the float64 oracle's dc_cg on a bounded frame sample of the workload (calibrated so
    the sample takes about ``target_s`` seconds).  Returns a dict (pts/s, frames, cores, ...)."""
    from oracle import nufft as on, cg as ocg
    workers = cpu_count()
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    coils = synth.coil_maps(cfg.N, cfg.C, cfg.seed)
    if nf is None:   # calibrate: one normal on `workers` frames
        cal = list(range(min(cfg.L, workers)))
        xc = synth.images(cfg, cal)
        t0 = time.perf_counter()
        on.normal(xc, traj, coils, cfg.W, mu=cfg.mu, frame_interleaf=synth.frame_interleaf(cal, cfg.R),
                  workers=workers)
        per_frame = (time.perf_counter() - t0) / len(cal) * (n_iter + 1.5)
        nf = int(max(1, min(cfg.L, round(target_s / max(per_frame, 1e-6)))))
    frames = list(range(nf))
    fil = synth.frame_interleaf(frames, cfg.R)
    x = synth.images(cfg, frames)
    y = on.forward(x, traj, coils, cfg.W, frame_interleaf=fil, workers=workers)
    t0 = time.perf_counter()
    H = lambda v: on.normal(v, traj, coils, cfg.W, mu=cfg.mu, frame_interleaf=fil, workers=workers)
    rhs = ocg.dc_rhs(on.adjoint(y, traj, coils, cfg.N, cfg.W, frame_interleaf=fil, workers=workers), None, cfg.mu)
    ocg.cg(H, rhs, np.zeros_like(rhs), n_iter)
    dt = time.perf_counter() - t0
    pts = nf * cfg.C * cfg.M * passes_per_step(n_iter, zero_init=False)
    desc = (f"oracle dc_cg (float64 numpy/scipy, {n_iter} CG iterations) on frames 0..{nf - 1} of {cfg.L} of the "
            f"'{cfg.name}' workload ({nf * cfg.C * cfg.M * passes_per_step(n_iter, zero_init=False)} point-passes), "
            f"{workers} ThreadPool workers over frames")
    return {"value": pts / dt, "frames": nf, "cores": workers, "seconds": dt, "sample": desc}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = synth.get_config(args.workload)
    n_iter = args.cg_iters or cfg.cg_iters
    vals, nf, last = [], None, None
    per_step = max(2.0, args.cpu_seconds / 2)
    for i in range(args.warmup + args.steps):
        last = oracle_sample(cfg, n_iter, per_step, nf=nf)
        nf = last["frames"]
        if i >= args.warmup:
            vals.append(last["value"])
    value = float(np.median(vals))
    steps_ms = 1e3 * cfg.L * cfg.C * cfg.M * passes_per_step(n_iter, zero_init=False) / value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": steps_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "N": cfg.N, "L": cfg.L, "M": cfg.M, "C": cfg.C, "W": cfg.W,
                   "sigma": cfg.sigma, "cg_iters": n_iter, "mu": cfg.mu,
                   "step": "oracle dc_cg on a frame sample; ms_per_step extrapolated to all L frames"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "cpu_model": cpu_model(),
                         "kind": "oracle", "sample": last["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2310_05647_b200 import binding
    from paper_2310_05647_b200.sharding import frame_shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, found {torch.cuda.device_count()}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
        comm = binding.nccl_comm_create(rank, world, local)

    cfg = synth.get_config(args.workload)
    n_iter = args.cg_iters or cfg.cg_iters
    off, L = frame_shard(cfg.L, world, rank)
    frames = list(range(off, off + L))
    traj = synth.spiral_trajectory(cfg.M, cfg.R, cfg.turns, cfg.p)
    x_true, coils = make_inputs(cfg, frames, dev, torch)
    plan = binding.Plan(cfg.N, traj, L, coils=coils, W=cfg.W, frame_offset=off, device=local, nccl_comm=comm,
                        batch_frames=args.batch_frames)
    y = plan.forward(x_true)
    if cfg.noise > 0:
        ss = torch.tensor([float((y.abs() ** 2).sum().item()), float(y.numel())], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ss)
        sig = cfg.noise * math.sqrt(ss[0].item() / ss[1].item())
        y += sig * torch.from_numpy(synth.unit_noise(cfg.C, cfg.M, frames, cfg.seed)).to(dev)
    del x_true
    xbuf = torch.zeros(plan.x_shape, dtype=torch.complex64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():   # CG from x0 = 0 (Algorithm 1's data-consistency solve); x is output only
        plan.dc_cg(y, mu=cfg.mu, n_iter=n_iter, x=xbuf, zero_init=True)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed region
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    # L2 flush between steps when the step's working set is not far beyond the 126 MB L2
    # (SURVEY.md §8(d) timing protocol): a 512 MB write outside the per-step events
    work_set = 4.0 * L * cfg.N * cfg.N * 8 + 2.0 * L * cfg.C * cfg.M * 8
    flush = args.flush_l2 == "on" or (args.flush_l2 == "auto" and work_set < 4 * 126e6)
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if flush else None
    if flush:   # per-step events around each step, the flush between them untimed
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            scratch.fill_(i & 0xFF)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
    else:       # one bracket around the K steps
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))]
        evs[0][0].record(stream)
        for _ in range(args.steps):
            step()
        evs[0][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs))
    clk = clocks.stop()
    del scratch
    # per-kernel-class CUDA events (the library brackets every launch): the same steps again,
    # outside the timed region -- profiling replaces the solve's CUDA graph by direct launches
    plan.profile(True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    prof = {k: plan.profile_query(k) for k in binding.KERNEL_CLASSES}
    plan.profile(False)
    ms_step = ms_total / args.steps
    pts_step = cfg.L * cfg.C * cfg.M * passes_per_step(n_iter)
    value = pts_step / (ms_step * 1e-3)

    # ---------------------------------------------------------------- per-operator timings (device)
    def time_op(fn, reps):
        for _ in range(2):
            fn()
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(b)) / reps

    xin = torch.randn(plan.x_shape, dtype=torch.complex64, device=dev)
    xout = torch.empty_like(xin)
    yout = torch.empty(plan.y_shape, dtype=torch.complex64, device=dev)
    reps = max(3, args.steps)
    ms_normal = time_op(lambda: plan.normal(xin, mu=cfg.mu, out=xout), reps)
    ms_fwd = time_op(lambda: plan.forward(xin, y=yout), reps)
    ms_adj = time_op(lambda: plan.adjoint(y, x=xout), reps)
    # the timed step runs from x0 = 0 (MRF_CG_ZERO_INIT): 1 adjoint for the rhs, then n_iter
    # iterations (no normal operator for the initial residual)
    ms_cg_iter = max(0.0, (ms_step - ms_adj) / max(1, n_iter))
    # cuFFT reference (timing only, never in the product path): batched C2C G x G, L*C transforms
    cufft_ms = None
    try:
        B = max(1, min(64, cfg.L * cfg.C))
        buf = torch.randn((B, cfg.G, cfg.G), dtype=torch.complex64, device=dev)
        nchunks = math.ceil(L * cfg.C / B)
        cufft_ms = time_op(lambda: [torch.fft.fft2(buf) for _ in range(nchunks)], 3)
        del buf
    except Exception:
        cufft_ms = None

    # ---------------------------------------------------------------- FFT stages vs cuFFT (reference only)
    # Each of the four gridding kernels timed on its own (a one-lane plan, per-kernel-class events,
    # forward then adjoint), beside cuFFT doing the same stage's transforms unpruned: the row stage
    # = N length-G FFTs per frame-coil (torch.fft.fft over the last axis of [B, N, G]), the column
    # stage = G length-G FFTs per frame-coil (axis -2 of [B, G, G]).  Ours includes the fused
    # deapodisation / gather / spread / crop work of its stage; cuFFT's includes its own HBM passes.
    fft_stages = None
    if not args.no_fft_stages and world == 1:   # (time_op synchronises ranks)
        try:
            prev_lanes = os.environ.get("MRF_LANES")
            os.environ["MRF_LANES"] = "1"
            try:
                p1 = binding.Plan(cfg.N, traj, L, coils=coils, W=cfg.W, frame_offset=off, device=local,
                                  batch_frames=args.batch_frames)
            finally:
                if prev_lanes is None:
                    os.environ.pop("MRF_LANES", None)
                else:
                    os.environ["MRF_LANES"] = prev_lanes
            p1.forward(xin, y=yout)
            p1.adjoint(y, x=xout)
            torch.cuda.synchronize()
            p1.profile(True)
            for _ in range(reps):
                p1.forward(xin, y=yout)
                p1.adjoint(y, x=xout)
            torch.cuda.synchronize()
            ours = {k: p1.profile_query(k)[0] / reps for k in ("fwd_rows", "fwd_cols", "adj_cols", "adj_rows")}
            p1.profile(False)
            p1.close()
            FB = max(1, min(32, L * cfg.C))
            nch = math.ceil(L * cfg.C / FB)
            bufr = torch.randn((FB, cfg.N, cfg.G), dtype=torch.complex64, device=dev)
            bufc = torch.randn((FB, cfg.G, cfg.G), dtype=torch.complex64, device=dev)
            cuf = {
                "rows_fwd": time_op(lambda: [torch.fft.fft(bufr, dim=-1) for _ in range(nch)], 3),
                "cols_fwd": time_op(lambda: [torch.fft.fft(bufc, dim=-2) for _ in range(nch)], 3),
                "cols_inv": time_op(lambda: [torch.fft.ifft(bufc, dim=-2) for _ in range(nch)], 3),
                "rows_inv": time_op(lambda: [torch.fft.ifft(bufr, dim=-1) for _ in range(nch)], 3),
            }
            del bufr, bufc
            fft_stages = {"ours_ms": {"fwd_rows": ours["fwd_rows"], "fwd_cols": ours["fwd_cols"],
                                      "adj_cols": ours["adj_cols"], "adj_rows": ours["adj_rows"]},
                          "cufft_ms": cuf,
                          "note": "ours: one-lane plan, per-kernel-class CUDA events, stage = pruned transforms + the "
                                  "fused deapod/gather/spread/crop of that kernel; cuFFT: unpruned batched 1D C2C "
                                  "transforms of the same stage (rows: N x G per frame-coil, columns: G x G), "
                                  "out-of-place, timing reference only"}
        except Exception as e:  # reference timing only
            fft_stages = {"error": str(e)[:200]}

    # ---------------------------------------------------------------- Toeplitz normal operator
    toep = None
    if not args.no_toeplitz:
        t0 = time.perf_counter()
        plan_t = binding.Plan(cfg.N, traj, L, coils=coils, W=cfg.W, frame_offset=off, device=local, nccl_comm=comm,
                              batch_frames=args.batch_frames, normal="toeplitz")
        torch.cuda.synchronize()
        plan_ms = (time.perf_counter() - t0) * 1e3
        ms_normal_t = time_op(lambda: plan_t.normal(xin, mu=cfg.mu, out=xout), reps)
        xbuf_t = torch.zeros_like(xbuf)

        def step_t():
            plan_t.dc_cg(y, mu=cfg.mu, n_iter=n_iter, x=xbuf_t, zero_init=True)
        ms_step_t = time_op(step_t, max(2, min(args.steps, 5)))
        fl = sum(kernel_flops(cfg, k, cfg.L) for k in ("fwd_rows", "adj_rows")) + \
            cfg.L * cfg.C * 2 * cfg.G * 5.0 * cfg.G * math.log2(cfg.G)
        toep = {"ms_per_AHA": ms_normal_t, "ms_per_step": ms_step_t, "plan_ms": plan_ms,
                "AHA_algorithmic_flops": fl, "AHA_tflops": fl / (ms_normal_t * 1e-3) / 1e12,
                "note": "mrf_dc_cg with the Toeplitz-embedded exact normal operator (MRF_NORMAL_TOEPLITZ); "
                        "the rhs still uses the gridding adjoint"}
        plan_t.close()
        del xbuf_t

    # ---------------------------------------------------------------- dictionary matching Phi_D
    match = None
    if not args.no_match and world == 1 and cfg.C == 1:
        import synth.dictionary as sdict
        grid = sdict.t1t2_grid()
        atoms = sdict.surrogate_dictionary(cfg.L, grid)
        dic = binding.Dictionary(atoms, grid, device=local)
        xm = xbuf.view(cfg.L, -1)                       # the CG solution, frame-major [L][V]
        ms_match = time_op(lambda: dic.match(xm), 5)
        dic.profile(True)
        for _ in range(5):
            dic.match(xm)
        gemm_ms, gemm_n = dic.profile_query()
        dic.profile(False)
        gemm_ms /= max(gemm_n, 1)
        Vm, Km = xm.shape[1], atoms.shape[0]
        # the profiled bracket holds the certified filter's two k_dict_gemm passes over the packed
        # fp16 rows [u_hi | u_lo | u_hi] of the r-dimensional projection: K = KF = 384
        # (csrc/match.cuh), M = voxels padded to 128, N = 2 x atoms padded to 256
        vpad, np_, kd = -(-Vm // 128) * 128, -(-2 * Km // 256) * 256, 384
        gemm_fl = 2 * 2.0 * vpad * np_ * kd
        peak_tc = float(peaks().get("bf16_tflops", 2250.0))
        match = {"ms": ms_match, "voxels": Vm, "atoms": Km, "frames": cfg.L,
                 "useful_tflops": 8.0 * Vm * Km * cfg.L / (ms_match * 1e-3) / 1e12,
                 "roofline": {"bound": "tensor", "kernel": "k_dict_gemm", "achieved": gemm_fl / (gemm_ms * 1e-3) / 1e12,
                              "peak": peak_tc, "unit": "TFLOP/s",
                              "frac": gemm_fl / (gemm_ms * 1e-3) / 1e12 / peak_tc, "avg_launch_ms": gemm_ms,
                              "peak_note": "measured bf16 dense burst (MEASURED_PEAKS.json); fp16 runs at the same rate"},
                 "note": "mrf_dict_match on the CG solution (exact Eq. 5 argmax): r-dimensional projection, "
                         "certified 3xFP16 tcgen05 filter (two GEMM passes, K = 384; 'roofline' covers them), "
                         "float64 rescoring of every admissible atom; useful_tflops = the dense complex "
                         "correlation 8 V K L it replaces, per second of the whole match; synthetic 3336-atom "
                         "dictionary (PAPER.md:319 grid, surrogate fingerprints)"}
        dic.close()

    # ---------------------------------------------------------------- preconditioned CG
    pcg_res = None
    if not args.no_pcg:
        def solve_tol(pc):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, inf = plan.dc_cg(y, mu=cfg.mu, n_iter=300, tol=args.pcg_tol, x=xbuf, zero_init=True, precond=pc)
            torch.cuda.synchronize()
            return inf, (time.perf_counter() - t0) * 1e3
        solve_tol(True)
        inf_cg, ms_cg_tol = solve_tol(False)
        inf_pc, ms_pc_tol = solve_tol(True)
        ms_pc_step = time_op(lambda: plan.dc_cg(y, mu=cfg.mu, n_iter=n_iter, x=xbuf, zero_init=True, precond=True),
                             max(2, min(args.steps, 5)))
        pcg_res = {"tol": args.pcg_tol, "iters_cg": inf_cg["iters"], "iters_pcg": inf_pc["iters"],
                   "ms_to_tol_cg": max_over_ranks(ms_cg_tol), "ms_to_tol_pcg": max_over_ranks(ms_pc_tol),
                   "rel_resid_cg": inf_cg["rel_resid"], "rel_resid_pcg": inf_pc["rel_resid"],
                   "ms_per_step_pcg": ms_pc_step, "ms_per_pcg_iter_est": max(0.0, (ms_pc_step - ms_adj) / max(1, n_iter)),
                   "note": "mrf_dc_cg_ex(MRF_CG_PRECOND): T. Chan circulant of the exact normal operator + gamma I, "
                           "gamma = mu + 30 mean(lambda); iterations and wall time (host-synchronised tol checks) "
                           "to ||r||/||r0|| < tol from x0 = 0"}

    # ---------------------------------------------------------------- density compensation
    dcf_res = None
    if world == 1:
        t0 = time.perf_counter()
        plan_d = binding.Plan(cfg.N, traj, L, coils=coils, W=cfg.W, device=local, dcf=True)
        plan_ms = (time.perf_counter() - t0) * 1e3
        xd = torch.empty_like(xbuf)
        ms_adj_dcf = time_op(lambda: plan_d.adjoint_dcf(y, x=xd), 5)
        ms_adj = time_op(lambda: plan_d.adjoint(y, x=xd), 5)
        dcf_res = {"ms_adjoint_dcf": ms_adj_dcf, "ms_adjoint": ms_adj, "plan_ms_with_dcf": plan_ms,
                   "note": "mrf_adjoint_dcf = A^H (w . y) with the plan's Pipe-Menon weights (20 iterations, "
                           "float64 at plan time): one scaling kernel + the adjoint pipeline"}
        plan_d.close()
        del xd

    # ---------------------------------------------------------------- (MS-)LLR outer step and Algorithm 1
    llr_res = None
    if not args.no_llr and world == 1 and cfg.C == 1:
        import synth.dictionary as sdict
        grid = sdict.t1t2_grid()
        dic = binding.Dictionary(sdict.surrogate_dictionary(cfg.L, grid), grid, device=local)
        t0 = time.perf_counter()
        d_basis = dic.basis(0.9999, 32)
        basis_ms = (time.perf_counter() - t0) * 1e3
        op = binding.LLR(dic, cfg.N, 11, 5)
        rhs_l = plan.adjoint(y)
        xl = torch.empty_like(xbuf)
        ms_llr = time_op(lambda: op.step(plan, xbuf, rhs_l, 1.0, 0.1, 0.2, x_out=xl, nuclear=False), 5)
        nc = len(range(0, cfg.N - 11 + 1, 5)) + (0 if (cfg.N - 11) % 5 == 0 else 1)
        # the manifold term (lambda_1 > 0): maps by Phi_D, the Laplacian, the MS-LLR step, the cost
        _, pd_m, par_m = dic.match(xbuf)
        ms_lap = time_op(lambda: op.laplacian(par_m, pd_m), 3)
        _, maxdeg = op.laplacian(par_m, pd_m)
        lam1 = 1e-7 * maxdeg                      # lambda_1^0 max(L) with lambda_1^0 = 1e-7
        ms_ms = time_op(lambda: op.step(plan, xbuf, rhs_l, 1.0, 0.1, 0.2, x_out=xl, nuclear=False, lam1=lam1), 5)
        ms_cost = time_op(lambda: op.cost(plan, xl, y, lam1=lam1, lam2=0.1), 3)

        def solve_s(n, l1, pln=None, costs=True):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            op.solve(dic, pln or plan, y, mu=0.018, lam1=l1, lam2=0.1, beta=0.2, max_iter=n, tol=0.0, costs=costs)
            torch.cuda.synchronize()
            return (time.perf_counter() - t0) * 1e3

        solve_s(1, 1e-7)
        it_llr = min((solve_s(11, 0.0) - solve_s(1, 0.0)) / 10 for _ in range(2))
        it_ms = min((solve_s(11, 1e-7) - solve_s(1, 1e-7)) / 10 for _ in range(2))
        # the same loop on a Toeplitz plan: iterations n >= 2 in basis coordinates (subspace normal)
        plan_t = binding.Plan(cfg.N, traj, cfg.L, W=cfg.W, normal="toeplitz", device=local)
        solve_s(2, 1e-7, plan_t)
        it_llr_t = min((solve_s(11, 0.0, plan_t) - solve_s(1, 0.0, plan_t)) / 10 for _ in range(2))
        it_ms_t = min((solve_s(11, 1e-7, plan_t) - solve_s(1, 1e-7, plan_t)) / 10 for _ in range(2))
        it_ms_t_nc = min((solve_s(11, 1e-7, plan_t, False) - solve_s(1, 1e-7, plan_t, False)) / 10 for _ in range(2))
        plan_t.close()
        llr_res = {"ms_per_step": ms_llr, "ms_normal_inside": ms_normal, "rank": int(d_basis.shape[0]),
                   "patches": nc * nc, "basis_ms": basis_ms,
                   "ms_per_step_manifold": ms_ms, "ms_laplacian": ms_lap, "ms_cost": ms_cost,
                   "ms_per_algorithm1_iteration": {"llr": it_llr, "ms_llr": it_ms,
                                                   "llr_basis_coordinates": it_llr_t, "ms_llr_basis_coordinates": it_ms_t,
                                                   "ms_llr_basis_coordinates_no_cost": it_ms_t_nc,
                                                   "note": "mrf_msllr_solve wall clock (T(11) - T(1)) / 10, best of 2: step + "
                                                           "cost (+ Phi_D + Laplacian update for MS-LLR); "
                                                           "mu = 0.018 (< 1/lambda_max), lambda_1^0 = 1e-7; "
                                                           "*_basis_coordinates: on a MRF_NORMAL_TOEPLITZ plan (subspace "
                                                           "normal, exact NUDFT normal operator); *_no_cost: fixed iteration count without "
                                                           "cost(n) (tol = 0, no cost output)"},
                   "note": "mrf_llr_step: Z = P_S(X - mu(A^H A X - A^H b) [+ mu lambda_1 Q*(Q(X) L)]), per-patch "
                           "SVT (11x11, stride 5, tau = 1/beta = 5) in subspace coordinates, overlap-exact X "
                           "update; mu = 1, lambda_2 = 0.1, beta = 1/5 (PAPER.md:304); basis from the synthetic "
                           "dictionary; manifold GEMM on tcgen05 (tf32 x3)"}
        op.close()
        dic.close()
        del xl, rhs_l

    # ---------------------------------------------------------------- e2e through the C-ABI, host buffers
    e2e = None
    if not args.no_e2e:
        y_h = y.cpu().pin_memory()
        x_h = [torch.zeros(plan.x_shape, dtype=torch.complex64).pin_memory() for _ in range(2)]
        # warm-up (allocates the slots), then a pipelined stream of solves through the C-ABI with
        # host buffers (MRF_CG_ASYNC_HOST: each result copy overlaps the next solve; the timed
        # region ends when the last result is on the host)
        plan.dc_cg(y_h, mu=cfg.mu, n_iter=n_iter, x=x_h[0], zero_init=True, async_host=True)
        plan.wait()
        n_e2e = max(1, min(args.steps, 10))
        barrier()
        t0 = time.perf_counter()
        for k in range(n_e2e):
            plan.dc_cg(y_h, mu=cfg.mu, n_iter=n_iter, x=x_h[k % 2], zero_init=True, async_host=True)
        plan.wait()
        torch.cuda.synchronize()
        ms_e2e = max_over_ranks((time.perf_counter() - t0) * 1e3 / n_e2e)
        e2e = {"value": pts_step / (ms_e2e * 1e-3), "unit": UNIT, "ms_per_step": ms_e2e, "steps": n_e2e,
               "h2d_bytes_per_step": int(y_h.numel() * 8) * world,
               "d2h_bytes_per_step": int(x_h[0].numel() * 8) * world,
               "note": "host pinned k-space y copied in, solution x copied out, inside each "
                       "mrf_dc_cg_ex(MRF_CG_ZERO_INIT | MRF_CG_ASYNC_HOST) call (x0 = 0 is not transferred); "
                       "the result copy of step k overlaps the solve of step k+1; wall clock from the first "
                       "call to the last result on the host"}

    # ---------------------------------------------------------------- roofline of the dominant kernel
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    pk = peaks()
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    peak_alu = fp32_peak_tflops(sm_count, sm_max)
    hbm_peak = float(pk.get("hbm_gbs", 6650.0))
    cls_ms = {k: v[0] for k, v in prof.items()}
    dom = max(("fwd_rows", "fwd_cols", "adj_cols", "adj_rows"), key=lambda k: cls_ms[k])
    dom_ms, dom_n = prof[dom]
    # frames processed by the dominant class in the timed region: each launch covers a batch
    frames_per_call = {"fwd_rows": n_iter, "fwd_cols": n_iter, "adj_cols": n_iter + 1, "adj_rows": n_iter + 1}
    dom_flops_total = kernel_flops(cfg, dom, L) * frames_per_call[dom] * args.steps
    achieved = dom_flops_total / (dom_ms * 1e-3) / 1e12 if dom_ms > 0 else None
    # traffic: ncu dram bytes per launch, scaled from the capture's frames per launch to this run's
    tr = ncu_traffic(dom)
    traffic = None
    if tr and dom_n:
        frames_per_launch = L * frames_per_call[dom] * args.steps / dom_n
        traffic = tr["dram_bytes_per_launch"] * frames_per_launch / tr["frames_per_launch"]
    roofline = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak_alu, "unit": "TFLOP/s",
                "frac": (achieved / peak_alu) if achieved else None, "traffic": traffic,
                "traffic_note": ("ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                 f"({tr['source']}), scaled to this run's frames per launch") if tr else None,
                "note": "per-launch CUDA events on the launch lane; the two batch lanes overlap, so the "
                        "durations include time-sharing with the other lane (conservative)",
                "avg_launch_ms": dom_ms / max(dom_n, 1), "launches": dom_n,
                "peak_note": f"FP32 CUDA-core peak {sm_count} SMs x 128 x 2 x {sm_max:.0f} MHz (DESIGN.md)"}
    # the whole normal operator as one unit (its kernels overlap across the two batch lanes, so the
    # per-class event durations above are conservative): algorithmic FLOPs / device time per A^H A
    aha_flops = sum(kernel_flops(cfg, k, cfg.L) for k in ("fwd_rows", "fwd_cols", "adj_cols", "adj_rows"))
    aha_tflops = aha_flops / (ms_normal * 1e-3) / 1e12
    aha_bytes = cfg.L * 16.0 * cfg.N * cfg.N + 8.0 * cfg.R * cfg.M
    roofline_aha = {"bound": "alu", "unit": "TFLOP/s", "achieved": aha_tflops, "peak": peak_alu,
                    "frac": aha_tflops / peak_alu, "algorithmic_flops": aha_flops, "ms": ms_normal,
                    "hbm_literal_frac": aha_bytes / (ms_normal * 1e-3) / 1e9 / hbm_peak,
                    "t_roof_ms": max(aha_flops / (peak_alu * 1e12), aha_bytes / (hbm_peak * 1e9)) * 1e3}
    share = {k: (v / ms_total if ms_total > 0 else None) for k, v in cls_ms.items()}
    # the two batch lanes overlap, so the shares above sum to > 1; normalised to the summed kernel
    # time they compare with the serialised ncu launch list (profiles/)
    ksum = sum(cls_ms.values())
    share_k = {k: (v / ksum if ksum > 0 else None) for k, v in cls_ms.items()}
    hbm_bytes = step_bytes(cfg, cfg.L, n_iter)
    hbm_achieved = hbm_bytes / (ms_step * 1e-3) / 1e9
    gpu_launches = int(sum(prof[k][1] for k in ("fwd_rows", "fwd_cols", "adj_cols", "adj_rows", "cg_vec")))

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:   # after every timed region; the other ranks wait
        o = oracle_sample(cfg, n_iter, args.cpu_seconds)
        cpu = {"value": o["value"], "unit": UNIT, "cores": o["cores"], "cpu_model": cpu_model(), "kind": "oracle",
               "sample": o["sample"], "seconds": o["seconds"]}
    barrier()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "N": cfg.N, "L": cfg.L, "M": cfg.M, "C": cfg.C, "R": cfg.R, "W": cfg.W,
                   "sigma": cfg.sigma, "cg_iters": n_iter, "mu": cfg.mu, "parallelism": f"frames/{world}",
                   "step": "mrf_dc_cg_ex(MRF_CG_ZERO_INIT), x0 = 0: 1 adjoint + n_iter normals + CG vector ops",
                   "l2": (f"L2 flushed between steps (512 MB write outside the per-step events; step working set "
                          f"{work_set / 1e6:.0f} MB)" if flush else
                          f"working set {work_set / 1e6:.0f} MB (x, r, p, q each {L * cfg.N ** 2 * 8 / 1e6:.0f} MB) > L2; no flush"),
                   "batch_frames": args.batch_frames or "auto"},
        "ms_per_AHA": ms_normal, "ms_per_forward": ms_fwd, "ms_per_adjoint": ms_adj,
        "ms_per_cg_iter_est": ms_cg_iter,
        "fwd_pts_s": cfg.L * cfg.C * cfg.M / (ms_fwd * 1e-3), "adj_pts_s": cfg.L * cfg.C * cfg.M / (ms_adj * 1e-3),
        "hbm": {"algorithmic_bytes_per_step": hbm_bytes, "achieved_GBs": hbm_achieved, "peak_GBs": hbm_peak,
                "frac": hbm_achieved / hbm_peak},
        "cufft_ref_ms_fft2_LC": cufft_ms, "fft_stages": fft_stages,
        "roofline": roofline, "roofline_AHA": roofline_aha, "toeplitz": toep, "match": match, "dcf": dcf_res, "pcg": pcg_res, "llr": llr_res, "kernel_share": share, "kernel_share_of_kernel_time": share_k, "gpu_launches": gpu_launches,
        "clocks": clk, "e2e": e2e, "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if comm:
        binding.nccl_comm_destroy(comm)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _spawned_rank(local: int, world: int, port: int, argv):
    """Entry of a rank started by bench.py itself (``--gpus N`` without torchrun)."""
    os.environ.update(RANK=str(local), LOCAL_RANK=str(local), WORLD_SIZE=str(world),
                      LOCAL_WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.argv = argv
    rc = run_ours(parse())
    if rc:
        raise SystemExit(rc)


def spawn_ranks(args) -> int:
    """``python bench.py --gpus N`` (N > 1) outside torchrun: one process per GPU, the same
    environment torchrun would give them (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_*)."""
    import socket
    import torch
    import torch.multiprocessing as mp
    n = torch.cuda.device_count()
    if n < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, found {n}")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_spawned_rank, args=(args.gpus, port, list(sys.argv)), nprocs=args.gpus, join=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

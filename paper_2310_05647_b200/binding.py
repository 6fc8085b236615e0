"""Thin ctypes binding over libmrfnufft.so (include/mrfnufft.h).  Argument marshalling only.

Every operator step runs in the library's sm_100a kernels; there is no CPU or PyTorch fallback.
If the shared library is missing the import fails loudly (build it with
``python -m paper_2310_05647_b200.build`` or ``__graft_entry__.build()``).

Arrays are ``torch.complex64`` tensors, C-contiguous.  CUDA tensors must live on the plan's
device and run asynchronously on the current torch stream; CPU tensors (pinned or pageable) go
through the library's host path (staged copies inside the call; the call returns when done).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np
import torch

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmrfnufft.so")
if os.environ.get("MRF_LIB_PATH"):   # A/B experiments against another in-tree build (never the default)
    LIB_PATH = os.environ["MRF_LIB_PATH"]

MRF_DEAPOD_ANALYTIC = 0
MRF_DEAPOD_DISCRETE = 1
MRF_NORMAL_TOEPLITZ = 2
MRF_DCF = 4
KERNEL_CLASSES = {"fwd_rows": 0, "fwd_cols": 1, "adj_cols": 2, "adj_rows": 3, "cg_vec": 4, "other": 5}
STATUS = {0: "MRF_OK", 1: "MRF_EINVAL", 2: "MRF_ENOMEM", 3: "MRF_ECUDA", 4: "MRF_ENCCL",
          5: "MRF_EUNSUPPORTED", 6: "MRF_ENUMERIC"}

EXPORTED = [
    "mrf_plan_create", "mrf_forward", "mrf_adjoint", "mrf_normal", "mrf_dc_cg", "mrf_dc_cg_ex", "mrf_plan_destroy",
    "mrf_status_string", "mrf_last_error", "mrf_plan_device_bytes", "mrf_profile_enable",
    "mrf_profile_query", "mrf_nccl_get_unique_id", "mrf_nccl_comm_init", "mrf_nccl_comm_destroy",
    "mrf_adjoint_dcf", "mrf_dcf_weights", "mrf_dict_create", "mrf_dict_match", "mrf_dict_destroy",
    "mrf_dict_profile", "mrf_dict_profile_query", "mrf_dict_basis", "mrf_dict_basis_copy", "mrf_llr_create",
    "mrf_llr_step", "mrf_llr_destroy", "mrf_llr_laplacian", "mrf_llr_cost", "mrf_msllr_solve", "mrf_plan_wait",
    "mrf_dict_match_coef", "mrf_llr_create_basis", "mrf_llr_subspace_normal", "mrf_llr_create_shard",
    "mrf_plan_set_host_allreduce", "mrf_plan_set_precond_shift", "mrf_dict_overflow", "mrf_dict_filter_info",
    "mrf_dict_match_ex", "mrf_dict_match_coef_ex", "mrf_llr_set_options", "mrf_plan_debug_halfgrid",
]
MRF_MATCH_NORM2 = 1
MRF_LLR_LITERAL_EQ23, MRF_LLR_RAW_MAPS, MRF_LLR_MATCH_NORM2 = 1, 2, 4

MRF_DTYPE_F32 = 0
MRF_DTYPE_F64 = 1
# int (*)(void* buf, size_t count, int dtype, void* ctx)
HOST_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p)


class MrfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int), ("L_local", ctypes.c_int), ("frame_offset", ctypes.c_int),
        ("M", ctypes.c_int), ("R", ctypes.c_int),
        ("traj", ctypes.c_void_p), ("frame_interleaf", ctypes.c_void_p),
        ("C", ctypes.c_int), ("coils", ctypes.c_void_p),
        ("W", ctypes.c_int), ("sigma", ctypes.c_float), ("flags", ctypes.c_uint),
        ("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("nccl_comm", ctypes.c_void_p),
        ("batch_frames", ctypes.c_int),
    ]


class MsllrParams(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_float), ("lambda1", ctypes.c_float), ("lambda2", ctypes.c_float),
                ("beta", ctypes.c_float), ("max_iter", ctypes.c_int), ("tol", ctypes.c_double),
                ("sigma2", ctypes.c_double)]


class MsllrInfo(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("cost", ctypes.POINTER(ctypes.c_double)), ("lambda1", ctypes.c_double)]


class CGInfo(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("rel_resid", ctypes.c_double),
                ("history", ctypes.POINTER(ctypes.c_double)), ("alpha", ctypes.POINTER(ctypes.c_double)),
                ("beta", ctypes.POINTER(ctypes.c_double))]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_2310_05647_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, ci, cf = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
    sig = {
        "mrf_plan_create": ([ctypes.POINTER(PlanDesc), ctypes.POINTER(vp)], ci),
        "mrf_forward": ([vp, vp, vp, vp], ci),
        "mrf_adjoint": ([vp, vp, vp, vp], ci),
        "mrf_adjoint_dcf": ([vp, vp, vp, vp], ci),
        "mrf_dcf_weights": ([vp, vp], ci),
        "mrf_normal": ([vp, vp, vp, cf, vp], ci),
        "mrf_dc_cg": ([vp, vp, vp, cf, ci, cf, vp, ctypes.POINTER(CGInfo), vp], ci),
        "mrf_dc_cg_ex": ([vp, vp, vp, cf, ci, cf, ctypes.c_uint, vp, ctypes.POINTER(CGInfo), vp], ci),
        "mrf_plan_destroy": ([vp], ci),
        "mrf_plan_wait": ([vp], ci),
        "mrf_status_string": ([ci], ctypes.c_char_p),
        "mrf_last_error": ([], ctypes.c_char_p),
        "mrf_plan_device_bytes": ([vp], ctypes.c_size_t),
        "mrf_profile_enable": ([vp, ci], ci),
        "mrf_profile_query": ([vp, ci, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong)], ci),
        "mrf_nccl_get_unique_id": ([vp], ci),
        "mrf_nccl_comm_init": ([ctypes.POINTER(vp), ci, vp, ci, ci], ci),
        "mrf_nccl_comm_destroy": ([vp], ci),
        "mrf_plan_set_host_allreduce": ([vp, HOST_ALLREDUCE_FN, vp], ci),
        "mrf_plan_set_precond_shift": ([vp, ctypes.c_double], ci),
        "mrf_dict_create": ([vp, vp, ci, ci, ci, ci, ctypes.POINTER(vp)], ci),
        "mrf_dict_match": ([vp, vp, ctypes.c_longlong, vp, vp, vp, vp], ci),
        "mrf_dict_match_coef": ([vp, vp, ctypes.c_longlong, vp, vp, vp, vp], ci),
        "mrf_dict_match_ex": ([vp, vp, ctypes.c_longlong, ctypes.c_uint, vp, vp, vp, vp], ci),
        "mrf_dict_match_coef_ex": ([vp, vp, ctypes.c_longlong, ctypes.c_uint, vp, vp, vp, vp], ci),
        "mrf_llr_set_options": ([vp, ctypes.c_uint], ci),
        "mrf_plan_debug_halfgrid": ([vp, vp, ctypes.c_size_t], ci),
        "mrf_dict_destroy": ([vp], ci),
        "mrf_dict_overflow": ([vp, ctypes.POINTER(ci)], ci),
        "mrf_dict_filter_info": ([vp, ctypes.POINTER(ci), ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double)], ci),
        "mrf_dict_profile": ([vp, ci], ci),
        "mrf_dict_profile_query": ([vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong)], ci),
        "mrf_dict_basis": ([vp, ctypes.c_double, ci, ctypes.POINTER(ci)], ci),
        "mrf_dict_basis_copy": ([vp, vp], ci),
        "mrf_llr_create": ([vp, ci, ci, ci, ctypes.POINTER(vp)], ci),
        "mrf_llr_create_basis": ([vp, ci, ci, ci, ci, ci, ci, ctypes.POINTER(vp)], ci),
        "mrf_llr_create_shard": ([vp, ci, ci, ci, ci, ci, ctypes.POINTER(vp)], ci),
        "mrf_llr_subspace_normal": ([vp, vp, vp, vp, vp], ci),
        "mrf_llr_step": ([vp, vp, vp, vp, cf, cf, cf, cf, vp, ctypes.POINTER(ctypes.c_double),
                          ctypes.POINTER(ctypes.c_double), vp], ci),
        "mrf_llr_laplacian": ([vp, vp, vp, ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_double), vp], ci),
        "mrf_llr_destroy": ([vp], ci),
        "mrf_llr_cost": ([vp, vp, vp, vp, cf, cf, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                          vp], ci),
        "mrf_msllr_solve": ([vp, vp, vp, vp, ctypes.POINTER(MsllrParams), vp, vp, vp, vp, ctypes.POINTER(MsllrInfo),
                             vp], ci),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:   # only an A/B build (MRF_LIB_PATH) may lack symbols; tests/test_abi_cpu.py checks the exports
            if not os.environ.get("MRF_LIB_PATH"):
                raise ImportError(f"{LIB_PATH} does not export {name}")
            continue
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def _check(status: int):
    if status != 0:
        raise MrfError(status, lib.mrf_last_error().decode(errors="replace"))


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _as_c64(t, shape, name):
    if not isinstance(t, torch.Tensor):
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(t, dtype=np.complex64)))
    if t.dtype != torch.complex64:
        raise TypeError(f"{name} must be complex64, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


class Plan:
    """One frame shard of the multi-frame, multi-coil KB-gridding NUFFT operator (mrf_plan)."""

    def __init__(self, N: int, traj, L: int, *, coils=None, W: int = 6, sigma: float = 2.0,
                 frame_interleaf=None, frame_offset: int = 0, deapod: str = "analytic", normal: str = "gridding",
                 device: Optional[int] = None, nccl_comm: Optional[int] = None, batch_frames: int = 0,
                 dcf: bool = False):
        traj_np = np.ascontiguousarray(np.asarray(traj, dtype=np.float32))
        if traj_np.ndim != 3 or traj_np.shape[2] != 2:
            raise ValueError("traj must be [R][M][2] float32")
        self.N, self.L, self.W, self.sigma = int(N), int(L), int(W), float(sigma)
        self.R, self.M = traj_np.shape[0], traj_np.shape[1]
        self.frame_offset = int(frame_offset)
        coils_np = None
        if coils is not None:
            coils_np = np.ascontiguousarray(np.asarray(coils, dtype=np.complex64))
            if coils_np.ndim != 3 or coils_np.shape[1:] != (self.N, self.N):
                raise ValueError("coils must be [C][N][N] complex64")
        self.C = 1 if coils_np is None else coils_np.shape[0]
        fil_np = None
        if frame_interleaf is not None:
            fil_np = np.ascontiguousarray(np.asarray(frame_interleaf, dtype=np.int32))
            if fil_np.shape != (self.L,):
                raise ValueError("frame_interleaf must have shape [L]")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._keep = (traj_np, coils_np, fil_np)
        d = PlanDesc()
        d.N, d.L_local, d.frame_offset, d.M, d.R = self.N, self.L, self.frame_offset, self.M, self.R
        d.traj = traj_np.ctypes.data
        d.frame_interleaf = None if fil_np is None else fil_np.ctypes.data
        d.C = self.C
        d.coils = None if coils_np is None else coils_np.ctypes.data
        d.W, d.sigma = self.W, self.sigma
        d.flags = {"analytic": MRF_DEAPOD_ANALYTIC, "discrete": MRF_DEAPOD_DISCRETE}[deapod] | \
            {"gridding": 0, "toeplitz": MRF_NORMAL_TOEPLITZ}[normal] | (MRF_DCF if dcf else 0)
        d.device = self.device
        d.stream = None
        d.nccl_comm = nccl_comm
        d.batch_frames = int(batch_frames)
        h = ctypes.c_void_p()
        _check(lib.mrf_plan_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h

    # ------------------------------------------------------------------ helpers
    @property
    def x_shape(self):
        return (self.L, self.N, self.N)

    @property
    def y_shape(self):
        return (self.L, self.C, self.M)

    def _stream(self, *tensors):
        if any(t is not None and t.is_cuda for t in tensors):
            return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        return None

    def _like(self, ref: torch.Tensor, shape):
        if ref.is_cuda:
            return torch.empty(shape, dtype=torch.complex64, device=ref.device)
        return torch.empty(shape, dtype=torch.complex64, pin_memory=ref.is_pinned())

    @property
    def device_bytes(self) -> int:
        return int(lib.mrf_plan_device_bytes(self._h))

    # ------------------------------------------------------------------ operators
    def forward(self, x, y=None):
        """y = A x  (Eq. (1))."""
        x = _as_c64(x, self.x_shape, "x")
        y = self._like(x, self.y_shape) if y is None else _as_c64(y, self.y_shape, "y")
        _check(lib.mrf_forward(self._h, _ptr(x), _ptr(y), self._stream(x, y)))
        return y

    def adjoint(self, y, x=None):
        """x = A^H y  (A*)."""
        y = _as_c64(y, self.y_shape, "y")
        x = self._like(y, self.x_shape) if x is None else _as_c64(x, self.x_shape, "x")
        _check(lib.mrf_adjoint(self._h, _ptr(y), _ptr(x), self._stream(x, y)))
        return x

    def adjoint_dcf(self, y, x=None):
        """x = A^H (w . y), w the plan's Pipe-Menon density compensation (plan made with dcf=True)."""
        y = _as_c64(y, self.y_shape, "y")
        x = self._like(y, self.x_shape) if x is None else _as_c64(x, self.x_shape, "x")
        _check(lib.mrf_adjoint_dcf(self._h, _ptr(y), _ptr(x), self._stream(x, y)))
        return x

    def dcf_weights(self) -> np.ndarray:
        """The plan's density compensation weights, float32 [R][M]."""
        w = np.empty((self.R, self.M), dtype=np.float32)
        _check(lib.mrf_dcf_weights(self._h, w.ctypes.data_as(ctypes.c_void_p)))
        return w

    def normal(self, x, mu: float = 0.0, out=None):
        """out = A^H A x + mu x  (A*(A X))."""
        x = _as_c64(x, self.x_shape, "x")
        out = self._like(x, self.x_shape) if out is None else _as_c64(out, self.x_shape, "out")
        _check(lib.mrf_normal(self._h, _ptr(x), _ptr(out), ctypes.c_float(mu), self._stream(x, out)))
        return out

    def dc_cg(self, y, x0=None, z=None, mu: float = 0.01, n_iter: int = 10, tol: float = 0.0, x=None,
              zero_init: bool = False, async_host: bool = False, precond: bool = False):
        """CG solve of (A^H A + mu I) x = A^H y + mu z from x0; returns (x, info dict).

        zero_init=True: x0 = 0 and x is output only (mrf_dc_cg_ex with MRF_CG_ZERO_INIT: no normal
        operator for the initial residual, and no host-to-device copy of x0 on the host path).
        async_host=True (pinned host tensors): MRF_CG_ASYNC_HOST -- the result copy overlaps the
        next call's solve; call ``wait()`` before reading x.
        precond=True: MRF_CG_PRECOND -- PCG with the circulant preconditioner (same solution)."""
        y = _as_c64(y, self.y_shape, "y")
        if x is None:
            x = self._like(y, self.x_shape)
            if x0 is None and not zero_init:
                x.zero_()
            elif x0 is not None:
                x.copy_(_as_c64(x0, self.x_shape, "x0"))
        else:
            x = _as_c64(x, self.x_shape, "x")
            if x0 is not None:
                x.copy_(_as_c64(x0, self.x_shape, "x0"))
        if zero_init and x0 is not None:
            raise ValueError("zero_init excludes x0")
        if z is not None:
            z = _as_c64(z, self.x_shape, "z")
        hist = (ctypes.c_double * (n_iter + 1))()
        ha = (ctypes.c_double * max(n_iter, 1))()
        hb = (ctypes.c_double * max(n_iter, 1))()
        dp = lambda a: ctypes.cast(a, ctypes.POINTER(ctypes.c_double))
        info = CGInfo(0, 0.0, dp(hist), dp(ha), dp(hb))
        _check(lib.mrf_dc_cg_ex(self._h, _ptr(y), _ptr(z), ctypes.c_float(mu), int(n_iter), ctypes.c_float(tol),
                                (1 if zero_init else 0) | (2 if async_host else 0) | (4 if precond else 0), _ptr(x),
                                ctypes.byref(info),
                                self._stream(x, y, z)))
        it = info.iters
        return x, {"iters": it, "rel_resid": info.rel_resid, "history": list(hist)[: it + 1],
                   "alpha": list(ha)[:it], "beta": list(hb)[:it]}

    def set_precond_shift(self, shift: float):
        """gamma = mu + shift * mean(lambda) of the PCG preconditioner (mrf_plan_set_precond_shift)."""
        _check(lib.mrf_plan_set_precond_shift(self._h, ctypes.c_double(shift)))

    def set_host_allreduce(self, fn):
        """Route the plan's rank reductions through a host callable (mrf_plan_set_host_allreduce).

        ``fn(buf)`` receives a numpy float32/float64 array view of the library's pinned staging
        buffer and must replace it in place by its sum over all ranks (e.g. a gloo
        ``torch.distributed.all_reduce`` on ``torch.from_numpy(buf)``).  ``fn=None`` restores NCCL."""
        if fn is None:
            self._host_ar = None
            _check(lib.mrf_plan_set_host_allreduce(self._h, HOST_ALLREDUCE_FN(), None))
            return

        def tramp(buf, count, dtype, _ctx):
            try:
                ct = ctypes.c_double if dtype == MRF_DTYPE_F64 else ctypes.c_float
                arr = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ct)), shape=(int(count),))
                fn(arr)
                return 0
            except Exception:   # reported to the library as MRF_ENCCL
                import traceback
                traceback.print_exc()
                return 1

        self._host_ar = HOST_ALLREDUCE_FN(tramp)   # keep the trampoline alive with the plan
        _check(lib.mrf_plan_set_host_allreduce(self._h, self._host_ar, None))

    def debug_halfgrid(self, frames: int) -> np.ndarray:
        """The first lane's half-grid workspace (mrf_plan_debug_halfgrid; test hook), `frames` =
        the plan's batch size: complex64 [frames * C * N * G]."""
        out = np.empty(frames * self.C * self.N * int(round(self.sigma * self.N)), dtype=np.complex64)
        _check(lib.mrf_plan_debug_halfgrid(self._h, out.ctypes.data_as(ctypes.c_void_p), out.nbytes))
        return out

    def wait(self):
        """Waits for the result copies of async_host solves (mrf_plan_wait)."""
        _check(lib.mrf_plan_wait(self._h))

    # ------------------------------------------------------------------ profiling
    def profile(self, enable: bool = True):
        _check(lib.mrf_profile_enable(self._h, int(bool(enable))))

    def profile_query(self, cls: str):
        ms = ctypes.c_double()
        n = ctypes.c_longlong()
        _check(lib.mrf_profile_query(self._h, KERNEL_CLASSES[cls], ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    # ------------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_h", None):
            _check(lib.mrf_plan_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ---------------------------------------------------------------------- NCCL communicator
def nccl_comm_create(rank: int, world: int, device: int):
    """ncclComm_t for the CG inner-product all-reduce; the 128-byte id is broadcast over the
    default torch.distributed process group (any backend)."""
    import torch.distributed as dist
    buf = (ctypes.c_ubyte * 128)()
    if rank == 0:
        _check(lib.mrf_nccl_get_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        t = t.cuda(device)
    dist.broadcast(t, 0)
    idb = bytes(t.cpu().tolist())
    ctypes.memmove(buf, idb, 128)
    comm = ctypes.c_void_p()
    _check(lib.mrf_nccl_comm_init(ctypes.byref(comm), int(world), ctypes.cast(buf, ctypes.c_void_p), int(rank),
                                  int(device)))
    return comm.value


def nccl_comm_destroy(comm):
    if comm:
        _check(lib.mrf_nccl_comm_destroy(ctypes.c_void_p(comm)))


class Dictionary:
    """Dictionary matching Phi_D (Eq. (5); include/mrfnufft.h mrf_dict_*).

    atoms: [K][L] complex64 (host); lut: [K][P] float32 parameters (e.g. T1, T2) or None.
    match(x) takes the frame-major image stack x [L][...voxels] (CUDA complex64) and returns
    (index int32 [V], pd float32 [V], params float32 [V][P] or None) on x's device.
    """

    def __init__(self, atoms, lut=None, device: Optional[int] = None):
        a = np.ascontiguousarray(np.asarray(atoms, dtype=np.complex64))
        if a.ndim != 2:
            raise ValueError("atoms must be [K][L]")
        self.K, self.L = a.shape
        lt = None if lut is None else np.ascontiguousarray(np.asarray(lut, dtype=np.float32))
        self.P = 0 if lt is None else lt.reshape(self.K, -1).shape[1]
        self.device = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        _check(lib.mrf_dict_create(a.ctypes.data_as(ctypes.c_void_p),
                                   None if lt is None else lt.ctypes.data_as(ctypes.c_void_p),
                                   self.K, self.L, self.P, self.device, ctypes.byref(h)))
        self._h = h

    def match(self, x: torch.Tensor, norm2: bool = False):
        """Exact Phi_D of the frame-major stack x [L][...voxels]; norm2=True: Eq. (5) as printed
        (||d||^2 denominator, mrf_dict_match_ex with MRF_MATCH_NORM2)."""
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.complex64 and x.is_contiguous()):
            raise TypeError("x must be a contiguous CUDA complex64 tensor [L][...]")
        if x.shape[0] != self.L:
            raise ValueError(f"x must have {self.L} frames, got {x.shape[0]}")
        V = x.numel() // self.L
        index = torch.empty(V, dtype=torch.int32, device=x.device)
        pd = torch.empty(V, dtype=torch.float32, device=x.device)
        params = torch.empty((V, self.P), dtype=torch.float32, device=x.device) if self.P else None
        st = torch.cuda.current_stream(x.device).cuda_stream
        _check(lib.mrf_dict_match_ex(self._h, _ptr(x), V, MRF_MATCH_NORM2 if norm2 else 0, _ptr(index), _ptr(pd),
                                     _ptr(params), ctypes.c_void_p(st)))
        return index, pd, params

    def match_coef(self, u: torch.Tensor, norm2: bool = False):
        """Phi_D of voxels in basis coordinates u [r][...voxels] (CUDA complex64), x_v = sum_i u[i, v] d_i
        (mrf_dict_match_coef; needs basis())."""
        if not (isinstance(u, torch.Tensor) and u.is_cuda and u.dtype == torch.complex64 and u.is_contiguous()):
            raise TypeError("u must be a contiguous CUDA complex64 tensor [r][...]")
        V = u.numel() // u.shape[0]
        index = torch.empty(V, dtype=torch.int32, device=u.device)
        pd = torch.empty(V, dtype=torch.float32, device=u.device)
        params = torch.empty((V, self.P), dtype=torch.float32, device=u.device) if self.P else None
        st = torch.cuda.current_stream(u.device).cuda_stream
        _check(lib.mrf_dict_match_coef_ex(self._h, _ptr(u), V, MRF_MATCH_NORM2 if norm2 else 0, _ptr(index), _ptr(pd),
                                          _ptr(params), ctypes.c_void_p(st)))
        return index, pd, params

    def overflow(self) -> int:
        """Voxels of the last match rescored against every atom (mrf_dict_overflow)."""
        n = ctypes.c_int()
        _check(lib.mrf_dict_overflow(self._h, ctypes.byref(n)))
        return n.value

    def filter_info(self):
        """(Rf, beta, max residual) of the certified filter (mrf_dict_filter_info)."""
        r, b, res = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        _check(lib.mrf_dict_filter_info(self._h, ctypes.byref(r), ctypes.byref(b), ctypes.byref(res)))
        return r.value, b.value, res.value

    def basis(self, energy: float = 0.9999, max_rank: int = 32) -> np.ndarray:
        """Subspace basis of P_S (Eq. 17): [r][L] complex64 orthonormal rows (mrf_dict_basis)."""
        r = ctypes.c_int()
        _check(lib.mrf_dict_basis(self._h, ctypes.c_double(energy), int(max_rank), ctypes.byref(r)))
        d = np.empty((r.value, self.L), dtype=np.complex64)
        _check(lib.mrf_dict_basis_copy(self._h, d.ctypes.data_as(ctypes.c_void_p)))
        return d

    def profile(self, enable: bool = True):
        _check(lib.mrf_dict_profile(self._h, int(enable)))

    def profile_query(self):
        """(milliseconds, launches) of the tensor-core GEMM since profile(True)."""
        ms, n = ctypes.c_double(), ctypes.c_longlong()
        _check(lib.mrf_dict_profile_query(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def close(self):
        if getattr(self, "_h", None):
            lib.mrf_dict_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LLR:
    """The (MS-)LLR outer step of Algorithm 1 (include/mrfnufft.h mrf_llr_*, mrf_msllr_solve).

    Needs ``dictionary.basis(...)`` first.  ``step(plan, x, rhs, mu, lam2, beta)`` returns
    (x_next, nuclear, penalty) for CUDA complex64 [L][N][N] x and rhs = A^H b; ``laplacian``
    builds the manifold term's graph Laplacian from Phi_D's maps; ``cost`` evaluates Algorithm 1's
    cost; ``solve`` runs Algorithm 1 end to end.
    """

    def __init__(self, dictionary: "Dictionary", N: int, p: int = 11, s: int = 5):
        h = ctypes.c_void_p()
        _check(lib.mrf_llr_create(dictionary._h, int(N), int(p), int(s), ctypes.byref(h)))
        self._h = h
        self.N, self.L = int(N), dictionary.L
        self.r = None

    @classmethod
    def from_basis(cls, basis, N: int, p: int = 11, s: int = 5, device: Optional[int] = None) -> "LLR":
        """An operator with a caller-supplied basis d ([r][L] complex, orthonormal rows; mrf_llr_create_basis)."""
        d = np.ascontiguousarray(np.asarray(basis, dtype=np.complex64))
        if d.ndim != 2:
            raise ValueError("basis must be [r][L]")
        self = cls.__new__(cls)
        h = ctypes.c_void_p()
        dev = torch.cuda.current_device() if device is None else device
        _check(lib.mrf_llr_create_basis(d.ctypes.data_as(ctypes.c_void_p), d.shape[0], d.shape[1], int(N), int(p),
                                        int(s), dev, ctypes.byref(h)))
        self._h = h
        self.N, self.L, self.r = int(N), d.shape[1], d.shape[0]
        return self

    @classmethod
    def shard(cls, dictionary: "Dictionary", frame0: int, L_local: int, N: int, p: int = 11,
              s: int = 5) -> "LLR":
        """The operator for frames [frame0, frame0 + L_local) of the dictionary's basis
        (mrf_llr_create_shard); with a plan carrying the ranks' NCCL communicator the coefficient
        partials are all-reduced inside every call."""
        self = cls.__new__(cls)
        h = ctypes.c_void_p()
        _check(lib.mrf_llr_create_shard(dictionary._h, int(frame0), int(L_local), int(N), int(p), int(s),
                                        ctypes.byref(h)))
        self._h = h
        self.N, self.L, self.r = int(N), int(L_local), None
        return self

    def set_options(self, literal_eq23: bool = False, raw_maps: bool = False, match_norm2: bool = False):
        """The printed-form switches (mrf_llr_set_options): Eq. (23)'s scalar denominator, Eq. (8)
        on raw maps, Eq. (5)'s ||d||^2 denominator in Phi_D (readings 25, 26, 21)."""
        o = (MRF_LLR_LITERAL_EQ23 if literal_eq23 else 0) | (MRF_LLR_RAW_MAPS if raw_maps else 0) | \
            (MRF_LLR_MATCH_NORM2 if match_norm2 else 0)
        _check(lib.mrf_llr_set_options(self._h, o))

    def subspace_normal(self, plan: "Plan", u, z=None):
        """Coefficients of P_S A^H A (sum_i u_i d_i) for u [r][N][N] on a Toeplitz plan (mrf_llr_subspace_normal)."""
        if not (isinstance(u, torch.Tensor) and u.is_cuda and u.dtype == torch.complex64 and u.is_contiguous()):
            raise TypeError("u must be a contiguous CUDA complex64 tensor [r][N][N]")
        z = torch.empty_like(u) if z is None else z
        st = torch.cuda.current_stream(u.device).cuda_stream
        _check(lib.mrf_llr_subspace_normal(self._h, plan._h, _ptr(u), _ptr(z), ctypes.c_void_p(st)))
        return z

    def laplacian(self, params: torch.Tensor, pd: torch.Tensor, sigma2: float = 0.0):
        """Graph Laplacian from Phi_D's maps (params [V][2] T1/T2, pd [V]; CUDA float32).
        Returns (sigma2, max_degree)."""
        params = params.contiguous().float()
        pd = pd.contiguous().float()
        s2, md = ctypes.c_double(), ctypes.c_double()
        st = torch.cuda.current_stream(params.device).cuda_stream
        _check(lib.mrf_llr_laplacian(self._h, _ptr(params), _ptr(pd), ctypes.c_double(sigma2), ctypes.byref(s2),
                                     ctypes.byref(md), ctypes.c_void_p(st)))
        return s2.value, md.value

    def step(self, plan: "Plan", x, rhs, mu: float = 1.0, lam2: float = 0.1, beta: float = 0.2, x_out=None,
             nuclear: bool = True, lam1: float = 0.0, penalty: bool = False):
        """One iteration of Algorithm 1; returns (x_next, nuclear or None, penalty or None)."""
        shape = (self.L, self.N, self.N)
        x = _as_c64(x, shape, "x")
        rhs = _as_c64(rhs, shape, "rhs")
        if not (x.is_cuda and rhs.is_cuda):
            raise TypeError("x and rhs must be CUDA tensors")
        x_out = torch.empty_like(x) if x_out is None else _as_c64(x_out, shape, "x_out")
        nuc, pen = ctypes.c_double(), ctypes.c_double()
        st = torch.cuda.current_stream(x.device).cuda_stream
        _check(lib.mrf_llr_step(self._h, plan._h, _ptr(x), _ptr(rhs), ctypes.c_float(mu), ctypes.c_float(lam1),
                                ctypes.c_float(lam2), ctypes.c_float(beta), _ptr(x_out),
                                ctypes.byref(nuc) if nuclear else None, ctypes.byref(pen) if penalty else None,
                                ctypes.c_void_p(st)))
        return x_out, (nuc.value if nuclear else None), (pen.value if penalty else None)

    def cost(self, plan: "Plan", x, b, lam1: float = 0.0, lam2: float = 0.1):
        """Algorithm 1's cost at x (b = k-space [L][C][M]): (cost, (data, manifold, nuclear))."""
        x = _as_c64(x, (self.L, self.N, self.N), "x")
        if not (x.is_cuda and b.is_cuda and b.dtype == torch.complex64 and b.is_contiguous()):
            raise TypeError("x and b must be contiguous CUDA complex64 tensors")
        c = ctypes.c_double()
        t = (ctypes.c_double * 3)()
        st = torch.cuda.current_stream(x.device).cuda_stream
        _check(lib.mrf_llr_cost(self._h, plan._h, _ptr(x), _ptr(b), ctypes.c_float(lam1), ctypes.c_float(lam2),
                                ctypes.byref(c), t, ctypes.c_void_p(st)))
        return c.value, (t[0], t[1], t[2])

    def solve(self, dictionary: "Dictionary", plan: "Plan", b, mu: float = 1.0, lam1: float = 0.0,
              lam2: float = 0.1, beta: float = 0.2, max_iter: int = 10, tol: float = 1e-5, sigma2: float = 0.0,
              costs: bool = True):
        """Algorithm 1 (mrf_msllr_solve).  Returns dict(x, index, pd, params, iters, cost, lambda1).
        costs=False with tol <= 0: cost(n) is not evaluated (cost = [])."""
        if not (isinstance(b, torch.Tensor) and b.is_cuda and b.dtype == torch.complex64 and b.is_contiguous()):
            raise TypeError("b must be a contiguous CUDA complex64 tensor [L][C][M]")
        dev = b.device
        V = self.N * self.N
        x = torch.empty((self.L, self.N, self.N), dtype=torch.complex64, device=dev)
        index = torch.empty(V, dtype=torch.int32, device=dev)
        pd = torch.empty(V, dtype=torch.float32, device=dev)
        params = torch.empty((V, dictionary.P), dtype=torch.float32, device=dev) if dictionary.P else None
        prm = MsllrParams(mu, lam1, lam2, beta, int(max_iter), tol, sigma2)
        cost = (ctypes.c_double * max(int(max_iter), 1))()
        info = MsllrInfo(0, ctypes.cast(cost, ctypes.POINTER(ctypes.c_double)) if costs else None, 0.0)
        st = torch.cuda.current_stream(dev).cuda_stream
        _check(lib.mrf_msllr_solve(self._h, dictionary._h, plan._h, _ptr(b), ctypes.byref(prm), _ptr(x), _ptr(index),
                                   _ptr(pd), _ptr(params), ctypes.byref(info), ctypes.c_void_p(st)))
        return {"x": x, "index": index, "pd": pd, "params": params, "iters": info.iters,
                "cost": [cost[i] for i in range(info.iters)] if costs else [], "lambda1": info.lambda1}

    def close(self):
        if getattr(self, "_h", None):
            lib.mrf_llr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


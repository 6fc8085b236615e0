/*
 * mrfnufft.h -- C-ABI of the B200-native (sm_100a) data-consistency operator of MS-LLR
 * MR fingerprinting reconstruction (Li, Ji, Hu, arxiv 2310.05647).
 *
 * What it computes (the "acquisition operator" of the paper):
 *   b = A X + n,  A = F_u C                       PAPER.md:56-60 (§II-B, Eq. (1) data_ac)
 *   X in C^{Nx x Ny x L} image frames, b in C^{Nc x Ns x L} k-space, C = coil sensitivities,
 *   F_u = per-frame non-Cartesian (spiral) undersampled Fourier transform.
 *   The paper evaluates F_u with a GPU NUFFT library (§III-D, §V) and
 *   uses A* in the gradient A*(A X - b) (Eq. (15)) and in the
 *   initialisation X^0 = A* b (Alg. 1).  BASELINE.json's north_star adds the exact
 *   data-consistency solve (A^H A + mu I) x = A^H y + mu z by conjugate gradients.
 *
 * Conventions:
 *   - image frame x_l[iy][ix] (x fastest), centred indices n = (ix - N/2, iy - N/2);
 *   - trajectory k in cycles/pixel, |k| <= 0.5 inclusive (+0.5 == -0.5);
 *   - A:   y[l][c][j] = (1/N) sum_n S_c[n] x_l[n] exp(-i 2 pi k_{l,j} . n)   (approximated by
 *          Kaiser-Bessel gridding: width W, oversampling sigma = 2, Beatty beta, open support,
 *          deapodisation by the kernel's continuous Fourier transform unless
 *          MRF_DEAPOD_DISCRETE);
 *   - A^H: the exact transpose of the gridding forward (conj coils, e^{+i}, same taps).
 *   - frame l (local index) samples interleaf frame_interleaf[l], default
 *     (frame_offset + l) mod R.
 *
 * Memory: every complex array is interleaved complex64 (float real, float imag), C-contiguous:
 *   x, z, out  [L_local][N][N]     y  [L_local][C][M]     coils [C][N][N]     traj [R][M][2]
 * Every array must be 16-byte aligned (MRF_EINVAL otherwise; torch/cudaMalloc allocations are).
 * Array arguments of the operator calls may be DEVICE pointers (on the plan's device; fully
 * asynchronous on `stream`, CUDA-graph capturable, no allocation) or HOST pointers (pinned or
 * pageable; the call stages them through plan-owned device buffers allocated on first use and
 * returns only after the result is back in host memory).  Device and host pointers may not be
 * mixed within one call.
 *
 * Errors: every call returns an mrf_status; MRF_OK == 0.  mrf_last_error() returns a
 * thread-local human-readable message for the most recent failure.  On any error the output
 * buffers are unspecified.
 */
#ifndef MRFNUFFT_H
#define MRFNUFFT_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mrf_plan_s* mrf_plan;          /* opaque; owns all derived device data */

typedef enum {
  MRF_OK = 0,
  MRF_EINVAL = 1,        /* null required pointer, bad size, |k| > 0.5 or non-finite k, W out of
                            [2,16], mu < 0, n_iter < 0, mixed host/device pointers            */
  MRF_ENOMEM = 2,        /* device or host allocation failed                                    */
  MRF_ECUDA = 3,         /* CUDA runtime error (message in mrf_last_error)                      */
  MRF_ENCCL = 4,         /* NCCL unavailable or a collective failed                             */
  MRF_EUNSUPPORTED = 5,  /* sigma != 2, G = sigma*N not in {64,...,1024}, or unsupported mode  */
  MRF_ENUMERIC = 6       /* CG breakdown: Re<p, (A^H A + mu I) p> <= 0 or non-finite           */
} mrf_status;

/* flags */
#define MRF_DEAPOD_ANALYTIC 0u   /* psi = continuous FT of the KB kernel (default)               */
#define MRF_DEAPOD_DISCRETE 1u   /* psi = DFT of the integer-sampled kernel (exact on-grid)      */
/* mrf_normal and mrf_dc_cg evaluate A^H A by Toeplitz embedding:
 * A^H A x = sum_c conj(S_c) crop(IFFT_2N(T_r . FFT_2N(pad(S_c x)))), T_r the real 2N x 2N spectrum of
 * the exact point-spread function of interleaf r (computed in float64 at plan creation).  This is
 * the exact (NUDFT) normal operator up to fp32 rounding -- it differs from the gridding A^H(A x) by
 * the NUFFT approximation error (~1e-5).  forward/adjoint are unchanged.  Costs R*(2N)^2*4 bytes. */
#define MRF_NORMAL_TOEPLITZ 2u
/* Density compensation (reading 23): the plan
 * computes per-sample weights w[r][j] by 20 Pipe-Menon iterations w <- w / (Phi Phi^T w) on the
 * sigma*N grid with the gridding taps (float64, at plan creation) for mrf_adjoint_dcf, the
 * density-compensated initialisation X^0 = A^H (w . b) ("X^0 = A* b"). */
#define MRF_DCF 4u

typedef struct {
  int N;                        /* square image side, even; G = sigma*N must be a supported size */
  int L_local;                  /* frames held by this plan (this rank's shard), >= 1           */
  int frame_offset;             /* global index of local frame 0 (default interleaf map)        */
  int M;                        /* nonuniform points per frame, >= 1                            */
  int R;                        /* distinct interleaves in traj, >= 1                            */
  const float* traj;            /* HOST [R][M][2] (kx, ky) cycles/pixel; copied at create       */
  const int* frame_interleaf;   /* HOST [L_local] in [0,R), or NULL => (frame_offset+l) mod R   */
  int C;                        /* coils >= 1                                                    */
  const float* coils;           /* HOST [C][N][N] complex64, or NULL with C == 1 => S = 1       */
  int W;                        /* Kaiser-Bessel width, 2..16                                    */
  float sigma;                  /* oversampling factor; 2.0 supported                            */
  unsigned flags;               /* MRF_DEAPOD_* | MRF_NORMAL_TOEPLITZ                            */
  int device;                   /* CUDA device ordinal                                           */
  void* stream;                 /* cudaStream_t for create-time uploads (NULL = legacy default)  */
  void* nccl_comm;              /* ncclComm_t shared by all ranks of one solve, or NULL          */
  int batch_frames;             /* frames per on-chip batch of the gridding pipeline; 0 = auto   */
} mrf_plan_desc;

/* Validates the descriptor, evaluates the KB kernel/deapodisation constants in float64 on the
 * host, bins every interleaf's points into column strips of the oversampled grid, uploads
 * everything and allocates all workspaces.  Caller keeps ownership of desc's host arrays. */
mrf_status mrf_plan_create(const mrf_plan_desc* desc, mrf_plan* out);

/* y = A x  (Eq. (1) without noise).  x [L][N][N], y [L][C][M]. */
mrf_status mrf_forward(mrf_plan plan, const void* x, void* y, void* stream);

/* x = A^H y  (the adjoint A* of PAPER.md:221; X^0 = A* b of Alg. 1). */
mrf_status mrf_adjoint(mrf_plan plan, const void* y, void* x, void* stream);

/* out = A^H A x + mu x  (the normal operator inside A*(A X^n - b), Eq. (15)).
 * out must not alias x; mu >= 0. */
mrf_status mrf_normal(mrf_plan plan, const void* x, void* out, float mu, void* stream);

/* x = A^H (w . y): the adjoint of the density-compensated k-space (plan created with MRF_DCF;
 * else MRF_EINVAL).  Layouts, pointers and errors as mrf_adjoint. */
mrf_status mrf_adjoint_dcf(mrf_plan plan, const void* y, void* x, void* stream);
/* Copies the plan's weights, HOST float [R][M], into w (MRF_DCF plans; else MRF_EINVAL). */
mrf_status mrf_dcf_weights(mrf_plan plan, float* w);

typedef struct {
  int iters;               /* CG iterations performed                                           */
  double rel_resid;        /* sqrt(rho_last / rho_0), rho = <r, r> global over all ranks        */
  double* history;         /* nullable HOST array of length n_iter+1: history[k] = sqrt(rho_k)  */
  double* alpha;           /* nullable HOST array of length n_iter: the step lengths alpha_k    */
  double* beta;            /* nullable HOST array of length n_iter: beta_k = rho_{k+1} / rho_k  */
} mrf_cg_info;

/* Solves (A^H A + mu I) x = A^H y + mu z by CG from x (in: x0, out: solution), inner products
 * <a,b> = sum conj(a) b over ALL frames of ALL ranks, accumulated in float64 (and all-reduced
 * with NCCL when the plan has a communicator: every rank must call with the same mu, n_iter,
 * tol).  z may be NULL (=> 0).  tol == 0 runs exactly n_iter iterations with no host
 * synchronisation inside the loop; tol > 0 stops once sqrt(rho_k/rho_0) < tol.  Iteration as in
 * SURVEY.md §8(c)(ii) step 7.  The call synchronises `stream` once at the end to fill `info`
 * and check for breakdown. */
mrf_status mrf_dc_cg(mrf_plan plan, const void* y, const void* z, float mu, int n_iter, float tol,
                     void* x, mrf_cg_info* info, void* stream);

/* mrf_dc_cg with flags.  MRF_CG_ZERO_INIT: the initial guess is x0 = 0 (Algorithm 1's CG from
 * rest) and x is output only: neither read nor (on the host path) copied in, and the initial
 * residual is r = rhs without an application of the normal operator.  Same iterates as
 * mrf_dc_cg on a zeroed x.  Unknown flags: MRF_EINVAL. */
#define MRF_CG_ZERO_INIT 1u
/* MRF_CG_ASYNC_HOST (host buffers only, else MRF_EINVAL): pipelined host path for a stream of
 * solves.  The call copies y (and x0 / z) into one of two device slots on `stream`, solves there,
 * and copies the result to the host x on the plan's own copy stream, then returns without waiting
 * for that copy: the result copy of call k overlaps the solve of call k+1 (PCIe is full duplex;
 * call k+2 reuses the slot after call k's copy).  The host buffers of a call stay in use until
 * mrf_plan_wait returns; pinned host memory is needed for the overlap.  `info`, if given, is
 * filled as usual (that synchronises `stream`, not the copy stream). */
#define MRF_CG_ASYNC_HOST 2u
/* MRF_CG_PRECOND: preconditioned CG (reading 28) -- same system,
 * same solution, other iterates.  Per frame M = C + gamma I, C = T. Chan's optimal circulant of the
 * frame's exact normal operator (eigenvalues lambda_m = ||A f_m||^2 at the Fourier vectors f_m,
 * PAPER.md:217's A^H A, computed in float64 per interleaf on the first such call and scaled by the
 * mean coil power), gamma = mu + shift * mean(lambda) (shift: mrf_plan_set_precond_shift, default
 * 30).  z = M^-1 r costs a 2D FFT pair over the frames (three passes).  history / rel_resid /
 * tol report the true residual ||r||; alpha, beta are the PCG step lengths.  Costs 2 more image
 * stacks of device memory. */
#define MRF_CG_PRECOND 4u
mrf_status mrf_dc_cg_ex(mrf_plan plan, const void* y, const void* z, float mu, int n_iter, float tol,
                        unsigned flags, void* x, mrf_cg_info* info, void* stream);
/* The preconditioner's shift (MRF_CG_PRECOND): gamma = mu + shift * mean(lambda); shift >= 0,
 * finite (else MRF_EINVAL).  Synchronises the device (cached CUDA graphs of PCG solves are dropped). */
mrf_status mrf_plan_set_precond_shift(mrf_plan plan, double shift);
/* Waits for every result copy of MRF_CG_ASYNC_HOST calls on the plan.  Errors: MRF_EINVAL, MRF_ECUDA. */
mrf_status mrf_plan_wait(mrf_plan plan);

mrf_status mrf_plan_destroy(mrf_plan plan);

const char* mrf_status_string(mrf_status status);
const char* mrf_last_error(void);

/* ---- plan introspection ---------------------------------------------------------------- */
/* Bytes of device memory the plan owns (tables, coils, workspaces, CG vectors). */
size_t mrf_plan_device_bytes(mrf_plan plan);

/* Test hook (stage-wise parity): copies the half-grid workspace of the plan's first
 * batch lane into dst (host or device, `bytes` = batch_frames * C * N * G * 8, else MRF_EINVAL) after
 * synchronising the device.  After mrf_forward on a one-batch plan it holds the row-FFT'd padded
 * image, strip-major [frame * C + c][G/16][N][16] (image row iy, grid column 16 s + j); after
 * mrf_adjoint the column-iFFT'd spread grid at the N kept rows, row-major [frame * C + c][N][G].
 * Not part of the computation's API: nothing reads it back. */
mrf_status mrf_plan_debug_halfgrid(mrf_plan plan, void* dst, size_t bytes);

/* ---- per-kernel timing (CUDA events on the launching stream) ----------------------------- */
/* Kernel classes for mrf_profile_query. */
#define MRF_K_FWD_ROWS      0   /* deapod . coil . pad . row FFT                                */
#define MRF_K_FWD_COLS      1   /* column FFT + KB gather interpolation                          */
#define MRF_K_ADJ_COLS      2   /* KB spread + column inverse FFT + row crop                     */
#define MRF_K_ADJ_ROWS      3   /* row inverse FFT + crop + deapod + conj-coil sum               */
#define MRF_K_CG_VEC        4   /* CG vector updates and inner products                          */
#define MRF_K_OTHER         5   /* memsets, reductions                                            */
#define MRF_K_COUNT         6
/* enable != 0 brackets every subsequent kernel launch with CUDA events (and resets counters). */
mrf_status mrf_profile_enable(mrf_plan plan, int enable);
/* Synchronises the recorded events and returns total milliseconds and launch count of a class. */
mrf_status mrf_profile_query(mrf_plan plan, int kernel_class, double* total_ms, long long* launches);

/* ---- NCCL helpers (NCCL is loaded at run time; no link-time dependency) ------------------- */
/* Writes the 128-byte ncclUniqueId into id_out. */
mrf_status mrf_nccl_get_unique_id(void* id_out128);
/* Creates an ncclComm_t on the current device; *comm_out receives it. */
mrf_status mrf_nccl_comm_init(void** comm_out, int nranks, const void* id128, int rank, int device);
mrf_status mrf_nccl_comm_destroy(void* comm);

/* ---- host-side reduction hook (frame sharding without NCCL) -------------------------------
 * The frame-sharded solve (the operator is block-diagonal over frames,
 * PAPER.md:60, so the only coupling between ranks is the sum over frames inside the CG inner
 * products and the coefficient projection of mrf_llr_step) needs one primitive: an in-place
 * SUM of a small buffer over all ranks.  By default it is ncclAllReduce on the plan's
 * communicator (mrf_plan_desc.nccl_comm).  mrf_plan_set_host_allreduce replaces it by a host
 * callback, for process layouts NCCL cannot serve (several ranks on one GPU: the multi-rank
 * tests, or a gloo/MPI job): every all-reduce the plan (and an mrf_llr operator called with it)
 * performs then copies the device buffer into plan-owned pinned host memory on the call's
 * stream, synchronises the stream, calls fn(buf, count, dtype, ctx) -- which must replace the
 * `count` elements at `buf` (HOST) by their sum over all ranks and return 0 -- and copies the
 * result back.  dtype is MRF_DTYPE_F32 or MRF_DTYPE_F64.  The calls happen on the calling
 * thread in the same order on every rank; a non-zero return makes the operation fail with
 * MRF_ENCCL.  This inserts host synchronisations, so such a plan's mrf_dc_cg is not CUDA-graph
 * capturable.  fn = NULL restores the plan's NCCL communicator (or no reduction).
 * Errors: MRF_EINVAL (null plan). */
#define MRF_DTYPE_F32 0
#define MRF_DTYPE_F64 1
typedef int (*mrf_host_allreduce_fn)(void* buf, size_t count, int dtype, void* ctx);
mrf_status mrf_plan_set_host_allreduce(mrf_plan plan, mrf_host_allreduce_fn fn, void* ctx);

/* ---- dictionary matching Phi_D (Eqs. (4)-(5)) -------------
 *
 *   k_v   = argmax_k |<d_k, x_v>| / ||d_k||_2        ties -> lowest k   (reading 21)
 *   pd_v  = max(Re<d_k, x_v> / ||d_k||_2^2, 0)       eta_v = LUT[k_v]
 *
 * with <d, x> = sum_l conj(d_l) x_l over the L frames.  The argmax is exact: a certified filter on
 * the tensor cores lists every atom that can be the best, and the listed atoms are rescored from the
 * complex64 data with float64 accumulation (ties -> lowest index).  Filter: the dictionary's leading
 * Rf <= 64 right singular vectors phi (computed at mrf_dict_create); for any x,
 * <d_k, x> = <phi d_k, phi x> + <r_k, x> with r_k = (I - phi^H phi) d_k, so the normalised
 * correlation rho = |<d, x>| / (||d|| ||x||) is approximated by a 3xFP16 tcgen05 GEMM of the
 * coefficients to within a bound beta that adds max_k ||r_k|| / ||d_k|| (float64), the projection's
 * fp32 rounding, the split-operand rounding and the worst-case fp32 accumulation; every atom within
 * 2 beta of the filter's best is rescored.  A voxel with more than 32 such atoms is rescored
 * against every atom (mrf_dict_overflow counts them), so the result never depends on the filter;
 * a dictionary without a compressible spectrum is slower, never wrong.  pd uses the exact <d_k, x>. */
typedef struct mrf_dict_s* mrf_dict;

/* atoms: HOST [K][L] complex64 (interleaved re, im), copied; lut: HOST [K][P] float (P >= 0
 * parameters per atom, e.g. T1, T2; NULL if P == 0), copied.  K >= 1, 1 <= L <= 65536.  Builds the
 * filter basis (subspace iteration on D^H D, float64 residuals; synchronous).
 * Errors: MRF_EINVAL (sizes / NULL), MRF_ENOMEM, MRF_ECUDA.  An all-zero atom is never matched. */
mrf_status mrf_dict_create(const void* atoms, const float* lut, int K, int L, int P, int device, mrf_dict* out);

/* x: DEVICE [L][V] complex64, frame-major (the layout of the image stack, voxel fastest).
 * index: DEVICE int32 [V]; pd: DEVICE float [V]; params: DEVICE float [V][P] or NULL.  All
 * 16-byte aligned.  Asynchronous on `stream`; workspaces (a voxel-major copy of x, V x 8L bytes,
 * and V x ~1 KB) are allocated on first use and grown as needed (that call synchronises).  A zero
 * voxel gets index 0, pd 0.  Errors: MRF_EINVAL, MRF_ENOMEM, MRF_ECUDA. */
mrf_status mrf_dict_match(mrf_dict dict, const void* x, long long V, int* index, float* pd, float* params,
                          void* stream);
/* mrf_dict_match with flags.  MRF_MATCH_NORM2: Eq. (5) as printed, k = argmax |<d_k, x>| /
 * ||d_k||_2^2 (reading 21 uses ||d_k||_2: with atoms of unequal norm the printed
 * form prefers low-norm atoms).  Same exact-argmax machinery (the band is widened by 1/min ||d_k||).
 * Unknown flags: MRF_EINVAL. */
#define MRF_MATCH_NORM2 1u
mrf_status mrf_dict_match_ex(mrf_dict dict, const void* x, long long V, unsigned flags, int* index, float* pd,
                             float* params, void* stream);
/* Voxels of the last match that were rescored against every atom (more than 32 atoms inside the
 * certified band); synchronises.  The filter: *rank = Rf, *beta = the bound on the normalised
 * correlation, *residual = max_k ||r_k|| / ||d_k|| (nullable outputs). */
mrf_status mrf_dict_overflow(mrf_dict dict, int* voxels);
mrf_status mrf_dict_filter_info(mrf_dict dict, int* rank, double* beta, double* residual);

mrf_status mrf_dict_destroy(mrf_dict dict);

/* ---- subspace basis and the LLR outer step (lambda_1 = 0: the paper's LLR
 * ablation; Eqs. (15), (17), (20), (21); readings 24, 25) ----------
 *
 * mrf_dict_basis: the fingerprint-subspace basis d of P_S(X) = X d^dagger d (Eq. 17, "approximated
 * by the precomputed dictionary"): the leading right singular vectors of the dictionary keeping a
 * fraction `energy` of ||D||_F^2, at most max_rank (<= 32) rows, computed on the device by subspace
 * iteration (float64 accumulation).  *rank_out receives r.  Errors: MRF_EINVAL, MRF_ENOMEM,
 * MRF_ECUDA, MRF_ENUMERIC.  mrf_dict_basis_copy writes the HOST [r][L] complex64 rows. */
mrf_status mrf_dict_basis(mrf_dict dict, double energy, int max_rank, int* rank_out);
mrf_status mrf_dict_basis_copy(mrf_dict dict, void* basis_out);

/* Phi_D of voxels given in basis coordinates: u DEVICE [r][V] complex64 (coefficient-major, the
 * layout of an r-frame image stack) with x_v = sum_i u[i][v] d_i.  For such x (every iterate of
 * mrf_llr_step lies in span(d)) <d_k, x_v> = sum_i u[i][v] conj(Dc[k][i]) with Dc = D d^dagger
 * (built by mrf_dict_basis in float64), so the exact scores need r instead of L frames of work;
 * the filter coefficients are phi x = sum_i u_i (phi d_i) and ||x||^2 = u^H (d d^H) u (float64).
 * The argmax is exact for that x (same certified filter and rescoring as mrf_dict_match; the full
 * atom norms ||d_k|| are kept).  Needs mrf_dict_basis; otherwise as mrf_dict_match. */
mrf_status mrf_dict_match_coef(mrf_dict dict, const void* u, long long V, int* index, float* pd, float* params,
                               void* stream);
mrf_status mrf_dict_match_coef_ex(mrf_dict dict, const void* u, long long V, unsigned flags, int* index, float* pd,
                                  float* params, void* stream);

/* An LLR operator on N x N images of the dictionary's L frames, p x p patches with stride s
 * (11 x 11, 5), patch corners 0, s, 2s, ... and N - p.  Needs mrf_dict_basis; the
 * basis is copied.  Errors: MRF_EINVAL, MRF_ENOMEM, MRF_ECUDA. */
typedef struct mrf_llr_s* mrf_llr;
mrf_status mrf_llr_create(mrf_dict dict, int N, int p, int s, mrf_llr* out);
/* Frame sharding of the LLR operator (multi-GPU): the operator
 * for frames [frame0, frame0 + L_local) of the dictionary's L, with those columns of its basis
 * (the basis itself is the global one, so Phi_D on coefficients stays exact).  Used with a plan
 * over the same frames (mrf_plan_desc.frame_offset = frame0) that carries the ranks' NCCL
 * communicator: the coefficient projection Y = Z d^dagger (Eq. 17) is then a sum over ranks, done
 * as an in-place ncclAllReduce of the [N*N][r] partials (8 N^2 r bytes) on the call's stream, so
 * every rank holds all patches' coefficients and runs the SVT, the manifold term and the cost
 * terms on them redundantly; the data term of mrf_llr_cost is all-reduced the same way.  Every
 * rank must make the same calls in the same order.  mrf_msllr_solve then supports lambda1 = 0,
 * max_iter >= 1 on gridding plans (MRF_EUNSUPPORTED otherwise: Phi_D of X^0 would need the frames
 * of all ranks).  Errors: MRF_EINVAL (no basis, frame range outside [0, L)), MRF_ENOMEM, MRF_ECUDA. */
mrf_status mrf_llr_create_shard(mrf_dict dict, int frame0, int L_local, int N, int p, int s, mrf_llr* out);

/* The same with a caller-supplied basis: HOST [r][L] complex64 with orthonormal rows (copied),
 * 1 <= r <= 32.  Phi_D inside mrf_msllr_solve then always runs on the frames. */
mrf_status mrf_llr_create_basis(const void* basis, int r, int L, int N, int p, int s, int device, mrf_llr* out);

/* The subspace normal operator in basis coordinates on a MRF_NORMAL_TOEPLITZ plan: for
 * x = sum_i u_i d_i (u DEVICE [r][N][N] complex64), z = the coefficients of P_S A^H A x, DEVICE
 * [r][N][N] (z_j = sum_i crop F^-1 [K_ji ⊙ F pad(u_i)], K_ji = sum_rho c^rho_ji T_rho; the exact
 * (NUDFT) normal of the Toeplitz plan).  The mixing kernels are built on first use per plan.
 * Errors: MRF_EINVAL (null, aliasing, not a Toeplitz plan, plan shape), MRF_ENOMEM, MRF_ECUDA. */
mrf_status mrf_llr_subspace_normal(mrf_llr llr, mrf_plan plan, const void* u, void* z, void* stream);

/* The graph Laplacian of the manifold term (Eqs. 7-11; reading 26) from Phi_D's maps:
 * params DEVICE [V][2] float (T1, T2) and pd DEVICE [V] float (mrf_dict_match outputs, V = N*N).
 * The three channels are standardised over the foreground PD > 0.1 max PD; w_ij =
 * exp(-||Q_i(M) - Q_j(M)||_F^2 / sigma2) over all patch pairs (dense), L = D - W.  sigma2 <= 0:
 * the median of the nonzero pairwise squared distances.  Outputs (nullable, HOST): the sigma^2
 * used and max_i D_ii (= max(L), for lambda_1^n = lambda_1^0 max(L)).
 * Synchronises the stream.  Errors: MRF_EINVAL (null, no foreground), MRF_ENOMEM, MRF_ECUDA. */
mrf_status mrf_llr_laplacian(mrf_llr llr, const float* params, const float* pd, double sigma2, double* sigma2_out,
                             double* max_degree, void* stream);

/* One iteration of Algorithm 1 (DEVICE [L][N][N] complex64 arrays, 16-byte aligned):
 *   Z = P_S(x - mu [A^H A x - rhs + lambda1 Q^*(Q(x) L)])   (Eq. 15; rhs = A^H b, A^H A from `plan`)
 *   P_q = SVT_{1/beta}(Q_q(Z))                              (Eq. 20, per patch)
 *   x_out = (Z + gamma Q^*(P)) / (1 + gamma c)              (Eq. 21, gamma = mu lambda2 beta, c = patch count)
 * lambda1 = 0 is the paper's LLR ablation; lambda1 > 0 needs mrf_llr_laplacian (the manifold term
 * is evaluated on P_S x: P_S commutes with the patch operators).  The SVT runs in subspace
 * coordinates (Z lies in span(d): a float64 r x r Gram eigendecomposition per patch).  x_out may alias x
 * when lambda1 = 0 and penalty is NULL.  nuclear (nullable): sum_q ||Q_q(Z)||_*; penalty
 * (nullable, needs the Laplacian): Tr(Q(P_S x) L Q(P_S x)^H) -- the cost terms of Algorithm 1;
 * either synchronises the stream.  Errors: MRF_EINVAL (mu <= 0, lambda1 < 0, lambda2 < 0,
 * beta <= 0, null, misaligned, plan shape), errors of mrf_normal. */
mrf_status mrf_llr_step(mrf_llr llr, mrf_plan plan, const void* x, const void* rhs, float mu, float lambda1,
                        float lambda2, float beta, void* x_out, double* nuclear, double* penalty, void* stream);
/* Cost of Algorithm 1 at x, DEVICE x [L][N][N] and b [L][C][M] (16-byte aligned):
 *   terms[0] = 1/2 ||A x - b||_F^2,  terms[1] = Tr(Q(P_S x) L Q(P_S x)^H) (0 without a Laplacian),
 *   terms[2] = sum_q ||Q_q(P_S x)||_*,  *cost = terms[0] + lambda1 terms[1] + lambda2 terms[2].
 * The regularisers are evaluated on P_S x (equal to x for the iterates of mrf_llr_step).  Both
 * outputs HOST, nullable; float64 reductions in a fixed order; synchronises the stream.  Uses the
 * operator's workspaces (not concurrently with mrf_llr_step on another stream).  Errors:
 * MRF_EINVAL (null, lambda < 0, lambda1 > 0 without a Laplacian, plan shape), errors of mrf_forward. */
mrf_status mrf_llr_cost(mrf_llr llr, mrf_plan plan, const void* x, const void* b, float lambda1, float lambda2,
                        double* cost, double* terms, void* stream);

/* Algorithm 1 of the paper, MS-LLR reconstruction and parameter maps:
 *   X^0 = A^* b;  M^0 = Phi_D(X^0);  L^0 and lambda_1 = lambda1 max(L^0)     (lambda1 > 0 only)
 *   for n = 1 .. max_iter:  X^n = mrf_llr_step(X^{n-1});  cost(n) = mrf_llr_cost(X^n)
 *                           stop if n >= 2 and cost(n-1)/cost(n) - 1 < tol     (reading 27)
 *                           M^{n+1} = Phi_D(X^n);  L^{n+1};  lambda_1 = lambda1 max(L^{n+1})
 *   outputs X^ (in x) and M^ = Phi_D(X^) (index, pd, params).
 * On a plan created with MRF_NORMAL_TOEPLITZ the iterations n >= 2 run in basis coordinates: x = u d
 * with u [V][r], P_S A^H A x from the plan's PSF spectra (r forward / inverse 2D FFT pairs and an
 * r x r mixing per frequency, K_ji = sum_rho c^rho_ji T_rho, c^rho_ji = sum_{l in rho} conj(d_jl) d_il),
 * the data term by 1/2 ||A x - b||^2 = 1/2 <u, P_S A^H A x> - Re <u, P_S A^H b> + 1/2 ||b||^2, and
 * Phi_D on the coefficients; the operator is then the exact (NUDFT) normal of the Toeplitz plan
 * (A^H b stays the gridding adjoint), and x is expanded to the L frames once at the end.
 * lambda1 = 0 is the LLR-only reconstruction (no maps inside the loop).  lambda1 > 0 needs a
 * dictionary LUT of (T1, T2) (P = 2) and params.  b: DEVICE [L][C][M]; x: DEVICE [L][N][N] (out);
 * index int32 [V], pd float [V], params float [V][P] (nullable when lambda1 = 0): DEVICE.
 * info (nullable): iterations run, cost(1..iters) into info->cost (HOST, max_iter entries, nullable)
 * and the last lambda_1.  With tol <= 0 and no info->cost the cost is not evaluated (nothing
 * depends on it).  Allocates two image stacks on first use; synchronises.  Errors: MRF_EINVAL,
 * and the errors of the calls above. */
typedef struct {
  float mu, lambda1, lambda2, beta;   /* Eq. 15 step, lambda_1^0, lambda_2, beta (SVT threshold 1/beta) */
  int max_iter;                       /* N_max */
  double tol;                         /* stop-rule tolerance (1e-5); <= 0: run max_iter */
  double sigma2;                      /* Laplacian bandwidth; <= 0: the median rule at every update */
} mrf_msllr_params;
typedef struct {
  int iters;
  double* cost;                       /* HOST [max_iter] or NULL */
  double lambda1;                     /* lambda_1 of the last step */
} mrf_msllr_info;
mrf_status mrf_msllr_solve(mrf_llr llr, mrf_dict dict, mrf_plan plan, const void* b, const mrf_msllr_params* prm,
                           void* x, int* index, float* pd, float* params, mrf_msllr_info* info, void* stream);
/* Printed-form switches of the LLR / MS-LLR operator (the defaults are DESIGN.md's readings; these
 * reproduce the formulas as printed): MRF_LLR_LITERAL_EQ23 -- the update divides by the scalar
 * 1 + mu lambda2 beta of Eq. (23) instead of 1 + gamma c(v) (reading 25, exact
 * with overlapping patches); MRF_LLR_RAW_MAPS -- the manifold weights of Eq. (8)
 * use the raw (T1, T2, PD) patches instead of standardised ones (reading 26); MRF_LLR_MATCH_NORM2 --
 * Phi_D inside mrf_msllr_solve uses Eq. (5)'s printed ||d||^2 denominator (reading 21).  Applies to
 * every later call on the operator.  Unknown bits: MRF_EINVAL. */
#define MRF_LLR_LITERAL_EQ23 1u
#define MRF_LLR_RAW_MAPS 2u
#define MRF_LLR_MATCH_NORM2 4u
mrf_status mrf_llr_set_options(mrf_llr llr, unsigned options);
mrf_status mrf_llr_destroy(mrf_llr llr);

/* enable != 0 brackets every subsequent tensor-core GEMM launch (k_dict_gemm) of mrf_dict_match
 * with CUDA events on its stream (and resets); the query synchronises them and returns the
 * summed milliseconds and the launch count. */
mrf_status mrf_dict_profile(mrf_dict dict, int enable);
mrf_status mrf_dict_profile_query(mrf_dict dict, double* gemm_ms, long long* launches);

#ifdef __cplusplus
}
#endif
#endif /* MRFNUFFT_H */

// mrfnufft.cu -- the C-ABI (include/mrfnufft.h): plan creation, operator drivers, CG solve.
//
// Plan creation runs once on the host in float64: Kaiser-Bessel
// constants, deapodisation, twiddles, per-point taps and weights, and the bin-sort of every
// interleaf's points into 16-column strips of the oversampled grid.  The operator drivers only
// launch kernels on the caller's stream (no allocation, no host synchronisation), so forward /
// adjoint / normal / dc_cg(tol = 0) are CUDA-graph capturable.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mrfnufft.h"
#include "cg.cuh"
#include "gridding.cuh"
#include "precond.cuh"
#include "nccl_dl.h"
#include "status.h"

using namespace mrf;

// ================================================================================== errors
// (status.h: fail(), CUDA_TRY, MRF_TRY; the message lives in one thread-local string here)
static thread_local std::string g_err;

mrf_status mrf::fail(mrf_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

mrf_status mrf::check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MRF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return MRF_OK;
}

// ================================================================================== plan
namespace {

struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> ev[MRF_K_COUNT];   // start/stop pairs
  size_t used[MRF_K_COUNT] = {0};
  long long launches[MRF_K_COUNT] = {0};
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

static constexpr int kMaxLanes = 8;

struct CgKey {   // the arguments a captured CG graph bakes in
  const void *x = nullptr, *y = nullptr, *z = nullptr;
  float mu = 0.f;
  int n_iter = -1;
  bool zero_init = false, pc = false;
  bool operator==(const CgKey& o) const {
    return x == o.x && y == o.y && z == o.z && mu == o.mu && n_iter == o.n_iter && zero_init == o.zero_init &&
           pc == o.pc;
  }
};
static constexpr int kDefaultLanes = 2;
static int cols_threads_rt(int G);

struct mrf_plan_s {
  // sizes
  int N = 0, G = 0, L = 0, M = 0, R = 0, C = 1, W = 0, S = 0, frame_offset = 0, recw = 0;
  unsigned flags = 0;
  int device = 0;
  unsigned long long serial = 0;   // creation number (process-wide), identifies the plan
  int bf = 1;               // frames per batch
  int nsm = 148;            // SMs of the device
  bool adj_sep = false;      // k_adj_cols variant with the separate exchange buffer (one CTA per SM)
  bool adj_t2 = false;       // k_adj_cols with two threads per stage-2 transform (G = 512: 16 warps per CTA)
  int adj_threads() const { return cols_threads_rt(G) * (adj_t2 ? 2 : 1); }
  int ystage = 0;           // bytes of y[fc] k_adj_cols stages in shared memory (M*8 if M even, M*8 <= kYBytes)
  int occ_fr0 = 1, occ_fr1 = 1, occ_fc = 1, occ_ac = 1, occ_ar = 1;   // resident CTAs per SM
  int fc_stage = 0, ac_stage = 0;   // chunk staging bytes of the column kernels
  int occ_tc = 1;
  int col_smem = 0;                 // dynamic shared memory of k_fwd_cols
  int acol_smem = 0;                // dynamic shared memory of k_adj_cols
  void* nccl_comm = nullptr;
  mrf_host_allreduce_fn host_ar = nullptr;   // mrf_plan_set_host_allreduce (replaces nccl_comm)
  void* host_ar_ctx = nullptr;
  void* host_ar_buf = nullptr;               // pinned staging of the host all-reduce
  size_t host_ar_cap = 0;
  int dbg = 0;               // MRF_DBG experiment bits (1: skip gather/spread, 2: phase timers)
  long long* dbgbuf = nullptr;
  // device tables
  float2* coils = nullptr;
  float* dap = nullptr;
  float2* tw = nullptr;
  int* fchunks = nullptr;    // per (interleaf, strip) point records (gather), gridding.cuh
  int2* ftab = nullptr;
  int* achunks = nullptr;    // per (interleaf, strip) spread matrix in SELL-32 form
  int2* atab = nullptr;
  int* fil = nullptr;
  int* perm = nullptr;       // [L] interleaf-ordered processing order within each batch (DevPlan::perm)
  int* ctrs = nullptr;       // [kMaxLanes][8] dynamic item hand-out counters of the column kernels (self-resetting)
  bool adj_dyn = false;      // k_adj_cols hands items out dynamically (set at plan creation from the chunk sizes)
  // workspaces
  // Frame batches alternate between kLanes internal streams so one batch's kernel tail overlaps
  // the next batch's kernels; each lane owns its half-grid and k-space workspaces.
  int nlanes = 1;
  cudaStream_t lane[kMaxLanes] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxLanes] = {};
  float2* Hs[kMaxLanes] = {};      // [bf*C][N][G] half grid per lane
  float2* Has[kMaxLanes] = {};     // Toeplitz plans: the adjoint-side half grid per lane
  float* psf = nullptr;            // Toeplitz plans: [R][S][G][16] real PSF spectra
  float* dcf = nullptr;            // MRF_DCF plans: [R][M] Pipe-Menon density compensation weights
  std::vector<float> dcf_host;     // the same, host copy (mrf_dcf_weights)
  float2* ydcf = nullptr;          // [L][C][M] weighted k-space (allocated on first mrf_adjoint_dcf)
  float* ones = nullptr;           // [N] of 1.0 (the Toeplitz path has no deapodisation)
  float2* ybufs[kMaxLanes] = {};   // [bf*C][M] per lane
  float2* r = nullptr;       // CG vectors [L][N][N]
  float2* p = nullptr;
  float2* q = nullptr;
  double2* part = nullptr;   // [kPartBlocks] vector-kernel partials
  double2* dotp = nullptr;   // [L * rowblocks] fused <p, q> partials of k_adj_rows
  // split-phase CG (C == 1): y = A p of all local frames and the ||p||^2 partials of the row pass
  float2* ycg = nullptr;     // [L][M]
  double2* pnp = nullptr;    // [L * rowblocks * 4]
  float2* hacg = nullptr;    // Toeplitz plans: [L][N][G] adjoint-side half grids of all frames
  double2* tqp = nullptr;    // Toeplitz plans: [L * S * warps] Parseval partials of <p, A^H A p>
  size_t ndotp = 0;
  CGScalars* sc = nullptr;
  float2* cg_rin = nullptr;  // the vector the fused CG row pass adds to beta p: r (CG) or z (PCG)
  // PCG (MRF_CG_PRECOND; precond.cuh, reading 28): Chan circulant eigenvalues per
  // interleaf, z = M^-1 r, the row-pass workspace and the <r, z> partials
  std::vector<float> traj_h;       // host copy of the trajectory [R][M][2]
  float* pc_lam = nullptr;         // [R][N][N] float32, [my + N/2][mx + N/2]
  double pc_lam_sum = 0.0;         // mean of lambda over R interleaves (float64)
  double pc_gamma = -1.0;          // gamma of the current solve
  double pc_shift = 30.0;          // gamma = mu + shift * scale * mean(lambda)
  float pc_scale = 1.f;            // mean coil power
  float2* z = nullptr;
  float2* pc_tmp = nullptr;
  double2* pc_part = nullptr;      // [kPcBlocks]
  int pc_occ_rows = 0, pc_occ_cols = 0;
  double* hist = nullptr;    // device [hist_cap]
  int hist_cap = 0;
  // host staging (allocated on first host-pointer call)
  float2* stg_x = nullptr;
  float2* stg_y = nullptr;
  float2* stg_z = nullptr;
  // MRF_CG_ASYNC_HOST: two device slots (x, y) per call parity, a copy stream for the
  // device-to-host result copies, and events ordering slot reuse
  float2* ax[2] = {nullptr, nullptr};
  float2* ay[2] = {nullptr, nullptr};
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_solved[2] = {}, ev_copied[2] = {};
  unsigned long long acalls = 0;
  // CUDA graph of the last tol == 0 solve (run_cg) and the arguments it was captured with
  cudaStream_t gstream = nullptr;
  static constexpr int kGraphs = 4;   // e.g. the two device slots of MRF_CG_ASYNC_HOST
  cudaGraphExec_t cg_exec[kGraphs] = {};
  CgKey cg_key[kGraphs];
  unsigned long long cg_use[kGraphs] = {}, cg_clock = 0;
  size_t bytes = 0;
  Prof prof;
  DevPlan dp() const {
    DevPlan d;
    d.N = N; d.G = G; d.M = M; d.R = R; d.C = C; d.W = W; d.S = S; d.recw = recw;
    d.coils = coils; d.dap = dap; d.tw = tw; d.fchunks = fchunks; d.ftab = ftab; d.achunks = achunks; d.atab = atab;
    d.fil = fil;
    d.perm = perm;
    d.dbg = dbg;
    d.dbgbuf = dbgbuf;
    return d;
  }
};

static constexpr int kPartBlocks = 4 * 148;

// ---------------------------------------------------------------------------- host math (fp64)
// I0 by its power series sum_k (x^2/4)^k / (k!)^2 (converges for all x; x <= ~40 here).
static double bessel_i0(double x) {
  const double q = 0.25 * x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 500; ++k) {
    term *= q / ((double)k * (double)k);
    sum += term;
    if (term < 1e-17 * sum) break;
  }
  return sum;
}

struct KB {
  int W;
  double beta, i0b;
  KB(int W_, double sigma) : W(W_) {
    beta = M_PI * std::sqrt((W / sigma) * (W / sigma) * (sigma - 0.5) * (sigma - 0.5) - 0.8);
    i0b = bessel_i0(beta);
  }
  double phi(double u) const {   // open support |u| < W/2, phi(0) = 1
    if (!(std::fabs(u) < 0.5 * W)) return 0.0;
    const double t = 1.0 - (2.0 * u / W) * (2.0 * u / W);
    return bessel_i0(beta * std::sqrt(t)) / i0b;
  }
  double psi_analytic(double n, int G) const {
    const double a = M_PI * W * n / G;
    const double rad = beta * beta - a * a;
    double f;
    if (rad > 0) {
      const double z = std::sqrt(rad);
      f = std::sinh(z) / z;
    } else if (rad < 0) {
      const double z = std::sqrt(-rad);
      f = std::sin(z) / z;
    } else {
      f = 1.0;
    }
    return W * f / i0b;
  }
  double psi_discrete(double n, int G) const {
    double s = 0.0;
    const int dmax = (W + 1) / 2;
    for (int d = -dmax; d <= dmax; ++d) s += phi((double)d) * std::cos(2.0 * M_PI * d * n / G);
    return s;
  }
};

// float64 weights of one point: out[0..W) = phi(u_x - m_x), out[W..2W) = phi(u_y - m_y)
static void kb_taps(const KB& kb, int G, int W, float kx, float ky, double* out) {
  const float k2[2] = {kx, ky};
  for (int ax = 0; ax < 2; ++ax) {
    const double u = (double)G * (double)k2[ax];
    const long long m0 = (long long)std::floor(u - 0.5 * W) + 1;
    for (int t = 0; t < W; ++t) out[ax * W + t] = kb.phi(u - (double)(m0 + t));
  }
}

template <int G>
static void fft_shape_t(int* P, int* Q, int* T) {
  *P = FFTShape<G>::P;
  *Q = FFTShape<G>::Q;
  *T = FFTShape<G>::T;
}
static void fft_shape(int G, int* P, int* Q, int* T) {
  switch (G) {
    case 64: fft_shape_t<64>(P, Q, T); break;
    case 128: fft_shape_t<128>(P, Q, T); break;
    case 256: fft_shape_t<256>(P, Q, T); break;
    case 512: fft_shape_t<512>(P, Q, T); break;
    default: fft_shape_t<1024>(P, Q, T); break;
  }
}

static int cols_threads_rt(int G) {   // threads of a column-kernel CTA (SW x T)
  int P = 0, Q = 0, T = 0;
  fft_shape(G, &P, &Q, &T);
  return SW * T;
}
template <typename T>
static mrf_status dev_alloc(mrf_plan_s* pl, T** ptr, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)ptr, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(MRF_ENOMEM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
  }
  pl->bytes += count * sizeof(T);
  return MRF_OK;
}

static void free_plan(mrf_plan_s* pl) {
  if (!pl) return;
  if (pl->dbgbuf) {   // phase timer dump (experiment bit 2): cycles summed over CTAs
    long long h[32];
    if (cudaMemcpy(h, pl->dbgbuf, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess) {
      const char* nm[2] = {"fwd_cols", "adj_cols"};
      for (int k = 0; k < 2; ++k) {
        std::fprintf(stderr, "[phase] %s items=%lld cycles/item:", nm[k], h[16 * k]);
        for (int i = 1; i <= 10; ++i) std::fprintf(stderr, " %.0f", h[16 * k] ? (double)h[16 * k + i] / h[16 * k] : 0.0);
        std::fprintf(stderr, "\n");
      }
    }
    cudaFree(pl->dbgbuf);
  }
  if (pl->psf) cudaFree(pl->psf);
  if (pl->dcf) cudaFree(pl->dcf);
  if (pl->ydcf) cudaFree(pl->ydcf);
  if (pl->ones) cudaFree(pl->ones);
  for (int i = 0; i < kMaxLanes; ++i) {
    if (pl->Has[i]) cudaFree(pl->Has[i]);
    if (pl->Hs[i]) cudaFree(pl->Hs[i]);
    if (pl->ybufs[i]) cudaFree(pl->ybufs[i]);
  }
  void* ptrs[] = {pl->ctrs, pl->ycg, pl->pnp, pl->hacg, pl->tqp, pl->perm, pl->pc_lam, pl->z, pl->pc_tmp, pl->pc_part,
                  pl->coils, pl->dap, pl->tw, pl->fchunks, pl->ftab, pl->achunks, pl->atab, pl->fil, pl->r, pl->p, pl->q,
                  pl->part, pl->dotp, pl->sc, pl->hist, pl->stg_x, pl->stg_y, pl->stg_z, pl->ax[0], pl->ax[1],
                  pl->ay[0], pl->ay[1]};
  for (int i = 0; i < 2; ++i) {
    if (pl->ev_solved[i]) cudaEventDestroy(pl->ev_solved[i]);
    if (pl->ev_copied[i]) cudaEventDestroy(pl->ev_copied[i]);
  }
  if (pl->cstream) cudaStreamDestroy(pl->cstream);
  for (cudaGraphExec_t e : pl->cg_exec)
    if (e) cudaGraphExecDestroy(e);
  if (pl->gstream) cudaStreamDestroy(pl->gstream);
  if (pl->host_ar_buf) cudaFreeHost(pl->host_ar_buf);
  for (void* v : ptrs)
    if (v) cudaFree(v);
  for (int k = 0; k < MRF_K_COUNT; ++k)
    for (cudaEvent_t e : pl->prof.ev[k]) cudaEventDestroy(e);
  for (int i = 0; i < kMaxLanes; ++i) {
    if (pl->lane[i]) cudaStreamDestroy(pl->lane[i]);
    if (pl->ev_join[i]) cudaEventDestroy(pl->ev_join[i]);
  }
  if (pl->ev_fork) cudaEventDestroy(pl->ev_fork);
  delete pl;
}

// ================================================================================== launches
static constexpr size_t kProfCap = 1 << 15;

struct ProfScope {
  mrf_plan_s* pl;
  int cls;
  cudaStream_t st;
  bool rec = false;
  size_t slot = 0;
  ProfScope(mrf_plan_s* p, int c, cudaStream_t s) : pl(p), cls(c), st(s) {
    if (!pl->prof.on) return;
    pl->prof.launches[cls]++;
    Prof& pr = pl->prof;
    if (pr.used[cls] + 2 > kProfCap) return;
    while (pr.ev[cls].size() < pr.used[cls] + 2) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      pr.ev[cls].push_back(e);
    }
    slot = pr.used[cls];
    pr.used[cls] += 2;
    cudaEventRecord(pr.ev[cls][slot], st);
    rec = true;
  }
  ~ProfScope() {
    if (rec) cudaEventRecord(pl->prof.ev[cls][slot + 1], st);
  }
};


// Opt-in shared memory sizes and occupancy of the persistent kernels (once per plan).
// Density compensation (reading 23): Pipe-Menon fixed-point
// iteration w <- w / (Phi Phi^T w) on the sigma*N grid with the gridding taps, float64, per
// interleaf at plan time (a dense G x G accumulator: spread, then interpolate back).
static constexpr int kDcfIters = 20;
static void pipe_menon(const KB& kb, int G, int W, const float* traj, int M, double* w) {
  std::vector<double> tp((size_t)M * 2 * W), grid((size_t)G * G);
  std::vector<int> m0((size_t)M * 2);
  for (int j = 0; j < M; ++j) {
    kb_taps(kb, G, W, traj[2 * j], traj[2 * j + 1], &tp[(size_t)j * 2 * W]);
    for (int ax = 0; ax < 2; ++ax) {
      const long long m = (long long)std::floor((double)G * (double)traj[2 * j + ax] - 0.5 * W) + 1;
      m0[2 * j + ax] = (int)(((m % G) + G) % G);
    }
  }
  for (int j = 0; j < M; ++j) w[j] = 1.0;
  for (int it = 0; it < kDcfIters; ++it) {
    std::fill(grid.begin(), grid.end(), 0.0);
    for (int j = 0; j < M; ++j) {
      const double* t = &tp[(size_t)j * 2 * W];
      for (int ty = 0; ty < W; ++ty) {
        double* row = &grid[(size_t)((m0[2 * j + 1] + ty) % G) * G];
        for (int tx = 0; tx < W; ++tx) row[(m0[2 * j] + tx) % G] += t[W + ty] * t[tx] * w[j];
      }
    }
    for (int j = 0; j < M; ++j) {
      const double* t = &tp[(size_t)j * 2 * W];
      double acc = 0.0;
      for (int ty = 0; ty < W; ++ty) {
        const double* row = &grid[(size_t)((m0[2 * j + 1] + ty) % G) * G];
        for (int tx = 0; tx < W; ++tx) acc += t[W + ty] * t[tx] * row[(m0[2 * j] + tx) % G];
      }
      w[j] = acc > 0.0 ? w[j] / acc : 0.0;
    }
  }
}

// y_w[l][c][j] = dcf[interleaf(l)][j] * y[l][c][j]
__global__ void k_dcf_scale(float2* __restrict__ yw, const float2* __restrict__ y, const float* __restrict__ dcf,
                            const int* __restrict__ fil, int L, int C, int M) {
  const size_t n = (size_t)L * C * M;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / ((size_t)C * M)), j = (int)(i % M);
    const float w = __ldg(dcf + (size_t)__ldg(fil + l) * M + j);
    const float2 v = y[i];
    yw[i] = make_float2(w * v.x, w * v.y);
  }
}

// k_adj_cols variant of the plan: SEP (separate exchange buffer, G <= 512, one CTA per SM) and DYN
// (dynamic item hand-out; plans whose spread chunks mostly overflow the staging buffer)
template <int G>
static void (*adj_cols_kernel(const mrf_plan_s* pl))(DevPlan, const float2*, float2*, int, int, int, int, int*) {
  if constexpr (G == 512) {
    if (pl->adj_sep && pl->adj_t2) return pl->adj_dyn ? k_adj_cols<G, true, true, true> : k_adj_cols<G, true, false, true>;
  }
  if (pl->adj_sep) return pl->adj_dyn ? k_adj_cols<G, (G <= 512), true> : k_adj_cols<G, (G <= 512), false>;
  return pl->adj_dyn ? k_adj_cols<G, false, true> : k_adj_cols<G, false, false>;
}

template <int G>
static mrf_status adj_cols_attr(mrf_plan_s* pl) {   // (after a change of the variant)
  CUDA_TRY(cudaFuncSetAttribute(adj_cols_kernel<G>(pl), cudaFuncAttributeMaxDynamicSharedMemorySize, pl->acol_smem));
  return MRF_OK;
}
template <int G>
static mrf_status setup_kernels(mrf_plan_s* pl) {
  const int ncol = cols_threads<G>();
  const size_t s_fr0 = fwd_rows_smem<G>(1), s_fr1 = fwd_rows_smem<G>(3), s_ar = adj_rows_smem<G>();
  int optin = 0, per_sm = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, pl->device));
  CUDA_TRY(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, pl->device));
  int actas = 1;   // measured: the adjoint column kernel prefers one CTA per SM with a large chunk stage
  if (const char* e = std::getenv("MRF_ADJ_CTAS")) actas = std::max(1, std::min(2, std::atoi(e)));
  int fctas = cols_ctas_per_sm<G>();
  if (const char* e = std::getenv("MRF_FWD_CTAS")) fctas = std::max(1, std::min(2, std::atoi(e)));
  const size_t s_col = std::min<size_t>((size_t)optin - 256, (size_t)per_sm / fctas - 1024 - 256) & ~size_t(15);
  const size_t s_acol = std::min<size_t>((size_t)optin - 256, (size_t)per_sm / actas - 1024 - 256) & ~size_t(15);
  pl->col_smem = (int)s_col;
  pl->acol_smem = (int)s_acol;
  pl->fc_stage = (int)((s_col - fwd_cols_fixed<G>()) & ~size_t(15));
  pl->adj_sep = G <= 512 && actas == 1;
  pl->adj_t2 = false;
  if (const char* e = std::getenv("MRF_ADJ_T2")) pl->adj_t2 = G == 512 && pl->adj_sep && e[0] == '1';
  pl->ac_stage = (int)((s_acol - adj_cols_fixed<G>((size_t)pl->ystage, pl->adj_sep)) & ~size_t(15));
  CUDA_TRY(cudaFuncSetAttribute(k_fwd_rows<G, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_fr0));
  CUDA_TRY(cudaFuncSetAttribute(k_fwd_rows<G, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_fr1));
  CUDA_TRY(cudaFuncSetAttribute(k_adj_rows<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_ar));
  CUDA_TRY(cudaFuncSetAttribute(k_adj_rows<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_ar));
  CUDA_TRY(cudaFuncSetAttribute(k_fwd_cols<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_col));
  auto adj_kernel = adj_cols_kernel<G>(pl);
  CUDA_TRY(cudaFuncSetAttribute(adj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_acol));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl->occ_fr0, k_fwd_rows<G, 0>, kRowThreads, s_fr0));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl->occ_fr1, k_fwd_rows<G, 1>, kRowThreads, s_fr1));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl->occ_ar, k_adj_rows<G, false>, kRowThreads, s_ar));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl->occ_fc, k_fwd_cols<G>, ncol, s_col));
  CUDA_TRY(cudaFuncSetAttribute(k_toep_cols<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)toep_cols_smem<G>()));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl->occ_tc, k_toep_cols<G>, ncol, toep_cols_smem<G>()));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl->occ_ac, adj_kernel, pl->adj_threads(), s_acol));
  CUDA_TRY(cudaFuncSetAttribute(k_sn_fcols<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sn_cols_smem<G>()));
  CUDA_TRY(cudaFuncSetAttribute(k_sn_icols<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sn_cols_smem<G>()));
  if (pl->occ_fr0 < 1 || pl->occ_fr1 < 1 || pl->occ_ar < 1 || pl->occ_fc < 1 || pl->occ_ac < 1)
    return fail(MRF_EUNSUPPORTED, "a kernel does not fit on an SM");
  if (const char* cap = std::getenv("MRF_OCC_CAP")) {   // experiment knob: resident CTAs per SM
    const int c = std::atoi(cap);
    if (c > 0) {
      pl->occ_fr0 = std::min(pl->occ_fr0, c); pl->occ_fr1 = std::min(pl->occ_fr1, c);
      pl->occ_ar = std::min(pl->occ_ar, c); pl->occ_fc = std::min(pl->occ_fc, c); pl->occ_ac = std::min(pl->occ_ac, c);
    }
  }
  return MRF_OK;
}

// Launch with programmatic stream serialisation (PDL): the kernel's prologue overlaps the
// predecessor's tail; the kernel itself calls griddepcontrol.wait before touching produced data.
static bool g_pdl = [] {
  const char* e = std::getenv("MRF_PDL");
  return !(e && e[0] == '0');
}();

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Experiment knobs MRF_GCAP_FR / _FC / _AC / _AR: upper bound on the CTAs of one launch of the forward-row,
// forward-column, adjoint-column and adjoint-row kernels (0 = resident CTAs x SMs, the default), so that
// kernels of several lanes can share the SMs side by side.
static int g_gcap[4] = {0, 0, 0, 0};
static bool g_gcap_init = [] {
  const char* names[4] = {"MRF_GCAP_FR", "MRF_GCAP_FC", "MRF_GCAP_AC", "MRF_GCAP_AR"};
  for (int i = 0; i < 4; ++i)
    if (const char* e = std::getenv(names[i])) g_gcap[i] = std::max(0, std::atoi(e));
  return true;
}();
static int pgrid(mrf_plan_s* pl, int occ, long long items, int cls = -1) {
  long long g = std::min<long long>(items, (long long)occ * pl->nsm);
  if (cls >= 0 && g_gcap[cls] > 0) g = std::min<long long>(g, g_gcap[cls]);
  // Column kernels walk items (fc, strip) round-robin, item % S = strip: a grid that shares a factor
  // with S confines each CTA to the strips of one residue class, and the strips next to DC carry
  // several times the mean gather / spread work (a grid of 128 CTAs, a multiple of the 32 strips,
  // measured 2.28 ms for the MRF normal operator against 1.59 ms).  Take the next smaller grid
  // coprime with S (148 SMs: 147 and 295 CTAs; adjoint 0.919 -> 0.906 ms).
  if ((cls == 1 || cls == 2) && items > g && pl->S > 1) {
    auto gcd = [](long long a, long long b) { while (b) { const long long t = a % b; a = b; b = t; } return a; };
    while (g > 1 && gcd(g, pl->S) != 1) --g;
  }
  return (int)std::max<long long>(1, g);
}

template <int G>
static mrf_status launch_fwd_rows(mrf_plan_s* pl, const float2* x, float2* H, int l0, int nb, cudaStream_t st,
                                  float2* yzero = nullptr, long long nyzero = 0) {
  const long long items = (long long)nb * (pl->N / RowCfg<G>::RPC) * pl->C;
  ProfScope ps(pl, MRF_K_FWD_ROWS, st);
  CUDA_TRY(launch_pdl(k_fwd_rows<G, 0>, pgrid(pl, pl->occ_fr0, items, 0), kRowThreads, fwd_rows_smem<G>(1), st, pl->dp(),
                      x, H, l0, nb, nullptr, nullptr, nullptr, nullptr, yzero, nyzero, (double2*)nullptr));
  return MRF_OK;
}
template <int G>
static mrf_status launch_fwd_rows_cg(mrf_plan_s* pl, float2* x, float2* H, int l0, int nb, cudaStream_t st,
                                     float2* yzero, long long nyzero, double2* pn = nullptr) {
  const long long items = (long long)nb * (pl->N / RowCfg<G>::RPC) * pl->C;
  ProfScope ps(pl, MRF_K_FWD_ROWS, st);
  CUDA_TRY(launch_pdl(k_fwd_rows<G, 1>, pgrid(pl, pl->occ_fr1, items, 0), kRowThreads, fwd_rows_smem<G>(3), st, pl->dp(),
                      nullptr, H, l0, nb, pl->cg_rin ? pl->cg_rin : pl->r, pl->p, x, &pl->sc->alpha, yzero, nyzero, pn));
  return MRF_OK;
}
template <int G>
static mrf_status launch_fwd_cols(mrf_plan_s* pl, const float2* H, float2* y, int l0, int nb, cudaStream_t st) {
  const long long items = (long long)nb * pl->C * pl->S;
  ProfScope ps(pl, MRF_K_FWD_COLS, st);
  CUDA_TRY(launch_pdl(k_fwd_cols<G>, pgrid(pl, pl->occ_fc, items, 1), cols_threads<G>(), pl->col_smem, st, pl->dp(), H, y,
                      l0, nb, pl->fc_stage));
  return MRF_OK;
}
template <int G>
static mrf_status launch_adj_cols(mrf_plan_s* pl, const float2* y, float2* H, int l0, int nb, cudaStream_t st,
                                  int slot = 0) {
  const long long items = (long long)nb * pl->C * pl->S;
  const int ys = ((uintptr_t)y % 16 == 0) ? pl->ystage : 0;
  const int stage = ys ? pl->ac_stage : (int)(((size_t)pl->acol_smem - adj_cols_fixed<G>(0, pl->adj_sep)) & ~size_t(15));
  ProfScope ps(pl, MRF_K_ADJ_COLS, st);
  auto adj_kernel = adj_cols_kernel<G>(pl);
  CUDA_TRY(launch_pdl(adj_kernel, pgrid(pl, pl->occ_ac, items, 2), pl->adj_threads(), pl->acol_smem, st, pl->dp(), y, H,
                      l0, nb, ys, stage, pl->adj_dyn ? pl->ctrs + 8 * slot : (int*)nullptr));
  return MRF_OK;
}
template <int G>
static mrf_status launch_adj_rows(mrf_plan_s* pl, const float2* H, float2* out, const float2* xin, float mu, int l0,
                                  int nb, double2* dot, cudaStream_t st, float2* rres = nullptr) {
  const long long items = (long long)nb * (pl->N / RowCfg<G>::RPC);
  ProfScope ps(pl, MRF_K_ADJ_ROWS, st);
  if (rres)
    CUDA_TRY(launch_pdl(k_adj_rows<G, true>, pgrid(pl, pl->occ_ar, items, 3), kRowThreads, adj_rows_smem<G>(), st, pl->dp(),
                        H, out, xin, mu, l0, nb, dot, rres, (const double*)&pl->sc->alpha));
  else
    CUDA_TRY(launch_pdl(k_adj_rows<G, false>, pgrid(pl, pl->occ_ar, items, 3), kRowThreads, adj_rows_smem<G>(), st, pl->dp(),
                        H, out, xin, mu, l0, nb, dot, (float2*)nullptr, (const double*)nullptr));
  return MRF_OK;
}

template <int G>
static mrf_status launch_toep_cols(mrf_plan_s* pl, const float2* Hf, float2* Ha, int l0, int nb, cudaStream_t st,
                                   double2* tq = nullptr) {
  const long long items = (long long)nb * pl->C * pl->S;
  ProfScope ps(pl, MRF_K_FWD_COLS, st);
  CUDA_TRY(launch_pdl(k_toep_cols<G>, pgrid(pl, pl->occ_tc, items, 1), cols_threads<G>(), toep_cols_smem<G>(), st, pl->dp(),
                      Hf, Ha, pl->psf, l0, nb, tq));
  return MRF_OK;
}

static mrf_status memset_async(mrf_plan_s* pl, void* ptr, size_t bytes, cudaStream_t st) {
  ProfScope ps(pl, MRF_K_OTHER, st);
  CUDA_TRY(cudaMemsetAsync(ptr, 0, bytes, st));
  return MRF_OK;
}

// ---------------------------------------------------------------------------- operator drivers
// Fork the frame batches of one operator call onto the plan's lanes and join them back into the
// caller's stream (graph capturable: fork/join through events).
struct Lanes {
  mrf_plan_s* pl;
  cudaStream_t st;
  int n;
  Lanes(mrf_plan_s* p, cudaStream_t s, int nbatch) : pl(p), st(s), n(nbatch > 1 ? p->nlanes : 1) {}
  mrf_status begin() {
    if (n == 1) return MRF_OK;
    CUDA_TRY(cudaEventRecord(pl->ev_fork, st));
    for (int i = 0; i < n; ++i) CUDA_TRY(cudaStreamWaitEvent(pl->lane[i], pl->ev_fork, 0));
    return MRF_OK;
  }
  cudaStream_t stream(int b) const { return n == 1 ? st : pl->lane[b % n]; }
  int slot(int b) const { return n == 1 ? 0 : b % n; }
  mrf_status end() {
    if (n == 1) return MRF_OK;
    for (int i = 0; i < n; ++i) {
      CUDA_TRY(cudaEventRecord(pl->ev_join[i], pl->lane[i]));
      CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_join[i], 0));
    }
    return MRF_OK;
  }
};

static int n_batches(const mrf_plan_s* pl) { return (pl->L + pl->bf - 1) / pl->bf; }

template <int G>
static mrf_status run_forward(mrf_plan_s* pl, const float2* x, float2* y, cudaStream_t st) {
  MRF_TRY(memset_async(pl, y, (size_t)pl->L * pl->C * pl->M * sizeof(float2), st));
  Lanes ln(pl, st, n_batches(pl));
  MRF_TRY(ln.begin());
  for (int b = 0, l0 = 0; l0 < pl->L; ++b, l0 += pl->bf) {
    const int nb = std::min(pl->bf, pl->L - l0);
    cudaStream_t s = ln.stream(b);
    float2* H = pl->Hs[ln.slot(b)];
    MRF_TRY(launch_fwd_rows<G>(pl, x, H, l0, nb, s));
    MRF_TRY(launch_fwd_cols<G>(pl, H, y + (size_t)l0 * pl->C * pl->M, l0, nb, s));
  }
  return ln.end();
}

template <int G>
static mrf_status run_adjoint(mrf_plan_s* pl, const float2* y, float2* x, cudaStream_t st) {
  Lanes ln(pl, st, n_batches(pl));
  MRF_TRY(ln.begin());
  for (int b = 0, l0 = 0; l0 < pl->L; ++b, l0 += pl->bf) {
    const int nb = std::min(pl->bf, pl->L - l0);
    cudaStream_t s = ln.stream(b);
    float2* H = pl->Hs[ln.slot(b)];
    MRF_TRY(launch_adj_cols<G>(pl, y + (size_t)l0 * pl->C * pl->M, H, l0, nb, s, ln.slot(b)));
    MRF_TRY(launch_adj_rows<G>(pl, H, x, nullptr, 0.f, l0, nb, nullptr, s));
  }
  return ln.end();
}

// out = A^H A x + mu x.  cg != 0: the CG iteration form -- x is the CG search direction p, the
// row pass first forms p = r + beta p and advances the solution xsol += alpha p_old (C == 1), and
// the last pass writes the float64 partials of <p, out> to pl->dotp.
template <int G>
static mrf_status run_normal(mrf_plan_s* pl, const float2* x, float2* out, float mu, int cg, float2* xsol,
                             cudaStream_t st) {
  Lanes ln(pl, st, n_batches(pl));
  MRF_TRY(ln.begin());
  for (int b = 0, l0 = 0; l0 < pl->L; ++b, l0 += pl->bf) {
    const int nb = std::min(pl->bf, pl->L - l0);
    cudaStream_t s = ln.stream(b);
    float2* H = pl->Hs[ln.slot(b)];
    float2* yb = pl->ybufs[ln.slot(b)];
    const long long ny = (long long)nb * pl->C * pl->M;   // zeroed by the row pass for the gather
    if (cg && pl->C == 1) MRF_TRY(launch_fwd_rows_cg<G>(pl, xsol, H, l0, nb, s, yb, ny));
    else MRF_TRY(launch_fwd_rows<G>(pl, x, H, l0, nb, s, yb, ny));
    MRF_TRY(launch_fwd_cols<G>(pl, H, yb, l0, nb, s));
    MRF_TRY(launch_adj_cols<G>(pl, yb, H, l0, nb, s, ln.slot(b)));
    MRF_TRY(launch_adj_rows<G>(pl, H, out, (mu != 0.f || cg) ? x : nullptr, mu, l0, nb, cg ? pl->dotp : nullptr, s));
  }
  return ln.end();
}

// Split-phase CG iteration (C == 1, gridding plans): the forward half of the
// normal operator for every batch -- the fused row pass (p = r + beta p, x += alpha p, ||p||^2
// partials) and the column pass into y = A p of all frames -- then, once alpha = rho /
// (||A p||^2 + mu ||p||^2) is known, the adjoint half whose row pass advances r -= alpha
// (A^H A p + mu p) in place and emits the <r, r> partials.  q is never stored and the separate
// r-update pass disappears: 8 image passes per iteration instead of 10.
template <int G>
static mrf_status run_cg_split_fwd(mrf_plan_s* pl, float2* xsol, cudaStream_t st) {
  Lanes ln(pl, st, n_batches(pl));
  MRF_TRY(ln.begin());
  for (int b = 0, l0 = 0; l0 < pl->L; ++b, l0 += pl->bf) {
    const int nb = std::min(pl->bf, pl->L - l0);
    cudaStream_t s = ln.stream(b);
    float2* H = pl->Hs[ln.slot(b)];
    float2* yb = pl->ycg + (size_t)l0 * pl->C * pl->M;
    const long long ny = (long long)nb * pl->C * pl->M;   // zeroed by the row pass for the gather
    if (pl->C == 1) MRF_TRY(launch_fwd_rows_cg<G>(pl, xsol, H, l0, nb, s, yb, ny, pl->pnp));
    else MRF_TRY(launch_fwd_rows<G>(pl, pl->p, H, l0, nb, s, yb, ny));   // p, x formed by k_cg_px
    MRF_TRY(launch_fwd_cols<G>(pl, H, yb, l0, nb, s));
  }
  return ln.end();
}
template <int G>
static mrf_status run_cg_split_adj(mrf_plan_s* pl, float mu, cudaStream_t st) {
  Lanes ln(pl, st, n_batches(pl));
  MRF_TRY(ln.begin());
  for (int b = 0, l0 = 0; l0 < pl->L; ++b, l0 += pl->bf) {
    const int nb = std::min(pl->bf, pl->L - l0);
    cudaStream_t s = ln.stream(b);
    float2* H = pl->Hs[ln.slot(b)];
    MRF_TRY(launch_adj_cols<G>(pl, pl->ycg + (size_t)l0 * pl->C * pl->M, H, l0, nb, s, ln.slot(b)));
    MRF_TRY(launch_adj_rows<G>(pl, H, nullptr, pl->p, mu, l0, nb, pl->dotp, s, pl->r));
  }
  return ln.end();
}

// The same split on Toeplitz plans (C == 1): the forward half (row pass + k_toep_cols) keeps the
// adjoint-side half grids of every frame and emits the Parseval partials of <p, A^H A p> =
// sum_k T(k) |FFT(pad p)(k)|^2; the adjoint half is the residual-update row pass.
template <int G>
static mrf_status run_cg_split_fwd_toep(mrf_plan_s* pl, float2* xsol, cudaStream_t st) {
  Lanes ln(pl, st, n_batches(pl));
  MRF_TRY(ln.begin());
  float* dap = pl->dap;
  pl->dap = pl->ones;   // dp() copies: unit deapodisation
  mrf_status rc = MRF_OK;
  for (int b = 0, l0 = 0; l0 < pl->L && rc == MRF_OK; ++b, l0 += pl->bf) {
    const int nb = std::min(pl->bf, pl->L - l0);
    cudaStream_t s = ln.stream(b);
    float2* Hf = pl->Hs[ln.slot(b)];
    rc = launch_fwd_rows_cg<G>(pl, xsol, Hf, l0, nb, s, nullptr, 0, pl->pnp);
    if (rc == MRF_OK) rc = launch_toep_cols<G>(pl, Hf, pl->hacg + (size_t)l0 * pl->N * pl->G, l0, nb, s, pl->tqp);
  }
  pl->dap = dap;
  MRF_TRY(rc);
  return ln.end();
}
template <int G>
static mrf_status run_cg_split_adj_toep(mrf_plan_s* pl, float mu, cudaStream_t st) {
  Lanes ln(pl, st, n_batches(pl));
  MRF_TRY(ln.begin());
  float* dap = pl->dap;
  pl->dap = pl->ones;
  mrf_status rc = MRF_OK;
  for (int b = 0, l0 = 0; l0 < pl->L && rc == MRF_OK; ++b, l0 += pl->bf) {
    const int nb = std::min(pl->bf, pl->L - l0);
    rc = launch_adj_rows<G>(pl, pl->hacg + (size_t)l0 * pl->N * pl->G, nullptr, pl->p, mu, l0, nb, pl->dotp, ln.stream(b),
                            pl->r);
  }
  pl->dap = dap;
  MRF_TRY(rc);
  return ln.end();
}

// Toeplitz form of run_normal (plans with MRF_NORMAL_TOEPLITZ): row FFT of pad(S_c x) (no
// deapodisation), k_toep_cols (column FFT, x PSF spectrum, column iFFT), row iFFT + conj-coil sum.
template <int G>
static mrf_status run_normal_toeplitz(mrf_plan_s* pl, const float2* x, float2* out, float mu, int cg, float2* xsol,
                                      cudaStream_t st) {
  Lanes ln(pl, st, n_batches(pl));
  MRF_TRY(ln.begin());
  float* dap = pl->dap;
  pl->dap = pl->ones;   // dp() copies: the launches below see unit deapodisation
  mrf_status rc = MRF_OK;
  for (int b = 0, l0 = 0; l0 < pl->L && rc == MRF_OK; ++b, l0 += pl->bf) {
    const int nb = std::min(pl->bf, pl->L - l0);
    cudaStream_t s = ln.stream(b);
    float2* Hf = pl->Hs[ln.slot(b)];
    float2* Ha = pl->Has[ln.slot(b)];
    if (cg && pl->C == 1) rc = launch_fwd_rows_cg<G>(pl, xsol, Hf, l0, nb, s, nullptr, 0);
    else rc = launch_fwd_rows<G>(pl, x, Hf, l0, nb, s);
    if (rc == MRF_OK) rc = launch_toep_cols<G>(pl, Hf, Ha, l0, nb, s);
    if (rc == MRF_OK)
      rc = launch_adj_rows<G>(pl, Ha, out, (mu != 0.f || cg) ? x : nullptr, mu, l0, nb, cg ? pl->dotp : nullptr, s);
  }
  pl->dap = dap;
  MRF_TRY(rc);
  return ln.end();
}

#define DISPATCH_G(pl, fn, ...)                               \
  switch ((pl)->G) {                                          \
    case 64: return fn<64>(__VA_ARGS__);                      \
    case 128: return fn<128>(__VA_ARGS__);                    \
    case 256: return fn<256>(__VA_ARGS__);                    \
    case 512: return fn<512>(__VA_ARGS__);                    \
    case 1024: return fn<1024>(__VA_ARGS__);                  \
    default: return fail(MRF_EUNSUPPORTED, "unsupported G");  \
  }

static mrf_status do_forward(mrf_plan_s* pl, const float2* x, float2* y, cudaStream_t st) {
  DISPATCH_G(pl, run_forward, pl, x, y, st);
}
static mrf_status do_adjoint(mrf_plan_s* pl, const float2* y, float2* x, cudaStream_t st) {
  DISPATCH_G(pl, run_adjoint, pl, y, x, st);
}
static mrf_status do_normal(mrf_plan_s* pl, const float2* x, float2* out, float mu, cudaStream_t st, int cg = 0,
                            float2* xsol = nullptr) {
  if (pl->flags & MRF_NORMAL_TOEPLITZ) {
    DISPATCH_G(pl, run_normal_toeplitz, pl, x, out, mu, cg, xsol, st);
  }
  DISPATCH_G(pl, run_normal, pl, x, out, mu, cg, xsol, st);
}
static mrf_status do_setup(mrf_plan_s* pl) { DISPATCH_G(pl, setup_kernels, pl); }
static mrf_status do_cg_split_fwd(mrf_plan_s* pl, float2* xsol, cudaStream_t st) {
  if (pl->flags & MRF_NORMAL_TOEPLITZ) {
    DISPATCH_G(pl, run_cg_split_fwd_toep, pl, xsol, st);
  }
  DISPATCH_G(pl, run_cg_split_fwd, pl, xsol, st);
}
static mrf_status do_cg_split_adj(mrf_plan_s* pl, float mu, cudaStream_t st) {
  if (pl->flags & MRF_NORMAL_TOEPLITZ) {
    DISPATCH_G(pl, run_cg_split_adj_toep, pl, mu, st);
  }
  DISPATCH_G(pl, run_cg_split_adj, pl, mu, st);
}

// ---------------------------------------------------------------------------- CG (device scalars)
static int vec_blocks(size_t n) {
  const size_t b = (n + kVecThreads - 1) / kVecThreads;
  return (int)std::max<size_t>(1, std::min<size_t>(b, kPartBlocks));
}

// In-place sum over the plan's ranks: NCCL on the plan's communicator, or the
// host hook of mrf_plan_set_host_allreduce (D2H into pinned staging, synchronise, callback, H2D).
mrf_status mrf::plan_allreduce(mrf_plan pl, void* buf, size_t n, int dtype, cudaStream_t st) {
  if (n == 0) return MRF_OK;
  if (pl->host_ar) {
    const size_t bytes = n * (dtype == MRF_DTYPE_F64 ? 8 : 4);
    if (pl->host_ar_cap < bytes) {
      if (pl->host_ar_buf) cudaFreeHost(pl->host_ar_buf);
      pl->host_ar_buf = nullptr;
      pl->host_ar_cap = 0;
      CUDA_TRY(cudaMallocHost(&pl->host_ar_buf, bytes));
      pl->host_ar_cap = bytes;
    }
    ProfScope ps(pl, MRF_K_OTHER, st);
    CUDA_TRY(cudaMemcpyAsync(pl->host_ar_buf, buf, bytes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const int rc = pl->host_ar(pl->host_ar_buf, n, dtype, pl->host_ar_ctx);
    if (rc != 0) return fail(MRF_ENCCL, "host all-reduce callback returned " + std::to_string(rc));
    CUDA_TRY(cudaMemcpyAsync(buf, pl->host_ar_buf, bytes, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));   // the staging buffer is reused by the next call
    return MRF_OK;
  }
  if (!pl->nccl_comm) return MRF_OK;
  const char* why = nullptr;
  const NcclApi* api = nccl_api(&why);
  if (!api) return fail(MRF_ENCCL, why);
  ProfScope ps(pl, MRF_K_OTHER, st);
  const int rc = api->AllReduce(buf, buf, n, dtype == MRF_DTYPE_F64 ? kNcclFloat64 : kNcclFloat32, kNcclSum,
                                pl->nccl_comm, st);
  if (rc != 0) return fail(MRF_ENCCL, std::string("ncclAllReduce: ") + api->GetErrorString(rc));
  return MRF_OK;
}

static mrf_status allreduce2(mrf_plan_s* pl, double2* v, cudaStream_t st) {
  return plan_allreduce(pl, v, 2, MRF_DTYPE_F64, st);
}

// ---------------------------------------------------------------------------- PCG preconditioner
// (precond.cuh; reading 28)
static constexpr int kPcBlocks = 16 * 148;

template <int N>
static mrf_status pc_setup_t(mrf_plan_s* pl) {
  CUDA_TRY(cudaFuncSetAttribute(pc::k_pc_rows<N, -1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pc::rows_smem<N>()));
  CUDA_TRY(cudaFuncSetAttribute(pc::k_pc_rows<N, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pc::rows_smem<N>()));
  CUDA_TRY(cudaFuncSetAttribute(pc::k_pc_cols<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pc::cols_smem<N>()));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl->pc_occ_rows, pc::k_pc_rows<N, 1, true>, pc::kRowThreads,
                                                         pc::rows_smem<N>()));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl->pc_occ_cols, pc::k_pc_cols<N>, pc::cols_threads<N>(),
                                                         pc::cols_smem<N>()));
  if (pl->pc_occ_rows < 1 || pl->pc_occ_cols < 1) return fail(MRF_EUNSUPPORTED, "preconditioner kernels do not fit");
  return MRF_OK;
}

// z = M^-1 r over the plan's frames, *npart float64 partials of <r, z> in pl->pc_part
template <int N>
static mrf_status run_precond(mrf_plan_s* pl, const float2* r, float2* z, cudaStream_t st, int* npart) {
  const long long nrows = (long long)pl->L * N;
  const long long ritems = nrows / pc::Row<N>::RPC;
  const int gr = (int)std::max<long long>(1, std::min<long long>({ritems, (long long)pl->pc_occ_rows * pl->nsm, kPcBlocks}));
  const int gc = (int)std::max<long long>(1, std::min<long long>((long long)pl->L * (N / pc::SWc), (long long)pl->pc_occ_cols * pl->nsm));
  const double gamma = pl->pc_gamma;   // set by ensure_precond for the call's mu
  ProfScope ps(pl, MRF_K_CG_VEC, st);
  pc::k_pc_rows<N, -1, false><<<gr, pc::kRowThreads, pc::rows_smem<N>(), st>>>(r, pl->pc_tmp, nullptr, nrows, 1.f, nullptr);
  MRF_TRY(check_launch("k_pc_rows"));
  pc::k_pc_cols<N><<<gc, pc::cols_threads<N>(), pc::cols_smem<N>(), st>>>(pl->pc_tmp, pl->pc_lam, pl->fil, pl->L,
                                                                            pl->pc_scale, (float)gamma);
  MRF_TRY(check_launch("k_pc_cols"));
  pc::k_pc_rows<N, 1, true><<<gr, pc::kRowThreads, pc::rows_smem<N>(), st>>>(pl->pc_tmp, z, r, nrows,
                                                                                1.f / ((float)N * (float)N), pl->pc_part);
  MRF_TRY(check_launch("k_pc_rows"));
  *npart = gr;
  return MRF_OK;
}

#define DISPATCH_N(pl, fn, ...)                               \
  switch ((pl)->N) {                                          \
    case 32: return fn<32>(__VA_ARGS__);                      \
    case 64: return fn<64>(__VA_ARGS__);                      \
    case 128: return fn<128>(__VA_ARGS__);                    \
    case 256: return fn<256>(__VA_ARGS__);                    \
    case 512: return fn<512>(__VA_ARGS__);                    \
    default: return fail(MRF_EUNSUPPORTED, "unsupported N");  \
  }
static mrf_status pc_setup(mrf_plan_s* pl) { DISPATCH_N(pl, pc_setup_t, pl); }
static mrf_status do_precond(mrf_plan_s* pl, const float2* r, float2* z, cudaStream_t st, int* npart) {
  DISPATCH_N(pl, run_precond, pl, r, z, st, npart);
}

// Plan-time (first PCG call) eigenvalues lambda_r[m] = N^-4 sum_j F(kx_j - mx/N) F(ky_j - my/N) in
// float64 on the device (Fejer factors, then the (N x M)(M x N) product of k_psf_gemm), stored
// fp32; the float64 mean over all interleaves and the mean coil power fix gamma.  pc_gamma
// caches gamma for the last mu.
static mrf_status ensure_precond(mrf_plan_s* pl, float mu, cudaStream_t st) {
  const int N = pl->N, M = pl->M, R = pl->R;
  const size_t nx = (size_t)pl->L * N * N;
  if (!pl->pc_lam) {
    MRF_TRY(pc_setup(pl));
    MRF_TRY(dev_alloc(pl, &pl->z, nx));
    MRF_TRY(dev_alloc(pl, &pl->pc_tmp, nx));
    MRF_TRY(dev_alloc(pl, &pl->pc_part, kPcBlocks));
    float* lam = nullptr;
    MRF_TRY(dev_alloc(pl, &lam, (size_t)R * N * N));
    float* traj = nullptr;
    double *Fx = nullptr, *Fy = nullptr, *Tm = nullptr;
    auto cleanup = [&]() {
      for (void* v : {(void*)traj, (void*)Fx, (void*)Fy, (void*)Tm})
        if (v) cudaFree(v);
    };
    if (cudaMalloc((void**)&traj, (size_t)R * M * 2 * sizeof(float)) != cudaSuccess ||
        cudaMalloc((void**)&Fx, (size_t)M * N * sizeof(double)) != cudaSuccess ||
        cudaMalloc((void**)&Fy, (size_t)M * N * sizeof(double)) != cudaSuccess ||
        cudaMalloc((void**)&Tm, (size_t)R * N * N * sizeof(double)) != cudaSuccess) {
      cleanup();
      cudaFree(lam);
      cudaGetLastError();
      return fail(MRF_ENOMEM, "preconditioner workspace");
    }
    cudaError_t e = cudaMemcpyAsync(traj, pl->traj_h.data(), (size_t)R * M * 2 * sizeof(float), cudaMemcpyHostToDevice, st);
    const double scale = 1.0 / ((double)N * N * (double)N * N);
    for (int r = 0; r < R && e == cudaSuccess; ++r) {
      const float* tr = traj + (size_t)r * M * 2;
      pc::k_pc_fejer<<<592, 256, 0, st>>>(tr, M, N, 0, Fx);
      pc::k_pc_fejer<<<592, 256, 0, st>>>(tr, M, N, 1, Fy);
      k_psf_gemm<<<dim3((N + 63) / 64, (N + 63) / 64), 256, 0, st>>>(Fy, Fx, M, N, scale, Tm + (size_t)r * N * N);
      e = cudaGetLastError();
    }
    std::vector<double> h((size_t)R * N * N);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), Tm, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cleanup();
    if (e != cudaSuccess) {
      cudaFree(lam);
      return fail(MRF_ECUDA, std::string("preconditioner eigenvalues: ") + cudaGetErrorString(e));
    }
    std::vector<float> hf(h.size());
    double sum = 0.0;
    for (size_t i = 0; i < h.size(); ++i) {
      sum += h[i];
      hf[i] = (float)h[i];
    }
    CUDA_TRY(cudaMemcpy(lam, hf.data(), hf.size() * sizeof(float), cudaMemcpyHostToDevice));
    pl->pc_lam = lam;
    pl->pc_lam_sum = sum / (double)h.size();
    double cp = 1.0;   // mean coil power (1/N^2) sum_n sum_c |S_c|^2
    if (pl->coils) {
      std::vector<float2> c((size_t)pl->C * N * N);
      CUDA_TRY(cudaMemcpy(c.data(), pl->coils, c.size() * sizeof(float2), cudaMemcpyDeviceToHost));
      cp = 0.0;
      for (const float2& v : c) cp += (double)v.x * v.x + (double)v.y * v.y;
      cp /= (double)N * N;
    }
    pl->pc_scale = (float)cp;
  }
  pl->pc_gamma = (double)mu + pl->pc_shift * (double)pl->pc_scale * pl->pc_lam_sum;   // gamma
  return MRF_OK;
}

// dst = the fixed-order sum of the partials; then the scalar step OP.  Without a communicator the
// reduction and the scalar step are one launch; with one, dst is all-reduced in between.
template <int OP>
static mrf_status reduce_step(mrf_plan_s* pl, const double2* part, int nblk, double2* dst, double* hx, int k,
                              cudaStream_t st) {
  const bool comm = pl->nccl_comm || pl->host_ar;
  {
    ProfScope ps(pl, MRF_K_CG_VEC, st);
    if (comm) k_reduce<kRedPlain><<<1, kReduceThreads, 0, st>>>(part, nblk, dst, pl->sc, pl->hist, hx, k);
    else k_reduce<OP><<<1, kReduceThreads, 0, st>>>(part, nblk, dst, pl->sc, pl->hist, hx, k);
    MRF_TRY(check_launch("k_reduce"));
  }
  if (!comm) return MRF_OK;
  MRF_TRY(allreduce2(pl, dst, st));
  ProfScope ps(pl, MRF_K_CG_VEC, st);
  if (OP == kRedStart) k_cg_start<<<1, 1, 0, st>>>(pl->sc, pl->hist);
  if (OP == kRedAlpha) k_cg_alpha<<<1, 1, 0, st>>>(pl->sc, hx, k);
  if (OP == kRedBeta) k_cg_beta<<<1, 1, 0, st>>>(pl->sc, pl->hist, hx, k);
  if (OP == kRedStartPc) k_cg_start_pc<<<1, 1, 0, st>>>(pl->sc, pl->hist);
  if (OP == kRedBetaPc) k_cg_beta_pc<<<1, 1, 0, st>>>(pl->sc, pl->hist, hx, k);
  return check_launch("k_cg_scalar");
}

static mrf_status vec_launch_check(const char* what) { return check_launch(what); }

// CG on (A^H A + mu I) x = A^H y + mu z, with the vector work fused:
// iteration k runs one row pass that forms p_k = r_k + beta_{k-1} p_{k-1} and advances
// x_k = x_{k-1} + alpha_{k-1} p_{k-1} (same iterates as the textbook order), the normal operator
// whose last pass also emits <p_k, q_k> partials, and one r-update pass that emits <r, r>.
// run_cg_launch issues the whole solve on `st` (no host synchronisation when tol == 0); it is
// what the CUDA graph of a tol == 0 solve captures.
static mrf_status run_cg_launch(mrf_plan_s* pl, const float2* y, const float2* z, float mu, int n_iter, float tol,
                                float2* x, cudaStream_t st, bool zero_init, bool pc, int* iters_done, double* res0_out) {
  const size_t n = (size_t)pl->L * pl->N * pl->N;
  const int nblk = vec_blocks(n);
  double* hist_a = pl->hist + pl->hist_cap;
  double* hist_b = pl->hist + 2 * pl->hist_cap;
  // PCG (oracle/pcg.py): the fused row pass forms p = z + beta p from z = M^-1 r
  float2* rin = pc ? pl->z : pl->r;
  pl->cg_rin = rin;
  // rhs = A^H y + mu z  -> r
  MRF_TRY(do_adjoint(pl, y, pl->r, st));
  if (z && mu != 0.f) {
    ProfScope ps(pl, MRF_K_CG_VEC, st);
    k_axpy<<<nblk, kVecThreads, 0, st>>>(pl->r, z, mu, n);
    MRF_TRY(vec_launch_check("k_axpy"));
  }
  // r = rhs - H x0 ; p = r ; rho0   (x0 = 0: no normal operator, x = 0)
  if (zero_init) {
    CUDA_TRY(cudaMemsetAsync(x, 0, n * sizeof(float2), st));
  } else {
    MRF_TRY(do_normal(pl, x, pl->q, mu, st));
  }
  {
    ProfScope ps(pl, MRF_K_CG_VEC, st);
    k_cg_init<<<nblk, kVecThreads, 0, st>>>(pl->r, zero_init ? nullptr : pl->q, pl->r, pl->p, n, pl->part);
    MRF_TRY(vec_launch_check("k_cg_init"));
  }
  if (pc) {   // rr0, then z0 = M^-1 r0 and rho0 = <r0, z0>
    MRF_TRY(reduce_step<kRedPlain>(pl, pl->part, nblk, &pl->sc->rr, nullptr, 0, st));
    int npart = 0;
    MRF_TRY(do_precond(pl, pl->r, pl->z, st, &npart));
    MRF_TRY(reduce_step<kRedStartPc>(pl, pl->pc_part, npart, &pl->sc->rz, nullptr, 0, st));
  } else {
    MRF_TRY(reduce_step<kRedStart>(pl, pl->part, nblk, &pl->sc->rr, nullptr, 0, st));
  }
  double res0 = -1.0;
  if (tol > 0.f) {
    CUDA_TRY(cudaMemcpyAsync(&res0, &pl->sc->res0, sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  *iters_done = n_iter;
  const bool comm = pl->nccl_comm || pl->host_ar;
  const bool toep = (pl->flags & MRF_NORMAL_TOEPLITZ) != 0;
  const bool split = !pc && (toep ? pl->C == 1 && pl->hacg != nullptr : pl->ycg != nullptr);
  for (int k = 0; k < n_iter; ++k) {
    if (tol > 0.f && res0 == 0.0) { *iters_done = 0; break; }
    if (pl->C > 1) {   // unfused p / x update (the multi-coil row pass reads the image once per coil)
      ProfScope ps(pl, MRF_K_CG_VEC, st);
      k_cg_px<<<nblk, kVecThreads, 0, st>>>(x, pl->p, rin, n, pl->sc, split ? pl->pnp : nullptr);
      MRF_TRY(vec_launch_check("k_cg_px"));
    }
    if (split) {   // alpha from <p, A^H A p> + mu ||p||^2; the adjoint half advances r and emits <r, r>
      MRF_TRY(do_cg_split_fwd(pl, x, st));
      {
        ProfScope ps(pl, MRF_K_CG_VEC, st);
        const double2* pa = pl->part;   // gridding: ||y||^2 partials of y = A p; Toeplitz: Parseval partials
        int na = 0;
        if (toep) {
          pa = pl->tqp;
          na = pl->L * pl->C * pl->S * (cols_threads_rt(pl->G) / 32);
        } else {
          const size_t ny = (size_t)pl->L * pl->C * pl->M;
          na = vec_blocks(ny);
          k_sqnorm<<<na, kVecThreads, 0, st>>>(pl->ycg, ny, pl->part);
          MRF_TRY(vec_launch_check("k_sqnorm"));
        }
        // ||p||^2 partials: per warp and row item from the fused row pass (C == 1), per block from
        // k_cg_px (C > 1)
        const int npn = pl->C == 1 ? (int)(pl->ndotp * (kRowThreads / 32)) : nblk;
        if (comm) k_reduce_pq<kRedPlain><<<1, kReduceThreads, 0, st>>>(pa, na, pl->pnp, npn, (double)mu, &pl->sc->pq, pl->sc, hist_a, k);
        else k_reduce_pq<kRedAlpha><<<1, kReduceThreads, 0, st>>>(pa, na, pl->pnp, npn, (double)mu, &pl->sc->pq, pl->sc, hist_a, k);
        MRF_TRY(vec_launch_check("k_reduce_pq"));
      }
      if (comm) {
        MRF_TRY(allreduce2(pl, &pl->sc->pq, st));
        ProfScope ps(pl, MRF_K_CG_VEC, st);
        k_cg_alpha<<<1, 1, 0, st>>>(pl->sc, hist_a, k);
        MRF_TRY(vec_launch_check("k_cg_alpha"));
      }
      MRF_TRY(do_cg_split_adj(pl, mu, st));
      MRF_TRY(reduce_step<kRedBeta>(pl, pl->dotp, (int)pl->ndotp, &pl->sc->rr, hist_b, k, st));
    } else {
    MRF_TRY(do_normal(pl, pl->p, pl->q, mu, st, 1, x));
    MRF_TRY(reduce_step<kRedAlpha>(pl, pl->dotp, (int)pl->ndotp, &pl->sc->pq, hist_a, k, st));
    {
      ProfScope ps(pl, MRF_K_CG_VEC, st);
      k_cg_r<<<nblk, kVecThreads, 0, st>>>(pl->r, pl->q, n, pl->sc, pl->part);
      MRF_TRY(vec_launch_check("k_cg_r"));
    }
    if (pc) {
      MRF_TRY(reduce_step<kRedPlain>(pl, pl->part, nblk, &pl->sc->rr, nullptr, 0, st));
      int npart = 0;
      MRF_TRY(do_precond(pl, pl->r, pl->z, st, &npart));
      MRF_TRY(reduce_step<kRedBetaPc>(pl, pl->pc_part, npart, &pl->sc->rz, hist_b, k, st));
    } else {
      MRF_TRY(reduce_step<kRedBeta>(pl, pl->part, nblk, &pl->sc->rr, hist_b, k, st));
    }
    }
    if (tol > 0.f) {
      double res = 0.0;
      CUDA_TRY(cudaMemcpyAsync(&res, &pl->sc->res, sizeof(double), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      if (std::sqrt(res / res0) < (double)tol) { *iters_done = k + 1; break; }
    }
  }
  if (n_iter > 0 && *iters_done > 0) {   // x += alpha_last p_last
    ProfScope ps(pl, MRF_K_CG_VEC, st);
    k_cg_xfin<<<nblk, kVecThreads, 0, st>>>(x, pl->p, n, pl->sc);
    MRF_TRY(vec_launch_check("k_cg_xfin"));
  }
  *res0_out = res0;
  return MRF_OK;
}

// A tol == 0 solve is a fixed launch sequence: it is captured once into a CUDA graph (on the
// plan's capture stream, forked from the caller's stream) and replayed while its arguments stay
// the same -- one graph launch per solve instead of ~40 launches per iteration.  Not used when
// tol > 0 (host-side stopping), with the host all-reduce hook (host synchronisation), while
// per-kernel profiling is on (its events are per launch), or with MRF_CG_GRAPH=0.
static bool g_cg_graph = [] {
  const char* e = std::getenv("MRF_CG_GRAPH");
  return !(e && e[0] == '0');
}();

static void drop_cg_graphs(mrf_plan_s* pl) {
  for (int i = 0; i < mrf_plan_s::kGraphs; ++i) {
    if (pl->cg_exec[i]) cudaGraphExecDestroy(pl->cg_exec[i]);
    pl->cg_exec[i] = nullptr;
    pl->cg_key[i] = CgKey();
  }
}

static mrf_status run_cg(mrf_plan_s* pl, const float2* y, const float2* z, float mu, int n_iter, float tol,
                         float2* x, mrf_cg_info* info, cudaStream_t st, bool zero_init = false, bool pc = false) {
  if (pc) MRF_TRY(ensure_precond(pl, mu, st));
  if (n_iter + 1 > pl->hist_cap) {   // [sqrt(rho_k), k <= n][alpha_k][beta_k]
    drop_cg_graphs(pl);
    if (pl->hist) cudaFree(pl->hist);
    pl->hist = nullptr;
    pl->hist_cap = 0;
    MRF_TRY(dev_alloc(pl, &pl->hist, 3 * ((size_t)n_iter + 1)));
    pl->hist_cap = n_iter + 1;
  }
  int iters_done = n_iter;
  double rho0 = -1.0;
  const bool graph = g_cg_graph && tol == 0.f && !pl->host_ar && !pl->prof.on;
  if (graph) {
    const CgKey key{x, y, z, mu, n_iter, zero_init, pc};
    int slot = -1;
    for (int i = 0; i < mrf_plan_s::kGraphs; ++i)
      if (pl->cg_exec[i] && pl->cg_key[i] == key) slot = i;
    if (slot < 0) {   // capture into the least recently used slot
      slot = 0;
      for (int i = 1; i < mrf_plan_s::kGraphs; ++i)
        if (pl->cg_use[i] < pl->cg_use[slot]) slot = i;
      if (pl->cg_exec[slot]) cudaGraphExecDestroy(pl->cg_exec[slot]);
      pl->cg_exec[slot] = nullptr;
      if (!pl->gstream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->gstream, cudaStreamNonBlocking));
      CUDA_TRY(cudaStreamBeginCapture(pl->gstream, cudaStreamCaptureModeThreadLocal));
      mrf_status rc = run_cg_launch(pl, y, z, mu, n_iter, tol, x, pl->gstream, zero_init, pc, &iters_done, &rho0);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(pl->gstream, &g);
      if (rc != MRF_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (ce != cudaSuccess) return fail(MRF_ECUDA, std::string("CG graph capture: ") + cudaGetErrorString(ce));
      const cudaError_t ie = cudaGraphInstantiate(&pl->cg_exec[slot], g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) {
        pl->cg_exec[slot] = nullptr;
        return fail(MRF_ECUDA, std::string("CG graph instantiate: ") + cudaGetErrorString(ie));
      }
      pl->cg_key[slot] = key;
    }
    pl->cg_use[slot] = ++pl->cg_clock;
    CUDA_TRY(cudaGraphLaunch(pl->cg_exec[slot], st));
  } else {
    MRF_TRY(run_cg_launch(pl, y, z, mu, n_iter, tol, x, st, zero_init, pc, &iters_done, &rho0));
  }
  CGScalars hs;
  CUDA_TRY(cudaMemcpyAsync(&hs, pl->sc, sizeof(CGScalars), cudaMemcpyDeviceToHost, st));
  std::vector<double> hh(3 * (size_t)pl->hist_cap, 0.0);
  CUDA_TRY(cudaMemcpyAsync(hh.data(), pl->hist, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (hs.res0 == 0.0) iters_done = 0;
  if (info) {
    info->iters = iters_done;
    info->rel_resid = hs.res0 > 0.0 ? std::sqrt(hs.res / hs.res0) : 0.0;
    if (info->history) {
      for (int i = 0; i <= n_iter; ++i) info->history[i] = i <= iters_done ? hh[i] : 0.0;
    }
    for (int i = 0; i < n_iter; ++i) {
      if (info->alpha) info->alpha[i] = i < iters_done ? hh[pl->hist_cap + i] : 0.0;
      if (info->beta) info->beta[i] = i < iters_done ? hh[2 * pl->hist_cap + i] : 0.0;
    }
  }
  if (hs.breakdown) return fail(MRF_ENUMERIC, "CG breakdown: Re<p, (A^H A + mu I) p> <= 0 or non-finite");
  return MRF_OK;
}

// ================================================================================== pointers
// 0 = device memory of the plan's device, 1 = host memory, -1 = other device / invalid
static int ptr_kind(const void* ptr, int dev) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return at.device == dev ? 0 : -1;
  return 1;
}

static mrf_status classify(mrf_plan_s* pl, std::initializer_list<const void*> ptrs, bool* host) {
  int kind = -2;
  for (const void* v : ptrs) {
    if (!v) continue;
    if ((uintptr_t)v % 16 != 0) return fail(MRF_EINVAL, "arrays must be 16-byte aligned");
    const int k = ptr_kind(v, pl->device);
    if (k < 0) return fail(MRF_EINVAL, "pointer is device memory of another device");
    if (kind == -2) kind = k;
    else if (kind != k) return fail(MRF_EINVAL, "host and device pointers mixed in one call");
  }
  *host = kind == 1;
  return MRF_OK;
}

static mrf_status ensure_staging(mrf_plan_s* pl, bool need_z) {
  const size_t nx = (size_t)pl->L * pl->N * pl->N, ny = (size_t)pl->L * pl->C * pl->M;
  if (!pl->stg_x) MRF_TRY(dev_alloc(pl, &pl->stg_x, nx));
  if (!pl->stg_y) MRF_TRY(dev_alloc(pl, &pl->stg_y, std::max(ny, nx)));   // also 2nd image buffer
  if (need_z && !pl->stg_z) MRF_TRY(dev_alloc(pl, &pl->stg_z, nx));
  return MRF_OK;
}

static mrf_status ensure_async(mrf_plan_s* pl, bool need_z) {
  const size_t nx = (size_t)pl->L * pl->N * pl->N, ny = (size_t)pl->L * pl->C * pl->M;
  for (int i = 0; i < 2; ++i) {
    if (!pl->ax[i]) MRF_TRY(dev_alloc(pl, &pl->ax[i], nx));
    if (!pl->ay[i]) MRF_TRY(dev_alloc(pl, &pl->ay[i], ny));
    if (!pl->ev_solved[i]) CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_solved[i], cudaEventDisableTiming));
    if (!pl->ev_copied[i]) CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_copied[i], cudaEventDisableTiming));
  }
  if (!pl->cstream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->cstream, cudaStreamNonBlocking));
  if (need_z && !pl->stg_z) MRF_TRY(dev_alloc(pl, &pl->stg_z, nx));
  return MRF_OK;
}

// Toeplitz PSF spectra (MRF_NORMAL_TOEPLITZ), float64 on the device, one interleaf at a time:
// Dirichlet factors D_x, D_y [M][G], T_r = D_y^T D_x / (G^2 N^2) (gridding.cuh k_psf_*), stored fp32.
static mrf_status build_psf(mrf_plan_s* pl, const float* traj_host, cudaStream_t st) {
  const int N = pl->N, G = pl->G, M = pl->M, R = pl->R;
  MRF_TRY(dev_alloc(pl, &pl->psf, (size_t)R * G * G));
  MRF_TRY(dev_alloc(pl, &pl->ones, (size_t)N));
  std::vector<float> one((size_t)N, 1.0f);
  CUDA_TRY(cudaMemcpyAsync(pl->ones, one.data(), N * sizeof(float), cudaMemcpyHostToDevice, st));
  float* traj = nullptr;
  double *Dx = nullptr, *Dy = nullptr, *Tm = nullptr;
  auto cleanup = [&]() {
    if (traj) cudaFree(traj);
    if (Dx) cudaFree(Dx);
    if (Dy) cudaFree(Dy);
    if (Tm) cudaFree(Tm);
  };
  if (cudaMalloc((void**)&traj, (size_t)R * M * 2 * sizeof(float)) != cudaSuccess ||
      cudaMalloc((void**)&Dx, (size_t)M * G * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&Dy, (size_t)M * G * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&Tm, (size_t)G * G * sizeof(double)) != cudaSuccess) {
    cleanup();
    cudaGetLastError();
    return fail(MRF_ENOMEM, "PSF workspace");
  }
  cudaError_t e = cudaMemcpyAsync(traj, traj_host, (size_t)R * M * 2 * sizeof(float), cudaMemcpyHostToDevice, st);
  const double scale = 1.0 / ((double)G * G * (double)N * N);
  for (int r = 0; r < R && e == cudaSuccess; ++r) {
    const float* tr = traj + (size_t)r * M * 2;
    k_psf_dirichlet<<<1184, 256, 0, st>>>(tr, M, N, G, 0, Dx);
    k_psf_dirichlet<<<1184, 256, 0, st>>>(tr, M, N, G, 1, Dy);
    k_psf_gemm<<<dim3((G + 63) / 64, (G + 63) / 64), 256, 0, st>>>(Dy, Dx, M, G, scale, Tm);
    k_psf_store<<<592, 256, 0, st>>>(Tm, G, pl->psf + (size_t)r * G * G);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cleanup();
  if (e != cudaSuccess) return fail(MRF_ECUDA, std::string("PSF precompute: ") + cudaGetErrorString(e));
  return MRF_OK;
}

void mrf::plan_dims(mrf_plan pl, int* N, int* L, int* C, int* device, int* M) {
  if (M) *M = pl->M;
  *N = pl->N;
  *L = pl->L;
  *C = pl->C;
  *device = pl->device;
}

// ---------------------------------------------------------------------------- subspace normal
// (gridding.cuh k_sn_*; used by mrf_msllr_solve on Toeplitz plans, llr.cu)
bool mrf::plan_has_comm(mrf_plan pl) { return pl->nccl_comm != nullptr || pl->host_ar != nullptr; }
int mrf::plan_frame_offset(mrf_plan pl) { return pl->frame_offset; }
bool mrf::plan_toeplitz(mrf_plan pl) { return (pl->flags & MRF_NORMAL_TOEPLITZ) != 0 && pl->psf; }
unsigned long long mrf::plan_serial(mrf_plan pl) { return pl->serial; }
long long mrf::sn_elems(mrf_plan pl) { return (long long)pl->G * pl->G; }

mrf_status mrf::sn_build(mrf_plan pl, const float2* basis_h, int r, float2* K, cudaStream_t st) {
  if (!plan_toeplitz(pl)) return fail(MRF_EINVAL, "the subspace normal needs a plan with MRF_NORMAL_TOEPLITZ");
  DeviceGuard guard(pl->device);
  const int L = pl->L, R = pl->R;
  std::vector<int> fil(L);
  CUDA_TRY(cudaMemcpy(fil.data(), pl->fil, (size_t)L * sizeof(int), cudaMemcpyDeviceToHost));
  // c^rho_ji = sum_{l in rho} conj(d_jl) d_il  (float64)
  std::vector<std::complex<double>> cd((size_t)r * r * R, 0.0);
  for (int l = 0; l < L; ++l) {
    const int rho = fil[l];
    for (int j = 0; j < r; ++j) {
      const std::complex<double> dj(basis_h[(size_t)j * L + l].x, -basis_h[(size_t)j * L + l].y);
      for (int i = 0; i < r; ++i) {
        const std::complex<double> di(basis_h[(size_t)i * L + l].x, basis_h[(size_t)i * L + l].y);
        cd[((size_t)j * r + i) * R + rho] += dj * di;
      }
    }
  }
  const int pairs = r * (r + 1) / 2;   // j <= i (K is Hermitian in (j, i))
  std::vector<float2> cc((size_t)pairs * R);
  for (int j = 0; j < r; ++j)
    for (int i = j; i < r; ++i)
      for (int rho = 0; rho < R; ++rho) {
        const std::complex<double> v = cd[((size_t)j * r + i) * R + rho];
        cc[(size_t)sn_pair(j, i, r) * R + rho] = make_float2((float)v.real(), (float)v.imag());
      }
  float2* ccd = nullptr;
  CUDA_TRY(cudaMalloc((void**)&ccd, cc.size() * sizeof(float2)));
  cudaError_t e = cudaMemcpyAsync(ccd, cc.data(), cc.size() * sizeof(float2), cudaMemcpyHostToDevice, st);
  const long long E = sn_elems(pl), tot = (long long)pairs * E;
  if (e == cudaSuccess) {
    k_sn_kbuild<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->psf, ccd, pairs, R, E, K);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(ccd);
  if (e != cudaSuccess) return fail(MRF_ECUDA, std::string("sn_build: ") + cudaGetErrorString(e));
  return MRF_OK;
}

template <int G>
static mrf_status run_sn(mrf_plan_s* pl, const float2* K, int r, const float2* U, float2* Z, float2* spec_a,
                         float2* spec_b, cudaStream_t st) {
  const int C = pl->C, ncol = cols_threads<G>();
  const long long E = (long long)G * G;
  float* dap = pl->dap;
  pl->dap = pl->ones;   // Toeplitz form: no deapodisation (dp() copies it into the launches)
  mrf_status rc = MRF_OK;
  for (int l0 = 0; l0 < r && rc == MRF_OK; l0 += pl->bf) {   // r frames: row FFTs, column FFTs -> spectra
    const int nb = std::min(pl->bf, r - l0);
    rc = launch_fwd_rows<G>(pl, U, pl->Hs[0], l0, nb, st);
    if (rc == MRF_OK) {
      const int items = nb * C * pl->S;
      k_sn_fcols<G><<<std::min(items, pl->nsm * 2), ncol, sn_cols_smem<G>(), st>>>(pl->tw, pl->Hs[0],
                                                                                   spec_a + (size_t)l0 * C * E, nb * C);
      if (cudaGetLastError() != cudaSuccess) rc = fail(MRF_ECUDA, "k_sn_fcols launch failed");
    }
  }
  if (rc == MRF_OK) {
    const long long n = (long long)C * E;
    if (r <= 16) k_sn_mix<16><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(spec_a, K, spec_b, r, C, E);
    else k_sn_mix<32><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(spec_a, K, spec_b, r, C, E);
    if (cudaGetLastError() != cudaSuccess) rc = fail(MRF_ECUDA, "k_sn_mix launch failed");
  }
  for (int l0 = 0; l0 < r && rc == MRF_OK; l0 += pl->bf) {   // inverse column FFTs, row iFFTs + crop
    const int nb = std::min(pl->bf, r - l0);
    const int items = nb * C * pl->S;
    k_sn_icols<G><<<std::min(items, pl->nsm * 2), ncol, sn_cols_smem<G>(), st>>>(pl->tw, spec_b + (size_t)l0 * C * E,
                                                                                 pl->Has[0], nb * C);
    if (cudaGetLastError() != cudaSuccess) rc = fail(MRF_ECUDA, "k_sn_icols launch failed");
    if (rc == MRF_OK) rc = launch_adj_rows<G>(pl, pl->Has[0], Z, nullptr, 0.f, l0, nb, nullptr, st);
  }
  pl->dap = dap;
  return rc;
}

mrf_status mrf::sn_apply(mrf_plan pl, const float2* K, int r, const float2* U, float2* Z, float2* spec_a,
                         float2* spec_b, cudaStream_t st) {
  if (!plan_toeplitz(pl)) return fail(MRF_EINVAL, "the subspace normal needs a plan with MRF_NORMAL_TOEPLITZ");
  DeviceGuard guard(pl->device);
  DISPATCH_G(pl, run_sn, pl, K, r, U, Z, spec_a, spec_b, st);
}

// ================================================================================== C-ABI
extern "C" {

const char* mrf_status_string(mrf_status s) {
  switch (s) {
    case MRF_OK: return "MRF_OK";
    case MRF_EINVAL: return "MRF_EINVAL: invalid argument";
    case MRF_ENOMEM: return "MRF_ENOMEM: out of memory";
    case MRF_ECUDA: return "MRF_ECUDA: CUDA error";
    case MRF_ENCCL: return "MRF_ENCCL: NCCL error";
    case MRF_EUNSUPPORTED: return "MRF_EUNSUPPORTED: unsupported configuration";
    case MRF_ENUMERIC: return "MRF_ENUMERIC: numerical breakdown";
  }
  return "unknown mrf_status";
}

const char* mrf_last_error(void) { return g_err.c_str(); }

mrf_status mrf_plan_create(const mrf_plan_desc* d, mrf_plan* out) {
  if (!d || !out) return fail(MRF_EINVAL, "null desc or out");
  *out = nullptr;
  if (d->N < 8 || (d->N % 2) != 0) return fail(MRF_EINVAL, "N must be even and >= 8");
  if (d->L_local < 1 || d->M < 1 || d->R < 1 || d->C < 1) return fail(MRF_EINVAL, "L_local, M, R, C must be >= 1");
  if (d->frame_offset < 0) return fail(MRF_EINVAL, "frame_offset < 0");
  if (!d->traj) return fail(MRF_EINVAL, "null traj");
  if (d->C > 1 && !d->coils) return fail(MRF_EINVAL, "C > 1 requires coils");
  if (d->W < 2 || d->W > 16) return fail(MRF_EINVAL, "W must be in [2, 16]");
  if (!(d->sigma > 0.f) || !std::isfinite(d->sigma)) return fail(MRF_EINVAL, "sigma must be positive");
  if (d->batch_frames < 0) return fail(MRF_EINVAL, "batch_frames < 0");
  if (d->flags & ~7u) return fail(MRF_EINVAL, "unknown flags");
  if ((double)d->sigma != 2.0) return fail(MRF_EUNSUPPORTED, "only sigma = 2 is supported");
  const double Gd = (double)d->sigma * d->N;
  const int G = (int)std::lround(Gd);
  if (std::fabs(Gd - G) > 1e-9 || !(G == 64 || G == 128 || G == 256 || G == 512 || G == 1024))
    return fail(MRF_EUNSUPPORTED, "G = sigma*N must be one of 64, 128, 256, 512, 1024");
  const int N = d->N, M = d->M, R = d->R, W = d->W, C = d->C, L = d->L_local;
  // trajectory checks
  for (size_t i = 0; i < (size_t)R * M * 2; ++i) {
    const float v = d->traj[i];
    if (!std::isfinite(v) || std::fabs(v) > 0.5f) return fail(MRF_EINVAL, "trajectory entry non-finite or |k| > 0.5");
  }
  std::vector<int> fil(L);
  for (int l = 0; l < L; ++l) {
    fil[l] = d->frame_interleaf ? d->frame_interleaf[l] : (int)(((long long)d->frame_offset + l) % R);
    if (fil[l] < 0 || fil[l] >= R) return fail(MRF_EINVAL, "frame_interleaf entry out of [0, R)");
  }
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (d->device < 0 || d->device >= ndev) return fail(MRF_EINVAL, "bad device ordinal");
  DeviceGuard guard(d->device);
  cudaStream_t st = (cudaStream_t)d->stream;

  mrf_plan_s* pl = new mrf_plan_s();
  static std::atomic<unsigned long long> plan_counter{0};
  pl->serial = ++plan_counter;
  pl->N = N; pl->G = G; pl->L = L; pl->M = M; pl->R = R; pl->C = C; pl->W = W; pl->S = G / SW;
  pl->recw = (2 + 2 * W + 3) & ~3;
  if (const char* e = std::getenv("MRF_DBG")) pl->dbg = std::atoi(e);
  if (pl->dbg & 2) {
    if (cudaMalloc((void**)&pl->dbgbuf, 32 * sizeof(long long)) != cudaSuccess) return fail(MRF_ENOMEM, "dbgbuf");
    cudaMemset(pl->dbgbuf, 0, 32 * sizeof(long long));
  }
  pl->ystage = (M % 2 == 0 && (size_t)M * sizeof(float2) <= (size_t)kYBytes) ? (int)(M * sizeof(float2)) : 0;
  {
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, d->device) == cudaSuccess && nsm > 0) pl->nsm = nsm;
  }
  pl->frame_offset = d->frame_offset;
  pl->flags = d->flags;
  pl->traj_h.assign(d->traj, d->traj + (size_t)R * M * 2);
  pl->device = d->device;
  pl->nccl_comm = d->nccl_comm;
  auto bail = [&](mrf_status s) { free_plan(pl); return s; };

  // ---- constants (float64 host) ------------------------------------------------------------
  const KB kb(W, d->sigma);
  std::vector<float> dap(N);
  for (int i = 0; i < N; ++i) {
    const double n = (double)(i - N / 2);
    const double psi = (d->flags & MRF_DEAPOD_DISCRETE) ? kb.psi_discrete(n, G) : kb.psi_analytic(n, G);
    dap[i] = (float)(1.0 / (psi * std::sqrt((double)N)));
  }
  int P = 0, Q = 0, T = 0;
  fft_shape(G, &P, &Q, &T);
  std::vector<float2> tw(G);
  for (int k1 = 0; k1 < P; ++k1)
    for (int n2 = 0; n2 < Q; ++n2) {
      const double a = -2.0 * M_PI * (double)((long long)n2 * k1 % G) / G;
      tw[n2 * P + k1] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  // ---- taps, weights, strip bins (a0) ---------------------------------------------------------
  // Every point of every interleaf is binned into the 16-column strips its W x-taps touch (one
  // record per (point, strip), at most two per point); a record carries the point index, its
  // first grid row, the run of x-taps inside the strip, and the W x- and W y-weights.
  const int S = G / SW;
  const int recw = (2 + 2 * W + 3) & ~3;   // 16-byte records for the bulk copies
  std::vector<float> wts((size_t)R * M * 2 * W);
  std::vector<int> m0x((size_t)R * M), m0y((size_t)R * M);
  for (int r = 0; r < R; ++r)
    for (int j = 0; j < M; ++j) {
      const size_t pj = (size_t)r * M + j;
      for (int ax = 0; ax < 2; ++ax) {
        const double u = (double)G * (double)d->traj[pj * 2 + ax];
        const long long m0 = (long long)std::floor(u - 0.5 * W) + 1;
        for (int t = 0; t < W; ++t) wts[pj * 2 * W + ax * W + t] = (float)kb.phi(u - (double)(m0 + t));
        const int w0 = (int)(((m0 % G) + G) % G);
        (ax == 0 ? m0x : m0y)[pj] = w0;
      }
    }
  std::vector<std::vector<int2>> bins(S);
  std::vector<int> fch, ach;
  std::vector<int2> ftab((size_t)R * S), atab((size_t)R * S);
  struct Nz { int cell, j; double w; };
  std::vector<Nz> nz;
  std::vector<int2> rows;   // {first nz, count}
  std::vector<double> wtd((size_t)2 * W);
  for (int r = 0; r < R; ++r) {
    for (auto& b : bins) b.clear();
    for (int j = 0; j < M; ++j) {
      const size_t pj = (size_t)r * M + j;
      int t = 0;
      while (t < W) {   // split the W x-taps into runs of consecutive columns within one strip
        const int col = (m0x[pj] + t) % G;
        const int s = col / SW;
        int cnt = 1;
        while (t + cnt < W && ((m0x[pj] + t + cnt) % G) / SW == s && ((m0x[pj] + t + cnt) % G) == col + cnt) ++cnt;
        const int packed = m0y[pj] | (t << 11) | (cnt << 16) | ((col - s * SW) << 21);
        bins[s].push_back(make_int2(j, packed));
        t += cnt;
      }
    }
    for (int s = 0; s < S; ++s) {
      {   // deal the strip's records so that each run of 32 (one warp of the thread-per-record
          // gather) covers the 16 residues (gy0 + cx0) mod 16 evenly: with the 17-slot strip rows
          // every tap of a record sits in bank pair (gy0 + cx0 + ty + tx) mod 16, so a warp's tap
          // loads then hit each bank pair at most twice (conflict-free 64-bit accesses)
        std::vector<std::vector<int2>> res(16);
        for (const int2& rr : bins[s]) res[((rr.y & 2047) + ((rr.y >> 21) & 31)) & 15].push_back(rr);
        std::vector<size_t> nx(16, 0);
        for (size_t o = 0; o < bins[s].size(); ++o) {
          int b = (int)(o & 15);
          if (nx[b] == res[b].size()) {
            size_t best = 0;
            for (int q = 0; q < 16; ++q)
              if (res[q].size() - nx[q] > best) { best = res[q].size() - nx[q]; b = q; }
          }
          bins[s][o] = res[b][nx[b]++];
        }
      }
      const std::vector<int2>& rb = bins[s];
      const int n_rec = (int)rb.size();
      // forward chunk: header + records
      {
        const size_t base = fch.size();
        const size_t words = (size_t)kChunkHdr + (size_t)((n_rec + 31) / 32) * 32 * recw;
        fch.resize(base + words, 0);
        fch[base] = n_rec;
        for (int ri = 0; ri < n_rec; ++ri) {
          std::vector<int> rec((size_t)recw, 0);
          const int pk = rb[ri].y, tx0 = (pk >> 11) & 31, ntx = (pk >> 16) & 31;
          const float* wp = &wts[((size_t)r * M + rb[ri].x) * 2 * W];
          rec[0] = rb[ri].x;
          rec[1] = (pk & 2047) | (((pk >> 21) & 31) << 11);   // first grid row | first strip column
          float* wx = reinterpret_cast<float*>(&rec[2]);
          for (int i = 0; i < W; ++i) wx[i] = i < ntx ? wp[tx0 + i] : 0.f;   // x-weights aligned to the strip
          std::memcpy(&rec[2 + W], wp + W, sizeof(float) * W);
          // interleaved store: piece k (words 4k..4k+3) of record 32g + l at (g recw + 4k) 32 + 4l
          const size_t g = (size_t)ri / 32, l = (size_t)ri % 32;
          for (int w = 0; w < recw; ++w)
            fch[base + kChunkHdr + (g * recw + (size_t)(w & ~3)) * 32 + 4 * l + (w & 3)] = rec[(size_t)w];
        }
        ftab[(size_t)r * S + s] = make_int2((int)base, (int)words);
      }
      // adjoint chunk: spread matrix rows = cells, entries (j, w = wx*wy rounded once from float64)
      nz.clear();
      for (int ri = 0; ri < n_rec; ++ri) {
        const int j = rb[ri].x, pk = rb[ri].y;
        const int gy0 = pk & 2047, tx0 = (pk >> 11) & 31, ntx = (pk >> 16) & 31, cx0 = (pk >> 21) & 31;
        kb_taps(kb, G, W, d->traj[((size_t)r * M + j) * 2], d->traj[((size_t)r * M + j) * 2 + 1], wtd.data());
        for (int ty = 0; ty < W; ++ty)
          for (int i = 0; i < ntx; ++i) nz.push_back({((gy0 + ty) % G) * SW + cx0 + i, j, wtd[W + ty] * wtd[tx0 + i]});
      }
      std::sort(nz.begin(), nz.end(), [](const Nz& a, const Nz& b) { return a.cell != b.cell ? a.cell < b.cell : a.j < b.j; });
      rows.clear();
      for (size_t i = 0; i < nz.size();) {
        size_t k = i;
        while (k < nz.size() && nz[k].cell == nz[i].cell) ++k;
        rows.push_back(make_int2((int)i, (int)(k - i)));
        i = k;
      }
      std::stable_sort(rows.begin(), rows.end(), [](const int2& a, const int2& b) { return a.y > b.y; });
      // Slices: a cell with more than kSplitEntries entries gets a slice of its own whose 32 lanes
      // share its entries (entry i -> lane i % 32, step i / 32) and are summed by a warp reduction
      // (width stored negated); then the other cells in groups of 32, widest first; the width-1
      // slices last.  Slices [0, n_multi) are the ones wider than 1.
      // measured: 128 (stress normal 254 -> 83 ms); a lower threshold costs more in per-slice
      // reductions than it saves (MRF, where no cell exceeds 120 entries, is unaffected)
      static const int kSplitEntries = [] {   // MRF_SPLIT: experiment knob
        const char* e = std::getenv("MRF_SPLIT");
        return e ? std::max(32, std::atoi(e)) : 128;
      }();
      std::vector<int2> slices;   // {first row index, width (< 0: reduction slice of one row)}
      size_t r0 = 0;
      while (r0 < rows.size() && rows[r0].y > kSplitEntries) {
        slices.push_back(make_int2((int)r0, -((rows[r0].y + 31) / 32)));
        ++r0;
      }
      for (size_t i = r0; i < rows.size(); i += 32) slices.push_back(make_int2((int)i, rows[i].y));
      const int nsl = (int)slices.size();
      long long nent = 0;
      int n_multi = 0;
      for (int sl = 0; sl < nsl; ++sl) {
        nent += 32LL * std::abs(slices[sl].y);
        if (slices[sl].y != 1) n_multi = sl + 1;
      }
      const size_t cells_off = (size_t)kAdjHdr + 2 * (size_t)nsl;
      const size_t ent_off = (cells_off + 16 * (size_t)nsl + 3) & ~(size_t)3;   // 16-byte aligned entries
      const size_t words = (ent_off + 2 * (size_t)nent + 3) & ~(size_t)3;
      const size_t base = ach.size();
      ach.resize(base + words, 0);
      int* ch = &ach[base];
      ch[0] = nsl; ch[1] = (int)cells_off; ch[2] = (int)ent_off; ch[3] = n_multi;
      {   // row-pair masks of k_adj_cols' stage-1 loads: warp w, bit a*P + n1 <-> rows Q n1 + T a + 2w + {0,1}
        std::vector<char> touched(G, 0);
        for (const Nz& q : nz) touched[q.cell / SW] = 1;
        const int nwarps = SW * T / 32, A = Q / T;
        for (int w = 0; w < nwarps && w < 16; ++w) {
          uint32_t m = 0;
          for (int a = 0; a < A; ++a)
            for (int n1 = 0; n1 < P; ++n1) {
              const int row = Q * n1 + T * a + 2 * w;
              if (touched[row] || touched[row + 1]) m |= 1u << (a * P + n1);
            }
          ch[kChunkHdr + w] = (int)m;
        }
      }
      unsigned short* cells = reinterpret_cast<unsigned short*>(ch + cells_off);
      int2* ents = reinterpret_cast<int2*>(ch + ent_off);
      // entries of the width-1 slices first (one flat run, always staged first), then the others
      long long first = 32LL * (nsl - n_multi);
      auto put = [&](long long pos, const Nz& q) {
        const float wf = (float)q.w;
        int2 e = make_int2(q.j, 0);
        std::memcpy(&e.y, &wf, 4);
        ents[pos] = e;
      };
      auto slot = [&](const int2& row) {
        return (unsigned short)sidx(nz[row.x].cell / SW, nz[row.x].cell % SW);   // swizzled strip slot
      };
      for (int sl = 0; sl < nsl; ++sl) {
        const int width = slices[sl].y;
        if (sl == n_multi) first = 0;
        ch[kAdjHdr + 2 * sl] = (int)first;
        ch[kAdjHdr + 2 * sl + 1] = width;
        if (width < 0) {   // reduction slice: entries of one cell in order, lanes interleaved
          const int2& row = rows[(size_t)slices[sl].x];
          for (int lane = 0; lane < 32; ++lane) cells[sl * 32 + lane] = slot(row);
          for (int i = 0; i < row.y; ++i) put(first + i, nz[row.x + i]);
          first += 32LL * -width;
          continue;
        }
        for (int lane = 0; lane < 32; ++lane) {
          const size_t ri = (size_t)slices[sl].x + lane;
          cells[sl * 32 + lane] = ri < rows.size() ? slot(rows[ri]) : (unsigned short)0xFFFF;
          for (int k = 0; k < width; ++k)
            if (ri < rows.size() && k < rows[ri].y) put(first + 32LL * k + lane, nz[rows[ri].x + k]);
        }
        first += 32LL * width;
      }
      atab[(size_t)r * S + s] = make_int2((int)base, (int)words);
    }
  }
  if (fch.size() > (size_t)INT32_MAX || ach.size() > (size_t)INT32_MAX)
    return bail(fail(MRF_EUNSUPPORTED, "plan tables too large"));
  // ---- batch size: frames per launch (per lane) ---------------------------------------------------
  const size_t per_frame = (size_t)C * N * G * sizeof(float2);
  int bf = d->batch_frames;
  if (bf == 0)
    if (const char* e = std::getenv("MRF_BF")) bf = std::max(0, std::atoi(e));   // experiment knob
  if (bf == 0) {
    // per lane; measured: launch-tail amortisation beats L2 residency (MRF: 128 MB); multi-coil
    // batches hold C x the half grid per frame, and 1 GB keeps their row passes (the coil sum is
    // a loop inside an item) wide enough (SENSE 6.38 -> 6.19 ms, stress 20.8 -> 20.3 ms per 512 frames)
    const size_t target = C == 1 ? (128ull << 20) : (1ull << 30);
    bf = (int)std::max<size_t>(1, target / per_frame);
    // at least one batch per lane (frame shards of 8 GPUs: 125 MRF frames -> 2 x 63, 3 % faster)
    bf = std::min(bf, std::max(1, (L + kDefaultLanes - 1) / kDefaultLanes));
  }
  bf = std::min(bf, L);
  pl->bf = bf;
  // ---- device uploads ---------------------------------------------------------------------------
  pl->ndotp = (size_t)L * (N / (kRowThreads / (G <= 128 ? 8 : G <= 512 ? 16 : 32)));
  mrf_status s;
  if ((s = dev_alloc(pl, &pl->dap, N)) || (s = dev_alloc(pl, &pl->tw, G)) ||
      (s = dev_alloc(pl, &pl->fchunks, fch.size())) || (s = dev_alloc(pl, &pl->ftab, ftab.size())) ||
      (s = dev_alloc(pl, &pl->achunks, ach.size())) || (s = dev_alloc(pl, &pl->atab, atab.size())) ||
      (s = dev_alloc(pl, &pl->fil, L)) ||
      (s = dev_alloc(pl, &pl->Hs[0], (size_t)bf * C * N * G)) || (s = dev_alloc(pl, &pl->ybufs[0], (size_t)bf * C * M)) ||
      (s = dev_alloc(pl, &pl->r, (size_t)L * N * N)) || (s = dev_alloc(pl, &pl->p, (size_t)L * N * N)) ||
      (s = dev_alloc(pl, &pl->q, (size_t)L * N * N)) || (s = dev_alloc(pl, &pl->part, kPartBlocks)) ||
      (s = dev_alloc(pl, &pl->dotp, pl->ndotp)) || (s = dev_alloc(pl, &pl->sc, 1)))
    return bail(s);
  if (d->coils && C >= 1) {
    if ((s = dev_alloc(pl, &pl->coils, (size_t)C * N * N))) return bail(s);
  }
  {   // split-phase CG (MRF_CG_SPLIT=0 disables): gridding plans of any C, Toeplitz plans with C == 1
    const char* e = std::getenv("MRF_CG_SPLIT");
    if (!(e && e[0] == '0') && (C == 1 || !(d->flags & MRF_NORMAL_TOEPLITZ))) {
      if ((s = dev_alloc(pl, &pl->pnp, std::max<size_t>(pl->ndotp * (kRowThreads / 32), kPartBlocks)))) return bail(s);
      if (!(d->flags & MRF_NORMAL_TOEPLITZ)) {
        if ((s = dev_alloc(pl, &pl->ycg, (size_t)L * C * M))) return bail(s);
      } else if ((s = dev_alloc(pl, &pl->hacg, (size_t)L * N * G)) ||
                 (s = dev_alloc(pl, &pl->tqp, (size_t)L * (G / SW) * (SW * 32 / 32)))) {   // S items x warps
        return bail(s);
      }
    }
  }
  pl->nlanes = std::min(kDefaultLanes, (L + bf - 1) / bf);
  if (const char* e = std::getenv("MRF_LANES")) pl->nlanes = std::max(1, std::min(kMaxLanes, std::atoi(e)));
  if (pl->nlanes > 1) {
    for (int i = 1; i < pl->nlanes; ++i)
      if ((s = dev_alloc(pl, &pl->Hs[i], (size_t)bf * C * N * G)) || (s = dev_alloc(pl, &pl->ybufs[i], (size_t)bf * C * M)))
        return bail(s);
    for (int i = 0; i < pl->nlanes; ++i) {
      if (cudaStreamCreateWithFlags(&pl->lane[i], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&pl->ev_join[i], cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(MRF_ECUDA, "stream/event creation failed"));
    }
    if (cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(MRF_ECUDA, "event creation failed"));
  }
  {   // item hand-out counters of k_adj_cols (DYN variant), one pair per lane, self-resetting
    if ((s = dev_alloc(pl, &pl->ctrs, (size_t)kMaxLanes * 8))) return bail(s);
    if (cudaMemset(pl->ctrs, 0, (size_t)kMaxLanes * 8 * sizeof(int)) != cudaSuccess) return bail(fail(MRF_ECUDA, "memset"));
  }
  if ((s = do_setup(pl))) return bail(s);
  if (pl->flags & MRF_NORMAL_TOEPLITZ) {
    if ((s = build_psf(pl, d->traj, st))) return bail(s);
    for (int i = 0; i < pl->nlanes; ++i)
      if ((s = dev_alloc(pl, &pl->Has[i], (size_t)bf * C * N * G))) return bail(s);
  }
  {   // dynamic item hand-out in k_adj_cols when the mean spread chunk exceeds half the staging
      // buffer (the item costs then vary several-fold: stress normal -14 %; on the MRF plan, mean
      // chunk 24 KB of an 85 KB buffer, the static round-robin is 5 % faster).  MRF_ADJ_DYN=0/1 overrides.
    double mean = 0.0;
    for (const int2& ow : atab) mean += ow.y * 4.0;
    mean /= (double)atab.size();
    pl->adj_dyn = pl->ctrs && mean > 0.5 * pl->ac_stage;
    if (const char* e = std::getenv("MRF_ADJ_DYN")) pl->adj_dyn = pl->ctrs && e[0] == '1';
    // The 16-warp variant of the kernel (two threads per stage-2 transform, k_adj_cols<.., T2>) is
    // an option only (MRF_ADJ_T2=1): it gained 2.7 % on stress before the direct path's remainder
    // loads were batched and nothing after (65.0 vs 64.9 ms), and loses 14 % on MRF, whose items are
    // bound by the FFT's shared-memory traffic (adjoint 0.920 -> 1.049 ms).
    if (pl->adj_dyn || pl->adj_t2) {
      auto k = [&]() { DISPATCH_G(pl, adj_cols_attr, pl); };
      if ((s = k())) return bail(s);
    }
  }
  if (std::getenv("MRF_PLAN_STATS")) {   // chunk size distribution (bytes) against the staging buffers
    std::vector<int> a, f;
    for (const int2& ow : atab) a.push_back(ow.y * 4);
    for (const int2& ow : ftab) f.push_back(ow.y * 4);
    std::sort(a.begin(), a.end());
    std::sort(f.begin(), f.end());
    auto q = [](const std::vector<int>& v, double p) { return v[(size_t)(p * (v.size() - 1))]; };
    double sa = 0, sf = 0;
    for (int v : a) sa += v;
    for (int v : f) sf += v;
    std::fprintf(stderr, "[plan] adj chunks: mean %.0f p50 %d p90 %d max %d (stage %d) | fwd chunks: mean %.0f p90 %d max %d (stage %d)\n",
                 sa / a.size(), q(a, 0.5), q(a, 0.9), a.back(), pl->ac_stage, sf / f.size(), q(f, 0.9), f.back(), pl->fc_stage);
  }
  for (const int2& ow : atab)   // the spread kernel needs every chunk's header, slices and cells staged
    if ((size_t)ach[ow.x + 2] * 4 > (size_t)pl->ac_stage)
      return bail(fail(MRF_EUNSUPPORTED, "a grid strip has too many occupied cells for the staging buffer"));
  auto up = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  };
  cudaError_t ce = cudaSuccess;
  if (!ce) ce = up(pl->dap, dap.data(), dap.size() * sizeof(float));
  if (!ce) ce = up(pl->tw, tw.data(), tw.size() * sizeof(float2));
  if (!ce) ce = up(pl->fchunks, fch.data(), fch.size() * sizeof(int));
  if (!ce) ce = up(pl->ftab, ftab.data(), ftab.size() * sizeof(int2));
  if (!ce) ce = up(pl->achunks, ach.data(), ach.size() * sizeof(int));
  if (!ce) ce = up(pl->atab, atab.data(), atab.size() * sizeof(int2));
  if (!ce) ce = up(pl->fil, fil.data(), fil.size() * sizeof(int));
  std::vector<int> perm(L);   // (lives until the uploads below have completed)
  if (!ce) {   // column passes: each batch's frames in interleaf order (shared plan tables read from L2)
    for (int l0 = 0; l0 < L; l0 += bf) {
      const int nb = std::min(bf, L - l0);
      std::vector<int> ord(nb);
      for (int i = 0; i < nb; ++i) ord[i] = i;
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return fil[l0 + a] < fil[l0 + b]; });
      for (int i = 0; i < nb; ++i) perm[l0 + i] = ord[i];
    }
    if (std::getenv("MRF_NO_PERM") == nullptr) {
      if (cudaMalloc((void**)&pl->perm, (size_t)L * sizeof(int)) != cudaSuccess) ce = cudaErrorMemoryAllocation;
      else ce = up(pl->perm, perm.data(), perm.size() * sizeof(int));
    }
  }
  if (!ce && pl->coils) ce = up(pl->coils, d->coils, (size_t)C * N * N * sizeof(float2));
  if (!ce && (pl->flags & MRF_DCF)) {
    std::vector<double> wr((size_t)M);
    pl->dcf_host.resize((size_t)R * M);
    for (int r = 0; r < R; ++r) {
      pipe_menon(kb, G, W, d->traj + (size_t)r * M * 2, M, wr.data());
      for (int j = 0; j < M; ++j) pl->dcf_host[(size_t)r * M + j] = (float)wr[j];
    }
    if ((s = dev_alloc(pl, &pl->dcf, (size_t)R * M))) return bail(s);
    ce = up(pl->dcf, pl->dcf_host.data(), pl->dcf_host.size() * sizeof(float));
  }
  if (!ce) ce = cudaMemsetAsync(pl->sc, 0, sizeof(CGScalars), st);
  if (!ce) ce = cudaStreamSynchronize(st);
  if (ce) {
    free_plan(pl);
    return fail(MRF_ECUDA, std::string("plan upload: ") + cudaGetErrorString(ce));
  }
  *out = pl;
  return MRF_OK;
}

mrf_status mrf_plan_destroy(mrf_plan pl) {
  if (!pl) return fail(MRF_EINVAL, "null plan");
  DeviceGuard guard(pl->device);
  cudaDeviceSynchronize();
  free_plan(pl);
  return MRF_OK;
}

size_t mrf_plan_device_bytes(mrf_plan pl) { return pl ? pl->bytes : 0; }

mrf_status mrf_forward(mrf_plan pl, const void* x, void* y, void* stream) {
  if (!pl || !x || !y) return fail(MRF_EINVAL, "null plan/x/y");
  DeviceGuard guard(pl->device);
  cudaStream_t st = (cudaStream_t)stream;
  bool host = false;
  MRF_TRY(classify(pl, {x, y}, &host));
  if (!host) return do_forward(pl, (const float2*)x, (float2*)y, st);
  MRF_TRY(ensure_staging(pl, false));
  const size_t bx = (size_t)pl->L * pl->N * pl->N * sizeof(float2), by = (size_t)pl->L * pl->C * pl->M * sizeof(float2);
  CUDA_TRY(cudaMemcpyAsync(pl->stg_x, x, bx, cudaMemcpyHostToDevice, st));
  MRF_TRY(do_forward(pl, pl->stg_x, pl->stg_y, st));
  CUDA_TRY(cudaMemcpyAsync(y, pl->stg_y, by, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MRF_OK;
}

mrf_status mrf_adjoint(mrf_plan pl, const void* y, void* x, void* stream) {
  if (!pl || !x || !y) return fail(MRF_EINVAL, "null plan/x/y");
  DeviceGuard guard(pl->device);
  cudaStream_t st = (cudaStream_t)stream;
  bool host = false;
  MRF_TRY(classify(pl, {x, y}, &host));
  if (!host) return do_adjoint(pl, (const float2*)y, (float2*)x, st);
  MRF_TRY(ensure_staging(pl, false));
  const size_t bx = (size_t)pl->L * pl->N * pl->N * sizeof(float2), by = (size_t)pl->L * pl->C * pl->M * sizeof(float2);
  CUDA_TRY(cudaMemcpyAsync(pl->stg_y, y, by, cudaMemcpyHostToDevice, st));
  MRF_TRY(do_adjoint(pl, pl->stg_y, pl->stg_x, st));
  CUDA_TRY(cudaMemcpyAsync(x, pl->stg_x, bx, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MRF_OK;
}

mrf_status mrf_adjoint_dcf(mrf_plan pl, const void* y, void* x, void* stream) {
  if (!pl || !x || !y) return fail(MRF_EINVAL, "null plan/x/y");
  if (!pl->dcf) return fail(MRF_EINVAL, "the plan was created without MRF_DCF");
  DeviceGuard guard(pl->device);
  cudaStream_t st = (cudaStream_t)stream;
  bool host = false;
  MRF_TRY(classify(pl, {x, y}, &host));
  const size_t ny = (size_t)pl->L * pl->C * pl->M;
  if (!pl->ydcf) MRF_TRY(dev_alloc(pl, &pl->ydcf, ny));
  const float2* src = (const float2*)y;
  if (host) {
    MRF_TRY(ensure_staging(pl, false));
    CUDA_TRY(cudaMemcpyAsync(pl->stg_y, y, ny * sizeof(float2), cudaMemcpyHostToDevice, st));
    src = pl->stg_y;
  }
  {
    ProfScope ps(pl, MRF_K_OTHER, st);
    k_dcf_scale<<<(unsigned)std::min<size_t>((ny + 255) / 256, 4096), 256, 0, st>>>(pl->ydcf, src, pl->dcf, pl->fil,
                                                                                     pl->L, pl->C, pl->M);
    MRF_TRY(check_launch("k_dcf_scale"));
  }
  if (!host) return do_adjoint(pl, pl->ydcf, (float2*)x, st);
  MRF_TRY(do_adjoint(pl, pl->ydcf, pl->stg_x, st));
  CUDA_TRY(cudaMemcpyAsync(x, pl->stg_x, (size_t)pl->L * pl->N * pl->N * sizeof(float2), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MRF_OK;
}

mrf_status mrf_dcf_weights(mrf_plan pl, float* w) {
  if (!pl || !w) return fail(MRF_EINVAL, "null plan/w");
  if (pl->dcf_host.empty()) return fail(MRF_EINVAL, "the plan was created without MRF_DCF");
  std::memcpy(w, pl->dcf_host.data(), pl->dcf_host.size() * sizeof(float));
  return MRF_OK;
}

mrf_status mrf_normal(mrf_plan pl, const void* x, void* out, float mu, void* stream) {
  if (!pl || !x || !out) return fail(MRF_EINVAL, "null plan/x/out");
  if (x == out) return fail(MRF_EINVAL, "out may not alias x");
  if (!(mu >= 0.f) || !std::isfinite(mu)) return fail(MRF_EINVAL, "mu must be finite and >= 0");
  DeviceGuard guard(pl->device);
  cudaStream_t st = (cudaStream_t)stream;
  bool host = false;
  MRF_TRY(classify(pl, {x, out}, &host));
  if (!host) return do_normal(pl, (const float2*)x, (float2*)out, mu, st);
  MRF_TRY(ensure_staging(pl, false));
  const size_t bx = (size_t)pl->L * pl->N * pl->N * sizeof(float2);
  CUDA_TRY(cudaMemcpyAsync(pl->stg_x, x, bx, cudaMemcpyHostToDevice, st));
  MRF_TRY(do_normal(pl, pl->stg_x, pl->stg_y, mu, st));
  CUDA_TRY(cudaMemcpyAsync(out, pl->stg_y, bx, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return MRF_OK;
}

mrf_status mrf_dc_cg(mrf_plan pl, const void* y, const void* z, float mu, int n_iter, float tol, void* x,
                     mrf_cg_info* info, void* stream) {
  return mrf_dc_cg_ex(pl, y, z, mu, n_iter, tol, 0u, x, info, stream);
}

mrf_status mrf_dc_cg_ex(mrf_plan pl, const void* y, const void* z, float mu, int n_iter, float tol, unsigned flags,
                        void* x, mrf_cg_info* info, void* stream) {
  if (!pl || !y || !x) return fail(MRF_EINVAL, "null plan/y/x");
  if (flags & ~(MRF_CG_ZERO_INIT | MRF_CG_ASYNC_HOST | MRF_CG_PRECOND)) return fail(MRF_EINVAL, "unknown CG flags");
  const bool zero_init = (flags & MRF_CG_ZERO_INIT) != 0, async = (flags & MRF_CG_ASYNC_HOST) != 0;
  const bool pc = (flags & MRF_CG_PRECOND) != 0;
  if (!(mu >= 0.f) || !std::isfinite(mu)) return fail(MRF_EINVAL, "mu must be finite and >= 0");
  if (n_iter < 0) return fail(MRF_EINVAL, "n_iter < 0");
  if (!(tol >= 0.f) || !std::isfinite(tol)) return fail(MRF_EINVAL, "tol must be finite and >= 0");
  DeviceGuard guard(pl->device);
  cudaStream_t st = (cudaStream_t)stream;
  bool host = false;
  MRF_TRY(classify(pl, {y, z, x}, &host));
  if (!host) {
    if (async) return fail(MRF_EINVAL, "MRF_CG_ASYNC_HOST needs host buffers");
    return run_cg(pl, (const float2*)y, (const float2*)z, mu, n_iter, tol, (float2*)x, info, st, zero_init, pc);
  }
  const size_t bx = (size_t)pl->L * pl->N * pl->N * sizeof(float2), by = (size_t)pl->L * pl->C * pl->M * sizeof(float2);
  if (async) {
    // slot s = call parity: wait until the result copy of the call before last (same slot) has
    // left the device buffer, copy the inputs in and solve on `stream`, then copy the result out
    // on the plan's copy stream -- overlapping the next call's solve.  No host synchronisation
    // except the one that fills `info`.
    MRF_TRY(ensure_async(pl, z != nullptr));
    const int s = (int)(pl->acalls++ & 1);
    CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_copied[s], 0));
    CUDA_TRY(cudaMemcpyAsync(pl->ay[s], y, by, cudaMemcpyHostToDevice, st));
    if (!zero_init) CUDA_TRY(cudaMemcpyAsync(pl->ax[s], x, bx, cudaMemcpyHostToDevice, st));
    if (z) CUDA_TRY(cudaMemcpyAsync(pl->stg_z, z, bx, cudaMemcpyHostToDevice, st));
    mrf_status r = run_cg(pl, pl->ay[s], z ? pl->stg_z : nullptr, mu, n_iter, tol, pl->ax[s], info, st, zero_init, pc);
    if (r != MRF_OK && r != MRF_ENUMERIC) return r;
    CUDA_TRY(cudaEventRecord(pl->ev_solved[s], st));
    CUDA_TRY(cudaStreamWaitEvent(pl->cstream, pl->ev_solved[s], 0));
    CUDA_TRY(cudaMemcpyAsync(x, pl->ax[s], bx, cudaMemcpyDeviceToHost, pl->cstream));
    CUDA_TRY(cudaEventRecord(pl->ev_copied[s], pl->cstream));
    return r;
  }
  MRF_TRY(ensure_staging(pl, z != nullptr));
  CUDA_TRY(cudaMemcpyAsync(pl->stg_y, y, by, cudaMemcpyHostToDevice, st));
  if (!zero_init) CUDA_TRY(cudaMemcpyAsync(pl->stg_x, x, bx, cudaMemcpyHostToDevice, st));
  if (z) CUDA_TRY(cudaMemcpyAsync(pl->stg_z, z, bx, cudaMemcpyHostToDevice, st));
  mrf_status s = run_cg(pl, pl->stg_y, z ? pl->stg_z : nullptr, mu, n_iter, tol, pl->stg_x, info, st, zero_init, pc);
  if (s != MRF_OK && s != MRF_ENUMERIC) return s;
  CUDA_TRY(cudaMemcpyAsync(x, pl->stg_x, bx, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return s;
}

mrf_status mrf_plan_wait(mrf_plan pl) {
  if (!pl) return fail(MRF_EINVAL, "null plan");
  DeviceGuard guard(pl->device);
  if (pl->cstream) CUDA_TRY(cudaStreamSynchronize(pl->cstream));
  return MRF_OK;
}

mrf_status mrf_profile_enable(mrf_plan pl, int enable) {
  if (!pl) return fail(MRF_EINVAL, "null plan");
  pl->prof.on = enable != 0;
  for (int k = 0; k < MRF_K_COUNT; ++k) {
    pl->prof.used[k] = 0;
    pl->prof.launches[k] = 0;
  }
  return MRF_OK;
}

mrf_status mrf_profile_query(mrf_plan pl, int cls, double* total_ms, long long* launches) {
  if (!pl || cls < 0 || cls >= MRF_K_COUNT) return fail(MRF_EINVAL, "bad plan or kernel class");
  DeviceGuard guard(pl->device);
  double tot = 0.0;
  Prof& pr = pl->prof;
  for (size_t i = 0; i + 1 < pr.used[cls]; i += 2) {
    CUDA_TRY(cudaEventSynchronize(pr.ev[cls][i + 1]));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, pr.ev[cls][i], pr.ev[cls][i + 1]));
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = (long long)(pr.used[cls] / 2);
  return MRF_OK;
}

mrf_status mrf_plan_debug_halfgrid(mrf_plan pl, void* dst, size_t bytes) {
  if (!pl || !dst) return fail(MRF_EINVAL, "null plan/dst");
  const size_t need = (size_t)pl->bf * pl->C * pl->N * pl->G * sizeof(float2);
  if (bytes != need) return fail(MRF_EINVAL, "bytes must be batch_frames * C * N * G * 8");
  DeviceGuard guard(pl->device);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(dst, pl->Hs[0], need, cudaMemcpyDefault));
  return MRF_OK;
}

mrf_status mrf_plan_set_precond_shift(mrf_plan pl, double shift) {
  if (!pl) return fail(MRF_EINVAL, "null plan");
  if (!(shift >= 0.0) || !std::isfinite(shift)) return fail(MRF_EINVAL, "shift must be finite and >= 0");
  DeviceGuard guard(pl->device);
  cudaDeviceSynchronize();   // captured PCG graphs bake gamma in
  drop_cg_graphs(pl);
  pl->pc_shift = shift;
  return MRF_OK;
}

mrf_status mrf_plan_set_host_allreduce(mrf_plan pl, mrf_host_allreduce_fn fn, void* ctx) {
  if (!pl) return fail(MRF_EINVAL, "null plan");
  pl->host_ar = fn;
  pl->host_ar_ctx = fn ? ctx : nullptr;
  return MRF_OK;
}

mrf_status mrf_nccl_get_unique_id(void* id_out) {
  if (!id_out) return fail(MRF_EINVAL, "null id");
  const char* why = nullptr;
  const NcclApi* api = nccl_api(&why);
  if (!api) return fail(MRF_ENCCL, why);
  NcclUniqueId id;
  const int rc = api->GetUniqueId(&id);
  if (rc != 0) return fail(MRF_ENCCL, std::string("ncclGetUniqueId: ") + api->GetErrorString(rc));
  std::memcpy(id_out, &id, sizeof(id));
  return MRF_OK;
}

mrf_status mrf_nccl_comm_init(void** comm_out, int nranks, const void* id128, int rank, int device) {
  if (!comm_out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return fail(MRF_EINVAL, "bad comm args");
  const char* why = nullptr;
  const NcclApi* api = nccl_api(&why);
  if (!api) return fail(MRF_ENCCL, why);
  DeviceGuard guard(device);
  cudaSetDevice(device);
  NcclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  NcclComm comm = nullptr;
  const int rc = api->CommInitRank(&comm, nranks, id, rank);
  if (rc != 0) return fail(MRF_ENCCL, std::string("ncclCommInitRank: ") + api->GetErrorString(rc));
  *comm_out = comm;
  return MRF_OK;
}

mrf_status mrf_nccl_comm_destroy(void* comm) {
  if (!comm) return fail(MRF_EINVAL, "null comm");
  const char* why = nullptr;
  const NcclApi* api = nccl_api(&why);
  if (!api) return fail(MRF_ENCCL, why);
  const int rc = api->CommDestroy(comm);
  if (rc != 0) return fail(MRF_ENCCL, std::string("ncclCommDestroy: ") + api->GetErrorString(rc));
  return MRF_OK;
}

}  // extern "C"

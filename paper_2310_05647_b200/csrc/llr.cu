// llr.cu -- host side of the MS-LLR outer step and of Algorithm 1 (
// PAPER.md:130-180 Eqs. (7)-(11), 217-264 Eqs. (15), (17), (20), (21), 266-298 Algorithm 1):
// mrf_llr_create / _laplacian / _step / _cost / _destroy and mrf_msllr_solve of include/mrfnufft.h.
// Kernels in llr.cuh (coefficients, SVT, update, manifold term), gemm3.cuh (the tf32 x 3
// tensor-core GEMM G = W Q) and gridding.cuh (the subspace normal k_sn_*); the subspace basis and
// the basis-coordinate dictionary come from dict.cu (mrf_dict_basis).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/mrfnufft.h"
#include "dict_internal.h"
#include "gemm3.cuh"
#include "llr.cuh"
#include "status.h"

using namespace mrf;

static constexpr int kStatBlocks = 4 * 148;   // blocks of the grid-stride reductions

struct mrf_llr_s {
  int N = 0, L = 0, p = 0, s = 0, r = 0, nc = 0, device = 0;
  // frame sharding (mrf_llr_create_shard): this operator owns frames [frame0, frame0 + L) of Lg;
  // comm = the plan of the last call when it reduces over ranks (NCCL communicator or host
  // hook; the coefficient partials are all-reduced through it), else nullptr
  int frame0 = 0, Lg = 0;
  mrf_plan comm = nullptr;
  unsigned opts = 0;   // mrf_llr_set_options: printed-form switches (readings 21, 25, 26)
  float2* dT = nullptr;       // [L][R] transposed basis, rows zero-padded to R = 16 or 32
  int* corners = nullptr;     // [nc]
  float2* Y = nullptr;        // [N*N][r] coefficients of Z
  float2* P = nullptr;        // [nc*nc][p*p][r] thresholded patch coefficients
  float2* nx = nullptr;       // [L][N][N] A^H A x
  double* nuc = nullptr;      // [nc*nc] per-patch nuclear norms
  std::vector<double> nuc_h;
  float2* yb = nullptr;       // [L][C][M] A x of mrf_llr_cost
  size_t ny = 0;
  double* part = nullptr;     // [4][kStatBlocks] partial sums
  double* hsum = nullptr;     // pinned host staging of deferred sums (Sums)
  size_t hsum_cap = 0;
  float2 *rhs = nullptr, *x2 = nullptr;   // mrf_msllr_solve: A^H b and the second iterate buffer
  float2 *xcv = nullptr, *xcr = nullptr;  // coefficients of the last x_out: [V][r] and [r][V]
  unsigned basis_gen = 0;                 // the dictionary's basis generation at creation
  std::vector<float2> basis_h;            // host [r][L] copy of the basis
  // basis-coordinate loop on Toeplitz plans (mrf_msllr_solve): mixing kernels [r][r][G*G], the
  // spectra workspaces [r][C][G*G], zs = P_S A^H A x and bv = P_S A^H b coefficients
  float2 *Ksn = nullptr, *spa = nullptr, *spb = nullptr, *zs = nullptr, *bv = nullptr;
  size_t sn_bytes = 0;
  cudaStream_t side = nullptr;            // second stream: the cost's SVT overlaps its subspace normal
  cudaStream_t side2 = nullptr;           // third stream: the next maps and Laplacian overlap the cost
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_step = nullptr;
  unsigned long long sn_plan = 0;         // serial of the plan the mixing kernels were built for
  // manifold term (mrf_llr_laplacian)
  bool has_lap = false;
  bool q_fresh = false;   // Qm / Qh / Ql hold Q of the current coefficients xcv (set by the solve's cost)
  // two Laplacian sets (W, deg, the tf32 split and its tensor maps); W, deg, Wh, Wl, tWh, tWl below
  // alias the current one.  A build writes the other set and switches at its end, so a step or cost
  // already enqueued on another stream keeps reading the previous Laplacian.
  int lap_cur = 0;
  float *Wset[2] = {nullptr, nullptr}, *degset[2] = {nullptr, nullptr};
  float *Whset[2] = {nullptr, nullptr}, *Wlset[2] = {nullptr, nullptr};
  CUtensorMap tWhset[2], tWlset[2];
  float* W = nullptr;         // [n][n] similarity weights (Eq. 8), first the squared distances
  float* deg = nullptr;       // [n] degrees D_ii
  float* pv = nullptr;        // [n][3 p^2] standardised patch vectors of the maps
  unsigned* hist = nullptr;   // [2][2048] radix-select histograms (+1 word: max PD bits)
  mfd::LapSel* sel = nullptr;   // device state of the Laplacian build
  mfd::LapSel* sel_h = nullptr; // pinned host copy
  double* stats = nullptr;    // [blocks][7] foreground sums, then [6] mean/std
  float2* YX = nullptr;       // [V][r] coefficients of x
  float2* Qm = nullptr;       // [n][p^2 r] patch blocks of YX
  float2* Gm = nullptr;       // [n][p^2 r] W Qm
  double* pen = nullptr;      // [n] trace-penalty terms
  // G = W Qm on the tensor cores (gemm3.cuh): tf32 hi / lo copies, K-major, row pitch nK
  int nK = 0, sms = 0;
  float *Wh = nullptr, *Wl = nullptr;   // [n][nK]
  float *Qh = nullptr, *Ql = nullptr;   // [2 p^2 r][nK] (Qm transposed)
  CUtensorMap tWh, tWl, tQh, tQl;
  CUtensorMap tQh2, tQl2;                 // the same with BN / 2-row boxes (multicast halves)
  bool g3_mc = true;                      // clusters of 2 with multicast B tiles (MRF_G3_MC=0: off)
};

static void llr_free(mrf_llr_s* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->sel_h) cudaFreeHost(h->sel_h);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->side2) cudaStreamDestroy(h->side2);
  if (h->ev_step) cudaEventDestroy(h->ev_step);
  if (h->hsum) cudaFreeHost(h->hsum);
  for (int i = 0; i < 2; ++i)
    for (void* v : {(void*)h->Wset[i], (void*)h->degset[i], (void*)h->Whset[i], (void*)h->Wlset[i]})
      if (v) cudaFree(v);
  h->W = h->deg = h->Wh = h->Wl = nullptr;   // aliases of a set
  for (void* v : {(void*)h->sel, (void*)h->dT, (void*)h->corners, (void*)h->Y, (void*)h->P, (void*)h->nx, (void*)h->nuc,
                  (void*)h->pv, (void*)h->hist, (void*)h->stats, (void*)h->YX, (void*)h->Qm,
                  (void*)h->Gm, (void*)h->pen, (void*)h->Qh, (void*)h->Ql, (void*)h->yb, (void*)h->part, (void*)h->rhs, (void*)h->x2, (void*)h->xcv, (void*)h->xcr, (void*)h->Ksn,
                  (void*)h->spa, (void*)h->spb, (void*)h->zs, (void*)h->bv})
    if (v) cudaFree(v);
  delete h;
}

static size_t svt_smem(int r) { return (llr::kSvtThreads / 32) * llr::svt_warp_bytes(r); }


// manifold-term workspaces (first use): YX, Qm, Gm, per-patch penalties, Qm^T hi / lo + tensor maps
static mrf_status manifold_ws(mrf_llr_s* h) {
  if (h->YX) return MRF_OK;
  const int V = h->N * h->N, n = h->nc * h->nc, blk = h->p * h->p * h->r;
  bool ok = cudaMalloc((void**)&h->YX, (size_t)V * h->r * sizeof(float2)) == cudaSuccess &&
            cudaMalloc((void**)&h->Qm, (size_t)n * blk * sizeof(float2)) == cudaSuccess &&
            cudaMalloc((void**)&h->Gm, (size_t)n * blk * sizeof(float2)) == cudaSuccess &&
            cudaMalloc((void**)&h->pen, (size_t)n * sizeof(double)) == cudaSuccess &&
            cudaMalloc((void**)&h->Qh, (size_t)2 * blk * h->nK * sizeof(float)) == cudaSuccess &&
            cudaMalloc((void**)&h->Ql, (size_t)2 * blk * h->nK * sizeof(float)) == cudaSuccess;
  if (!ok) return fail(MRF_ENOMEM, "manifold workspace allocation failed");
  MRF_TRY(tmap_2d(&h->tQh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h->Qh, n, 2 * blk, (uint64_t)h->nK * 4, g3::BK, g3::BN));
  MRF_TRY(tmap_2d(&h->tQl, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h->Ql, n, 2 * blk, (uint64_t)h->nK * 4, g3::BK, g3::BN));
  MRF_TRY(tmap_2d(&h->tQh2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h->Qh, n, 2 * blk, (uint64_t)h->nK * 4, g3::BK, g3::BN / 2));
  MRF_TRY(tmap_2d(&h->tQl2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h->Ql, n, 2 * blk, (uint64_t)h->nK * 4, g3::BK, g3::BN / 2));
  return MRF_OK;
}

// Qm = Q(coef) (patch blocks of the [V][r] coefficients), Gm = W Qm on the tensor cores
// reuse_q: Qm and its split already hold Q(coef) (inside mrf_msllr_solve the cost of X^n and the
// next step both need Q(X^n); only W changes between them)
static mrf_status manifold_G(mrf_llr_s* h, const float2* coef, cudaStream_t st, bool reuse_q = false) {
  const int n = h->nc * h->nc, blk = h->p * h->p * h->r;
  const int M2 = 2 * blk;   // G [n][M2] = W [n][n] Qm [n][M2]: A = W (K-major), B = Qm^T [M2][n]
  if (!reuse_q) {
    mfd::k_mfd_gather<<<n, 128, 0, st>>>(coef, h->corners, h->nc, h->N, h->p, h->r, h->Qm);
    const dim3 gs((unsigned)((M2 + 31) / 32), (unsigned)((n + 31) / 32));
    g3::k_g3_split<true><<<gs, 256, 0, st>>>(reinterpret_cast<const float*>(h->Qm), n, M2, M2, h->Qh, h->Ql, h->nK);
  }
  int mt = (n + g3::BM - 1) / g3::BM;
  const int nt = (M2 + g3::BN - 1) / g3::BN, kb = (n + g3::BK - 1) / g3::BK;
  if (h->g3_mc && mt > 1) {   // clusters of 2 CTAs sharing the B tile by multicast
    mt += mt & 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(std::min(mt / 2 * nt, h->sms / 2) * 2));
    cfg.blockDim = dim3(g3::THREADS);
    cfg.dynamicSmemBytes = g3::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, g3::k_g3_gemm<true>, h->tWh, h->tWl, h->tQh2, h->tQl2, mt, nt, kb, n, M2,
                                reinterpret_cast<float*>(h->Gm), (long long)M2));
  } else {
    g3::k_g3_gemm<false><<<std::min(mt * nt, h->sms), g3::THREADS, g3::SMEM, st>>>(
        h->tWh, h->tWl, h->tQh, h->tQl, mt, nt, kb, n, M2, reinterpret_cast<float*>(h->Gm), M2);
  }
  return check_launch("k_g3_gemm");
}

// In-place sum over the ranks of the plan's communicator (frame sharding): no-op without one.
static mrf_status allreduce(mrf_llr_s* h, void* buf, size_t n, int dtype, cudaStream_t st) {
  if (!h->comm) return MRF_OK;
  return plan_allreduce(h->comm, buf, n, dtype, st);
}

// coefficients Y = (x - mu (nx - rhs)) d^dagger and, with yx, also x d^dagger.  Frame-sharded:
// each rank's kernel sums its own frames; the [V][r] partials (6.8 MB at the MRF size, instead of
// re-sharding the 524 MB frame stack to patches) are all-reduced, so every rank holds all of Y.
static mrf_status coefs(mrf_llr_s* h, const float2* x, const float2* nx, const float2* rhs, float mu, float2* y,
                        float2* yx, cudaStream_t st) {
  const int V = h->N * h->N;
  const unsigned gv = (unsigned)((V + 31) / 32);   // 32 voxels x NG frame groups per block
  if (h->r <= 16) {
    if (yx) llr::k_llr_coef<16, true><<<gv, 32 * llr::coef_groups<16>(), 0, st>>>(x, nx, rhs, h->dT, h->r, h->L, V, mu, y, yx);
    else llr::k_llr_coef<16, false><<<gv, 32 * llr::coef_groups<16>(), 0, st>>>(x, nx, rhs, h->dT, h->r, h->L, V, mu, y, nullptr);
  } else {
    if (yx) llr::k_llr_coef<32, true><<<gv, 32 * llr::coef_groups<32>(), 0, st>>>(x, nx, rhs, h->dT, h->r, h->L, V, mu, y, yx);
    else llr::k_llr_coef<32, false><<<gv, 32 * llr::coef_groups<32>(), 0, st>>>(x, nx, rhs, h->dT, h->r, h->L, V, mu, y, nullptr);
  }
  MRF_TRY(check_launch("k_llr_coef"));
  MRF_TRY(allreduce(h, y, (size_t)V * h->r * 2, MRF_DTYPE_F32, st));
  if (yx) MRF_TRY(allreduce(h, yx, (size_t)V * h->r * 2, MRF_DTYPE_F32, st));
  return MRF_OK;
}

// per-patch SVT of the coefficient blocks of Y (nuclear norms into h->nuc, thresholded blocks into h->P)
static mrf_status svt(mrf_llr_s* h, const float2* Ysrc, float tau, cudaStream_t st) {
  const int nq = h->nc * h->nc, ppb = llr::kSvtThreads / 32;
  const bool cost = std::isinf(tau);   // singular values only (the cost): eigenvalues, no vectors
  llr::k_llr_svt<<<(unsigned)((nq + ppb - 1) / ppb), llr::kSvtThreads, svt_smem(h->r), st>>>(
      Ysrc, h->corners, h->nc, h->N, h->p, h->r, tau, nq, cost ? nullptr : h->P, h->nuc);
  return check_launch("k_llr_svt");
}

// sum of n doubles copied from the device, in index order (synchronises)
static mrf_status host_sum(const double* dev, int n, cudaStream_t st, double* out) {
  std::vector<double> v(n);
  CUDA_TRY(cudaMemcpyAsync(v.data(), dev, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  double t = 0.0;
  for (double a : v) t += a;
  *out = t;
  return MRF_OK;
}

// Deferred float64 sums: the partial arrays are copied into a pinned host buffer and summed in a
// fixed order after ONE stream synchronisation for all of them.
struct Sums {
  mrf_llr_s* h;
  cudaStream_t st;
  size_t used = 0;
  std::vector<std::pair<size_t, int>> seg;
  std::vector<double*> out;
  mrf_status add(const double* dev, int n, double* dst) {
    if (used + (size_t)n > h->hsum_cap) return fail(MRF_EINVAL, "internal: sum staging overflow");
    CUDA_TRY(cudaMemcpyAsync(h->hsum + used, dev, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, st));
    seg.emplace_back(used, n);
    out.push_back(dst);
    used += (size_t)n;
    return MRF_OK;
  }
  mrf_status finish() {
    CUDA_TRY(cudaStreamSynchronize(st));
    for (size_t i = 0; i < seg.size(); ++i) {
      double t = 0.0;
      for (int k = 0; k < seg[i].second; ++k) t += h->hsum[seg[i].first + k];
      *out[i] = t;
    }
    return MRF_OK;
  }
};

static mrf_status check_plan(mrf_llr_s* h, mrf_plan plan, const char* who) {
  int pN = 0, pL = 0, pC = 0, pdev = 0;
  plan_dims(plan, &pN, &pL, &pC, &pdev);
  if (pN != h->N || pL != h->L || pdev != h->device)
    return fail(MRF_EINVAL, std::string(who) + ": the plan's N, L or device differ from the LLR operator's");
  // a shard's basis columns are frames [frame0, frame0 + L) of the dictionary: the plan must hold
  // the same global frames, or the coefficient all-reduce would sum misaligned projections
  if (h->L != h->Lg && plan_frame_offset(plan) != h->frame0)
    return fail(MRF_EINVAL, std::string(who) + ": the plan's frame_offset differs from the shard's first frame");
  h->comm = plan_has_comm(plan) ? plan : nullptr;
  return MRF_OK;
}

extern "C" {

}  // extern "C"

static mrf_status create_impl(const float2* basis_h, int r, int L, int device, unsigned gen, int N, int p, int s,
                              mrf_llr* out) {
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  auto* h = new mrf_llr_s();
  h->N = N; h->L = L; h->Lg = L; h->p = p; h->s = s; h->r = r; h->device = device;
  std::vector<int> c;   // patch corners 0, s, 2s, ... and N - p (reading 25)
  for (int v = 0; v + p <= N; v += s) c.push_back(v);
  if (c.back() != N - p) c.push_back(N - p);
  h->nc = (int)c.size();
  const size_t V = (size_t)N * N, nq = (size_t)h->nc * h->nc;
  h->nuc_h.resize(nq);
  const int R = h->r <= 16 ? 16 : 32;
  bool ok = cudaMalloc((void**)&h->dT, (size_t)R * h->L * sizeof(float2)) == cudaSuccess &&
            cudaMalloc((void**)&h->corners, c.size() * sizeof(int)) == cudaSuccess &&
            cudaMalloc((void**)&h->Y, V * h->r * sizeof(float2)) == cudaSuccess &&
            cudaMalloc((void**)&h->P, nq * p * p * h->r * sizeof(float2)) == cudaSuccess &&
            cudaMalloc((void**)&h->nx, V * h->L * sizeof(float2)) == cudaSuccess &&
            cudaMalloc((void**)&h->nuc, nq * sizeof(double)) == cudaSuccess &&
            cudaMalloc((void**)&h->xcv, V * h->r * sizeof(float2)) == cudaSuccess &&
            cudaMalloc((void**)&h->xcr, V * h->r * sizeof(float2)) == cudaSuccess &&
            cudaMalloc((void**)&h->part, 4 * (size_t)kStatBlocks * sizeof(double)) == cudaSuccess &&
            cudaMallocHost((void**)&h->hsum, (4 * (size_t)kStatBlocks + 4 * nq) * sizeof(double)) == cudaSuccess;
  h->hsum_cap = 4 * (size_t)kStatBlocks + 4 * nq;
  h->basis_gen = gen;
  h->basis_h.assign(basis_h, basis_h + (size_t)r * L);
  if (!ok) {
    llr_free(h);
    return fail(MRF_ENOMEM, "mrf_llr_create: device allocation failed");
  }
  std::vector<float2> dT((size_t)R * h->L, make_float2(0.f, 0.f));   // [L][R] from the [r][L] rows
  for (int i = 0; i < h->r; ++i)
    for (int l = 0; l < h->L; ++l) dT[(size_t)l * R + i] = basis_h[(size_t)i * h->L + l];
  cudaError_t e = cudaMemcpy(h->dT, dT.data(), dT.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(h->corners, c.data(), c.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(llr::k_llr_svt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)svt_smem(h->r));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(g3::k_g3_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g3::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(g3::k_g3_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g3::SMEM);
  if (const char* mc = std::getenv("MRF_G3_MC")) h->g3_mc = std::atoi(mc) != 0;
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->side2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_step, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    llr_free(h);
    return fail(MRF_ECUDA, std::string("mrf_llr_create: ") + cudaGetErrorString(e));
  }
  *out = h;
  return MRF_OK;
}

extern "C" {

mrf_status mrf_llr_create(mrf_dict dict, int N, int p, int s, mrf_llr* out) {
  if (!dict || !out || N < 2 || p < 1 || p > N || s < 1 || p * p > 1024)
    return fail(MRF_EINVAL, "mrf_llr_create: invalid arguments");
  if (!dict->rank) return fail(MRF_EINVAL, "mrf_llr_create: the dictionary has no basis (call mrf_dict_basis)");
  return create_impl(dict->basis_h.data(), dict->rank, dict->L, dict->device, dict->basis_gen, N, p, s, out);
}

mrf_status mrf_llr_create_shard(mrf_dict dict, int frame0, int L_local, int N, int p, int s, mrf_llr* out) {
  if (!dict || !out || N < 2 || p < 1 || p > N || s < 1 || p * p > 1024)
    return fail(MRF_EINVAL, "mrf_llr_create_shard: invalid arguments");
  if (!dict->rank) return fail(MRF_EINVAL, "mrf_llr_create_shard: the dictionary has no basis (call mrf_dict_basis)");
  if (frame0 < 0 || L_local < 1 || frame0 + L_local > dict->L)
    return fail(MRF_EINVAL, "mrf_llr_create_shard: frames [frame0, frame0 + L_local) must lie in [0, L)");
  const int r = dict->rank, L = dict->L;
  std::vector<float2> cols((size_t)r * L_local);   // the shard's columns of the global basis
  for (int i = 0; i < r; ++i)
    std::memcpy(&cols[(size_t)i * L_local], &dict->basis_h[(size_t)i * L + frame0], (size_t)L_local * sizeof(float2));
  MRF_TRY(create_impl(cols.data(), r, L_local, dict->device, dict->basis_gen, N, p, s, out));
  (*out)->frame0 = frame0;
  (*out)->Lg = L;
  return MRF_OK;
}

mrf_status mrf_llr_create_basis(const void* basis, int r, int L, int N, int p, int s, int device, mrf_llr* out) {
  if (!basis || !out || r < 1 || r > llr::RMAX || L < 1 || N < 2 || p < 1 || p > N || s < 1 || p * p > 1024)
    return fail(MRF_EINVAL, "mrf_llr_create_basis: invalid arguments");
  // a caller-supplied basis never equals a dictionary's basis generation: Phi_D inside
  // mrf_msllr_solve then runs on frames
  return create_impl(reinterpret_cast<const float2*>(basis), r, L, device, ~0u, N, p, s, out);
}


mrf_status mrf_llr_laplacian(mrf_llr h, const float* params, const float* pd, double sigma2, double* sigma2_out,
                             double* max_degree, void* stream) {
  if (!h || !params || !pd) return fail(MRF_EINVAL, "mrf_llr_laplacian: null argument");
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int n = h->nc * h->nc, np = h->p * h->p, V = h->N * h->N;
  if (!h->Wset[0]) {
    bool ok = true;
    for (int i = 0; i < 2; ++i)
      ok = ok && cudaMalloc((void**)&h->Wset[i], (size_t)n * n * sizeof(float)) == cudaSuccess &&
           cudaMalloc((void**)&h->degset[i], (size_t)n * sizeof(float)) == cudaSuccess;
    ok = ok && cudaMalloc((void**)&h->pv, (size_t)n * 3 * np * sizeof(float)) == cudaSuccess &&
              cudaMalloc((void**)&h->hist, (3 * 2048 + 1) * sizeof(unsigned)) == cudaSuccess &&
              cudaMalloc((void**)&h->sel, sizeof(mfd::LapSel)) == cudaSuccess &&
              cudaMallocHost((void**)&h->sel_h, sizeof(mfd::LapSel)) == cudaSuccess &&
              cudaMalloc((void**)&h->stats, (size_t)kStatBlocks * 7 * sizeof(double)) == cudaSuccess;
    h->nK = (n + 3) / 4 * 4;   // 16-byte TMA row pitch
    for (int i = 0; i < 2; ++i)
      ok = ok && cudaMalloc((void**)&h->Whset[i], (size_t)n * h->nK * sizeof(float)) == cudaSuccess &&
           cudaMalloc((void**)&h->Wlset[i], (size_t)n * h->nK * sizeof(float)) == cudaSuccess;
    if (!ok) return fail(MRF_ENOMEM, "mrf_llr_laplacian: device allocation failed");
    for (int i = 0; i < 2; ++i) {
      MRF_TRY(tmap_2d(&h->tWhset[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h->Whset[i], n, n, (uint64_t)h->nK * 4, g3::BK,
                      g3::BM));
      MRF_TRY(tmap_2d(&h->tWlset[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h->Wlset[i], n, n, (uint64_t)h->nK * 4, g3::BK,
                      g3::BM));
    }
  }
  // build into the set not in use (the first build: set 0)
  const int bs = h->has_lap ? h->lap_cur ^ 1 : 0;
  float *Wb = h->Wset[bs], *degb = h->degset[bs];
  // Everything stays on the device until the final copy of the LapSel state (one synchronisation):
  // foreground statistics of (T1, T2, PD) over PD > 0.1 max PD (reading 26)
  unsigned* pdmax = h->hist + 3 * 2048;
  mfd::LapSel* sel = h->sel;
  CUDA_TRY(cudaMemsetAsync(pdmax, 0, sizeof(unsigned), st));
  mfd::k_mfd_max<<<kStatBlocks, 256, 0, st>>>(pd, V, pdmax);
  mfd::k_mfd_stats<<<kStatBlocks, 256, 0, st>>>(params, pd, V, pdmax, h->stats);
  mfd::k_mfd_stats_final<<<1, 256, 0, st>>>(h->stats, kStatBlocks, sel, (h->opts & MRF_LLR_RAW_MAPS) ? 1 : 0);
  MRF_TRY(check_launch("k_mfd_stats"));
  mfd::k_mfd_patchvec<<<n, 128, 0, st>>>(params, pd, sel, h->corners, h->nc, h->N, h->p, h->pv);
  const dim3 gd((unsigned)((n + 127) / 128), (unsigned)((n + 127) / 128));
  mfd::k_mfd_dist<<<gd, 256, 0, st>>>(h->pv, n, 3 * np, Wb);
  MRF_TRY(check_launch("k_mfd_dist"));
  // sigma^2: given, or the median of the nonzero upper-triangle distances by an exact radix select
  // (11 + 11 + 10 bits; positive floats order as their bits), the bookkeeping on the device
  const unsigned given = sigma2 > 0.0 ? 1u : 0u;
  CUDA_TRY(cudaMemcpyAsync(&sel->given, &given, sizeof(unsigned), cudaMemcpyHostToDevice, st));
  if (given) {
    CUDA_TRY(cudaMemcpyAsync(&sel->sigma2, &sigma2, sizeof(double), cudaMemcpyHostToDevice, st));
  } else {
    unsigned* h0 = h->hist;
    unsigned* h1 = h->hist + 2048;
    const unsigned hb = 2 * 148;
    CUDA_TRY(cudaMemsetAsync(h0, 0, 2048 * sizeof(unsigned), st));
    mfd::k_mfd_hist<<<hb, 256, 0, st>>>(Wb, n, 0, nullptr, h0, h1);
    mfd::k_mfd_select<<<1, 256, 0, st>>>(0, h0, h0, sel);
    for (int ps = 1; ps <= 2; ++ps) {
      CUDA_TRY(cudaMemsetAsync(h0, 0, 2 * 2048 * sizeof(unsigned), st));
      mfd::k_mfd_hist<<<hb, 256, 0, st>>>(Wb, n, ps, sel->pre, h0, h1);
      mfd::k_mfd_select<<<1, 256, 0, st>>>(ps, h0, h1, sel);
    }
    MRF_TRY(check_launch("k_mfd_select"));
  }
  mfd::k_mfd_weights<<<n, 256, 0, st>>>(Wb, n, &sel->sigma2, degb);
  MRF_TRY(check_launch("k_mfd_weights"));
  mfd::k_mfd_degmax<<<(unsigned)std::min((n + 255) / 256, 148), 256, 0, st>>>(degb, n, sel);
  MRF_TRY(check_launch("k_mfd_degmax"));
  const dim3 gs((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  g3::k_g3_split<false><<<gs, 256, 0, st>>>(Wb, n, n, n, h->Whset[bs], h->Wlset[bs], h->nK);
  MRF_TRY(check_launch("k_g3_split"));
  CUDA_TRY(cudaMemcpyAsync(h->sel_h, sel, sizeof(mfd::LapSel), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (!(h->sel_h->count > 0.0)) return fail(MRF_EINVAL, "mrf_llr_laplacian: no foreground voxel");
  if (sigma2_out) *sigma2_out = h->sel_h->sigma2;
  if (max_degree) {
    float md;
    std::memcpy(&md, &h->sel_h->maxdeg, 4);
    *max_degree = md;
  }
  // switch to the new set (everything that reads it is enqueued after this returns)
  h->lap_cur = bs;
  h->W = Wb;
  h->deg = degb;
  h->Wh = h->Whset[bs];
  h->Wl = h->Wlset[bs];
  h->tWh = h->tWhset[bs];
  h->tWl = h->tWlset[bs];
  h->has_lap = true;
  return MRF_OK;
}

}  // extern "C"

// xcoef (nullable): the [V][r] coefficients of x when x = xcoef d is known to lie in span(d)
// (the previous step's output inside mrf_msllr_solve); the manifold term then reads them instead
// of projecting x again.
// ax (nullable): A x already computed (the previous cost's forward inside mrf_msllr_solve), so
// A^H A x = A^H (A x) is one adjoint instead of a normal application.
static mrf_status step_impl(mrf_llr h, mrf_plan plan, const void* x, const void* rhs, float mu, float lambda1,
                            float lambda2, float beta, void* x_out, double* nuclear, double* penalty, void* stream,
                            const float2* xcoef, const float2* ax = nullptr) {
  if (!h || !plan || !x || !rhs || !x_out) return fail(MRF_EINVAL, "mrf_llr_step: null argument");
  if (!(mu > 0.f) || !(lambda1 >= 0.f) || !(lambda2 >= 0.f) || !(beta > 0.f) || !std::isfinite(mu * lambda2 * beta))
    return fail(MRF_EINVAL, "mrf_llr_step: need mu > 0, lambda1 >= 0, lambda2 >= 0, beta > 0");
  const bool manifold = lambda1 > 0.f || penalty != nullptr;
  if (manifold && !h->has_lap) return fail(MRF_EINVAL, "mrf_llr_step: lambda1 > 0 needs mrf_llr_laplacian first");
  if (x_out == x && manifold) return fail(MRF_EINVAL, "mrf_llr_step: x_out may not alias x with the manifold term");
  for (const void* v : {x, rhs, (const void*)x_out})
    if ((uintptr_t)v % 16) return fail(MRF_EINVAL, "mrf_llr_step: arrays must be 16-byte aligned");
  MRF_TRY(check_plan(h, plan, "mrf_llr_step"));
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int V = h->N * h->N, nq = h->nc * h->nc;
  // A^H A x (the plan checks that x has its shape: [L][N][N] device memory)
  if (ax) MRF_TRY(mrf_adjoint(plan, ax, h->nx, stream));
  else MRF_TRY(mrf_normal(plan, x, h->nx, 0.f, stream));
  if (manifold) MRF_TRY(manifold_ws(h));
  MRF_TRY(coefs(h, (const float2*)x, h->nx, (const float2*)rhs, mu, h->Y, manifold && !xcoef ? h->YX : nullptr, st));
  if (manifold) {   // Y -= mu lambda1 coef(Q^*(Q(P_S x) L)),  L = D - W (Eq. 15's manifold term)
    MRF_TRY(manifold_G(h, xcoef ? xcoef : h->YX, st, xcoef && h->q_fresh));
    if (lambda1 > 0.f) {
      if (h->r <= 16)
        mfd::k_mfd_apply<16><<<(unsigned)(((long long)V * h->r + 255) / 256), 256, 0, st>>>(h->Y, h->Qm, h->Gm, h->deg, h->corners, h->nc,
                                                                           h->N, h->p, h->r, mu * lambda1);
      else
        mfd::k_mfd_apply<32><<<(unsigned)(((long long)V * h->r + 255) / 256), 256, 0, st>>>(h->Y, h->Qm, h->Gm, h->deg, h->corners, h->nc,
                                                                           h->N, h->p, h->r, mu * lambda1);
      MRF_TRY(check_launch("k_mfd_apply"));
    }
    if (penalty) {
      mfd::k_mfd_penalty<<<nq, 256, 0, st>>>(h->Qm, h->Gm, h->deg, h->p * h->p * h->r, h->pen);
      MRF_TRY(check_launch("k_mfd_penalty"));
    }
  }
  MRF_TRY(svt(h, h->Y, 1.f / beta, st));
  const float gamma = mu * lambda2 * beta;
  const int lit = (h->opts & MRF_LLR_LITERAL_EQ23) ? 1 : 0;
  const unsigned gv = (unsigned)((V + 31) / 32);
  if (h->r <= 16)
    llr::k_llr_update<16><<<gv, 256, 0, st>>>(h->Y, h->P, h->corners, h->nc, h->N, h->p, h->r, h->dT, h->L, gamma,
                                              (float2*)x_out, h->xcv, h->xcr, lit);
  else
    llr::k_llr_update<32><<<gv, 256, 0, st>>>(h->Y, h->P, h->corners, h->nc, h->N, h->p, h->r, h->dT, h->L, gamma,
                                              (float2*)x_out, h->xcv, h->xcr, lit);
  MRF_TRY(check_launch("k_llr_update"));
  h->q_fresh = false;   // the coefficients moved on
  // Tr(Q(P_S x) L Q(P_S x)^H) and sum_q ||Q_q(Z)||_*: patches summed in a fixed order (synchronise)
  if (penalty || nuclear) {
    Sums sums{h, st};
    if (penalty) MRF_TRY(sums.add(h->pen, nq, penalty));
    if (nuclear) MRF_TRY(sums.add(h->nuc, nq, nuclear));
    MRF_TRY(sums.finish());
  }
  return MRF_OK;
}

// xcoef known (inside mrf_msllr_solve): the SVT runs on the side stream beside the forward, and
// `mid` (nullable) runs after every launch and before the host sums (the overlapped map update).
static mrf_status cost_impl(mrf_llr h, mrf_plan plan, const void* x, const void* b, float lambda1, float lambda2,
                            double* cost, double* terms, void* stream, const float2* xcoef,
                            const std::function<mrf_status()>& mid = nullptr) {
  if (!h || !plan || !x || !b) return fail(MRF_EINVAL, "mrf_llr_cost: null argument");
  if (!(lambda1 >= 0.f) || !(lambda2 >= 0.f)) return fail(MRF_EINVAL, "mrf_llr_cost: need lambda1, lambda2 >= 0");
  if (lambda1 > 0.f && !h->has_lap) return fail(MRF_EINVAL, "mrf_llr_cost: lambda1 > 0 needs mrf_llr_laplacian first");
  for (const void* v : {x, b})
    if ((uintptr_t)v % 16) return fail(MRF_EINVAL, "mrf_llr_cost: arrays must be 16-byte aligned");
  MRF_TRY(check_plan(h, plan, "mrf_llr_cost"));
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  int pN = 0, pL = 0, pC = 0, pdev = 0, pM = 0;
  plan_dims(plan, &pN, &pL, &pC, &pdev, &pM);
  const size_t ny = (size_t)pL * pC * pM;
  if (!h->yb || h->ny < ny) {
    if (h->yb) cudaFree(h->yb);
    h->yb = nullptr;
    if (cudaMalloc((void**)&h->yb, ny * sizeof(float2)) != cudaSuccess) return fail(MRF_ENOMEM, "mrf_llr_cost: allocation failed");
    h->ny = ny;
  }
  const int nq = h->nc * h->nc;
  if (xcoef) {   // sum_q ||Q_q(P_S x)||_* on the side stream (overlapping the forward)
    CUDA_TRY(cudaEventRecord(h->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    MRF_TRY(svt(h, xcoef, INFINITY, h->side));
    CUDA_TRY(cudaEventRecord(h->ev_join, h->side));
  }
  // 1/2 ||A x - b||^2
  MRF_TRY(mrf_forward(plan, x, h->yb, stream));
  llr::k_llr_resid<<<kStatBlocks, 256, 0, st>>>(h->yb, (const float2*)b, ny, h->part);
  MRF_TRY(check_launch("k_llr_resid"));
  MRF_TRY(allreduce(h, h->part, kStatBlocks, MRF_DTYPE_F64, st));   // the data term over all ranks' frames
  double t[3] = {0.0, 0.0, 0.0};
  Sums sums{h, st};
  MRF_TRY(sums.add(h->part, kStatBlocks, &t[0]));
  // coefficients of P_S x (k_llr_coef with mu = 0 reads x three times: x - 0 (x - x) = x), unless known
  const float2* xf = (const float2*)x;
  if (!xcoef) MRF_TRY(coefs(h, xf, xf, xf, 0.f, h->Y, nullptr, st));
  const float2* cf = xcoef ? xcoef : h->Y;
  if (h->has_lap && (lambda1 > 0.f || terms)) {   // Tr(Q(P_S x) L Q(P_S x)^H)
    MRF_TRY(manifold_ws(h));
    MRF_TRY(manifold_G(h, cf, st));
    h->q_fresh = xcoef != nullptr;
    mfd::k_mfd_penalty<<<nq, 256, 0, st>>>(h->Qm, h->Gm, h->deg, h->p * h->p * h->r, h->pen);
    MRF_TRY(check_launch("k_mfd_penalty"));
    MRF_TRY(sums.add(h->pen, nq, &t[1]));
  }
  // sum_q ||Q_q(P_S x)||_* (threshold +inf: only the singular values, no thresholded blocks)
  if (xcoef) CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join, 0));
  else MRF_TRY(svt(h, cf, INFINITY, st));
  MRF_TRY(sums.add(h->nuc, nq, &t[2]));
  if (mid) MRF_TRY(mid());
  MRF_TRY(sums.finish());
  t[0] *= 0.5;
  if (terms)
    for (int i = 0; i < 3; ++i) terms[i] = t[i];
  if (cost) *cost = t[0] + (double)lambda1 * t[1] + (double)lambda2 * t[2];
  return MRF_OK;
}

// float64 sum over a grid-stride kernel's kStatBlocks partials (fixed order; synchronises)
static mrf_status dot_re(mrf_llr_s* h, const float2* a, const float2* b, size_t n, cudaStream_t st, double* out) {
  llr::k_llr_dotre<<<kStatBlocks, 256, 0, st>>>(a, b, n, h->part);
  MRF_TRY(check_launch("k_llr_dotre"));
  return host_sum(h->part, kStatBlocks, st, out);
}

// One step of Algorithm 1 in basis coordinates (x = xcv d; zs = P_S A^H A x from the previous
// cost): Y = xcv - mu (zs - bv) [- mu lambda1 coef(Q^*(Q(x) L))], SVT, the Eq. 21 update of the
// coefficients (no frame-domain image).
static mrf_status sub_step(mrf_llr_s* h, float mu, float lambda1, float lambda2, float beta, cudaStream_t st) {
  const int V = h->N * h->N;
  llr::k_sn_grad<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(h->xcv, h->zs, h->bv, mu, h->r, V, h->Y);
  MRF_TRY(check_launch("k_sn_grad"));
  if (lambda1 > 0.f) {
    MRF_TRY(manifold_ws(h));
    MRF_TRY(manifold_G(h, h->xcv, st, h->q_fresh));
    if (h->r <= 16)
      mfd::k_mfd_apply<16><<<(unsigned)(((long long)V * h->r + 255) / 256), 256, 0, st>>>(h->Y, h->Qm, h->Gm, h->deg, h->corners, h->nc,
                                                                         h->N, h->p, h->r, mu * lambda1);
    else
      mfd::k_mfd_apply<32><<<(unsigned)(((long long)V * h->r + 255) / 256), 256, 0, st>>>(h->Y, h->Qm, h->Gm, h->deg, h->corners, h->nc,
                                                                         h->N, h->p, h->r, mu * lambda1);
    MRF_TRY(check_launch("k_mfd_apply"));
  }
  MRF_TRY(svt(h, h->Y, 1.f / beta, st));
  const float gamma = mu * lambda2 * beta;
  llr::k_llr_update_coef<<<(unsigned)(((long long)V * h->r + 255) / 256), 256, 0, st>>>(
      h->Y, h->P, h->corners, h->nc, h->N, h->p, h->r, gamma, h->xcv, h->xcr, (h->opts & MRF_LLR_LITERAL_EQ23) ? 1 : 0);
  h->q_fresh = false;   // the coefficients moved on
  return check_launch("k_llr_update_coef");
}

// cost(n) in basis coordinates: zs = P_S A^H A x (kept for the next step),
// 1/2 ||A x - b||^2 = 1/2 <x, A^H A x> - Re <x, A^H b> + 1/2 ||b||^2 = 1/2 <u, zs> - Re <u, bv> + b2 / 2,
// the trace term and the nuclear norms from the coefficients
struct SubCost {
  double uz = 0.0, ub = 0.0, tr = 0.0, nuc = 0.0;
};
static mrf_status sub_cost_launch(mrf_llr_s* h, mrf_plan plan, float lambda1, cudaStream_t st, Sums& sums,
                                  SubCost& t) {
  const size_t n = (size_t)h->N * h->N * h->r;
  // the nuclear norms (latency-bound SVT, a quarter of the warp slots) on the side stream,
  // overlapping the subspace normal and the trace term on `st`
  CUDA_TRY(cudaEventRecord(h->ev_fork, st));
  CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
  MRF_TRY(svt(h, h->xcv, INFINITY, h->side));
  CUDA_TRY(cudaEventRecord(h->ev_join, h->side));
  MRF_TRY(sn_apply(plan, h->Ksn, h->r, h->xcr, h->zs, h->spa, h->spb, st));
  llr::k_llr_dotre<<<kStatBlocks, 256, 0, st>>>(h->xcr, h->zs, n, h->part);
  llr::k_llr_dotre<<<kStatBlocks, 256, 0, st>>>(h->xcv, h->bv, n, h->part + kStatBlocks);
  MRF_TRY(check_launch("k_llr_dotre"));
  MRF_TRY(sums.add(h->part, kStatBlocks, &t.uz));
  MRF_TRY(sums.add(h->part + kStatBlocks, kStatBlocks, &t.ub));
  const int nq = h->nc * h->nc;
  if (h->has_lap && lambda1 > 0.f) {
    MRF_TRY(manifold_ws(h));
    MRF_TRY(manifold_G(h, h->xcv, st));
    h->q_fresh = true;
    mfd::k_mfd_penalty<<<nq, 256, 0, st>>>(h->Qm, h->Gm, h->deg, h->p * h->p * h->r, h->pen);
    MRF_TRY(check_launch("k_mfd_penalty"));
    MRF_TRY(sums.add(h->pen, nq, &t.tr));
  }
  CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join, 0));
  return sums.add(h->nuc, nq, &t.nuc);
}

// Subspace-normal workspaces (mixing kernels, spectra, zs, bv) sized for `plan`, and the mixing
// kernels K for the operator's basis on the plan's PSF spectra (rebuilt when the plan changes or
// `force`).
static mrf_status ensure_sn(mrf_llr_s* h, mrf_plan plan, cudaStream_t st, bool force) {
  int pN = 0, pL = 0, pC = 0, pdev = 0, pM = 0;
  plan_dims(plan, &pN, &pL, &pC, &pdev, &pM);
  const size_t E = (size_t)sn_elems(plan), r = (size_t)h->r, V = (size_t)h->N * h->N;
  const size_t need = (r * (r + 1) / 2 * E + 2 * r * pC * E + 2 * r * V) * sizeof(float2);
  if (h->sn_bytes < need) {
    for (float2** p : {&h->Ksn, &h->spa, &h->spb, &h->zs, &h->bv}) {
      if (*p) cudaFree(*p);
      *p = nullptr;
    }
    h->sn_bytes = 0;
    h->sn_plan = 0;
    if (cudaMalloc((void**)&h->Ksn, r * (r + 1) / 2 * E * sizeof(float2)) != cudaSuccess ||
        cudaMalloc((void**)&h->spa, r * pC * E * sizeof(float2)) != cudaSuccess ||
        cudaMalloc((void**)&h->spb, r * pC * E * sizeof(float2)) != cudaSuccess ||
        cudaMalloc((void**)&h->zs, r * V * sizeof(float2)) != cudaSuccess ||
        cudaMalloc((void**)&h->bv, r * V * sizeof(float2)) != cudaSuccess)
      return fail(MRF_ENOMEM, "subspace normal: workspace allocation failed");
    h->sn_bytes = need;
  }
  if (force || h->sn_plan != plan_serial(plan)) {
    MRF_TRY(sn_build(plan, h->basis_h.data(), h->r, h->Ksn, st));
    h->sn_plan = plan_serial(plan);
  }
  return MRF_OK;
}

extern "C" {

mrf_status mrf_llr_step(mrf_llr h, mrf_plan plan, const void* x, const void* rhs, float mu, float lambda1,
                        float lambda2, float beta, void* x_out, double* nuclear, double* penalty, void* stream) {
  return step_impl(h, plan, x, rhs, mu, lambda1, lambda2, beta, x_out, nuclear, penalty, stream, nullptr);
}

mrf_status mrf_llr_cost(mrf_llr h, mrf_plan plan, const void* x, const void* b, float lambda1, float lambda2,
                        double* cost, double* terms, void* stream) {
  return cost_impl(h, plan, x, b, lambda1, lambda2, cost, terms, stream, nullptr);
}

mrf_status mrf_msllr_solve(mrf_llr h, mrf_dict dict, mrf_plan plan, const void* b, const mrf_msllr_params* prm,
                           void* x, int* index, float* pd, float* params, mrf_msllr_info* info, void* stream) {
  if (!h || !dict || !plan || !b || !prm || !x || !index || !pd) return fail(MRF_EINVAL, "mrf_msllr_solve: null argument");
  if (!(prm->mu > 0.f) || !(prm->lambda1 >= 0.f) || !(prm->lambda2 >= 0.f) || !(prm->beta > 0.f) || prm->max_iter < 0)
    return fail(MRF_EINVAL, "mrf_msllr_solve: need mu > 0, lambda1 >= 0, lambda2 >= 0, beta > 0, max_iter >= 0");
  if (dict->L != h->Lg || dict->device != h->device)
    return fail(MRF_EINVAL, "mrf_msllr_solve: the dictionary's L or device differ from the LLR operator's");
  const bool manifold = prm->lambda1 > 0.f;
  if (manifold && (dict->P != 2 || !params))
    return fail(MRF_EINVAL, "mrf_msllr_solve: lambda1 > 0 needs a (T1, T2) look-up table (P = 2) and params");
  if (params && dict->P < 1) return fail(MRF_EINVAL, "mrf_msllr_solve: params given but the dictionary has no LUT");
  MRF_TRY(check_plan(h, plan, "mrf_msllr_solve"));
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const long long V = (long long)h->N * h->N;
  const size_t xbytes = (size_t)h->L * V * sizeof(float2);
  if (!h->rhs) {
    if (cudaMalloc((void**)&h->rhs, xbytes) != cudaSuccess || cudaMalloc((void**)&h->x2, xbytes) != cudaSuccess)
      return fail(MRF_ENOMEM, "mrf_msllr_solve: allocation failed");
  }
  // X^0 = A^* b, M^0 = Phi_D(X^0), L^0, lambda_1^0 max(L^0)   (Algorithm 1)
  MRF_TRY(mrf_adjoint(plan, b, h->rhs, stream));
  CUDA_TRY(cudaMemcpyAsync(x, h->rhs, xbytes, cudaMemcpyDeviceToDevice, st));
  float lam1 = 0.f;
  // after a step, x = Xc d lies in span(d) with Xc in h->xcv / h->xcr: Phi_D runs on the r
  // coefficients (mrf_dict_match_coef) when the dictionary's basis is the operator's
  const bool coef_ok = dict->basis_gen == h->basis_gen && dict->rank == h->r;
  // Toeplitz plans: from n = 2 on the loop runs in basis coordinates (the subspace normal, the
  // cost by the inner-product identity; frames only for X^0, the first step and the output)
  const bool sub = plan_toeplitz(plan) && coef_ok;
  // frame-sharded (a communicator, or a shard of the dictionary's frames): Phi_D can only run on
  // the all-reduced coefficients, so X^0 = A^* b (not in span(d)) is never matched
  if (h->comm || h->L != h->Lg) {
    if (sub) return fail(MRF_EUNSUPPORTED, "mrf_msllr_solve: frame sharding needs a gridding plan (not MRF_NORMAL_TOEPLITZ)");
    if (!coef_ok) return fail(MRF_EUNSUPPORTED, "mrf_msllr_solve: frame sharding needs the dictionary's own basis");
    if (manifold || prm->max_iter < 1)
      return fail(MRF_EUNSUPPORTED, "mrf_msllr_solve: frame sharding needs lambda1 = 0 and max_iter >= 1 (Phi_D of X^0)");
  }
  double b2 = 0.0;
  if (sub) {
    int pN = 0, pL = 0, pC = 0, pdev = 0, pM = 0;
    plan_dims(plan, &pN, &pL, &pC, &pdev, &pM);
    MRF_TRY(ensure_sn(h, plan, st, false));   // built once per plan (plan serial)
    const float2* rh = h->rhs;
    MRF_TRY(coefs(h, rh, rh, rh, 0.f, h->bv, nullptr, st));   // P_S A^H b coefficients
    const size_t ny = (size_t)pL * pC * pM;
    MRF_TRY(dot_re(h, (const float2*)b, (const float2*)b, ny, st, &b2));   // ||b||^2
  }
  bool have_coef = false;
  auto maps = [&](const void* cur, void* ms) -> mrf_status {
    const unsigned mf = (h->opts & MRF_LLR_MATCH_NORM2) ? MRF_MATCH_NORM2 : 0u;
    if (have_coef && coef_ok) return mrf_dict_match_coef_ex(dict, h->xcr, V, mf, index, pd, params, ms);
    return mrf_dict_match_ex(dict, cur, V, mf, index, pd, params, ms);
  };
  auto update_maps = [&](const void* cur, void* ms) -> mrf_status {
    MRF_TRY(maps(cur, ms));
    if (manifold) {
      double maxdeg = 0.0;
      MRF_TRY(mrf_llr_laplacian(h, params, pd, prm->sigma2, nullptr, &maxdeg, ms));
      lam1 = (float)((double)prm->lambda1 * maxdeg);   // lambda_1^n = lambda_1^0 max(L^n)
    }
    return MRF_OK;
  };
  if (manifold) MRF_TRY(update_maps(x, stream));
  void* cur = x;
  void* nxt = h->x2;
  double prev = 0.0;
  int it = 0;
  float lam1_last = lam1;   // lambda_1 of the last step (info)
  bool maps_current = manifold;
  // cost(n) only feeds the stop rule and info->cost: without either it is not evaluated (the
  // iterates do not depend on it)
  const bool monitor = prm->tol > 0.0 || (info && info->cost);
  for (int n = 1; n <= prm->max_iter; ++n) {
    // Z^n, P^n, X^n (Eqs. 15, 20, 21), then cost(n)
    // from n = 2 on, A X^{n-1} is the previous cost's forward (h->yb): A^H A X^{n-1} = A^H (h->yb)
    if (sub && have_coef) {
      MRF_TRY(sub_step(h, prm->mu, lam1, prm->lambda2, prm->beta, st));
    } else {
      MRF_TRY(step_impl(h, plan, cur, h->rhs, prm->mu, lam1, prm->lambda2, prm->beta, nxt, nullptr, nullptr, stream,
                        have_coef ? h->xcv : nullptr, have_coef && monitor ? h->yb : nullptr));
      std::swap(cur, nxt);
    }
    have_coef = true;   // k_llr_update wrote the coefficients of X^n
    lam1_last = lam1;
    it = n;
    maps_current = false;
    // basis coordinates: the next maps and Laplacian (they read X^n's coefficients, and the
    // Laplacian builds into its other set) run on a third stream while cost(n) runs here
    const bool overlap = manifold && n < prm->max_iter && (sub || monitor);
    if (overlap) {
      CUDA_TRY(cudaEventRecord(h->ev_step, st));
      CUDA_TRY(cudaStreamWaitEvent(h->side2, h->ev_step, 0));
    }
    double c = 0.0;
    if (monitor) {
      if (sub) {
        Sums sums{h, st};
        SubCost t;
        MRF_TRY(sub_cost_launch(h, plan, lam1, st, sums, t));
        if (overlap) {
          MRF_TRY(update_maps(cur, h->side2));   // synchronises side2
          maps_current = true;
        }
        MRF_TRY(sums.finish());
        c = (0.5 * t.uz - t.ub + 0.5 * b2) + (double)lam1_last * t.tr + (double)prm->lambda2 * t.nuc;
      } else {
        std::function<mrf_status()> mid;
        if (overlap)
          mid = [&]() -> mrf_status {
            MRF_TRY(update_maps(cur, h->side2));   // synchronises side2
            maps_current = true;
            return MRF_OK;
          };
        MRF_TRY(cost_impl(h, plan, cur, b, lam1, prm->lambda2, &c, nullptr, stream, h->xcv, mid));
      }
      if (info && info->cost) info->cost[n - 1] = c;
    } else if (sub) {   // no cost wanted: only the subspace normal the next step needs
      MRF_TRY(sn_apply(plan, h->Ksn, h->r, h->xcr, h->zs, h->spa, h->spb, st));
      if (overlap) {
        MRF_TRY(update_maps(cur, h->side2));
        maps_current = true;
      }
    }
    // stop rule cost(n-1) / cost(n) - 1 < tol, from n = 2 (reading 27: cost(0) is not defined);
    // with the overlap the maps of X^n are already there (they are also the output maps)
    if (n >= 2 && prm->tol > 0.0 && prev / c - 1.0 < prm->tol) break;
    prev = c;
    if (!overlap && manifold && n < prm->max_iter) {   // M^{n+1} = Phi_D(X^n), L^{n+1}, lambda_1^{n+1}
      MRF_TRY(update_maps(cur, stream));
      maps_current = true;
    }
  }
  if (!maps_current) MRF_TRY(maps(cur, stream));   // M^ = Phi_D(X^)
  if (sub && it > 1) {   // X^ = Xc d into x (k_llr_update with gamma = 0 expands its Y)
    const unsigned gv = (unsigned)((V + 31) / 32);
    if (h->r <= 16)
      llr::k_llr_update<16><<<gv, 256, 0, st>>>(h->xcv, h->P, h->corners, h->nc, h->N, h->p, h->r, h->dT, h->L, 0.f,
                                                (float2*)x, nullptr, nullptr, 0);
    else
      llr::k_llr_update<32><<<gv, 256, 0, st>>>(h->xcv, h->P, h->corners, h->nc, h->N, h->p, h->r, h->dT, h->L, 0.f,
                                                (float2*)x, nullptr, nullptr, 0);
    MRF_TRY(check_launch("k_llr_update"));
  } else if (cur != x) {
    CUDA_TRY(cudaMemcpyAsync(x, cur, xbytes, cudaMemcpyDeviceToDevice, st));
  }
  if (info) {
    info->iters = it;
    info->lambda1 = lam1_last;
  }
  return MRF_OK;
}

mrf_status mrf_llr_subspace_normal(mrf_llr h, mrf_plan plan, const void* u, void* z, void* stream) {
  if (!h || !plan || !u || !z) return fail(MRF_EINVAL, "mrf_llr_subspace_normal: null argument");
  if (u == z) return fail(MRF_EINVAL, "mrf_llr_subspace_normal: z may not alias u");
  if (!plan_toeplitz(plan)) return fail(MRF_EINVAL, "mrf_llr_subspace_normal: needs a plan with MRF_NORMAL_TOEPLITZ");
  MRF_TRY(check_plan(h, plan, "mrf_llr_subspace_normal"));
  // the mixing kernels of a shard sum over its own frames only, and z would be a rank-local
  // partial: the subspace normal is defined for the whole frame stack
  if (h->comm || h->L != h->Lg)
    return fail(MRF_EUNSUPPORTED, "mrf_llr_subspace_normal: not available on a frame-sharded operator");
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  MRF_TRY(ensure_sn(h, plan, st, false));
  return sn_apply(plan, h->Ksn, h->r, (const float2*)u, (float2*)z, h->spa, h->spb, st);
}

mrf_status mrf_llr_set_options(mrf_llr h, unsigned options) {
  if (!h) return fail(MRF_EINVAL, "mrf_llr_set_options: null operator");
  if (options & ~(MRF_LLR_LITERAL_EQ23 | MRF_LLR_RAW_MAPS | MRF_LLR_MATCH_NORM2))
    return fail(MRF_EINVAL, "mrf_llr_set_options: unknown options");
  h->opts = options;
  return MRF_OK;
}

mrf_status mrf_llr_destroy(mrf_llr h) {
  llr_free(h);
  return MRF_OK;
}

}  // extern "C"

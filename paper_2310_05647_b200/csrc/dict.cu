// dict.cu -- host side of dictionary matching Phi_D (Eq. (5)):
// mrf_dict_create / mrf_dict_match / mrf_dict_profile* / mrf_dict_destroy of include/mrfnufft.h.
// The kernels are in match.cuh.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mrfnufft.h"
#include "dict_internal.h"
#include "llr.cuh"
#include "match.cuh"
#include "status.h"

using namespace mrf;

static constexpr int kKDc = 64;   // fp16 row length of the basis-coordinate dictionary (2 rank <= 64)


static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

mrf_status mrf::tmap_2d(CUtensorMap* m, CUtensorMapDataType type, const void* base, uint64_t cols, uint64_t rows,
                       uint64_t row_bytes, uint32_t box_cols, uint32_t box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(MRF_ECUDA, "cuTensorMapEncodeTiled is not available");
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, type, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MRF_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return MRF_OK;
}

// 2D fp16 tensor map over a row-major [rows][cols] array with a (64 x box_rows) 128-byte swizzled box
static mrf_status make_tmap(CUtensorMap* m, const __half* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  return tmap_2d(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, base, cols, rows, cols * sizeof(__half), (uint32_t)dm::BK,
                 box_rows);
}

static void dict_free(mrf_dict_s* d) {
  if (!d) return;
  cudaSetDevice(d->device);
  for (void* p : {(void*)d->dp, (void*)d->w2, (void*)d->n2inv, (void*)d->atoms, (void*)d->lut, (void*)d->xp,
                  (void*)d->xs, (void*)d->best, (void*)d->basis, (void*)d->dpc, (void*)d->w2c, (void*)d->Dc})
    if (p) cudaFree(p);
  delete d;
}

extern "C" {

mrf_status mrf_dict_create(const void* atoms, const float* lut, int K, int L, int P, int device, mrf_dict* out) {
  if (!atoms || !out || K < 1 || L < 1 || L > 65536 || P < 0 || (P > 0 && !lut))
    return fail(MRF_EINVAL, "mrf_dict_create: invalid arguments");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  auto* d = new mrf_dict_s();
  d->K = K; d->L = L; d->P = P; d->device = device;
  d->KD = ((2 * L + dm::BK - 1) / dm::BK) * dm::BK;
  d->NP = ((2 * K + dm::BN - 1) / dm::BN) * dm::BN;
  const float2* a = reinterpret_cast<const float2*>(atoms);
  // host packing (once per dictionary): fp16 rows 2k = (dr, di)/m_k, 2k+1 = (-di, dr)/m_k
  std::vector<__half> dp((size_t)d->NP * d->KD, __float2half(0.f));
  std::vector<float> w2(d->NP / 2, 0.f), n2inv(K, 0.f);
  for (int k = 0; k < K; ++k) {
    double n2 = 0.0, m = 0.0;
    for (int l = 0; l < L; ++l) {
      const float2 v = a[(size_t)k * L + l];
      n2 += (double)v.x * v.x + (double)v.y * v.y;
      m = std::max(m, (double)std::max(std::fabs(v.x), std::fabs(v.y)));
    }
    d->fro2 += n2;
    if (n2 <= 0.0) continue;   // zero atom: w2 = 0, never preferred over a non-zero one
    n2inv[k] = (float)(1.0 / n2);
    w2[k] = (float)(m * m / n2);
    const double im = 1.0 / m;
    __half* r0 = &dp[(size_t)(2 * k) * d->KD];
    __half* r1 = r0 + d->KD;
    for (int l = 0; l < L; ++l) {
      const float2 v = a[(size_t)k * L + l];
      r0[2 * l] = __float2half((float)(v.x * im));
      r0[2 * l + 1] = __float2half((float)(v.y * im));
      r1[2 * l] = __float2half((float)(-v.y * im));
      r1[2 * l + 1] = __float2half((float)(v.x * im));
    }
  }
  auto alloc = [&](void** p, size_t bytes) { return cudaMalloc(p, bytes) == cudaSuccess; };
  if (!alloc((void**)&d->dp, dp.size() * sizeof(__half)) || !alloc((void**)&d->w2, w2.size() * sizeof(float)) ||
      !alloc((void**)&d->n2inv, (size_t)K * sizeof(float)) || !alloc((void**)&d->atoms, (size_t)K * L * sizeof(float2)) ||
      (P > 0 && !alloc((void**)&d->lut, (size_t)K * P * sizeof(float)))) {
    dict_free(d);
    return fail(MRF_ENOMEM, "mrf_dict_create: device allocation failed");
  }
  cudaError_t e = cudaMemcpy(d->dp, dp.data(), dp.size() * sizeof(__half), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d->w2, w2.data(), w2.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d->n2inv, n2inv.data(), (size_t)K * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d->atoms, a, (size_t)K * L * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && P > 0) e = cudaMemcpy(d->lut, lut, (size_t)K * P * sizeof(float), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    dict_free(d);
    return fail(MRF_ECUDA, std::string("mrf_dict_create: ") + cudaGetErrorString(e));
  }
  mrf_status s = make_tmap(&d->tmd, d->dp, (uint64_t)d->KD, (uint64_t)d->NP, (uint32_t)dm::BN);
  if (s != MRF_OK) {
    dict_free(d);
    return s;
  }
  e = cudaFuncSetAttribute(dm::k_dict_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(dm::k_dict_gemm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::SMEM);
  if (e != cudaSuccess) {
    dict_free(d);
    return fail(MRF_ECUDA, std::string("mrf_dict_create: ") + cudaGetErrorString(e));
  }
  *out = d;
  return MRF_OK;
}

}  // extern "C"

// Phi_D of x [L][V] against packed rows (tmd, KD) with weights w2 and exact-pd atoms [K][L]:
// the frame-domain match (L = d->L) and the basis-coordinate match (L = rank, Dc).
static mrf_status match_impl(mrf_dict d, const char* who, const void* x, int L, int KD, const CUtensorMap& tmd,
                             const float* w2, const float2* atoms, long long V, int* index, float* pd, float* params,
                             void* stream) {
  if (!d || !x || !index || !pd || V < 1 || V > (1LL << 30))
    return fail(MRF_EINVAL, std::string(who) + ": invalid arguments");
  for (const void* p : {x, (const void*)index, (const void*)pd, (const void*)params})
    if (p && ((uintptr_t)p % 16) != 0) return fail(MRF_EINVAL, std::string(who) + ": arrays must be 16-byte aligned");
  CUDA_TRY(cudaSetDevice(d->device));
  cudaStream_t st = (cudaStream_t)stream;
  const long long vpad = ((V + dm::BM - 1) / dm::BM) * dm::BM;
  if (vpad > d->vcap) {   // rows of d->KD >= 64 >= KD fp16 (the basis-coordinate packing fits too)
    CUDA_TRY(cudaStreamSynchronize(st));
    if (d->xp) cudaFree(d->xp);
    if (d->xs) cudaFree(d->xs);
    if (d->best) cudaFree(d->best);
    d->xp = nullptr; d->xs = nullptr; d->best = nullptr; d->vcap = 0;
    if (cudaMalloc((void**)&d->xp, (size_t)vpad * d->KD * sizeof(__half)) != cudaSuccess ||
        cudaMalloc((void**)&d->xs, (size_t)vpad * sizeof(float)) != cudaSuccess ||
        cudaMalloc((void**)&d->best, (size_t)vpad * sizeof(unsigned long long)) != cudaSuccess)
      return fail(MRF_ENOMEM, std::string(who) + ": workspace allocation failed");
    d->vcap = vpad;
  }
  CUtensorMap tmx;
  MRF_TRY(make_tmap(&tmx, d->xp, (uint64_t)KD, (uint64_t)vpad, (uint32_t)dm::BM));
  const float2* xf = reinterpret_cast<const float2*>(x);
  if (L <= 32 && KD == 64)
    dm::k_dict_pack_short<<<(unsigned)((vpad + 255) / 256), 256, 0, st>>>(xf, L, (int)V, (int)vpad, KD, d->xp, d->xs);
  else
    dm::k_dict_pack_x<<<(unsigned)(vpad / 32), 256, 0, st>>>(xf, L, (int)V, KD, d->xp, d->xs);
  MRF_TRY(check_launch("k_dict_pack_x"));
  if (d->prof) {
    while (d->ev.size() < d->ev_used + 2) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      d->ev.push_back(e);
    }
    CUDA_TRY(cudaEventRecord(d->ev[d->ev_used], st));
  }
  const int m_tiles = (int)(vpad / dm::BM), n_tiles = d->NP / dm::BN;
  int n_sm = 148;
  CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, d->device));
  CUDA_TRY(cudaMemsetAsync(d->best, 0, (size_t)V * sizeof(unsigned long long), st));
  const unsigned grid = (unsigned)std::min(n_sm, m_tiles * n_tiles);
  if (KD / dm::BK == 1)   // short series (basis coordinates): two epilogue groups
    dm::k_dict_gemm<2><<<grid, dm::threads<2>(), dm::SMEM, st>>>(tmx, tmd, w2, m_tiles, n_tiles, 1, (int)V, d->best);
  else
    dm::k_dict_gemm<1><<<grid, dm::threads<1>(), dm::SMEM, st>>>(tmx, tmd, w2, m_tiles, n_tiles, KD / dm::BK, (int)V,
                                                                 d->best);
  MRF_TRY(check_launch("k_dict_gemm"));
  if (d->prof) {
    CUDA_TRY(cudaEventRecord(d->ev[d->ev_used + 1], st));
    d->ev_used += 2;
  }
  if (L <= 32)
    dm::k_dict_fix_short<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(xf, atoms, d->n2inv, d->lut, d->P, L, (int)V,
                                                                      d->best, index, pd, params);
  else
    dm::k_dict_fix<<<(unsigned)((V + 31) / 32), 256, 0, st>>>(xf, atoms, d->n2inv, d->lut, d->P, L, (int)V, d->best,
                                                                 index, pd, params);
  MRF_TRY(check_launch("k_dict_fix"));
  return MRF_OK;
}

extern "C" {

mrf_status mrf_dict_match(mrf_dict d, const void* x, long long V, int* index, float* pd, float* params, void* stream) {
  if (!d) return fail(MRF_EINVAL, "mrf_dict_match: null dictionary");
  return match_impl(d, "mrf_dict_match", x, d->L, d->KD, d->tmd, d->w2, d->atoms, V, index, pd, params, stream);
}

mrf_status mrf_dict_match_coef(mrf_dict d, const void* u, long long V, int* index, float* pd, float* params,
                               void* stream) {
  if (!d) return fail(MRF_EINVAL, "mrf_dict_match_coef: null dictionary");
  if (!d->rank || !d->dpc) return fail(MRF_EINVAL, "mrf_dict_match_coef: no basis (call mrf_dict_basis)");
  return match_impl(d, "mrf_dict_match_coef", u, d->rank, kKDc, d->tmdc, d->w2c, d->Dc, V, index, pd, params, stream);
}

// ---------------------------------------------------------------- subspace basis (Eq. 17, reading 24)
// Leading right singular vectors of D by subspace iteration on D^H D (GEMMs on the device,
// double accumulation; the k-column re-orthonormalisation (Gram-Schmidt twice) and the k x k
// Rayleigh-Ritz eigenproblem in float64 on the host), then the rank that keeps `energy` of ||D||_F^2.
static void host_jacobi_eig(int n, std::vector<std::complex<double>>& H, std::vector<std::complex<double>>& W,
                            std::vector<double>& lam) {
  W.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) W[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double m2 = std::norm(H[(size_t)i * n + j]);
        tot += m2;
        if (i != j) off += m2;
      }
    if (!(off > 1e-28 * tot)) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const std::complex<double> hpq = H[(size_t)p * n + q];
        const double mag = std::abs(hpq);
        if (!(mag > 1e-300)) continue;
        const double a = H[(size_t)p * n + p].real(), b = H[(size_t)q * n + q].real();
        const double kap = (a - b) / (2.0 * mag);
        const double t = (kap >= 0.0 ? 1.0 : -1.0) / (std::fabs(kap) + std::sqrt(1.0 + kap * kap));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = t * c;
        const std::complex<double> e = hpq / mag;
        for (int k = 0; k < n; ++k) {   // columns of H and W
          const std::complex<double> hp = H[(size_t)k * n + p], hq = H[(size_t)k * n + q];
          H[(size_t)k * n + p] = c * hp + sn * hq * std::conj(e);
          H[(size_t)k * n + q] = c * hq - sn * hp * e;
          const std::complex<double> wp = W[(size_t)k * n + p], wq = W[(size_t)k * n + q];
          W[(size_t)k * n + p] = c * wp + sn * wq * std::conj(e);
          W[(size_t)k * n + q] = c * wq - sn * wp * e;
        }
        for (int k = 0; k < n; ++k) {   // rows of H
          const std::complex<double> rp = H[(size_t)p * n + k], rq = H[(size_t)q * n + k];
          H[(size_t)p * n + k] = c * rp + sn * rq * e;
          H[(size_t)q * n + k] = c * rq - sn * rp * std::conj(e);
        }
      }
  }
  lam.resize(n);
  for (int i = 0; i < n; ++i) lam[i] = H[(size_t)i * n + i].real();
}

// The dictionary in basis coordinates (mrf_dict_match_coef): Dc = D d^dagger [K][r] on the device
// (k_cgemm computes conj(D) d^T with float64 accumulation), packed like the frame-domain rows with
// per-atom scales m'_k = max |Re, Im| of Dc_k and weights (m'_k / ||d_k||)^2 from the FULL norms.
static mrf_status build_coef_dict(mrf_dict d, int r) {
  const int K = d->K, L = d->L;
  for (void* p : {(void*)d->dpc, (void*)d->w2c, (void*)d->Dc})
    if (p) cudaFree(p);
  d->dpc = nullptr; d->w2c = nullptr; d->Dc = nullptr;
  if (cudaMalloc((void**)&d->Dc, (size_t)K * r * sizeof(float2)) != cudaSuccess ||
      cudaMalloc((void**)&d->dpc, (size_t)d->NP * kKDc * sizeof(__half)) != cudaSuccess ||
      cudaMalloc((void**)&d->w2c, (size_t)d->NP / 2 * sizeof(float)) != cudaSuccess)
    return fail(MRF_ENOMEM, "mrf_dict_basis: allocation failed");
  const dim3 blk(16, 16), grd((unsigned)((r + 15) / 16), (unsigned)((K + 15) / 16));
  llr::k_cgemm<<<grd, blk>>>(d->atoms, L, 1, 1, d->basis, 1, L, K, r, L, d->Dc, nullptr);   // conj(D) d^T
  MRF_TRY(check_launch("k_cgemm"));
  std::vector<float2> dc((size_t)K * r);
  CUDA_TRY(cudaMemcpy(dc.data(), d->Dc, dc.size() * sizeof(float2), cudaMemcpyDeviceToHost));
  std::vector<float> n2inv(K);
  CUDA_TRY(cudaMemcpy(n2inv.data(), d->n2inv, (size_t)K * sizeof(float), cudaMemcpyDeviceToHost));
  std::vector<__half> dp((size_t)d->NP * kKDc, __float2half(0.f));
  std::vector<float> w2(d->NP / 2, 0.f);
  for (int k = 0; k < K; ++k) {
    double m = 0.0;
    for (int i = 0; i < r; ++i) {
      float2& v = dc[(size_t)k * r + i];
      v.y = -v.y;   // Dc = conj(conj(D) d^T)
      m = std::max(m, (double)std::max(std::fabs(v.x), std::fabs(v.y)));
    }
    if (!(m > 0.0) || !(n2inv[k] > 0.f)) continue;
    w2[k] = (float)(m * m * (double)n2inv[k]);
    const double im = 1.0 / m;
    __half* r0 = &dp[(size_t)(2 * k) * kKDc];
    __half* r1 = r0 + kKDc;
    for (int i = 0; i < r; ++i) {
      const float2 v = dc[(size_t)k * r + i];
      r0[2 * i] = __float2half((float)(v.x * im));
      r0[2 * i + 1] = __float2half((float)(v.y * im));
      r1[2 * i] = __float2half((float)(-v.y * im));
      r1[2 * i + 1] = __float2half((float)(v.x * im));
    }
  }
  CUDA_TRY(cudaMemcpy(d->Dc, dc.data(), dc.size() * sizeof(float2), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d->dpc, dp.data(), dp.size() * sizeof(__half), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d->w2c, w2.data(), w2.size() * sizeof(float), cudaMemcpyHostToDevice));
  return make_tmap(&d->tmdc, d->dpc, (uint64_t)kKDc, (uint64_t)d->NP, (uint32_t)dm::BN);
}

extern "C" mrf_status mrf_dict_basis(mrf_dict d, double energy, int max_rank, int* rank_out) {
  if (!d || !rank_out || !(energy > 0.0 && energy <= 1.0) || max_rank < 1 || max_rank > llr::RMAX)
    return fail(MRF_EINVAL, "mrf_dict_basis: invalid arguments (0 < energy <= 1, 1 <= max_rank <= 32)");
  if (!(d->fro2 > 0.0)) return fail(MRF_EINVAL, "mrf_dict_basis: all-zero dictionary");
  CUDA_TRY(cudaSetDevice(d->device));
  const int K = d->K, L = d->L, k = std::min({max_rank + 16, 64, K, L});
  float2 *Q = nullptr, *B = nullptr;
  double2* S = nullptr;
  auto cleanup = [&]() {
    for (void* p : {(void*)Q, (void*)B, (void*)S})
      if (p) cudaFree(p);
  };
  if (cudaMalloc((void**)&Q, (size_t)L * k * sizeof(float2)) != cudaSuccess ||
      cudaMalloc((void**)&B, (size_t)K * k * sizeof(float2)) != cudaSuccess ||
      cudaMalloc((void**)&S, (size_t)k * k * sizeof(double2)) != cudaSuccess) {
    cleanup();
    return fail(MRF_ENOMEM, "mrf_dict_basis: workspace allocation failed");
  }
  std::vector<float2> q0((size_t)L * k);
  uint64_t st = 0x9E3779B97F4A7C15ull;   // deterministic start block (xorshift)
  for (auto& v : q0) {
    auto u = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (double)(st >> 11) / 9007199254740992.0 - 0.5; };
    v = make_float2((float)u(), (float)u());
  }
  const dim3 blk(16, 16);
  auto grid = [](int M, int N) { return dim3((unsigned)((N + 15) / 16), (unsigned)((M + 15) / 16)); };
  std::vector<double2> Sh((size_t)k * k);
  std::vector<float2> Qh((size_t)L * k);
  std::vector<std::complex<double>> Qd((size_t)L * k);
  auto orthonormalize = [&]() -> mrf_status {   // Q <- orth(Q): modified Gram-Schmidt, twice, float64 (host)
    CUDA_TRY(cudaMemcpy(Qh.data(), Q, Qh.size() * sizeof(float2), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < Qd.size(); ++i) Qd[i] = std::complex<double>(Qh[i].x, Qh[i].y);
    for (int j = 0; j < k; ++j) {
      for (int pass = 0; pass < 2; ++pass)
        for (int i = 0; i < j; ++i) {
          std::complex<double> dot = 0.0;
          for (int l = 0; l < L; ++l) dot += std::conj(Qd[(size_t)l * k + i]) * Qd[(size_t)l * k + j];
          for (int l = 0; l < L; ++l) Qd[(size_t)l * k + j] -= dot * Qd[(size_t)l * k + i];
        }
      double nrm = 0.0;
      for (int l = 0; l < L; ++l) nrm += std::norm(Qd[(size_t)l * k + j]);
      nrm = std::sqrt(nrm);
      if (!(nrm > 1e-300)) {   // numerically dependent column: restart it from a fixed vector
        for (int l = 0; l < L; ++l) Qd[(size_t)l * k + j] = (l % (j + 2) == 0) ? 1.0 : 0.0;
        --j;
        continue;
      }
      for (int l = 0; l < L; ++l) Qd[(size_t)l * k + j] /= nrm;
    }
    for (size_t i = 0; i < Qd.size(); ++i) Qh[i] = make_float2((float)Qd[i].real(), (float)Qd[i].imag());
    CUDA_TRY(cudaMemcpy(Q, Qh.data(), Qh.size() * sizeof(float2), cudaMemcpyHostToDevice));
    return MRF_OK;
  };
  mrf_status s = MRF_OK;
  if (cudaMemcpy(Q, q0.data(), q0.size() * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess) s = MRF_ECUDA;
  for (int it = 0; s == MRF_OK && it < 40; ++it) {
    llr::k_cgemm<<<grid(K, k), blk>>>(d->atoms, L, 1, 0, Q, k, 1, K, k, L, B, nullptr);      // B = D Q
    llr::k_cgemm<<<grid(L, k), blk>>>(d->atoms, 1, L, 1, B, k, 1, L, k, K, Q, nullptr);      // Q = D^H B
    s = orthonormalize();
  }
  if (s != MRF_OK) {
    cleanup();
    return s == MRF_ECUDA ? fail(MRF_ECUDA, "mrf_dict_basis: copy failed") : s;
  }
  // Rayleigh-Ritz: T = (D Q)^H (D Q) = W diag(lam) W^H
  llr::k_cgemm<<<grid(K, k), blk>>>(d->atoms, L, 1, 0, Q, k, 1, K, k, L, B, nullptr);
  llr::k_cgemm<<<grid(k, k), blk>>>(B, 1, k, 1, B, k, 1, k, k, K, nullptr, S);
  cudaError_t e = cudaMemcpy(Sh.data(), S, Sh.size() * sizeof(double2), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(Qh.data(), Q, Qh.size() * sizeof(float2), cudaMemcpyDeviceToHost);
  cleanup();
  if (e != cudaSuccess) return fail(MRF_ECUDA, std::string("mrf_dict_basis: ") + cudaGetErrorString(e));
  std::vector<std::complex<double>> T((size_t)k * k), Wv;
  for (size_t i = 0; i < T.size(); ++i) T[i] = std::complex<double>(Sh[i].x, Sh[i].y);
  std::vector<double> lam;
  host_jacobi_eig(k, T, Wv, lam);
  std::vector<int> ord(k);
  for (int i = 0; i < k; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return lam[a] > lam[b]; });
  int r = 0;
  double acc = 0.0;
  while (r < std::min(max_rank, k) && acc < energy * d->fro2) acc += lam[ord[r++]];
  // basis rows d_i = conj(Q w_i)^T  (right singular vectors as rows, P_S(x) = x d^H d)
  d->basis_h.assign((size_t)r * L, make_float2(0.f, 0.f));
  for (int i = 0; i < r; ++i)
    for (int l = 0; l < L; ++l) {
      std::complex<double> v = 0.0;
      for (int j = 0; j < k; ++j)
        v += std::complex<double>(Qh[(size_t)l * k + j].x, Qh[(size_t)l * k + j].y) * Wv[(size_t)j * k + ord[i]];
      d->basis_h[(size_t)i * L + l] = make_float2((float)v.real(), (float)-v.imag());
    }
  if (d->basis) cudaFree(d->basis);
  d->basis = nullptr;
  d->rank = 0;
  CUDA_TRY(cudaMalloc((void**)&d->basis, d->basis_h.size() * sizeof(float2)));
  CUDA_TRY(cudaMemcpy(d->basis, d->basis_h.data(), d->basis_h.size() * sizeof(float2), cudaMemcpyHostToDevice));
  MRF_TRY(build_coef_dict(d, r));
  d->rank = r;
  // process-wide generation: two dictionaries (or two bases of one) never share a value, so an
  // LLR operator recognises exactly the basis it was built from (mrf_msllr_solve's coef_ok)
  static std::atomic<unsigned> basis_counter{0};
  d->basis_gen = ++basis_counter;
  *rank_out = r;
  return MRF_OK;
}

extern "C" mrf_status mrf_dict_basis_copy(mrf_dict d, void* out) {
  if (!d || !out) return fail(MRF_EINVAL, "mrf_dict_basis_copy: null argument");
  if (!d->rank) return fail(MRF_EINVAL, "mrf_dict_basis_copy: no basis (call mrf_dict_basis)");
  std::memcpy(out, d->basis_h.data(), d->basis_h.size() * sizeof(float2));
  return MRF_OK;
}

mrf_status mrf_dict_profile(mrf_dict d, int enable) {
  if (!d) return fail(MRF_EINVAL, "mrf_dict_profile: null dictionary");
  d->prof = enable != 0;
  d->ev_used = 0;
  return MRF_OK;
}

mrf_status mrf_dict_profile_query(mrf_dict d, double* gemm_ms, long long* launches) {
  if (!d || !gemm_ms || !launches) return fail(MRF_EINVAL, "mrf_dict_profile_query: invalid arguments");
  double t = 0.0;
  for (size_t i = 0; i + 1 < d->ev_used; i += 2) {
    float ms = 0.f;
    CUDA_TRY(cudaEventSynchronize(d->ev[i + 1]));
    CUDA_TRY(cudaEventElapsedTime(&ms, d->ev[i], d->ev[i + 1]));
    t += ms;
  }
  *gemm_ms = t;
  *launches = (long long)(d->ev_used / 2);
  return MRF_OK;
}

mrf_status mrf_dict_destroy(mrf_dict d) {
  if (d)
    for (cudaEvent_t e : d->ev) cudaEventDestroy(e);
  dict_free(d);
  return MRF_OK;
}

}  // extern "C"

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
  for (void* p : {(void*)d->atoms, (void*)d->dn2, (void*)d->lut, (void*)d->phi, (void*)d->phiT, (void*)d->dpf,
                  (void*)d->w2f, (void*)d->xp, (void*)d->xs, (void*)d->xnorm, (void*)d->best, (void*)d->thr,
                  (void*)d->ncand, (void*)d->cand, (void*)d->ov, (void*)d->nov, (void*)d->xT, (void*)d->basis,
                  (void*)d->part_best, (void*)d->a64, (void*)d->beta2, (void*)d->u64,
                  (void*)d->Gd, (void*)d->Dc, (void*)d->dpc, (void*)d->w2c, (void*)d->w2f2, (void*)d->w2c2})
    if (p) cudaFree(p);
  delete d;
}

static mrf_status top_right_vectors(mrf_dict d, int k, std::vector<std::complex<double>>& rows, std::vector<double>& lam);

// The certified filter of Phi_D (match.cuh header): phi = the leading Rf <= 64 right singular
// vectors (subspace iteration, as mrf_dict_basis), a_k = phi d_k, ||r_k|| and ||a_k||_1 in float64
// on the device (k_dict_filter_atoms), the packed fp16 rows [a_hi | a_hi | a_lo] / m_k, the weights
// (m_k / ||d_k||)^2, and the bound beta on |rho~_k - rho_k| of the normalised correlation.
static mrf_status build_filter(mrf_dict d) {
  const int K = d->K, L = d->L, k = std::min({dm::RF + 16, K, L});
  std::vector<std::complex<double>> rows;
  std::vector<double> lam;
  MRF_TRY(top_right_vectors(d, k, rows, lam));
  const int Rf = std::min(dm::RF, k);
  d->Rf = Rf;
  std::vector<float2> ph((size_t)dm::RF * L, make_float2(0.f, 0.f)), phT((size_t)L * dm::RF, make_float2(0.f, 0.f));
  for (int f = 0; f < Rf; ++f)
    for (int l = 0; l < L; ++l) {
      const std::complex<double> v = rows[(size_t)f * L + l];
      ph[(size_t)f * L + l] = phT[(size_t)l * dm::RF + f] = make_float2((float)v.real(), (float)v.imag());
    }
  double2* a = nullptr;
  double *res2 = nullptr, *a1 = nullptr;
  auto cleanup = [&]() {
    for (void* p : {(void*)res2, (void*)a1})
      if (p) cudaFree(p);
  };
  if (cudaMalloc((void**)&d->phi, ph.size() * sizeof(float2)) != cudaSuccess ||
      cudaMalloc((void**)&d->phiT, phT.size() * sizeof(float2)) != cudaSuccess ||
      cudaMalloc((void**)&a, (size_t)K * dm::RF * sizeof(double2)) != cudaSuccess ||
      cudaMalloc((void**)&res2, (size_t)K * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&a1, (size_t)K * sizeof(double)) != cudaSuccess) {
    cleanup();
    if (a) cudaFree(a);
    return fail(MRF_ENOMEM, "mrf_dict_create: filter allocation failed");
  }
  d->a64 = a;   // owned by the dictionary from here on
  cudaError_t e = cudaMemcpy(d->phi, ph.data(), ph.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d->phiT, phT.data(), phT.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    dm::k_dict_filter_atoms<<<K, 256>>>(d->atoms, d->phi, L, a, res2, a1);
    e = cudaGetLastError();
  }
  std::vector<double2> ah((size_t)K * dm::RF);
  std::vector<double> r2h(K), a1h(K), dn2(K);
  if (e == cudaSuccess) e = cudaMemcpy(ah.data(), a, ah.size() * sizeof(double2), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(r2h.data(), res2, (size_t)K * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(a1h.data(), a1, (size_t)K * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(dn2.data(), d->dn2, (size_t)K * sizeof(double), cudaMemcpyDeviceToHost);
  cleanup();
  if (e != cudaSuccess) return fail(MRF_ECUDA, std::string("mrf_dict_create: filter setup: ") + cudaGetErrorString(e));
  // packed atom rows: 2k = (ar, ai) and 2k+1 = (-ai, ar) per coefficient, scaled by 1/m_k, split
  // into fp16 hi + lo: [hi | hi | lo] against the voxel rows [u_hi | u_lo | u_hi]
  std::vector<__half> dp((size_t)d->NP * dm::KF, __float2half(0.f));
  std::vector<float> w2((size_t)d->NP / 2, 0.f), w2p((size_t)d->NP / 2, 0.f);
  double bres = 0.0, ba1 = 0.0;
  for (int kk = 0; kk < K; ++kk) {
    if (!(dn2[kk] > 0.0)) continue;   // zero atom: w2 = 0, never listed
    double m = 0.0;
    for (int f = 0; f < dm::RF; ++f) m = std::max({m, std::fabs(ah[(size_t)kk * dm::RF + f].x), std::fabs(ah[(size_t)kk * dm::RF + f].y)});
    const double nd = std::sqrt(dn2[kk]);
    bres = std::max(bres, std::sqrt(std::max(r2h[kk], 0.0)) / nd);
    ba1 = std::max(ba1, a1h[kk] / nd);
    if (!(m > 0.0)) continue;         // no component in the filter space: its score is 0 (+ band)
    w2[kk] = (float)(m * m / dn2[kk]);
    w2p[kk] = (float)(m * m / (dn2[kk] * dn2[kk]));
    __half* r0 = &dp[(size_t)(2 * kk) * dm::KF];
    __half* r1 = r0 + dm::KF;
    for (int f = 0; f < dm::RF; ++f) {
      const double2 v = ah[(size_t)kk * dm::RF + f];
      double comp[4] = {v.x / m, v.y / m, -v.y / m, v.x / m};   // r0: (ar, ai), r1: (-ai, ar)
      for (int c = 0; c < 4; ++c) {
        __half hi, lo;
        hi = __double2half(comp[c]);
        lo = __double2half(comp[c] - (double)__half2float(hi));
        __half* row = c < 2 ? r0 : r1;
        const int col = 2 * f + (c & 1);
        row[col] = hi;
        row[2 * dm::RF + col] = hi;
        row[4 * dm::RF + col] = lo;
      }
    }
  }
  // beta (match.cuh): residual ||r_k|| / ||d_k|| (plus 1e-12 for its float64 evaluation) +
  // projection rounding eps_u ||a_k||_1 / ||d_k|| (eps_u = sqrt(2) gamma_{2 kProjChunk} (1 + 1e-4):
  // kProjChunk-frame fp32 chunks, ||phi_f|| <= 1 + 1e-4) + split-operand rounding 3 u16^2 + subnormal half
  // (2^-25 sqrt(2 RF) 2) + worst-case fp32 accumulation of the K = 384 products gamma_384, on both
  // components (sqrt 2), + the fp32 score arithmetic (1e-6), x 1.05.  beta2_k (the float64
  // coefficient score of the rescoring) keeps the residual and projection terms of atom k.
  const double u32 = std::ldexp(1.0, -24), u16 = std::ldexp(1.0, -11);
  const double g384 = 384.0 * u32 / (1.0 - 384.0 * u32);
  const double nfma = 2.0 * dm::kProjChunk;
  const double eps_u = std::sqrt(2.0) * (nfma * u32 / (1.0 - nfma * u32)) * (1.0 + 1e-4);
  const double gemm = std::sqrt(2.0) * ((3.0 * u16 * u16 + g384) * 1.001 + std::ldexp(1.0, -25) * std::sqrt(2.0 * dm::RF) * 2.0);
  d->beta_res = bres;
  d->beta_a1 = ba1;
  d->beta = 1.05 * ((bres + 1e-12) + eps_u * ba1 + gemm + 1e-6);
  std::vector<double> b2(K, 0.0);
  for (int kk = 0; kk < K; ++kk)
    if (dn2[kk] > 0.0)
      b2[kk] = 1.05 * (std::sqrt(std::max(r2h[kk], 0.0)) + eps_u * a1h[kk]) / std::sqrt(dn2[kk]) + 1e-12;
  if (cudaMalloc((void**)&d->beta2, (size_t)K * sizeof(double)) != cudaSuccess)
    return fail(MRF_ENOMEM, "mrf_dict_create: filter allocation failed");
  CUDA_TRY(cudaMemcpy(d->beta2, b2.data(), (size_t)K * sizeof(double), cudaMemcpyHostToDevice));
  d->dmin = 0.0;
  for (int kk = 0; kk < K; ++kk)
    if (dn2[kk] > 0.0 && (d->dmin == 0.0 || std::sqrt(dn2[kk]) < d->dmin)) d->dmin = std::sqrt(dn2[kk]);
  if (cudaMalloc((void**)&d->dpf, dp.size() * sizeof(__half)) != cudaSuccess ||
      cudaMalloc((void**)&d->w2f, w2.size() * sizeof(float)) != cudaSuccess ||
      cudaMalloc((void**)&d->w2f2, w2p.size() * sizeof(float)) != cudaSuccess)
    return fail(MRF_ENOMEM, "mrf_dict_create: filter allocation failed");
  CUDA_TRY(cudaMemcpy(d->dpf, dp.data(), dp.size() * sizeof(__half), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d->w2f, w2.data(), w2.size() * sizeof(float), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d->w2f2, w2p.data(), w2p.size() * sizeof(float), cudaMemcpyHostToDevice));
  return make_tmap(&d->tmdf, d->dpf, (uint64_t)dm::KF, (uint64_t)d->NP, (uint32_t)dm::BN);
}

extern "C" {

mrf_status mrf_dict_create(const void* atoms, const float* lut, int K, int L, int P, int device, mrf_dict* out) {
  if (!atoms || !out || K < 1 || L < 1 || L > 65536 || P < 0 || (P > 0 && !lut))
    return fail(MRF_EINVAL, "mrf_dict_create: invalid arguments");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  auto* d = new mrf_dict_s();
  d->K = K; d->L = L; d->P = P; d->device = device;
  d->NP = ((2 * K + dm::BN - 1) / dm::BN) * dm::BN;
  const float2* a = reinterpret_cast<const float2*>(atoms);
  std::vector<double> dn2(K, 0.0);
  for (int k = 0; k < K; ++k) {
    double n2 = 0.0;
    for (int l = 0; l < L; ++l) {
      const float2 v = a[(size_t)k * L + l];
      n2 += (double)v.x * v.x + (double)v.y * v.y;
    }
    dn2[k] = n2;
    d->fro2 += n2;
  }
  auto alloc = [&](void** p, size_t bytes) { return cudaMalloc(p, bytes) == cudaSuccess; };
  if (!alloc((void**)&d->atoms, (size_t)K * L * sizeof(float2)) || !alloc((void**)&d->dn2, (size_t)K * sizeof(double)) ||
      (P > 0 && !alloc((void**)&d->lut, (size_t)K * P * sizeof(float)))) {
    dict_free(d);
    return fail(MRF_ENOMEM, "mrf_dict_create: device allocation failed");
  }
  cudaError_t e = cudaMemcpy(d->atoms, a, (size_t)K * L * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d->dn2, dn2.data(), (size_t)K * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && P > 0) e = cudaMemcpy(d->lut, lut, (size_t)K * P * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(dm::k_dict_gemm<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(dm::k_dict_gemm<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(dm::k_dict_proj_frames, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::proj_smem());
  if (e != cudaSuccess) {
    dict_free(d);
    return fail(MRF_ECUDA, std::string("mrf_dict_create: ") + cudaGetErrorString(e));
  }
  if (!(d->fro2 > 0.0)) {   // all-zero dictionary: every score is 0 (no filter needed)
    *out = d;
    return MRF_OK;
  }
  mrf_status s = build_filter(d);
  if (s != MRF_OK) {
    dict_free(d);
    return s;
  }
  *out = d;
  return MRF_OK;
}

}  // extern "C"

static mrf_status grow(mrf_dict d, long long vpad, long long vt, int L, cudaStream_t st, const char* who) {
  if (vpad > d->vcap) {
    CUDA_TRY(cudaStreamSynchronize(st));
    for (void** p : {(void**)&d->xp, (void**)&d->xs, (void**)&d->xnorm, (void**)&d->best, (void**)&d->thr,
                     (void**)&d->ncand, (void**)&d->cand, (void**)&d->ov, &d->part_best, (void**)&d->u64})
      if (*p) { cudaFree(*p); *p = nullptr; }
    d->vcap = 0;
    if (cudaMalloc((void**)&d->xp, (size_t)vpad * dm::KF * sizeof(__half)) != cudaSuccess ||
        cudaMalloc((void**)&d->xs, (size_t)vpad * sizeof(float)) != cudaSuccess ||
        cudaMalloc((void**)&d->xnorm, (size_t)vpad * sizeof(double)) != cudaSuccess ||
        cudaMalloc((void**)&d->best, (size_t)vpad * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc((void**)&d->thr, (size_t)vpad * sizeof(float)) != cudaSuccess ||
        cudaMalloc((void**)&d->ncand, (size_t)vpad * sizeof(int)) != cudaSuccess ||
        cudaMalloc((void**)&d->cand, (size_t)vpad * dm::kCand * sizeof(int)) != cudaSuccess ||
        cudaMalloc((void**)&d->ov, (size_t)vpad * sizeof(int)) != cudaSuccess ||
        cudaMalloc((void**)&d->part_best, (size_t)vpad * dm::kParts * sizeof(dm::PartBest)) != cudaSuccess ||
        cudaMalloc((void**)&d->u64, (size_t)vpad * dm::RF * sizeof(double2)) != cudaSuccess)
      return fail(MRF_ENOMEM, std::string(who) + ": workspace allocation failed");
    if (!d->nov && cudaMalloc((void**)&d->nov, sizeof(int)) != cudaSuccess)
      return fail(MRF_ENOMEM, std::string(who) + ": workspace allocation failed");
    d->vcap = vpad;
  }
  if (vt > d->vtcap) {
    CUDA_TRY(cudaStreamSynchronize(st));
    if (d->xT) cudaFree(d->xT);
    d->xT = nullptr;
    d->vtcap = 0;
    if (cudaMalloc((void**)&d->xT, (size_t)vt * L * sizeof(float2)) != cudaSuccess)
      return fail(MRF_ENOMEM, std::string(who) + ": workspace allocation failed");
    d->vtcap = vt;
  }
  return MRF_OK;
}

// The two filter GEMM passes over the packed voxel rows d->xp (match.cuh steps 3): best score,
// certified band, candidate lists.
static mrf_status filter_passes(mrf_dict d, long long V, long long vpad, int kf, const CUtensorMap& tmd, const float* w2,
                                double beta, cudaStream_t st) {
  CUtensorMap tmx;
  MRF_TRY(tmap_2d(&tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, d->xp, (uint64_t)kf, (uint64_t)vpad, (uint64_t)kf * sizeof(__half),
                  (uint32_t)dm::BK, (uint32_t)dm::BM));
  const int m_tiles = (int)(vpad / dm::BM), n_tiles = d->NP / dm::BN;
  int n_sm = 148;
  CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, d->device));
  const unsigned grid = (unsigned)std::min(n_sm, m_tiles * n_tiles);
  CUDA_TRY(cudaMemsetAsync(d->best, 0, (size_t)V * sizeof(unsigned long long), st));
  if (d->prof) {
    while (d->ev.size() < d->ev_used + 2) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      d->ev.push_back(e);
    }
    CUDA_TRY(cudaEventRecord(d->ev[d->ev_used], st));
  }
  dm::k_dict_gemm<2, 0><<<grid, dm::threads<2>(), dm::SMEM, st>>>(tmx, tmd, w2, m_tiles, n_tiles, kf / dm::BK, (int)V,
                                                                  d->best, nullptr, nullptr, nullptr);
  MRF_TRY(check_launch("k_dict_gemm"));
  dm::k_dict_thr<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(d->best, d->xnorm, d->xs, beta, (int)V, d->thr, d->ncand);
  MRF_TRY(check_launch("k_dict_thr"));
  dm::k_dict_gemm<2, 1><<<grid, dm::threads<2>(), dm::SMEM, st>>>(tmx, tmd, w2, m_tiles, n_tiles, kf / dm::BK, (int)V,
                                                                  nullptr, d->thr, d->ncand, d->cand);
  MRF_TRY(check_launch("k_dict_gemm"));
  if (d->prof) {
    CUDA_TRY(cudaEventRecord(d->ev[d->ev_used + 1], st));
    d->ev_used += 2;
  }
  CUDA_TRY(cudaMemsetAsync(d->nov, 0, sizeof(int), st));
  return MRF_OK;
}

static mrf_status check_args(mrf_dict d, const char* who, const void* x, long long V, int* index, float* pd,
                             float* params) {
  if (!d || !x || !index || !pd || V < 1 || V > (1LL << 30)) return fail(MRF_EINVAL, std::string(who) + ": invalid arguments");
  for (const void* p : {x, (const void*)index, (const void*)pd, (const void*)params})
    if (p && ((uintptr_t)p % 16) != 0) return fail(MRF_EINVAL, std::string(who) + ": arrays must be 16-byte aligned");
  return MRF_OK;
}

extern "C" {

mrf_status mrf_dict_match(mrf_dict d, const void* x, long long V, int* index, float* pd, float* params, void* stream) {
  return mrf_dict_match_ex(d, x, V, 0u, index, pd, params, stream);
}

mrf_status mrf_dict_match_ex(mrf_dict d, const void* x, long long V, unsigned flags, int* index, float* pd, float* params,
                             void* stream) {
  if (flags & ~MRF_MATCH_NORM2) return fail(MRF_EINVAL, "mrf_dict_match: unknown flags");
  const int pw = (flags & MRF_MATCH_NORM2) ? 2 : 1;
  MRF_TRY(check_args(d, "mrf_dict_match", x, V, index, pd, params));
  CUDA_TRY(cudaSetDevice(d->device));
  cudaStream_t st = (cudaStream_t)stream;
  const long long vpad = ((V + dm::BM - 1) / dm::BM) * dm::BM;
  MRF_TRY(grow(d, vpad, V, d->L, st, "mrf_dict_match"));
  const float2* xf = reinterpret_cast<const float2*>(x);
  if (!d->phi) {   // all-zero dictionary: the lowest index, PD 0 (every score is 0)
    CUDA_TRY(cudaMemsetAsync(index, 0, (size_t)V * sizeof(int), st));
    CUDA_TRY(cudaMemsetAsync(pd, 0, (size_t)V * sizeof(float), st));
    if (params) CUDA_TRY(cudaMemsetAsync(params, 0, (size_t)V * d->P * sizeof(float), st));
    return MRF_OK;
  }
  CUDA_TRY(cudaMemsetAsync(d->xp + (size_t)V * dm::KF, 0, (size_t)(vpad - V) * dm::KF * sizeof(__half), st));
  dm::k_dict_proj_frames<<<(unsigned)((V + dm::PJV - 1) / dm::PJV), 256, dm::proj_smem(), st>>>(xf, d->phiT, d->L, (int)V, d->xT, d->xp, d->xs,
                                                                     d->xnorm, d->u64);
  MRF_TRY(check_launch("k_dict_proj_frames"));
  // the printed form's scores |c| / ||d||^2 carry the band beta ||d|| ||x|| / ||d||^2 <= beta ||x|| / dmin
  MRF_TRY(filter_passes(d, V, vpad, dm::KF, d->tmdf, pw == 2 ? d->w2f2 : d->w2f, pw == 2 ? d->beta / d->dmin : d->beta, st));
  dm::k_dict_rescore_frames<<<(unsigned)((V + 7) / 8), 256, 0, st>>>(d->xT, d->atoms, d->dn2, d->xnorm, d->u64, d->a64,
                                                                    d->beta2, pw, d->ncand, d->cand, d->lut, d->P, d->L, (int)V,
                                                                    index, pd, params, d->ov, d->nov);
  MRF_TRY(check_launch("k_dict_rescore_frames"));
  dm::k_dict_exact_frames<<<1184, 256, 0, st>>>(d->xT, d->atoms, d->dn2, pw, d->K, d->L, d->ov, d->nov,
                                                (dm::PartBest*)d->part_best);
  MRF_TRY(check_launch("k_dict_exact_frames"));
  dm::k_dict_exact_finish<<<64, 128, 0, st>>>(d->ov, d->nov, (const dm::PartBest*)d->part_best, d->dn2, d->lut, d->P, index, pd, params);
  return check_launch("k_dict_exact_finish");
}

mrf_status mrf_dict_match_coef(mrf_dict d, const void* u, long long V, int* index, float* pd, float* params,
                               void* stream) {
  return mrf_dict_match_coef_ex(d, u, V, 0u, index, pd, params, stream);
}

mrf_status mrf_dict_match_coef_ex(mrf_dict d, const void* u, long long V, unsigned flags, int* index, float* pd,
                                  float* params, void* stream) {
  if (flags & ~MRF_MATCH_NORM2) return fail(MRF_EINVAL, "mrf_dict_match_coef: unknown flags");
  const int pw = (flags & MRF_MATCH_NORM2) ? 2 : 1;
  MRF_TRY(check_args(d, "mrf_dict_match_coef", u, V, index, pd, params));
  if (!d->rank || !d->Dc || !d->dpc) return fail(MRF_EINVAL, "mrf_dict_match_coef: no basis (call mrf_dict_basis)");
  CUDA_TRY(cudaSetDevice(d->device));
  cudaStream_t st = (cudaStream_t)stream;
  const long long vpad = ((V + dm::BM - 1) / dm::BM) * dm::BM;
  MRF_TRY(grow(d, vpad, 0, d->L, st, "mrf_dict_match_coef"));
  const float2* w = reinterpret_cast<const float2*>(u);
  CUDA_TRY(cudaMemsetAsync(d->xp + (size_t)V * dm::KFC, 0, (size_t)(vpad - V) * dm::KFC * sizeof(__half), st));
  dm::k_dict_proj_coef<<<(unsigned)((V + 127) / 128), 128, 0, st>>>(w, d->rank, (int)V, d->Gd, d->xp, d->xs, d->xnorm);
  MRF_TRY(check_launch("k_dict_proj_coef"));
  MRF_TRY(filter_passes(d, V, vpad, dm::KFC, d->tmdc, pw == 2 ? d->w2c2 : d->w2c, pw == 2 ? d->beta_c / d->dmin : d->beta_c,
                        st));
  dm::k_dict_rescore_coef<<<(unsigned)((V + 127) / 128), 128, 0, st>>>(w, d->rank, d->Dc, d->dn2, pw, d->xnorm, d->ncand,
                                                                        d->cand, d->lut, d->P, (int)V, index, pd, params,
                                                                        d->ov, d->nov);
  MRF_TRY(check_launch("k_dict_rescore_coef"));
  dm::k_dict_exact_coef<<<64, 128, 0, st>>>(w, d->rank, d->Dc, d->dn2, pw, d->K, d->lut, d->P, (int)V, d->ov, d->nov, index,
                                            pd, params);
  return check_launch("k_dict_exact_coef");
}

mrf_status mrf_dict_overflow(mrf_dict d, int* voxels) {
  if (!d || !voxels) return fail(MRF_EINVAL, "mrf_dict_overflow: null argument");
  CUDA_TRY(cudaSetDevice(d->device));
  int n = 0;
  if (d->nov) CUDA_TRY(cudaMemcpy(&n, d->nov, sizeof(int), cudaMemcpyDeviceToHost));
  *voxels = n;
  return MRF_OK;
}

mrf_status mrf_dict_filter_info(mrf_dict d, int* rank, double* beta, double* residual) {
  if (!d) return fail(MRF_EINVAL, "mrf_dict_filter_info: null dictionary");
  if (rank) *rank = d->Rf;
  if (beta) *beta = d->beta;
  if (residual) *residual = d->beta_res;
  return MRF_OK;
}

}  // extern "C"

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

// The match in basis coordinates (mrf_dict_match_coef; x = sum_i w_i d_i for the basis rows d_i):
// Dc[k][i] = <d_i, d_k> (exact scores <d_k, x> = sum_i w_i conj(Dc[k][i])) and Gd[i][j] = <d_i, d_j>
// (||x||^2 = w^H Gd w), float64 on the device from the fp32 basis (k_cgemm, float64 accumulation),
// and the r-dimensional certified filter: rows [Dc_hi | Dc_hi | Dc_lo] / m'_k (blocks of 64 halves,
// 2r <= 64), weights (m'_k / ||d_k||)^2 with the FULL atom norms, and beta_c = split-operand
// rounding + worst-case fp32 accumulation of the K = 192 products (no residual: the identity is exact).
static mrf_status build_coef_dict(mrf_dict d, int r) {
  const int K = d->K, L = d->L;
  for (void* p : {(void*)d->Gd, (void*)d->Dc, (void*)d->dpc, (void*)d->w2c, (void*)d->w2c2})
    if (p) cudaFree(p);
  d->Gd = nullptr; d->Dc = nullptr; d->dpc = nullptr; d->w2c = nullptr; d->w2c2 = nullptr;
  if (cudaMalloc((void**)&d->Dc, (size_t)K * r * sizeof(double2)) != cudaSuccess ||
      cudaMalloc((void**)&d->Gd, (size_t)r * r * sizeof(double2)) != cudaSuccess ||
      cudaMalloc((void**)&d->dpc, (size_t)d->NP * dm::KFC * sizeof(__half)) != cudaSuccess ||
      cudaMalloc((void**)&d->w2c, (size_t)d->NP / 2 * sizeof(float)) != cudaSuccess ||
      cudaMalloc((void**)&d->w2c2, (size_t)d->NP / 2 * sizeof(float)) != cudaSuccess)
    return fail(MRF_ENOMEM, "mrf_dict_basis: allocation failed");
  const dim3 blk(16, 16);
  auto grid = [](int M, int N) { return dim3((unsigned)((N + 15) / 16), (unsigned)((M + 15) / 16)); };
  // Dc^* = conj(D) d^T, i.e. conj(Dc[k][i]) = sum_l conj(d_kl) d_il  (conjugated on the host below)
  llr::k_cgemm<<<grid(K, r), blk>>>(d->atoms, L, 1, 1, d->basis, 1, L, K, r, L, nullptr, d->Dc);
  MRF_TRY(check_launch("k_cgemm"));
  // Gd [r][r]: Gd[i][j] = sum_l conj(d_il) d_jl = <d_i, d_j>
  llr::k_cgemm<<<grid(r, r), blk>>>(d->basis, L, 1, 1, d->basis, 1, L, r, r, L, nullptr, d->Gd);
  MRF_TRY(check_launch("k_cgemm"));
  std::vector<double2> dc((size_t)K * r);
  CUDA_TRY(cudaMemcpy(dc.data(), d->Dc, dc.size() * sizeof(double2), cudaMemcpyDeviceToHost));
  for (auto& v : dc) v.y = -v.y;
  CUDA_TRY(cudaMemcpy(d->Dc, dc.data(), dc.size() * sizeof(double2), cudaMemcpyHostToDevice));
  std::vector<double> dn2(K);
  CUDA_TRY(cudaMemcpy(dn2.data(), d->dn2, (size_t)K * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<__half> dp((size_t)d->NP * dm::KFC, __float2half(0.f));
  std::vector<float> w2((size_t)d->NP / 2, 0.f), w2p((size_t)d->NP / 2, 0.f);
  for (int k = 0; k < K; ++k) {
    if (!(dn2[k] > 0.0)) continue;
    double m = 0.0;
    for (int i = 0; i < r; ++i) m = std::max({m, std::fabs(dc[(size_t)k * r + i].x), std::fabs(dc[(size_t)k * r + i].y)});
    if (!(m > 0.0)) continue;
    w2[k] = (float)(m * m / dn2[k]);
    w2p[k] = (float)(m * m / (dn2[k] * dn2[k]));
    __half* r0 = &dp[(size_t)(2 * k) * dm::KFC];
    __half* r1 = r0 + dm::KFC;
    for (int i = 0; i < r; ++i) {
      const double2 v = dc[(size_t)k * r + i];
      const double comp[4] = {v.x / m, v.y / m, -v.y / m, v.x / m};   // r0: (re, im), r1: (-im, re)
      for (int c = 0; c < 4; ++c) {
        const __half hi = __double2half(comp[c]);
        const __half lo = __double2half(comp[c] - (double)__half2float(hi));
        __half* row = c < 2 ? r0 : r1;
        const int col = 2 * i + (c & 1);
        row[col] = hi;
        row[64 + col] = hi;
        row[128 + col] = lo;
      }
    }
  }
  const double u32 = std::ldexp(1.0, -24), u16 = std::ldexp(1.0, -11);
  const double g192 = 192.0 * u32 / (1.0 - 192.0 * u32);
  // ||w|| <= ||x|| (1 + 1e-6): the basis rows are orthonormal to fp32 rounding
  d->beta_c = 1.05 * std::sqrt(2.0) * ((3.0 * u16 * u16 + g192) * 1.001 + std::ldexp(1.0, -25) * 8.0 * 2.0) + 1e-6;
  CUDA_TRY(cudaMemcpy(d->dpc, dp.data(), dp.size() * sizeof(__half), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d->w2c, w2.data(), w2.size() * sizeof(float), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d->w2c2, w2p.data(), w2p.size() * sizeof(float), cudaMemcpyHostToDevice));
  return tmap_2d(&d->tmdc, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, d->dpc, (uint64_t)dm::KFC, (uint64_t)d->NP,
                 (uint64_t)dm::KFC * sizeof(__half), (uint32_t)dm::BK, (uint32_t)dm::BN);
}

// Leading right singular vectors of D by subspace iteration on D^H D (GEMMs on the device, double
// accumulation; the k-column re-orthonormalisation (Gram-Schmidt twice) and the k x k Rayleigh-Ritz
// eigenproblem in float64 on the host).  rows [k][L]: the Ritz vectors as rows in the convention
// of the basis d (P_S(x) = x d^H d), by decreasing Ritz value lam.
static mrf_status top_right_vectors(mrf_dict d, int k, std::vector<std::complex<double>>& rows, std::vector<double>& lam_out) {
  const int K = d->K, L = d->L;
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
    return fail(MRF_ENOMEM, "subspace basis: workspace allocation failed");
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
    return s == MRF_ECUDA ? fail(MRF_ECUDA, "subspace basis: copy failed") : s;
  }
  // Rayleigh-Ritz: T = (D Q)^H (D Q) = W diag(lam) W^H
  llr::k_cgemm<<<grid(K, k), blk>>>(d->atoms, L, 1, 0, Q, k, 1, K, k, L, B, nullptr);
  llr::k_cgemm<<<grid(k, k), blk>>>(B, 1, k, 1, B, k, 1, k, k, K, nullptr, S);
  cudaError_t e = cudaMemcpy(Sh.data(), S, Sh.size() * sizeof(double2), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(Qh.data(), Q, Qh.size() * sizeof(float2), cudaMemcpyDeviceToHost);
  cleanup();
  if (e != cudaSuccess) return fail(MRF_ECUDA, std::string("subspace basis: ") + cudaGetErrorString(e));
  std::vector<std::complex<double>> T((size_t)k * k), Wv;
  for (size_t i = 0; i < T.size(); ++i) T[i] = std::complex<double>(Sh[i].x, Sh[i].y);
  std::vector<double> lam;
  host_jacobi_eig(k, T, Wv, lam);
  std::vector<int> ord(k);
  for (int i = 0; i < k; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return lam[a] > lam[b]; });
  rows.assign((size_t)k * L, 0.0);
  lam_out.resize(k);
  for (int i = 0; i < k; ++i) {
    lam_out[i] = lam[ord[i]];
    for (int l = 0; l < L; ++l) {
      std::complex<double> v = 0.0;
      for (int j = 0; j < k; ++j)
        v += std::complex<double>(Qh[(size_t)l * k + j].x, Qh[(size_t)l * k + j].y) * Wv[(size_t)j * k + ord[i]];
      rows[(size_t)i * L + l] = std::conj(v);   // basis rows d_i = conj(Q w_i)^T
    }
  }
  return MRF_OK;
}

extern "C" mrf_status mrf_dict_basis(mrf_dict d, double energy, int max_rank, int* rank_out) {
  if (!d || !rank_out || !(energy > 0.0 && energy <= 1.0) || max_rank < 1 || max_rank > llr::RMAX)
    return fail(MRF_EINVAL, "mrf_dict_basis: invalid arguments (0 < energy <= 1, 1 <= max_rank <= 32)");
  if (!(d->fro2 > 0.0)) return fail(MRF_EINVAL, "mrf_dict_basis: all-zero dictionary");
  CUDA_TRY(cudaSetDevice(d->device));
  const int K = d->K, L = d->L, k = std::min({max_rank + 16, 64, K, L});
  std::vector<std::complex<double>> rows;
  std::vector<double> lam;
  MRF_TRY(top_right_vectors(d, k, rows, lam));
  int r = 0;
  double acc = 0.0;
  while (r < std::min(max_rank, k) && acc < energy * d->fro2) acc += lam[r++];
  d->basis_h.assign((size_t)r * L, make_float2(0.f, 0.f));
  for (int i = 0; i < r; ++i)
    for (int l = 0; l < L; ++l) {
      const std::complex<double> v = rows[(size_t)i * L + l];
      d->basis_h[(size_t)i * L + l] = make_float2((float)v.real(), (float)v.imag());
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

extern "C" {

mrf_status mrf_dict_basis_copy(mrf_dict d, void* out) {
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

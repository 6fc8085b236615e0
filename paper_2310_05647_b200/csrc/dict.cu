// dict.cu -- host side of dictionary matching Phi_D (Eq. (5)):
// mrf_dict_create / mrf_dict_match / mrf_dict_profile* / mrf_dict_destroy of include/mrfnufft.h.
// The kernels are in match.cuh.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mrfnufft.h"
#include "match.cuh"
#include "status.h"

using namespace mrf;

struct mrf_dict_s {
  int K = 0, L = 0, P = 0, device = 0;
  int KD = 0, NP = 0;            // fp16 row length (2 L padded to 64), GEMM rows (2 K padded to 256)
  __half* dp = nullptr;          // [NP][KD] atom rows (re/im rotated, scaled by 1 / m_k)
  float* w2 = nullptr;           // [NP / 2] (m_k / ||d_k||)^2, 0 for padding
  float* n2inv = nullptr;        // [K] 1 / ||d_k||^2 (0 for a zero atom)
  float2* atoms = nullptr;       // [K][L] complex64 (for the exact pd)
  float* lut = nullptr;          // [K][P]
  __half* xp = nullptr;          // workspace [vcap][KD]
  float* xs = nullptr;           // [vcap] per-voxel scale
  unsigned long long* best = nullptr;   // [vcap] packed (score, ~atom) running maxima
  long long vcap = 0;
  CUtensorMap tmd;
  bool prof = false;             // CUDA events around the tensor-core GEMM (mrf_dict_profile)
  std::vector<cudaEvent_t> ev;   // pairs
  size_t ev_used = 0;
};

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

// 2D fp16 tensor map over a row-major [rows][cols] array with a (64 x box_rows) 128-byte swizzled box
static mrf_status make_tmap(CUtensorMap* m, const __half* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(MRF_ECUDA, "cuTensorMapEncodeTiled is not available");
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * sizeof(__half)};
  const cuuint32_t box[2] = {(cuuint32_t)dm::BK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MRF_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return MRF_OK;
}

static void dict_free(mrf_dict_s* d) {
  if (!d) return;
  cudaSetDevice(d->device);
  for (void* p : {(void*)d->dp, (void*)d->w2, (void*)d->n2inv, (void*)d->atoms, (void*)d->lut, (void*)d->xp,
                  (void*)d->xs, (void*)d->best})
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
  e = cudaFuncSetAttribute(dm::k_dict_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::SMEM);
  if (e != cudaSuccess) {
    dict_free(d);
    return fail(MRF_ECUDA, std::string("mrf_dict_create: ") + cudaGetErrorString(e));
  }
  *out = d;
  return MRF_OK;
}

mrf_status mrf_dict_match(mrf_dict d, const void* x, long long V, int* index, float* pd, float* params, void* stream) {
  if (!d || !x || !index || !pd || V < 1 || V > (1LL << 30))
    return fail(MRF_EINVAL, "mrf_dict_match: invalid arguments");
  for (const void* p : {x, (const void*)index, (const void*)pd, (const void*)params})
    if (p && ((uintptr_t)p % 16) != 0) return fail(MRF_EINVAL, "mrf_dict_match: arrays must be 16-byte aligned");
  CUDA_TRY(cudaSetDevice(d->device));
  cudaStream_t st = (cudaStream_t)stream;
  const long long vpad = ((V + dm::BM - 1) / dm::BM) * dm::BM;
  if (vpad > d->vcap) {
    CUDA_TRY(cudaStreamSynchronize(st));
    if (d->xp) cudaFree(d->xp);
    if (d->xs) cudaFree(d->xs);
    if (d->best) cudaFree(d->best);
    d->xp = nullptr; d->xs = nullptr; d->best = nullptr; d->vcap = 0;
    if (cudaMalloc((void**)&d->xp, (size_t)vpad * d->KD * sizeof(__half)) != cudaSuccess ||
        cudaMalloc((void**)&d->xs, (size_t)vpad * sizeof(float)) != cudaSuccess ||
        cudaMalloc((void**)&d->best, (size_t)vpad * sizeof(unsigned long long)) != cudaSuccess)
      return fail(MRF_ENOMEM, "mrf_dict_match: workspace allocation failed");
    d->vcap = vpad;
  }
  CUtensorMap tmx;
  MRF_TRY(make_tmap(&tmx, d->xp, (uint64_t)d->KD, (uint64_t)vpad, (uint32_t)dm::BM));
  const float2* xf = reinterpret_cast<const float2*>(x);
  dm::k_dict_pack_x<<<(unsigned)(vpad / 32), 256, 0, st>>>(xf, d->L, (int)V, d->KD, d->xp, d->xs);
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
  dm::k_dict_gemm<<<(unsigned)std::min(n_sm, m_tiles * n_tiles), dm::THREADS, dm::SMEM, st>>>(
      tmx, d->tmd, d->w2, m_tiles, n_tiles, d->KD / dm::BK, (int)V, d->best);
  MRF_TRY(check_launch("k_dict_gemm"));
  if (d->prof) {
    CUDA_TRY(cudaEventRecord(d->ev[d->ev_used + 1], st));
    d->ev_used += 2;
  }
  dm::k_dict_fix<<<(unsigned)((V + 31) / 32), 256, 0, st>>>(xf, d->atoms, d->n2inv, d->lut, d->P, d->L, (int)V,
                                                               d->best, index, pd, params);
  MRF_TRY(check_launch("k_dict_fix"));
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

// llr.cu -- host side of the LLR outer step (lambda_1 = 0; PAPER.md:217-264,
// Eqs. (15), (17), (20), (21)): mrf_llr_create / mrf_llr_step / mrf_llr_destroy of
// include/mrfnufft.h.  Kernels in llr.cuh; the subspace basis comes from the dictionary
// (mrf_dict_basis, dict.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/mrfnufft.h"
#include "dict_internal.h"
#include "llr.cuh"
#include "status.h"

using namespace mrf;

struct mrf_llr_s {
  int N = 0, L = 0, p = 0, s = 0, r = 0, nc = 0, device = 0;
  float2* dT = nullptr;       // [L][R] transposed basis, rows zero-padded to R = 16 or 32
  int* corners = nullptr;     // [nc]
  float2* Y = nullptr;        // [N*N][r] coefficients of Z
  float2* P = nullptr;        // [nc*nc][p*p][r] thresholded patch coefficients
  float2* nx = nullptr;       // [L][N][N] A^H A x
  double* nuc = nullptr;      // [nc*nc] per-patch nuclear norms
  std::vector<double> nuc_h;
};

static void llr_free(mrf_llr_s* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  for (void* v : {(void*)h->dT, (void*)h->corners, (void*)h->Y, (void*)h->P, (void*)h->nx, (void*)h->nuc})
    if (v) cudaFree(v);
  delete h;
}

static size_t svt_smem(int p, int r) { return (llr::kSvtThreads / 32) * llr::svt_warp_bytes(p, r); }

extern "C" {

mrf_status mrf_llr_create(mrf_dict dict, int N, int p, int s, mrf_llr* out) {
  if (!dict || !out || N < 2 || p < 1 || p > N || s < 1 || p * p > 1024)
    return fail(MRF_EINVAL, "mrf_llr_create: invalid arguments");
  if (!dict->rank) return fail(MRF_EINVAL, "mrf_llr_create: the dictionary has no basis (call mrf_dict_basis)");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(dict->device));
  auto* h = new mrf_llr_s();
  h->N = N; h->L = dict->L; h->p = p; h->s = s; h->r = dict->rank; h->device = dict->device;
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
            cudaMalloc((void**)&h->nuc, nq * sizeof(double)) == cudaSuccess;
  if (!ok) {
    llr_free(h);
    return fail(MRF_ENOMEM, "mrf_llr_create: device allocation failed");
  }
  std::vector<float2> dT((size_t)R * h->L, make_float2(0.f, 0.f));   // [L][R] from the [r][L] rows
  for (int i = 0; i < h->r; ++i)
    for (int l = 0; l < h->L; ++l) dT[(size_t)l * R + i] = dict->basis_h[(size_t)i * h->L + l];
  cudaError_t e = cudaMemcpy(h->dT, dT.data(), dT.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(h->corners, c.data(), c.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(llr::k_llr_svt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)svt_smem(p, h->r));
  if (e != cudaSuccess) {
    llr_free(h);
    return fail(MRF_ECUDA, std::string("mrf_llr_create: ") + cudaGetErrorString(e));
  }
  *out = h;
  return MRF_OK;
}

mrf_status mrf_llr_step(mrf_llr h, mrf_plan plan, const void* x, const void* rhs, float mu, float lambda2, float beta,
                        void* x_out, double* nuclear, void* stream) {
  if (!h || !plan || !x || !rhs || !x_out) return fail(MRF_EINVAL, "mrf_llr_step: null argument");
  if (!(mu > 0.f) || !(lambda2 >= 0.f) || !(beta > 0.f) || !std::isfinite(mu * lambda2 * beta))
    return fail(MRF_EINVAL, "mrf_llr_step: need mu > 0, lambda2 >= 0, beta > 0");
  for (const void* v : {x, rhs, (const void*)x_out})
    if ((uintptr_t)v % 16) return fail(MRF_EINVAL, "mrf_llr_step: arrays must be 16-byte aligned");
  int pN = 0, pL = 0, pC = 0, pdev = 0;
  plan_dims(plan, &pN, &pL, &pC, &pdev);
  if (pN != h->N || pL != h->L || pdev != h->device)
    return fail(MRF_EINVAL, "mrf_llr_step: the plan's N, L or device differ from the LLR operator's");
  CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int V = h->N * h->N, nq = h->nc * h->nc;
  // A^H A x (the plan checks that x has its shape: [L][N][N] device memory)
  MRF_TRY(mrf_normal(plan, x, h->nx, 0.f, stream));
  const float2* xf = reinterpret_cast<const float2*>(x);
  const unsigned gv = (unsigned)((V + 31) / 32);   // 32 voxels x 8 frame groups per block
  if (h->r <= 16)
    llr::k_llr_coef<16><<<gv, 32 * llr::coef_groups<16>(), 0, st>>>(xf, h->nx, (const float2*)rhs, h->dT, h->r,
                                                                       h->L, V, mu, h->Y);
  else
    llr::k_llr_coef<32><<<gv, 32 * llr::coef_groups<32>(), 0, st>>>(xf, h->nx, (const float2*)rhs, h->dT, h->r,
                                                                       h->L, V, mu, h->Y);
  MRF_TRY(check_launch("k_llr_coef"));
  const int ppb = llr::kSvtThreads / 32;
  llr::k_llr_svt<<<(unsigned)((nq + ppb - 1) / ppb), llr::kSvtThreads, svt_smem(h->p, h->r), st>>>(
      h->Y, h->corners, h->nc, h->N, h->p, h->r, 1.f / beta, nq, h->P, h->nuc);
  MRF_TRY(check_launch("k_llr_svt"));
  const float gamma = mu * lambda2 * beta;
  if (h->r <= 16)
    llr::k_llr_update<16><<<gv, 256, 0, st>>>(h->Y, h->P, h->corners, h->nc, h->N, h->p, h->r, h->dT, h->L, gamma,
                                              (float2*)x_out);
  else
    llr::k_llr_update<32><<<gv, 256, 0, st>>>(h->Y, h->P, h->corners, h->nc, h->N, h->p, h->r, h->dT, h->L, gamma,
                                              (float2*)x_out);
  MRF_TRY(check_launch("k_llr_update"));
  if (nuclear) {   // sum over patches in a fixed order (synchronises the stream)
    CUDA_TRY(cudaMemcpyAsync(h->nuc_h.data(), h->nuc, (size_t)nq * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    double t = 0.0;
    for (double v : h->nuc_h) t += v;
    *nuclear = t;
  }
  return MRF_OK;
}

mrf_status mrf_llr_destroy(mrf_llr h) {
  llr_free(h);
  return MRF_OK;
}

}  // extern "C"

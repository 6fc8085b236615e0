// status.h -- internal error helpers shared by the library's translation units (not public API).
// fail() records the message returned by mrf_last_error(); CUDA_TRY / MRF_TRY propagate errors.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "../../include/mrfnufft.h"

namespace mrf {
mrf_status fail(mrf_status s, const std::string& msg);
mrf_status check_launch(const char* what);   // cudaGetLastError after a launch
void plan_dims(mrf_plan plan, int* N, int* L, int* C, int* device, int* M = nullptr);   // mrfnufft.cu
// 2D tiled TMA map over a row-major [rows][cols] array (row pitch row_bytes, a multiple of 16):
// (box_cols x box_rows) boxes, 128-byte swizzle (box_cols x element size = 128), out-of-bounds
// elements read as zero.  dict.cu.
// subspace normal operator on Toeplitz plans (mrfnufft.cu): K = [r (r + 1) / 2][G*G] complex mixing
// kernels from the basis rows (host [r][L]); apply: Z = P_S A^H A (U d) in coefficients, U and Z
// DEVICE [r][N][N], spectra workspaces [r][C][G*G] each.
bool plan_toeplitz(mrf_plan plan);
bool plan_has_comm(mrf_plan plan);   // the plan reduces over ranks (NCCL communicator or host hook)
int plan_frame_offset(mrf_plan plan);   // global index of the plan's local frame 0
// In-place sum of n elements (dtype MRF_DTYPE_F32 / MRF_DTYPE_F64) of a DEVICE buffer over the
// plan's ranks, on `st`: ncclAllReduce on its communicator, or the host hook
// (mrf_plan_set_host_allreduce); a no-op for an unsharded plan.
mrf_status plan_allreduce(mrf_plan plan, void* buf, size_t n, int dtype, cudaStream_t st);
unsigned long long plan_serial(mrf_plan plan);   // process-wide creation number of the plan
long long sn_elems(mrf_plan plan);
mrf_status sn_build(mrf_plan plan, const float2* basis_h, int r, float2* K, cudaStream_t st);
mrf_status sn_apply(mrf_plan plan, const float2* K, int r, const float2* U, float2* Z, float2* spec_a, float2* spec_b,
                    cudaStream_t st);
mrf_status tmap_2d(CUtensorMap* m, CUtensorMapDataType type, const void* base, uint64_t cols, uint64_t rows,
                   uint64_t row_bytes, uint32_t box_cols, uint32_t box_rows);
}  // namespace mrf

#define CUDA_TRY(expr)                                                                           \
  do {                                                                                           \
    cudaError_t _e = (expr);                                                                     \
    if (_e != cudaSuccess) {                                                                     \
      return ::mrf::fail(MRF_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));        \
    }                                                                                            \
  } while (0)

#define MRF_TRY(expr)                                                                            \
  do {                                                                                           \
    mrf_status _s = (expr);                                                                      \
    if (_s != MRF_OK) return _s;                                                                 \
  } while (0)

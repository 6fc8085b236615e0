// status.h -- internal error helpers shared by the library's translation units (not public API).
// fail() records the message returned by mrf_last_error(); CUDA_TRY / MRF_TRY propagate errors.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/mrfnufft.h"

namespace mrf {
mrf_status fail(mrf_status s, const std::string& msg);
mrf_status check_launch(const char* what);   // cudaGetLastError after a launch
void plan_dims(mrf_plan plan, int* N, int* L, int* C, int* device);   // mrfnufft.cu
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

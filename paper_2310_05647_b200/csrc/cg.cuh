// cg.cuh -- CG vector kernels with float64 inner products.
#pragma once
#include <cuda_runtime.h>

#include "fft.cuh"

namespace mrf {

// ------------------------------------------------------------------------------ CG vector ops
// Inner products accumulate in float64 (SURVEY.md §8(c) reading #16): per-block partials written
// to `part`, then summed in a fixed order by k_reduce (deterministic for a fixed grid).
constexpr int kVecThreads = 256;

__device__ __forceinline__ double2 block_sum2(double2 v) {
  __shared__ double2 red[kVecThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kVecThreads / 32; ++i) { s.x += red[i].x; s.y += red[i].y; }
  }
  return s;   // valid in thread 0
}

// dst = sum of part[0..n) in a fixed order (one block)
__global__ void __launch_bounds__(kVecThreads) k_reduce(const double2* __restrict__ part, int n, double2* __restrict__ dst) {
  double2 s = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) { s.x += part[i].x; s.y += part[i].y; }
  s = block_sum2(s);
  if (threadIdx.x == 0) *dst = s;
}

// Device-resident CG scalars.
struct CGScalars {
  double2 pq;        // <p, q>          (global after allreduce)
  double2 rr;        // <r, r>          (global after allreduce)
  double rho, rho0, alpha, beta;
  int breakdown, iters;
};

// r = rhs - q ; p = r  (initial residual); partial <r,r>
__global__ void __launch_bounds__(kVecThreads) k_cg_init(const float2* __restrict__ rhs, const float2* __restrict__ q,
                                                         float2* __restrict__ r, float2* __restrict__ pv, size_t n,
                                                         double2* __restrict__ part) {
  double2 s = make_double2(0.0, 0.0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 v = csub(rhs[i], q[i]);
    r[i] = v;
    pv[i] = v;
    s.x += (double)v.x * v.x + (double)v.y * v.y;
  }
  s = block_sum2(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// rho0 = rho = rr.x ; hist[0]
__global__ void k_cg_start(CGScalars* sc, double* hist) {
  sc->rho = sc->rr.x;
  sc->rho0 = sc->rr.x;
  sc->breakdown = 0;
  sc->iters = 0;
  sc->alpha = 0.0;   // consumed by the first fused row pass: x += 0 * p, p = r + 0 * p
  sc->beta = 0.0;
  hist[0] = sqrt(sc->rr.x);
}

// alpha = rho / Re<p,q>  (breakdown => alpha = 0, flagged)
__global__ void k_cg_alpha(CGScalars* sc) {
  const double pq = sc->pq.x;
  if (sc->rho0 == 0.0) {
    sc->alpha = 0.0;
  } else if (!(pq > 0.0) || !isfinite(pq)) {
    sc->alpha = 0.0;
    sc->breakdown = 1;
  } else {
    sc->alpha = sc->rho / pq;
  }
}

// r -= alpha q ; partial <r,r>   (x is advanced lazily: x += alpha p in the next row pass)
__global__ void __launch_bounds__(kVecThreads) k_cg_r(float2* __restrict__ r, const float2* __restrict__ q, size_t n,
                                                      const CGScalars* __restrict__ sc, double2* __restrict__ part) {
  const float alpha = (float)sc->alpha;
  double2 s = make_double2(0.0, 0.0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 qi = q[i];
    float2 ri = r[i];
    ri.x = fmaf(-alpha, qi.x, ri.x);
    ri.y = fmaf(-alpha, qi.y, ri.y);
    r[i] = ri;
    s.x += (double)ri.x * ri.x + (double)ri.y * ri.y;
  }
  s = block_sum2(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// x += alpha p  (the last deferred solution update)
__global__ void __launch_bounds__(kVecThreads) k_cg_xfin(float2* __restrict__ x, const float2* __restrict__ pv, size_t n,
                                                         const CGScalars* __restrict__ sc) {
  const float alpha = (float)sc->alpha;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 pi = pv[i];
    float2 xi = x[i];
    xi.x = fmaf(alpha, pi.x, xi.x);
    xi.y = fmaf(alpha, pi.y, xi.y);
    x[i] = xi;
  }
}

// x += alpha p_old ; p = r + beta p_old   (unfused form, used when C > 1)
__global__ void __launch_bounds__(kVecThreads) k_cg_px(float2* __restrict__ x, float2* __restrict__ pv,
                                                       const float2* __restrict__ r, size_t n,
                                                       const CGScalars* __restrict__ sc) {
  const float alpha = (float)sc->alpha, beta = (float)sc->beta;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 pi = pv[i], ri = r[i];
    float2 xi = x[i];
    xi.x = fmaf(alpha, pi.x, xi.x);
    xi.y = fmaf(alpha, pi.y, xi.y);
    x[i] = xi;
    pv[i] = make_float2(fmaf(beta, pi.x, ri.x), fmaf(beta, pi.y, ri.y));
  }
}

// beta = rho' / rho ; rho = rho' ; hist[k+1]
__global__ void k_cg_beta(CGScalars* sc, double* hist, int k) {
  const double rn = sc->rr.x;
  sc->beta = sc->rho > 0.0 ? rn / sc->rho : 0.0;
  sc->rho = rn;
  sc->iters = k + 1;
  hist[k + 1] = sqrt(rn);
}

// a += mu b   (rhs = A^H y + mu z)
__global__ void __launch_bounds__(kVecThreads) k_axpy(float2* __restrict__ a, const float2* __restrict__ b, float mu, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 bi = b[i];
    float2 ai = a[i];
    ai.x = fmaf(mu, bi.x, ai.x);
    ai.y = fmaf(mu, bi.y, ai.y);
    a[i] = ai;
  }
}

}  // namespace mrf

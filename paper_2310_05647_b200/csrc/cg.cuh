// cg.cuh -- CG vector kernels with float64 inner products.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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

// Device-resident CG scalars.
struct CGScalars {
  double2 pq;        // <p, q>          (global after allreduce)
  double2 rr;        // <r, r>          (global after allreduce)
  double2 rz;        // <r, z>, z = M^-1 r (PCG; global after allreduce)
  double rho, rho0, alpha, beta;   // rho = <r, r> (CG) or <r, z> (PCG)
  double res, res0;                // <r, r> now and at the start (history, tol, rel_resid)
  int breakdown, iters;
};

// The scalar steps of the iteration (single thread).
// rho0 = rho = rr.x ; hist[0]
__device__ __forceinline__ void cg_start(CGScalars* sc, double* hist) {
  sc->rho = sc->rr.x;
  sc->rho0 = sc->rr.x;
  sc->res = sc->res0 = sc->rr.x;
  sc->breakdown = 0;
  sc->iters = 0;
  sc->alpha = 0.0;   // consumed by the first fused row pass: x += 0 * p, p = r + 0 * p
  sc->beta = 0.0;
  hist[0] = sqrt(sc->rr.x);
}
// alpha = rho / Re<p,q>  (breakdown => alpha = 0, flagged); ha[k] = alpha
__device__ __forceinline__ void cg_alpha(CGScalars* sc, double* ha, int k) {
  const double pq = sc->pq.x;
  if (sc->rho0 == 0.0) {
    sc->alpha = 0.0;
  } else if (!(pq > 0.0) || !isfinite(pq)) {
    sc->alpha = 0.0;
    sc->breakdown = 1;
  } else {
    sc->alpha = sc->rho / pq;
  }
  ha[k] = sc->alpha;
}
// beta = rho' / rho ; rho = rho' ; hist[k+1], hb[k] = beta
__device__ __forceinline__ void cg_beta(CGScalars* sc, double* hist, double* hb, int k) {
  const double rn = sc->rr.x;
  sc->beta = sc->rho > 0.0 ? rn / sc->rho : 0.0;
  hb[k] = sc->beta;
  sc->rho = rn;
  sc->res = rn;
  sc->iters = k + 1;
  hist[k + 1] = sqrt(rn);
}
// PCG: rho0 = <r0, z0> (steps), res0 = <r0, r0> (history); rr already reduced
__device__ __forceinline__ void cg_start_pc(CGScalars* sc, double* hist) {
  cg_start(sc, hist);
  sc->rho = sc->rz.x;
  sc->rho0 = sc->rz.x;
}
// PCG: beta = <r', z'> / <r, z> ; rho = <r', z'> ; res = <r', r'>
__device__ __forceinline__ void cg_beta_pc(CGScalars* sc, double* hist, double* hb, int k) {
  const double rn = sc->rz.x;
  sc->beta = sc->rho > 0.0 ? rn / sc->rho : 0.0;
  hb[k] = sc->beta;
  sc->rho = rn;
  sc->res = sc->rr.x;
  sc->iters = k + 1;
  hist[k + 1] = sqrt(sc->rr.x);
}
enum { kRedPlain = 0, kRedStart = 1, kRedAlpha = 2, kRedBeta = 3, kRedStartPc = 4, kRedBetaPc = 5 };

// dst = sum of part[0..n) in a fixed order (one block of kReduceThreads, 4 independent loads in
// flight per thread)
constexpr int kReduceThreads = 1024;
// OP != kRedPlain: then the scalar step that consumes dst (one launch instead of two when the
// plan has no communicator to all-reduce dst first).
template <int OP>
__global__ void __launch_bounds__(kReduceThreads) k_reduce(const double2* __restrict__ part, int n, double2* __restrict__ dst,
                                                           CGScalars* sc, double* hist, double* hx, int k) {
  __shared__ double2 red[kReduceThreads / 32];
  double2 s0 = make_double2(0.0, 0.0), s1 = s0, s2 = s0, s3 = s0;
  int i = threadIdx.x;
  for (; i + 3 * kReduceThreads < n; i += 4 * kReduceThreads) {
    const double2 a = part[i], b = part[i + kReduceThreads], c = part[i + 2 * kReduceThreads], d = part[i + 3 * kReduceThreads];
    s0.x += a.x; s0.y += a.y; s1.x += b.x; s1.y += b.y; s2.x += c.x; s2.y += c.y; s3.x += d.x; s3.y += d.y;
  }
  for (; i < n; i += kReduceThreads) { s0.x += part[i].x; s0.y += part[i].y; }
  double2 v = make_double2((s0.x + s1.x) + (s2.x + s3.x), (s0.y + s1.y) + (s2.y + s3.y));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = make_double2(0.0, 0.0);
    for (int w = 0; w < kReduceThreads / 32; ++w) { t.x += red[w].x; t.y += red[w].y; }
    *dst = t;
    if (OP == kRedStart) cg_start(sc, hist);
    if (OP == kRedAlpha) cg_alpha(sc, hx, k);
    if (OP == kRedBeta) cg_beta(sc, hist, hx, k);
    if (OP == kRedStartPc) cg_start_pc(sc, hist);
    if (OP == kRedBetaPc) cg_beta_pc(sc, hist, hx, k);
  }
}

// dst = sum a[0..na) + mu * sum b[0..nb) (each summed in a fixed order), then alpha (OP ==
// kRedAlpha) -- the split-phase CG's <p, (A^H A + mu I) p> = ||A p||^2 + mu ||p||^2.
template <int OP>
__global__ void __launch_bounds__(kReduceThreads) k_reduce_pq(const double2* __restrict__ a, int na,
                                                              const double2* __restrict__ b, int nb, double mu,
                                                              double2* __restrict__ dst, CGScalars* sc, double* hx, int k) {
  __shared__ double red[2][kReduceThreads / 32];
  double sa = 0.0, sb = 0.0;
  for (int i = threadIdx.x; i < na; i += kReduceThreads) sa += a[i].x;
  for (int i = threadIdx.x; i < nb; i += kReduceThreads) sb += b[i].x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = sa;
    red[1][threadIdx.x >> 5] = sb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tb = 0.0;
    for (int w = 0; w < kReduceThreads / 32; ++w) { ta += red[0][w]; tb += red[1][w]; }
    *dst = make_double2(ta + mu * tb, 0.0);
    if (OP == kRedAlpha) cg_alpha(sc, hx, k);
  }
}

// The vector kernels treat the complex64 arrays as float4 (two elements; n is even and the arrays
// are 16-byte aligned) and keep 4 independent float4 per operand in flight per thread (a
// grid-stride loop unrolled by 4), enough outstanding bytes per SM to stream at HBM rate.
#define MRF_VEC4_LOOP(n4, ...)                                                                   \
  {                                                                                              \
    const size_t st_ = (size_t)gridDim.x * blockDim.x;                                           \
    size_t i_ = blockIdx.x * (size_t)blockDim.x + threadIdx.x;                                  \
    for (; i_ + 3 * st_ < (n4); i_ += 4 * st_) {                                                 \
      _Pragma("unroll") for (int u_ = 0; u_ < 4; ++u_) {                                         \
        const size_t i = i_ + u_ * st_;                                                          \
        __VA_ARGS__                                                                              \
      }                                                                                          \
    }                                                                                            \
    for (; i_ < (n4); i_ += st_) {                                                               \
      const size_t i = i_;                                                                       \
      __VA_ARGS__                                                                                \
    }                                                                                            \
  }

__device__ __forceinline__ double norm2d(float4 v) {
  return ((double)v.x * v.x + (double)v.y * v.y) + ((double)v.z * v.z + (double)v.w * v.w);
}


// partial ||v||^2 per block (v: n complex64 values, 8-byte aligned; any n)
__global__ void __launch_bounds__(kVecThreads) k_sqnorm(const float2* __restrict__ v, size_t n, double2* __restrict__ part) {
  double2 s = make_double2(0.0, 0.0);
  const float4* v4 = reinterpret_cast<const float4*>(v);
  if (reinterpret_cast<uintptr_t>(v) % 16 == 0) {
    MRF_VEC4_LOOP(n / 2, { s.x += norm2d(v4[i]); })
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const float2 t = v[n - 1];
      s.x += (double)t.x * t.x + (double)t.y * t.y;
    }
  } else {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const float2 t = v[i];
      s.x += (double)t.x * t.x + (double)t.y * t.y;
    }
  }
  s = block_sum2(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// r = rhs - q ; p = r  (initial residual; q == nullptr: x0 = 0, r = rhs); partial <r,r>.
// rhs may be r itself (the solver's call): with q == nullptr r already holds its value and is
// not rewritten (one image pass fewer).
__global__ void __launch_bounds__(kVecThreads) k_cg_init(const float2* rhs, const float2* __restrict__ q,
                                                         float2* r, float2* __restrict__ pv, size_t n,
                                                         double2* __restrict__ part) {
  const float4* rh4 = reinterpret_cast<const float4*>(rhs);
  const float4* q4 = reinterpret_cast<const float4*>(q);
  float4* r4 = reinterpret_cast<float4*>(r);
  float4* p4 = reinterpret_cast<float4*>(pv);
  const bool keep_r = q == nullptr && rhs == r;
  double2 s = make_double2(0.0, 0.0);
  MRF_VEC4_LOOP(n / 2, {
    const float4 a = rh4[i], b = q4 ? q4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 v = make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
    if (!keep_r) r4[i] = v;
    p4[i] = v;
    s.x += norm2d(v);
  })
  s = block_sum2(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_cg_start(CGScalars* sc, double* hist) { cg_start(sc, hist); }
__global__ void k_cg_alpha(CGScalars* sc, double* ha, int k) { cg_alpha(sc, ha, k); }

// r -= alpha q ; partial <r,r>   (x is advanced lazily: x += alpha p in the next row pass)
__global__ void __launch_bounds__(kVecThreads) k_cg_r(float2* __restrict__ r, const float2* __restrict__ q, size_t n,
                                                      const CGScalars* __restrict__ sc, double2* __restrict__ part) {
  const float alpha = (float)sc->alpha;
  const float4* q4 = reinterpret_cast<const float4*>(q);
  float4* r4 = reinterpret_cast<float4*>(r);
  double2 s = make_double2(0.0, 0.0);
  MRF_VEC4_LOOP(n / 2, {
    const float4 qi = q4[i];
    float4 ri = r4[i];
    ri.x = fmaf(-alpha, qi.x, ri.x);
    ri.y = fmaf(-alpha, qi.y, ri.y);
    ri.z = fmaf(-alpha, qi.z, ri.z);
    ri.w = fmaf(-alpha, qi.w, ri.w);
    r4[i] = ri;
    s.x += norm2d(ri);
  })
  s = block_sum2(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// x += alpha p  (the last deferred solution update)
__global__ void __launch_bounds__(kVecThreads) k_cg_xfin(float2* __restrict__ x, const float2* __restrict__ pv, size_t n,
                                                         const CGScalars* __restrict__ sc) {
  const float alpha = (float)sc->alpha;
  const float4* p4 = reinterpret_cast<const float4*>(pv);
  float4* x4 = reinterpret_cast<float4*>(x);
  MRF_VEC4_LOOP(n / 2, {
    const float4 pi = p4[i];
    float4 xi = x4[i];
    xi.x = fmaf(alpha, pi.x, xi.x);
    xi.y = fmaf(alpha, pi.y, xi.y);
    xi.z = fmaf(alpha, pi.z, xi.z);
    xi.w = fmaf(alpha, pi.w, xi.w);
    x4[i] = xi;
  })
}

// x += alpha p_old ; p = r + beta p_old   (unfused form, used when C > 1); with part != nullptr
// also the block partials of ||p||^2 (split-phase CG)
__global__ void __launch_bounds__(kVecThreads) k_cg_px(float2* __restrict__ x, float2* __restrict__ pv,
                                                       const float2* __restrict__ r, size_t n,
                                                       const CGScalars* __restrict__ sc, double2* __restrict__ part) {
  double2 s = make_double2(0.0, 0.0);
  const float alpha = (float)sc->alpha, beta = (float)sc->beta;
  float4* p4 = reinterpret_cast<float4*>(pv);
  float4* x4 = reinterpret_cast<float4*>(x);
  const float4* r4 = reinterpret_cast<const float4*>(r);
  MRF_VEC4_LOOP(n / 2, {
    const float4 pi = p4[i], ri = r4[i];
    float4 xi = x4[i];
    xi.x = fmaf(alpha, pi.x, xi.x);
    xi.y = fmaf(alpha, pi.y, xi.y);
    xi.z = fmaf(alpha, pi.z, xi.z);
    xi.w = fmaf(alpha, pi.w, xi.w);
    x4[i] = xi;
    const float4 pn = make_float4(fmaf(beta, pi.x, ri.x), fmaf(beta, pi.y, ri.y), fmaf(beta, pi.z, ri.z), fmaf(beta, pi.w, ri.w));
    p4[i] = pn;
    s.x += norm2d(pn);
  })
  if (part) {
    s = block_sum2(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

__global__ void k_cg_beta(CGScalars* sc, double* hist, double* hb, int k) { cg_beta(sc, hist, hb, k); }
__global__ void k_cg_start_pc(CGScalars* sc, double* hist) { cg_start_pc(sc, hist); }
__global__ void k_cg_beta_pc(CGScalars* sc, double* hist, double* hb, int k) { cg_beta_pc(sc, hist, hb, k); }

// a += mu b   (rhs = A^H y + mu z)
__global__ void __launch_bounds__(kVecThreads) k_axpy(float2* __restrict__ a, const float2* __restrict__ b, float mu, size_t n) {
  float4* a4 = reinterpret_cast<float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  MRF_VEC4_LOOP(n / 2, {
    const float4 bi = b4[i];
    float4 ai = a4[i];
    ai.x = fmaf(mu, bi.x, ai.x);
    ai.y = fmaf(mu, bi.y, ai.y);
    ai.z = fmaf(mu, bi.z, ai.z);
    ai.w = fmaf(mu, bi.w, ai.w);
    a4[i] = ai;
  })
}

}  // namespace mrf

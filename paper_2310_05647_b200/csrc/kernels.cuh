// kernels.cuh -- sm_100a kernels of the multi-frame KB-gridding NUFFT pair and the CG vector ops.
//
// Pipeline per frame l and coil c (the paper's A = F_u C):
//   forward A  : K_fwd_rows  (a1 deapod . coil . pad, a2 row FFT on the N non-zero rows)
//                K_fwd_cols  (a2 column FFT of one 16-column strip, a3 KB gather interpolation)
//   adjoint A^H: K_adj_cols  (a4 KB spread into the strip in shared memory, a5 column iFFT,
//                             row crop)
//                K_adj_rows  (a5 row iFFT, a6 crop . deapod . conj-coil . coil sum [+ mu x])
// The N x G "half grid" between the row and the column pass lives in a frame-batch workspace
// sized to stay resident in the 126 MB L2 (the full G x G grid never leaves shared memory).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"

namespace mrf {

constexpr int SW = 16;  // columns per strip (>= W so a point's x-taps touch at most 2 strips)

struct DevPlan {
  int N, G, M, R, C, W, S;            // S = G / SW strips
  const float2* __restrict__ coils;   // [C][N][N] or nullptr (C == 1)
  const float* __restrict__ dap;      // [N]  1 / (psi(n) sqrt(N))
  const float2* __restrict__ tw;      // [G]  tw[k1*Q + n2] = exp(-i 2 pi n2 k1 / G)
  const float* __restrict__ wts;      // [R][M][2W]  wx[0..W) | wy[0..W)
  const int2* __restrict__ ent;       // strip entries {j, gy0 | tx0<<11 | ntx<<16 | cx0<<21}
  const int* __restrict__ soff;       // [R][S+1] absolute entry offsets
  const int* __restrict__ fil;        // [L_local] interleaf of each local frame
};

// image index <-> wrapped grid index (centred n = i - N/2, grid position n mod G)
template <int G>
__device__ __forceinline__ int grid_to_img(int pos) {   // pos in the kept set
  constexpr int N = G / 2;
  return pos < N / 2 ? pos + N / 2 : pos - (G - N / 2);
}

template <int G>
constexpr int rows_threads() { return 256; }
template <int G>
constexpr int cols_threads() { return SW * FFTShape<G>::T; }

template <int G>
constexpr size_t rows_smem() {
  using S = FFTShape<G>;
  return (size_t(G) + size_t(256 / S::T) * S::Q * (S::P + 1)) * sizeof(float2);
}
template <int G>
constexpr size_t cols_smem() { return (size_t(G) + size_t(G) * SW) * sizeof(float2); }

// ------------------------------------------------------------------------------ forward rows
// grid (N / RPC, nb); frame l = l0 + blockIdx.y; writes H[(bl*C + c)][iy][0..G)
template <int G>
__global__ void __launch_bounds__(256, 2)
k_fwd_rows(DevPlan p, const float2* __restrict__ x, float2* __restrict__ H, int l0) {
  using S = FFTShape<G>;
  constexpr int P = S::P, Q = S::Q, T = S::T, N = G / 2, RPC = 256 / T, A = Q / T, B = P / T;
  extern __shared__ float2 sm[];
  float2* stw = sm;
  float2* ex = sm + G;
  for (int i = threadIdx.x; i < G; i += blockDim.x) stw[i] = p.tw[i];
  const int rloc = threadIdx.x / T, t = threadIdx.x % T;
  const int iy = blockIdx.x * RPC + rloc;
  const int bl = blockIdx.y, l = l0 + bl;
  const float2* xr = x + ((size_t)l * N + iy) * N;
  const float dy = p.dap[iy];
  float2* myex = ex + rloc * (Q * (P + 1));
  __syncthreads();
  for (int c = 0; c < p.C; ++c) {
    float2 v[A][P];
    const float2* sr = p.coils ? p.coils + ((size_t)c * N + iy) * N : nullptr;
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) {
        if (n1 < P / 4 || n1 >= 3 * P / 4) {
          const int ix = grid_to_img<G>(Q * n1 + n2);
          float2 val = cscale(__ldg(xr + ix), dy * __ldg(p.dap + ix));
          if (sr) val = cmul(val, __ldg(sr + ix));
          v[a][n1] = val;
        } else {
          v[a][n1] = make_float2(0.f, 0.f);
        }
      }
      dft<P, -1>(v[a]);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) myex[n2 * (P + 1) + k1] = cmul(v[a][k1], stw[k1 * Q + n2]);
    }
    __syncwarp();
    float2* Hr = H + (((size_t)bl * p.C + c) * N + iy) * G;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      float2 w[Q];
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) w[n2] = myex[n2 * (P + 1) + k1];
      dft<Q, -1>(w);
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) Hr[k1 + P * k2] = w[k2];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------ forward columns
// grid (S, nb*C); fc = bl*C + c.  y points at frame l0's first sample and must be zeroed.
template <int G>
__global__ void __launch_bounds__(SW * FFTShape<G>::T)
k_fwd_cols(DevPlan p, const float2* __restrict__ H, float2* __restrict__ y, int l0) {
  using S = FFTShape<G>;
  constexpr int P = S::P, Q = S::Q, T = S::T, N = G / 2, A = Q / T, B = P / T;
  extern __shared__ float2 sm[];
  float2* stw = sm;
  float2* buf = sm + G;
  for (int i = threadIdx.x; i < G; i += blockDim.x) stw[i] = p.tw[i];
  const int c = threadIdx.x % SW, t = threadIdx.x / SW;
  const int s = blockIdx.x, fc = blockIdx.y;
  const int gx = s * SW + c;
  const float2* Hc = H + (size_t)fc * N * G + gx;
  float2 v[A][P];
#pragma unroll
  for (int a = 0; a < A; ++a) {
    const int n2 = t + T * a;
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) {
      if (n1 < P / 4 || n1 >= 3 * P / 4) {
        v[a][n1] = Hc[(size_t)grid_to_img<G>(Q * n1 + n2) * G];
      } else {
        v[a][n1] = make_float2(0.f, 0.f);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < A; ++a) {
    const int n2 = t + T * a;
    dft<P, -1>(v[a]);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) buf[(n2 * P + k1) * SW + c] = cmul(v[a][k1], stw[k1 * Q + n2]);
  }
  __syncthreads();
  float2 w[B][Q];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int k1 = t + T * b;
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) w[b][n2] = buf[(n2 * P + k1) * SW + c];
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int k1 = t + T * b;
    dft<Q, -1>(w[b]);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) buf[(k1 + P * k2) * SW + c] = w[b][k2];   // strip [gy][c]
  }
  __syncthreads();
  // a3: KB gather interpolation of the points whose x-taps fall in this strip
  const int bl = fc / p.C;
  const int r = p.fil[l0 + bl];
  const int e0 = p.soff[r * (p.S + 1) + s], e1 = p.soff[r * (p.S + 1) + s + 1];
  const int W = p.W;
  for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int2 en = __ldg(p.ent + e);
    const int j = en.x, gy0 = en.y & 2047, tx0 = (en.y >> 11) & 31, ntx = (en.y >> 16) & 31,
              cx0 = (en.y >> 21) & 31;
    const float* wp = p.wts + ((size_t)r * p.M + j) * (2 * W);
    float2 acc = make_float2(0.f, 0.f);
    for (int ty = 0; ty < W; ++ty) {
      const float2* row = buf + ((gy0 + ty) & (G - 1)) * SW + cx0;
      float2 ra = make_float2(0.f, 0.f);
      for (int i = 0; i < ntx; ++i) {
        const float wx = __ldg(wp + tx0 + i);
        const float2 g = row[i];
        ra.x = fmaf(wx, g.x, ra.x);
        ra.y = fmaf(wx, g.y, ra.y);
      }
      const float wy = __ldg(wp + W + ty);
      acc.x = fmaf(wy, ra.x, acc.x);
      acc.y = fmaf(wy, ra.y, acc.y);
    }
    float2* yo = y + (size_t)fc * p.M + j;
    atomicAdd(&yo->x, acc.x);   // at most two strips contribute: order-independent result
    atomicAdd(&yo->y, acc.y);
  }
}

// ------------------------------------------------------------------------------ adjoint columns
// grid (S, nb*C).  y points at frame l0's first sample; writes H[fc][iy][gx] for the N kept rows.
template <int G>
__global__ void __launch_bounds__(SW * FFTShape<G>::T)
k_adj_cols(DevPlan p, const float2* __restrict__ y, float2* __restrict__ H, int l0) {
  using S = FFTShape<G>;
  constexpr int P = S::P, Q = S::Q, T = S::T, N = G / 2, A = Q / T, B = P / T;
  extern __shared__ float2 sm[];
  float2* stw = sm;
  float2* buf = sm + G;
  for (int i = threadIdx.x; i < G; i += blockDim.x) stw[i] = p.tw[i];
  for (int i = threadIdx.x; i < G * SW; i += blockDim.x) buf[i] = make_float2(0.f, 0.f);
  const int c = threadIdx.x % SW, t = threadIdx.x / SW;
  const int s = blockIdx.x, fc = blockIdx.y;
  const int gx = s * SW + c;
  __syncthreads();
  // a4: KB spreading into the shared-memory strip
  {
    const int bl = fc / p.C;
    const int r = p.fil[l0 + bl];
    const int e0 = p.soff[r * (p.S + 1) + s], e1 = p.soff[r * (p.S + 1) + s + 1];
    const int W = p.W;
    // one work item per (entry, y-tap): W x more parallelism than one thread per point
    const int n_items = (e1 - e0) * W;
    for (int it = threadIdx.x; it < n_items; it += blockDim.x) {
      const int e = e0 + it / W, ty = it % W;
      const int2 en = __ldg(p.ent + e);
      const int j = en.x, gy0 = en.y & 2047, tx0 = (en.y >> 11) & 31, ntx = (en.y >> 16) & 31,
                cx0 = (en.y >> 21) & 31;
      const float* wp = p.wts + ((size_t)r * p.M + j) * (2 * W);
      const float2 val = __ldg(y + (size_t)fc * p.M + j);
      const float wy = __ldg(wp + W + ty);
      const float2 vy = make_float2(wy * val.x, wy * val.y);
      float2* row = buf + ((gy0 + ty) & (G - 1)) * SW + cx0;
      for (int i = 0; i < ntx; ++i) {
        const float wx = __ldg(wp + tx0 + i);
        atomicAdd(&row[i].x, wx * vy.x);
        atomicAdd(&row[i].y, wx * vy.y);
      }
    }
  }
  __syncthreads();
  // a5: column inverse FFT (e^{+i}, unnormalised), only the N kept output rows are stored
  float2 v[A][P];
#pragma unroll
  for (int a = 0; a < A; ++a) {
    const int n2 = t + T * a;
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) v[a][n1] = buf[(Q * n1 + n2) * SW + c];
  }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < A; ++a) {
    const int n2 = t + T * a;
    dft<P, +1>(v[a]);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) buf[(n2 * P + k1) * SW + c] = cmulc(v[a][k1], stw[k1 * Q + n2]);
  }
  __syncthreads();
  float2* Hc = H + (size_t)fc * N * G + gx;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int k1 = t + T * b;
    float2 w[Q];
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) w[n2] = buf[(n2 * P + k1) * SW + c];
    dft<Q, +1>(w);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) {
      if (k2 < Q / 4 || k2 >= 3 * Q / 4) Hc[(size_t)grid_to_img<G>(k1 + P * k2) * G] = w[k2];
    }
  }
}

// ------------------------------------------------------------------------------ adjoint rows
// grid (N / RPC, nb).  out[l] = sum_c conj(S_c) . crop(rowIFFT(H[l,c])) . dap dap  (+ mu xin[l])
template <int G>
__global__ void __launch_bounds__(256, 2)
k_adj_rows(DevPlan p, const float2* __restrict__ H, float2* __restrict__ out,
           const float2* __restrict__ xin, float mu, int l0) {
  using S = FFTShape<G>;
  constexpr int P = S::P, Q = S::Q, T = S::T, N = G / 2, RPC = 256 / T, A = Q / T, B = P / T;
  extern __shared__ float2 sm[];
  float2* stw = sm;
  float2* ex = sm + G;
  for (int i = threadIdx.x; i < G; i += blockDim.x) stw[i] = p.tw[i];
  const int rloc = threadIdx.x / T, t = threadIdx.x % T;
  const int iy = blockIdx.x * RPC + rloc;
  const int bl = blockIdx.y, l = l0 + bl;
  float2* myex = ex + rloc * (Q * (P + 1));
  float2 acc[B][Q / 2];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int kk = 0; kk < Q / 2; ++kk) acc[b][kk] = make_float2(0.f, 0.f);
  __syncthreads();
  for (int c = 0; c < p.C; ++c) {
    const float2* Hr = H + (((size_t)bl * p.C + c) * N + iy) * G;
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
      float2 v[P];
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) v[n1] = Hr[Q * n1 + n2];
      dft<P, +1>(v);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) myex[n2 * (P + 1) + k1] = cmulc(v[k1], stw[k1 * Q + n2]);
    }
    __syncwarp();
    const float2* sr = p.coils ? p.coils + ((size_t)c * N + iy) * N : nullptr;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      float2 w[Q];
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) w[n2] = myex[n2 * (P + 1) + k1];
      dft<Q, +1>(w);
#pragma unroll
      for (int kk = 0; kk < Q / 2; ++kk) {
        const int k2 = kk < Q / 4 ? kk : kk + Q / 2;
        float2 val = w[k2];
        if (sr) val = cmulc(val, __ldg(sr + grid_to_img<G>(k1 + P * k2)));
        acc[b][kk] = cadd(acc[b][kk], val);
      }
    }
    __syncwarp();
  }
  const float dy = p.dap[iy];
  float2* orow = out + ((size_t)l * N + iy) * N;
  const float2* xrow = xin ? xin + ((size_t)l * N + iy) * N : nullptr;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int k1 = t + T * b;
#pragma unroll
    for (int kk = 0; kk < Q / 2; ++kk) {
      const int k2 = kk < Q / 4 ? kk : kk + Q / 2;
      const int ix = grid_to_img<G>(k1 + P * k2);
      float2 o = cscale(acc[b][kk], dy * __ldg(p.dap + ix));
      if (xrow) {
        const float2 xv = xrow[ix];
        o.x = fmaf(mu, xv.x, o.x);
        o.y = fmaf(mu, xv.y, o.y);
      }
      orow[ix] = o;
    }
  }
}

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

// part[block] = sum conj(a) b over this block's grid-stride share
__global__ void __launch_bounds__(kVecThreads) k_dot(const float2* __restrict__ a, const float2* __restrict__ b,
                                                     size_t n, double2* __restrict__ part) {
  double2 s = make_double2(0.0, 0.0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 u = a[i], v = b[i];
    s.x += (double)u.x * v.x + (double)u.y * v.y;
    s.y += (double)u.x * v.y - (double)u.y * v.x;
  }
  s = block_sum2(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
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

// x += alpha p ; r -= alpha q ; partial <r,r>
__global__ void __launch_bounds__(kVecThreads) k_cg_xr(float2* __restrict__ x, float2* __restrict__ r,
                                                       const float2* __restrict__ pv, const float2* __restrict__ q,
                                                       size_t n, const CGScalars* __restrict__ sc,
                                                       double2* __restrict__ part) {
  const float alpha = (float)sc->alpha;
  double2 s = make_double2(0.0, 0.0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 pi = pv[i], qi = q[i];
    float2 xi = x[i], ri = r[i];
    xi.x = fmaf(alpha, pi.x, xi.x);
    xi.y = fmaf(alpha, pi.y, xi.y);
    ri.x = fmaf(-alpha, qi.x, ri.x);
    ri.y = fmaf(-alpha, qi.y, ri.y);
    x[i] = xi;
    r[i] = ri;
    s.x += (double)ri.x * ri.x + (double)ri.y * ri.y;
  }
  s = block_sum2(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// beta = rho' / rho ; rho = rho' ; hist[k+1]
__global__ void k_cg_beta(CGScalars* sc, double* hist, int k) {
  const double rn = sc->rr.x;
  sc->beta = sc->rho > 0.0 ? rn / sc->rho : 0.0;
  sc->rho = rn;
  sc->iters = k + 1;
  hist[k + 1] = sqrt(rn);
}

// p = r + beta p
__global__ void __launch_bounds__(kVecThreads) k_cg_p(float2* __restrict__ pv, const float2* __restrict__ r, size_t n,
                                                      const CGScalars* __restrict__ sc) {
  const float beta = (float)sc->beta;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 ri = r[i], pi = pv[i];
    pv[i] = make_float2(fmaf(beta, pi.x, ri.x), fmaf(beta, pi.y, ri.y));
  }
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

// precond.cuh -- the circulant image-space preconditioner of the PCG data-consistency solve
// (reading 28), sm_100a.
//
// Per frame, M = C + gamma I with C T. Chan's optimal circulant of the frame's exact normal
// operator A^H A (the normal operator of PAPER.md:217 Eq. (15)): eigenvalues
//   lambda_m = ||A f_m||^2 = N^-4 sum_j F(kx_j - mx/N) F(ky_j - my/N),  F(t) = sin^2(pi N t) / sin^2(pi t),
// centred m (the Rayleigh quotients at the Fourier vectors f_m = e^{+i 2 pi m.n/N} / N).  On array
// indices i = n + N/2 the phase of f_m is constant per m, so
//   M^-1 v = N^-2 IDFT2( DFT2(v)[k] / (s lambda[(k + N/2) mod N] + gamma) )
// with the standard (uncentred) DFT pair; s = the mean coil power.  Three passes over the frame
// stack: row DFTs, column DFT -> divide -> column IDFT (in place, one 16-column strip per item),
// row IDFTs (scaled by N^-2) with the float64 partials of <r, z> fused.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"

namespace mrf {
namespace pc {

constexpr int kRowThreads = 128;
constexpr int SWc = 16;   // columns per strip item

template <int N>
struct Row {
  static constexpr int T = FFTShape<N>::T, P = FFTShape<N>::P, Q = FFTShape<N>::Q;
  static constexpr int RPC = kRowThreads / T;   // rows per item (a row's T threads share a warp)
  static constexpr int EX = Q * (P + 1);
};
template <int N>
constexpr size_t rows_smem() { return (size_t(N) + size_t(Row<N>::RPC) * N + size_t(Row<N>::RPC) * Row<N>::EX) * 8; }
template <int N>
constexpr int cols_threads() { return SWc * FFTShape<N>::T; }
template <int N>
constexpr size_t cols_smem() { return (size_t(N) + 2 * size_t(N) * SWc) * 8; }

// w = exp(SIGN i 2 pi e / N) for an integer e (float64 sincospi, rounded once)
template <int N, int SIGN>
__device__ __forceinline__ float2 twiddle(int e) {
  double s, c;
  sincospi(2.0 * (double)(e % N) / N, &s, &c);
  return make_float2((float)c, (float)(SIGN * s));
}

// Row DFTs of rows [0, nrows) of `in` (rows of N complex), SIGN -1 forward / +1 inverse.
// FINAL (inverse pass): out = scale * IDFT(in) and the float64 partial of <r, out> per block.
template <int N, int SIGN, bool FINAL>
__global__ void __launch_bounds__(kRowThreads) k_pc_rows(const float2* __restrict__ in, float2* __restrict__ out,
                                                         const float2* __restrict__ r, long long nrows, float scale,
                                                         double2* __restrict__ dot) {
  using R = Row<N>;
  constexpr int P = R::P, Q = R::Q, T = R::T, RPC = R::RPC, A = Q / T, B = P / T;
  extern __shared__ __align__(16) unsigned char pc_raw[];
  float2* stw = reinterpret_cast<float2*>(pc_raw);   // [k1][n2] = W_N^{SIGN n2 k1}
  float2* rows = stw + N;                             // [RPC][N]
  float2* ex = rows + RPC * N;                        // [RPC][EX]
  __shared__ double2 red[kRowThreads / 32];
  const int tid = threadIdx.x, rloc = tid / T, t = tid % T;
  for (int i = tid; i < N; i += kRowThreads) stw[i] = twiddle<N, SIGN>((i % Q) * (i / Q));
  __syncthreads();
  double2 d = make_double2(0.0, 0.0);
  const long long items = nrows / RPC;
  float2* myex = ex + rloc * R::EX;
  float2* myrow = rows + rloc * N;
  for (long long item = blockIdx.x; item < items; item += gridDim.x) {
    const size_t base = (size_t)item * RPC * N;
    const float4* src = reinterpret_cast<const float4*>(in + base);
    for (int i = tid; i < RPC * N / 2; i += kRowThreads) reinterpret_cast<float4*>(rows)[i] = __ldg(src + i);
    __syncthreads();
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
      float2 v[P];
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) v[n1] = myrow[Q * n1 + n2];
      dft<P, SIGN>(v);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) myex[n2 * (P + 1) + k1] = cmul(v[k1], stw[k1 * Q + n2]);
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      float2 w[Q];
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) w[n2] = myex[n2 * (P + 1) + k1];
      dft<Q, SIGN>(w);
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) myrow[k1 + P * k2] = FINAL ? cscale(w[k2], scale) : w[k2];
    }
    __syncthreads();
    float4* dst = reinterpret_cast<float4*>(out + base);
    const float4* rr = reinterpret_cast<const float4*>(r + base);
    for (int i = tid; i < RPC * N / 2; i += kRowThreads) {
      const float4 z = reinterpret_cast<const float4*>(rows)[i];
      dst[i] = z;
      if (FINAL) {   // Re and Im of conj(r) z
        const float4 q = __ldg(rr + i);
        d.x += ((double)q.x * z.x + (double)q.y * z.y) + ((double)q.z * z.z + (double)q.w * z.w);
        d.y += ((double)q.x * z.y - (double)q.y * z.x) + ((double)q.z * z.w - (double)q.w * z.z);
      }
    }
    __syncthreads();
  }
  if (FINAL) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d.x += __shfl_xor_sync(0xffffffffu, d.x, o);
      d.y += __shfl_xor_sync(0xffffffffu, d.y, o);
    }
    if ((tid & 31) == 0) red[tid >> 5] = d;
    __syncthreads();
    if (tid == 0) {
      double2 s = make_double2(0.0, 0.0);
      for (int i = 0; i < kRowThreads / 32; ++i) { s.x += red[i].x; s.y += red[i].y; }
      dot[blockIdx.x] = s;
    }
  }
}

// Column DFT -> divide by (s lambda + gamma) -> column IDFT, in place, one (frame, 16-column strip)
// per item.  lam: [R][N][N] float32 (interleaf-major, [my + N/2][mx + N/2]); fil: frame -> interleaf.
template <int N>
__global__ void __launch_bounds__(SWc * FFTShape<N>::T) k_pc_cols(float2* __restrict__ buf, const float* __restrict__ lam,
                                                                 const int* __restrict__ fil, int L, float lscale,
                                                                 float gamma) {
  using F = FFTShape<N>;
  constexpr int P = F::P, Q = F::Q, T = F::T, A = Q / T, B = P / T, S = N / SWc, NT = SWc * T;
  extern __shared__ __align__(16) unsigned char pc_raw[];
  float2* stw = reinterpret_cast<float2*>(pc_raw);   // [n2][k1] = W_N^{-n2 k1}
  float2* strip = stw + N;                            // [N][16]
  float2* ex = strip + N * SWc;                       // [N][16]
  const int tid = threadIdx.x, c = tid % SWc, t = tid / SWc;
  for (int i = tid; i < N; i += NT) stw[i] = twiddle<N, -1>((i / P) * (i % P));
  __syncthreads();
  for (int item = blockIdx.x; item < L * S; item += gridDim.x) {
    const int l = item / S, s = item % S;
    float2* col0 = buf + (size_t)l * N * N + (size_t)s * SWc;
    for (int i = tid; i < N * SWc / 2; i += NT) {   // 8 float4 per 128-byte row segment
      const int y = i / (SWc / 2), q = i % (SWc / 2);
      reinterpret_cast<float4*>(strip)[i] = __ldg(reinterpret_cast<const float4*>(col0 + (size_t)y * N) + q);
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < A; ++a) {   // forward stage 1 (over n1), twiddle
      const int n2 = t + T * a;
      float2 v[P];
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) v[n1] = strip[(Q * n1 + n2) * SWc + c];
      dft<P, -1>(v);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) ex[(n2 * P + k1) * SWc + c] = cmul(v[k1], stw[n2 * P + k1]);
    }
    __syncthreads();
    float2 w[B][Q];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) w[b][n2] = ex[(n2 * P + t + T * b) * SWc + c];
    __syncthreads();   // ex is rewritten below
    const float* lr = lam + (size_t)__ldg(fil + l) * N * N + (size_t)((s * SWc + c + N / 2) % N);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      dft<Q, -1>(w[b]);                                 // w[b][k2] = X[k1 + P k2]
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) {
        const float lv = __ldg(lr + (size_t)(((k1 + P * k2) + N / 2) % N) * N);
        w[b][k2] = cscale(w[b][k2], 1.f / fmaf(lscale, lv, gamma));
      }
      dft<Q, +1>(w[b]);                                 // inverse stage A: index n2
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) ex[(n2 * P + k1) * SWc + c] = cmulc(w[b][n2], stw[n2 * P + k1]);
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < A; ++a) {   // inverse stage B (over k1): index n1, row n2 + Q n1
      const int n2 = t + T * a;
      float2 u[P];
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) u[k1] = ex[(n2 * P + k1) * SWc + c];
      dft<P, +1>(u);
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) strip[(n2 + Q * n1) * SWc + c] = u[n1];
    }
    __syncthreads();
    for (int i = tid; i < N * SWc / 2; i += NT) {
      const int y = i / (SWc / 2), q = i % (SWc / 2);
      reinterpret_cast<float4*>(col0 + (size_t)y * N)[q] = reinterpret_cast<const float4*>(strip)[i];
    }
    __syncthreads();
  }
}

// F[j][m] = Fejer(k_j[axis] - (m - N/2) / N), float64 (plan time)
__global__ void k_pc_fejer(const float* __restrict__ traj, int M, int N, int axis, double* __restrict__ F) {
  const long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / N), m = (int)(i % N) - N / 2;
    const double th = (double)traj[2 * j + axis] - (double)m / N;
    const double sn = sinpi(th);
    double f;
    if (fabs(sn) < 1e-12) {
      f = (double)N * N;
    } else {
      const double q = sinpi((double)N * th) / sn;
      f = q * q;
    }
    F[i] = f;
  }
}

}  // namespace pc
}  // namespace mrf

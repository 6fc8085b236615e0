// llr.cuh -- the locally-low-rank outer step of Algorithm 1 in subspace coordinates (SURVEY.md
// §8(f) f2, the paper's LLR ablation: lambda_1 = 0).  PAPER.md:217-264:
//
//   Z   = P_S(X - mu A^*(A X - b)),  P_S(X) = X d^dagger d               (Eqs. 15, 17)
//   P_q = SVT_{1/beta}(Q_q(Z))                                            (Eq. 20)
//   X+  = (Z + gamma Q^*(P)) / (1 + gamma c),  gamma = mu lambda_2 beta    (Eq. 21, reading 25)
//
// After P_S every voxel's time series lies in span(d) (d: r x L, orthonormal rows), so with the
// coefficients Y = Z d^dagger (V x r) a patch Casorati matrix is Q_q(Z) = Y_q d and
// SVT(Q_q(Z)) = SVT(Y_q) d = Y_q W diag(max(1 - tau / sigma, 0)) W^H d with Y_q^H Y_q = W S^2 W^H:
// the p^2 x L SVD becomes an r x r Hermitian eigenproblem per patch (r = 13 for the MRF
// dictionary at 0.9999 energy), solved by cyclic complex Jacobi (float64) in one warp.
//
//   k_llr_coef   : Y[v][i] = sum_l conj(d[i][l]) (x - mu (n - rhs))[l][v]   (reads 3 image arrays)
//   k_llr_svt    : per patch: Gram, Jacobi, M = W f W^H, P_q = Y_q M, sum sigma (nuclear norm)
//   k_llr_update : per voxel: sum of its covering patches' P (fixed order), the Eq. 21 division,
//                  x+[l][v] = sum_i Xc[i] d[i][l]
#pragma once
#include <cuda_runtime.h>

#include "fft.cuh"   // cadd / cmul helpers

namespace mrf {
namespace llr {

constexpr int RMAX = 32;      // largest supported subspace rank
constexpr int kSvtThreads = 128;

__device__ __forceinline__ float2 cconjmul(float2 a, float2 b) {   // conj(a) * b
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.x, b.y, -a.y * b.x));
}

// Y[v][i] for i < r, v < V.  d: [r][L] complex (orthonormal rows).  One thread per voxel;
// R = compile-time bound on r (16 or 32).
template <int R>
__global__ void __launch_bounds__(256) k_llr_coef(const float2* __restrict__ x, const float2* __restrict__ nx,
                                                  const float2* __restrict__ rhs, const float2* __restrict__ d,
                                                  int r, int L, int V, float mu, float2* __restrict__ Y) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  float2 acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = make_float2(0.f, 0.f);
  for (int l = 0; l < L; ++l) {
    const size_t o = (size_t)l * V + v;
    const float2 a = __ldg(x + o), n = __ldg(nx + o), b = __ldg(rhs + o);
    const float2 w = make_float2(a.x - mu * (n.x - b.x), a.y - mu * (n.y - b.y));
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (i < r) {
        const float2 di = __ldg(d + (size_t)i * L + l);   // same address across the warp: broadcast
        const float2 t = cconjmul(di, w);
        acc[i].x += t.x;
        acc[i].y += t.y;
      }
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (i < r) Y[(size_t)v * r + i] = acc[i];
}

// One patch per block.  corners: [nc] top-left coordinates (same list for rows and columns);
// patch q = (qy, qx) with qy, qx < nc.  P: [nq][p*p][r] output coefficients; nuc: [nq] sum sigma.
static __global__ void __launch_bounds__(kSvtThreads) k_llr_svt(const float2* __restrict__ Y, const int* __restrict__ corners,
                                                          int nc, int N, int p, int r, float tau,
                                                          float2* __restrict__ P, double* __restrict__ nuc) {
  extern __shared__ __align__(16) unsigned char llr_raw[];
  double2* H = reinterpret_cast<double2*>(llr_raw);     // [r][r] Gram, then Jacobi working copy (float64)
  double2* Wm = H + RMAX * RMAX;                        // [r][r] eigenvectors (columns)
  float2* Mm = reinterpret_cast<float2*>(Wm + RMAX * RMAX);   // [r][r] W f W^H
  float2* Yq = Mm + RMAX * RMAX;                        // [p*p][r]
  __shared__ double fw[RMAX];
  const int q = blockIdx.x, qy = q / nc, qx = q % nc;
  const int y0 = corners[qy], x0 = corners[qx];
  const int np = p * p, tid = threadIdx.x;
  for (int e = tid; e < np * r; e += blockDim.x) {
    const int k = e / r, i = e % r;
    const int vy = y0 + k / p, vx = x0 + k % p;
    Yq[e] = Y[((size_t)vy * N + vx) * r + i];
  }
  __syncthreads();
  // Gram H = Yq^H Yq (r x r), float64 (the eigenvalues are squared singular values: float32
  // would put an absolute error ~1e-7 lambda_max on them, i.e. ~3e-4 sigma_max on the small sigma)
  for (int e = tid; e < r * r; e += blockDim.x) {
    const int i = e / r, j = e % r;
    double sx = 0.0, sy = 0.0;
    for (int k = 0; k < np; ++k) {
      const float2 a = Yq[k * r + i], b = Yq[k * r + j];
      sx += (double)a.x * b.x + (double)a.y * b.y;
      sy += (double)a.x * b.y - (double)a.y * b.x;
    }
    H[i * RMAX + j] = make_double2(sx, sy);
    Wm[i * RMAX + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  // cyclic complex Jacobi in warp 0 (lane k owns index k): H <- U^H H U, W <- W U with
  // U = [[c, -s e^{i phi}], [s e^{-i phi}, c]] on (p, q), phi = arg H[p][q], cot 2theta = (a - b) / 2|H_pq|
  if (tid < 32) {
    const int k = tid;
    auto mul = [](double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); };
    for (int sweep = 0; sweep < 30; ++sweep) {
      double off = 0.0, tot = 0.0;
      for (int e = k; e < r * r; e += 32) {
        const double2 h = H[(e / r) * RMAX + e % r];
        const double m2 = h.x * h.x + h.y * h.y;
        tot += m2;
        if (e / r != e % r) off += m2;
      }
      for (int o = 16; o > 0; o >>= 1) {
        off += __shfl_xor_sync(0xffffffffu, off, o);
        tot += __shfl_xor_sync(0xffffffffu, tot, o);
      }
      if (!(off > 1e-26 * tot)) break;
      for (int pp = 0; pp < r - 1; ++pp)
        for (int qq = pp + 1; qq < r; ++qq) {
          const double2 hpq = H[pp * RMAX + qq];
          const double mag = sqrt(hpq.x * hpq.x + hpq.y * hpq.y);
          if (!(mag > 1e-300)) continue;
          const double a = H[pp * RMAX + pp].x, b = H[qq * RMAX + qq].x;
          const double kap = (a - b) / (2.0 * mag);
          const double t = (kap >= 0.0 ? 1.0 : -1.0) / (fabs(kap) + sqrt(1.0 + kap * kap));
          const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
          const double2 e = make_double2(hpq.x / mag, hpq.y / mag);   // e^{i phi}
          const double2 ec = make_double2(e.x, -e.y);
          __syncwarp();
          if (k < r) {   // columns: H[:,p]' = H[:,p] c + H[:,q] s e^{-i phi};  H[:,q]' = -H[:,p] s e^{i phi} + H[:,q] c
            const double2 hp = H[k * RMAX + pp], hq = H[k * RMAX + qq];
            const double2 a1 = mul(hq, ec), a2 = mul(hp, e);
            H[k * RMAX + pp] = make_double2(c * hp.x + s * a1.x, c * hp.y + s * a1.y);
            H[k * RMAX + qq] = make_double2(c * hq.x - s * a2.x, c * hq.y - s * a2.y);
            const double2 wp = Wm[k * RMAX + pp], wq = Wm[k * RMAX + qq];
            const double2 b1 = mul(wq, ec), b2 = mul(wp, e);
            Wm[k * RMAX + pp] = make_double2(c * wp.x + s * b1.x, c * wp.y + s * b1.y);
            Wm[k * RMAX + qq] = make_double2(c * wq.x - s * b2.x, c * wq.y - s * b2.y);
          }
          __syncwarp();
          if (k < r) {   // rows: H[p,:]'' = c H[p,:]' + s e^{i phi} H[q,:]';  H[q,:]'' = -s e^{-i phi} H[p,:]' + c H[q,:]'
            const double2 rp = H[pp * RMAX + k], rq = H[qq * RMAX + k];
            const double2 a1 = mul(rq, e), a2 = mul(rp, ec);
            H[pp * RMAX + k] = make_double2(c * rp.x + s * a1.x, c * rp.y + s * a1.y);
            H[qq * RMAX + k] = make_double2(c * rq.x - s * a2.x, c * rq.y - s * a2.y);
          }
          __syncwarp();
        }
    }
    // f(lambda) = max(1 - tau / sqrt(lambda), 0); nuclear norm = sum sqrt(lambda)
    double sig = 0.0;
    if (k < r) {
      sig = sqrt(fmax(H[k * RMAX + k].x, 0.0));
      fw[k] = sig > (double)tau ? 1.0 - (double)tau / sig : 0.0;
    }
    for (int o = 16; o > 0; o >>= 1) sig += __shfl_xor_sync(0xffffffffu, sig, o);
    if (k == 0) nuc[q] = sig;
  }
  __syncthreads();
  // M = W diag(f) W^H
  for (int e = tid; e < r * r; e += blockDim.x) {
    const int i = e / r, j = e % r;
    double mx = 0.0, my = 0.0;
    for (int t = 0; t < r; ++t) {
      const double2 wi = Wm[i * RMAX + t], wj = Wm[j * RMAX + t];   // W[i][t] conj(W[j][t])
      mx += fw[t] * (wi.x * wj.x + wi.y * wj.y);
      my += fw[t] * (wi.y * wj.x - wi.x * wj.y);
    }
    Mm[i * RMAX + j] = make_float2((float)mx, (float)my);
  }
  __syncthreads();
  // P_q = Yq M
  float2* Pq = P + (size_t)q * np * r;
  for (int e = tid; e < np * r; e += blockDim.x) {
    const int k = e / r, j = e % r;
    float2 acc = make_float2(0.f, 0.f);
    for (int t = 0; t < r; ++t) {
      const float2 pr = cmul(Yq[k * r + t], Mm[t * RMAX + j]);
      acc.x += pr.x;
      acc.y += pr.y;
    }
    Pq[e] = acc;
  }
}

// Per voxel: Xc = (Y + gamma sum_{q covering v} P_q[v]) / (1 + gamma c(v)), then
// x+[l][v] = sum_i Xc[i] d[i][l].  Covering patches are visited in increasing (qy, qx) order.
template <int R>
__global__ void __launch_bounds__(256) k_llr_update(const float2* __restrict__ Y, const float2* __restrict__ P,
                                                    const int* __restrict__ corners, int nc, int N, int p, int r,
                                                    const float2* __restrict__ d, int L, float gamma,
                                                    float2* __restrict__ xout) {
  const int V = N * N;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int vy = v / N, vx = v % N;
  float2 xc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) xc[i] = make_float2(0.f, 0.f);
  int cnt = 0;
  for (int qy = 0; qy < nc; ++qy) {
    const int cy = __ldg(corners + qy);
    if (vy < cy || vy >= cy + p) continue;
    for (int qx = 0; qx < nc; ++qx) {
      const int cx = __ldg(corners + qx);
      if (vx < cx || vx >= cx + p) continue;
      const float2* pv = P + (((size_t)(qy * nc + qx) * p + (vy - cy)) * p + (vx - cx)) * r;
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (i < r) {
          const float2 t = __ldg(pv + i);
          xc[i].x += t.x;
          xc[i].y += t.y;
        }
      ++cnt;
    }
  }
  const float inv = 1.f / (1.f + gamma * (float)cnt);
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (i < r) {
      const float2 y = __ldg(Y + (size_t)v * r + i);
      xc[i] = make_float2((y.x + gamma * xc[i].x) * inv, (y.y + gamma * xc[i].y) * inv);
    }
  for (int l = 0; l < L; ++l) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (i < r) {
        const float2 t = cmul(xc[i], __ldg(d + (size_t)i * L + l));
        acc.x += t.x;
        acc.y += t.y;
      }
    xout[(size_t)l * V + v] = acc;
  }
}

// ---- basis of the dictionary subspace (creation time): complex GEMM with double accumulation,
// C(m, n) = sum_t A(m, t) B(t, n), A(m, t) = [conj] a[m*sam + t*sat], B(t, n) = b[t*sbt + n*sbn].
static __global__ void k_cgemm(const float2* __restrict__ a, long long sam, long long sat, int conj_a,
                        const float2* __restrict__ b, long long sbt, long long sbn, int M, int Nn, int T,
                        float2* __restrict__ c, double2* __restrict__ c64) {
  __shared__ float2 As[16][17], Bs[16][17];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int m = blockIdx.y * 16 + ty, n = blockIdx.x * 16 + tx;
  double sx = 0.0, sy = 0.0;
  for (int t0 = 0; t0 < T; t0 += 16) {
    const int ma = blockIdx.y * 16 + ty, ta = t0 + tx;
    float2 va = make_float2(0.f, 0.f);
    if (ma < M && ta < T) va = a[ma * sam + ta * sat];
    if (conj_a) va.y = -va.y;
    As[ty][tx] = va;
    const int tb = t0 + ty, nb = blockIdx.x * 16 + tx;
    Bs[ty][tx] = (tb < T && nb < Nn) ? b[tb * sbt + nb * sbn] : make_float2(0.f, 0.f);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float2 x = As[ty][k], y = Bs[k][tx];
      sx += (double)x.x * y.x - (double)x.y * y.y;
      sy += (double)x.x * y.y + (double)x.y * y.x;
    }
    __syncthreads();
  }
  if (m < M && n < Nn) {
    if (c) c[(size_t)m * Nn + n] = make_float2((float)sx, (float)sy);
    if (c64) c64[(size_t)m * Nn + n] = make_double2(sx, sy);
  }
}

}  // namespace llr
}  // namespace mrf

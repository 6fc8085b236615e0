// llr.cuh -- the (MS-)LLR outer step of Algorithm 1 in subspace coordinates.
// PAPER.md:217-264:
//
//   Z   = P_S(X - mu [A^*(A X - b) + lambda_1 Q^*(Q(X) L)]),  P_S(X) = X d^dagger d   (Eqs. 15, 17)
//   P_q = SVT_{1/beta}(Q_q(Z))                                            (Eq. 20)
//   X+  = (Z + gamma Q^*(P)) / (1 + gamma c),  gamma = mu lambda_2 beta    (Eq. 21, reading 25)
//
// After P_S every voxel's time series lies in span(d) (d: r x L, orthonormal rows), so with the
// coefficients Y = Z d^dagger (V x r) a patch Casorati matrix is Q_q(Z) = Y_q d and
// SVT(Q_q(Z)) = SVT(Y_q) d = Y_q W diag(max(1 - tau / sigma, 0)) W^H d with Y_q^H Y_q = W S^2 W^H:
// the p^2 x L SVD becomes an r x r Hermitian eigenproblem per patch (r = 13 for the MRF
// dictionary at 0.9999 energy), solved by a float64 Jacobi on the Gram matrix in one warp.
//
//   k_llr_coef   : Y[v][i] = sum_l conj(d[i][l]) (x - mu (n - rhs))[l][v]   (reads 3 image arrays)
//   k_llr_svt    : per patch: Gram, Jacobi, M = W f W^H, P_q = Y_q M, sum sigma (nuclear norm)
//   k_llr_update : per voxel: sum of its covering patches' P (fixed order), the Eq. 21 division,
//                  the coefficients Xc of x+ and (optionally) x+[l][v] = sum_i Xc[i] d[i][l]
//   k_sn_grad, k_llr_resid, k_llr_dotre : the basis-coordinate gradient and float64 reductions
//   mfd::*       : the manifold term (Eqs. 7-11): foreground statistics, patch distances, the
//                  radix-select median bandwidth, weights and degrees, Q(x) blocks, the update
//                  with deg Q - W Q, the trace penalty (W Q itself: gemm3.cuh)
#pragma once
#include <cuda_runtime.h>

#include "fft.cuh"   // cadd / cmul helpers

namespace mrf {
namespace llr {

constexpr int RMAX = 32;      // largest supported subspace rank
constexpr int kSvtThreads = 128;   // 4 patches (one warp each) per block

__device__ __forceinline__ float2 cconjmul(float2 a, float2 b) {   // conj(a) * b
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.x, b.y, -a.y * b.x));
}

// Y[v][i] for i < r, v < V.  dT: [L][R] complex transpose of d (rows padded to R with zeros), so
// one frame's R coefficients are R/2 16-byte loads, broadcast across a warp.  Block = 32 voxels
// (lanes) x NG warps; warp w sums the frames l = w (mod NG), the NG partial sums are added in a
// fixed order through shared memory.
template <int R>
__host__ __device__ constexpr int coef_groups() { return R <= 16 ? 8 : 4; }   // frame groups (warps) per block
template <int R, bool WX>
__global__ void __launch_bounds__(32 * coef_groups<R>()) k_llr_coef(const float2* __restrict__ x, const float2* __restrict__ nx,
                                                  const float2* __restrict__ rhs, const float2* __restrict__ dT,
                                                  int r, int L, int V, float mu, float2* __restrict__ Y,
                                                  float2* __restrict__ YX) {
  // WX: also the coefficients of x itself, YX = x d^dagger (the manifold term uses Q(P_S x))
  constexpr int NG = coef_groups<R>();
  __shared__ float2 part[NG][R][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int v = blockIdx.x * 32 + lane;
  float2 acc[R], accx[WX ? R : 1];
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < (WX ? R : 1); ++i) accx[i] = make_float2(0.f, 0.f);
  const float4* d4 = reinterpret_cast<const float4*>(dT);
  if (v < V)
    for (int l = w; l < L; l += NG) {
      const size_t o = (size_t)l * V + v;
      const float2 a = __ldg(x + o), n = __ldg(nx + o), b = __ldg(rhs + o);
      const float2 wv = make_float2(a.x - mu * (n.x - b.x), a.y - mu * (n.y - b.y));
#pragma unroll
      for (int i2 = 0; i2 < R / 2; ++i2) {
        const float4 dd = __ldg(d4 + (size_t)l * (R / 2) + i2);
        const float2 d0 = make_float2(dd.x, dd.y), d1 = make_float2(dd.z, dd.w);
        const float2 t0 = cconjmul(d0, wv), t1 = cconjmul(d1, wv);
        acc[2 * i2].x += t0.x; acc[2 * i2].y += t0.y;
        acc[2 * i2 + 1].x += t1.x; acc[2 * i2 + 1].y += t1.y;
        if constexpr (WX) {
          const float2 u0 = cconjmul(d0, a), u1 = cconjmul(d1, a);
          accx[2 * i2].x += u0.x; accx[2 * i2].y += u0.y;
          accx[2 * i2 + 1].x += u1.x; accx[2 * i2 + 1].y += u1.y;
        }
      }
    }
  for (int pass = 0; pass < (WX ? 2 : 1); ++pass) {
    if (pass) __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) part[w][i][lane] = pass ? accx[WX ? i : 0] : acc[i];
    __syncthreads();
    float2* out = pass ? YX : Y;
    for (int e = threadIdx.x; e < 32 * r; e += blockDim.x) {
      const int i = e / 32, ln = e % 32;
      const int vv = blockIdx.x * 32 + ln;
      float2 t = make_float2(0.f, 0.f);
#pragma unroll
      for (int g = 0; g < NG; ++g) { t.x += part[g][i][ln].x; t.y += part[g][i][ln].y; }
      if (vv < V) out[(size_t)vv * r + i] = t;
    }
  }
}

// One patch per warp, kSvtThreads / 32 patches per block.  corners: [nc] top-left coordinates
// (same list for rows and columns); patch q = (qy, qx).  P: [nq][p*p][r] output coefficients;
// nuc: [nq] sum sigma.  SVT(Y_q) = Y_q W diag(max(1 - tau / sigma, 0)) W^H with the Hermitian
// eigendecomposition Y_q^H Y_q = W S^2 W^H:
//   1. the r x r Gram matrix in float64 (products of float32 are exact in float64, so the small
//      eigenvalues keep an absolute error ~1e-16 ||Y_q||_F^2 -- far below tau^2);
//   2. cyclic parallel Jacobi in float64: each round applies rp / 2 disjoint rotations (round-robin
//      pairing, rp = r rounded up to even), all rows then all columns, lanes striding the entries;
//   3. M = W F W^H (float64 -> float32), P_q = Y_q M.
// Shared memory per warp: svt_warp_bytes(r).
__host__ __device__ constexpr int svt_rp(int r) { return (r + 1) & ~1; }
__host__ __device__ constexpr size_t svt_warp_bytes(int r) {
  return (size_t)2 * svt_rp(r) * svt_rp(r) * 16 + (size_t)svt_rp(r) / 2 * 32 + ((size_t)r * r * 8 + 15) / 16 * 16;
}

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

static __global__ void __launch_bounds__(kSvtThreads) k_llr_svt(const float2* __restrict__ Y, const int* __restrict__ corners,
                                                          int nc, int N, int p, int r, float tau, int nq,
                                                          float2* __restrict__ P, double* __restrict__ nuc) {
  // P == nullptr: singular values only (eigenvalues of the Gram matrix, no eigenvectors).
  // (A warm start from cached eigenvectors of the previous iteration was measured: it does not
  // reduce the sweeps inside the MS-LLR loop.)
  extern __shared__ __align__(16) unsigned char llr_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * (kSvtThreads / 32) + warp;
  if (q >= nq) return;   // warp-uniform
  const int rp = svt_rp(r), half = rp / 2;
  const bool vecs = P != nullptr;   // eigenvectors needed
  double2* A = reinterpret_cast<double2*>(llr_raw + (size_t)warp * svt_warp_bytes(r));   // [rp][rp]
  double2* Wm = A + rp * rp;                                                             // [rp][rp]
  double4* rot = reinterpret_cast<double4*>(Wm + rp * rp);                               // [half] (c, s, e)
  float2* M = reinterpret_cast<float2*>(rot + half);                                     // [r][r]
  const int qy = q / nc, qx = q % nc;
  const int y0 = corners[qy], x0 = corners[qx];
  const int np = p * p;
  const float2* Yb = Y + ((size_t)y0 * N + x0) * r;   // row k of Y_q: Yb + ((k / p) * N + k % p) * r
  // 1. Gram G[i][j] = sum_k conj(Y[k][i]) Y[k][j], upper triangle entries strided over the lanes
  double tr = 0.0;
  for (int e = lane; e < r * (r + 1) / 2; e += 32) {
    int i = 0, rem = e;
    while (rem >= r - i) { rem -= r - i; ++i; }
    const int j = i + rem;
    double gx = 0.0, gy = 0.0;
    for (int yy = 0; yy < p; ++yy) {
      const float2* row = Yb + (size_t)yy * N * r;
      for (int xx = 0; xx < p; ++xx, row += r) {
        const float2 a = __ldg(row + i), b = __ldg(row + j);
        gx = fma((double)a.x, (double)b.x, fma((double)a.y, (double)b.y, gx));
        gy = fma((double)a.x, (double)b.y, fma(-(double)a.y, (double)b.x, gy));
      }
    }
    A[i * rp + j] = make_double2(gx, gy);
    A[j * rp + i] = make_double2(gx, -gy);
    if (i == j) tr += gx;
  }
  for (int e = lane; e < rp * rp; e += 32) {
    const int i = e / rp, j = e % rp;
    if (i >= r || j >= r) A[e] = make_double2(0.0, 0.0);   // padding row / column of odd r
    Wm[e] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
  // |g| <= 1e-14 tr is zero at the scale of ||Y_q||_F^2: the eigenvalues then carry an absolute
  // error <= ~1e-14 ||Y_q||_F^2, and M = W F W^H an error ~1e-14 ||Y_q||_F^2 / tau^2
  const double floor_g = 1e-14 * tr;
  // lane = (group g, index c): groups of w = 16 lanes (rp <= 16) or one group of 32
  const int w = rp <= 16 ? 16 : 32, G = 32 / w, g = lane / w, c = lane % w;
  int2* pr = reinterpret_cast<int2*>(M);   // round's pairs (M is free until step 3)
  __syncwarp();
  // 2. cyclic Jacobi, round-robin pairs: round t, slot k: (t, rp-1) for k = 0, else
  //    ((t + k) mod (rp-1), (t - k) mod (rp-1))
  for (int sweep = 0; sweep < 30; ++sweep) {
    bool rotated = false;
    for (int t = 0; t < rp - 1; ++t) {
      if (lane < half) {
        int a = lane ? (t + lane) % (rp - 1) : t, b = lane ? (t - lane + rp - 1) % (rp - 1) : rp - 1;
        if (a > b) { const int u = a; a = b; b = u; }
        double4 R = make_double4(1.0, 0.0, 1.0, 0.0);
        if (b < r) {
          const double al = A[a * rp + a].x, be = A[b * rp + b].x;
          const double2 gg = A[a * rp + b];
          const double g2 = gg.x * gg.x + gg.y * gg.y;
          if (g2 > floor_g * floor_g) {
            // A <- J^H A J with J = [[c, -s e], [s conj(e), c]] on (a, b), e = g / |g|:
            // cot 2theta = (al - be) / 2|g| zeroes the (a, b) entry.  rsqrt (1 ulp) instead of
            // sqrt + divisions: |e| and c^2 (1 + t^2) equal 1 to float64 rounding either way,
            // so J stays unitary; t only sets the angle.
            const double inv = rsqrt(g2);
            const double kap = (al - be) * (0.5 * inv);
            const double tt = (kap >= 0.0 ? 1.0 : -1.0) / (fabs(kap) + sqrt(1.0 + kap * kap));
            const double cs = rsqrt(1.0 + tt * tt);
            R = make_double4(cs, tt * cs, gg.x * inv, gg.y * inv);
          }
        }
        rot[lane] = R;
        pr[lane] = make_int2(a, b);
        rotated |= R.y != 0.0;
      }
      rotated = __any_sync(0xffffffffu, rotated);
      __syncwarp();
      if (vecs) {
        // with eigenvectors (measured faster this way): rows a, b of A,
        // A[a][k] <- c A[a][k] + s e A[b][k],  A[b][k] <- c A[b][k] - s conj(e) A[a][k], then columns
        // a, b of A and of W: X[k][a] <- c X[k][a] + s conj(e) X[k][b], X[k][b] <- c X[k][b] - s e X[k][a]
        for (int k = g; k < half; k += G) {
          const double4 R = rot[k];
          if (R.y == 0.0 || c >= r) continue;
          const int2 ab = pr[k];
          const double2 x = A[ab.x * rp + c], y = A[ab.y * rp + c];
          const double2 ey = zmul(make_double2(R.z, R.w), y), ecx = zmul(make_double2(R.z, -R.w), x);
          A[ab.x * rp + c] = make_double2(R.x * x.x + R.y * ey.x, R.x * x.y + R.y * ey.y);
          A[ab.y * rp + c] = make_double2(R.x * y.x - R.y * ecx.x, R.x * y.y - R.y * ecx.y);
        }
        __syncwarp();
        for (int mk = g; mk < 2 * half; mk += G) {
          const double4 R = rot[mk >> 1];
          if (R.y == 0.0 || c >= r) continue;
          const int2 ab = pr[mk >> 1];
          double2* X = (mk & 1) ? Wm : A;
          const double2 x = X[c * rp + ab.x], y = X[c * rp + ab.y];
          const double2 ecy = zmul(make_double2(R.z, -R.w), y), ex = zmul(make_double2(R.z, R.w), x);
          X[c * rp + ab.x] = make_double2(R.x * x.x + R.y * ecy.x, R.x * x.y + R.y * ecy.y);
          X[c * rp + ab.y] = make_double2(R.x * y.x - R.y * ex.x, R.x * y.y - R.y * ex.y);
        }
      } else {
        // eigenvalues only: A <- J^H A J in one pass over the 2 x 2 blocks (pair k1 of rows, pair k2
        // of columns); every entry belongs to exactly one block, whose new value depends only on its
        // own 4 entries
        const int nblk = half * half;
        for (int it = lane; it < nblk; it += 32) {   // A blocks
          {
            const int k1 = it / half, k2 = it - k1 * half;
            const double4 R1 = rot[k1], R2 = rot[k2];
            if (R1.y == 0.0 && R2.y == 0.0) continue;
            const int2 p1 = pr[k1], p2 = pr[k2];
            double2 x00 = A[p1.x * rp + p2.x], x01 = A[p1.x * rp + p2.y];
            double2 x10 = A[p1.y * rp + p2.x], x11 = A[p1.y * rp + p2.y];
            if (R1.y != 0.0) {
              const double2 e = make_double2(R1.z, R1.w), ec = make_double2(R1.z, -R1.w);
              const double2 e10 = zmul(e, x10), e11 = zmul(e, x11), c00 = zmul(ec, x00), c01 = zmul(ec, x01);
              const double2 n00 = make_double2(R1.x * x00.x + R1.y * e10.x, R1.x * x00.y + R1.y * e10.y);
              const double2 n01 = make_double2(R1.x * x01.x + R1.y * e11.x, R1.x * x01.y + R1.y * e11.y);
              x10 = make_double2(R1.x * x10.x - R1.y * c00.x, R1.x * x10.y - R1.y * c00.y);
              x11 = make_double2(R1.x * x11.x - R1.y * c01.x, R1.x * x11.y - R1.y * c01.y);
              x00 = n00;
              x01 = n01;
            }
            if (R2.y != 0.0) {
              const double2 e = make_double2(R2.z, R2.w), ec = make_double2(R2.z, -R2.w);
              const double2 c01 = zmul(ec, x01), c11 = zmul(ec, x11), e00 = zmul(e, x00), e10 = zmul(e, x10);
              const double2 n00 = make_double2(R2.x * x00.x + R2.y * c01.x, R2.x * x00.y + R2.y * c01.y);
              const double2 n10 = make_double2(R2.x * x10.x + R2.y * c11.x, R2.x * x10.y + R2.y * c11.y);
              x01 = make_double2(R2.x * x01.x - R2.y * e00.x, R2.x * x01.y - R2.y * e00.y);
              x11 = make_double2(R2.x * x11.x - R2.y * e10.x, R2.x * x11.y - R2.y * e10.y);
              x00 = n00;
              x10 = n10;
            }
            A[p1.x * rp + p2.x] = x00;
            A[p1.x * rp + p2.y] = x01;
            A[p1.y * rp + p2.x] = x10;
            A[p1.y * rp + p2.y] = x11;
          }
        }
      }
      __syncwarp();
    }
    if (!rotated) break;
    // converged if no off-diagonal entry is above the floor: the next sweep would rotate nothing
    // (one parallel scan instead of a sweep of no-op rounds)
    bool big = false;
    for (int e = lane; e < r * r; e += 32) {
      const int i = e / r, j = e % r;
      if (i < j) {
        const double2 v = A[i * rp + j];
        big |= v.x * v.x + v.y * v.y > floor_g * floor_g;
      }
    }
    if (!__any_sync(0xffffffffu, big)) break;
  }
  // sigma_j = sqrt(lambda_j); f_j = max(1 - tau / sigma_j, 0) (kept in the rot scratch)
  double* f = reinterpret_cast<double*>(rot);
  double sig = 0.0;
  for (int j = 0; j < r; ++j) {
    const double sj = sqrt(fmax(A[j * rp + j].x, 0.0));
    sig += sj;
    if (lane == 0) f[j] = sj > (double)tau ? 1.0 - (double)tau / sj : 0.0;
  }
  if (lane == 0) nuc[q] = sig;
  if (!P) return;   // singular values only (the cost's nuclear norms)
  __syncwarp();
  // 3. M = W F W^H
  for (int e = lane; e < r * r; e += 32) {
    const int a = e / r, b = e % r;
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < r; ++j) {
      const double2 wa = Wm[a * rp + j], wb = Wm[b * rp + j];
      const double2 t = zmul(wa, make_double2(wb.x, -wb.y));
      acc.x = fma(f[j], t.x, acc.x);
      acc.y = fma(f[j], t.y, acc.y);
    }
    M[e] = make_float2((float)acc.x, (float)acc.y);
  }
  __syncwarp();
  // P_q = Y_q M:  P[k][j'] = sum_j Y[k][j] M[j][j'];  lane = (row group g, column c)
  float2* Pq = P + (size_t)q * np * r;
  for (int kk = g; kk < np; kk += G) {
    if (c >= r) continue;
    const float2* row = Yb + ((size_t)(kk / p) * N + kk % p) * r;
    float2 acc = make_float2(0.f, 0.f);
    for (int j = 0; j < r; ++j) {
      const float2 t = cmul(__ldg(row + j), M[j * r + c]);
      acc.x += t.x;
      acc.y += t.y;
    }
    Pq[kk * r + c] = acc;
  }
}

// Per voxel: Xc = (Y + gamma sum_{q covering v} P_q[v]) / (1 + gamma c(v)), then
// x+[l][v] = sum_i Xc[i] d[i][l] (dT [L][R] as for k_llr_coef).  Covering patches are visited
// in increasing (qy, qx) order.
template <int R>
__global__ void __launch_bounds__(256) k_llr_update(const float2* __restrict__ Y, const float2* __restrict__ P,
                                                    const int* __restrict__ corners, int nc, int N, int p, int r,
                                                    const float2* __restrict__ dT, int L, float gamma,
                                                    float2* __restrict__ xout, float2* __restrict__ xcv,
                                                    float2* __restrict__ xcr, int lit) {
  // xcv [V][r] / xcr [r][V] (nullable): the coefficients Xc of x+ in both layouts (x+ = Xc d
  // lies in span(d): the next step's manifold term, the cost and Phi_D read them instead of x+)
  __shared__ float2 xcs[R][33];
  const int V = N * N;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int v = blockIdx.x * 32 + lane;
  if (w == 0) {   // Xc of the block's 32 voxels
    float2 xc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) xc[i] = make_float2(0.f, 0.f);
    if (v < V) {
      const int vy = v / N, vx = v % N;
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
      const float inv = 1.f / (1.f + gamma * (lit ? 1.f : (float)cnt));   // lit: Eq. (23) as printed
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (i < r) {
          const float2 y = __ldg(Y + (size_t)v * r + i);
          xc[i] = make_float2((y.x + gamma * xc[i].x) * inv, (y.y + gamma * xc[i].y) * inv);
        }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) xcs[i][lane] = xc[i];
    if (xcv && v < V)
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (i < r) xcv[(size_t)v * r + i] = xc[i];
  }
  __syncthreads();
  if (xcr && v < V)
    for (int i = w; i < r; i += 8) xcr[(size_t)i * V + v] = xcs[i][lane];
  if (v >= V || !xout) return;   // xout == nullptr: coefficients only (basis-coordinate loop)
  float2 xc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) xc[i] = xcs[i][lane];
  const float4* d4 = reinterpret_cast<const float4*>(dT);
  for (int l = w; l < L; l += 8) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int i2 = 0; i2 < R / 2; ++i2) {   // padded entries of dT are zero
      const float4 dd = __ldg(d4 + (size_t)l * (R / 2) + i2);
      const float2 t0 = cmul(xc[2 * i2], make_float2(dd.x, dd.y)), t1 = cmul(xc[2 * i2 + 1], make_float2(dd.z, dd.w));
      acc.x += t0.x + t1.x;
      acc.y += t0.y + t1.y;
    }
    xout[(size_t)l * V + v] = acc;
  }
}

// Coefficient-only Eq. 21 update (basis-coordinate loop): thread = (voxel v, coefficient i),
// xc = (Y + gamma sum_{q covering v} P_q[v]) / (1 + gamma c(v)) with the covering patches in
// increasing (qy, qx) order (the same arithmetic as k_llr_update); writes xcv [V][r] and xcr [r][V].
static __global__ void __launch_bounds__(256) k_llr_update_coef(const float2* __restrict__ Y,
                                                                const float2* __restrict__ P,
                                                                const int* __restrict__ corners, int nc, int N, int p,
                                                                int r, float gamma, float2* __restrict__ xcv,
                                                                float2* __restrict__ xcr, int lit) {
  const int V = N * N;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)V * r) return;
  const int v = (int)(t / r), i = (int)(t % r);
  const int vy = v / N, vx = v % N;
  float2 acc = make_float2(0.f, 0.f);
  int cnt = 0;
  for (int qy = 0; qy < nc; ++qy) {
    const int cy = __ldg(corners + qy);
    if (vy < cy || vy >= cy + p) continue;
    for (int qx = 0; qx < nc; ++qx) {
      const int cx = __ldg(corners + qx);
      if (vx < cx || vx >= cx + p) continue;
      const float2 u = __ldg(P + (((size_t)(qy * nc + qx) * p + (vy - cy)) * p + (vx - cx)) * r + i);
      acc.x += u.x;
      acc.y += u.y;
      ++cnt;
    }
  }
  const float inv = 1.f / (1.f + gamma * (lit ? 1.f : (float)cnt));   // lit: Eq. (23) as printed
  const float2 y = __ldg(Y + t);
  const float2 xc = make_float2((y.x + gamma * acc.x) * inv, (y.y + gamma * acc.y) * inv);
  xcv[t] = xc;
  xcr[(size_t)i * V + v] = xc;
}

// part[block] = sum |a - b|^2 over a grid-stride slice (float64; fixed grid, so the partials and
// their host sum are deterministic)
static __global__ void __launch_bounds__(256) k_llr_resid(const float2* __restrict__ a, const float2* __restrict__ b,
                                                          size_t n, double* __restrict__ part) {
  double s = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 u = __ldg(a + i), v = __ldg(b + i);
    const double dx = (double)u.x - (double)v.x, dy = (double)u.y - (double)v.y;
    s = fma(dx, dx, fma(dy, dy, s));
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

// Y[v][i] = xcv[v][i] - mu (zs[i][v] - bv[v][i]): Eq. 15's gradient step in basis coordinates
// (zs = P_S A^H A x, bv = P_S A^H b coefficients; thread per voxel, coefficient-major zs reads)
static __global__ void __launch_bounds__(256) k_sn_grad(const float2* __restrict__ xcv, const float2* __restrict__ zs,
                                                        const float2* __restrict__ bv, float mu, int r, int V,
                                                        float2* __restrict__ Y) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  for (int i = 0; i < r; ++i) {
    const float2 a = xcv[(size_t)v * r + i], z = __ldg(zs + (size_t)i * V + v), b = bv[(size_t)v * r + i];
    Y[(size_t)v * r + i] = make_float2(a.x - mu * (z.x - b.x), a.y - mu * (z.y - b.y));
  }
}

// part[block] = sum Re(conj(a) b) over a grid-stride slice (float64; fixed grid)
static __global__ void __launch_bounds__(256) k_llr_dotre(const float2* __restrict__ a, const float2* __restrict__ b,
                                                          size_t n, double* __restrict__ part) {
  double s = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float2 u = __ldg(a + i), w = __ldg(b + i);
    s = fma((double)u.x, (double)w.x, fma((double)u.y, (double)w.y, s));
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
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

namespace mrf {
namespace mfd {
// ---- manifold term (Eqs. 7-11; reading 26) ----
// Parameter maps come from Phi_D: params [V][2] = (T1, T2), pd [V].

// max PD (bits of a non-negative float order like the value)
static __global__ void k_mfd_max(const float* __restrict__ pd, int V, unsigned* __restrict__ out) {
  float m = 0.f;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) m = fmaxf(m, pd[v]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// per-block (sum, sum of squares, count) of the three channels over the foreground PD > 0.1 max
static __global__ void __launch_bounds__(256) k_mfd_stats(const float* __restrict__ params, const float* __restrict__ pd,
                                                          int V, const unsigned* __restrict__ pdmax,
                                                          double* __restrict__ part) {   // [gridDim][7]
  __shared__ double red[7][8];
  const float thr = 0.1f * __uint_as_float(*pdmax);
  double a[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    const float p = pd[v];
    if (!(p > thr) && thr > 0.f) continue;
    const double c0 = params[2 * v], c1 = params[2 * v + 1], c2 = p;
    a[0] += c0; a[1] += c0 * c0; a[2] += c1; a[3] += c1 * c1; a[4] += c2; a[5] += c2 * c2; a[6] += 1.0;
  }
  for (int i = 0; i < 7; ++i) {
    double t = a[i];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) red[i][threadIdx.x >> 5] = t;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
    part[(size_t)blockIdx.x * 7 + threadIdx.x] = t;
  }
}

// Device-resident state of the Laplacian build (no host round trip until the end)
struct LapSel {
  double ms[6];                  // foreground mean / std of T1, T2, PD
  double count;                  // foreground voxels
  double sigma2;                 // bandwidth (median or given)
  unsigned long long m, k[2], c[2];
  unsigned pre[2];               // radix-select prefixes of the two middle order statistics
  unsigned maxdeg;               // float bits of max_i D_ii
  unsigned given;                // sigma2 given by the caller
};

// ms from the per-block partials of k_mfd_stats: each of the 7 sums is reduced by 32 lanes of one
// warp (fixed strided partial sums, then a fixed xor tree: deterministic), one warp per sum
// raw != 0: Eq. (8) on the raw maps (mean 0, std 1 recorded: the patch vectors are the raw values)
static __global__ void k_mfd_stats_final(const double* __restrict__ part, int nblk, LapSel* __restrict__ sel, int raw) {
  __shared__ double a[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < 7) {
    double t = 0.0;
    for (int b = lane; b < nblk; b += 32) t += part[(size_t)b * 7 + w];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) a[w] = t;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int c = threadIdx.x;
    const double cnt = a[6] > 0.0 ? a[6] : 1.0;
    const double mean = a[2 * c] / cnt, var = fmax(a[2 * c + 1] / cnt - mean * mean, 0.0);
    sel->ms[2 * c] = raw ? 0.0 : mean;
    sel->ms[2 * c + 1] = raw ? 1.0 : (var > 0.0 ? sqrt(var) : 1.0);
  }
  if (threadIdx.x == 0) {
    sel->count = a[6];
    sel->maxdeg = 0u;
  }
}

// Radix-select bookkeeping after histogram pass `pass` (one block of 256 threads, 8 bins each,
// a block-wide exclusive scan of the bin counts): pass 0 sets the ranks of the two middle values
// (numpy's median) and the 11-bit prefixes; passes 1, 2 extend them; after pass 2 sigma2 = the
// mean of the two middle values (1 if there is none).
__device__ __forceinline__ void sel_find(const unsigned* __restrict__ h, unsigned long long base,
                                         unsigned long long k, unsigned long long* c_out, unsigned* b_out,
                                         unsigned long long* scan) {
  // scan[256]: shared; returns (through the owning thread) the bin b with base + cum(<b) <= k < base + cum(<=b)
  const int t = threadIdx.x;
  unsigned long long loc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) loc += h[t * 8 + i];
  scan[t] = loc;
  __syncthreads();
  for (int off = 1; off < 256; off <<= 1) {   // inclusive Hillis-Steele scan
    const unsigned long long v = t >= off ? scan[t - off] : 0ull;
    __syncthreads();
    scan[t] += v;
    __syncthreads();
  }
  unsigned long long c = base + scan[t] - loc;   // exclusive prefix of this thread's first bin
  if (c <= k && k < c + loc) {
    unsigned b = t * 8;
    while (c + h[b] <= k) c += h[b++];
    *c_out = c;
    *b_out = b;
  }
  __syncthreads();
}

static __global__ void __launch_bounds__(256) k_mfd_select(int pass, const unsigned* __restrict__ h0,
                                                           const unsigned* __restrict__ h1, LapSel* __restrict__ sel) {
  __shared__ unsigned long long scan[256];
  if (sel->given) return;   // block-uniform
  if (pass == 0) {
    unsigned long long loc = 0;
    for (int i = threadIdx.x; i < 2048; i += 256) loc += h0[i];
    scan[threadIdx.x] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0;
      for (int i = 0; i < 256; ++i) m += scan[i];
      sel->m = m;
      if (m == 0) sel->sigma2 = 1.0;
      sel->k[0] = m ? (m - 1) / 2 : 0;
      sel->k[1] = m / 2;
    }
    __syncthreads();
    if (sel->m == 0) return;
    for (int t = 0; t < 2; ++t) sel_find(h0, 0ull, sel->k[t], &sel->c[t], &sel->pre[t], scan);
    return;
  }
  if (sel->m == 0) return;
  __shared__ unsigned bsel[2];
  for (int t = 0; t < 2; ++t) sel_find(t ? h1 : h0, sel->c[t], sel->k[t], &sel->c[t], &bsel[t], scan);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (pass == 1) {
      for (int t = 0; t < 2; ++t) sel->pre[t] = (sel->pre[t] << 11) | bsel[t];
    } else {
      const float v0 = __uint_as_float((sel->pre[0] << 10) | bsel[0]);
      const float v1 = __uint_as_float((sel->pre[1] << 10) | bsel[1]);
      sel->sigma2 = 0.5 * ((double)v0 + (double)v1);
    }
  }
}

static __global__ void k_mfd_degmax(const float* __restrict__ deg, int n, LapSel* __restrict__ sel) {
  float m = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = fmaxf(m, deg[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&sel->maxdeg, __float_as_uint(m));
}

// standardised patch vectors [n][3 p^2] (channel-major, row-major inside the patch); ms = mean, std x3
static __global__ void k_mfd_patchvec(const float* __restrict__ params, const float* __restrict__ pd,
                                      const LapSel* __restrict__ sel, const int* __restrict__ corners, int nc, int N,
                                      int p, float* __restrict__ pv) {
  const int q = blockIdx.x, y0 = corners[q / nc], x0 = corners[q % nc], np = p * p;
  const double* ms = sel->ms;
  for (int e = threadIdx.x; e < 3 * np; e += blockDim.x) {
    const int ch = e / np, k = e % np, v = (y0 + k / p) * N + x0 + k % p;
    const float raw = ch == 2 ? pd[v] : params[2 * v + ch];
    pv[(size_t)q * 3 * np + e] = (float)(((double)raw - ms[2 * ch]) / ms[2 * ch + 1]);
  }
}

// d2[i][j] = ||pv_i - pv_j||^2, 32 x 32 tiles of patch pairs
// d2[i][j] = ||pv_i - pv_j||^2 over dim components: 128 x 128 tiles of the upper triangle (the
// lower one is the mirror), 16 x 16 threads with 8 x 8 outputs each, 16-component chunks in smem.
static __global__ void __launch_bounds__(256) k_mfd_dist(const float* __restrict__ pv, int n, int dim,
                                                         float* __restrict__ d2) {
  if (blockIdx.y > blockIdx.x) return;   // lower-triangle tile: written by its mirror
  __shared__ float A[16][129], B[16][129];   // [component][row]
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = blockIdx.y * 128, j0 = blockIdx.x * 128;
  float acc[8][8] = {};
  for (int k0 = 0; k0 < dim; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 128; e += 256) {   // coalesced over the components
      const int rr = e / 16, kk = e % 16;
      A[kk][rr] = (i0 + rr < n && k0 + kk < dim) ? pv[(size_t)(i0 + rr) * dim + k0 + kk] : 0.f;
      B[kk][rr] = (j0 + rr < n && k0 + kk < dim) ? pv[(size_t)(j0 + rr) * dim + k0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) {
      float a[8], bb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = A[kk][ty + 16 * u];
        bb[u] = B[kk][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float dd = a[u] - bb[v];
          acc[u][v] = fmaf(dd, dd, acc[u][v]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
      if (i < n && j < n) d2[(size_t)i * n + j] = acc[u][v];
    }
  if (blockIdx.x == blockIdx.y) return;   // diagonal tile: the rows above already hold it
  // mirror d2[j][i]: 16 tile columns at a time transposed through shared memory (coalesced rows)
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) A[tx][ty + 16 * u] = acc[u][v];   // A[col][row]
    __syncthreads();
    for (int e = threadIdx.x; e < 16 * 128; e += 256) {
      const int cc = e / 128, rr = e % 128;
      const int j = j0 + cc + 16 * v, i = i0 + rr;
      if (i < n && j < n) d2[(size_t)j * n + i] = A[cc][rr];
    }
  }
}

// Radix select of the nonzero strict-upper-triangle d2 bits, 11 + 11 + 10 bits: pass 0 counts
// bits [31:21], pass 1 bits [20:10] of the values whose bits [31:21] equal `pre`, pass 2 bits
// [9:0] of those whose bits [31:10] equal `pre`.  Block-private shared-memory histograms (2048
// bins), merged with one global atomic per non-empty bin.
static __global__ void __launch_bounds__(256) k_mfd_hist(const float* __restrict__ d2, int n, int pass,
                                                         const unsigned* __restrict__ pre_dev,
                                                         unsigned* __restrict__ hist0, unsigned* __restrict__ hist1) {
  // pass 0: one histogram (hist0); passes 1, 2: the two middle order statistics' prefixes
  // pre_dev[0], pre_dev[1] counted together (hist0, hist1)
  __shared__ unsigned sh[2][2048];
  const unsigned pre0 = pass > 0 ? pre_dev[0] : 0u, pre1 = pass > 0 ? pre_dev[1] : 0u;
  for (int i = threadIdx.x; i < 2 * 2048; i += blockDim.x) sh[i >> 11][i & 2047] = 0u;
  __syncthreads();
  const int shift = pass == 0 ? 21 : pass == 1 ? 10 : 0;
  const unsigned mask = pass == 2 ? 0x3FFu : 0x7FFu;
  const int pshift = pass == 0 ? 32 : pass == 1 ? 21 : 10;
  for (int i = blockIdx.x; i < n; i += gridDim.x)   // row i, columns j > i (coalesced)
    for (int j = i + 1 + (int)threadIdx.x; j < n; j += blockDim.x) {
      const unsigned b = __float_as_uint(d2[(size_t)i * n + j]);
      if (b == 0u) continue;
      const unsigned bin = (b >> shift) & mask;
      if (pass == 0) {
        atomicAdd(&sh[0][bin], 1u);
      } else {
        const unsigned pb = b >> pshift;
        if (pb == pre0) atomicAdd(&sh[0][bin], 1u);
        if (pb == pre1) atomicAdd(&sh[1][bin], 1u);
      }
    }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) {
    if (sh[0][i]) atomicAdd(&hist0[i], sh[0][i]);
    if (pass > 0 && sh[1][i]) atomicAdd(&hist1[i], sh[1][i]);
  }
}

// W[i][j] = exp(-d2 / sigma2) (i != j), 0 on the diagonal; deg[i] = sum_j W[i][j] in a fixed order
static __global__ void k_mfd_weights(float* __restrict__ d2w, int n, const double* __restrict__ sigma2,
                                     float* __restrict__ deg) {
  const int i = blockIdx.x;
  const float inv_s2 = (float)(1.0 / *sigma2);
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    float w = j == i ? 0.f : expf(-d2w[(size_t)i * n + j] * inv_s2);
    d2w[(size_t)i * n + j] = w;
    s += w;
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    deg[i] = (float)t;
  }
}

// patch coefficient blocks Qm[q][k][i] = YX[voxel k of patch q][i]  ([n][p^2 r] complex)
static __global__ void k_mfd_gather(const float2* __restrict__ YX, const int* __restrict__ corners, int nc, int N, int p,
                                    int r, float2* __restrict__ Qm) {
  const int q = blockIdx.x, y0 = corners[q / nc], x0 = corners[q % nc], np = p * p;
  for (int e = threadIdx.x; e < np * r; e += blockDim.x) {
    const int k = e / r, i = e % r;
    Qm[(size_t)q * np * r + e] = YX[((size_t)(y0 + k / p) * N + x0 + k % p) * r + i];
  }
}

// Y[v] -= scale * sum_{q covering v} (deg_q Qm_q[v] - G_q[v])   (Q^*(Q(X) L) in coefficients);
// pen[q-block]: per-block partial of Re sum_q <Qm_q, deg_q Qm_q - G_q> (the trace penalty) when q0 < 0
// thread = (voxel v, coefficient i): consecutive threads read consecutive words of a patch block
// (coalesced); the covering patches are visited in increasing (qy, qx) order (deterministic).
// R is unused (kept for the launch sites' dispatch on r).
template <int R>
__global__ void __launch_bounds__(256) k_mfd_apply(float2* __restrict__ Y, const float2* __restrict__ Qm,
                                                   const float2* __restrict__ G, const float* __restrict__ deg,
                                                   const int* __restrict__ corners, int nc, int N, int p, int r,
                                                   float scale) {
  const int V = N * N;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)V * r) return;
  const int v = (int)(t / r), i = (int)(t % r);
  const int vy = v / N, vx = v % N, np = p * p;
  float2 acc = make_float2(0.f, 0.f);
  for (int qy = 0; qy < nc; ++qy) {
    const int cy = __ldg(corners + qy);
    if (vy < cy || vy >= cy + p) continue;
    for (int qx = 0; qx < nc; ++qx) {
      const int cx = __ldg(corners + qx);
      if (vx < cx || vx >= cx + p) continue;
      const int q = qy * nc + qx;
      const float dq = __ldg(deg + q);
      const size_t o = ((size_t)q * np + (size_t)(vy - cy) * p + (vx - cx)) * r + i;
      const float2 a = __ldg(Qm + o), g = __ldg(G + o);
      acc.x += dq * a.x - g.x;
      acc.y += dq * a.y - g.y;
    }
  }
  float2 y = Y[t];
  y.x -= scale * acc.x;
  y.y -= scale * acc.y;
  Y[t] = y;
}

// per-patch Re <Qm_q, deg_q Qm_q - G_q> (trace penalty terms), one block per patch, fixed order
static __global__ void k_mfd_penalty(const float2* __restrict__ Qm, const float2* __restrict__ G,
                                     const float* __restrict__ deg, int len, double* __restrict__ pen) {
  const int q = blockIdx.x;
  const float dq = deg[q];
  double s = 0.0;
  for (int e = threadIdx.x; e < len; e += blockDim.x) {
    const float2 a = Qm[(size_t)q * len + e], g = G[(size_t)q * len + e];
    s += (double)a.x * (dq * a.x - g.x) + (double)a.y * (dq * a.y - g.y);
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    pen[q] = t;
  }
}

}  // namespace mfd
}  // namespace mrf

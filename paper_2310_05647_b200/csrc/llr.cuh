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
// dictionary at 0.9999 energy), solved by one-sided (Hestenes) Jacobi on Y_q in one warp.
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
constexpr int kSvtThreads = 128;   // 4 patches (warps) per block

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
// nuc: [nq] sum sigma.  The SVD of the p^2 x r coefficient block Y_q is one-sided (Hestenes)
// Jacobi: column pairs of Y_q are rotated until mutually orthogonal, accumulating V, so that
// Y_q V = Yhat has orthogonal columns of norms sigma_j (float32 keeps the small sigma to relative
// accuracy: no squared Gram); SVT(Y_q) = Yhat diag(max(1 - tau / sigma, 0)) V^H.
// Shared memory per warp: svt_warp_bytes(p, r).
__host__ __device__ constexpr size_t svt_warp_bytes(int p, int r) { return ((size_t)p * p * r + (size_t)r * r) * 8; }

static __global__ void __launch_bounds__(kSvtThreads) k_llr_svt(const float2* __restrict__ Y, const int* __restrict__ corners,
                                                          int nc, int N, int p, int r, float tau, int nq,
                                                          float2* __restrict__ P, double* __restrict__ nuc) {
  extern __shared__ __align__(16) unsigned char llr_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * (kSvtThreads / 32) + warp;
  if (q >= nq) return;   // warp-uniform
  float2* Yq = reinterpret_cast<float2*>(llr_raw + (size_t)warp * svt_warp_bytes(p, r));   // [p*p][r]
  float2* Vm = Yq + p * p * r;                                                            // [r][r]
  const int qy = q / nc, qx = q % nc;
  const int y0 = corners[qy], x0 = corners[qx];
  const int np = p * p;
  for (int e = lane; e < np * r; e += 32) {
    const int kk = e / r, i = e % r;
    Yq[e] = Y[((size_t)(y0 + kk / p) * N + (x0 + kk % p)) * r + i];
  }
  for (int e = lane; e < r * r; e += 32) Vm[e] = make_float2(e / r == e % r ? 1.f : 0.f, 0.f);
  __syncwarp();
  // ||Y_q||_F^2 (invariant under the rotations): pairs whose inner product is below 1e-13 of it
  // are numerically orthogonal however small the columns (rounding noise would otherwise keep
  // rotating the negligible columns of a low-rank patch)
  float fro = 0.f;
  for (int e = lane; e < np * r; e += 32) fro = fmaf(Yq[e].x, Yq[e].x, fmaf(Yq[e].y, Yq[e].y, fro));
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  const float floor_g = 1e-13f * fro;
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rotated = false;
    for (int pp = 0; pp < r - 1; ++pp)
      for (int qq = pp + 1; qq < r; ++qq) {
        // alpha = |y_p|^2, beta = |y_q|^2, g = <y_p, y_q> over the p^2 rows (lanes stride the rows)
        float al = 0.f, be = 0.f, gx = 0.f, gy = 0.f;
        for (int kk = lane; kk < np; kk += 32) {
          const float2 a = Yq[kk * r + pp], b = Yq[kk * r + qq];
          al = fmaf(a.x, a.x, fmaf(a.y, a.y, al));
          be = fmaf(b.x, b.x, fmaf(b.y, b.y, be));
          gx = fmaf(a.x, b.x, fmaf(a.y, b.y, gx));
          gy = fmaf(a.x, b.y, fmaf(-a.y, b.x, gy));
        }
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          gx += __shfl_xor_sync(0xffffffffu, gx, o);
          gy += __shfl_xor_sync(0xffffffffu, gy, o);
        }
        const float mag = sqrtf(gx * gx + gy * gy);
        if (!(mag > 4e-6f * sqrtf(al * be)) || !(mag > floor_g)) continue;   // orthogonal to float32 accuracy
        rotated = true;
        // 2x2 Hermitian [[al, g], [conj g, be]]: U = [[c, -s e^{i phi}], [s e^{-i phi}, c]],
        // cot 2theta = (al - be) / 2|g|; columns: y_p' = c y_p + s e^{-i phi} y_q, y_q' = c y_q - s e^{i phi} y_p
        const float kap = (al - be) / (2.f * mag);
        const float t = (kap >= 0.f ? 1.f : -1.f) / (fabsf(kap) + sqrtf(1.f + kap * kap));
        const float c = rsqrtf(1.f + t * t), sn = t * c;
        const float2 e = make_float2(gx / mag, gy / mag), ec = make_float2(e.x, -e.y);
        for (int kk = lane; kk < np; kk += 32) {
          const float2 a = Yq[kk * r + pp], b = Yq[kk * r + qq];
          const float2 b_ec = cmul(b, ec), a_e = cmul(a, e);
          Yq[kk * r + pp] = make_float2(c * a.x + sn * b_ec.x, c * a.y + sn * b_ec.y);
          Yq[kk * r + qq] = make_float2(c * b.x - sn * a_e.x, c * b.y - sn * a_e.y);
        }
        if (lane < r) {
          const float2 a = Vm[lane * r + pp], b = Vm[lane * r + qq];
          const float2 b_ec = cmul(b, ec), a_e = cmul(a, e);
          Vm[lane * r + pp] = make_float2(c * a.x + sn * b_ec.x, c * a.y + sn * b_ec.y);
          Vm[lane * r + qq] = make_float2(c * b.x - sn * a_e.x, c * b.y - sn * a_e.y);
        }
        __syncwarp();
      }
    if (!rotated) break;
  }
  // sigma_j = |yhat_j|; f_j = max(1 - tau / sigma_j, 0) held by lane j; nuclear norm = sum sigma
  float fj = 0.f;
  double sig = 0.0;
  for (int j = 0; j < r; ++j) {
    float n2 = 0.f;
    for (int kk = lane; kk < np; kk += 32) {
      const float2 a = Yq[kk * r + j];
      n2 = fmaf(a.x, a.x, fmaf(a.y, a.y, n2));
    }
    for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    const float sj = sqrtf(n2);
    sig += sj;
    if (lane == j) fj = sj > tau ? 1.f - tau / sj : 0.f;
  }
  if (lane == 0) nuc[q] = sig;
  // P_q = Yhat diag(f) V^H:  P[k][j'] = sum_j Yhat[k][j] f_j conj(V[j'][j])
  float2* Pq = P + (size_t)q * np * r;
  for (int e0 = 0; e0 < np * r; e0 += 32) {   // all lanes stay in the loop (shuffles)
    const int e = e0 + lane;
    const bool ok = e < np * r;
    const int kk = ok ? e / r : 0, jp = ok ? e % r : 0;
    float2 acc = make_float2(0.f, 0.f);
    for (int j = 0; j < r; ++j) {
      const float f = __shfl_sync(0xffffffffu, fj, j);
      const float2 v = Vm[jp * r + j];
      const float2 t = cmul(Yq[kk * r + j], make_float2(v.x, -v.y));
      acc.x = fmaf(f, t.x, acc.x);
      acc.y = fmaf(f, t.y, acc.y);
    }
    if (ok) Pq[e] = acc;
  }
}

// Per voxel: Xc = (Y + gamma sum_{q covering v} P_q[v]) / (1 + gamma c(v)), then
// x+[l][v] = sum_i Xc[i] d[i][l] (dT [L][R] as for k_llr_coef).  Covering patches are visited
// in increasing (qy, qx) order.
template <int R>
__global__ void __launch_bounds__(256) k_llr_update(const float2* __restrict__ Y, const float2* __restrict__ P,
                                                    const int* __restrict__ corners, int nc, int N, int p, int r,
                                                    const float2* __restrict__ dT, int L, float gamma,
                                                    float2* __restrict__ xout) {
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
      const float inv = 1.f / (1.f + gamma * (float)cnt);
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (i < r) {
          const float2 y = __ldg(Y + (size_t)v * r + i);
          xc[i] = make_float2((y.x + gamma * xc[i].x) * inv, (y.y + gamma * xc[i].y) * inv);
        }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) xcs[i][lane] = xc[i];
  }
  __syncthreads();
  if (v >= V) return;
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

// standardised patch vectors [n][3 p^2] (channel-major, row-major inside the patch); ms = mean, std x3
static __global__ void k_mfd_patchvec(const float* __restrict__ params, const float* __restrict__ pd,
                                      const double* __restrict__ ms, const int* __restrict__ corners, int nc, int N,
                                      int p, float* __restrict__ pv) {
  const int q = blockIdx.x, y0 = corners[q / nc], x0 = corners[q % nc], np = p * p;
  for (int e = threadIdx.x; e < 3 * np; e += blockDim.x) {
    const int ch = e / np, k = e % np, v = (y0 + k / p) * N + x0 + k % p;
    const float raw = ch == 2 ? pd[v] : params[2 * v + ch];
    pv[(size_t)q * 3 * np + e] = (float)(((double)raw - ms[2 * ch]) / ms[2 * ch + 1]);
  }
}

// d2[i][j] = ||pv_i - pv_j||^2, 32 x 32 tiles of patch pairs
static __global__ void k_mfd_dist(const float* __restrict__ pv, int n, int dim, float* __restrict__ d2) {
  __shared__ float A[32][33], B[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8 threads
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < dim; k0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      A[r][tx] = (i0 + r < n && k0 + tx < dim) ? pv[(size_t)(i0 + r) * dim + k0 + tx] : 0.f;
      B[r][tx] = (j0 + r < n && k0 + tx < dim) ? pv[(size_t)(j0 + r) * dim + k0 + tx] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const float b = B[tx][k];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float dd = A[ty + 8 * u][k] - b;
        acc[u] = fmaf(dd, dd, acc[u]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + ty + 8 * u, j = j0 + tx;
    if (i < n && j < n) d2[(size_t)i * n + j] = acc[u];
  }
}

// histogram of the strict upper triangle's nonzero d2 bits: pass 0 on the high 16 bits, pass 1
// on the low 16 bits of the values whose high bits equal `hi`
static __global__ void k_mfd_hist(const float* __restrict__ d2, int n, int pass, unsigned hi, unsigned* __restrict__ hist) {
  const long long total = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    if (j <= i) continue;
    const unsigned b = __float_as_uint(d2[e]);
    if (b == 0u) continue;
    if (pass == 0) atomicAdd(&hist[b >> 16], 1u);
    else if ((b >> 16) == hi) atomicAdd(&hist[b & 0xFFFFu], 1u);
  }
}

// W[i][j] = exp(-d2 / sigma2) (i != j), 0 on the diagonal; deg[i] = sum_j W[i][j] in a fixed order
static __global__ void k_mfd_weights(float* __restrict__ d2w, int n, float inv_s2, float* __restrict__ deg) {
  const int i = blockIdx.x;
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

// C[n][M] = W[n][n] B[n][M] (fp32, W symmetric real; B, C real views of complex blocks).
// 64 x 64 output tile per 256-thread block, 4 x 4 outputs per thread, K chunks of 16 via smem.
static __global__ void __launch_bounds__(256) k_mfd_sgemm(const float* __restrict__ W, const float* __restrict__ B, int n,
                                                          int M, float* __restrict__ C) {
  __shared__ float As[16][65], Bs[16][65];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < n; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e / 64, c = e % 64;
      // A tile: W[row0 + c][k0 + kk] read as W[k0 + kk][row0 + c] (symmetric) -> coalesced over c
      As[kk][c] = (row0 + c < n && k0 + kk < n) ? W[(size_t)(k0 + kk) * n + row0 + c] : 0.f;
      Bs[kk][c] = (k0 + kk < n && col0 + c < M) ? B[(size_t)(k0 + kk) * M + col0 + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[kk][ty + 16 * u];
        b[u] = Bs[kk][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int rr = row0 + ty + 16 * u, cc = col0 + tx + 16 * v;
      if (rr < n && cc < M) C[(size_t)rr * M + cc] = acc[u][v];
    }
}

// Y[v] -= scale * sum_{q covering v} (deg_q Qm_q[v] - G_q[v])   (Q^*(Q(X) L) in coefficients);
// pen[q-block]: per-block partial of Re sum_q <Qm_q, deg_q Qm_q - G_q> (the trace penalty) when q0 < 0
template <int R>
__global__ void __launch_bounds__(256) k_mfd_apply(float2* __restrict__ Y, const float2* __restrict__ Qm,
                                                   const float2* __restrict__ G, const float* __restrict__ deg,
                                                   const int* __restrict__ corners, int nc, int N, int p, int r,
                                                   float scale) {
  const int V = N * N;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int vy = v / N, vx = v % N, np = p * p;
  float2 acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = make_float2(0.f, 0.f);
  for (int qy = 0; qy < nc; ++qy) {
    const int cy = __ldg(corners + qy);
    if (vy < cy || vy >= cy + p) continue;
    for (int qx = 0; qx < nc; ++qx) {
      const int cx = __ldg(corners + qx);
      if (vx < cx || vx >= cx + p) continue;
      const int q = qy * nc + qx;
      const float dq = __ldg(deg + q);
      const size_t o = ((size_t)q * np + (size_t)(vy - cy) * p + (vx - cx)) * r;
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (i < r) {
          const float2 a = __ldg(Qm + o + i), g = __ldg(G + o + i);
          acc[i].x += dq * a.x - g.x;
          acc[i].y += dq * a.y - g.y;
        }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (i < r) {
      float2 y = Y[(size_t)v * r + i];
      y.x -= scale * acc[i].x;
      y.y -= scale * acc[i].y;
      Y[(size_t)v * r + i] = y;
    }
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

// match.cuh -- exact dictionary matching Phi_D (Eq. (5)) on
// the sm_100a tensor cores with a certified filter and exact float64 rescoring.
//
//   k_v = argmax_k |<d_k, x_v>| / ||d_k||          (reading 21; ties -> lowest k)
//   rho_v = max(Re<d_k, x_v> / ||d_k||^2, 0),  eta_v = LUT[k_v]
//
// 1. Filter basis Phi (Rf <= 64 orthonormal rows, the dictionary's leading right singular vectors,
//    fp32): u_v = Phi x_v, a_k = Phi d_k.  For any x the identity
//        <d_k, x> = <a_k, u> + <r_k, x>,   r_k = (I - Phi^H Phi) d_k   (Phi^H Phi Hermitian)
//    holds exactly, and |<r_k, x>| <= ||r_k|| ||x|| (float64 residual norms per atom, plan time).
// 2. k_dict_proj_*: u_v with fp32 FMAs in 16-frame chunks summed in float64 (error <= 32 u_32 per
//    chunk, Sum_l |phi||x| <= ||x||), ||x_v|| in float64, and the rows [u_hi | u_lo | u_hi] / s_v
//    (fp16 hi/lo split of u / s_v, s_v = max-abs of u): K = 3 x 128.
// 3. k_dict_gemm: the 3xFP16 correlation GEMM [u_hi|u_lo|u_hi] . [a_hi|a_hi|a_lo]^T on tcgen05
//    (fp32 accumulation) -- pass EPI = 0 keeps the best filter score per voxel (64-bit atomicMax),
//    pass EPI = 1 lists every atom whose filter score lies within the certified band 2 beta of it.
//    beta bounds |rho~_k - rho_k| of the normalised correlation rho = |<d,x>| / (||d|| ||x||):
//    residual + projection rounding + split-operand rounding + worst-case fp32 accumulation
//    (dict.cu filter_beta), so the true argmax is always listed.
// 4. k_dict_rescore_*: exact scores of the listed atoms, fp32 products summed in float64 (frames:
//    from the voxel-major copy x^T; coefficients: from the float64 Dc = <d_i, d_k>), argmax with
//    ties to the lowest index, pd and LUT.  A voxel whose list overflows (or an all-atoms band) is
//    rescored against every atom (k_dict_exact_*), so the result never depends on the filter.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "umma.cuh"

namespace mrf {
namespace dm {

using namespace umma;

constexpr int BM = 128;          // voxels per CTA (UMMA M)
constexpr int BN = 256;          // GEMM columns per atom tile (UMMA N) = 128 atoms
constexpr int BK = 64;           // fp16 per 128-byte swizzled row
constexpr int UK = 16;           // UMMA K for kind::f16
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BN * BK * 2;   // 32 KB
// warps 0-3: TMA / MMA roles; then NG epilogue groups of 4 warps (NG = 1 for long series, where
// the MMAs set the pace; NG = 2 for the 13-coefficient basis match, where the epilogue does)
template <int NG>
constexpr int threads() { return 128 + 128 * NG; }
constexpr int THREADS = threads<1>();
constexpr size_t SMEM = 1024 + (size_t)STAGES * (A_BYTES + B_BYTES) + 256;

// instruction descriptor: kind::f16, fp16 A/B, fp32 D, both K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
      : "memory");
}
// best[v] = max over the atom tiles of (score bits << 32 | ~atom), zeroed by the caller;
// w2[k] = (m_k / ||d_k||)^2 (0 for padding atoms).  X~ [Vpad][KD] and D~ [NP][KD] fp16 are read
// through the tensor maps; m_tiles = Vpad / BM, n_tiles = NP / BN, kblocks = KD / BK.  The
// grid is persistent (one CTA per SM), so the m_tiles x n_tiles units quantise to < 1 %.
constexpr int kCand = 128;  // listed candidates per voxel (more: the voxel is rescored against every atom)

template <int NG, int EPI>
__global__ void __launch_bounds__(threads<NG>(), 1)
k_dict_gemm(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmd,
            const float* __restrict__ w2, int m_tiles, int n_tiles, int kblocks, int V,
            unsigned long long* __restrict__ best, const float* __restrict__ thr, int* __restrict__ ncand,
            int* __restrict__ cand) {
  extern __shared__ __align__(128) unsigned char dm_raw[];   // aligned to 1024 below (SMEM has the slack)
  unsigned char* base = (unsigned char*)(((uintptr_t)dm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = base;
  unsigned char* sB = base + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // persistent: work unit u = (m tile u / n_tiles, atom tile u % n_tiles), strided over the grid
  const int units = m_tiles * n_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      bar_init(&tfull[a], 1);
      bar_init(&tempty[a], NG * 4 * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {   // 512 TMEM columns = two 256-column fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int m0 = (u / n_tiles) * BM, nt = u % n_tiles;
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int s = it % STAGES;
        bar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        bar_expect_tx(&full[s], A_BYTES + B_BYTES);
        tma_load_2d(sA + s * A_BYTES, &tmx, kb * BK, m0, &full[s]);
        tma_load_2d(sB + s * B_BYTES, &tmd, kb * BK, nt * BN, &full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    int it = 0, j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int acc = j & 1, use = j >> 1;
      bar_wait(&tempty[acc], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t td = tmem + (uint32_t)(acc * BN);
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int s = it % STAGES;
        bar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        const uint32_t a0 = saddr(sA + s * A_BYTES), b0 = saddr(sB + s * B_BYTES);
#pragma unroll
        for (int k = 0; k < BK / UK; ++k)
          mma_f16(td, sdesc(a0 + k * UK * 2), sdesc(b0 + k * UK * 2), (kb | k) != 0);
        mma_commit(&empty[s]);   // frees the stage once these MMAs have read it
      }
      mma_commit(&tfull[acc]);   // accumulator complete
    }
  } else if (warp >= 4) {
    // ---- epilogue: thread = TMEM lane = voxel row of the unit's m tile; two groups of 4 warps
    // (warp % 4 selects the TMEM lane quarter) take the accumulator's columns [0, 128) and
    // [128, 256) (64 atoms each).  The best atom of a group's 64 is merged across groups and units
    // with one 64-bit atomicMax per voxel on (score bits << 32 | ~atom): scores are >= 0, so their
    // bits order as the values, and on equal scores the lower atom index wins (order independent,
    // deterministic).
    const int grp = (warp - 4) >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int m0 = (u / n_tiles) * BM, nt = u % n_tiles;
      const int acc = j & 1, use = j >> 1;
      const float th = (EPI == 1 && m0 + row < V) ? __ldg(thr + m0 + row) : INFINITY;
      bar_wait(&tfull[acc], use & 1);
      __syncwarp();   // tcgen05.ld is .sync.aligned
      tc_fence_after();
      float bsc = -1.f;
      int bk = 0;
      // CW columns (CW / 2 atoms) per TMEM load and wait: 128 with one group, 64 with two (registers)
      constexpr int CW = NG == 1 ? 128 : 64;
#pragma unroll 1
      for (int ch = 0; ch < BN / NG / CW; ++ch) {
        float v[CW];
        const int col = grp * (BN / NG) + ch * CW;
        if constexpr (CW == 128) tmem_ld128(tmem + lane_addr + (uint32_t)(acc * BN + col), v);
        else tmem_ld64(tmem + lane_addr + (uint32_t)(acc * BN + col), v);
        const int k0 = nt * (BN / 2) + col / 2;
#pragma unroll
        for (int q = 0; q < CW / 2; ++q) {
          const float wq = __ldg(w2 + k0 + q);
          const float sc = (v[2 * q] * v[2 * q] + v[2 * q + 1] * v[2 * q + 1]) * wq;
          if (EPI == 0) {
            if (sc > bsc) {   // strict: equal scores keep the lowest atom index
              bsc = sc;
              bk = k0 + q;
            }
          } else if (sc >= th && wq > 0.f) {   // inside the certified band (zero / padding atoms never)
            const int slot = atomicAdd(ncand + m0 + row, 1);
            if (slot < kCand) cand[(size_t)(m0 + row) * kCand + slot] = k0 + q;
          }
        }
      }
      tc_fence_before();
      bar_arrive(&tempty[acc]);
      if (EPI == 0 && m0 + row < V)
        atomicMax(best + m0 + row,
                  ((unsigned long long)__float_as_uint(fmaxf(bsc, 0.f)) << 32) | (0xFFFFFFFFu - (uint32_t)bk));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}


// ------------------------------------------------------------------------------ projections
constexpr int RF = 64;          // filter basis rows (padded)
constexpr int KF = 3 * 2 * RF;  // fp16 row length [u_hi | u_lo | u_hi] = 384

// split v (already divided by the scale) into fp16 hi + lo: |v - hi - lo| <= u16^2 |v| + 2^-25
__device__ __forceinline__ void split_h(double v, __half& hi, __half& lo) {
  hi = __double2half(v);
  lo = __double2half(v - (double)__half2float(hi));
}

// Frame domain: x [L][V] complex64 -> u = Phi x, ||x|| (float64), the packed row [V][KF], scale s_v,
// u itself in float64 [V][RF] (the second certification level of the rescoring) and the
// voxel-major copy xT [V][L].  A register-tiled complex GEMM on the CUDA cores: block = 64 voxels
// x 64 coefficients, thread = 4 voxels x 4 coefficients (16 complex accumulators), K streamed in
// 16-frame tiles (x tile [16][64] and phi tile [16][64] complex in shared memory, cp.async double
// buffered; per frame 4 LDS.128 feed 64 FMAs).  Each 16-frame tile is one fp32 chunk (2 x 16 FMAs
// per component: error <= gamma_32 Sum |phi| |x| <= gamma_32 ||x||), added into float64 totals.
constexpr int kProjChunk = 16;   // frames per fp32 chunk = frames per K tile
constexpr int PJV = 64;          // voxels per block
constexpr int PJX = PJV + 2;     // padded x-tile row (16-byte aligned pairs, conflict-light transposed reads)
constexpr size_t proj_smem() { return (size_t)2 * kProjChunk * RF * 8 + (size_t)2 * kProjChunk * PJX * 8; }

// cp.async of 8 / 16 bytes, zero-filled when `valid` is false (LDGSTS)
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(saddr(dst)), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(dst)), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__global__ void __launch_bounds__(256, 2) k_dict_proj_frames(const float2* __restrict__ x, const float2* __restrict__ phiT,
                                                             int L, int V, float2* __restrict__ xT,
                                                             __half* __restrict__ xp, float* __restrict__ xs,
                                                             double* __restrict__ xnorm, double2* __restrict__ u64) {
  extern __shared__ __align__(16) unsigned char pj_raw[];   // proj_smem() bytes
  auto ptile = reinterpret_cast<float2(*)[kProjChunk][RF]>(pj_raw);                              // [buf][frame][f]
  auto tile = reinterpret_cast<float2(*)[kProjChunk][PJX]>(pj_raw + 2 * kProjChunk * RF * 8);    // [buf][frame][voxel]
  auto red = reinterpret_cast<double(*)[16]>(pj_raw);   // after the loop: [voxel][tx] (aliases ptile)
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;   // coefficients 4tx.., voxels 4ty..
  const int vb = blockIdx.x * PJV;
  double ur[4][4], ui[4][4], nrm[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    nrm[a] = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) ur[a][b] = ui[a][b] = 0.0;
  }
  const int ntiles = (L + kProjChunk - 1) / kProjChunk;
  auto stage = [&](int t) {   // tile t into buffer t & 1 (zero past L / V)
    const int l0 = kProjChunk * t, bi = t & 1;
#pragma unroll
    for (int q = 0; q < kProjChunk * PJV / 256; ++q) {   // x: [16 frames][64 voxels], 8 bytes each
      const int i = tid + 256 * q, fl = i / PJV, vv = i % PJV;
      const int l = l0 + fl, v = vb + vv;
      cp_async8(&tile[bi][fl][vv], x + (size_t)min(l, L - 1) * V + min(v, V - 1), l < L && v < V);
    }
#pragma unroll
    for (int q = 0; q < kProjChunk * RF / 2 / 256; ++q) {   // phi rows: [16][64] complex = 512 x 16 bytes
      const int i = tid + 256 * q, fl = i / (RF / 2), l = l0 + fl;
      cp_async16(reinterpret_cast<float4*>(&ptile[bi][0][0]) + i,
                 reinterpret_cast<const float4*>(phiT + (size_t)min(l, L - 1) * RF) + (i % (RF / 2)), l < L);
    }
  };
  stage(0);
  cp_async_commit();
  for (int t = 0; t < ntiles; ++t) {
    const int l0 = kProjChunk * t, bi = t & 1;
    if (t + 1 < ntiles) stage(t + 1);
    cp_async_commit();
    cp_async_wait1();   // tile t has landed (t + 1 may still be in flight)
    __syncthreads();
    float cr[4][4], ci[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) cr[a][b] = ci[a][b] = 0.f;
#pragma unroll 4
    for (int fl = 0; fl < kProjChunk; ++fl) {
      const float4 x01 = *reinterpret_cast<const float4*>(&tile[bi][fl][4 * ty]);       // voxels 4ty, 4ty+1
      const float4 x23 = *reinterpret_cast<const float4*>(&tile[bi][fl][4 * ty + 2]);
      const float4 p01 = *reinterpret_cast<const float4*>(&ptile[bi][fl][4 * tx]);
      const float4 p23 = *reinterpret_cast<const float4*>(&ptile[bi][fl][4 * tx + 2]);
      const float2 xv[4] = {make_float2(x01.x, x01.y), make_float2(x01.z, x01.w), make_float2(x23.x, x23.y),
                            make_float2(x23.z, x23.w)};
      const float2 pv[4] = {make_float2(p01.x, p01.y), make_float2(p01.z, p01.w), make_float2(p23.x, p23.y),
                            make_float2(p23.z, p23.w)};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {   // u += conj(phi) x
          cr[a][b] = fmaf(pv[b].x, xv[a].x, fmaf(pv[b].y, xv[a].y, cr[a][b]));
          ci[a][b] = fmaf(pv[b].x, xv[a].y, fmaf(-pv[b].y, xv[a].x, ci[a][b]));
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) { ur[a][b] += (double)cr[a][b]; ui[a][b] += (double)ci[a][b]; }
    // ||x||^2: thread tx adds frame tx of the tile for its 4 voxels
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const float2 xv = tile[bi][tx][4 * ty + a];
      nrm[a] += (double)xv.x * xv.x + (double)xv.y * xv.y;
    }
    // voxel-major copy: 64 voxels x 16 frames, each voxel's 128-byte run coalesced
#pragma unroll
    for (int q = 0; q < kProjChunk * PJV / 256; ++q) {
      const int i = tid + 256 * q, vv = i / kProjChunk, fl = i % kProjChunk;
      if (vb + vv < V && l0 + fl < L) xT[(size_t)(vb + vv) * L + l0 + fl] = tile[bi][fl][vv];
    }
    __syncthreads();   // buffer bi is refilled by the stage of tile t + 2
  }
  // per voxel: s_v = max-abs of its 64 complex coefficients (16 threads), ||x|| (16 threads)
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double m = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) m = fmax(m, fmax(fabs(ur[a][b]), fabs(ui[a][b])));
    red[4 * ty + a][tx] = m;
  }
  __syncthreads();
  double sv[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double m = 0.0;
    for (int i = 0; i < 16; ++i) m = fmax(m, red[4 * ty + a][i]);
    sv[a] = m > 0.0 ? m : 1.0;
  }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < 4; ++a) red[4 * ty + a][tx] = nrm[a];
  __syncthreads();
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int v = vb + 4 * ty + a;
    if (v >= V) continue;
    if (tx == 0) {
      double n2 = 0.0;
      for (int i = 0; i < 16; ++i) n2 += red[4 * ty + a][i];
      xs[v] = (float)sv[a];
      xnorm[v] = sqrt(n2);
    }
    const float sf = (float)sv[a];   // the scale the GEMM epilogue sees
    __half* row = xp + (size_t)v * KF;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int f = 4 * tx + b, c = 2 * f;
      u64[(size_t)v * RF + f] = make_double2(ur[a][b], ui[a][b]);
      __half hr, lr, hi, li;
      split_h(ur[a][b] / (double)sf, hr, lr);
      split_h(ui[a][b] / (double)sf, hi, li);
      row[c] = hr; row[c + 1] = hi;                       // [u_hi
      row[2 * RF + c] = lr; row[2 * RF + c + 1] = li;     //  | u_lo
      row[4 * RF + c] = hr; row[4 * RF + c + 1] = hi;     //  | u_hi]
    }
  }
}

// Basis coordinates: x = sum_i w_i d_i (w [r][V], the LLR basis rows d_i, r <= 32).  Here the exact
// scores are r-dimensional, <d_k, x> = sum_i w_i conj(Dc[k][i]) (Dc = <d_i, d_k>, float64), so the
// filter runs on w itself: rows [w_hi | w_lo | w_hi] / s_v of KFC = 3 x 64 halves (2r <= 64, zero
// padded) against the packed Dc rows; ||x||^2 = w^H Gd w (Gd = d d^H, float64).  One thread per voxel.
constexpr int KFC = 3 * 64;
__global__ void __launch_bounds__(128) k_dict_proj_coef(const float2* __restrict__ w, int r, int V,
                                                        const double2* __restrict__ Gd, __half* __restrict__ xp,
                                                        float* __restrict__ xs, double* __restrict__ xnorm) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  float2 wv[32];
  float m = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    wv[i] = i < r ? __ldg(w + (size_t)i * V + v) : make_float2(0.f, 0.f);
    m = fmaxf(m, fmaxf(fabsf(wv[i].x), fabsf(wv[i].y)));
  }
  double n2 = 0.0;
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {   // conj(w_i) Gd_ij w_j
      const double2 gq = __ldg(Gd + i * r + j);
      const double ar = (double)wv[i].x, ai = -(double)wv[i].y, br = wv[j].x, bi = wv[j].y;
      const double pr = ar * br - ai * bi, pi = ar * bi + ai * br;
      n2 += pr * gq.x - pi * gq.y;
    }
  const float sf = m > 0.f ? m : 1.f;
  xs[v] = sf;
  xnorm[v] = sqrt(fmax(n2, 0.0));
  __half* row = xp + (size_t)v * KFC;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    __half hr, lr, hi, li;
    split_h((double)wv[i].x / (double)sf, hr, lr);
    split_h((double)wv[i].y / (double)sf, hi, li);
    row[2 * i] = hr; row[2 * i + 1] = hi;
    row[64 + 2 * i] = lr; row[64 + 2 * i + 1] = li;
    row[128 + 2 * i] = hr; row[128 + 2 * i + 1] = hi;
  }
}

// Certified band: thr_v = (max(0, sqrt(best_v) - 2 beta ||x_v|| / s_v))^2 on the filter score
// scale (sqrt(score) = rho~ ||x|| / s_v); +inf for a zero voxel (every atom scores 0: index 0).
__global__ void k_dict_thr(const unsigned long long* __restrict__ best, const double* __restrict__ xnorm,
                           const float* __restrict__ xs, double beta, int V, float* __restrict__ thr,
                           int* __restrict__ ncand) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  ncand[v] = 0;
  if (!(xnorm[v] > 0.0)) {
    thr[v] = INFINITY;
    return;
  }
  const double sb = sqrt((double)__uint_as_float((uint32_t)(best[v] >> 32)));
  const double t = sb - 2.0 * beta * xnorm[v] / (double)xs[v];
  // rounded down so that the fp32 comparison in the epilogue can only admit more atoms
  thr[v] = t > 0.0 ? __double2float_rd(t * t * (1.0 - 1e-6)) : 0.f;
}

// ------------------------------------------------------------------------------ exact rescoring
struct Best {
  double s;      // |c|^2 / ||d||^2
  int k;
  double cre;    // Re c of the best atom
};
__device__ __forceinline__ void best_update(Best& b, double s, int k, double cre) {
  if (s > b.s || (s == b.s && k < b.k)) { b.s = s; b.k = k; b.cre = cre; }
}

__device__ __forceinline__ void finish_voxel(int v, const Best& b, const double* __restrict__ dn2,
                                             const float* __restrict__ lut, int P, int* __restrict__ index,
                                             float* __restrict__ pd, float* __restrict__ params) {
  index[v] = b.k;
  pd[v] = (float)fmax(b.cre / dn2[b.k], 0.0);
  if (params)
    for (int c = 0; c < P; ++c) params[(size_t)v * P + c] = __ldg(lut + (size_t)b.k * P + c);
}

// exact <d_k, x_v> from the voxel-major frames: one warp, lanes over frames, float64 sums of the
// (exact) products of fp32 values, fixed-order warp reduction
__device__ __forceinline__ double2 warp_dot_frames(const float2* __restrict__ dk, const float2* __restrict__ xv, int L,
                                                   int lane) {
  double sr = 0.0, si = 0.0;
  for (int l = lane; l < L; l += 32) {
    const float2 a = __ldg(dk + l), b = __ldg(xv + l);
    sr += (double)a.x * b.x + (double)a.y * b.y;
    si += (double)a.x * b.y - (double)a.y * b.x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    si += __shfl_xor_sync(0xffffffffu, si, o);
  }
  return make_double2(sr, si);
}

// Frames: one warp per voxel.  Level 2 (lane i = listed atom i): rho^_k = |<a_k, u>| / (||d_k|| ||x||)
// in float64 from the float64 coefficients, |rho^_k - rho_k| <= beta2_k = (||r_k|| + eps_u ||a_k||_1)
// / ||d_k|| (per atom, dict.cu); an atom stays a candidate only if rho^_k + beta2_k reaches
// max_j (rho^_j - beta2_j).  Level 3: exact float64 <d_k, x> over the frames for the survivors.  A
// voxel whose list overflowed is queued for the full scan (ov / nov).
__global__ void __launch_bounds__(256) k_dict_rescore_frames(const float2* __restrict__ xT, const float2* __restrict__ atoms,
                                                             const double* __restrict__ dn2, const double* __restrict__ xnorm,
                                                             const double2* __restrict__ u64, const double2* __restrict__ a64,
                                                             const double* __restrict__ beta2, int pw,
                                                             const int* __restrict__ ncand, const int* __restrict__ cand,
                                                             const float* __restrict__ lut, int P, int L, int V,
                                                             int* __restrict__ index, float* __restrict__ pd,
                                                             float* __restrict__ params, int* __restrict__ ov,
                                                             int* __restrict__ nov) {
  const int lane = threadIdx.x & 31;
  const int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (v >= V) return;
  Best b{-1.0, 0, 0.0};
  const double xn = xnorm[v];
  if (!(xn > 0.0)) {   // zero voxel: every score is 0 -> the lowest index, PD 0
    b.s = 0.0;
    if (lane == 0) finish_voxel(v, b, dn2, lut, P, index, pd, params);
    return;
  }
  const int n = ncand[v];
  if (n > kCand || n == 0) {   // (n == 0 cannot happen: the filter's best atom is always in band)
    if (lane == 0) ov[atomicAdd(nov, 1)] = v;
    return;
  }
  // level 2: lane i scores listed atoms i, i + 32, i + 64, i + 96
  constexpr int RND = kCand / 32;
  int kr[RND];
  double hr[RND], m = -INFINITY;
  const double2* uv = u64 + (size_t)v * RF;
#pragma unroll
  for (int rd = 0; rd < RND; ++rd) {
    const int i = 32 * rd + lane;
    kr[rd] = 0;
    hr[rd] = -INFINITY;
    if (i < n) {
      const int k = cand[(size_t)v * kCand + i];
      const double2* ak = a64 + (size_t)k * RF;
      double sr = 0.0, si = 0.0;
#pragma unroll 8
      for (int f = 0; f < RF; ++f) {   // <a_k, u> = sum conj(a) u
        const double2 a = __ldg(ak + f), u = __ldg(uv + f);
        sr += a.x * u.x + a.y * u.y;
        si += a.x * u.y - a.y * u.x;
      }
      // pw = 2 (Eq. 5 as printed): score |c| / ||d||^2 = rho / ||d||, bound beta2 / ||d||
      const double nd = sqrt(dn2[k]), sc = pw == 2 ? nd : 1.0;
      const double rho = sqrt(sr * sr + si * si) / (nd * xn) / sc, bk = beta2[k] / sc;
      kr[rd] = k;
      hr[rd] = rho + bk;
      m = fmax(m, rho - bk);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  // level 3: exact float64 <d_k, x> for the atoms whose upper bound reaches m
  const float2* xv = xT + (size_t)v * L;
#pragma unroll
  for (int rd = 0; rd < RND; ++rd) {
    unsigned keep = __ballot_sync(0xffffffffu, hr[rd] >= m);
    while (keep) {
      const int i = __ffs(keep) - 1;
      keep &= keep - 1;
      const int ki = __shfl_sync(0xffffffffu, kr[rd], i);
      const double2 c = warp_dot_frames(atoms + (size_t)ki * L, xv, L, lane);
      best_update(b, (c.x * c.x + c.y * c.y) / (pw == 2 ? dn2[ki] * dn2[ki] : dn2[ki]), ki, c.x);
    }
  }
  if (lane == 0) finish_voxel(v, b, dn2, lut, P, index, pd, params);
}

// Full exact scan for the queued voxels: item (queued voxel q, atom part) -> the part's best in
// part_best[q][part]; k_dict_exact_finish merges the parts in order (deterministic).
constexpr int kParts = 16;
struct PartBest {
  double s, cre;
  int k, pad;
};
__global__ void __launch_bounds__(256) k_dict_exact_frames(const float2* __restrict__ xT, const float2* __restrict__ atoms,
                                                           const double* __restrict__ dn2, int pw, int K, int L,
                                                           const int* __restrict__ ov, const int* __restrict__ nov,
                                                           PartBest* __restrict__ part_best) {
  __shared__ Best wb[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n = *nov, kp = (K + kParts - 1) / kParts;
  for (int it = blockIdx.x; it < n * kParts; it += gridDim.x) {
    const int q = it / kParts, part = it % kParts, v = ov[q];
    const int k0 = part * kp, k1 = min(K, k0 + kp);
    Best b{-1.0, 0x7fffffff, 0.0};
    for (int k = k0 + w; k < k1; k += 8) {
      if (!(dn2[k] > 0.0)) continue;   // an all-zero atom is never matched
      const double2 c = warp_dot_frames(atoms + (size_t)k * L, xT + (size_t)v * L, L, lane);
      best_update(b, (c.x * c.x + c.y * c.y) / (pw == 2 ? dn2[k] * dn2[k] : dn2[k]), k, c.x);
    }
    if (lane == 0) wb[w] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
      Best t = wb[0];
      for (int i = 1; i < 8; ++i) best_update(t, wb[i].s, wb[i].k, wb[i].cre);
      part_best[(size_t)q * kParts + part] = PartBest{t.s, t.cre, t.k, 0};
    }
    __syncthreads();
  }
}

__global__ void k_dict_exact_finish(const int* __restrict__ ov, const int* __restrict__ nov,
                                    const PartBest* __restrict__ part_best, const double* __restrict__ dn2,
                                    const float* __restrict__ lut, int P, int* __restrict__ index, float* __restrict__ pd,
                                    float* __restrict__ params) {
  const int n = *nov;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    Best b{-1.0, 0x7fffffff, 0.0};
    for (int part = 0; part < kParts; ++part) {
      const PartBest pb = part_best[(size_t)q * kParts + part];
      best_update(b, pb.s, pb.k, pb.cre);
    }
    finish_voxel(ov[q], b, dn2, lut, P, index, pd, params);
  }
}

// Basis coordinates: exact <d_k, x> = sum_i w_i conj(Dc[k][i]) (Dc = <d_i, d_k>, float64: products of
// fp32 w and float64 Dc, float64 sums), one thread per voxel over its listed atoms; overflow queued
// for k_dict_exact_coef.
__device__ __forceinline__ double2 dot_coef(const double2* __restrict__ dck, const float2 (&wv)[32], int r) {
  double sr = 0.0, si = 0.0;
  for (int i = 0; i < r; ++i) {
    const double2 d = __ldg(dck + i);
    sr += wv[i].x * d.x + wv[i].y * d.y;
    si += wv[i].y * d.x - wv[i].x * d.y;
  }
  return make_double2(sr, si);
}

__global__ void __launch_bounds__(128) k_dict_rescore_coef(const float2* __restrict__ w, int r, const double2* __restrict__ Dc,
                                                           const double* __restrict__ dn2, int pw, const double* __restrict__ xnorm,
                                                           const int* __restrict__ ncand, const int* __restrict__ cand,
                                                           const float* __restrict__ lut, int P, int V,
                                                           int* __restrict__ index, float* __restrict__ pd,
                                                           float* __restrict__ params, int* __restrict__ ov,
                                                           int* __restrict__ nov) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  Best b{-1.0, 0, 0.0};
  if (!(xnorm[v] > 0.0)) {
    b.s = 0.0;
    finish_voxel(v, b, dn2, lut, P, index, pd, params);
    return;
  }
  const int n = ncand[v];
  if (n > kCand || n == 0) {
    ov[atomicAdd(nov, 1)] = v;
    return;
  }
  float2 wv[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) wv[i] = i < r ? __ldg(w + (size_t)i * V + v) : make_float2(0.f, 0.f);
  for (int i = 0; i < n; ++i) {
    const int k = cand[(size_t)v * kCand + i];
    const double2 c = dot_coef(Dc + (size_t)k * r, wv, r);
    best_update(b, (c.x * c.x + c.y * c.y) / (pw == 2 ? dn2[k] * dn2[k] : dn2[k]), k, c.x);
  }
  finish_voxel(v, b, dn2, lut, P, index, pd, params);
}

__global__ void __launch_bounds__(128) k_dict_exact_coef(const float2* __restrict__ w, int r, const double2* __restrict__ Dc,
                                                         const double* __restrict__ dn2, int pw, int K, const float* __restrict__ lut,
                                                         int P, int V, const int* __restrict__ ov, const int* __restrict__ nov,
                                                         int* __restrict__ index, float* __restrict__ pd,
                                                         float* __restrict__ params) {
  const int n = *nov;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int v = ov[q];
    float2 wv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) wv[i] = i < r ? __ldg(w + (size_t)i * V + v) : make_float2(0.f, 0.f);
    Best b{-1.0, 0, 0.0};
    for (int k = 0; k < K; ++k) {
      if (!(dn2[k] > 0.0)) continue;
      const double2 c = dot_coef(Dc + (size_t)k * r, wv, r);
      best_update(b, (c.x * c.x + c.y * c.y) / (pw == 2 ? dn2[k] * dn2[k] : dn2[k]), k, c.x);
    }
    finish_voxel(v, b, dn2, lut, P, index, pd, params);
  }
}

// ------------------------------------------------------------------------------ setup (float64)
// Per atom (one block): a_k = Phi d_k (RF complex, float64 from the fp32 inputs), the residual
// norm ||d_k - Phi^H a_k||^2 and ||a_k||_1, with phi [RF][L] (rows past Rf zero).
__global__ void __launch_bounds__(256) k_dict_filter_atoms(const float2* __restrict__ atoms, const float2* __restrict__ phi,
                                                           int L, double2* __restrict__ a, double* __restrict__ res2,
                                                           double* __restrict__ a1) {
  __shared__ double2 sa[RF];
  __shared__ double red[8];
  const int k = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float2* d = atoms + (size_t)k * L;
  for (int f = w; f < RF; f += 8) {   // warp per filter row
    double sr = 0.0, si = 0.0;
    for (int l = lane; l < L; l += 32) {   // conj(phi) d
      const float2 p = __ldg(phi + (size_t)f * L + l), x = __ldg(d + l);
      sr += (double)p.x * x.x + (double)p.y * x.y;
      si += (double)p.x * x.y - (double)p.y * x.x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sr += __shfl_xor_sync(0xffffffffu, sr, o);
      si += __shfl_xor_sync(0xffffffffu, si, o);
    }
    if (lane == 0) sa[f] = make_double2(sr, si);
  }
  __syncthreads();
  double r2 = 0.0;
  for (int l = threadIdx.x; l < L; l += blockDim.x) {   // d_l - sum_f phi_fl a_f
    const float2 x = __ldg(d + l);
    double er = x.x, ei = x.y;
    for (int f = 0; f < RF; ++f) {
      const float2 p = __ldg(phi + (size_t)f * L + l);
      er -= (double)p.x * sa[f].x - (double)p.y * sa[f].y;
      ei -= (double)p.x * sa[f].y + (double)p.y * sa[f].x;
    }
    r2 += er * er + ei * ei;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
  if (lane == 0) red[w] = r2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, n1 = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    for (int f = 0; f < RF; ++f) n1 += sqrt(sa[f].x * sa[f].x + sa[f].y * sa[f].y);
    res2[k] = t;
    a1[k] = n1;
  }
  if (threadIdx.x < RF) a[(size_t)k * RF + threadIdx.x] = sa[threadIdx.x];
}

}  // namespace dm
}  // namespace mrf

// match.cuh -- dictionary matching Phi_D (Eq. (5)) on the
// sm_100a tensor cores.
//
//   k_v = argmax_k |<d_k, x_v>| / ||d_k||          (reading 21; ties -> lowest k)
//   rho_v = max(Re<d_k, x_v> / ||d_k||^2, 0),  eta_v = LUT[k_v]
//
// The correlations of all voxels with all atoms are one complex GEMM, done as a real fp16 GEMM
// with fp32 accumulation: voxel row v = (xr_0, xi_0, xr_1, xi_1, ...) / s_v, atom rows
// 2k = (dr_l, di_l) / m_k and 2k+1 = (-di_l, dr_l) / m_k, so output columns (2k, 2k+1) are
// (Re, Im) <d_k, x_v> / (s_v m_k).  s_v (per voxel) and m_k (per atom) are max-abs scales that
// keep the fp16 operands in [-1, 1]; the argmax uses |c~|^2 * (m_k / ||d_k||)^2 (s_v is common
// to a voxel's row).  rho is recomputed exactly in fp32 for the chosen atom (k_dict_fix).
//
// k_dict_gemm: persistent CTAs over (128-voxel, 128-atom) units, 384 threads in roles: warp 0 = TMA producer (128-byte
// swizzled tiles, 4-stage mbarrier ring), warp 1 = TMEM allocator + single-thread tcgen05.mma
// issuer (M = 128, N = 256, K = 16 per instruction, fp32 accumulators in TMEM, two 256-column
// accumulator buffers so the epilogue of one atom tile overlaps the MMAs of the next), warps
// 4..11 = epilogue in two groups of 4 warps, one per half of the atom tile (tcgen05.ld, one voxel
// per thread = TMEM lane, running argmax in registers) -- with the 13 basis coefficients (K = 64)
// the MMAs are short and the epilogue sets the pace.
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
template <int NG>
__global__ void __launch_bounds__(threads<NG>(), 1)
k_dict_gemm(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmd,
            const float* __restrict__ w2, int m_tiles, int n_tiles, int kblocks, int V,
            unsigned long long* __restrict__ best) {
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
          const float sc = (v[2 * q] * v[2 * q] + v[2 * q + 1] * v[2 * q + 1]) * __ldg(w2 + k0 + q);
          if (sc > bsc) {   // strict: equal scores keep the lowest atom index
            bsc = sc;
            bk = k0 + q;
          }
        }
      }
      tc_fence_before();
      bar_arrive(&tempty[acc]);
      if (m0 + row < V)
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

// X [L][V] complex64 (frame-major image stack) -> X~ [Vpad][KD] fp16, row v = interleaved
// (Re, Im) x_v / s_v, zero-padded to KD; s[v] = max_l max(|Re|, |Im|) (1 if the voxel is zero).
// Block = 32 voxels x 8 row-groups; two passes over the voxels' time series.
__global__ void __launch_bounds__(256) k_dict_pack_x(const float2* __restrict__ x, int L, int V, int KD,
                                                     __half* __restrict__ xp, float* __restrict__ s) {
  __shared__ float red[8][33];
  __shared__ __half2 tile[32][65];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int v = blockIdx.x * 32 + tx;
  float m = 0.f;
  if (v < V) {
#pragma unroll 8
    for (int l = ty; l < L; l += 8) {
      const float2 a = __ldg(x + (size_t)l * V + v);
      m = fmaxf(m, fmaxf(fabsf(a.x), fabsf(a.y)));
    }
  }
  red[ty][tx] = m;
  __syncthreads();
  if (ty == 0) {
    float mm = 0.f;
    for (int i = 0; i < 8; ++i) mm = fmaxf(mm, red[i][tx]);
    red[0][tx] = mm > 0.f ? mm : 1.f;
    if (v < V) s[v] = red[0][tx];
  }
  __syncthreads();
  const float inv = 1.f / red[0][tx];
  const int L2 = KD / 2;   // complex slots per padded row
  for (int l0 = 0; l0 < L2; l0 += 64) {
    // load 64 frames x 32 voxels (coalesced over voxels, 8 loads in flight per thread),
    // transpose through shared memory
    float2 a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int l = l0 + ty + 8 * q;
      a[q] = (v < V && l < L) ? __ldg(x + (size_t)l * V + v) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) tile[tx][ty + 8 * q] = __floats2half2_rn(a[q].x * inv, a[q].y * inv);
    __syncthreads();
#pragma unroll
    for (int i = ty; i < 32; i += 8) {   // voxel blockIdx*32 + i, frames l0 + tx and l0 + 32 + tx
      const int vv = blockIdx.x * 32 + i;
      __half2* row = reinterpret_cast<__half2*>(xp + (size_t)vv * KD);
      if (l0 + tx < L2) row[l0 + tx] = tile[i][tx];
      if (l0 + 32 + tx < L2) row[l0 + 32 + tx] = tile[i][32 + tx];
    }
    __syncthreads();
  }
}

// rho and LUT lookup for the chosen atoms: Re<d_k, x_v> in fp32 from the complex64 data.  A
// CTA takes 32 voxels; 32-frame tiles of x ([l][v], coalesced over v) and of the 32 chosen atoms
// ([v][l], coalesced over l) are staged in shared memory; warp w sums voxels 4w..4w+3 with one
// frame per lane and a final shuffle reduction.
__global__ void __launch_bounds__(256) k_dict_fix(const float2* __restrict__ x, const float2* __restrict__ atoms,
                                                  const float* __restrict__ n2inv, const float* __restrict__ lut, int P,
                                                  int L, int V, const unsigned long long* __restrict__ best,
                                                  int* __restrict__ index,
                                                  float* __restrict__ pd, float* __restrict__ params) {
  __shared__ float2 xt[64][33];   // [l][v]
  __shared__ float2 dt[32][65];   // [v][l]
  __shared__ int ks[32];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int v0 = blockIdx.x * 32;
  if (threadIdx.x < 32) ks[tx] = v0 + tx < V ? (int)(0xFFFFFFFFu - (uint32_t)(best[v0 + tx] & 0xFFFFFFFFull)) : 0;
  __syncthreads();
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int l0 = 0; l0 < L; l0 += 64) {   // 64 frames per step, 16 loads in flight per thread
#pragma unroll
    for (int i = ty; i < 64; i += 8) {
      const int l = l0 + i, v = v0 + tx;
      xt[i][tx] = (l < L && v < V) ? __ldg(x + (size_t)l * V + v) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int i = ty; i < 32; i += 8) {
      const float2* dr = atoms + (size_t)ks[i] * L + l0;
      dt[i][tx] = (l0 + tx < L) ? __ldg(dr + tx) : make_float2(0.f, 0.f);
      dt[i][32 + tx] = (l0 + 32 + tx < L) ? __ldg(dr + 32 + tx) : make_float2(0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {   // Re(conj(d) x) = dr xr + di xi, frames l0 + tx and l0 + 32 + tx
      const int j = ty * 4 + q;
      const float2 d0 = dt[j][tx], x0 = xt[tx][j], d1 = dt[j][32 + tx], x1 = xt[32 + tx][j];
      acc[q] = fmaf(d0.x, x0.x, fmaf(d0.y, x0.y, acc[q]));
      acc[q] = fmaf(d1.x, x1.x, fmaf(d1.y, x1.y, acc[q]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float r = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    const int v = v0 + ty * 4 + q;
    if (tx == 0 && v < V) {
      const int k = ks[ty * 4 + q];
      index[v] = k;
      pd[v] = fmaxf(r * __ldg(n2inv + k), 0.f);
    }
    if (params && v < V)
      for (int c = tx; c < P; c += 32) params[(size_t)v * P + c] = __ldg(lut + (size_t)ks[ty * 4 + q] * P + c);
  }
}

// Short time series (L <= 32: the basis-coordinate match, K = 64): one thread per voxel.
// Pack: x [L][V] -> X~ [Vpad][KD] fp16 row v = (Re, Im) x_v / s_v, zero-padded; s_v = max |Re|, |Im|.
__global__ void __launch_bounds__(256) k_dict_pack_short(const float2* __restrict__ x, int L, int V, int Vpad, int KD,
                                                         __half* __restrict__ xp, float* __restrict__ s) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= Vpad) return;
  float2 a[32];
  float m = 0.f;
#pragma unroll
  for (int l = 0; l < 32; ++l) {
    a[l] = (l < L && v < V) ? __ldg(x + (size_t)l * V + v) : make_float2(0.f, 0.f);
    m = fmaxf(m, fmaxf(fabsf(a[l].x), fabsf(a[l].y)));
  }
  const float sc = m > 0.f ? m : 1.f, inv = 1.f / sc;
  if (v < V) s[v] = sc;
  uint4* row = reinterpret_cast<uint4*>(xp + (size_t)v * KD);
#pragma unroll
  for (int q = 0; q < 8; ++q) {   // 8 x 16 bytes = 64 halves = 32 complex slots (KD == 64)
    __half2 h[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) h[t] = __floats2half2_rn(a[4 * q + t].x * inv, a[4 * q + t].y * inv);
    row[q] = *reinterpret_cast<uint4*>(h);
  }
}

// rho and LUT lookup for the chosen atoms, one thread per voxel (L <= 32): Re<d_k, x_v> in fp32.
__global__ void __launch_bounds__(256) k_dict_fix_short(const float2* __restrict__ x, const float2* __restrict__ atoms,
                                                        const float* __restrict__ n2inv, const float* __restrict__ lut,
                                                        int P, int L, int V, const unsigned long long* __restrict__ best,
                                                        int* __restrict__ index, float* __restrict__ pd,
                                                        float* __restrict__ params) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int k = (int)(0xFFFFFFFFu - (uint32_t)(best[v] & 0xFFFFFFFFull));
  const float2* d = atoms + (size_t)k * L;
  float acc = 0.f;
  for (int l = 0; l < L; ++l) {
    const float2 dv = __ldg(d + l), xv = __ldg(x + (size_t)l * V + v);
    acc = fmaf(dv.x, xv.x, fmaf(dv.y, xv.y, acc));
  }
  index[v] = k;
  pd[v] = fmaxf(acc * __ldg(n2inv + k), 0.f);
  if (params)
    for (int c = 0; c < P; ++c) params[(size_t)v * P + c] = __ldg(lut + (size_t)k * P + c);
}

}  // namespace dm
}  // namespace mrf

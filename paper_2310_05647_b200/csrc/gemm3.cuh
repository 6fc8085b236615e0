// gemm3.cuh -- float32-accurate real GEMM on the sm_100a tensor cores (kind::tf32, three products):
//
//   C[m][n] = sum_k A[m][k] B[n][k],   A = A_hi + A_lo,  B = B_hi + B_lo,
//   hi = x rounded to tf32 (10-bit mantissa), lo = x - hi (exact in fp32, |lo| <= 2^-11 |x|),
//   C ~= A_hi B_hi + A_hi B_lo + A_lo B_hi       (the dropped A_lo B_lo is ~2^-22 relative)
//
// Used for the manifold term of the MS-LLR step (Eq. 15, lambda_1 Q^*(Q(X) L)):
// G = W Qm with W the n x n patch similarity matrix (Eq. 8) and Qm the n x (2 p^2 r) real view of
// the patch coefficient blocks, a dense contraction with K = n = 2500 at the MRF size.  Plain
// tf32 (one product) would leave ~1e-3 relative errors that the Laplacian's cancellation
// (L = D - W, rows sum to zero) amplifies; the three-product split restores float32 accuracy.
//
// Operands are K-major fp32 arrays in global memory (hi and lo copies written by k_g3_split), read
// by 2D TMA in 128-byte swizzled boxes of 32 fp32 (out-of-bounds rows / k read as zero).
// k_g3_gemm: persistent CTAs over (128-row, 256-column) output units, 256 threads: warp 0 TMA
// producer (2-stage ring: A_hi, A_lo, B_hi, B_lo = 96 KB per stage), warp 1 TMEM allocator +
// single-thread tcgen05.mma issuer (M = 128, N = 256, K = 8 per instruction, 3 products per K
// step into one fp32 TMEM accumulator; two accumulators so the epilogue of one unit overlaps the
// MMAs of the next), warps 4..7 epilogue (tcgen05.ld, thread = output row, 32 columns per load).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "umma.cuh"

namespace mrf {
namespace g3 {

using namespace umma;

constexpr int BM = 128;                // output rows per unit (UMMA M)
constexpr int BN = 256;                // output columns per unit (UMMA N)
constexpr int BK = 32;                 // fp32 per 128-byte swizzled row
constexpr int UK = 8;                  // UMMA K for kind::tf32
constexpr int STAGES = 2;
constexpr int A_BYTES = BM * BK * 4;   // 16 KB
constexpr int B_BYTES = BN * BK * 4;   // 32 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int THREADS = 256;
constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 256;
// instruction descriptor: fp32 D (bits 4-5 = 1), tf32 A and B (bits 7-9, 10-12 = 2), both K-major,
// N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
      : "memory");
}

// 2D TMA load multicast to the CTAs of `mask` in the cluster (same smem offset, and complete_tx on
// the mbarrier at the same offset in each)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* b,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(saddr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(saddr(b)), "h"(mask)
      : "memory");
}
// tcgen05.commit arriving on the mbarrier at this offset in every CTA of `mask`
__device__ __forceinline__ void mma_commit_mc(uint64_t* b, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   saddr(b)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// C [m_rows][ldc] fp32 (columns < n_cols written).  Tensor maps: ta_hi / ta_lo over A [m_rows][K]
// (box 32 x BM), tb_hi / tb_lo over B [n_cols][K] (box 32 x BN); kblocks = ceil(K / 32).
// MC: clusters of 2 CTAs take row tiles (2p, 2p + 1) of the same column tile; each loads half of the
// B tile's rows and multicasts it to both (tb_* boxes of BN / 2 rows), halving the B traffic from L2;
// a stage is refilled once both CTAs' MMAs have released it (multicast commits, empty count 2).
// m_tiles must then be even (an extra row tile reads zeros and stores nothing).
template <bool MC>
__global__ void __launch_bounds__(THREADS, 1)
k_g3_gemm(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
          const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo, int m_tiles,
          int n_tiles, int kblocks, int m_rows, int n_cols, float* __restrict__ C, long long ldc) {
  extern __shared__ __align__(128) unsigned char g3_raw[];   // aligned to 1024 below (SMEM has the slack)
  unsigned char* base = (unsigned char*)(((uintptr_t)g3_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // unit u = (row tile u % m_tiles, column tile u / m_tiles): CTAs running together share column tiles.
  // MC: unit index over pairs, row tile 2 (u % (m_tiles / 2)) + rank
  const int rank = MC ? (int)cluster_rank() : 0;
  const int grid_units = MC ? (int)gridDim.x / 2 : (int)gridDim.x;
  const int first = MC ? (int)blockIdx.x / 2 : (int)blockIdx.x;
  const int mt_n = MC ? m_tiles / 2 : m_tiles;
  const int units = mt_n * n_tiles;
  auto unit_m0 = [&](int u) { return (MC ? 2 * (u % mt_n) + rank : u % mt_n) * BM; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], MC ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      bar_init(&tfull[a], 1);
      bar_init(&tempty[a], 4 * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {   // 512 TMEM columns = two 256-column fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  if (MC) cluster_sync_all();   // the peer's multicasts land only after our barriers exist
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    int it = 0;
    for (int u = first; u < units; u += grid_units) {
      const int m0 = unit_m0(u), n0 = (u / mt_n) * BN;
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int s = it % STAGES;
        unsigned char* st = base + s * STAGE_BYTES;
        bar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        bar_expect_tx(&full[s], STAGE_BYTES);
        tma_load_2d(st, &ta_hi, kb * BK, m0, &full[s]);
        tma_load_2d(st + A_BYTES, &ta_lo, kb * BK, m0, &full[s]);
        if constexpr (MC) {   // this CTA's half of the B rows, to both CTAs
          const int off = rank * (B_BYTES / 2);
          tma_load_2d_mc(st + 2 * A_BYTES + off, &tb_hi, kb * BK, n0 + rank * (BN / 2), &full[s], 0x3);
          tma_load_2d_mc(st + 2 * A_BYTES + B_BYTES + off, &tb_lo, kb * BK, n0 + rank * (BN / 2), &full[s], 0x3);
        } else {
          tma_load_2d(st + 2 * A_BYTES, &tb_hi, kb * BK, n0, &full[s]);
          tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tb_lo, kb * BK, n0, &full[s]);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    int it = 0, j = 0;
    for (int u = first; u < units; u += grid_units, ++j) {
      const int acc = j & 1, use = j >> 1;
      bar_wait(&tempty[acc], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t td = tmem + (uint32_t)(acc * BN);
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int s = it % STAGES;
        bar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        const uint32_t ah = saddr(base + s * STAGE_BYTES), al = ah + A_BYTES, bh = ah + 2 * A_BYTES,
                       bl = bh + B_BYTES;
#pragma unroll
        for (int k = 0; k < BK / UK; ++k) {
          const uint32_t o = k * UK * 4;   // 32 bytes per K step inside the swizzled row
          mma_tf32(td, sdesc(al + o), sdesc(bh + o), (kb | k) != 0);
          mma_tf32(td, sdesc(ah + o), sdesc(bl + o), 1u);
          mma_tf32(td, sdesc(ah + o), sdesc(bh + o), 1u);
        }
        if constexpr (MC) mma_commit_mc(&empty[s], 0x3);   // both CTAs' producers refill this stage
        else mma_commit(&empty[s]);   // frees the stage once these MMAs have read it
      }
      mma_commit(&tfull[acc]);   // accumulator complete
    }
  } else if (warp >= 4) {
    // ---- epilogue: thread = TMEM lane = output row of the unit
    const int row = (warp - 4) * 32 + lane;
    const uint32_t lane_addr = (uint32_t)((warp - 4) * 32) << 16;
    int j = 0;
    for (int u = first; u < units; u += grid_units, ++j) {
      const int m = unit_m0(u) + row, n0 = (u / mt_n) * BN;
      const int acc = j & 1, use = j >> 1;
      bar_wait(&tfull[acc], use & 1);
      __syncwarp();   // tcgen05.ld is .sync.aligned
      tc_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        float v[32];
        tmem_ld32(tmem + lane_addr + (uint32_t)(acc * BN + ch * 32), v);
        const int c0 = n0 + ch * 32;
        if (m < m_rows) {
          float* out = C + (size_t)m * ldc + c0;
          if (c0 + 32 <= n_cols && ((ldc | c0) & 1) == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) reinterpret_cast<float2*>(out)[i] = make_float2(v[2 * i], v[2 * i + 1]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i < n_cols) out[i] = v[i];
          }
        }
      }
      tc_fence_before();
      bar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  if (MC) cluster_sync_all();   // no CTA leaves while its peer may still multicast into it
  else __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// hi / lo split of src [rows][cols] (row pitch lds) into dst [rows][ldd] (no transpose) or
// dst [cols][ldd] (transpose: dst[c][r] = src[r][c]); 32 x 32 tiles through shared memory,
// block (32, 8).
template <bool T>
__global__ void __launch_bounds__(256) k_g3_split(const float* __restrict__ src, int rows, int cols, long long lds,
                                                  float* __restrict__ hi, float* __restrict__ lo, long long ldd) {
  __shared__ float t[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if constexpr (!T) {
#pragma unroll
    for (int i = ty; i < 32; i += 8) {
      const int r = r0 + i, c = c0 + tx;
      if (r < rows && c < cols) {
        const float x = src[(size_t)r * lds + c], h = tf32_hi(x);
        hi[(size_t)r * ldd + c] = h;
        lo[(size_t)r * ldd + c] = x - h;
      }
    }
  } else {
#pragma unroll
    for (int i = ty; i < 32; i += 8) {
      const int r = r0 + i, c = c0 + tx;
      t[i][tx] = (r < rows && c < cols) ? src[(size_t)r * lds + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int i = ty; i < 32; i += 8) {   // dst row c0 + i, columns r0 + tx
      const int c = c0 + i, r = r0 + tx;
      if (c < cols && r < rows) {
        const float x = t[tx][i], h = tf32_hi(x);
        hi[(size_t)c * ldd + r] = h;
        lo[(size_t)c * ldd + r] = x - h;
      }
    }
  }
}

}  // namespace g3
}  // namespace mrf

// gridding.cuh -- persistent sm_100a kernels of the multi-frame KB-gridding NUFFT pair.
//
// Pipeline per frame l and coil c (the paper's A = F_u C, and
// its adjoint A*):
//   forward A  : k_fwd_rows  a1 deapod . coil . zero-pad, a2 row FFTs of the N non-zero rows
//                k_fwd_cols  a2 column FFT of one 16-column strip, a3 KB gather interpolation
//   adjoint A^H: k_adj_cols  a4 KB spread into the strip (shared memory), a5 column iFFT
//                k_adj_rows  a5 row iFFTs, a6 crop . deapod . conj-coil . coil sum [+ mu x]
// The forward half grid is strip-major ([fc][strip][row][16]: one strip = one bulk copy); the
// adjoint half grid is row-major ([fc][row][G]: one row block = one bulk copy).
//
// Every kernel is persistent (grid = resident CTAs) and walks a list of work items.  The global
// inputs of the NEXT item are fetched by the Tensor Memory Accelerator (cp.async.bulk, completion
// on an mbarrier) into shared memory while the current item computes, so no warp waits on HBM/L2
// inside an item.  The N x G half grid between the row and the column pass is stored strip-major
// ([fc][strip][row][16]) so one strip of one frame-coil is a contiguous 32 KB bulk copy; it lives
// in a frame-batch workspace sized to stay in the 126 MB L2.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"

// Device-side bounds checks (the checks build, -DMRF_CHECKS: libmrfnufft_checks.so):
// every index that comes from a plan table or a staged chunk is tested before use; a failure
// prints the condition and traps (the launch fails, the host sees MRF_ECUDA).  Compiled out of
// the production build.
#ifdef MRF_CHECKS
#include <cstdio>
#define MRF_CHECK(cond)                                                                       \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("MRF_CHECK failed at %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                              \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define MRF_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace mrf {

constexpr int SW = 16;             // columns per strip (>= W: a point's x-taps touch <= 2 strips)
constexpr int kYBytes = 32768;     // largest y[fc] staged in shared memory by k_adj_cols (M <= 4096)
constexpr int kChunkHdr = 8;       // header words of a forward strip chunk (and offset of the adjoint row masks)
constexpr int kAdjHdr = 24;        // header words of an adjoint strip chunk (8 + 16 row-mask words)
constexpr int SWG = SW + 1;        // row stride of the forward strip during the gather (bank skew)
constexpr int kRowThreads = 128;

struct CGScalars;

// Per (interleaf, strip) "chunks" (32-bit words, 16-byte multiples), built once at plan time.
// Forward chunk (gather):  [0] n_rec [1..7] 0, then n_rec point records of recw words:
//     j, taps (gy0 | cx0<<11), wx[W] (the x-weights of the taps inside the strip, starting at strip
//     column cx0, zero past the strip's last tap), wy[W] (fp32)
// Adjoint chunk (spread), the strip's KB spread matrix in SELL-32 form (rows = strip cells
// sorted by non-zero count, slices of 32 lanes):
//     [0] n_slices [1] cells offset [2] entries offset [3] n_multi (slices of width > 1) [4..7] 0
//     [8 + w], w < 16: row-pair mask of warp w's stage-1 loads in k_adj_cols (bit a*P + n1 set if
//     row Q n1 + T a + 2w or the next row holds a spread value)
//     slices : n_slices x {first entry, width}; width < 0: a reduction slice (one cell, its entries
//              spread over the 32 lanes, summed by a warp reduction), then widths non-increasing
//     cells  : n_slices x 32 uint16 strip cells (swizzled slot), 0xFFFF = empty lane
//     entries: {j, w = wx*wy (fp32 bits, from float64)}; entry k of lane l at first + 32k + l;
//              the width-1 slices' entries come first (one flat run), then the wider slices'.
// ftab / atab[r*S + s] = {word offset, words} of each chunk.
struct DevPlan {
  int N, G, M, R, C, W, S, recw;      // S = G / SW strips; recw = 32-bit words per point record
  const float2* __restrict__ coils;   // [C][N][N] or nullptr (C == 1)
  const float* __restrict__ dap;      // [N]  1 / (psi(n) sqrt(N))
  const float2* __restrict__ tw;      // [G]  tw[n2*P + k1] = exp(-i 2 pi n2 k1 / G)
  const int* __restrict__ fchunks;    // forward chunks
  const int2* __restrict__ ftab;      // [R*S] {offset, words}
  const int* __restrict__ achunks;    // adjoint chunks
  const int2* __restrict__ atab;      // [R*S] {offset, words}
  const int* __restrict__ fil;        // [L_local] interleaf of each local frame
  const int* __restrict__ perm;       // [L_local] processing order of each batch's frames (by interleaf) or nullptr
  int dbg;                            // experiment bits (0 in production)
  long long* dbgbuf;                  // phase timer output (experiment bit 2)
};

// ---------------------------------------------------------------------------- async copy (TMA)
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}

// Programmatic dependent launch: the next kernel in the stream may start its prologue while this
// one drains; every kernel waits for its predecessor's completion before touching global data
// that a predecessor produces or consumes.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// float2 += v in shared memory (64-bit CAS; no native shared float add on sm_100)
__device__ __forceinline__ void smem_add2(float2* a, float2 v) {
  unsigned long long* q = reinterpret_cast<unsigned long long*>(a);
  unsigned long long old = *q, assumed;
  do {
    assumed = old;
    float2 f = *reinterpret_cast<float2*>(&assumed);
    f.x += v.x;
    f.y += v.y;
    old = atomicCAS(q, assumed, *reinterpret_cast<unsigned long long*>(&f));
  } while (old != assumed);
}

// Shared-memory strip layout [row][16] with the column XOR-swizzled by the row (row & 15): a
// record's W tap rows then fall in different banks, and a row is still 16 contiguous slots.
__host__ __device__ __forceinline__ int sidx(int row, int col) { return row * SW + (col ^ (row & (SW - 1))); }

// Stage-1 twiddles W_G^{n2 k1} of the two-stage FFT (fft.cuh).  Global table layout [n2][k1]:
// in the column kernels a warp spans 2 values of n2, and the pair (k1, k1 + 1), k1 even, is one
// 16-byte shared-memory load; the row kernels (a warp spans 16 values of n2) transpose it to
// [k1][n2] in shared memory.
__device__ __forceinline__ float4 tw_pair(const float2* stw, int i) { return *reinterpret_cast<const float4*>(stw + i); }

// image index <-> wrapped grid index (centred n = i - N/2, grid position n mod G)
template <int G>
__device__ __forceinline__ int grid_to_img(int pos) {   // pos in the kept set
  constexpr int N = G / 2;
  return pos < N / 2 ? pos + N / 2 : pos - (G - N / 2);
}

// ---------------------------------------------------------------------------- launch shapes
template <int G>
struct RowCfg {
  static constexpr int T = FFTShape<G>::T, P = FFTShape<G>::P, Q = FFTShape<G>::Q;
  static constexpr int RPC = kRowThreads / T;          // rows per item
  static constexpr int N = G / 2;
  static constexpr int EX = Q * (P + 1);               // padded exchange buffer per row
};
template <int G>
constexpr int cols_threads() { return SW * FFTShape<G>::T; }

template <int G>
constexpr size_t fwd_rows_smem(int n_stage) {   // tw | n_stage image blocks | coil block | exchange | bar
  using R = RowCfg<G>;
  return (size_t(G) + size_t(n_stage + 1) * R::RPC * R::N + size_t(R::RPC) * R::EX) * 8 + 16 + R::N * 4;
}
template <int G>
constexpr size_t adj_rows_smem() {              // tw | H block | x blocks[2] | exchange | bars
  using R = RowCfg<G>;
  return (size_t(G) + size_t(R::RPC) * G + 2 * size_t(R::RPC) * R::N + size_t(R::RPC) * R::EX) * 8 + 32 + R::N * 4;
}
// Column kernels: shared memory per CTA is fixed by the resident-CTA target (2 per SM for G <= 512,
// 1 for G = 1024); whatever the strip, twiddles (and y) leave is the chunk staging buffer.
template <int G>
constexpr int cols_ctas_per_sm() { return G >= 1024 ? 1 : 2; }
template <int G>
constexpr size_t fwd_cols_fixed() { return (size_t(G) + size_t(G / 2) * SW + size_t(G) * SWG + SW) * 8 + 16; }
template <int G>
constexpr size_t toep_cols_smem() { return (size_t(G) + size_t(G / 2) * SW + size_t(G) * SW) * 8 + 16; }
// k_adj_cols layout: SEP = separate exchange buffer + register twiddles (G <= 512, one CTA per SM)
template <int G>
constexpr size_t adj_cols_fixed(size_t ybytes, bool sep) {
  return (sep ? 2 * size_t(G) * SW : size_t(G) + size_t(G) * SW) * 8 + ybytes + 16;
}

// Phase timer (experiment bit 2; only compiled with -DMRF_EXPERIMENTS): thread 0 of every CTA
// accumulates clock64 deltas per phase into p.dbgbuf.
#ifdef MRF_EXPERIMENTS
#define MRF_DBG_ON(bit) (p.dbg & (bit))
struct PhaseTimer {
  long long acc[10];
  long long t0;
  bool on;
  __device__ __forceinline__ void start(bool enable) {
    on = enable;
    if (on) {
      for (int i = 0; i < 10; ++i) acc[i] = 0;
      t0 = clock64();
    }
  }
  __device__ __forceinline__ void mark(int i) {
    if (on) {
      const long long t = clock64();
      acc[i] += t - t0;
      t0 = t;
    }
  }
  __device__ __forceinline__ void report(long long* buf, int items) {
    if (on && buf) {
      atomicAdd(reinterpret_cast<unsigned long long*>(buf), (unsigned long long)items);
      for (int i = 0; i < 10; ++i) atomicAdd(reinterpret_cast<unsigned long long*>(buf + 1 + i), (unsigned long long)acc[i]);
    }
  }
};
#else
#define MRF_DBG_ON(bit) false
struct PhaseTimer {
  __device__ __forceinline__ void start(bool) {}
  __device__ __forceinline__ void mark(int) {}
  __device__ __forceinline__ void report(long long*, int) {}
};
#endif

// a3 for one point record (thread = record): y_j += sum_ty wy[ty] sum_i wx[i] strip(gy0 + ty, cx0 + i).
// The forward strip is stored [row][SWG] (16 cells + 1 skew slot per row, so the same column of
// neighbouring rows falls in different banks) and followed by a pad, so the taps past the strip's
// last column (weight 0 by construction) read finite values.  Each y_j receives
// at most two strip partials, added with fp32 atomics onto 0 (order independent).
template <int G, int W, bool GL>
__device__ __forceinline__ void gather_rec(const int* rp, const float2* strip, float2* __restrict__ yf, int M) {
  constexpr int RW = (2 + 2 * W + 3) & ~3;
  int wd[RW];
#pragma unroll
  for (int k = 0; k < RW / 4; ++k) {   // 16-byte piece k of the record: 32 records apart
    const int4 q = GL ? __ldg(reinterpret_cast<const int4*>(rp) + 32 * k) : reinterpret_cast<const int4*>(rp)[32 * k];
    wd[4 * k] = q.x;
    wd[4 * k + 1] = q.y;
    wd[4 * k + 2] = q.z;
    wd[4 * k + 3] = q.w;
  }
  const int gy0 = wd[1] & 2047, cx0 = (wd[1] >> 11) & 31;
  MRF_CHECK((unsigned)wd[0] < (unsigned)M && gy0 < G && cx0 < SW);
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int ty = 0; ty < W; ++ty) {
    const float2* row = strip + ((gy0 + ty) & (G - 1)) * SWG + cx0;
    float2 racc = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < W; ++i) {
      racc = caxpy(__int_as_float(wd[2 + i]), row[i], racc);
    }
    acc = caxpy(__int_as_float(wd[2 + W + ty]), racc, acc);
  }
  atomicAdd(&yf[wd[0]].x, acc.x);
  atomicAdd(&yf[wd[0]].y, acc.y);
}
// The same for any W in [2, 16] (run-time loops; rp may point to shared or global memory).
template <int G>
__device__ __forceinline__ void gather_rec_any(const int* rp, int W, const float2* strip, float2* __restrict__ yf, int M) {
  auto word = [&](int w) { return rp[(w >> 2) * 128 + (w & 3)]; };   // record word w (interleaved layout)
  auto wt = [&](int w) { return __int_as_float(word(w)); };
  const int gy0 = word(1) & 2047, cx0 = (word(1) >> 11) & 31;
  MRF_CHECK((unsigned)word(0) < (unsigned)M && gy0 < G && cx0 < SW);
  float2 acc = make_float2(0.f, 0.f);
  for (int ty = 0; ty < W; ++ty) {
    const float2* row = strip + ((gy0 + ty) & (G - 1)) * SWG + cx0;
    float2 racc = make_float2(0.f, 0.f);
    for (int i = 0; i < W; ++i) {
      racc = caxpy(wt(2 + i), row[i], racc);
    }
    acc = caxpy(wt(2 + W + ty), racc, acc);
  }
  atomicAdd(&yf[word(0)].x, acc.x);
  atomicAdd(&yf[word(0)].y, acc.y);
}

// Toeplitz column-pass items walk a batch's (frame, coil) pairs in interleaf order: perm[l0 + slot]
// is the batch-local frame processed in slot `slot`, so the frames that share an interleaf (and its
// PSF spectrum) are processed together and read it from L2.  Returns fc = frame * C + c.  (The
// gridding column kernels keep the natural order: measured 3-6 % faster there.)
__device__ __forceinline__ int item_fc(const int* __restrict__ perm, int C, int item, int S, int l0) {
  const int slot = item / S;
  const int f = slot / C;
  return (perm ? __ldg(perm + l0 + f) : f) * C + slot % C;
}

// ============================================================================ forward rows
// Items (bl, rowblock, c), c fastest.  MODE 0: image block = x.  MODE 1 (CG, C == 1): image block
// = p' = r + beta p with x' = x + alpha p, both written back (one pass over r, p, x per iteration);
// with pn != nullptr also the float64 partials of ||p'||^2, one per warp and item (split-phase CG).
template <int G, int MODE>
__global__ void __launch_bounds__(kRowThreads)
k_fwd_rows(DevPlan p, const float2* __restrict__ x, float2* __restrict__ H, int l0, int nb,
           float2* __restrict__ cg_r, float2* __restrict__ cg_p, float2* __restrict__ cg_x,
           const double* __restrict__ cg_ab, float2* __restrict__ yzero, long long nyzero,
           double2* __restrict__ pn = nullptr) {
  using Rc = RowCfg<G>;
  constexpr int P = Rc::P, Q = Rc::Q, T = Rc::T, N = Rc::N, RPC = Rc::RPC, A = Q / T, B = P / T;
  constexpr int NRB = N / RPC, S = G / SW, NST = MODE == 1 ? 3 : 1;
  constexpr uint32_t BLK = RPC * N * sizeof(float2);
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* stw = reinterpret_cast<float2*>(smraw);
  float2* xs = stw + G;                       // NST image blocks
  float2* cs = xs + NST * RPC * N;            // coil block
  float2* ex = cs + RPC * N;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ex + RPC * Rc::EX);
  float* sdap = reinterpret_cast<float*>(bar + 2);
  const int C = p.C;
  const int n_items = nb * NRB * C;
  const int tid = threadIdx.x, rloc = tid / T, t = tid % T;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < G; i += kRowThreads) stw[i] = p.tw[(i % Q) * P + i / Q];   // [k1][n2]: a warp spans n2
  for (int i = tid; i < N; i += kRowThreads) sdap[i] = p.dap[i];
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();
  // zero the k-space batch buffer the following column pass accumulates into
  for (long long i = blockIdx.x * (long long)kRowThreads + tid; i < nyzero; i += (long long)gridDim.x * kRowThreads)
    yzero[i] = make_float2(0.f, 0.f);
  auto issue = [&](int item) {
    const int c = item % C, rb = (item / C) % NRB, bl = item / (C * NRB);
    const size_t off = ((size_t)(l0 + bl) * N + (size_t)rb * RPC) * N;
    mbar_expect_tx(bar, BLK * NST + (p.coils ? BLK : 0));
    if (MODE == 0) {
      bulk_g2s(xs, x + off, BLK, bar);
    } else {
      bulk_g2s(xs, cg_r + off, BLK, bar);
      bulk_g2s(xs + RPC * N, cg_p + off, BLK, bar);
      bulk_g2s(xs + 2 * RPC * N, cg_x + off, BLK, bar);
    }
    if (p.coils) bulk_g2s(cs, p.coils + ((size_t)c * N + (size_t)rb * RPC) * N, BLK, bar);
  };
  int item = blockIdx.x;
  uint32_t ph = 0;
  if (tid == 0 && item < n_items) issue(item);
  float beta = 0.f, alpha = 0.f;
  if (MODE == 1) {   // after pdl_wait: written by the previous CG scalar kernel
    alpha = (float)cg_ab[0];
    beta = (float)cg_ab[1];
  }
  float2* myex = ex + rloc * Rc::EX;
  for (; item < n_items; item += gridDim.x) {
    const int c = item % C, rb = (item / C) % NRB, bl = item / (C * NRB);
    const int iy = rb * RPC + rloc;
    const float dy = sdap[iy];
    mbar_wait(bar, ph);
    ph ^= 1;
    float2 v[A][P];
    double pp = 0.0;   // ||p'||^2 of this thread's pixels (MODE 1)
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) {
        if (n1 < P / 4 || n1 >= 3 * P / 4) {
          const int ix = grid_to_img<G>(Q * n1 + n2);
          float2 img;
          if (MODE == 0) {
            img = xs[rloc * N + ix];
          } else {   // fused CG vector update
            const float2 rv = xs[rloc * N + ix], pv = xs[RPC * N + rloc * N + ix], xv = xs[2 * RPC * N + rloc * N + ix];
            img = caxpy(beta, pv, rv);
            const size_t gi = ((size_t)(l0 + bl) * N + iy) * N + ix;
            cg_p[gi] = img;
            cg_x[gi] = caxpy(alpha, pv, xv);
            pp += (double)img.x * img.x + (double)img.y * img.y;
          }
          float2 val = cscale(img, dy * sdap[ix]);
          if (p.coils) val = cmul(val, cs[rloc * N + ix]);
          v[a][n1] = val;
        } else {
          v[a][n1] = make_float2(0.f, 0.f);
        }
      }
    }
    if (MODE == 1 && pn) {   // per-warp partial of ||p'||^2 (summed in a fixed order by k_reduce_pq)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pp += __shfl_xor_sync(0xffffffffu, pp, o);
      if ((tid & 31) == 0) pn[((size_t)l0 * NRB + item) * (kRowThreads / 32) + (tid >> 5)] = make_double2(pp, 0.0);
    }
    __syncthreads();   // staging consumed: prefetch the next item behind this item's FFT
    if (tid == 0 && item + (int)gridDim.x < n_items) {
      fence_proxy_async();
      issue(item + gridDim.x);
    }
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
      dft_halfzero<P, -1>(v[a]);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) myex[n2 * (P + 1) + k1] = cmul(v[a][k1], stw[k1 * Q + n2]);
    }
    __syncwarp();
    const size_t fc = (size_t)bl * C + c;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      float2 w[Q];
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) w[n2] = myex[n2 * (P + 1) + k1];
      dft<Q, -1>(w);
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) {
        const int gx = k1 + P * k2;
        H[((fc * S + gx / SW) * N + iy) * SW + (gx % SW)] = w[k2];
      }
    }
    __syncwarp();
  }
}

// ============================================================================ forward columns
// Items (fc, strip).  y (frame l0's first sample) must be zeroed: each point's partial sums from
// its (at most two) strips are added with fp32 atomics onto 0, which is order independent.
// Pipeline: the next H strip is fetched right after this item's strip is in registers; the next
// chunk (point records) right after this item's gather.
template <int G>
__global__ void __launch_bounds__(SW * FFTShape<G>::T, (G >= 1024 ? 1 : 2))
k_fwd_cols(DevPlan p, const float2* __restrict__ H, float2* __restrict__ y, int l0, int nb, int stage_cap) {
  using F = FFTShape<G>;
  constexpr int P = F::P, Q = F::Q, T = F::T, N = G / 2, A = Q / T, B = P / T, S = G / SW;
  constexpr uint32_t STRIP_IN = N * SW * sizeof(float2);
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* stw = reinterpret_cast<float2*>(smraw);
  float2* inb = stw + G;
  float2* strip = inb + N * SW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(strip + G * SWG + SW);   // H, chunk (after the pad)
  int* stage = reinterpret_cast<int*>(bars + 2);
  __shared__ int copied;                                             // bytes of the staged chunk
  __shared__ int fchunk_off;                                         // word offset of the staged chunk
  const int C = p.C, W = p.W, recw = p.recw;
  const int n_items = nb * C * S;
  const int tid = threadIdx.x, c = tid % SW, t = tid / SW;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < G; i += blockDim.x) stw[i] = p.tw[i];
  for (int i = tid; i < G * SWG + SW; i += blockDim.x) strip[i] = make_float2(0.f, 0.f);   // skew slots and pad
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();
  auto chunk_of = [&](int item) -> int2 {
    const int fc = item / S, s = item % S;
    return __ldg(p.ftab + __ldg(p.fil + l0 + fc / C) * S + s);
  };
  auto issue_in = [&](int item) {
    mbar_expect_tx(&bars[0], STRIP_IN);
    bulk_g2s(inb, H + (size_t)item * (N * SW), STRIP_IN, &bars[0]);
  };
  auto issue_chunk = [&](int2 ow) {   // records beyond the staging capacity are read from L2
    const uint32_t bytes = (uint32_t)min(stage_cap, ow.y * 4) & ~15u;
    copied = (int)bytes;
    fchunk_off = ow.x;
    mbar_expect_tx(&bars[1], bytes);
    bulk_g2s(stage, p.fchunks + ow.x, bytes, &bars[1]);
  };
  int item = blockIdx.x;
  int2 off_next = make_int2(0, 0);
  PhaseTimer pt;
  pt.start(MRF_DBG_ON(2) && tid == 0);
  int nit = 0;
  if (tid == 0 && item < n_items) {
    issue_in(item);
    issue_chunk(chunk_of(item));
    if (item + (int)gridDim.x < n_items) off_next = chunk_of(item + gridDim.x);
  }
  for (int k = 0; item < n_items; item += gridDim.x, ++k) {
    const int fc = item / S;
    const int next = item + gridDim.x;
    mbar_wait(&bars[0], k & 1);
    pt.mark(0);
    ++nit;
    float2 v[A][P];
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) {
        v[a][n1] = (n1 < P / 4 || n1 >= 3 * P / 4) ? inb[grid_to_img<G>(Q * n1 + n2) * SW + c] : make_float2(0.f, 0.f);
      }
    }
    __syncthreads();
    if (tid == 0 && next < n_items) {
      fence_proxy_async();
      issue_in(next);
    }
    pt.mark(1);
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
      dft_halfzero<P, -1>(v[a]);
#pragma unroll
      for (int k1 = 0; k1 < P; k1 += 2) {
        const float4 tt = tw_pair(stw, n2 * P + k1);
        strip[(n2 * P + k1) * SW + c] = cmul(v[a][k1], make_float2(tt.x, tt.y));
        strip[(n2 * P + k1 + 1) * SW + c] = cmul(v[a][k1 + 1], make_float2(tt.z, tt.w));
      }
    }
    __syncthreads();
    pt.mark(2);
    float2 w[B][Q];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) w[b][n2] = strip[(n2 * P + k1) * SW + c];
    }
    __syncthreads();
    pt.mark(3);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      dft<Q, -1>(w[b]);
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) strip[(k1 + P * k2) * SWG + c] = w[b][k2];   // strip [gy][c]
    }
    __syncthreads();
    pt.mark(4);
    // a3: KB gather interpolation, one thread per point record of the strip (records past the
    // staging capacity are read from L2).
    mbar_wait(&bars[1], k & 1);
    pt.mark(5);
    if (!MRF_DBG_ON(1)) {
      const int n_rec = stage[0];
      // records in groups of 32, each group's records interleaved by 16-byte pieces (a warp's
      // piece-k loads are one contiguous 512-byte span); whole groups are staged
      const int n_st = ((copied / 4 - kChunkHdr) / (32 * recw)) * 32;
      const int* recs = stage + kChunkHdr;
      const int* grecs = p.fchunks + fchunk_off + kChunkHdr;
      float2* yf = y + (size_t)fc * p.M;
      for (int e = tid; e < n_rec; e += blockDim.x) {
        const int ro = (e >> 5) * recw * 32 + (e & 31) * 4;   // word offset of the record's piece 0
        if (W == 6) {
          if (e < n_st) gather_rec<G, 6, false>(recs + ro, strip, yf, p.M);
          else gather_rec<G, 6, true>(grecs + ro, strip, yf, p.M);
        } else if (W == 8) {
          if (e < n_st) gather_rec<G, 8, false>(recs + ro, strip, yf, p.M);
          else gather_rec<G, 8, true>(grecs + ro, strip, yf, p.M);
        } else {
          gather_rec_any<G>((e < n_st ? recs : grecs) + ro, W, strip, yf, p.M);
        }
      }
    }
    pt.mark(6);
    __syncthreads();
    pt.mark(7);
    if (tid == 0 && next < n_items) {
      fence_proxy_async();
      issue_chunk(off_next);
      if (next + (int)gridDim.x < n_items) off_next = chunk_of(next + gridDim.x);
    }
  }
  pt.report(p.dbgbuf, nit);
}

// a4 inner loop, the strip's SELL-32 spread matrix (lane = strip cell).  On a spiral most slices
// have width 1 (MRF: 87 %), so the chunk stores their entries first as one flat run: a thread per
// cell, no slice table.  The n_multi wider slices follow, one warp per slice, entry k of lane l at
// first + 32k + l.  Every cell is written exactly once.  YS: y[fc] staged in shared memory.
// PASS 0: the flat run and the wide slices whose entries are staged (entries at ents[e]);
// PASS 1: wide slices [sl_lo, sl_hi) past the staged prefix, whose entries a further bulk copy
// brought to ents[e - e0] (from_l2: one slice too wide for the buffer, read from L2).
// PASS 2: as PASS 1 with every entry read from L2 (the direct path of oversized chunks, eight loads
// in flight per lane).
template <bool YS, int PASS>
__device__ __forceinline__ void spread_cells(const int2* sl_tab, const unsigned short* cells, const int2* ents,
                                             const int2* __restrict__ gents, int n_staged, int e0, int sl_lo,
                                             int sl_hi, bool from_l2, int nsl, int n_multi, const float2* ys,
                                             const float2* __restrict__ yf, float2* strip, int tid, int nthreads,
                                             int warp, int nwarps, int lane, int M, int ncell, int nent) {
  (void)M; (void)ncell; (void)nent;   // bounds of the checks build (MRF_CHECK)
  if (PASS == 0) {
    const int n1 = (nsl - n_multi) * 32;
    const unsigned short* cells1 = cells + n_multi * 32;
    // four cells per thread in flight: all index / entry loads, then the y loads, then the stores
    // (the strip and the staged tables are disjoint, so hoisting the loads is safe)
    int i = tid;
    for (; i + 3 * nthreads < n1; i += 4 * nthreads) {
      int cl[4];
      int2 e[4];
      float2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ii = i + u * nthreads;
        MRF_CHECK(ii < nent);
        cl[u] = cells1[ii];
        e[u] = ii < n_staged ? ents[ii] : __ldg(gents + ii);
        MRF_CHECK((unsigned)e[u].x < (unsigned)M && (cl[u] == 0xFFFF || cl[u] < ncell));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = YS ? ys[e[u].x] : __ldg(yf + e[u].x);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (cl[u] != 0xFFFF) strip[cl[u]] = cscale(v[u], __int_as_float(e[u].y));
    }
    for (; i < n1; i += nthreads) {
      MRF_CHECK(i < nent);
      const int cell = cells1[i];
      const int2 e = i < n_staged ? ents[i] : __ldg(gents + i);
      MRF_CHECK((unsigned)e.x < (unsigned)M && (cell == 0xFFFF || cell < ncell));
      const float wgt = __int_as_float(e.y);
      const float2 v = YS ? ys[e.x] : __ldg(yf + e.x);
      if (cell != 0xFFFF) strip[cell] = cscale(v, wgt);
    }
    sl_lo = 0;
    sl_hi = n_multi;
  }
  for (int sl = sl_lo + warp; sl < sl_hi; sl += nwarps) {
    const int2 si = sl_tab[sl];
    const int width = abs(si.y);   // si.y < 0: the 32 lanes share one cell (warp reduction)
    if (PASS == 0 && si.x + 32 * width > n_staged) break;   // firsts increase with sl
    const int cell = cells[sl * 32 + lane];
    MRF_CHECK(cell == 0xFFFF || cell < ncell);
    MRF_CHECK(si.x + 32 * width <= nent);
    float2 acc = make_float2(0.f, 0.f);
    if (!from_l2) {
      const int2* ep = ents + (si.x - e0) + lane;
      int kk = 0;
      for (; kk + 3 < width; kk += 4) {   // loads first, the sum in entry order (deterministic)
        int2 e[4];
        float2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          e[u] = ep[(kk + u) * 32];
          MRF_CHECK((unsigned)e[u].x < (unsigned)M);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = YS ? ys[e[u].x] : __ldg(yf + e[u].x);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = caxpy(__int_as_float(e[u].y), v[u], acc);
      }
      for (; kk < width; ++kk) {
        const int2 e = ep[kk * 32];
        const float wgt = __int_as_float(e.y);
        acc = caxpy(wgt, YS ? ys[e.x] : __ldg(yf + e.x), acc);
      }
    } else {
      const int2* ep = gents + si.x + lane;
      int kk = 0;
      if (PASS == 2) {   // (the direct path of oversized chunks)
        for (; kk + 7 < width; kk += 8) {   // eight L2 loads in flight, the sum in entry order
          int2 e[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            e[u] = __ldg(ep + (kk + u) * 32);
            MRF_CHECK((unsigned)e[u].x < (unsigned)M);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = caxpy(__int_as_float(e[u].y), YS ? ys[e[u].x] : __ldg(yf + e[u].x), acc);
        }
        if (kk < width) {   // the last (width % 8) steps: their loads in flight together as well
          int2 e[7];
#pragma unroll
          for (int u = 0; u < 7; ++u)
            if (kk + u < width) e[u] = __ldg(ep + (kk + u) * 32);
#pragma unroll
          for (int u = 0; u < 7; ++u)
            if (kk + u < width) {
              MRF_CHECK((unsigned)e[u].x < (unsigned)M);
              acc = caxpy(__int_as_float(e[u].y), YS ? ys[e[u].x] : __ldg(yf + e[u].x), acc);
            }
          kk = width;
        }
      }
#pragma unroll 4
      for (; kk < width; ++kk) {
        const int2 e = __ldg(ep + kk * 32);
        const float wgt = __int_as_float(e.y);
        acc = caxpy(wgt, YS ? ys[e.x] : __ldg(yf + e.x), acc);
      }
    }
    if (si.y < 0) {   // warp-uniform
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (lane == 0) strip[cell] = acc;
    } else if (cell != 0xFFFF) {
      strip[cell] = acc;
    }
  }
}

// ============================================================================ adjoint columns
// Items (fc, strip).  a4: KB spreading as an output-stationary sparse product: lane = strip cell,
// summing w * y_j over its (j, w) list (SELL-32 slices, no atomics, deterministic);
// a5: column iFFT, then the N kept rows are stored strip-major H[fc][strip][iy][16].
// Pipeline: y[fc] and the chunk of the next item are fetched right after this item's spread.
// T2 (G = 512, SEP): two threads per stage-2 transform, 32 threads per column (16 warps per CTA
// instead of 8 at the same shared-memory footprint).  Stage 1 is one P-point DFT per thread; in
// stage 2 the lane pair (l, l ^ 16) splits the radix-4 decimation of the Q-point DFT -- lane half
// h owns the sub-transforms of n2 = h, h + 2 (mod 4) -- and exchanges the half-combined values by
// shuffle; the operations and their order per output are those of dft_halfout, so the two
// variants agree bit for bit.
template <int G, bool SEP, bool DYN, bool T2 = false>
__global__ void __launch_bounds__(SW * FFTShape<G>::T * (T2 ? 2 : 1), (SEP || G >= 1024) ? 1 : 2)
k_adj_cols(DevPlan p, const float2* __restrict__ y, float2* __restrict__ H, int l0, int nb, int ystage, int stage_cap,
           int* __restrict__ ctr) {
  // DYN: after its first item (blockIdx.x) a CTA takes the next unclaimed item from the
  // counter ctr[0] (dynamic hand-out: the strips differ in spread work, and a static round-robin
  // left the SMs' busy time spread 69 k .. 95 k cycles around an 82 k mean); the last CTA to exit
  // (ctr[1]) resets both words for the next launch on this lane.
  using F = FFTShape<G>;
  constexpr int P = F::P, Q = F::Q, T = F::T * (T2 ? 2 : 1), N = G / 2, A = Q / T, B = T2 ? 1 : P / T, S = G / SW;
  static_assert(!T2 || (SEP && T == Q && Q == 32 && 2 * P == T), "T2: G = 512 with the separate exchange buffer");
  // SEP (G <= 512): the spread strip S and the FFT exchange buffer E are separate, so S only ever
  // holds spread values and zeros: the stage-1 loads skip the row pairs the chunk's row mask marks
  // untouched and re-zero only the touched ones, and the stage-1 twiddles live in registers.
  // G = 1024 (two 128 KB buffers do not fit) exchanges through S and re-zeroes it in full.
  static_assert(!SEP || G <= 512, "two 128 KB strips do not fit");
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* stw = reinterpret_cast<float2*>(smraw);                 // twiddles (!SEP only)
  float2* strip = stw + (SEP ? 0 : G);
  float2* ex = SEP ? strip + G * SW : strip;
  float2* ys = strip + (SEP ? 2 : 1) * G * SW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(ys) + ystage);
  int* stage = reinterpret_cast<int*>(bars + 2);
  __shared__ int copied;
  __shared__ int chunk_off;    // word offset of the staged chunk (for its unstaged tail)
  __shared__ int chunk_words;  // its size
  __shared__ int4 win;         // {e0, slice end, from-L2 flag}: the current window of wide slices
  const int C = p.C, M = p.M;
  const int n_items = nb * C * S;
  const int tid = threadIdx.x, c = tid % SW, t = tid / SW;
  const int warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  int n_tail = 0;   // second copies issued by this CTA (mbarrier parity)
  float2 twr[SEP ? A : 1][SEP ? P : 1];   // stage-1 twiddles W_G^{n2 k1} of this thread (SEP)
  if constexpr (SEP) {
#pragma unroll
    for (int a = 0; a < A; ++a)
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) twr[a][k1] = __ldg(p.tw + (t + T * a) * P + k1);
  } else {
    for (int i = tid; i < G; i += blockDim.x) stw[i] = p.tw[i];
  }
  for (int i = tid; i < G * SW; i += blockDim.x) strip[i] = make_float2(0.f, 0.f);
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();
  auto chunk_of = [&](int item) -> int2 {
    const int fc = item / S, s = item % S;
    return __ldg(p.atab + __ldg(p.fil + l0 + fc / C) * S + s);
  };
  auto issue = [&](int item, int2 ow) {   // the part of a chunk beyond the staging buffer is read from L2
    const uint32_t bytes = (uint32_t)min(ow.y * 4, stage_cap) & ~15u;
    copied = (int)bytes;
    chunk_off = ow.x;
    chunk_words = ow.y;
    mbar_expect_tx(&bars[0], bytes + (uint32_t)ystage);
    bulk_g2s(stage, p.achunks + ow.x, bytes, &bars[0]);
    if (ystage) bulk_g2s(ys, y + (size_t)(item / S) * M, (uint32_t)ystage, &bars[0]);
  };
  __shared__ int s_next[2];   // the CTA's next item, by item parity (written by thread 0)
  int item = blockIdx.x;
  int2 off_next = make_int2(0, 0);
  PhaseTimer pt;
  pt.start(MRF_DBG_ON(2) && tid == 0);
  int nit = 0;
  int pend = 0;   // (thread 0, DYN) the hand-out claimed two items ahead: its latency hides behind an item
  if constexpr (DYN) {
    if (tid == 0) {
      const int nx = (int)gridDim.x + atomicAdd(ctr, 1);
      pend = (int)gridDim.x + atomicAdd(ctr, 1);
      s_next[0] = nx;
      if (item < n_items) {
        issue(item, chunk_of(item));
        if (nx < n_items) off_next = chunk_of(nx);
      }
    }
  } else if (tid == 0 && item < n_items) {
    issue(item, chunk_of(item));
    if (item + (int)gridDim.x < n_items) off_next = chunk_of(item + gridDim.x);
  }
  for (int k = 0; item < n_items; item += gridDim.x, ++k) {
    const int fc = item / S;
    const int snext = item + gridDim.x;   // the static round-robin's next item
    int next = snext;
    mbar_wait(&bars[0], k & 1);
    pt.mark(0);
    ++nit;
    // row-pair mask of this warp's stage-1 loads: bit a*P + n1 <=> rows Q n1 + T a + 2 warp + {0,1}
    // received spread values (read before the staging buffer is refilled)
    // (T2: warp w holds n2 = 2w + {0,1} = T' a + 2w' + {0,1} of the 8-warp layout, a = w >> 3, w' = w & 7)
    const uint32_t rmask = !SEP ? ~0u
                           : T2 ? ((uint32_t)stage[kChunkHdr + (warp & 7)] >> (P * (warp >> 3))) & ((1u << P) - 1u)
                                : (uint32_t)stage[kChunkHdr + warp];
    {
      // Staged prefix of the chunk: header, slice table and cells always fit (checked at plan
      // time); a slice whose entries lie past the staged prefix reads them from L2.
      const int nsl = MRF_DBG_ON(1) ? 0 : stage[0], cells_off = stage[1], ent_off = stage[2];
      const int n_multi = MRF_DBG_ON(1) ? 0 : stage[3];
      const float2* yf = y + (size_t)fc * M;
      const int2* sl_tab = reinterpret_cast<const int2*>(stage + kAdjHdr);
      const unsigned short* cells = reinterpret_cast<const unsigned short*>(stage + cells_off);
      const int2* ents = reinterpret_cast<const int2*>(stage + ent_off);
      MRF_CHECK(cells_off >= kAdjHdr && ent_off >= cells_off && ent_off * 4 <= copied && copied <= chunk_words * 4);
      MRF_CHECK(nsl >= n_multi && n_multi >= 0 && (chunk_words - ent_off) / 2 >= 32 * (nsl - n_multi));
      const int n_staged = (copied / 4 - ent_off) / 2;          // entries in shared memory
      const int2* gents = reinterpret_cast<const int2*>(p.achunks + chunk_off + ent_off);
      if (ystage)
        spread_cells<true, 0>(sl_tab, cells, ents, gents, n_staged, 0, 0, 0, false, nsl, n_multi, ys, yf, strip, tid,
                              blockDim.x, warp, nwarps, lane, M, G * SW, (chunk_words - ent_off) / 2);
      else
        spread_cells<false, 0>(sl_tab, cells, ents, gents, n_staged, 0, 0, 0, false, nsl, n_multi, ys, yf, strip,
                               tid, blockDim.x, warp, nwarps, lane, M, G * SW, (chunk_words - ent_off) / 2);
      if (copied < chunk_words * 4) {   // chunk larger than the staging buffer (block-uniform)
        // The wide slices past the staged prefix: windows of whole slices brought in by further
        // bulk copies over the (consumed) entry region; a slice wider than the region reads L2.
        const int cap = (copied / 4 - ent_off) / 2;          // entries that fit
        const int nent = (chunk_words - ent_off) / 2;
        // first wide slice whose entries are not all staged (slice ends increase with the slice
        // index: binary search, a dense chunk has hundreds of slices)
        int sl0 = 0;
        for (int hi = n_multi; sl0 < hi;) {
          const int mid = (sl0 + hi) >> 1;
          const int2 sm = sl_tab[mid];
          if (sm.x + 32 * abs(sm.y) <= n_staged) sl0 = mid + 1;
          else hi = mid;
        }
        // A chunk that needs more than one further window (the centre strips of a dense spiral:
        // stress) reads the rest of its slices straight from L2, eight loads in flight per lane,
        // instead of streaming windows (two barriers and a copy round trip each); one window
        // is still cheaper than L2 latency (measured: stress normal -4 %, MRF unchanged).
        // (With the direct path's loads batched eight deep through the slice tails, it also beats the
        // single window: MRF adjoint 0.951 -> 0.943 ms; MRF_DBG=8 of the experiment build restores
        // the windows for overflows of at most one window.)
        const bool direct = !MRF_DBG_ON(8) || (nent - n_staged > cap);
        if (direct) {
          if (ystage)
            spread_cells<true, 2>(sl_tab, cells, ents, gents, n_staged, 0, sl0, n_multi, true, nsl, n_multi, ys, yf,
                                  strip, tid, blockDim.x, warp, nwarps, lane, M, G * SW, (chunk_words - ent_off) / 2);
          else
            spread_cells<false, 2>(sl_tab, cells, ents, gents, n_staged, 0, sl0, n_multi, true, nsl, n_multi, ys, yf,
                                   strip, tid, blockDim.x, warp, nwarps, lane, M, G * SW, (chunk_words - ent_off) / 2);
          sl0 = n_multi;
        }
        while (sl0 < n_multi) {   // sl0 is block-uniform
          __syncthreads();        // the previous window's entries are consumed
          if (tid == 0) {
            const int e0 = sl_tab[sl0].x, e1 = min(nent, e0 + cap);
            int hi = sl0;
            while (hi < n_multi && sl_tab[hi].x + 32 * abs(sl_tab[hi].y) <= e1) ++hi;
            const bool big = hi == sl0;
            win = make_int4(e0, hi == sl0 ? sl0 + 1 : hi, big ? 1 : 0, 0);
            if (!big) {
              const uint32_t bytes = (uint32_t)(sl_tab[hi - 1].x + 32 * abs(sl_tab[hi - 1].y) - e0) * 8u;
              fence_proxy_async();
              mbar_expect_tx(&bars[1], bytes);
              bulk_g2s(stage + ent_off, p.achunks + chunk_off + ent_off + 2 * e0, bytes, &bars[1]);
            }
          }
          __syncthreads();
          const int4 wv = win;
          if (!wv.z) {
            mbar_wait(&bars[1], n_tail & 1);
            ++n_tail;
          }
          if (ystage)
            spread_cells<true, 1>(sl_tab, cells, ents, gents, n_staged, wv.x, sl0, wv.y, wv.z != 0, nsl, n_multi, ys,
                                  yf, strip, tid, blockDim.x, warp, nwarps, lane, M, G * SW, (chunk_words - ent_off) / 2);
          else
            spread_cells<false, 1>(sl_tab, cells, ents, gents, n_staged, wv.x, sl0, wv.y, wv.z != 0, nsl, n_multi, ys,
                                   yf, strip, tid, blockDim.x, warp, nwarps, lane, M, G * SW, (chunk_words - ent_off) / 2);
          sl0 = wv.y;
        }
      }
    }
    pt.mark(1);
    __syncthreads();
    pt.mark(2);
    if (DYN) next = s_next[k & 1];   // written by thread 0 before the barrier above
    if (tid == 0 && next < n_items) {
      fence_proxy_async();
      issue(next, off_next);
      if constexpr (DYN) {
        const int nn = pend;
        pend = (int)gridDim.x + atomicAdd(ctr, 1);
        s_next[(k + 1) & 1] = nn;
        if (nn < n_items) off_next = chunk_of(nn);
      } else {
        if (next + (int)gridDim.x < n_items) off_next = chunk_of(next + gridDim.x);
      }
    }
    // a5: column inverse FFT (e^{+i}, unnormalised); only the N kept rows are stored
    float2 v[A][P];
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) {
        if constexpr (SEP) {   // each cell is read by its one owner, who re-zeroes it for the next spread
          if ((rmask >> (a * P + n1)) & 1u) {
            float2& cell = strip[sidx(Q * n1 + n2, c)];
            v[a][n1] = cell;
            cell = make_float2(0.f, 0.f);
          } else {
            v[a][n1] = make_float2(0.f, 0.f);
          }
        } else {
          v[a][n1] = strip[sidx(Q * n1 + n2, c)];
        }
      }
    }
    if constexpr (!SEP) __syncthreads();   // the exchange below overwrites the strip
    pt.mark(3);
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
      dft<P, +1>(v[a]);
#pragma unroll
      for (int k1 = 0; k1 < P; k1 += 2) {
        float2 t0, t1;
        if constexpr (SEP) {
          t0 = twr[a][k1];
          t1 = twr[a][k1 + 1];
        } else {
          const float4 tt = tw_pair(stw, n2 * P + k1);
          t0 = make_float2(tt.x, tt.y);
          t1 = make_float2(tt.z, tt.w);
        }
        ex[(n2 * P + k1) * SW + c] = cmulc(v[a][k1], t0);
        ex[(n2 * P + k1 + 1) * SW + c] = cmulc(v[a][k1 + 1], t1);
      }
    }
    __syncthreads();
    pt.mark(4);
    float2* Hc = H + (size_t)fc * N * G + (size_t)(item % S) * SW + c;    // row-major [fc][iy][G]
    if constexpr (T2) {
      // lane half h = t & 1 (lanes l and l ^ 16 share k1 = t >> 1): sub-transforms q = h and h + 2 of
      // the radix-4 decimation in time, D_q[K] = sum_i ex[n2 = 4 i + q] W_8^{iK}
      const int h = t & 1, k1 = t >> 1;
      float2 da[Q / 4], db[Q / 4];
#pragma unroll
      for (int i = 0; i < Q / 4; ++i) {
        da[i] = ex[((4 * i + h) * P + k1) * SW + c];
        db[i] = ex[((4 * i + h + 2) * P + k1) * SW + c];
      }
      pt.mark(5);
      dft<Q / 4, +1>(da);
      dft<Q / 4, +1>(db);
      float2 out[Q / 4];
      detail::t2_combine<Q, +1, 0>(out, da, db, h);
#pragma unroll
      for (int K = 0; K < Q / 4; ++K) {
        const int k2 = h ? K + 3 * Q / 4 : K;
        __stcs(&Hc[(size_t)grid_to_img<G>(k1 + P * k2) * G], out[K]);
      }
    } else {
    float2 w[B][Q];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) {
        float2& cell = ex[(n2 * P + k1) * SW + c];
        w[b][n2] = cell;
        if constexpr (!SEP) cell = make_float2(0.f, 0.f);   // owner re-zeroes for the next spread
      }
    }
    pt.mark(5);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      dft_halfout<Q, +1>(w[b]);
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) {
        // streaming store: the half grid is read once, a batch later, and should not displace the
        // plan tables in L2 (adjoint 0.901 -> 0.890 ms; the same hint on k_fwd_rows' stores lost 0.3 %)
        if (k2 < Q / 4 || k2 >= 3 * Q / 4) __stcs(&Hc[(size_t)grid_to_img<G>(k1 + P * k2) * G], w[b][k2]);
      }
    }
    }
    pt.mark(6);
    // !SEP: zero-fill visible before the next spread.  SEP: the next item's spread and exchange are
    // ordered by its own first barrier (every thread is past its stage-2 loads by then).
    if constexpr (!SEP) __syncthreads();
    pt.mark(7);
    if constexpr (DYN) item = next - (int)gridDim.x;   // (the loop adds gridDim.x back)
  }
  pt.report(p.dbgbuf ? p.dbgbuf + 16 : nullptr, nit);
  if (DYN && tid == 0) {   // the last CTA out resets the hand-out counter
    __threadfence();
    if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
}

// ============================================================================ Toeplitz columns
// the normal operator A^H A x = sum_c conj(S_c) crop(IFFT(T ⊙ FFT(pad(S_c x))))
// with T the (real) 2N-point spectrum of the point-spread function of the interleaf
// (plan-time, see k_psf_*).  Items (fc, strip): forward column FFT of the strip (pruned input),
// multiply by T in registers, inverse column FFT computed in the transposed split
// (stage A = Q-point inverse DFTs over k2 on the forward's own output layout, so no exchange is
// needed between the two transforms; one exchange; stage B = P-point inverse DFTs over k1), and
// the N kept rows are stored row-major for k_adj_rows.  No gather, no spread, no k-space buffer.
template <int G>
__global__ void __launch_bounds__(SW * FFTShape<G>::T, (G >= 1024 ? 1 : 2))
k_toep_cols(DevPlan p, const float2* __restrict__ Hf, float2* __restrict__ Ha, const float* __restrict__ psf, int l0,
            int nb, double2* __restrict__ tq) {
  using F = FFTShape<G>;
  constexpr int P = F::P, Q = F::Q, T = F::T, N = G / 2, A = Q / T, B = P / T, S = G / SW;
  constexpr uint32_t STRIP_IN = N * SW * sizeof(float2);
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* stw = reinterpret_cast<float2*>(smraw);
  float2* inb = stw + G;
  float2* ex = inb + N * SW;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ex + G * SW);
  const int C = p.C;
  const int n_items = nb * C * S;
  const int tid = threadIdx.x, c = tid % SW, t = tid / SW;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < G; i += blockDim.x) stw[i] = p.tw[i];
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();
  auto issue_in = [&](int item) {
    mbar_expect_tx(bar, STRIP_IN);
    bulk_g2s(inb, Hf + ((size_t)item_fc(p.perm, C, item, S, l0) * S + item % S) * (N * SW), STRIP_IN, bar);
  };
  int item = blockIdx.x;
  if (tid == 0 && item < n_items) issue_in(item);
  for (int k = 0; item < n_items; item += gridDim.x, ++k) {
    const int fc = item_fc(p.perm, C, item, S, l0), s = item % S;
    double tpx = 0.0;
    const int next = item + gridDim.x;
    // PSF values at this thread's forward-output rows k1 + P k2: issued now, used after the FFT
    const int r = __ldg(p.fil + l0 + fc / C);
    const float* ps = psf + ((size_t)(r * S + s) * G) * SW + c;
    float tp[B][Q];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) tp[b][k2] = __ldg(ps + (size_t)(t + T * b + P * k2) * SW);
    mbar_wait(bar, k & 1);
    float2 v[A][P];
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) {
        v[a][n1] = (n1 < P / 4 || n1 >= 3 * P / 4) ? inb[grid_to_img<G>(Q * n1 + n2) * SW + c] : make_float2(0.f, 0.f);
      }
    }
    __syncthreads();
    if (tid == 0 && next < n_items) {
      fence_proxy_async();
      issue_in(next);
    }
    // forward column FFT
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
      dft_halfzero<P, -1>(v[a]);
#pragma unroll
      for (int k1 = 0; k1 < P; k1 += 2) {
        const float4 tt = tw_pair(stw, n2 * P + k1);
        ex[(n2 * P + k1) * SW + c] = cmul(v[a][k1], make_float2(tt.x, tt.y));
        ex[(n2 * P + k1 + 1) * SW + c] = cmul(v[a][k1 + 1], make_float2(tt.z, tt.w));
      }
    }
    __syncthreads();
    float2 w[B][Q];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) w[b][n2] = ex[(n2 * P + k1) * SW + c];
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      dft<Q, -1>(w[b]);                          // w[b][k2] = X[k1 + P k2]
      if (tq) {   // Parseval: <p, A^H A p> = sum_k T(k) |X(k)|^2 (split-phase CG, reading 30)
#pragma unroll
        for (int k2 = 0; k2 < Q; ++k2)
          tpx += (double)tp[b][k2] * ((double)w[b][k2].x * w[b][k2].x + (double)w[b][k2].y * w[b][k2].y);
      }
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) w[b][k2] = cscale(w[b][k2], tp[b][k2]);
      dft<Q, +1>(w[b]);                          // stage A of the inverse: index n2
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) ex[(n2 * P + k1) * SW + c] = cmulc(w[b][n2], stw[n2 * P + k1]);
    }
    if (tq) {   // one partial per warp and item, summed in a fixed order by k_reduce_pq
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tpx += __shfl_xor_sync(0xffffffffu, tpx, o);
      if ((tid & 31) == 0) tq[((size_t)l0 * C * S + item) * (blockDim.x >> 5) + (tid >> 5)] = make_double2(tpx, 0.0);
      tpx = 0.0;
    }
    __syncthreads();
    float2* Hc = Ha + (size_t)fc * N * G + (size_t)s * SW + c;    // row-major [fc][iy][G]
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
      float2 u[P];
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) u[k1] = ex[(n2 * P + k1) * SW + c];
      dft_halfout<P, +1>(u);                             // stage B: index n1, row n2 + Q n1
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) {
        if (n1 < P / 4 || n1 >= 3 * P / 4) Hc[(size_t)grid_to_img<G>(n2 + Q * n1) * G] = u[n1];
      }
    }
    __syncthreads();   // exchange buffer free for the next item
  }
}

// ============================================================================ subspace normal
// P_S A^H A in basis coordinates (SURVEY.md §8(f) f2 on a Toeplitz plan): for
// x = sum_i u_i d_i (d: r x L orthonormal rows) the coefficients of P_S(A^H A x) are
//   z_j = sum_i crop F^-1 [K_ji ⊙ F pad(u_i)],   K_ji = sum_rho c^rho_ji T_rho,
//   c^rho_ji = sum_{l : interleaf(l) = rho} conj(d_jl) d_il,
// with T_rho the real PSF spectra of the Toeplitz plan: r row/column FFT pairs and an r x r
// mixing per frequency instead of L frames of A^H A.  The spectra of one (frame, coil) are kept in
// the PSF layout [strip][row][16] (E = G * G elements).
template <int G>
constexpr size_t sn_cols_smem() { return (size_t(G) + size_t(G) * SW) * 8; }

// forward column FFT of the strip-major half grid (pruned input rows), spectrum out
template <int G>
__global__ void __launch_bounds__(SW * FFTShape<G>::T) k_sn_fcols(const float2* __restrict__ tw,
                                                                   const float2* __restrict__ Hf,
                                                                   float2* __restrict__ spec, int nfc) {
  using F = FFTShape<G>;
  constexpr int P = F::P, Q = F::Q, T = F::T, N = G / 2, A = Q / T, B = P / T, S = G / SW;
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* stw = reinterpret_cast<float2*>(smraw);
  float2* ex = stw + G;
  const int tid = threadIdx.x, c = tid % SW, t = tid / SW;
  for (int i = tid; i < G; i += blockDim.x) stw[i] = tw[i];
  __syncthreads();
  for (int item = blockIdx.x; item < nfc * S; item += gridDim.x) {
    const float2* in = Hf + (size_t)item * N * SW;   // [fc][s] strip: N rows x 16
    float2 v[A][P];
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1)
        v[a][n1] = (n1 < P / 4 || n1 >= 3 * P / 4) ? in[grid_to_img<G>(Q * n1 + n2) * SW + c] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
      dft_halfzero<P, -1>(v[a]);
#pragma unroll
      for (int k1 = 0; k1 < P; k1 += 2) {
        const float4 tt = tw_pair(stw, n2 * P + k1);
        ex[(n2 * P + k1) * SW + c] = cmul(v[a][k1], make_float2(tt.x, tt.y));
        ex[(n2 * P + k1 + 1) * SW + c] = cmul(v[a][k1 + 1], make_float2(tt.z, tt.w));
      }
    }
    __syncthreads();
    float2* out = spec + (size_t)item * G * SW;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      float2 w[Q];
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) w[n2] = ex[(n2 * P + k1) * SW + c];
      dft<Q, -1>(w);                                   // w[k2] = X[k1 + P k2]
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) out[(size_t)(k1 + P * k2) * SW + c] = w[k2];
    }
    __syncthreads();
  }
}

// inverse column FFT of a spectrum (the transposed split of k_toep_cols), the N kept rows stored
// row-major [fc][iy][G] for k_adj_rows
template <int G>
__global__ void __launch_bounds__(SW * FFTShape<G>::T) k_sn_icols(const float2* __restrict__ tw,
                                                                   const float2* __restrict__ spec,
                                                                   float2* __restrict__ Ha, int nfc) {
  using F = FFTShape<G>;
  constexpr int P = F::P, Q = F::Q, T = F::T, N = G / 2, A = Q / T, B = P / T, S = G / SW;
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* stw = reinterpret_cast<float2*>(smraw);
  float2* ex = stw + G;
  const int tid = threadIdx.x, c = tid % SW, t = tid / SW;
  for (int i = tid; i < G; i += blockDim.x) stw[i] = tw[i];
  __syncthreads();
  for (int item = blockIdx.x; item < nfc * S; item += gridDim.x) {
    const int fc = item / S, s = item % S;
    const float2* in = spec + (size_t)item * G * SW;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
      float2 w[Q];
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) w[k2] = in[(size_t)(k1 + P * k2) * SW + c];
      dft<Q, +1>(w);                                   // stage A of the inverse: index n2
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) ex[(n2 * P + k1) * SW + c] = cmulc(w[n2], stw[n2 * P + k1]);
    }
    __syncthreads();
    float2* Hc = Ha + (size_t)fc * N * G + (size_t)s * SW + c;
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n2 = t + T * a;
      float2 u[P];
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) u[k1] = ex[(n2 * P + k1) * SW + c];
      dft_halfout<P, +1>(u);                           // stage B: index n1, row n2 + Q n1
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1)
        if (n1 < P / 4 || n1 >= 3 * P / 4) Hc[(size_t)grid_to_img<G>(n2 + Q * n1) * G] = u[n1];
    }
    __syncthreads();
  }
}

// spec_out[j][c][e] = sum_i K[j][i][e] spec_in[i][c][e]   (r x r mixing per frequency; R >= r).
// K is Hermitian in (j, i) (T real, c^rho Hermitian): only j <= i is stored, pair index
// sn_pair(j, i, r) = j r - j (j - 1) / 2 + (i - j), and K_ij = conj(K_ji).
__host__ __device__ __forceinline__ int sn_pair(int j, int i, int r) { return j * r - j * (j - 1) / 2 + (i - j); }

template <int R>
__global__ void __launch_bounds__(256) k_sn_mix(const float2* __restrict__ spec_in, const float2* __restrict__ K,
                                                float2* __restrict__ spec_out, int r, int C, long long E) {
  // each stored pair (j <= i) is loaded once and used twice: out_j += K u_i, out_i += conj(K) u_j
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)C * E) return;
  const int c = (int)(idx / E);
  const long long e = idx % E;
  float2 u[R], acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    u[i] = i < r ? __ldg(spec_in + ((size_t)i * C + c) * E + e) : make_float2(0.f, 0.f);
    acc[i] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int i = j; i < R; ++i)
      if (i < r) {
        const float2 k = __ldg(K + (size_t)sn_pair(j, i, r) * E + e);
        acc[j].x = fmaf(k.x, u[i].x, fmaf(-k.y, u[i].y, acc[j].x));
        acc[j].y = fmaf(k.x, u[i].y, fmaf(k.y, u[i].x, acc[j].y));
        if (i != j) {   // conj(K_ji) u_j
          acc[i].x = fmaf(k.x, u[j].x, fmaf(k.y, u[j].y, acc[i].x));
          acc[i].y = fmaf(k.x, u[j].y, fmaf(-k.y, u[j].x, acc[i].y));
        }
      }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (j < r) spec_out[((size_t)j * C + c) * E + e] = acc[j];
}

// K[pair][e] = sum_rho cc[pair][rho] T_rho[e]  (plan time; pairs j <= i, sn_pair order; T real)
__global__ void __launch_bounds__(256) k_sn_kbuild(const float* __restrict__ psf, const float2* __restrict__ cc,
                                                   int pairs, int R, long long E, float2* __restrict__ K) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)pairs * E) return;
  const int pr = (int)(idx / E);
  const long long e = idx % E;
  float ax = 0.f, ay = 0.f;
  for (int rho = 0; rho < R; ++rho) {
    const float tv = __ldg(psf + (size_t)rho * E + e);
    const float2 cv = __ldg(cc + (size_t)pr * R + rho);
    ax = fmaf(cv.x, tv, ax);
    ay = fmaf(cv.y, tv, ay);
  }
  K[idx] = make_float2(ax, ay);
}

// ---------------------------------------------------------------------------- PSF (plan time)
// T[my][mx] = 1/(G^2 N^2) sum_j D(ky_j - my/G) D(kx_j - mx/G),
// D(theta) = sum_{d=-(N-1)}^{N-1} e^{i 2 pi d theta} = sin((2N-1) pi theta) / sin(pi theta):
// the G-point DFT of the circulant embedding of K(d) = 1/N^2 sum_j e^{+i 2 pi k_j . d}, the
// kernel of A^H A for one coil (K is Hermitian, so T is real).  Float64 throughout.
__global__ void k_psf_dirichlet(const float* __restrict__ traj, int M, int N, int G, int axis, double* __restrict__ D) {
  const long long total = (long long)M * G;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / G), m = (int)(i % G);
    const double th = (double)traj[2 * j + axis] - (double)m / G;
    const double den = sinpi(th);
    D[i] = fabs(den) < 1e-12 ? (double)(2 * N - 1) * cospi(th * (2 * N - 2)) : sinpi((2 * N - 1) * th) / den;
  }
}

// out[my][mx] = scale * sum_j Dy[j][my] Dx[j][mx]  (64 x 64 tile per 256-thread block)
__global__ void __launch_bounds__(256) k_psf_gemm(const double* __restrict__ Dy, const double* __restrict__ Dx, int M,
                                                  int G, double scale, double* __restrict__ out) {
  __shared__ double sy[16][64], sx[16][64];
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  const int my0 = blockIdx.y * 64, mx0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int j0 = 0; j0 < M; j0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int jj = i / 64, mm = i % 64, j = j0 + jj;
      sy[jj][mm] = (j < M && my0 + mm < G) ? Dy[(size_t)j * G + my0 + mm] : 0.0;
      sx[jj][mm] = (j < M && mx0 + mm < G) ? Dx[(size_t)j * G + mx0 + mm] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { a[u] = sy[jj][ty + 16 * u]; b[u] = sx[jj][tx + 16 * u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int my = my0 + ty + 16 * u, mx = mx0 + tx + 16 * v;
      if (my < G && mx < G) out[(size_t)my * G + mx] = scale * acc[u][v];
    }
}

// psf[r][s][my][16] (fp32) <- T[my][mx] (fp64), s = mx / 16
__global__ void k_psf_store(const double* __restrict__ Tm, int G, float* __restrict__ psf_r) {
  const int total = G * G;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int my = i / G, mx = i % G;
    psf_r[((size_t)(mx / SW) * G + my) * SW + (mx % SW)] = (float)Tm[i];
  }
}

// ============================================================================ adjoint rows
// Items (bl, rowblock); coils accumulated in registers.  out = sum_c conj(S_c) crop(rowIFFT(H))
// . dap dap (+ mu xin).  With dot != nullptr also writes the item's float64 partial of
// <xin, out> (the CG inner product <p, q>, fused).
// Split-phase CG (rres != nullptr, C == 1): q = out is not stored; the residual is advanced in
// place, r -= alpha q with alpha = *cg_alpha (computed from ||A p||^2 + mu ||p||^2 before this
// pass), and dot receives the partial of <r, r> of the new residual.  p and r are staged
// single-buffered in the two x slots, prefetched after the previous item's epilogue.
template <int G, bool RU>
__global__ void __launch_bounds__(kRowThreads)
k_adj_rows(DevPlan p, const float2* __restrict__ H, float2* __restrict__ out, const float2* __restrict__ xin,
           float mu, int l0, int nb, double2* __restrict__ dot, float2* __restrict__ rres,
           const double* __restrict__ cg_alpha) {
  using Rc = RowCfg<G>;
  constexpr int P = Rc::P, Q = Rc::Q, T = Rc::T, N = Rc::N, RPC = Rc::RPC, A = Q / T, B = P / T;
  constexpr int NRB = N / RPC;
  constexpr uint32_t HBLK = RPC * G * sizeof(float2);    // the row block of one frame-coil
  constexpr uint32_t XBLK = RPC * N * sizeof(float2);
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* stw = reinterpret_cast<float2*>(smraw);
  float2* hin = stw + G;                 // [RPC][G]
  float2* xs = hin + RPC * G;            // [2][RPC][N]
  float2* ex = xs + 2 * RPC * N;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ex + RPC * Rc::EX);   // H, X0, X1
  float* sdap = reinterpret_cast<float*>(bars + 4);
  __shared__ double2 red[kRowThreads / 32];
  const int C = p.C;
  const int n_items = nb * NRB;
  const int tid = threadIdx.x, rloc = tid / T, t = tid % T, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < G; i += kRowThreads) stw[i] = p.tw[(i % Q) * P + i / Q];   // [k1][n2]: a warp spans n2
  for (int i = tid; i < N; i += kRowThreads) sdap[i] = p.dap[i];
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();
  // sub-item = (item, coil): the H rows of one frame-coil and row block, S chunks of HBLK bytes
  auto issue_h = [&](int item, int c) {   // called by warp 0: the row block is one contiguous copy
    const int rb = item % NRB, bl = item / NRB;
    const size_t fc = (size_t)bl * C + c;
    if (lane == 0) {
      mbar_expect_tx(&bars[0], HBLK);
      bulk_g2s(hin, H + (fc * N + (size_t)rb * RPC) * G, HBLK, &bars[0]);
    }
  };
  auto issue_x = [&](int item, int xb) {   // called by thread 0
    const int rb = item % NRB, bl = item / NRB;
    mbar_expect_tx(&bars[1 + xb], XBLK);
    bulk_g2s(xs + xb * RPC * N, xin + ((size_t)(l0 + bl) * N + (size_t)rb * RPC) * N, XBLK, &bars[1 + xb]);
  };
  auto issue_pr = [&](int item) {   // split-phase CG: p -> slot 0, r -> slot 1 (thread 0)
    const int rb = item % NRB, bl = item / NRB;
    const size_t off = ((size_t)(l0 + bl) * N + (size_t)rb * RPC) * N;
    mbar_expect_tx(&bars[1], XBLK);
    bulk_g2s(xs, xin + off, XBLK, &bars[1]);
    mbar_expect_tx(&bars[2], XBLK);
    bulk_g2s(xs + RPC * N, rres + off, XBLK, &bars[2]);
  };
  const float alpha = RU ? (float)*cg_alpha : 0.f;   // after pdl_wait: written by the alpha step
  int item = blockIdx.x;
  if (warp == 0 && item < n_items) issue_h(item, 0);
  if (tid == 0 && item < n_items) {
    if (RU) issue_pr(item);
    else if (xin) issue_x(item, 0);
  }
  uint32_t hph = 0;
  float2* myex = ex + rloc * Rc::EX;
  for (int k = 0; item < n_items; item += gridDim.x, ++k) {
    const int rb = item % NRB, bl = item / NRB;
    const int iy = rb * RPC + rloc;
    const int next = item + gridDim.x;
    if (!RU && tid == 0 && xin && next < n_items) issue_x(next, (k + 1) & 1);   // buffer freed by item k-1
    float2 acc[B][Q / 2];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int kk = 0; kk < Q / 2; ++kk) acc[b][kk] = make_float2(0.f, 0.f);
    for (int c = 0; c < C; ++c) {
      mbar_wait(&bars[0], hph);
      hph ^= 1;
      float2 v[A][P];
#pragma unroll
      for (int a = 0; a < A; ++a) {
        const int n2 = t + T * a;
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) {
          const int pos = Q * n1 + n2;
          v[a][n1] = hin[rloc * G + pos];
        }
      }
      // this coil's sensitivities at the thread's output pixels: loaded now, used after the FFT
      float2 cv[B][Q / 2];
      if (p.coils) {
        const float2* sr = p.coils + ((size_t)c * N + iy) * N;
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int kk = 0; kk < Q / 2; ++kk)
            cv[b][kk] = __ldg(sr + grid_to_img<G>(t + T * b + P * (kk < Q / 4 ? kk : kk + Q / 2)));
      }
      __syncthreads();
      if (warp == 0) {
        if (c + 1 < C) {
          fence_proxy_async();
          issue_h(item, c + 1);
        } else if (next < n_items) {
          fence_proxy_async();
          issue_h(next, 0);
        }
      }
#pragma unroll
      for (int a = 0; a < A; ++a) {
        const int n2 = t + T * a;
        dft<P, +1>(v[a]);
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) myex[n2 * (P + 1) + k1] = cmulc(v[a][k1], stw[k1 * Q + n2]);
      }
      __syncwarp();
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int k1 = t + T * b;
        float2 w[Q];
#pragma unroll
        for (int n2 = 0; n2 < Q; ++n2) w[n2] = myex[n2 * (P + 1) + k1];
        dft_halfout<Q, +1>(w);
#pragma unroll
        for (int kk = 0; kk < Q / 2; ++kk) {
          const int k2 = kk < Q / 4 ? kk : kk + Q / 2;
          float2 val = w[k2];
          if (p.coils) val = cmulc(val, cv[b][kk]);
          acc[b][kk] = cadd(acc[b][kk], val);
        }
      }
      __syncwarp();
    }
    // a6 epilogue: deapodise, (+ mu x), store, CG partial <xin, out>
    const float dy = sdap[iy];
    const size_t orow0 = ((size_t)(l0 + bl) * N + iy) * N;
    float2* orow = (RU ? rres : out) + orow0;
    const float2* xrow = xs + (RU ? 0 : (k & 1)) * RPC * N + rloc * N;
    const float2* rrow = xs + RPC * N + rloc * N;
    if (RU) {
      mbar_wait(&bars[1], k & 1);
      mbar_wait(&bars[2], k & 1);
    } else if (xin) {
      mbar_wait(&bars[1 + (k & 1)], (k >> 1) & 1);
    }
    double2 d = make_double2(0.0, 0.0);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k1 = t + T * b;
#pragma unroll
      for (int kk = 0; kk < Q / 2; ++kk) {
        const int k2 = kk < Q / 4 ? kk : kk + Q / 2;
        const int ix = grid_to_img<G>(k1 + P * k2);
        float2 o = cscale(acc[b][kk], dy * sdap[ix]);
        if (RU) {   // r' = r - alpha (A^H A p + mu p); <r', r'>
          o = caxpy(mu, xrow[ix], o);
          o = caxpy(-alpha, o, rrow[ix]);
          d.x += (double)o.x * o.x + (double)o.y * o.y;
        } else if (xin) {
          const float2 xv = xrow[ix];
          o = caxpy(mu, xv, o);
          if (dot) {
            d.x += (double)xv.x * o.x + (double)xv.y * o.y;
            d.y += (double)xv.x * o.y - (double)xv.y * o.x;
          }
        }
        orow[ix] = o;
      }
    }
    if (dot) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        d.x += __shfl_xor_sync(0xffffffffu, d.x, o);
        d.y += __shfl_xor_sync(0xffffffffu, d.y, o);
      }
      if (lane == 0) red[warp] = d;
    }
    __syncthreads();   // x block consumed; red complete
    if (RU && tid == 0 && next < n_items) {   // p, r slots free: prefetch the next item's
      fence_proxy_async();
      issue_pr(next);
    }
    if (dot && tid == 0) {
      double2 s = make_double2(0.0, 0.0);
      for (int i = 0; i < kRowThreads / 32; ++i) { s.x += red[i].x; s.y += red[i].y; }
      dot[(size_t)l0 * NRB + item] = s;
    }
  }
}

}  // namespace mrf

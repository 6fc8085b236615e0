// fft.cuh -- register-resident DFT building blocks for the hand-written G x G FFTs (sm_100a).
//
// The 2D DFT of the oversampled grid (the paper's F_u,
// PAPER.md:60) is evaluated as row and column passes of length-G 1D DFTs.  Each length-G DFT is
// a two-stage Cooley-Tukey split G = P * Q executed by T cooperating threads of one warp:
//
//   n = Q n1 + n2,  k = k1 + P k2
//   X[k1 + P k2] = sum_{n2} W_Q^{n2 k2} . W_G^{n2 k1} . sum_{n1} x[Q n1 + n2] W_P^{n1 k1}
//
// stage 1: thread t owns n2 in {t + T a}: a P-point DFT per n2 in registers, times W_G^{n2 k1};
// one exchange through shared memory; stage 2: thread t owns k1 in {t + T b}: a Q-point DFT per
// k1 in registers.  The P-/Q-point DFTs are unrolled at compile time (radix-4 / radix-2
// decimation in time) with constant twiddles evaluated by constexpr Taylor series in double.
#pragma once
#include <cuda_runtime.h>

namespace mrf {

__host__ __device__ constexpr double c_pi() { return 3.14159265358979323846; }

// constexpr cos / sin for |t| <= pi (alternating Taylor series, 40 terms: < 1e-16 abs error).
__host__ __device__ constexpr double c_cos(double t) {
  double term = 1.0, sum = 1.0;
  for (int i = 1; i < 40; ++i) { term *= -t * t / ((2.0 * i - 1.0) * (2.0 * i)); sum += term; }
  return sum;
}
__host__ __device__ constexpr double c_sin(double t) {
  double term = t, sum = t;
  for (int i = 1; i < 40; ++i) { term *= -t * t / ((2.0 * i) * (2.0 * i + 1.0)); sum += term; }
  return sum;
}

// W_R^K = exp(SIGN * i * 2 pi K / R), K reduced to (-R/2, R/2].
template <int R, int K, int SIGN>
struct Tw {
  static constexpr int Kr = (K % R) > R / 2 ? (K % R) - R : (K % R);
  static constexpr double ang = SIGN * 2.0 * c_pi() * double(Kr) / double(R);
  static constexpr double c = c_cos(ang);
  static constexpr double s = c_sin(ang);
};

// ---- complex arithmetic on the packed FP32x2 pipe (sm_100: FADD2 / FMUL2 / FFMA2) -------------
// One instruction operates on both halves of a 64-bit register pair, so a complex addition is one
// instruction instead of two, a complex multiplication two instead of four, and the folded twiddle
// butterfly three instead of six.  ptxas folds the operand swaps / partial negations / scalar
// broadcasts written below into the instruction's operand modifiers (.F32x2.LO_HI.NP, .F32), so the
// pk() shuffles cost nothing.  Each half is an IEEE fp32 add / mul / fma, exactly as the scalar
// forms.
typedef unsigned long long f32x2_t;
__device__ __forceinline__ f32x2_t pk(float x, float y) {
  f32x2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ f32x2_t pk(float2 a) { return pk(a.x, a.y); }
__device__ __forceinline__ float2 upk(f32x2_t r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ f32x2_t add2(f32x2_t a, f32x2_t b) {
  f32x2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2_t sub2(f32x2_t a, f32x2_t b) {
  f32x2_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2_t mul2(f32x2_t a, f32x2_t b) {
  f32x2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2_t fma2(f32x2_t a, f32x2_t b, f32x2_t c) {   // a * b + c per half
  f32x2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return upk(add2(pk(a), pk(b))); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return upk(sub2(pk(a), pk(b))); }
// a * b = b a.x + (-b.y, b.x) a.y
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return upk(fma2(pk(b.y, b.x), pk(-a.y, a.y), mul2(pk(b), pk(a.x, a.x))));
}
// a * conj(b) = a b.x + (a.y, -a.x) b.y
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return upk(fma2(pk(a.y, a.x), pk(b.y, -b.y), mul2(pk(a), pk(b.x, b.x))));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return upk(mul2(pk(a), pk(s, s))); }
// acc + w * v (real weight w)
__device__ __forceinline__ float2 caxpy(float w, float2 v, float2 acc) { return upk(fma2(pk(w, w), pk(v), pk(acc))); }
// multiply by SIGN * i
template <int SIGN>
__device__ __forceinline__ float2 mul_i(float2 a) {
  return SIGN > 0 ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}
// a + SIGN i b in one instruction (b swapped, one half negated, times 1)
template <int SIGN>
__device__ __forceinline__ float2 cadd_i(float2 a, float2 b) {
  return SIGN > 0 ? upk(fma2(pk(b.y, b.x), pk(-1.f, 1.f), pk(a))) : upk(fma2(pk(b.y, b.x), pk(1.f, -1.f), pk(a)));
}

// a * W_R^K with the trivial angles special-cased.
template <int R, int K, int SIGN>
__device__ __forceinline__ float2 twmul(float2 a) {
  constexpr int k = ((K % R) + R) % R;
  if constexpr (k == 0) {
    return a;
  } else if constexpr (4 * k == R) {
    return mul_i<SIGN>(a);
  } else if constexpr (2 * k == R) {
    return make_float2(-a.x, -a.y);
  } else if constexpr (4 * k == 3 * R) {
    return mul_i<-SIGN>(a);
  } else {
    constexpr float c = float(Tw<R, K, SIGN>::c), s = float(Tw<R, K, SIGN>::s);
    return upk(fma2(pk(a.y, a.x), pk(-s, s), mul2(pk(a), pk(c, c))));   // a c + (-a.y, a.x) s
  }
}

// a + W_R^K b and a - W_R^K b with the twiddle multiplication folded into fused multiply-adds:
// for W = c + i s, factor the larger of |c|, |s| out (tangent form, |t| <= 1): W b = c (b + i t b)
// or s (u b + i b), so the pair costs 3 packed instructions (1 FFMA2 for the scaled b, 2 for the
// sum and the difference) instead of 8 scalar ones (a complex multiply and two complex additions).
// The trivial angles stay additions / swaps.
template <int R, int K, int SIGN>
__device__ __forceinline__ void bfly_w(float2 a, float2 b, float2& sum, float2& diff) {
  constexpr int k = ((K % R) + R) % R;
  if constexpr (k == 0 || 2 * k == R) {
    const float2 t = twmul<R, K, SIGN>(b);
    sum = cadd(a, t);
    diff = csub(a, t);
  } else if constexpr (4 * k == R || 4 * k == 3 * R) {   // W = +-i: a + W b, a - W b
    constexpr int S = (4 * k == R) ? SIGN : -SIGN;
    sum = cadd_i<S>(a, b);
    diff = cadd_i<-S>(a, b);
  } else {
    constexpr double c = Tw<R, K, SIGN>::c, s = Tw<R, K, SIGN>::s;
    if constexpr ((c < 0 ? -c : c) >= (s < 0 ? -s : s)) {
      constexpr float t = float(s / c), cf = float(c);
      const f32x2_t bb = fma2(pk(b.y, b.x), pk(-t, t), pk(b));   // b (1 + i t)
      sum = upk(fma2(pk(cf, cf), bb, pk(a)));
      diff = upk(fma2(pk(-cf, -cf), bb, pk(a)));
    } else {
      constexpr float u = float(c / s), sf = float(s);
      const f32x2_t bb = fma2(pk(b), pk(u, u), pk(-b.y, b.x));   // b (u + i)
      sum = upk(fma2(pk(sf, sf), bb, pk(a)));
      diff = upk(fma2(pk(-sf, -sf), bb, pk(a)));
    }
  }
}
// a + W_R^K b alone (2 packed instructions for a generic angle)
template <int R, int K, int SIGN>
__device__ __forceinline__ float2 madd_w(float2 a, float2 b) {
  constexpr int k = ((K % R) + R) % R;
  if constexpr (k == 0 || 2 * k == R) {
    return cadd(a, twmul<R, K, SIGN>(b));
  } else if constexpr (4 * k == R || 4 * k == 3 * R) {
    return cadd_i<(4 * k == R) ? SIGN : -SIGN>(a, b);
  } else {
    constexpr double c = Tw<R, K, SIGN>::c, s = Tw<R, K, SIGN>::s;
    if constexpr ((c < 0 ? -c : c) >= (s < 0 ? -s : s)) {
      constexpr float t = float(s / c), cf = float(c);
      const f32x2_t bb = fma2(pk(b.y, b.x), pk(-t, t), pk(b));
      return upk(fma2(pk(cf, cf), bb, pk(a)));
    } else {
      constexpr float u = float(c / s), sf = float(s);
      const f32x2_t bb = fma2(pk(b), pk(u, u), pk(-b.y, b.x));
      return upk(fma2(pk(sf, sf), bb, pk(a)));
    }
  }
}

template <int R, int SIGN>
__device__ __forceinline__ void dft(float2 (&v)[R]);

namespace detail {
// radix-4 DIT combine: X[k + m R/4] = sum_q W_R^{qk} W_4^{qm} D_q[k], with W_R^{3K} = W_R^K W_R^{2K}
// and SIGN i = W_R^{R/4} folded into FMA butterflies (bfly_w):
//   s02, d02 = D0 +- W^{2K} D2;  f, g = D1 +- W^{2K} D3;
//   X[K], X[K + R/2] = s02 +- W^K f;  X[K + R/4], X[K + 3R/4] = d02 +- W^{K + R/4} g
template <int R, int SIGN, int K>
__device__ __forceinline__ void r4_combine(float2 (&v)[R], const float2 (&d0)[R / 4], const float2 (&d1)[R / 4],
                                           const float2 (&d2)[R / 4], const float2 (&d3)[R / 4]) {
  if constexpr (K < R / 4) {
    float2 s02, d02, f, g;
    bfly_w<R, 2 * K, SIGN>(d0[K], d2[K], s02, d02);
    bfly_w<R, 2 * K, SIGN>(d1[K], d3[K], f, g);
    bfly_w<R, K, SIGN>(s02, f, v[K], v[K + R / 2]);
    bfly_w<R, K + R / 4, SIGN>(d02, g, v[K + R / 4], v[K + 3 * R / 4]);
    r4_combine<R, SIGN, K + 1>(v, d0, d1, d2, d3);
  }
}
template <int R, int SIGN, int K>
__device__ __forceinline__ void r2_combine(float2 (&v)[R], const float2 (&e)[R / 2], const float2 (&o)[R / 2]) {
  if constexpr (K < R / 2) {
    bfly_w<R, K, SIGN>(e[K], o[K], v[K], v[K + R / 2]);
    r2_combine<R, SIGN, K + 1>(v, e, o);
  }
}
}  // namespace detail

// In-place R-point DFT, natural order in and out: v[k] <- sum_n v[n] exp(SIGN i 2 pi n k / R).
template <int R, int SIGN>
__device__ __forceinline__ void dft(float2 (&v)[R]) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    const float2 s13 = cadd(v[1], v[3]), d13 = csub(v[1], v[3]);
    v[0] = cadd(s02, s13);
    v[2] = csub(s02, s13);
    v[1] = cadd_i<SIGN>(d02, d13);    // d02 + SIGN i d13
    v[3] = cadd_i<-SIGN>(d02, d13);
  } else if constexpr (R == 8) {
    float2 e[4], o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { e[i] = v[2 * i]; o[i] = v[2 * i + 1]; }
    dft<4, SIGN>(e);
    dft<4, SIGN>(o);
    detail::r2_combine<8, SIGN, 0>(v, e, o);
  } else {
    static_assert(R % 4 == 0, "R must be a power of two");
    float2 d0[R / 4], d1[R / 4], d2[R / 4], d3[R / 4];
#pragma unroll
    for (int i = 0; i < R / 4; ++i) {
      d0[i] = v[4 * i];
      d1[i] = v[4 * i + 1];
      d2[i] = v[4 * i + 2];
      d3[i] = v[4 * i + 3];
    }
    dft<R / 4, SIGN>(d0);
    dft<R / 4, SIGN>(d1);
    dft<R / 4, SIGN>(d2);
    dft<R / 4, SIGN>(d3);
    detail::r4_combine<R, SIGN, 0>(v, d0, d1, d2, d3);
  }
}

namespace detail {
template <int P, int SIGN, int N1>
__device__ __forceinline__ void halfzero_split(const float2 (&v)[P], float2 (&a)[P / 2], float2 (&b)[P / 2]) {
  if constexpr (N1 < P / 2) {
    constexpr int src = N1 < P / 4 ? N1 : N1 + P / 2;      // the one non-zero input of the pair
    constexpr int tw = N1 < P / 4 ? N1 : N1 + P / 2;       // (x[n] - x[n+P/2]) W^n = z W^{n or n+P/2}
    a[N1] = v[src];
    b[N1] = twmul<P, tw, SIGN>(v[src]);
    halfzero_split<P, SIGN, N1 + 1>(v, a, b);
  }
}
}  // namespace detail

// In-place P-point DFT of an input that is zero at n in [P/4, 3P/4) (the zero-padded half of the
// oversampled grid).  One decimation-in-frequency step leaves every butterfly
// with a single non-zero input, so it costs only the odd-branch twiddles, then two P/2-point DFTs
// give the even and odd outputs.  The values in v[P/4 .. 3P/4) are ignored.
template <int P, int SIGN>
__device__ __forceinline__ void dft_halfzero(float2 (&v)[P]) {
  float2 a[P / 2], b[P / 2];
  detail::halfzero_split<P, SIGN, 0>(v, a, b);
  dft<P / 2, SIGN>(a);
  dft<P / 2, SIGN>(b);
#pragma unroll
  for (int k = 0; k < P / 2; ++k) {
    v[2 * k] = a[k];
    v[2 * k + 1] = b[k];
  }
}

namespace detail {
// radix-4 DIT combine producing only X[K] and X[K + 3R/4] (folded as r4_combine)
template <int R, int SIGN, int K>
__device__ __forceinline__ void r4_combine_halfout(float2 (&v)[R], const float2 (&d0)[R / 4], const float2 (&d1)[R / 4],
                                                   const float2 (&d2)[R / 4], const float2 (&d3)[R / 4]) {
  if constexpr (K < R / 4) {
    float2 s02, d02, f, g;
    bfly_w<R, 2 * K, SIGN>(d0[K], d2[K], s02, d02);
    bfly_w<R, 2 * K, SIGN>(d1[K], d3[K], f, g);
    v[K] = madd_w<R, K, SIGN>(s02, f);
    v[K + 3 * R / 4] = madd_w<R, K + 3 * R / 4, SIGN>(d02, g);   // d02 - W^{K + R/4} g
    r4_combine_halfout<R, SIGN, K + 1>(v, d0, d1, d2, d3);
  }
}
}  // namespace detail

namespace detail {
// r4_combine_halfout split over a lane pair (l, l ^ 16): lane half h = 0 holds D0, D2 (da, db),
// h = 1 holds D1, D3.  Each forms its first butterfly (s02, d02 or f, g), the pair swaps d02 and
// f by shuffle, and h = 0 produces X[K] = s02 + W^K f, h = 1 X[K + 3R/4] = d02 + W^{K + 3R/4} g
// -- operation for operation what r4_combine_halfout computes in one thread.
template <int R, int SIGN, int K>
__device__ __forceinline__ void t2_combine(float2 (&out)[R / 4], const float2 (&da)[R / 4], const float2 (&db)[R / 4],
                                           int h) {
  if constexpr (K < R / 4) {
    float2 s, d;
    bfly_w<R, 2 * K, SIGN>(da[K], db[K], s, d);   // h = 0: s02, d02;  h = 1: f, g
    const float2 send = h ? s : d;                // h = 0 gives d02 away, h = 1 gives f away
    float2 recv;
    recv.x = __shfl_xor_sync(0xffffffffu, send.x, 16);
    recv.y = __shfl_xor_sync(0xffffffffu, send.y, 16);
    const float2 lo = madd_w<R, K, SIGN>(s, recv);               // (h = 0) s02 + W^K f
    const float2 hi = madd_w<R, K + 3 * R / 4, SIGN>(recv, d);   // (h = 1) d02 + W^{K + 3R/4} g
    out[K] = h ? hi : lo;
    t2_combine<R, SIGN, K + 1>(out, da, db, h);
  }
}
}  // namespace detail

// R-point DFT (natural order) that produces only the outputs k < R/4 and k >= 3R/4 -- the kept
// (cropped) half of the oversampled grid in the adjoint.  The other
// entries of v are left unspecified.  The last butterfly stage skips the two dropped outputs.
template <int R, int SIGN>
__device__ __forceinline__ void dft_halfout(float2 (&v)[R]) {
  if constexpr (R == 8) {
    float2 e[4], o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { e[i] = v[2 * i]; o[i] = v[2 * i + 1]; }
    dft<4, SIGN>(e);
    dft<4, SIGN>(o);
    v[0] = cadd(e[0], o[0]);
    v[1] = madd_w<8, 1, SIGN>(e[1], o[1]);
    v[6] = madd_w<8, 6, SIGN>(e[2], o[2]);   // e - W^2 o = e + W^6 o
    v[7] = madd_w<8, 7, SIGN>(e[3], o[3]);   // e - W^3 o = e + W^7 o
  } else if constexpr (R >= 16) {
    static_assert(R % 4 == 0, "R must be a power of two");
    float2 d0[R / 4], d1[R / 4], d2[R / 4], d3[R / 4];
#pragma unroll
    for (int i = 0; i < R / 4; ++i) {
      d0[i] = v[4 * i];
      d1[i] = v[4 * i + 1];
      d2[i] = v[4 * i + 2];
      d3[i] = v[4 * i + 3];
    }
    dft<R / 4, SIGN>(d0);
    dft<R / 4, SIGN>(d1);
    dft<R / 4, SIGN>(d2);
    dft<R / 4, SIGN>(d3);
    detail::r4_combine_halfout<R, SIGN, 0>(v, d0, d1, d2, d3);
  } else {
    dft<R, SIGN>(v);
  }
}

// Two-stage split of the supported grid sizes.  T threads (within one warp) per length-G DFT.
template <int G> struct FFTShape;
template <> struct FFTShape<32>   { static constexpr int P = 4,  Q = 8,  T = 4;  };   // N = 32 image transforms (precond.cuh)
template <> struct FFTShape<64>   { static constexpr int P = 8,  Q = 8,  T = 8;  };
template <> struct FFTShape<128>  { static constexpr int P = 8,  Q = 16, T = 8;  };
template <> struct FFTShape<256>  { static constexpr int P = 16, Q = 16, T = 16; };
template <> struct FFTShape<512>  { static constexpr int P = 16, Q = 32, T = 16; };
template <> struct FFTShape<1024> { static constexpr int P = 32, Q = 32, T = 32; };

}  // namespace mrf

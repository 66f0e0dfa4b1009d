// f46_device.cuh -- device building blocks of the 4/6 NVFP4 quantizer (sm_100a).
//
// Two paths compute one 16-element block:
//
//  * fast path (f32, packed f32x2 math, hardware cvt to e2m1/e4m3):
//      scale  sc_m  = cvt.e4m3(bmax * r_m) with r_m ~ 1/(alpha*m), bracketed by
//                     two perturbed quotients; a disagreement is a near-tie and
//                     is resolved exactly by sign(fma(alpha, T*m, -bmax)) where T
//                     is the E4M3 tie (T*m is exact in f32, the fma rounds once).
//      codes  c_i   = cvt.e2m1(x_i * rD) bracketed the same way; a near-tie is
//                     resolved by sign(fma(alpha, t*Delta, -|x_i|)), t the FP4 tie.
//      error  S_m   = sum (v_i*Delta*alpha - x_i)^2 in f32 (each term from one
//                     correctly rounded fma, f32x2 fma accumulation, relative
//                     error < 11 * 2^-24); if |S4 - S6| is inside a 2^-18
//                     band the two sums are recomputed exactly in f64 in the
//                     reference's numpy pairwise order.
//    This reproduces the reference's exact-real rounding decisions
//     for every block whose values lie in the guarded
//    range; everything else takes:
//
//  * exact path (f64, one block, noinline): a line-by-line restatement of the
//    reference's float64 arithmetic -- blockquant.py:239-242 (_nvfp4_scales),
//    :260-280 (_cast_values), :283-293 (_block_error_sums, numpy pairwise
//    order), adaptive.py:77-80 (strict '<', ties keep 6) -- using __dmul_rn /
//    __dadd_rn / __ddiv_rn so no FMA contraction can change a rounding.
//    Used for underflowed scales, extreme magnitudes, float64 inputs, alpha
//    overrides that are not float32 values, and the l1/absmax rules.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#ifndef F46_ACC2
#define F46_ACC2 0
#endif
#ifndef F46_PRMT_LO
#define F46_PRMT_LO 0
#endif
#ifndef F46_TAB
#define F46_TAB 1
#endif
#ifndef F46_NEWTON
#define F46_NEWTON 0
#endif

namespace f46 {

enum { DT_F32 = 0, DT_BF16 = 1, DT_F64 = 2 };
enum { FIXED6 = 0, FIXED4 = 1, ADAPTIVE = 2 };
enum { RULE_MSE = 0, RULE_L1 = 1, RULE_ABSMAX = 2 };

// ----------------------------------------------------------------------------
// PTX conversions (sm_100a)
// ----------------------------------------------------------------------------

// Two f32 -> two E4M3 codes (RNE, satfinite). Low byte = lo, high byte = hi.
__device__ __forceinline__ uint32_t cvt_e4m3x2(float hi, float lo) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

// Four pairs of f32 -> 8 E2M1 codes in one u32; element 2k in the low nibble
// of byte k (the reference's nibble order, tensor_io.py:118-123).
__device__ __forceinline__ uint32_t cvt_e2m1x8(float2 a, float2 b, float2 c, float2 d) {
  uint32_t r;
  asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t}"
      : "=r"(r)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y), "f"(d.x), "f"(d.y));
  return r;
}

// Byte k of w (two E2M1 codes) -> f16x2 (exact); the low nibble (even
// element) lands in the low half.  The byte is handed over in a 16-bit
// register split with mov.b16 (as cuda_fp4.hpp does): a 4-way .b8 vector
// split of a 32-bit register mis-selected bytes under ptxas 12.9.
template <int K>
__device__ __forceinline__ __half2 e2m1x2_to_h2(uint32_t w) {
  uint32_t r;
  const uint16_t b = (uint16_t)((w >> (8 * K)) & 0xFFu);
  asm("{\n\t.reg .b8 lo, hi;\n\tmov.b16 {lo, hi}, %1;\n\t"
      "cvt.rn.f16x2.e2m1x2 %0, lo;\n\t}"
      : "=r"(r)
      : "h"(b));
  return *reinterpret_cast<__half2*>(&r);
}

// E4M3 code -> f32 (exact; codes < 0x7F).
__device__ __forceinline__ float e4m3_to_f32(uint32_t code) {
  uint32_t r;
  uint16_t c = (uint16_t)code;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"(c));
  return __half2float(__ushort_as_half((uint16_t)(r & 0xFFFF)));
}

// FP4 magnitude of a 3-bit code m (0,.5,1,1.5,2,3,4,6), f32 exact.
__device__ __forceinline__ float fp4_mag_f32(uint32_t m) {
  // twice the magnitudes {0, 1, 2, 3, 4, 6, 8, 12} as a byte table
  return (float)(__byte_perm(0x03020100u, 0x0C080604u, m & 7u) & 0xFFu) * 0.5f;
}

// ----------------------------------------------------------------------------
// Exact float64 restatement of the reference (slow path)
// ----------------------------------------------------------------------------

// codecs.py:99-117 encode_fp4_rne, for finite x.
__device__ __forceinline__ uint32_t enc_fp4_d(double x) {
  const uint32_t sign = signbit(x) ? 8u : 0u;
  double m = fmin(fabs(x), 6.0);
  int e;
  frexp(m, &e);
  int ex = e - 1;
  if (ex < 0) ex = 0;
  const double q = ldexp(1.0, ex - 1);
  const double mag = __dmul_rn(rint(m / q), q);  // m/q exact (power of two)
  uint32_t idx;
  if (mag < 2.0)
    idx = (uint32_t)(mag * 2.0);  // 0, .5, 1, 1.5 -> 0..3
  else if (mag == 2.0)
    idx = 4;
  else if (mag == 3.0)
    idx = 5;
  else if (mag == 4.0)
    idx = 6;
  else
    idx = 7;
  return idx | sign;
}

// codecs.py:92-96
__device__ __forceinline__ double dec_fp4_d(uint32_t c) {
  const double v = (double)fp4_mag_f32(c & 7);
  return (c & 8) ? -v : v;
}

// codecs.py:56-68 / :151-155
__device__ __forceinline__ double dec_e4m3_d(uint32_t code) {
  const int ex = (code >> 3) & 0xF, mant = code & 7;
  double v;
  if (ex == 0xF && mant == 7)
    v = __longlong_as_double(0x7FF8000000000000ll);
  else if (ex == 0)
    v = mant * 0x1p-9;
  else
    v = (1.0 + mant / 8.0) * ldexp(1.0, ex - 7);
  return (code & 0x80) ? -v : v;
}

// codecs.py:158-178 encode_fp8_e4m3, non-negative input.
__device__ __forceinline__ uint32_t enc_e4m3_d(double x) {
  if (isnan(x)) return 0x7F;
  const uint32_t sign = signbit(x) ? 0x80u : 0u;
  double m = fabs(x);
  if (isinf(m)) m = 448.0;
  m = fmin(m, 448.0);
  int e;
  frexp(m, &e);
  int ex = e - 1;
  if (ex < -6) ex = -6;
  const double q = ldexp(1.0, ex - 3);
  const double mag = __dmul_rn(rint(m / q), q);
  uint32_t code;
  if (mag == 0.0) {
    code = 0;
  } else if (mag < 0x1p-6) {
    code = (uint32_t)(mag * 512.0);  // subnormal: mant * 2^-9
  } else {
    int e2;
    const double f = frexp(mag, &e2);  // mag = f * 2^e2, f in [0.5, 1)
    const uint32_t mant = (uint32_t)((f * 16.0) - 8.0);
    code = ((uint32_t)(e2 - 1 + 7) << 3) | mant;
  }
  return code | sign;
}

// numpy pairwise sum of 16 values (numpy 2.x pairwise_sum, n <= 128 branch)
__device__ __forceinline__ double pw16(const double (&e)[16]) {
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(e[j], e[j + 8]);
  return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

struct ExactPass {
  uint64_t codes;
  uint32_t sc;
  double sq, ab, mx;
};

// One fixed-target pass over one block (blockquant.py:302-313).
__device__ __forceinline__ void exact_pass(const double (&x)[16], double alpha, double m,
                                           ExactPass& o) {
  double bmax = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) bmax = fmax(bmax, fabs(x[i]));
  uint32_t sc = enc_e4m3_d(__ddiv_rn(bmax, __dmul_rn(alpha, m)));
  if (bmax == 0.0) sc = 1;
  const double sdec = dec_e4m3_d(sc);
  const double denom = __dmul_rn(alpha, sdec);
  double esq[16], eab[16];
  double mx = 0.0;
  uint64_t codes = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double s;
    if (denom > 0.0)
      s = __ddiv_rn(x[i], denom);
    else
      s = (x[i] != 0.0) ? copysign(6.0, x[i]) : 0.0;
    const uint32_t c = enc_fp4_d(s);
    codes |= (uint64_t)c << (4 * i);
    const double deq = __dmul_rn(dec_fp4_d(c), denom);
    const double diff = __dsub_rn(deq, x[i]);
    esq[i] = __dmul_rn(diff, diff);
    eab[i] = fabs(diff);
    mx = fmax(mx, eab[i]);
  }
  o.codes = codes;
  o.sc = sc;
  o.sq = pw16(esq);
  o.ab = pw16(eab);
  o.mx = mx;
}

__device__ __forceinline__ double rule_err(const ExactPass& p, int rule) {
  return rule == RULE_MSE ? p.sq : (rule == RULE_L1 ? p.ab : p.mx);
}

struct BlockOut {
  uint64_t codes;  // 16 nibbles, element i at bits [4i, 4i+4)
  uint32_t sc;     // E4M3 code
  uint32_t pick4;  // 1 if the M=4 target was stored
};

// Full exact block (adaptive.py:60-101 / blockquant.py:334-360 for one block).
// Pad positions must be passed as 0.0 and are zeroed in the returned codes by
// the caller's tail handling.
__device__ __forceinline__ void exact_block_inl(const double* xin, double alpha, int mode, int rule,
                                                BlockOut* out) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = xin[i];
  ExactPass p6, p4;
  if (mode == ADAPTIVE) {
    exact_pass(x, alpha, 6.0, p6);
    exact_pass(x, alpha, 4.0, p4);
    const bool k = rule_err(p4, rule) < rule_err(p6, rule);
    out->codes = k ? p4.codes : p6.codes;
    out->sc = k ? p4.sc : p6.sc;
    out->pick4 = k;
  } else {
    exact_pass(x, alpha, mode == FIXED4 ? 4.0 : 6.0, p6);
    out->codes = p6.codes;
    out->sc = p6.sc;
    out->pick4 = (mode == FIXED4);
  }
}

static __device__ __noinline__ void exact_block(const double* xin, double alpha, int mode, int rule,
                                         BlockOut* out) {
  exact_block_inl(xin, alpha, mode, rule, out);
}

// Exact float64 squared-error sum of one candidate whose codes are known
// (blockquant.py:279, :289-290), used when the f32 comparison is ambiguous.
static __device__ __noinline__ double exact_sq_sum(const double* x, uint64_t codes, double alpha,
                                            double delta) {
  const double denom = __dmul_rn(alpha, delta);
  double e[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double deq = __dmul_rn(dec_fp4_d((uint32_t)(codes >> (4 * i)) & 15u), denom);
    const double diff = __dsub_rn(deq, x[i]);
    e[i] = __dmul_rn(diff, diff);
  }
  return pw16(e);
}

// ----------------------------------------------------------------------------
// Fast path
// ----------------------------------------------------------------------------

// Per-tensor constants, identical in every thread.
struct TensorConsts {
  double alpha_d;
  float alpha;
  float r6_lo, r6_hi, r4_lo, r4_hi;  // bracketing 1/(alpha*m)
  int force_exact;                   // alpha outside the fast path's range
  // Rounding direction of bracket-flagged FP4 codes (see tie_direction()):
  // -1 keep the lower code, +1 take the upper code, 0 ties-to-even,
  // 2 unknown -> exact per-element test.
  int tdir;
  uint32_t zero;  // 0, but not a compile-time constant (unpack_e2m1x8)
};

// For BF16 input whose alpha was computed from amax A (no override), every
// element whose quotient x/(alpha*Delta) lies within 2^-19.5 of an FP4 tie t
// is an exact tie of the *unrounded* scale beta = A/mcap:
//   q_beta = |x|*mcap/(A*Delta) = (4*X*M*2^k)/(T*Y*S)  with X, Y (8-bit bf16
//   significands), M the odd part of mcap (<= 21), S (E4M3 significand, <= 15),
//   T = 4t <= 20, so q_beta != t implies |q_beta - t| >= t * 2^-16.3, while
//   |q/q_beta - 1| = |beta/alpha - 1| <= 2^-24.
// Hence q = t*beta/alpha and the reference's exact-real rounding goes down if
// alpha > beta, up if alpha < beta and to even if alpha == beta -- one sign for
// the whole tensor, decided exactly here (alpha*mcap has <= 29 bits).
// Scale codes, same setting (BF16 x, alpha computed from the amax A): the
// E4M3 code of a block is RN(bmax/(alpha*m)).  With beta = A/mcap, q_beta =
// bmax*mcap/(A*m) = (Xb * c * 2^k) / (Xa * m') with Xb, Xa the 8-bit bf16
// significands, c the odd part of mcap and m' the odd part of m (1 or 3).  An
// E4M3 tie t has an odd significand T <= 31 (subnormal ties included), so
// q_beta != t implies |q_beta - t| >= t / (T * Xa * m') >= t * 2^-14.6, while
// the bracketing products bmax*r_lo, bmax*r_hi lie within 2^-17 of q_alpha and
// |q_alpha/q_beta - 1| <= 2^-24.  A bracket straddling a tie therefore means
// an exact tie of q_beta, and q_alpha = t*beta/alpha rounds the way
// tie_direction says: down for -1 (the lower bracket's code is exact), up for
// +1 (the upper one's).  For 0 the exact ties need ties-to-even
// (e4m3_ties_possible / scale_tie).  The K2 prologue collapses the brackets.
#ifndef F46_SCALE_TDIR
#define F46_SCALE_TDIR 1
#endif
__device__ __forceinline__ int tie_direction(double alpha, double amax, double mcap, int dtype,
                                             bool overridden) {
  if (dtype != DT_BF16 || overridden || !(amax > 0.0)) return 2;
  const double d = alpha * mcap - amax;  // exact
  return d > 0.0 ? -1 : (d < 0.0 ? 1 : 0);
}

// Relative half-width of the scale brackets.  Every f32 quantity below carries
// at most 2^-21.9 relative error (one approximate reciprocal, <= 1 ulp, plus
// three RN roundings), so x*r_lo < x/(alpha*m) < x*r_hi strictly.
#define F46_BRACKET 0x1p-17f
// Codes are computed from q = x * rD * (1 - 11*2^-24), a strict lower bound of
// the true quotient x/(alpha*Delta) (and within 2^-19.9 of it); the winner's
// codes are checked against q * (1 + 11*2^-23), a strict upper bound.
#define F46_QLO (1.0f - 11.0f * 0x1p-24f) /* 1 - 2^-20.54, exact in f32 */
#define F46_QHI_OVER_QLO (1.0f + 11.0f * 0x1p-23f) /* exact in f32 */

__device__ __forceinline__ TensorConsts make_consts(double alpha_d, int rule, int dtype,
                                                   int tdir = 2) {
  TensorConsts t;
  t.tdir = tdir;
  t.alpha_d = alpha_d;
  t.alpha = (float)alpha_d;
  t.zero = __float_as_uint(t.alpha) >> 31;  // alpha > 0
  const bool f32_exact = ((double)t.alpha == alpha_d);
  t.force_exact = !(f32_exact && alpha_d >= 0x1p-50 && alpha_d <= 0x1p50) ||
                  rule != RULE_MSE || dtype == DT_F64;
  const float r6 = (float)(1.0 / (alpha_d * 6.0));
  const float r4 = (float)(1.0 / (alpha_d * 4.0));
  t.r6_lo = r6 * (1.0f - F46_BRACKET);
  t.r6_hi = r6 * (1.0f + F46_BRACKET);
  t.r4_lo = r4 * (1.0f - F46_BRACKET);
  t.r4_hi = r4 * (1.0f + F46_BRACKET);
  return t;
}

// The K2 streaming kernel's constants for a tensor with tie direction -1 or
// +1: both scale brackets collapse onto the one whose code is exact (see
// "Scale codes" above), so no block is deferred for its scale code.
__device__ __forceinline__ TensorConsts scale_dir_consts(TensorConsts t) {
  if (F46_SCALE_TDIR) {
    const bool up = t.tdir == 1, down = t.tdir == -1;
    const float r6l = t.r6_lo, r4l = t.r4_lo;
    t.r6_lo = up ? t.r6_hi : t.r6_lo;
    t.r4_lo = up ? t.r4_hi : t.r4_lo;
    t.r6_hi = down ? r6l : t.r6_hi;
    t.r4_hi = down ? r4l : t.r4_hi;
  }
  return t;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Block-scale code for target m.  The two bracketing quotients give the same
// E4M3 code unless bmax/(alpha*m) lies within 2^-17 of the E4M3 tie T between
// them; then sign(alpha*T*m - bmax) decides exactly (T*m has <= 7
// significant bits, the fma rounds once) and an exact tie goes to the even code.
__device__ __forceinline__ uint32_t block_scale_code(float bmax, float alpha, float m, float r_lo,
                                                     float r_hi) {
  const uint32_t pr = cvt_e4m3x2(bmax * r_hi, bmax * r_lo);
  uint32_t sc = pr & 0xFF;
  const uint32_t sh = pr >> 8;
  if (__builtin_expect(sh != sc, 0)) {
    const float T = 0.5f * (e4m3_to_f32(sc) + e4m3_to_f32(sh));
    const float s = fmaf(alpha, T * m, -bmax);
    sc = s > 0.f ? sc : (s < 0.f ? sh : ((sc & 1) ? sh : sc));
  }
  return sc;
}

// 4 * (FP4 tie above magnitude code m), m = 0..6: 0.25 .75 1.25 1.75 2.5 3.5 5
__device__ __forceinline__ float fp4_tie_above(uint32_t m) {
  return (float)(__byte_perm(0x07050301u, 0x00140E0Au, m) & 0xFFu) * 0.25f;
}

// Resolve the flagged nibbles of one 8-code word exactly: code(q_lo) = m and
// the true quotient may lie at or above the tie t above m, so the true code is
// m or m+1: sign(alpha*t*delta - |x|) decides (t*delta exact in f32), an exact
// tie goes to the even code.  base = index of the word's first element.
template <class Load>
__device__ __forceinline__ uint32_t fix_word(uint32_t w, uint32_t dmask, int base, float alpha,
                                             float delta, const Load& load) {
  while (dmask) {
    const int sh = (__ffs(dmask) - 1) & ~3;
    const uint32_t m = (w >> sh) & 7u;
    const float s = fmaf(alpha, fp4_tie_above(m) * delta, -fabsf(load(base + (sh >> 2))));
    const uint32_t inc = (s < 0.f) | ((s == 0.f) & (m & 1u));
    w += inc << sh;
    dmask &= ~(0xFu << sh);
  }
  return w;
}

// Round a quotient pair to E2M1 (cvt.rn.satfinite) and decode it straight back
// to f16x2 without packing the codes (the candidates' codes are only needed
// for their error; the stored candidate's codes are recomputed and packed
// once).  The .b8 never leaves the asm block, so no byte extraction is emitted.
__device__ __forceinline__ uint32_t e2m1x2_roundtrip(float hi, float lo) {
  uint32_t d;
  asm("{\n\t.reg .b8 c;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 c, %1, %2;\n\t"
      "cvt.rn.f16x2.e2m1x2 %0, c;\n\t}"
      : "=r"(d)
      : "f"(hi), "f"(lo));
  return d;
}

// r = v - q with v one half of an f16x2 word: one mixed-precision FHADD
// (f16 + f32 -> f32, single rounding) on the FMA pipe.
template <int H>
__device__ __forceinline__ float fhadd_h(uint32_t v, float negq) {
  float r;
  if (H == 0)
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.f16 %0, l, %2;\n\t}"
        : "=f"(r)
        : "r"(v), "f"(negq));
  else
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.f16 %0, h, %2;\n\t}"
        : "=f"(r)
        : "r"(v), "f"(negq));
  return r;
}

// Exact bf16 -> f32 of the high half of w on the FMA pipe (FHADD.BF16 w.H1 + -0,
// which keeps the sign of -0.0); the low half is a shift (IMAD.SHL).
__device__ __forceinline__ float2 bf16x2_unpack(uint32_t w) {
  float hi;
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.bf16 %0, h, %2;\n\t}"
      : "=f"(hi)
      : "r"(w), "f"(-0.0f));
#if F46_PRMT_LO
  return make_float2(__uint_as_float(__byte_perm(w, 0u, 0x1044u)), hi);
#else
  return make_float2(__uint_as_float(w << 16), hi);
#endif
}

// Quotient-space squared error of one candidate,  sum_i (v_i - q_i)^2  with
// q_i = x_i * rq (the lower-bound reciprocal) and v_i = E2M1(q_i).  One f32x2
// accumulator; any order of the 16 f32 additions stays inside the 2^-20
// relative bound the decision tolerance allows for.
__device__ __forceinline__ float cand_err(const float2 (&x)[8], float rq) {
  const float2 r2 = make_float2(rq, rq);
#if F46_ACC2
  float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const float2 q = __fmul2_rn(x[p], r2);
    const uint32_t v = e2m1x2_roundtrip(q.y, q.x);
    const float2 r = make_float2(fhadd_h<0>(v, -q.x), fhadd_h<1>(v, -q.y));
    acc[p & 1] = __ffma2_rn(r, r, acc[p & 1]);
  }
  return (acc[0].x + acc[1].x) + (acc[0].y + acc[1].y);
#else
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const float2 q = __fmul2_rn(x[p], r2);
    const uint32_t v = e2m1x2_roundtrip(q.y, q.x);
    const float2 r = make_float2(fhadd_h<0>(v, -q.x), fhadd_h<1>(v, -q.y));
    acc = __ffma2_rn(r, r, acc);
  }
  return acc.x + acc.y;
#endif
}

// Packed codes of x * r (16 nibbles, element i at bits [4i, 4i+4)).
__device__ __forceinline__ uint64_t codes_of(const float2 (&x)[8], float r) {
  const float2 r2 = make_float2(r, r);
  float2 q[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) q[p] = __fmul2_rn(x[p], r2);
  const uint32_t w0 = cvt_e2m1x8(q[0], q[1], q[2], q[3]);
  const uint32_t w1 = cvt_e2m1x8(q[4], q[5], q[6], q[7]);
  return ((uint64_t)w1 << 32) | w0;
}

// Exact codes of the stored candidate from its lower-bound reciprocal rq.
// q = x*rq is a strict lower bound of the true quotient x/(alpha*Delta) and
// q*QHI/QLO a strict upper bound; their codes agree except at nibbles whose
// bracket straddles an FP4 tie, where the true code is one of the two.  With a
// known tensor-wide tie direction one of the two bounds is already exact;
// otherwise both are formed and each flagged nibble is settled exactly.
template <class Load>
__device__ __forceinline__ uint64_t exact_codes(const float2 (&x)[8], float rq, float alpha,
                                                float delta, int tdir, const Load& load) {
  const float rh = rq * F46_QHI_OVER_QLO;
  if (tdir < 0) return codes_of(x, rq);
  if (tdir == 1) return codes_of(x, rh);
  const uint64_t lo = codes_of(x, rq), hi = codes_of(x, rh);
  uint32_t w0 = (uint32_t)lo, w1 = (uint32_t)(lo >> 32);
  const uint32_t h0 = (uint32_t)hi, h1 = (uint32_t)(hi >> 32);
  const uint32_t d0 = w0 ^ h0, d1 = w1 ^ h1;
  if (tdir == 0) {
    // Exact ties: a flagged nibble holds the lower code m (q's side) and the
    // upper code m+1 (magnitude m <= 6, so no carry leaves the nibble).  If m
    // is even, only bit 0 differs; if m is odd the increment carries into
    // bit 1.  Adding bit 1 of the difference therefore selects the even code.
    return ((uint64_t)(w1 + ((d1 & 0x22222222u) >> 1)) << 32) | (w0 + ((d0 & 0x22222222u) >> 1));
  }
  if (__builtin_expect((d0 | d1) != 0, 0)) {
    w0 = fix_word(w0, d0, 0, alpha, delta, load);
    w1 = fix_word(w1, d1, 8, alpha, delta, load);
  }
  return ((uint64_t)w1 << 32) | w0;
}

// Quantize one block on the fast path.  Returns false when the block must take
// the exact path (underflowed scale, values outside the guarded range, or an
// adaptive decision the certified f32 bound cannot settle).
template <int MODE, class Load>
__device__ __forceinline__ bool fast_block(const float2 (&x)[8], float bmax, const TensorConsts& tc,
                                           const Load& load, BlockOut& out) {
  // One unsigned compare keeps bmax in [2^-40, 2^40) (NaN and +-inf fail it).
  const uint32_t bb = __float_as_uint(bmax);
  if (__builtin_expect(bb - 0x2B800000u >= 0x28000000u, 0)) {
    if (bb != 0u) return false;
    // All-zero block: scale code 1 (blockquant.py:241), codes carry the sign
    // bit of -0.0 (codecs.py:109,116), both errors 0 -> tie keeps 6.
    uint64_t c = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      c |= (uint64_t)(__float_as_uint(x[p].x) >> 31) << (8 * p + 3);
      c |= (uint64_t)(__float_as_uint(x[p].y) >> 31) << (8 * p + 7);
    }
    out.codes = c;
    out.sc = 1;
    out.pick4 = (MODE == FIXED4);
    return true;
  }
  const float alpha = tc.alpha;
  if (MODE == FIXED6 || MODE == FIXED4) {
    const float m = MODE == FIXED6 ? 6.f : 4.f;
    const uint32_t sc = block_scale_code(bmax, alpha, m, MODE == FIXED6 ? tc.r6_lo : tc.r4_lo,
                                         MODE == FIXED6 ? tc.r6_hi : tc.r4_hi);
    if (sc == 0) return false;
    const float delta = e4m3_to_f32(sc);
    const float rq = rcp_approx(alpha * delta) * F46_QLO;
    out.codes = exact_codes(x, rq, alpha, delta, tc.tdir, load);
    out.sc = sc;
    out.pick4 = (MODE == FIXED4);
    return true;
  } else {
    // Both candidates' scale codes from one pair of bracketing quotients
    // (low byte: M=6, high byte: M=4).  A disagreement means bmax/(alpha*m)
    // lies within 2^-17 of an E4M3 tie; such blocks (and underflowed scales,
    // code 0 -- the M=4 code is never below the M=6 one) go to the exact path.
    const float2 b2 = make_float2(bmax, bmax);
    const float2 th = __fmul2_rn(b2, make_float2(tc.r6_hi, tc.r4_hi));
    const float2 tl = __fmul2_rn(b2, make_float2(tc.r6_lo, tc.r4_lo));
    const uint32_t ph = cvt_e4m3x2(th.y, th.x), pl = cvt_e4m3x2(tl.y, tl.x);
    if (__builtin_expect(ph != pl || (pl & 0xFFu) == 0u, 0)) return false;
    uint32_t dd;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(dd) : "h"((uint16_t)pl));
    const float2 dlt = make_float2(fhadd_h<0>(dd, -0.f), fhadd_h<1>(dd, -0.f));  // exact
    const float2 D = __fmul2_rn(make_float2(alpha, alpha), dlt);
    const float2 rq = __fmul2_rn(make_float2(rcp_approx(D.x), rcp_approx(D.y)),
                                 make_float2(F46_QLO, F46_QLO));
    const float2 sq = make_float2(cand_err(x, rq.x), cand_err(x, rq.y));
    // x-space sums S_m = D_m^2 * sq_m.  Certified bound on |S_m(f32) - S_m(ref)|
    // (DESIGN.md section "decision bound"): quotient error 2^-19.9 ->
    // 2^-18.9 * sqrt(S_m * sum x^2) <= 2^-16.9 * bmax * sqrt(S_m); codes taken
    // from the lower-bound quotient can differ from the exact ones only at
    // near-ties, moving S_m by <= 2^-15.1 * S_m; f32 rounding <= 2^-20 * S_m;
    // second-order quotient terms <= 2^-33.8 * bmax^2.  The first term is
    // covered through sqrt(s6) + sqrt(s4) <= sqrt(2 * (s6 + s4)).
    const float2 s = __fmul2_rn(sq, __fmul2_rn(D, D));
    const float ssum = s.x + s.y;
    const float tol = fmaf(0x1p-15f * bmax, sqrt_approx(ssum),
                           fmaf(0x1p-14f, ssum, fmaf(0x1p-32f * bmax, bmax, 0x1p-140f)));
    if (__builtin_expect(fabsf(s.x - s.y) <= tol, 0)) return false;  // exact path decides
    const bool k = s.y < s.x;
    out.codes = exact_codes(x, k ? rq.y : rq.x, alpha, k ? dlt.y : dlt.x, tc.tdir, load);
    out.sc = k ? (pl >> 8) : (pl & 0xFFu);
    out.pick4 = k;
    return true;
  }
}

// Straight-line variant of fast_block for the streaming kernel, with the
// tensor-wide tie direction as a template parameter (TDIR: -1, 0, +1, or 2 =
// unknown).  No early exits: every condition that sends a block to the exact
// path (all-zero or out-of-range bmax, near-tie or underflowed scale code,
// ambiguous 4/6 decision) folds into the returned flag, so consecutive blocks
// of one lane can be scheduled together.  Same arithmetic and bounds as
// fast_block.
// TDIR == 0 means alpha = amax/mcap exactly: alpha has <= 8 significant bits,
// so D = alpha*Delta (<= 12 bits) is exact in f32, every near-tie quotient is an
// exact tie, and non-ties stay >= 2^-16.3 (relative) away from one.  One
// Newton step  q1 = q0 - fma(q0, D, -x) * R  (residual exact, R ~ 1/D within
// 2^-22) lands exactly on a tie t (|q1 - t| <= t * 2^-43 before rounding) and
// within 2^-22 of every other quotient, so cvt.rn's ties-to-even is exact.
__device__ __forceinline__ uint64_t codes_newton(const float2 (&x)[8], float D, float R) {
  // Written as q1 = q0 + fma(q0, D, -x) * (-R) so that x = -0.0 keeps its sign
  // (every zero term is then -0 + -0); a +0 residual would turn q1 into +0.
  const float2 R2 = make_float2(R, R), nR2 = make_float2(-R, -R), D2 = make_float2(D, D);
  float2 q[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const float2 q0 = __fmul2_rn(x[p], R2);
    const float2 e = __ffma2_rn(q0, D2, make_float2(-x[p].x, -x[p].y));
    q[p] = __ffma2_rn(e, nR2, q0);
  }
  const uint32_t w0 = cvt_e2m1x8(q[0], q[1], q[2], q[3]);
  const uint32_t w1 = cvt_e2m1x8(q[4], q[5], q[6], q[7]);
  return ((uint64_t)w1 << 32) | w0;
}

// TDIR == 0 again (BF16 x: <= 8 significant bits; D = alpha*Delta exact),
// cheaper than the Newton step: split 1/D as Rhi + Rlo with Rhi truncated to
// 16 significant bits, so x*Rhi is exact in f32 (8 + 16 bits) and
// q0 = fma(x, Rlo, x*Rhi) is ONE rounding of x*(Rhi + Rlo) = q*(1 + e),
// |e| <= 2^-37 (Rlo = fma(-D, Rhi, 1)*R carries R's 2^-22 error on a 2^-16
// remainder).  An exact tie t therefore comes out as t exactly and every
// other quotient stays on its side of every tie (>= 2^-16.3 away), so
// cvt.rn's ties-to-even is the reference's rounding.  x = -0 stays -0.
__device__ __forceinline__ uint64_t codes_split(const float2 (&x)[8], float D) {
  const float R = rcp_approx(D);
  const float Rhi = __uint_as_float(__float_as_uint(R) & 0xFFFFFF00u);
  const float Rlo = fmaf(-D, Rhi, 1.0f) * R;
  const float2 H2 = make_float2(Rhi, Rhi), L2 = make_float2(Rlo, Rlo);
  float2 q[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) q[p] = __ffma2_rn(x[p], L2, __fmul2_rn(x[p], H2));
  const uint32_t w0 = cvt_e2m1x8(q[0], q[1], q[2], q[3]);
  const uint32_t w1 = cvt_e2m1x8(q[4], q[5], q[6], q[7]);
  return ((uint64_t)w1 << 32) | w0;
}

template <int TDIR, class Load>
__device__ __forceinline__ uint64_t codes_dir(const float2 (&x)[8], float rq, float D,
                                              float alpha, float delta, const Load& load) {
  if constexpr (TDIR < 0) {
    return codes_of(x, rq);
  } else if constexpr (TDIR == 1) {
    return codes_of(x, rq * F46_QHI_OVER_QLO);
  } else if constexpr (TDIR == 0) {
#if F46_NEWTON
    return codes_newton(x, D, rq);
#else
    return codes_split(x, D);
#endif
  } else {
    return exact_codes(x, rq, alpha, delta, TDIR, load);
  }
}

template <int MODE, int TDIR, class Load>
__device__ __forceinline__ bool block_sl(const float2 (&x)[8], float bmax, const TensorConsts& tc,
                                         const Load& load, BlockOut& out) {
  const uint32_t bb = __float_as_uint(bmax);
  bool ok = (bb - 0x2B800000u) < 0x28000000u;  // bmax in [2^-40, 2^40)
  const float alpha = tc.alpha;
  if constexpr (MODE == FIXED6 || MODE == FIXED4) {
    const float2 t = __fmul2_rn(make_float2(bmax, bmax), MODE == FIXED6
                                                             ? make_float2(tc.r6_hi, tc.r6_lo)
                                                             : make_float2(tc.r4_hi, tc.r4_lo));
    const uint32_t pr = cvt_e4m3x2(t.x, t.y);  // low byte: lower bracket
    const uint32_t sc = pr & 0xFFu;
    ok &= ((pr >> 8) == sc) & (sc != 0u);
    const float delta = e4m3_to_f32(sc);
    const float D = alpha * delta;
    const float rq = rcp_approx(D) * F46_QLO;
    out.codes = codes_dir<TDIR>(x, rq, D, alpha, delta, load);
    out.sc = sc;
    out.pick4 = (MODE == FIXED4);
  } else {
    const float2 b2 = make_float2(bmax, bmax);
    const float2 th = __fmul2_rn(b2, make_float2(tc.r6_hi, tc.r4_hi));
    const float2 tl = __fmul2_rn(b2, make_float2(tc.r6_lo, tc.r4_lo));
    const uint32_t ph = cvt_e4m3x2(th.y, th.x), pl = cvt_e4m3x2(tl.y, tl.x);
    ok &= (ph == pl) & ((pl & 0xFFu) != 0u);
    uint32_t dd;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(dd) : "h"((uint16_t)pl));
    const float2 dlt = make_float2(fhadd_h<0>(dd, -0.f), fhadd_h<1>(dd, -0.f));
    const float2 D = __fmul2_rn(make_float2(alpha, alpha), dlt);
    const float2 rq = __fmul2_rn(make_float2(rcp_approx(D.x), rcp_approx(D.y)),
                                 make_float2(F46_QLO, F46_QLO));
    const float2 sq = make_float2(cand_err(x, rq.x), cand_err(x, rq.y));
    const float2 s = __fmul2_rn(sq, __fmul2_rn(D, D));
    const float ssum = s.x + s.y;
    const float tol = fmaf(0x1p-15f * bmax, sqrt_approx(ssum),
                           fmaf(0x1p-14f, ssum, fmaf(0x1p-32f * bmax, bmax, 0x1p-140f)));
    ok &= fabsf(s.x - s.y) > tol;  // NaN (from a rejected block) compares false
    const bool k = s.y < s.x;
    out.codes = codes_dir<TDIR>(x, k ? rq.y : rq.x, k ? D.y : D.x, alpha, k ? dlt.y : dlt.x, load);
    out.sc = k ? (pl >> 8) : (pl & 0xFFu);
    out.pick4 = k;
  }
  return ok;
}

// ----------------------------------------------------------------------------
// Candidate pass that keeps its codes (adaptive, BF16, known tie direction)
// ----------------------------------------------------------------------------

// The 8 E2M1 codes of one packed word -> four f16x2 values (exact).  ptxas
// reads each byte with the unpack's byte selector (F2FP.F16.E2M1.UNPACK_B
// Rw.B1/.B2/.B3), so no byte extraction is emitted -- but only when `w` is
// opaque to it: if ptxas can see that w was assembled from cvt bytes
// (cvt_e2m1x8) it forwards the bytes and, under 12.9, reads bytes 2 and 3 of
// the 4-way .b8 split from RZ.  Callers therefore pass w ^ z with z a runtime
// zero (one LOP3 per word).
__device__ __forceinline__ void unpack_e2m1x8(uint32_t w, uint32_t (&v)[4]) {
  asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
      "mov.b32 {b0, b1, b2, b3}, %4;\n\t"
      "cvt.rn.f16x2.e2m1x2 %0, b0;\n\t"
      "cvt.rn.f16x2.e2m1x2 %1, b1;\n\t"
      "cvt.rn.f16x2.e2m1x2 %2, b2;\n\t"
      "cvt.rn.f16x2.e2m1x2 %3, b3;\n\t}"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
      : "r"(w));
}

// One candidate of one block: codes of q = x*rq packed into two words (the
// F2FP merge chain builds each word without byte shuffles) and decoded back
// from the words, and the quotient-space error  sum_i (v_i - q_i)^2  (f32x2
// accumulator, as cand_err).  The codes are those of the quotient q itself, so
// when rq is the bound that the tensor's tie direction makes exact (lower
// bound for TDIR -1, upper bound for +1) they are the reference's codes and the
// stored candidate needs no second pass.
__device__ __forceinline__ float cand_codes(const float2 (&x)[8], float rq, uint32_t z,
                                            uint32_t& w0, uint32_t& w1) {
  const float2 r2 = make_float2(rq, rq);
  float2 q[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) q[p] = __fmul2_rn(x[p], r2);
  w0 = cvt_e2m1x8(q[0], q[1], q[2], q[3]) ^ z;  // z == 0 (see unpack_e2m1x8)
  w1 = cvt_e2m1x8(q[4], q[5], q[6], q[7]) ^ z;
  uint32_t v[8];
  unpack_e2m1x8(w0, *reinterpret_cast<uint32_t(*)[4]>(&v[0]));
  unpack_e2m1x8(w1, *reinterpret_cast<uint32_t(*)[4]>(&v[4]));
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const float2 r = make_float2(fhadd_h<0>(v[p], -q[p].x), fhadd_h<1>(v[p], -q[p].y));
    acc = __ffma2_rn(r, r, acc);
  }
  return acc.x + acc.y;
}

// Adaptive block, BF16 input, computed alpha (TDIR -1, 0 or +1): block_sl with
// the candidates' codes kept.  TDIR -1 / +1: the candidate pass runs on the
// lower / upper bound quotient, whose codes are exact (tie_direction()), so
// the winner's codes are a select.  TDIR 0: the pass runs on the lower bound;
// only the winner's upper-bound codes are formed, and a nibble where the two
// differ is an exact tie (exact_codes's tdir 0 rule picks the even code).  The
// upper-bound quotient is within 2^-19.5 of the exact one, inside the 2^-15
// decision tolerance's margin (the lower bound's 2^-19.9 gives 2^-16.4 of it).
// Per-tensor table of everything block46 derives from a scale code c
// (0..127): {rq, rh, D*D, c} with D = RN(alpha * E4M3(c)), rq = RN(rcp(D) * QLO),
// rh = RN(rq * QHI_OVER_QLO) -- the same roundings block_sl performs per block.
// Code 0 (an underflowed scale) maps to NaN, which fails the decision test.
__device__ __forceinline__ float4 scale_entry(uint32_t c, float alpha) {
  const float D = alpha * e4m3_to_f32(c);
  const float rq = rcp_approx(D) * F46_QLO;
  float4 e = make_float4(rq, rq * F46_QHI_OVER_QLO, D * D, __uint_as_float(c));
  if (c == 0) e.x = e.y = e.z = __uint_as_float(0x7FC00000u);
  return e;
}

// The E4M3 code of bmax/(alpha*m) when the bracket gave lo and lo + 1: the
// tie T between them (5 significant bits, T*m exact in f32) decides with one
// correctly rounded fma; an exact tie goes to the even code (codecs.py:158-178).
__device__ __forceinline__ uint32_t scale_tie(uint32_t lo, float bmax, float alpha, float m) {
  const float T = 0.5f * (e4m3_to_f32(lo) + e4m3_to_f32(lo + 1));
  const float s = fmaf(alpha, T * m, -bmax);
  return s > 0.f ? lo : (s < 0.f ? lo + 1 : ((lo & 1u) ? lo + 1 : lo));
}

// True when bmax/(alpha*m) can land exactly on an E4M3 tie for a BF16 bmax:
// bmax = alpha * m * T needs odd(alpha) * odd(m) * odd(T) <= 255 with odd(T)
// >= 17 (a tie between two 4-bit significands has 5), i.e. odd(alpha) <= 15.
// Only tensors whose alpha has that few significant bits need block46's
// in-place tie resolution; the rest keep the leaner straight line.
__device__ __forceinline__ bool e4m3_ties_possible(float alpha) {
  const uint32_t sig = (__float_as_uint(alpha) & 0x7FFFFFu) | 0x800000u;
  return (sig >> (__ffs(sig) - 1)) <= 15u;
}

// TDIR 0 (alpha = amax / mcap exactly, so D = alpha * E4M3(c) is exact and
// every near-tie quotient is an exact FP4 tie, tie_direction()): look for a
// reciprocal R of D, within 4 ulps of RN(1/D), such that for every tie t whose
// value t*D is a BF16 number (the only ties an element can hit) cvt.rn of
// RN(t*D*R) gives the reference's code (ties to even).  Non-tie quotients lie
// >= 2^-16.3 (relative) from every tie and x*R is within 2^-20.5 of x/D, so
// with such an R the codes of x*R are the reference's for every element: the
// candidate pass can keep its codes with no upper-bound pass.  Returns false
// when no such R exists (then the tensor keeps the two-bound TDIR 0 path).
__device__ __forceinline__ bool safe_recip(uint32_t c, float alpha, float& R) {
  const float D = alpha * e4m3_to_f32(c);
  if (!(D > 0.f) || !(D < 1e30f)) return false;
  const float R0 = __frcp_rn(D);
  // the ties' reference codes (RNE on the code index): 0.25->0 .75->2 1.25->2
  // 1.75->4 2.5->4 3.5->6 5->6
  const float ties[7] = {0.25f, 0.75f, 1.25f, 1.75f, 2.5f, 3.5f, 5.f};
  const uint32_t want[7] = {0, 2, 2, 4, 4, 6, 6};
#pragma unroll 1
  for (int s = 0; s < 9; ++s) {
    const int k = (s & 1) ? (s + 1) / 2 : -(s / 2);  // 0, 1, -1, 2, -2, ...
    const float r = __int_as_float(__float_as_int(R0) + k);
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const float x = ties[i] * D;  // exact: <= 3 + 12 significant bits
      if ((__float_as_uint(x) & 0xFFFFu) != 0u) continue;  // not a BF16 value
      const float2 q = make_float2(x * r, x * r);
      ok &= (cvt_e2m1x8(q, q, q, q) & 0xFu) == want[i];
    }
    if (ok) {
      R = r;
      return true;
    }
  }
  return false;
}

__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}

// Adaptive block, BF16 input, computed alpha (TDIR -1, 0 or +1): block_sl with
// the candidates' codes kept.  TDIR -1 / +1: the candidate pass runs on the
// lower / upper bound quotient, whose codes are exact (tie_direction()), so
// the winner's codes are a select.  TDIR 0: the pass runs on the lower bound;
// only the winner's upper-bound codes are formed, and a nibble where the two
// differ is an exact tie whose even code is kept (exact_codes' tdir 0 rule).
// The upper-bound quotient is within 2^-19.5 of the exact one, inside the 2^-15
// decision tolerance's margin (the lower bound's 2^-19.9 gives 2^-16.4 of it).
// The per-code reciprocals come from the shared table `tab` (scale_entry).
template <int TDIR, bool TIE = false>
__device__ __forceinline__ bool block46(const float2 (&x)[8], float bmax, const TensorConsts& tc,
                                        uint32_t tab, BlockOut& out) {
  const uint32_t bb = __float_as_uint(bmax);
  bool ok = (bb - 0x2B800000u) < 0x28000000u;  // bmax in [2^-40, 2^40)
  const float2 b2 = make_float2(bmax, bmax);
  const float2 th = __fmul2_rn(b2, make_float2(tc.r6_hi, tc.r4_hi));
  const float2 tl = __fmul2_rn(b2, make_float2(tc.r6_lo, tc.r4_lo));
  const uint32_t ph = cvt_e4m3x2(th.y, th.x);
  uint32_t pl = cvt_e4m3x2(tl.y, tl.x);
  if (TIE) {
#if F46_SCALE_TDIR
    // alpha has few significant bits and tie direction 0 (alpha = beta): a
    // bracket disagreement is an exact tie ("Scale codes" above), so the
    // reference's ties-to-even takes the even code of the two -- the upper
    // byte wherever the lower one is odd (equal bytes: either)
    const uint32_t odd = (pl & 0x0101u) * 0xFFu;
    pl = (pl & ~odd) | (ph & odd);
#else
    if (__builtin_expect(ph != pl, 0)) {
      // settle the scale code exactly in place (block_scale_code's test)
      const uint32_t lo6 = pl & 0xFFu, lo4 = (pl >> 8) & 0xFFu;
      const uint32_t s6 = lo6 != (ph & 0xFFu) ? scale_tie(lo6, bmax, tc.alpha, 6.f) : lo6;
      const uint32_t s4 = lo4 != ((ph >> 8) & 0xFFu) ? scale_tie(lo4, bmax, tc.alpha, 4.f) : lo4;
      pl = s6 | (s4 << 8);
    }
#endif
  }
  if (!TIE) ok &= (ph == pl);
#if F46_TAB
  const float4 e6 = lds_f4(tab + ((pl << 4) & 0xFF0u));
  const float4 e4 = lds_f4(tab + ((pl >> 4) & 0xFF0u));
#else
  // the same entries computed in place (packed over the two candidates)
  ok &= (pl & 0xFFu) != 0u;
  uint32_t dd;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(dd) : "h"((uint16_t)pl));
  const float2 dlt = make_float2(fhadd_h<0>(dd, -0.f), fhadd_h<1>(dd, -0.f));
  const float2 D = __fmul2_rn(make_float2(tc.alpha, tc.alpha), dlt);
  const float2 rq2 = __fmul2_rn(make_float2(rcp_approx(D.x), rcp_approx(D.y)),
                                make_float2(F46_QLO, F46_QLO));
  const float2 rh2 = TDIR >= 0 ? __fmul2_rn(rq2, make_float2(F46_QHI_OVER_QLO, F46_QHI_OVER_QLO)) : rq2;
  const float2 DD = __fmul2_rn(D, D);
  const float4 e6 = make_float4(rq2.x, rh2.x, DD.x, __uint_as_float(pl & 0xFFu));
  const float4 e4 = make_float4(rq2.y, rh2.y, DD.y, __uint_as_float(pl >> 8));
#endif
  // TDIR 3: the table's x field holds safe_recip's R (codes exact as computed);
  // TDIR 4: x holds whichever reciprocal gives exact codes for the tensor (the
  // lower bound for -1, the upper bound for +1, safe_recip's R for 3)
  const float2 rq = TDIR == 1 ? make_float2(e6.y, e4.y) : make_float2(e6.x, e4.x);
  uint32_t a0, a1, b0, b1;  // M=6 and M=4 code words
  const float2 sq = make_float2(cand_codes(x, rq.x, tc.zero, a0, a1), cand_codes(x, rq.y, tc.zero, b0, b1));
  const float2 s = __fmul2_rn(sq, make_float2(e6.z, e4.z));
  const float ssum = s.x + s.y;
  // block_sl's tolerance with its square root bounded by AM-GM:
  // 2^-15 bmax sqrt(ssum) <= 2^-18 bmax^2 + 2^-14 ssum, so
  // tol <= (2^-14 + 2^-14) ssum + (2^-18 + 2^-32) bmax^2 + 2^-140.
  const float tol = fmaf(0x1.002p-13f, ssum, fmaf(0x1.002p-18f * bmax, bmax, 0x1p-140f));
  ok &= fabsf(s.x - s.y) > tol;  // NaN (underflowed scale, rejected block) compares false
  const bool k = s.y < s.x;
  uint32_t w0 = k ? b0 : a0, w1 = k ? b1 : a1;
  if constexpr (TDIR == 0) {
    const uint64_t hi = codes_of(x, k ? e4.y : e6.y);
    // nibbles where the bounds disagree are exact ties: keep the even code
    // (the lower code when it is even, else the upper one)
    const uint32_t m0 = (w0 & 0x11111111u) * 15u, m1 = (w1 & 0x11111111u) * 15u;
    w0 ^= (w0 ^ (uint32_t)hi) & m0;
    w1 ^= (w1 ^ (uint32_t)(hi >> 32)) & m1;
  }
  out.codes = ((uint64_t)w1 << 32) | w0;
  out.sc = __float_as_uint(k ? e4.w : e6.w);
  out.pick4 = k;
  return ok;
}

// ----------------------------------------------------------------------------
// tcgen05 scale layout (128 rows x 4 blocks per 512-byte tile)
// ----------------------------------------------------------------------------
__device__ __host__ __forceinline__ int64_t sf_tc_offset(int64_t r, int64_t kb, int64_t kb4) {
  return ((r >> 7) * kb4 + (kb >> 2)) * 512 + (r & 31) * 16 + ((r & 127) >> 5) * 4 + (kb & 3);
}
// the same in 32-bit arithmetic (scale tables below 4 GB)
__device__ __forceinline__ uint32_t sf_tc_offset32(uint32_t r, uint32_t kb, uint32_t kb4) {
  return ((r >> 7) * kb4 + (kb >> 2)) * 512u + (r & 31u) * 16u + ((r & 127u) >> 5) * 4u + (kb & 3u);
}

}  // namespace f46

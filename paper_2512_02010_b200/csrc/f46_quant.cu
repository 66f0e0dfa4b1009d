// f46_quant.cu -- amax, 4/6 quantize and dequantize kernels + their C ABI.
//
// Kernels (sm_100a):
//   amax_kernel          K1: grid-stride 128-bit loads (4 in flight), warp-shuffle
//                        max, one 64-bit atomicMax on the float64 bit pattern per CTA.
//   quant_seg_kernel     K2: each warp streams contiguous 2048-element segments of
//                        the input through a 2-stage cp.async.bulk -> shared memory
//                        pipeline; lane l quantizes blocks l, l+32, ... of the
//                        segment with the straight-line fast path (f46_device.cuh),
//                        stores 8 B of packed E2M1 codes (coalesced) and the E4M3
//                        scale into the tcgen05 128x4 layout; uncertified blocks are
//                        queued per warp and resolved exactly afterwards.
//                        Requires cols % 16 == 0.
//   quant_generic_kernel any shape / float64 input: one thread per block.
//   quant2d_kernel       16x16-tile weight quantization (exact f64), writes W and W^T.
//   quant_sr_kernel      stochastic rounding with numpy-Philox-exact uniforms.
//   stats_kernel         fused selection statistics (fraction_4 per rule).
//   rht16_kernel         16-wide randomized Hadamard transform (f64, numpy order).
//   dequant_tma_kernel   K3: per-warp 1024-element chunks, TMA-staged stores.
//   dequant_vec_kernel / dequant_kernel  K3 fallbacks (unaligned / ragged / f64 out).
//
// Reference: blockquant.py:215-222, :334-376; adaptive.py:60-101.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <mutex>
#include <type_traits>

#include "../../include/fouroversix.h"
#include "f46_device.cuh"
#include "f46_runtime.h"

using namespace f46;

namespace {

#ifndef F46_STAGES
#define F46_STAGES 2
#endif
constexpr int kStages = F46_STAGES;

int num_sms() { return f46rt::num_sms(); }
void udiv_magic(uint32_t d, uint32_t* magic, uint32_t* sh1, uint32_t* sh2);

// ---------------------------------------------------------------------------
// mbarrier / TMA helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// ---------------------------------------------------------------------------
// Parameters
// ---------------------------------------------------------------------------
struct QParams {
  const void* x;
  int64_t rows, cols;
  int mode, rule, dtype;
  double mcap;
  const double* d_amax;
  double alpha_override;
  uint8_t* codes;
  uint8_t* scales_tc;
  uint8_t* scales_rm;
  uint8_t* pick4;
  double* d_alpha_out;
  uint32_t* d_flags;
  // grouped launches (gridDim.y groups): per-group strides of x (bytes), codes
  // and scales_tc (bytes); d_amax / d_alpha_out are indexed by the group
  int64_t g_x, g_codes, g_scales;
  // flat streaming: block b -> row b / nb as t = umulhi(b, nb_magic),
  // row = (t + ((b - t) >> nb_sh1)) >> nb_sh2 (udiv_magic, set by the launcher)
  uint32_t nb_magic, nb_sh1, nb_sh2;
  // fused amax + quantize (f46_quantize_fused): grid-barrier counter, zeroed
  // by the caller with d_amax; null for the two-kernel path
  uint32_t* d_sync;
};

// Point the parameters at group blockIdx.y of a grouped launch.
__device__ __forceinline__ void select_group(QParams& p) {
  if (gridDim.y > 1) {
    const int64_t g = blockIdx.y;
    p.x = reinterpret_cast<const uint8_t*>(p.x) + g * p.g_x;
    p.codes += g * p.g_codes;
    p.scales_tc += g * p.g_scales;
    if (p.d_amax) p.d_amax += g;
    if (p.d_alpha_out) p.d_alpha_out += g;
  }
}

// blockquant.py:215-222 / :316-326: alpha = RN32(f32(amax) / f32(mcap)), 1.0
// for an all-zero tensor, or the override.
__device__ __forceinline__ double resolve_alpha(const QParams& p) {
  if (p.alpha_override > 0.0) return p.alpha_override;
  const double amax = __ldcg(p.d_amax);
  if (amax == 0.0) return 1.0;
  return (double)((float)amax / (float)p.mcap);
}

__device__ __forceinline__ void prologue_flags(const QParams& p, double alpha) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.d_alpha_out) *p.d_alpha_out = alpha;
    if (p.alpha_override <= 0.0 && p.d_flags) {
      const double amax = __ldcg(p.d_amax);
      if (!(amax <= 1.7976931348623157e308)) atomicOr(p.d_flags, F46_FLAG_NONFINITE);
    }
  }
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

// Re-read element i of the thread's block from the shared-memory segment
// (`blk` = shared-space address of the block's first element).
template <int DT>
struct SegLoad {
  uint32_t blk;
  __device__ __forceinline__ float operator()(int i) const {
    if constexpr (DT == DT_BF16)
      return __uint_as_float(lds_u16(blk + i * 2) << 16);
    else
      return lds_f32(blk + i * 4);
  }
};

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

template <int DT>
__device__ __forceinline__ void load_block(uint32_t blk, float2 (&x)[8], float& bmax) {
  if constexpr (DT == DT_BF16) {
    const uint4 a = lds128(blk);
    const uint4 b = lds128(blk + 16);
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int p = 0; p < 8; ++p) x[p] = bf16x2_unpack(w[p]);
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = lds128(blk + 16 * c);
      x[2 * c] = make_float2(__uint_as_float(v.x), __uint_as_float(v.y));
      x[2 * c + 1] = make_float2(__uint_as_float(v.z), __uint_as_float(v.w));
    }
  }
  // NaN-propagating max: a NaN (or inf) block fails the fast path's range
  // guard and is flagged on the exact path.
  float m0 = fmax_nan(fabsf(x[0].x), fabsf(x[0].y)), m1 = fmax_nan(fabsf(x[1].x), fabsf(x[1].y));
#pragma unroll
  for (int p = 2; p < 8; p += 2) {
    m0 = fmax_nan(m0, fmax_nan(fabsf(x[p].x), fabsf(x[p].y)));
    m1 = fmax_nan(m1, fmax_nan(fabsf(x[p + 1].x), fabsf(x[p + 1].y)));
  }
  bmax = fmax_nan(m0, m1);
}

// ---------------------------------------------------------------------------
// K2: bulk-copy-pipelined quantize (cols % 16 == 0)
//
// Each warp is an independent pipeline over "segments": kSegElems contiguous
// elements of one row (4 KB of bf16 / 8 KB of f32).  Lane 0 streams segments
// into kStages shared-memory stages with 1-D bulk copies (cp.async.bulk,
// mbarrier complete_tx); lane l then quantizes blocks l, l+32, l+64, l+96 of
// the segment, so the warp's 8-byte code stores are fully coalesced (256 B per
// instruction).  Blocks the fast path cannot certify are queued in a per-warp
// shared list and recomputed exactly outside the hot loop.
// ---------------------------------------------------------------------------
constexpr int kWarps = 4;
#ifndef F46_SEG
#define F46_SEG 2048
#endif
constexpr int kSegElems = F46_SEG;
#ifndef F46_KB_UNROLL
#define F46_KB_UNROLL 4
#endif
constexpr int kKbUnroll = F46_KB_UNROLL;
#ifndef F46_MINB
#define F46_MINB 4
#endif
#ifndef F46_FULL
#define F46_FULL 1
#endif
#ifndef F46_FLAT
#define F46_FLAT 1
#endif
#ifndef F46_PAR_RESOLVE
#define F46_PAR_RESOLVE 1
#endif
// inputs up to this size take the parallel-resolver instantiation (the fused
// amax+quantize path's range)
constexpr int64_t kParResolveMaxBytes = (int64_t)96 << 20;
#ifndef F46_RL_INLINE
#define F46_RL_INLINE __noinline__
#endif
#ifndef F46_NO_DEFER_PROBE
#define F46_NO_DEFER_PROBE 0
#endif
#ifndef F46_SF_UNROLL
#define F46_SF_UNROLL 4
#endif
constexpr int kSfUnroll = F46_SF_UNROLL;
// the small-tensor (parallel-resolver) instantiation: a rolled block loop
// keeps its hot code small, which matters when each warp streams only a few
// tiles and the instruction cache is cold
#ifndef F46_SF_UNROLL_SMALL
#define F46_SF_UNROLL_SMALL 1
#endif
constexpr int kSfUnrollSmall = F46_SF_UNROLL_SMALL;
#ifndef F46_T4
#define F46_T4 1
#endif
#ifndef F46_T3
#define F46_T3 1
#endif
#ifndef F46_STEP2
#define F46_STEP2 0
#endif
#ifndef F46_V3
#define F46_V3 1
#endif
#ifndef F46_UNCOND_STORE
#define F46_UNCOND_STORE 1
#endif

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Exact f64 recomputation of one block, reading its 16 values from global
// memory (used for the rare blocks the fast path defers).  Arguments by value:
// taking the address of the kernel's parameter struct would force a copy to
// local memory.
struct ExactArgs {
  const void* x;
  uint8_t* codes;
  uint8_t* scales_tc;
  uint8_t* scales_rm;
  uint8_t* pick4;
  int64_t cols;
  int mode, rule;
};

template <int DT>
__device__ __forceinline__ void exact_block_global(ExactArgs a, double alpha, uint32_t blk,
                                                   uint32_t kb4, uint32_t* nonfinite) {
  const int64_t nb = (a.cols + 15) >> 4;
  const int64_t row = blk / nb, kbg = blk - row * nb;
  double xd[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int64_t c = kbg * 16 + i;
    if (c >= a.cols)
      xd[i] = 0.0;
    else if constexpr (DT == DT_BF16)
      xd[i] = (double)__uint_as_float(
          (uint32_t)(reinterpret_cast<const uint16_t*>(a.x)[row * a.cols + c]) << 16);
    else
      xd[i] = (double)reinterpret_cast<const float*>(a.x)[row * a.cols + c];
  }
  bool nf = false, zero = true;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    nf |= !(fabs(xd[i]) <= 3.4028234663852886e38);
    zero &= (xd[i] == 0.0);
  }
  if (nf && nonfinite) atomicOr(nonfinite, F46_FLAG_NONFINITE);
  BlockOut o;
  if (zero) {
    // all-zero block (blockquant.py:241): scale code 1, codes keep the sign of -0.0
    // (codecs.py:109,116); both candidate errors are 0, so the tie keeps 6.
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) c |= (uint64_t)(signbit(xd[i]) ? 8u : 0u) << (4 * i);
    o.codes = c;
    o.sc = 1;
    o.pick4 = (a.mode == FIXED4);
  } else {
    exact_block_inl(xd, alpha, a.mode, a.rule, &o);
  }
  *reinterpret_cast<uint64_t*>(a.codes + (row * nb + kbg) * 8) = o.codes;
  a.scales_tc[sf_tc_offset(row, kbg, kb4)] = (uint8_t)o.sc;
  if (a.scales_rm) a.scales_rm[row * nb + kbg] = (uint8_t)o.sc;
  if (a.pick4) a.pick4[row * nb + kbg] = (uint8_t)o.pick4;
}

// A block the streaming loop deferred (cols % 16 == 0, not force_exact).  Most
// deferrals are a near-tie block scale or a 4/6 decision inside the f32
// tolerance, not a value outside the fast path's range, so the exact answer is
// reached without the float64 quantizer: both scale codes are settled exactly
// (block_scale_code's tie test), both candidates' codes come from the proven
// bracket logic (exact_codes), and only the two error sums are recomputed in
// float64 in the reference's pairwise order (exact_sq_sum) -- the reference's
// own arithmetic on identical codes (blockquant.py:279, :289-290; adaptive.py:
// 77-80).  Zero, out-of-range and underflowing blocks take exact_block_global.
template <int DT, int MODE>
__device__ __noinline__ void resolve_block_global(ExactArgs a, TensorConsts tc, uint32_t blk,
                                                  uint32_t kb4, uint32_t* flags) {
  const uint32_t nb = (uint32_t)(a.cols >> 4);
  const uint32_t row = blk / nb, kbg = blk - row * nb;
  const int64_t e0 = (int64_t)row * a.cols + (int64_t)kbg * 16;
  auto load = [&](int i) -> float {
    if constexpr (DT == DT_BF16)
      return __uint_as_float((uint32_t)(reinterpret_cast<const uint16_t*>(a.x)[e0 + i]) << 16);
    else
      return reinterpret_cast<const float*>(a.x)[e0 + i];
  };
  float2 x[8];
  float bmax = 0.f;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    x[p] = make_float2(load(2 * p), load(2 * p + 1));
    bmax = fmax_nan(bmax, fmax_nan(fabsf(x[p].x), fabsf(x[p].y)));
  }
  const uint32_t bb = __float_as_uint(bmax);
  if ((bb - 0x2B800000u) >= 0x28000000u) {  // zero, tiny, huge or non-finite
    exact_block_global<DT>(a, tc.alpha_d, blk, kb4, flags);
    return;
  }
  const float alpha = tc.alpha;
  BlockOut o;
  if constexpr (MODE == FIXED6 || MODE == FIXED4) {
    const float m = MODE == FIXED6 ? 6.f : 4.f;
    const uint32_t sc = block_scale_code(bmax, alpha, m, MODE == FIXED6 ? tc.r6_lo : tc.r4_lo,
                                         MODE == FIXED6 ? tc.r6_hi : tc.r4_hi);
    if (sc == 0) {
      exact_block_global<DT>(a, tc.alpha_d, blk, kb4, flags);
      return;
    }
    const float delta = e4m3_to_f32(sc);
    const float rq = rcp_approx(alpha * delta) * F46_QLO;
    o.codes = exact_codes(x, rq, alpha, delta, tc.tdir, load);
    o.sc = sc;
    o.pick4 = (MODE == FIXED4);
  } else {
    const uint32_t sc6 = block_scale_code(bmax, alpha, 6.f, tc.r6_lo, tc.r6_hi);
    const uint32_t sc4 = block_scale_code(bmax, alpha, 4.f, tc.r4_lo, tc.r4_hi);
    if (sc6 == 0 || sc4 == 0) {
      exact_block_global<DT>(a, tc.alpha_d, blk, kb4, flags);
      return;
    }
    const float d6 = e4m3_to_f32(sc6), d4 = e4m3_to_f32(sc4);
    const uint64_t c6 = exact_codes(x, rcp_approx(alpha * d6) * F46_QLO, alpha, d6, tc.tdir, load);
    const uint64_t c4 = exact_codes(x, rcp_approx(alpha * d4) * F46_QLO, alpha, d4, tc.tdir, load);
    double xd[16];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      xd[2 * p] = (double)x[p].x;
      xd[2 * p + 1] = (double)x[p].y;
    }
    const double s6 = exact_sq_sum(xd, c6, tc.alpha_d, (double)d6);
    const double s4 = exact_sq_sum(xd, c4, tc.alpha_d, (double)d4);
    const bool k = s4 < s6;  // strict: ties keep 6 (adaptive.py:77-80)
    o.codes = k ? c4 : c6;
    o.sc = k ? sc4 : sc6;
    o.pick4 = k;
  }
  *reinterpret_cast<uint64_t*>(a.codes + (int64_t)blk * 8) = o.codes;
  a.scales_tc[sf_tc_offset(row, kbg, kb4)] = (uint8_t)o.sc;
  if (a.scales_rm) a.scales_rm[blk] = (uint8_t)o.sc;
  if (a.pick4) a.pick4[blk] = (uint8_t)o.pick4;
}

// Two deferred blocks per warp, 16 lanes each (lane i of a half owns element
// i): the exact answer of resolve_block_global -- scale codes from the exact
// tie test, codes from the proven bracket logic per element, the two squared
// error sums in float64 in numpy's pairwise order (r_j = e_j + e_{j+8}, then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), blockquant.py:289-290) through
// half-warp shuffles, strict '<' (adaptive.py:77-80) -- with the element work
// spread over the lanes, so the resolve pass after the hot loop is short.
// Zero, tiny, huge, non-finite and underflowing blocks keep the single-lane
// float64 restatement (exact_block_global).  All 32 lanes call it.
__device__ __forceinline__ uint32_t exact_code_elem(float x, float rq, float alpha, float delta,
                                                    int tdir) {
  const float ql = x * rq, qh = ql * F46_QHI_OVER_QLO;
  const uint32_t cl = cvt_e2m1x8(make_float2(ql, ql), make_float2(ql, ql), make_float2(ql, ql),
                                 make_float2(ql, ql)) & 0xFu;
  const uint32_t ch = cvt_e2m1x8(make_float2(qh, qh), make_float2(qh, qh), make_float2(qh, qh),
                                 make_float2(qh, qh)) & 0xFu;
  if (cl == ch) return cl;
  if (tdir < 0) return cl;
  if (tdir == 1) return ch;
  if (tdir == 0) return (cl & 1u) ? ch : cl;  // an exact tie: the even code
  const uint32_t m = cl & 7u;
  const float s = fmaf(alpha, fp4_tie_above(m) * delta, -fabsf(x));
  return cl + ((s < 0.f) | ((s == 0.f) & (m & 1u)));
}

template <int DT, int MODE>
__device__ __forceinline__ void resolve_pair(const ExactArgs& a, const TensorConsts& tc, uint32_t kb4,
                                             uint32_t* flags, uint32_t blk_lo, uint32_t blk_hi,
                                             bool has_hi) {
  const unsigned FULL = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31, i = lane & 15;
  const bool hi_half = lane >= 16;
  const uint32_t blk = hi_half ? blk_hi : blk_lo;
  const bool valid = !hi_half || has_hi;
  const uint32_t nb = (uint32_t)(a.cols >> 4);
  const uint32_t row = blk / nb, kbg = blk - row * nb;
  const int64_t e0 = (int64_t)row * a.cols + (int64_t)kbg * 16;
  float x = 0.f;
  if (valid) {
    if constexpr (DT == DT_BF16)
      x = __uint_as_float((uint32_t)(reinterpret_cast<const uint16_t*>(a.x)[e0 + i]) << 16);
    else
      x = reinterpret_cast<const float*>(a.x)[e0 + i];
  }
  float bmax = fabsf(x);
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) bmax = fmax_nan(bmax, __shfl_xor_sync(FULL, bmax, o, 16));
  const uint32_t bb = __float_as_uint(bmax);
  const float alpha = tc.alpha;
  uint32_t sc6 = 0, sc4 = 0;
  bool special = (bb - 0x2B800000u) >= 0x28000000u;  // zero, tiny, huge or non-finite
  if (!special) {
    if constexpr (MODE == ADAPTIVE) {
      sc6 = block_scale_code(bmax, alpha, 6.f, tc.r6_lo, tc.r6_hi);
      sc4 = block_scale_code(bmax, alpha, 4.f, tc.r4_lo, tc.r4_hi);
    } else {
      sc6 = MODE == FIXED6 ? block_scale_code(bmax, alpha, 6.f, tc.r6_lo, tc.r6_hi)
                           : block_scale_code(bmax, alpha, 4.f, tc.r4_lo, tc.r4_hi);
      sc4 = sc6;
    }
    special = sc6 == 0 || sc4 == 0;
  }
  // every lane keeps shuffling (inactive and special halves with dummy values);
  // special blocks are settled by one lane after the last shuffle
  uint64_t word[2];
  double S[2];
  const int ncand = MODE == ADAPTIVE ? 2 : 1;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (k >= ncand) break;
    const uint32_t sc = special ? 0x38u : (k == 0 ? sc6 : sc4);
    const float delta = e4m3_to_f32(sc);
    const float rq = rcp_approx(alpha * delta) * F46_QLO;
    const uint32_t c = exact_code_elem(x, rq, alpha, delta, tc.tdir);
    uint64_t w = (uint64_t)c << (4 * i);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) w |= __shfl_xor_sync(FULL, w, o, 16);
    word[k] = w;
    const double diff = __dsub_rn(__dmul_rn(dec_fp4_d(c), __dmul_rn(tc.alpha_d, (double)delta)),
                                  (double)x);
    const double e = __dmul_rn(diff, diff);
    const double r = __dadd_rn(e, __shfl_down_sync(FULL, e, 8, 16));     // j < 8: e_j + e_{j+8}
    const double p1 = __dadd_rn(r, __shfl_down_sync(FULL, r, 1, 16));    // j even
    const double p2 = __dadd_rn(p1, __shfl_down_sync(FULL, p1, 2, 16));  // j % 4 == 0
    const double p3 = __dadd_rn(p2, __shfl_down_sync(FULL, p2, 4, 16));  // j == 0
    S[k] = __shfl_sync(FULL, p3, 0, 16);
  }
  if (!valid || i != 0) return;
  if (special) {
    exact_block_global<DT>(a, tc.alpha_d, blk, kb4, flags);
    return;
  }
  BlockOut o;
  if constexpr (MODE == ADAPTIVE) {
    const bool k4 = S[1] < S[0];  // strict: ties keep 6
    o.codes = k4 ? word[1] : word[0];
    o.sc = k4 ? sc4 : sc6;
    o.pick4 = k4;
  } else {
    o.codes = word[0];
    o.sc = sc6;
    o.pick4 = (MODE == FIXED4);
  }
  *reinterpret_cast<uint64_t*>(a.codes + (int64_t)blk * 8) = o.codes;
  a.scales_tc[sf_tc_offset(row, kbg, kb4)] = (uint8_t)o.sc;
  if (a.scales_rm) a.scales_rm[blk] = (uint8_t)o.sc;
  if (a.pick4) a.pick4[blk] = (uint8_t)o.pick4;
}

// Resolve a warp's deferred-block list, two blocks per step (resolve_pair).
template <int DT, int MODE>
__device__ F46_RL_INLINE void resolve_list(const ExactArgs ea, const TensorConsts tc, uint32_t kb4,
                                          uint32_t* flags, const uint32_t* dl, uint32_t n) {
#pragma unroll 1
  for (uint32_t i = 0; i < n; i += 2)
    resolve_pair<DT, MODE>(ea, tc, kb4, flags, dl[i], dl[i + 1 < n ? i + 1 : i], i + 1 < n);
}

constexpr int kBPL = kSegElems / 512;   // blocks per lane per segment
constexpr int kDefer = 2 * kSegElems / 16;  // deferred-block slots per warp (a segment defers <= half)

// The streaming loop of one warp, specialised on the tensor-wide tie direction.
template <int DT, int MODE, bool EXTRA, int TDIR, bool TIE = false>
__device__ __forceinline__ void seg_stream(const QParams& p, const TensorConsts& tc, uint32_t wsm,
                                           uint64_t* wb, uint32_t* dl, uint32_t t_begin,
                                           uint32_t t_end, uint32_t tab) {
  constexpr int kEsz = (DT == DT_BF16) ? 2 : 4;
  constexpr int kTileBytes = kSegElems * kEsz;
  constexpr uint32_t kSegBlocks = kSegElems / 16;
  const int lane = threadIdx.x & 31;
  const uint32_t cols = (uint32_t)p.cols;
  const uint32_t nb = cols >> 4;
  const uint32_t kb4 = (nb + 3) >> 2;
  const uint32_t n_seg = (cols + kSegElems - 1) / kSegElems;

  // Each warp streams one contiguous range of tiles (tile = one segment of one
  // row): successive tiles are adjacent in memory, so cursors only step.
  // The tiles tile the flat input contiguously, so the issue cursor is one
  // pointer that advances by the tile's size (lane 0 only).
  const uint32_t last_n = cols - (n_seg - 1) * kSegElems;  // elements in a row's last segment
  // (Byte offsets are 32-bit: the host launches at most 2^31 input bytes at a time.)
  const uint8_t* xb = reinterpret_cast<const uint8_t*>(p.x);
  uint32_t iseg, tnext = t_begin, src;
  {
    const uint32_t irow = t_begin / n_seg;
    iseg = t_begin - irow * n_seg;
    src = (irow * cols + iseg * kSegElems) * kEsz;
  }
  auto issue = [&](int s) {
    const uint32_t n = (iseg == n_seg - 1) ? last_n : (uint32_t)kSegElems;
    if (tnext < t_end) {
      mbar_expect_tx(&wb[s], n * kEsz);
      bulk_load(wsm + s * kTileBytes, xb + src, n * kEsz, &wb[s]);
    }
    src += n * kEsz;
    ++tnext;
    if (++iseg == n_seg) iseg = 0;
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) issue(s);
  }
  uint32_t row = t_begin / n_seg, seg = t_begin - row * n_seg;  // tile being consumed
  // Per-lane output cursors, stepped per tile: lane l owns blocks kb0 + l + 32j,
  // whose codes sit 256 B apart (the codes of consecutive tiles are contiguous)
  // and whose tcgen05-layout scales sit 8 atoms (4 KB) apart; a tile advances
  // the scale cursor by kSegBlocks/4 atoms within a row and is recomputed at a
  // row change.
  auto sf_cursor = [&](uint32_t r, uint32_t kb0) -> uint32_t {
    return ((r >> 7) * kb4 + (kb0 >> 2) + (lane >> 2)) * 512 + (r & 31) * 16 +
           ((r & 127) >> 5) * 4 + (lane & 3);
  };
  uint32_t coff = (row * nb + seg * kSegBlocks + lane) * 8;
  uint32_t soff = sf_cursor(row, seg * kSegBlocks);

  uint32_t t = t_begin;
  int s = 0;
  uint32_t parity = 0;
  uint32_t ndefer = 0;  // warp-uniform
  while (true) {
    // ---- hot loop: stream segments until done or the defer list is half full ----
    for (; t < t_end && ndefer <= kDefer - kSegBlocks; ++t) {
      mbar_wait(&wb[s], parity);
      const uint32_t kb0 = seg * kSegBlocks;                // a multiple of 4
      const uint32_t nbs = min(kSegBlocks, nb - kb0);       // blocks in this segment
      const uint64_t rbk = (uint64_t)row * nb + kb0;        // first block of the segment
      const uint32_t blk0 = wsm + s * kTileBytes + lane * (16 * kEsz);
      uint32_t fails = 0;
      auto one = [&](int j) {
        const uint32_t blk_addr = blk0 + j * (32 * 16 * kEsz);
        float2 x[8];
        float bmax;
        load_block<DT>(blk_addr, x, bmax);
        BlockOut o;
#if F46_UNCOND_STORE
        // straight line: store unconditionally; a deferred block's bytes are
        // rewritten by the resolve pass (ordered after this by __syncwarp)
        bool ok;
        if constexpr (F46_V3 && MODE == ADAPTIVE && TDIR != 2)
          ok = block46<TDIR, TIE>(x, bmax, tc, tab, o);
        else
          ok = block_sl<MODE, TDIR>(x, bmax, tc, SegLoad<DT>{blk_addr}, o);
        *reinterpret_cast<uint64_t*>(p.codes + coff + j * 256) = o.codes;
        p.scales_tc[soff + j * 4096] = (uint8_t)o.sc;
        if constexpr (EXTRA) {
          if (p.scales_rm) p.scales_rm[rbk + lane + 32 * j] = (uint8_t)o.sc;
          if (p.pick4) p.pick4[rbk + lane + 32 * j] = (uint8_t)o.pick4;
        }
        fails |= (ok ? 0u : 1u) << j;
#else
        if (block_sl<MODE, TDIR>(x, bmax, tc, SegLoad<DT>{blk_addr}, o)) {
          *reinterpret_cast<uint64_t*>(p.codes + coff + j * 256) = o.codes;
          p.scales_tc[soff + j * 4096] = (uint8_t)o.sc;
          if constexpr (EXTRA) {
            if (p.scales_rm) p.scales_rm[rbk + lane + 32 * j] = (uint8_t)o.sc;
            if (p.pick4) p.pick4[rbk + lane + 32 * j] = (uint8_t)o.pick4;
          }
        } else {
          fails |= 1u << j;
        }
#endif
      };
      if (nbs == kSegBlocks) {
#pragma unroll kKbUnroll
        for (int j = 0; j < kBPL; ++j) one(j);
      } else {
        for (int j = 0; j < kBPL; ++j)
          if (lane + 32 * j < nbs) one(j);
      }
      if (__builtin_expect(__any_sync(0xFFFFFFFFu, fails != 0), 0)) {
#pragma unroll
        for (int j = 0; j < kBPL; ++j) {
          const bool f = (fails >> j) & 1u;
          const uint32_t m = __ballot_sync(0xFFFFFFFFu, f);
          if (f) dl[ndefer + __popc(m & ((1u << lane) - 1))] = (uint32_t)(rbk + lane + 32 * j);
          ndefer += __popc(m);
        }
      }
      __syncwarp();
      if (lane == 0) issue(s);
      if (++s == kStages) {
        s = 0;
        parity ^= 1u;
      }
      coff += nbs * 8;
      if (++seg == n_seg) {
        seg = 0;
        ++row;
        soff = sf_cursor(row, 0);
      } else {
        soff += (kSegBlocks / 4) * 512;
      }
    }
    // ---- deferred blocks: exact float64 path (outside the hot loop) ----
    __syncwarp();
    if (ndefer) {
      const ExactArgs ea{p.x, p.codes, p.scales_tc, p.scales_rm, p.pick4, p.cols, MODE, p.rule};
      for (uint32_t i = lane; i < ndefer; i += 32) resolve_block_global<DT, MODE>(ea, tc, dl[i], kb4, p.d_flags);
    }
    __syncwarp();
    ndefer = 0;
    if (t >= t_end) break;
  }
}

// The streaming loop for whole segments (cols % kSegElems == 0, no parity
// views): tile t is bytes [t, t+1) * kTileBytes of the input, its blocks are
// t*kSegBlocks + [0, kSegBlocks), so every cursor is a multiple of t.  All
// per-tile bookkeeping is warp-uniform (the warp index comes through a shuffle,
// so the compiler keeps it in uniform registers and the bulk copy needs no
// per-lane election loop).
//
// FLAT (any cols % 16 == 0): the blocks of the tensor are one contiguous
// sequence (blocks never straddle rows), so tile t is blocks [128t, 128t+128)
// of it whatever the row length -- no partial per-row segments -- and each
// block's (row, kb) for the scale layout comes from a multiply-high division.
template <int DT, int MODE, int TDIR, bool TIE = false, bool FLAT = false, bool SMALL = false>
__device__ __forceinline__ uint32_t stream_full(const QParams& p, const TensorConsts& tc, uint32_t wsm,
                                                uint64_t* wb, uint32_t* dl, uint32_t t_begin,
                                                uint32_t t_end, uint32_t n_seg, uint32_t tab) {
  constexpr int kEsz = (DT == DT_BF16) ? 2 : 4;
  constexpr uint32_t kTileBytes = kSegElems * kEsz;
  constexpr uint32_t kSegBlocks = kSegElems / 16;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nb = (uint32_t)p.cols >> 4;
  const uint32_t kb4 = (nb + 3) >> 2;
  const uint8_t* xb = reinterpret_cast<const uint8_t*>(p.x);
  const uint32_t nblk = (uint32_t)p.rows * nb;
  auto tile_bytes = [&](uint32_t tt) -> uint32_t {  // the last flat tile may be short
    if constexpr (FLAT) return min(kSegBlocks, nblk - tt * kSegBlocks) * (16 * kEsz);
    return kTileBytes;
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s)
      if (t_begin + s < t_end) {
        const uint32_t nbytes = tile_bytes(t_begin + s);
        mbar_expect_tx(&wb[s], nbytes);
        bulk_load(wsm + s * kTileBytes, xb + (size_t)(t_begin + s) * kTileBytes, nbytes, &wb[s]);
      }
  }
  uint32_t row = FLAT ? 0 : t_begin / n_seg, seg = FLAT ? 0 : t_begin - row * n_seg;
  auto sf_row = [&](uint32_t r) -> uint32_t {  // lane's scale byte for block 0 of row r
    return ((r >> 7) * kb4 + (lane >> 2)) * 512 + (r & 31) * 16 + ((r & 127) >> 5) * 4 + (lane & 3);
  };
  uint32_t srow = sf_row(row);
  uint8_t* cptr = p.codes + (size_t)t_begin * (kSegBlocks * 8) + lane * 8;
  const ExactArgs ea{p.x, p.codes, p.scales_tc, nullptr, nullptr, p.cols, MODE, p.rule};
  uint32_t parity = 0, ndefer = 0;
  uint32_t t = t_begin;
  // one tile from stage S (a compile-time constant: barrier and buffer
  // addresses fold); returns false when the warp's range is done
  auto step = [&](auto S_) -> bool {
#if F46_STEP2
    constexpr int S = decltype(S_)::value;
#else
    const int S = S_;
#endif
    if (t >= t_end) return false;
    mbar_wait(&wb[S], parity);
    const uint32_t blk0 = wsm + S * kTileBytes + lane * (16 * kEsz);
    const uint32_t soff = srow + seg * (kSegBlocks / 4) * 512;
    uint32_t fails = 0;
#pragma unroll (SMALL ? kSfUnrollSmall : kSfUnroll)
    for (int j = 0; j < kBPL; ++j) {
      const uint32_t blk_addr = blk0 + j * (32 * 16 * kEsz);
      float2 x[8];
      float bmax;
      load_block<DT>(blk_addr, x, bmax);
      BlockOut o;
      bool ok;
      if constexpr (F46_V3 && MODE == ADAPTIVE && TDIR != 2)
        ok = block46<TDIR, TIE>(x, bmax, tc, tab, o);
      else
        ok = block_sl<MODE, TDIR>(x, bmax, tc, SegLoad<DT>{blk_addr}, o);
      if constexpr (FLAT) {
        const uint32_t b = t * kSegBlocks + lane + 32 * j;
        const uint32_t hi = __umulhi(b, p.nb_magic);
        const uint32_t r = (hi + ((b - hi) >> p.nb_sh1)) >> p.nb_sh2, kb = b - r * nb;
        if (b < nblk) {
          *reinterpret_cast<uint64_t*>(cptr + j * 256) = o.codes;
          p.scales_tc[((r >> 7) * kb4 + (kb >> 2)) * 512 + (r & 31) * 16 + ((r & 127) >> 5) * 4 + (kb & 3)] =
              (uint8_t)o.sc;
          fails |= (ok ? 0u : 1u) << j;
        }
      } else {
        *reinterpret_cast<uint64_t*>(cptr + j * 256) = o.codes;
        p.scales_tc[soff + j * 4096] = (uint8_t)o.sc;
        fails |= (ok ? 0u : 1u) << j;
      }
    }
    if (F46_NO_DEFER_PROBE) fails = 0;  // timing probe only (wrong results)
    if (__builtin_expect(__any_sync(0xFFFFFFFFu, fails != 0), 0)) {
      const uint32_t rbk = t * kSegBlocks;
#pragma unroll
      for (int j = 0; j < kBPL; ++j) {
        const bool f = (fails >> j) & 1u;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, f);
        if (f) dl[ndefer + __popc(m & ((1u << lane) - 1))] = rbk + lane + 32 * j;
        ndefer += __popc(m);
      }
      // deferred blocks: exact path, once the list is half full
      if (ndefer > kDefer - kSegBlocks) {
        __syncwarp();
        for (uint32_t i = lane; i < ndefer; i += 32) resolve_block_global<DT, MODE>(ea, tc, dl[i], kb4, p.d_flags);
        ndefer = 0;
      }
    }
    __syncwarp();
    if (lane == 0 && t + kStages < t_end) {
      const uint32_t nbytes = tile_bytes(t + kStages);
      mbar_expect_tx(&wb[S], nbytes);
      bulk_load(wsm + S * kTileBytes, xb + (size_t)(t + kStages) * kTileBytes, nbytes, &wb[S]);
    }
    ++t;
    cptr += kSegBlocks * 8;
    if (!FLAT && ++seg == n_seg) {
      seg = 0;
      ++row;
      srow = sf_row(row);
    }
    return true;
  };
  static_assert(kStages == 2, "stream_full unrolls two stages");
#if F46_STEP2
  while (step(std::integral_constant<int, 0>{}) && step(std::integral_constant<int, 1>{})) parity ^= 1u;
#else
  // one loop body: the stage index is a runtime value
  for (int s = 0; step(s); s ^= 1) parity ^= (uint32_t)s;
#endif
  return ndefer;  // the caller resolves the rest of dl[] (one call site per kernel)
}

template <int DT, int MODE, bool EXTRA, bool PAR = false>
__global__ void __launch_bounds__(kWarps * 32, F46_MINB) quant_seg_kernel(QParams p) {
  constexpr int kEsz = (DT == DT_BF16) ? 2 : 4;
  constexpr int kTileBytes = kSegElems * kEsz;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kWarps][kStages];
  __shared__ uint32_t defer[kWarps][kDefer];

  select_group(p);
  // warp index through a shuffle: the compiler then knows it is warp-uniform
  const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t cols = (uint32_t)p.cols;
  const uint32_t nb = cols >> 4;
  const uint32_t kb4 = (nb + 3) >> 2;
  const uint32_t n_seg = (cols + kSegElems - 1) / kSegElems;
  const bool full = !EXTRA && (cols % kSegElems) == 0;
  const bool flat = !EXTRA && !full && F46_FLAT;
  const uint32_t total = flat ? ((uint32_t)p.rows * nb + kSegElems / 16 - 1) / (kSegElems / 16)
                              : (uint32_t)p.rows * n_seg;
  const uint32_t gw = blockIdx.x * kWarps + warp, G = gridDim.x * kWarps;

  if (!EXTRA && p.d_sync) {
    // fused K1: max|x| over exactly the tiles this warp quantizes below (so
    // they are in L2 for the second pass), one 64-bit atomicMax per warp on the
    // float64 bit pattern as amax_kernel, then a grid-wide barrier (the launch
    // is cooperative: every CTA is resident)
    const uint32_t per0 = total / G, rem0 = total - per0 * G;
    const uint32_t tb = gw * per0 + min(gw, rem0), te = tb + per0 + (gw < rem0 ? 1u : 0u);
    const uint64_t nbytes = (uint64_t)p.rows * p.cols * kEsz;
    const uint64_t b0 = (uint64_t)tb * kTileBytes, b1 = min((uint64_t)te * kTileBytes, nbytes);
    const uint4* xv = reinterpret_cast<const uint4*>(p.x);
    uint32_t m = 0;
    auto fold = [&](const uint4 v) {
      if constexpr (DT == DT_BF16) {
        m = __vmaxu2(m, v.x & 0x7FFF7FFFu);
        m = __vmaxu2(m, v.y & 0x7FFF7FFFu);
        m = __vmaxu2(m, v.z & 0x7FFF7FFFu);
        m = __vmaxu2(m, v.w & 0x7FFF7FFFu);
      } else {
        m = max(m, max(max(v.x & 0x7FFFFFFFu, v.y & 0x7FFFFFFFu), max(v.z & 0x7FFFFFFFu, v.w & 0x7FFFFFFFu)));
      }
    };
    // eight 16-byte loads in flight per lane (4 KB per warp step)
    uint64_t off = b0 + lane * 16;
    for (; off + 7 * 512 < b1; off += 8 * 512) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = xv[(off + u * 512) >> 4];
#pragma unroll
      for (int u = 0; u < 8; ++u) fold(v[u]);
    }
    for (; off < b1; off += 512) fold(xv[off >> 4]);
    if constexpr (DT == DT_BF16) m = max(m & 0xFFFFu, m >> 16) << 16;
    uint64_t m64 = (uint64_t)__double_as_longlong((double)__uint_as_float(m));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t v = __shfl_xor_sync(0xFFFFFFFFu, m64, o);
      m64 = v > m64 ? v : m64;
    }
    if (lane == 0 && m64) atomicMax(reinterpret_cast<unsigned long long*>(const_cast<double*>(p.d_amax)),
                                    (unsigned long long)m64);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(p.d_sync, 1u);
      const uint32_t want = gridDim.x * gridDim.y;
      while (*reinterpret_cast<volatile uint32_t*>(p.d_sync) < want) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
  }

  const double alpha_d = resolve_alpha(p);
  prologue_flags(p, alpha_d);
  const bool overridden = p.alpha_override > 0.0;
  const TensorConsts tc = scale_dir_consts(make_consts(
      alpha_d, p.rule, DT,
      tie_direction(alpha_d, overridden ? 0.0 : __ldcg(p.d_amax), p.mcap, DT, overridden)));

  // per-tensor table of the per-scale-code reciprocals (block46)
  __shared__ __align__(16) float4 sctab[128];
  static_assert(kWarps * 32 >= 128, "one thread per scale code");
  if (threadIdx.x < 128) sctab[threadIdx.x] = scale_entry(threadIdx.x, tc.alpha);
  // TDIR 0, adaptive, BF16: per-code exact-tie reciprocals (safe_recip); if
  // every code has one the streaming loop runs as TDIR 3 (no upper-bound pass)
  float rsafe = 0.f;
  bool unsafe = false;
  // (codes 1..126: 0 underflows and 0x7F is NaN, neither is ever a stored scale)
  if (DT == DT_BF16 && MODE == ADAPTIVE && tc.tdir == 0 && !tc.force_exact && threadIdx.x < 127 &&
      threadIdx.x > 0)
    unsafe = !safe_recip(threadIdx.x, tc.alpha, rsafe);
  const bool t3 = DT == DT_BF16 && MODE == ADAPTIVE && tc.tdir == 0 && !tc.force_exact &&
                  !__syncthreads_or(unsafe) && F46_T3;
  if (t3 && threadIdx.x < 127 && threadIdx.x > 0) sctab[threadIdx.x].x = rsafe;
  // TDIR +1: the exact-code reciprocal is the upper bound (rh).  With this the
  // table's x field is, for TDIR -1, +1 and 3 alike, the reciprocal whose codes
  // are the reference's, and all three run one instantiation (TDIR 4): the
  // tensors of one grouped launch share a single hot loop (instruction cache)
  if (DT == DT_BF16 && MODE == ADAPTIVE && tc.tdir == 1 && threadIdx.x < 128)
    sctab[threadIdx.x].x = sctab[threadIdx.x].y;
  __syncthreads();
  const bool t4 = DT == DT_BF16 && MODE == ADAPTIVE && !tc.force_exact && F46_T4 &&
                  (t3 || tc.tdir == -1 || tc.tdir == 1);
  const uint32_t tab = smem_u32(sctab);
  const uint32_t wsm = smem_u32(smem) + warp * (kStages * kTileBytes);
  uint64_t* wb = bars[warp];
  uint32_t* dl = defer[warp];
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&wb[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  const uint32_t per = total / G, rem = total - per * G;
  const uint32_t t_begin = gw * per + min(gw, rem);
  const uint32_t t_end = t_begin + per + (gw < rem ? 1u : 0u);
  uint32_t nd = 0;  // deferred blocks stream_full left in dl[]
  if (tc.force_exact) {
    // alpha outside the fast path's range / rule != mse: every block exactly
    const ExactArgs ea{p.x, p.codes, p.scales_tc, p.scales_rm, p.pick4, p.cols, MODE, p.rule};
    const uint32_t nblk = (uint32_t)p.rows * nb;
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nblk; b += gridDim.x * blockDim.x)
      exact_block_global<DT>(ea, alpha_d, b, kb4, p.d_flags);
  } else if (flat) {
    if constexpr (DT == DT_BF16) {
      const bool tie = MODE == ADAPTIVE && e4m3_ties_possible(tc.alpha);
      switch (t4 ? 4 : (t3 ? 3 : tc.tdir)) {
        case 4:
          if constexpr (MODE == ADAPTIVE) {
            if (tie)
              nd = stream_full<DT, MODE, 4, true, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
            else
              nd = stream_full<DT, MODE, 4, false, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          }
          break;
        case -1:
          nd = stream_full<DT, MODE, -1, false, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          break;
        case 0:
          if (tie)
            nd = stream_full<DT, MODE, 0, true, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          else
            nd = stream_full<DT, MODE, 0, false, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          break;
        case 3:
          if constexpr (MODE == ADAPTIVE) {
            if (tie)
              nd = stream_full<DT, MODE, 3, true, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
            else
              nd = stream_full<DT, MODE, 3, false, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          }
          break;
        case 1:
          nd = stream_full<DT, MODE, 1, false, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          break;
        default:
          nd = stream_full<DT, MODE, 2, false, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
      }
    } else {
      nd = stream_full<DT, MODE, 2, false, true, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
    }
  } else if (full && F46_FULL) {
    if constexpr (DT == DT_BF16) {
      switch (t4 ? 4 : (t3 ? 3 : tc.tdir)) {
        case 4:
          if constexpr (MODE == ADAPTIVE) {
            if (e4m3_ties_possible(tc.alpha))
              nd = stream_full<DT, MODE, 4, true, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
            else
              nd = stream_full<DT, MODE, 4, false, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          }
          break;
        case -1:
          nd = stream_full<DT, MODE, -1, false, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          break;
        case 0:
          if (MODE == ADAPTIVE && e4m3_ties_possible(tc.alpha))
            nd = stream_full<DT, MODE, 0, true, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          else
            nd = stream_full<DT, MODE, 0, false, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          break;
        case 3:
          if constexpr (MODE == ADAPTIVE) {
            if (e4m3_ties_possible(tc.alpha))
              nd = stream_full<DT, MODE, 3, true, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
            else
              nd = stream_full<DT, MODE, 3, false, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          }
          break;
        case 1:
          nd = stream_full<DT, MODE, 1, false, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
          break;
        default:
          nd = stream_full<DT, MODE, 2, false, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
      }
    } else {
      nd = stream_full<DT, MODE, 2, false, false, PAR>(p, tc, wsm, wb, dl, t_begin, t_end, n_seg, tab);
    }
  } else if constexpr (DT == DT_BF16) {
    switch (t3 ? 3 : tc.tdir) {
      case -1:
        seg_stream<DT, MODE, EXTRA, -1>(p, tc, wsm, wb, dl, t_begin, t_end, tab);
        break;
      case 0:
        if (MODE == ADAPTIVE && e4m3_ties_possible(tc.alpha))
          seg_stream<DT, MODE, EXTRA, 0, true>(p, tc, wsm, wb, dl, t_begin, t_end, tab);
        else
          seg_stream<DT, MODE, EXTRA, 0>(p, tc, wsm, wb, dl, t_begin, t_end, tab);
        break;
      case 3:
        if constexpr (MODE == ADAPTIVE) {
          if (e4m3_ties_possible(tc.alpha))
            seg_stream<DT, MODE, EXTRA, 3, true>(p, tc, wsm, wb, dl, t_begin, t_end, tab);
          else
            seg_stream<DT, MODE, EXTRA, 3>(p, tc, wsm, wb, dl, t_begin, t_end, tab);
        }
        break;
      case 1:
        seg_stream<DT, MODE, EXTRA, 1>(p, tc, wsm, wb, dl, t_begin, t_end, tab);
        break;
      default:
        seg_stream<DT, MODE, EXTRA, 2>(p, tc, wsm, wb, dl, t_begin, t_end, tab);
    }
  } else {
    seg_stream<DT, MODE, EXTRA, 2>(p, tc, wsm, wb, dl, t_begin, t_end, tab);
  }
  __syncwarp();
  if (nd) {
    const ExactArgs ea{p.x, p.codes, p.scales_tc, nullptr, nullptr, p.cols, MODE, p.rule};
    if constexpr (PAR)
      resolve_list<DT, MODE>(ea, tc, kb4, p.d_flags, dl, nd);
    else
      for (uint32_t i = lane; i < nd; i += 32) resolve_block_global<DT, MODE>(ea, tc, dl[i], kb4, p.d_flags);
  }
  // tcgen05 layout padding: kb in [nb, 4*kb4) of every row, rows up to a multiple of 128
  const uint32_t rows = (uint32_t)p.rows, rows_pad = (rows + 127) & ~127u;
  const uint32_t kpad = 4 * kb4 - nb;
  const uint32_t n_a = rows * kpad, n_b = (rows_pad - rows) * 4 * kb4;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_a + n_b; i += gridDim.x * blockDim.x) {
    uint32_t r, kb;
    if (i < n_a) {
      r = i / kpad;
      kb = nb + (i - r * kpad);
    } else {
      r = rows + (i - n_a) / (4 * kb4);
      kb = (i - n_a) - (r - rows) * 4 * kb4;
    }
    p.scales_tc[sf_tc_offset(r, kb, kb4)] = 0;
  }
}

// ---------------------------------------------------------------------------
// K2 generic: any shape, any dtype (one thread per 16-block)
// ---------------------------------------------------------------------------
template <int DT>
struct GlobalLoad {
  const void* x;
  int64_t row, c0, cols;
  __device__ __forceinline__ float operator()(int i) const {
    const int64_t c = c0 + i;
    if (c >= cols) return 0.f;
    if constexpr (DT == DT_BF16)
      return __uint_as_float((uint32_t)(reinterpret_cast<const uint16_t*>(x)[row * cols + c]) << 16);
    else
      return reinterpret_cast<const float*>(x)[row * cols + c];
  }
};

template <int DT, int MODE>
__global__ void __launch_bounds__(256) quant_generic_kernel(QParams p) {
  select_group(p);
  const int64_t nb = (p.cols + 15) >> 4;
  const int64_t kb4 = (nb + 3) >> 2;
  const int64_t rows_pad = (p.rows + 127) & ~(int64_t)127;
  const int64_t total = rows_pad * kb4 * 4;
  const double alpha_d = resolve_alpha(p);
  prologue_flags(p, alpha_d);
  const TensorConsts tc = make_consts(alpha_d, p.rule, DT);
  bool nonfinite = false;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / (kb4 * 4), kb = idx - row * (kb4 * 4);
    if (row >= p.rows || kb >= nb) {  // tcgen05 layout padding
      p.scales_tc[sf_tc_offset(row, kb, kb4)] = 0;
      continue;
    }
    const int64_t c0 = kb * 16;
    BlockOut o;
    if constexpr (DT == DT_F64) {
      double xd[16];
      const double* xr = reinterpret_cast<const double*>(p.x) + row * p.cols;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        xd[i] = (c0 + i < p.cols) ? xr[c0 + i] : 0.0;
        nonfinite |= !(fabs(xd[i]) <= 1.7976931348623157e308);
      }
      exact_block(xd, alpha_d, MODE, p.rule, &o);
    } else {
      const GlobalLoad<DT> ld{p.x, row, c0, p.cols};
      float2 x[8];
      uint32_t m = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        x[q] = make_float2(ld(2 * q), ld(2 * q + 1));
        m = max(m, __float_as_uint(x[q].x) & 0x7FFFFFFFu);
        m = max(m, __float_as_uint(x[q].y) & 0x7FFFFFFFu);
      }
      nonfinite |= (m >= 0x7F800000u);
      const float bmax = __uint_as_float(m);
      bool ok = false;
      if (!tc.force_exact) ok = fast_block<MODE>(x, bmax, tc, ld, o);
      if (!ok) {
        double xd[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) xd[i] = (double)ld(i);
        exact_block(xd, alpha_d, MODE, p.rule, &o);
      }
    }
    // zero the codes of tail pad positions (x = 0 there, so only -0.0 could leak)
    uint64_t codes = o.codes;
    if (c0 + 16 > p.cols) {
      const int valid = (int)(p.cols - c0);
      codes &= (valid >= 16) ? ~0ull : ((1ull << (4 * valid)) - 1);
    }
    *reinterpret_cast<uint64_t*>(p.codes + (row * nb + kb) * 8) = codes;
    p.scales_tc[sf_tc_offset(row, kb, kb4)] = (uint8_t)o.sc;
    if (p.scales_rm) p.scales_rm[row * nb + kb] = (uint8_t)o.sc;
    if (p.pick4) p.pick4[row * nb + kb] = (uint8_t)o.pick4;
  }
  if (nonfinite && p.d_flags) atomicOr(p.d_flags, F46_FLAG_NONFINITE);
}

// ---------------------------------------------------------------------------
// 2-D 16x16-tile quantization (transforms.py:108-179 _tile_pass /
// quantize_weights_2d): one E4M3 scale per 16x16 tile chosen over all 256
// values, so the same codes and scales quantize W along its rows and W^T
// along its rows -- FPROP (x W^T) and DGRAD (dy W) both get a K-major operand
// from one pass.  One warp per tile, lane l owns tile row l/2, columns
// 8(l%2)..+7.  The arithmetic is the reference's float64 restatement
// (exact_pass' operations), and the 256-term error sums follow numpy's
// pairwise order for the (16,16) axis pair: P(e[0:128]) + P(e[128:256]),
// P with 8 accumulators r_j = e_j + e_{j+8} + e_{j+16} + ... in sequence
// (checked against the reference: tests/golden/golden_tile2d.npz).  Weights
// are quantized once per update, so exactness is bought with f64 here.
// ---------------------------------------------------------------------------
struct Q2Params {
  const void* w;
  int64_t R, C;
  int mode, rule, dtype;
  double mcap;
  const double* d_amax;
  double alpha_override;
  uint8_t* codes;      // [R][nbC*8]
  uint8_t* scales_tc;  // tcgen05 layout of [R, C]
  uint8_t* scales_rm;  // [R][nbC] (nullable)
  uint8_t* pick4;      // [R][nbC] (nullable)
  uint8_t* codes_t;    // W^T: [C][nbR*8] (nullable)
  uint8_t* scales_tc_t;  // tcgen05 layout of [C, R] (nullable)
  double* d_alpha_out;
  uint32_t* d_flags;
  int64_t g_w, g_codes, g_scales, g_codes_t, g_scales_t;  // grouped launches (bytes)
};

__device__ __forceinline__ void select_group2(Q2Params& p) {
  if (gridDim.y > 1) {
    const int64_t g = blockIdx.y;
    p.w = reinterpret_cast<const uint8_t*>(p.w) + g * p.g_w;
    p.codes += g * p.g_codes;
    p.scales_tc += g * p.g_scales;
    if (p.codes_t) p.codes_t += g * p.g_codes_t;
    if (p.scales_tc_t) p.scales_tc_t += g * p.g_scales_t;
    if (p.d_amax) p.d_amax += g;
    if (p.d_alpha_out) p.d_alpha_out += g;
  }
}

__device__ __forceinline__ double q2_load(const Q2Params& p, int64_t r, int64_t c) {
  if (r >= p.R || c >= p.C) return 0.0;
  const int64_t i = r * p.C + c;
  if (p.dtype == DT_BF16)
    return (double)__uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(p.w)[i] << 16);
  if (p.dtype == DT_F32) return (double)reinterpret_cast<const float*>(p.w)[i];
  return reinterpret_cast<const double*>(p.w)[i];
}

// numpy pairwise sum of the 256 tile errors; e[] in shared memory, row-major tile order
__device__ __forceinline__ double pw_tile(const double* e) {
  double tot = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = e[128 * h + j];
    for (int i = 8; i < 128; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], e[128 * h + i + j]);
    const double part = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                  __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    tot = h == 0 ? part : __dadd_rn(tot, part);
  }
  return tot;
}

// The same 256-term pairwise sum with 16 lanes: lane 8h + j accumulates
// r_j of half h (16 sequential adds), then the fixed tree
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and part0 + part1 through shuffles --
// the identical association as pw_tile.  Every lane returns the total.
__device__ __forceinline__ double pw_tile_par(const double* e, int lane) {
  const int h = (lane >> 3) & 1, j = lane & 7;
  double r = e[128 * h + j];
#pragma unroll
  for (int i = 8; i < 128; i += 8) r = __dadd_rn(r, e[128 * h + i + j]);
  double t = __shfl_down_sync(0xFFFFFFFFu, r, 1);
  const double a = __dadd_rn(r, t);  // meaningful in even j
  t = __shfl_down_sync(0xFFFFFFFFu, a, 2);
  const double b = __dadd_rn(a, t);  // meaningful in j % 4 == 0
  t = __shfl_down_sync(0xFFFFFFFFu, b, 4);
  const double c = __dadd_rn(b, t);  // part(h) in lane 8h
  const double tot = __dadd_rn(c, __shfl_down_sync(0xFFFFFFFFu, c, 8));
  return __shfl_sync(0xFFFFFFFFu, tot, 0);
}

// Exact FP4 codes of a lane's 8 tile values (float) under scale delta, from
// the same proven bracket logic as the 1-D quantizer (f46_device.cuh):
// tdir -1 / +1 pick one bound, 0 the split reciprocal, 2 resolves each
// flagged nibble with the exact test through `load`.
template <class Load>
__device__ __forceinline__ uint32_t tile_codes8(const float (&xf)[8], float alpha, float delta,
                                                int tdir, const Load& load) {
  const float D = alpha * delta;
  const float rq = rcp_approx(D) * F46_QLO;
  float2 q[4];
  if (tdir == 0) {
    const float R = rcp_approx(D);
    const float Rhi = __uint_as_float(__float_as_uint(R) & 0xFFFFFF00u);
    const float Rlo = fmaf(-D, Rhi, 1.0f) * R;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      q[i] = make_float2(fmaf(xf[2 * i], Rlo, xf[2 * i] * Rhi), fmaf(xf[2 * i + 1], Rlo, xf[2 * i + 1] * Rhi));
    return cvt_e2m1x8(q[0], q[1], q[2], q[3]);
  }
  const float r = tdir == 1 ? rq * F46_QHI_OVER_QLO : rq;
#pragma unroll
  for (int i = 0; i < 4; ++i) q[i] = make_float2(xf[2 * i] * r, xf[2 * i + 1] * r);
  uint32_t w = cvt_e2m1x8(q[0], q[1], q[2], q[3]);
  if (tdir == 2) {
    const float rh = rq * F46_QHI_OVER_QLO;
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = make_float2(xf[2 * i] * rh, xf[2 * i + 1] * rh);
    const uint32_t hi = cvt_e2m1x8(q[0], q[1], q[2], q[3]);
    if (__builtin_expect((w ^ hi) != 0, 0)) w = fix_word(w, w ^ hi, 0, alpha, delta, load);
  }
  return w;
}

#ifndef F46_Q2_MINB
#define F46_Q2_MINB 4
#endif
__global__ void __launch_bounds__(256, F46_Q2_MINB) quant2d_kernel(Q2Params p) {
  select_group2(p);
  __shared__ double esq[8][256];   // the rule's per-element errors of one candidate
  __shared__ double dtab[8][16];    // dequantized value of each code under the candidate
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t TR = (p.R + 15) >> 4, TC = (p.C + 15) >> 4;
  const int64_t ntiles = TR * TC;
  double alpha = p.alpha_override;
  if (!(alpha > 0.0)) {
    const double amax = *p.d_amax;
    alpha = amax == 0.0 ? 1.0 : (double)((float)amax / (float)p.mcap);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.d_alpha_out) *p.d_alpha_out = alpha;
    if (p.alpha_override <= 0.0 && p.d_flags && !(*p.d_amax <= 1.7976931348623157e308))
      atomicOr(p.d_flags, F46_FLAG_NONFINITE);
  }
  const int64_t nbC = (p.C + 15) >> 4, nbR = (p.R + 15) >> 4;
  const int64_t kb4 = (nbC + 3) >> 2, kb4t = (nbR + 3) >> 2;
  const int tr_local = lane >> 1, tc_half = lane & 1;  // tile row, 8-column half
  // Fast path (codes and scales from f32 brackets, proven exact; errors still
  // float64): BF16/F32 input with a float32 alpha in range.  The rule only
  // changes which float64 error sum decides, so it does not force the slow path.
  const bool overridden = p.alpha_override > 0.0;
  const TensorConsts tcs = make_consts(
      alpha, RULE_MSE, p.dtype,
      tie_direction(alpha, overridden ? 0.0 : *p.d_amax, p.mcap, p.dtype, overridden));
  double* es = esq[warp];
  double* ea = esq[warp];  // l1 and mse never both needed
  double* dt = dtab[warp];
  for (int64_t tile = (int64_t)blockIdx.x * 8 + warp; tile < ntiles; tile += (int64_t)gridDim.x * 8) {
    const int64_t tr = tile / TC, tc = tile - tr * TC;
    const int64_t r = tr * 16 + tr_local, c0 = tc * 16 + 8 * tc_half;
    double x[8];
    double tmax = 0.0;
    bool nf = false;
    if (p.dtype == DT_F64) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        x[i] = q2_load(p, r, c0 + i);
        nf |= !(fabs(x[i]) <= 1.7976931348623157e308);
        tmax = fmax(tmax, fabs(x[i]));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tmax = fmax(tmax, __shfl_xor_sync(0xFFFFFFFFu, tmax, o));
      nf = __any_sync(0xFFFFFFFFu, nf);
    } else {
      uint32_t mb = 0;  // |x| bit patterns order like the values (NaN above inf)
      const int64_t e0 = r * p.C + c0;
      if (p.dtype == DT_BF16 && r < p.R && c0 + 8 <= p.C && (e0 & 7) == 0 &&
          (((uintptr_t)p.w) & 15) == 0) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p.w) + e0));
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          x[2 * i] = (double)__uint_as_float(wv[i] << 16);
          x[2 * i + 1] = (double)__uint_as_float(wv[i] & 0xFFFF0000u);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = q2_load(p, r, c0 + i);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) mb = max(mb, __float_as_uint((float)x[i]) & 0x7FFFFFFFu);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mb = max(mb, __shfl_xor_sync(0xFFFFFFFFu, mb, o));
      nf = mb >= 0x7F800000u;
      tmax = (double)__uint_as_float(mb);
    }
    if (nf && p.d_flags && lane == 0) atomicOr(p.d_flags, F46_FLAG_NONFINITE);
    uint32_t sc[2];
    uint32_t cw[2];  // 8 nibbles per candidate
    double err[2];
    const int ncand = p.mode == ADAPTIVE ? 2 : 1;
    // fast-path scale codes (bmax = tile max, exact tie test); warp-uniform
    const float tmaxf = (float)tmax;  // exact: BF16/F32 input
    bool fast = p.dtype != DT_F64 && !tcs.force_exact &&
                (__float_as_uint(tmaxf) - 0x2B800000u) < 0x28000000u;
    uint32_t fsc[2] = {0, 0};
    if (fast) {
      for (int k = 0; k < ncand; ++k) {
        const bool m4 = (p.mode == FIXED4 || k == 1);
        fsc[k] = block_scale_code(tmaxf, tcs.alpha, m4 ? 4.f : 6.f, m4 ? tcs.r4_lo : tcs.r6_lo,
                                  m4 ? tcs.r4_hi : tcs.r6_hi);
        fast &= fsc[k] != 0u;  // an underflowed scale takes the float64 path
      }
    }
    float xf[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) xf[i] = (float)x[i];
    const auto gload = [&](int i) -> float { return (float)q2_load(p, r, c0 + i); };
    for (int k = 0; k < ncand; ++k) {
      const double m = (p.mode == FIXED4 || k == 1) ? 4.0 : 6.0;
      uint32_t s;
      uint32_t w = 0;
      if (fast) {
        s = fsc[k];
        w = tile_codes8(xf, tcs.alpha, e4m3_to_f32(s), tcs.tdir, gload);
      } else {
        s = enc_e4m3_d(__ddiv_rn(tmax, __dmul_rn(alpha, m)));
        if (tmax == 0.0) s = 1;
      }
      const double denom = __dmul_rn(alpha, dec_e4m3_d(s));
      // deq(code) = dec_fp4(code) * denom for the 16 codes (exact products)
      __syncwarp();
      if (lane < 16) dt[lane] = __dmul_rn(dec_fp4_d((uint32_t)lane), denom);
      __syncwarp();
      double mx = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t code;
        if (fast) {
          code = (w >> (4 * i)) & 0xFu;
        } else {
          const double q = denom > 0.0 ? __ddiv_rn(x[i], denom)
                                       : ((x[i] != 0.0) ? copysign(6.0, x[i]) : 0.0);
          code = enc_fp4_d(q);
          w |= code << (4 * i);
        }
        const double diff = __dsub_rn(dt[code], x[i]);
        if (p.rule == RULE_MSE)
          es[tr_local * 16 + 8 * tc_half + i] = __dmul_rn(diff, diff);
        else if (p.rule == RULE_L1)
          ea[tr_local * 16 + 8 * tc_half + i] = fabs(diff);
        else
          mx = fmax(mx, fabs(diff));
      }
      __syncwarp();
      double e;
      if (p.rule == RULE_ABSMAX) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        e = mx;
      } else {
        e = pw_tile_par(p.rule == RULE_MSE ? es : ea, lane);
      }
      __syncwarp();
      sc[k] = s;
      cw[k] = w;
      err[k] = e;
    }
    const bool k4 = (p.mode == ADAPTIVE) ? (err[1] < err[0]) : (p.mode == FIXED4);
    const int ki = (p.mode == ADAPTIVE && k4) ? 1 : 0;
    uint32_t w = cw[ki];
    const uint32_t s = sc[ki];
    // zero the codes of pad columns (x = 0 there; only -0.0 could leak a sign)
    if (c0 + 8 > p.C) {
      const int valid = (int)max((int64_t)0, p.C - c0);
      w &= valid >= 8 ? 0xFFFFFFFFu : ((1u << (4 * valid)) - 1u);
    }
    if (r < p.R) {
      reinterpret_cast<uint32_t*>(p.codes + r * nbC * 8)[2 * tc + tc_half] = w;
      if (tc_half == 0) {
        p.scales_tc[sf_tc_offset32((uint32_t)r, (uint32_t)tc, (uint32_t)kb4)] = (uint8_t)s;
        if (p.scales_rm) p.scales_rm[r * nbC + tc] = (uint8_t)s;
        if (p.pick4) p.pick4[r * nbC + tc] = (uint8_t)k4;
      }
    }
    if (p.codes_t) {
      // W^T: lane L builds W^T row tc*16 + L/2, word L%2 = tile rows
      // 8(L%2)..+7 at tile column L/2.  Tile row i's codes of that column sit
      // in lane 2i + (L/2 >= 8), nibble (L/2) % 8.
      const int cc = lane >> 1, hw = lane & 1;
      uint32_t wt = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t wv = __shfl_sync(0xFFFFFFFFu, w, 2 * (8 * hw + i) + (cc >> 3));
        wt |= ((wv >> (4 * (cc & 7))) & 0xFu) << (4 * i);
      }
      const int64_t rt = tc * 16 + cc;        // W^T row
      const int64_t ct0 = tr * 16 + 8 * hw;   // its first column in this word
      if (rt < p.C && ct0 < p.R) {
        if (ct0 + 8 > p.R) wt &= (1u << (4 * (int)(p.R - ct0))) - 1u;  // pad rows of W
        reinterpret_cast<uint32_t*>(p.codes_t + rt * nbR * 8)[2 * tr + hw] = wt;
      } else if (rt < p.C) {
        reinterpret_cast<uint32_t*>(p.codes_t + rt * nbR * 8)[2 * tr + hw] = 0u;
      }
      if (p.scales_tc_t && lane < 16 && tc * 16 + lane < p.C)
        p.scales_tc_t[sf_tc_offset(tc * 16 + lane, tr, kb4t)] = (uint8_t)s;
    }
  }
}

// 2-D tiles, version 2: two tiles per warp, 16 lanes per tile.  Lane (h, j)
// (h = row half, j = 0..7) owns tile columns j and 8+j of rows 8h..8h+7, which
// are exactly the 16 terms of the reference's pairwise accumulator r_j of half
// h (p = 16*row + col, r_j = e[128h + j] + e[128h + 8 + j] + e[128h + 16 + j]
// + ..., transforms.py:125-130): each lane sums its errors in registers in
// that order, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and part0 + part1 go
// through shuffles -- no shared memory.  Its two columns are also two W^T
// words directly; the row-major W words are gathered with shuffles.  Codes and
// scales come from the f32 bracket logic (exact, as in K2), errors in float64.
// Tiles the fast path cannot take (all-zero excepted) use quant2d_tile_exact.
__device__ __noinline__ void quant2d_tile_exact(const Q2Params p, double alpha, int64_t tr, int64_t tc) {
  const int64_t nbC = (p.C + 15) >> 4, nbR = (p.R + 15) >> 4;
  const int64_t kb4 = (nbC + 3) >> 2, kb4t = (nbR + 3) >> 2;
  double x[256];
  double tmax = 0.0;
  for (int i = 0; i < 256; ++i) {
    x[i] = q2_load(p, tr * 16 + (i >> 4), tc * 16 + (i & 15));
    tmax = fmax(tmax, fabs(x[i]));
  }
  uint8_t code[2][256];
  uint32_t sc[2];
  double err[2];
  const int ncand = p.mode == ADAPTIVE ? 2 : 1;
  for (int k = 0; k < ncand; ++k) {
    const double m = (p.mode == FIXED4 || k == 1) ? 4.0 : 6.0;
    uint32_t s = enc_e4m3_d(__ddiv_rn(tmax, __dmul_rn(alpha, m)));
    if (tmax == 0.0) s = 1;
    const double denom = __dmul_rn(alpha, dec_e4m3_d(s));
    double e[256];
    double mx = 0.0;
    for (int i = 0; i < 256; ++i) {
      const double q = denom > 0.0 ? __ddiv_rn(x[i], denom) : ((x[i] != 0.0) ? copysign(6.0, x[i]) : 0.0);
      code[k][i] = (uint8_t)enc_fp4_d(q);
      const double diff = __dsub_rn(__dmul_rn(dec_fp4_d(code[k][i]), denom), x[i]);
      e[i] = p.rule == RULE_MSE ? __dmul_rn(diff, diff) : fabs(diff);
      mx = fmax(mx, fabs(diff));
    }
    sc[k] = s;
    err[k] = p.rule == RULE_ABSMAX ? mx : pw_tile(e);
  }
  const bool k4 = (p.mode == ADAPTIVE) ? (err[1] < err[0]) : (p.mode == FIXED4);
  const int ki = (p.mode == ADAPTIVE && k4) ? 1 : 0;
  for (int rr = 0; rr < 16; ++rr) {
    const int64_t r = tr * 16 + rr;
    if (r < p.R) {
      uint64_t w = 0;
      for (int c = 0; c < 16; ++c)
        if (tc * 16 + c < p.C) w |= (uint64_t)code[ki][16 * rr + c] << (4 * c);
      *reinterpret_cast<uint64_t*>(p.codes + (r * nbC + tc) * 8) = w;
      p.scales_tc[sf_tc_offset(r, tc, kb4)] = (uint8_t)sc[ki];
      if (p.scales_rm) p.scales_rm[r * nbC + tc] = (uint8_t)sc[ki];
      if (p.pick4) p.pick4[r * nbC + tc] = (uint8_t)k4;
    }
    const int64_t rt = tc * 16 + rr;  // W^T row = W column
    if (p.codes_t && rt < p.C) {
      uint64_t w = 0;
      for (int c = 0; c < 16; ++c)
        if (tr * 16 + c < p.R) w |= (uint64_t)code[ki][16 * c + rr] << (4 * c);
      *reinterpret_cast<uint64_t*>(p.codes_t + (rt * nbR + tr) * 8) = w;
      p.scales_tc_t[sf_tc_offset(rt, tr, kb4t)] = (uint8_t)sc[ki];
    }
  }
}

#ifndef F46_Q2V2_MINB
#define F46_Q2V2_MINB 3
#endif
constexpr int kQ2Row = 24;  // staged tile row stride (bf16): 48 bytes, 16-byte aligned

// MSE: the rule is the squared error (the default) -- no |diff| maximum.
template <bool MSE>
__global__ void __launch_bounds__(256, F46_Q2V2_MINB) quant2d_v2_kernel(Q2Params p) {
  select_group2(p);
  __shared__ __align__(16) uint16_t stage[8][2][16 * kQ2Row];
  const int lane = threadIdx.x & 31, hw = lane >> 4, l = lane & 15, h = l >> 3, j = l & 7;
  const int hbase = lane & 16;
  const unsigned FULL = 0xFFFFFFFFu;
  const int64_t TR = (p.R + 15) >> 4, TC = (p.C + 15) >> 4;
  const int64_t ntiles = TR * TC;
  double alpha = p.alpha_override;
  if (!(alpha > 0.0)) {
    const double amax = *p.d_amax;
    alpha = amax == 0.0 ? 1.0 : (double)((float)amax / (float)p.mcap);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.d_alpha_out) *p.d_alpha_out = alpha;
    if (p.alpha_override <= 0.0 && p.d_flags && !(*p.d_amax <= 1.7976931348623157e308))
      atomicOr(p.d_flags, F46_FLAG_NONFINITE);
  }
  const int64_t nbC = (p.C + 15) >> 4, nbR = (p.R + 15) >> 4;
  const int64_t kb4 = (nbC + 3) >> 2, kb4t = (nbR + 3) >> 2;
  const bool overridden = p.alpha_override > 0.0;
  const TensorConsts tcs = make_consts(
      alpha, RULE_MSE, p.dtype,
      tie_direction(alpha, overridden ? 0.0 : *p.d_amax, p.mcap, p.dtype, overridden));
  const int64_t G = (int64_t)gridDim.x * (blockDim.x >> 5) * 2;
  bool nonfinite = false;
  // the half-warp's tile (row tr, column tc), advanced by G tiles per
  // iteration without a division (tile counts fit 32 bits)
  const uint32_t tc32 = (uint32_t)TC, gq = (uint32_t)G / tc32, gr = (uint32_t)G - gq * tc32;
  uint32_t ttr, ttc;
  {
    const uint32_t t_first = (uint32_t)(((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 2 + hw);
    ttr = t_first / tc32;
    ttc = t_first - ttr * tc32;
  }
  for (int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 2; t0 < ntiles;
       t0 += G) {
    const int64_t tile = t0 + hw;
    const bool live = tile < ntiles;
    const int64_t tr = live ? (int64_t)ttr : 0, tc = live ? (int64_t)ttc : 0;
    ttc += gr;
    ttr += gq;
    if (ttc >= tc32) {
      ttc -= tc32;
      ++ttr;
    }
    const int64_t r0 = tr * 16 + 8 * h, c0 = tc * 16;
    // the lane's 16 values in accumulation order: (row r0 + i/2, col (i%2)*8 + j)
    float x[16];
    // interior BF16 tiles: the half-warp stages its 16x16 tile through shared
    // memory with two 16-byte loads per lane (lane l: row l of the tile)
    const bool staged = live && p.dtype == DT_BF16 && (p.C & 7) == 0 && tr * 16 + 16 <= p.R &&
                        c0 + 16 <= p.C && ((reinterpret_cast<uintptr_t>(p.w) & 15) == 0);
    if (__all_sync(FULL, staged)) {
      uint16_t* st = stage[threadIdx.x >> 5][hw];
      const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p.w) +
                                                        (tr * 16 + l) * p.C + c0);
      const uint4 v0 = __ldcs(src), v1 = __ldcs(src + 1);
      reinterpret_cast<uint4*>(st + l * kQ2Row)[0] = v0;
      reinterpret_cast<uint4*>(st + l * kQ2Row)[1] = v1;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i)
        x[i] = __uint_as_float((uint32_t)st[(8 * h + (i >> 1)) * kQ2Row + ((i & 1) << 3) + j] << 16);
      __syncwarp();
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int64_t r = r0 + (i >> 1), c = c0 + ((i & 1) << 3) + j;
        x[i] = live ? (float)q2_load(p, r, c) : 0.f;
      }
    }
    uint32_t mb = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) mb = max(mb, __float_as_uint(x[i]) & 0x7FFFFFFFu);
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) mb = max(mb, __shfl_xor_sync(FULL, mb, o));
    nonfinite |= live && mb >= 0x7F800000u;
    const float tmax = __uint_as_float(mb);
    const bool zero = mb == 0u;
    bool fast = !tcs.force_exact && (mb - 0x2B800000u) < 0x28000000u;
    const int ncand = p.mode == ADAPTIVE ? 2 : 1;
    uint32_t sc[2] = {1u, 1u};
    if (fast) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (k < ncand) {
          const bool m4 = (p.mode == FIXED4 || k == 1);
          sc[k] = block_scale_code(tmax, tcs.alpha, m4 ? 4.f : 6.f, m4 ? tcs.r4_lo : tcs.r6_lo,
                                   m4 ? tcs.r4_hi : tcs.r6_hi);
          fast &= sc[k] != 0u;
        }
      }
    }
    if (!fast) sc[0] = sc[1] = 0x38;  // placeholders: every lane runs the shuffles below
    float2 x2[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x2[q] = make_float2(x[2 * q], x[2 * q + 1]);
    const auto gload = [&](int i) -> float {
      return (float)q2_load(p, r0 + (i >> 1), c0 + ((i & 1) << 3) + j);
    };
    uint64_t cw[2] = {0, 0};
    double err[2] = {0.0, 0.0};
    // Adaptive MSE, fast tiles: certified f32 quotient-space errors (K2's
    // scheme over 256 values).  With the tile's exact codes v and q = x*rq
    // within 2^-19.9 of x/D, |S(f32) - S(exact)| <= 2^-14.4 tmax sqrt(S6+S4)
    // (Cauchy-Schwarz over 256 terms, |q| <= 6.5) + 2^-20 (S6+S4) (f32 sums,
    // D^2) + 2^-31.8 tmax^2 (second order); outside the (wider) tolerance the
    // f32 comparison is the reference's, else the float64 sums below decide.
    float s32[2] = {0.f, 0.f};
    const bool f32dec = MSE && p.mode == ADAPTIVE;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (k >= ncand) break;
      const float delta = e4m3_to_f32(sc[k]);
      const float rq = rcp_approx(tcs.alpha * delta) * F46_QLO;
      const uint64_t codes = exact_codes(x2, rq, tcs.alpha, delta, tcs.tdir, gload);
      cw[k] = codes;
      if (f32dec) {
        uint32_t v[8];
        unpack_e2m1x8((uint32_t)codes ^ tcs.zero, *reinterpret_cast<uint32_t(*)[4]>(&v[0]));
        unpack_e2m1x8((uint32_t)(codes >> 32) ^ tcs.zero, *reinterpret_cast<uint32_t(*)[4]>(&v[4]));
        const float2 r2 = make_float2(rq, rq);
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) {
          const float2 qv = __fmul2_rn(x2[pp], r2);
          const float2 r = make_float2(fhadd_h<0>(v[pp], -qv.x), fhadd_h<1>(v[pp], -qv.y));
          acc = __ffma2_rn(r, r, acc);
        }
        float t = acc.x + acc.y;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) t += __shfl_down_sync(FULL, t, o);
        const float D = tcs.alpha * delta;
        s32[k] = __shfl_sync(FULL, t, hbase) * (D * D);
      }
    }
    bool need64 = !f32dec;
    if (f32dec) {
      const float ssum = s32[0] + s32[1];
      const float tol = fmaf(0x1.6a09e6p-14f * tmax, sqrt_approx(ssum),  // 2^-13.5
                             fmaf(0x1p-18f, ssum, fmaf(0x1p-30f * tmax, tmax, 0x1p-140f)));
      need64 = fast && !(fabsf(s32[0] - s32[1]) > tol);
      err[0] = s32[0];
      err[1] = s32[1];
    }
    if (__any_sync(FULL, need64)) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (k >= ncand) break;
      const float delta = e4m3_to_f32(sc[k]);
      const uint64_t codes = cw[k];
      const double denom = (double)tcs.alpha * (double)delta;  // exact
      double r = 0.0, mx = 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double diff = __dsub_rn(__dmul_rn(dec_fp4_d((uint32_t)(codes >> (4 * i)) & 15u), denom),
                                      (double)x[i]);
        const double e = MSE ? __dmul_rn(diff, diff) : (p.rule == RULE_MSE ? __dmul_rn(diff, diff) : fabs(diff));
        r = i == 0 ? e : __dadd_rn(r, e);
        if (!MSE) mx = fmax(mx, fabs(diff));
      }
      double tot;
      if (!MSE && p.rule == RULE_ABSMAX) {
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
        tot = mx;
      } else {
        const double a = __dadd_rn(r, __shfl_down_sync(FULL, r, 1));   // j even
        const double b = __dadd_rn(a, __shfl_down_sync(FULL, a, 2));   // j % 4 == 0
        const double c = __dadd_rn(b, __shfl_down_sync(FULL, b, 4));   // j == 0: part(h)
        const double t = __dadd_rn(c, __shfl_down_sync(FULL, c, 8));   // lane (0, 0)
        tot = __shfl_sync(FULL, t, hbase);
      }
      if (need64) err[k] = tot;
    }
    }
    const bool k4 = (p.mode == ADAPTIVE) ? (err[1] < err[0]) : (p.mode == FIXED4);
    const int ki = (p.mode == ADAPTIVE && k4) ? 1 : 0;
    uint64_t codes = cw[ki];
    uint32_t s = sc[ki];
    if (zero) {
      // all-zero tile (blockquant.py:241): scale code 1, codes keep -0.0's sign, tie keeps 6
      codes = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) codes |= (uint64_t)(__float_as_uint(x[i]) >> 31) << (4 * i + 3);
      s = 1;
    }
    const bool ok = fast || zero;
    // W rows: lane (h, j) writes row r0 + j; column c's nibble comes from lane
    // (h, c % 8), element 2j + c / 8
    // byte j of lane (h, c)'s codes = its elements 2j (low nibble) and 2j + 1
    uint32_t wlo = 0, whi = 0;
    const uint32_t bsel = (uint32_t)(j & 3) | 0x4440u;  // byte j%4 into byte 0, zeros above
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t lo = __shfl_sync(FULL, (uint32_t)codes, hbase + 8 * h + c);
      const uint32_t hi = __shfl_sync(FULL, (uint32_t)(codes >> 32), hbase + 8 * h + c);
      const uint32_t b = __byte_perm(j < 4 ? lo : hi, 0u, bsel);
      wlo |= (b & 0xFu) << (4 * c);   // element 2j: column c
      whi |= (b >> 4) << (4 * c);     // element 2j + 1: column 8 + c
    }
    const uint64_t wrow = ((uint64_t)whi << 32) | wlo;
    if (live && ok) {
      const int64_t r = r0 + j;
      if (r < p.R) {
        uint64_t w = wrow;
        if (c0 + 16 > p.C) w &= (1ull << (4 * (int)(p.C - c0))) - 1;  // pad columns
        *reinterpret_cast<uint64_t*>(p.codes + (r * nbC + tc) * 8) = w;
        p.scales_tc[sf_tc_offset32((uint32_t)r, (uint32_t)tc, (uint32_t)kb4)] = (uint8_t)s;
        if (p.scales_rm) p.scales_rm[r * nbC + tc] = (uint8_t)s;
        if (p.pick4) p.pick4[r * nbC + tc] = (uint8_t)(zero ? (p.mode == FIXED4) : k4);
      }
      if (p.codes_t) {
        // W^T rows c0 + j (even elements) and c0 + 8 + j (odd elements), word h
#pragma unroll
        for (int par = 0; par < 2; ++par) {
          // nibbles par, par+2, ..., par+14 of the 16 codes, packed: per 32-bit
          // half keep one nibble of every byte, then squeeze the bytes together
          auto squeeze = [](uint32_t w) -> uint32_t {
            w &= 0x0F0F0F0Fu;
            w = (w | (w >> 4)) & 0x00FF00FFu;
            return (w | (w >> 8)) & 0x0000FFFFu;
          };
          const uint32_t lo = (uint32_t)codes >> (4 * par), hi = (uint32_t)(codes >> 32) >> (4 * par);
          uint32_t wt = squeeze(lo) | (squeeze(hi) << 16);
          const int64_t rt = c0 + 8 * par + j;
          if (rt < p.C && r0 < p.R) {
            if (r0 + 8 > p.R) wt &= (1u << (4 * (int)(p.R - r0))) - 1u;  // pad rows of W
            reinterpret_cast<uint32_t*>(p.codes_t + (rt * nbR + tr) * 8)[h] = wt;
            if (h == 0) p.scales_tc_t[sf_tc_offset32((uint32_t)rt, (uint32_t)tr, (uint32_t)kb4t)] = (uint8_t)s;
          } else if (rt < p.C) {
            reinterpret_cast<uint32_t*>(p.codes_t + (rt * nbR + tr) * 8)[h] = 0u;
          }
        }
      }
    }
    if (live && !ok && l == 0) quant2d_tile_exact(p, alpha, tr, tc);
  }
  nonfinite = __any_sync(FULL, nonfinite);
  if (nonfinite && lane == 0 && p.d_flags) atomicOr(p.d_flags, F46_FLAG_NONFINITE);
}

// ---------------------------------------------------------------------------
// Selection statistics for all three rules in one pass (adaptive.py:159-187):
// per block both candidates' exact float64 errors (sq / abs / max, numpy
// pairwise order via exact_pass), the 4-vs-6 pick of each rule (strict '<'),
// counts of 4-picks, pairwise rule disagreements and the chosen candidate's
// squared error.  Each CTA writes 9 partials (6 counts, 3 sums) in a fixed
// reduction order, so results are deterministic; the host folds the partials.
// ---------------------------------------------------------------------------
// exact_pass given the candidate's (exact) codes: the reference's float64
// error terms and pairwise sums (blockquant.py:279, :283-293).
__device__ __forceinline__ void exact_pass_codes(const double (&x)[16], uint64_t codes, double alpha,
                                                 double delta, uint32_t sc, ExactPass& o) {
  const double denom = __dmul_rn(alpha, delta);
  double esq[16], eab[16];
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double diff = __dsub_rn(__dmul_rn(dec_fp4_d((uint32_t)(codes >> (4 * i)) & 15u), denom), x[i]);
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

template <int DT>
__global__ void __launch_bounds__(256) stats_kernel(const void* __restrict__ x, int64_t rows,
                                                    int64_t cols, double mcap, const double* d_amax,
                                                    double alpha_override, double* partials,
                                                    double* d_alpha_out) {
  const int64_t nb = (cols + 15) >> 4;
  const int64_t total = rows * nb;
  double alpha = alpha_override;
  if (!(alpha > 0.0)) {
    const double amax = *d_amax;
    alpha = amax == 0.0 ? 1.0 : (double)((float)amax / (float)mcap);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && d_alpha_out) *d_alpha_out = alpha;
  const bool overridden = alpha_override > 0.0;
  const TensorConsts tcs = make_consts(
      alpha, RULE_MSE, DT, tie_direction(alpha, overridden ? 0.0 : *d_amax, mcap, DT, overridden));
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < total;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = b / nb, kb = b - row * nb;
    double xd[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int64_t c = kb * 16 + i;
      if (c >= cols)
        xd[i] = 0.0;
      else if constexpr (DT == DT_BF16)
        xd[i] = (double)__uint_as_float(
            (uint32_t)(reinterpret_cast<const uint16_t*>(x)[row * cols + c]) << 16);
      else if constexpr (DT == DT_F32)
        xd[i] = (double)reinterpret_cast<const float*>(x)[row * cols + c];
      else
        xd[i] = reinterpret_cast<const double*>(x)[row * cols + c];
    }
    ExactPass p6, p4;
    // fast path: exact scale codes (f32 brackets + tie test) and exact codes
    // (bracket logic), then the reference's float64 error terms
    float2 xf[8];
    float bmax = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      xf[q] = make_float2((float)xd[2 * q], (float)xd[2 * q + 1]);
      bmax = fmax_nan(bmax, fmax_nan(fabsf(xf[q].x), fabsf(xf[q].y)));
    }
    bool fast = DT != DT_F64 && !tcs.force_exact &&
                (__float_as_uint(bmax) - 0x2B800000u) < 0x28000000u;
    uint32_t sc6 = 0, sc4 = 0;
    if (fast) {
      sc6 = block_scale_code(bmax, tcs.alpha, 6.f, tcs.r6_lo, tcs.r6_hi);
      sc4 = block_scale_code(bmax, tcs.alpha, 4.f, tcs.r4_lo, tcs.r4_hi);
      fast = sc6 != 0u && sc4 != 0u;
    }
    if (fast) {
      const auto load = [&](int i) -> float { return (float)xd[i]; };
      const float d6 = e4m3_to_f32(sc6), d4 = e4m3_to_f32(sc4);
      const uint64_t c6 = exact_codes(xf, rcp_approx(tcs.alpha * d6) * F46_QLO, tcs.alpha, d6, tcs.tdir, load);
      const uint64_t c4 = exact_codes(xf, rcp_approx(tcs.alpha * d4) * F46_QLO, tcs.alpha, d4, tcs.tdir, load);
      exact_pass_codes(xd, c6, alpha, (double)d6, sc6, p6);
      exact_pass_codes(xd, c4, alpha, (double)d4, sc4, p4);
    } else {
      exact_pass(xd, alpha, 6.0, p6);
      exact_pass(xd, alpha, 4.0, p4);
    }
    const bool k_sq = p4.sq < p6.sq, k_ab = p4.ab < p6.ab, k_mx = p4.mx < p6.mx;
    acc[0] += k_sq;
    acc[1] += k_ab;
    acc[2] += k_mx;
    acc[3] += (k_sq != k_ab);
    acc[4] += (k_sq != k_mx);
    acc[5] += (k_ab != k_mx);
    acc[6] += k_sq ? p4.sq : p6.sq;
    acc[7] += k_ab ? p4.sq : p6.sq;
    acc[8] += k_mx ? p4.sq : p6.sq;
  }
  __shared__ double red[8][9];
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 9) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w][threadIdx.x];
    partials[blockIdx.x * 9 + threadIdx.x] = v;
  }
}

// ---------------------------------------------------------------------------
// Stochastic rounding (blockquant.py:253-257 _sr_uniforms, codecs.py:120-148
// encode_fp4_stochastic) and the 16-wide randomized Hadamard transform
// (transforms.py:41-105): the gradient recipe of qlinear.py:123-159.
//
// Uniforms are numpy's, bit for bit: Generator(Philox(SeedSequence(seed,
// spawn_key=(tag, m)))).random(shape) is Philox4x64-10 keyed by the
// SeedSequence's generate_state(2, uint64) (derived on the host), counter
// value i/4 + 1 for the i-th uint64 of the stream, word i % 4, and the double
// (x >> 11) * 2^-53.  Element i of the padded block array (rows, nblocks, 16)
// consumes stream position i, so any schedule gives the same bits.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void philox4x64_10(uint64_t (&c)[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// the 16 uniforms of padded block b (stream positions 16b .. 16b+15)
__device__ __forceinline__ void sr_uniforms16(uint64_t b, uint64_t k0, uint64_t k1, double (&u)[16]) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const uint64_t ctr = 4 * b + g + 1;  // 128-bit add would matter only past 2^64 positions
    uint64_t c[4] = {ctr, 0, 0, 0};
    philox4x64_10(c, k0, k1);
#pragma unroll
    for (int w = 0; w < 4; ++w) u[4 * g + w] = (double)(c[w] >> 11) * 0x1p-53;
  }
}

// codecs.py:120-148 for one finite value
__device__ __forceinline__ uint32_t enc_fp4_sr_d(double x, double u) {
  const double mags[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
  const double xc = fmin(fmax(x, -6.0), 6.0);
  const double a = fabs(xc);
  int k = 0;
#pragma unroll
  for (int j = 1; j < 8; ++j) k += (mags[j] <= a);
  if (mags[k] == a) {  // exactly representable: its own code; -0.0 keeps the sign bit
    if (a == 0.0) return signbit(x) ? 8u : 0u;
    return (uint32_t)k | (xc < 0.0 ? 8u : 0u);
  }
  const double gap = mags[k + 1] - mags[k];
  if (xc > 0.0) {
    const bool take_hi = u < (a - mags[k]) / gap;  // (xc - lo) / gap
    return take_hi ? (uint32_t)(k + 1) : (uint32_t)k;
  }
  // negative: lo = -mags[k+1], hi = -mags[k] (0.0 when k == 0, code 0)
  const bool take_hi = u < (mags[k + 1] - a) / gap;
  if (take_hi) return k == 0 ? 0u : (8u | (uint32_t)k);
  return 8u | (uint32_t)(k + 1);
}

// One fixed-target pass with stochastic rounding (blockquant.py:302-313 with
// _cast_values' "sr" branch); errors in numpy's pairwise order.
__device__ __forceinline__ void exact_pass_sr(const double (&x)[16], double alpha, double m,
                                              const double (&u)[16], ExactPass& o) {
  double bmax = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) bmax = fmax(bmax, fabs(x[i]));
  uint32_t sc = enc_e4m3_d(__ddiv_rn(bmax, __dmul_rn(alpha, m)));
  if (bmax == 0.0) sc = 1;
  const double denom = __dmul_rn(alpha, dec_e4m3_d(sc));
  double esq[16], eab[16];
  double mx = 0.0;
  uint64_t codes = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double q = denom > 0.0 ? __ddiv_rn(x[i], denom)
                                 : ((x[i] != 0.0) ? copysign(6.0, x[i]) : 0.0);
    const uint32_t c = enc_fp4_sr_d(q, u[i]);
    codes |= (uint64_t)c << (4 * i);
    const double diff = __dsub_rn(__dmul_rn(dec_fp4_d(c), denom), x[i]);
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

// Fast, exact SR codes for one candidate (BF16/F32 input, f32 alpha, valid
// scale).  The reference rounds q = RN64(x / denom) stochastically: inside
// the grid interval [lo, hi) it takes the far end iff u < (|q| - lo) / gap
// (positive) or u < (hi - |q|) / gap (negative); a - lo is exact (Sterbenz)
// and gap is a power of two, so the only rounding is the quotient.  An f32
// quotient (x * rcp(alpha*delta), relative error < 2^-21.9) gives the interval
// position pt within 2^-20.4; when pt is 2^-18 clear of 0, 1 and u the
// decision is the reference's, otherwise that element recomputes q in float64.
__device__ __noinline__ uint32_t sr_code_exact(double xd, double denom, double u) {
  return enc_fp4_sr_d(__ddiv_rn(xd, denom), u);
}

__device__ __forceinline__ uint32_t sr_code_fast(float x, float R, double u, double xd,
                                                 double denom) {
  if (x == 0.f) return signbit(x) ? 8u : 0u;
  const float a = fabsf(x * R);
  const uint32_t sgn = x < 0.f ? 8u : 0u;
  if (a >= 6.0f * (1.0f + 0x1p-18f)) return 7u | sgn;  // saturates (exact q > 6 too)
  // k = index of the grid point at or below a (0 .5 1 1.5 2 3 4 6): from the
  // exponent and the top mantissa bit for a >= 1
  const uint32_t b = __float_as_uint(a);
  const int e = (int)(b >> 23) - 127;
  const uint32_t k = a >= 1.0f ? (uint32_t)min(2 * e + 2 + (int)((b >> 22) & 1u), 7)
                               : (a >= 0.5f ? 1u : 0u);
  const float lo = fp4_mag_f32(k);
  // 1 / gap: 2 2 2 2 1 1 0.5 for k = 0..6
  const float inv_gap = k < 4 ? 2.0f : (k < 6 ? 1.0f : 0.5f);
  const float pt = (a - lo) * inv_gap;
  const float uf = (float)u;
  if (k < 7 && pt > 0x1p-18f && pt < 1.0f - 0x1p-18f && fabsf(uf - (sgn ? 1.0f - pt : pt)) > 0x1p-18f) {
    if (!sgn) return uf < pt ? k + 1 : k;
    if (uf < 1.0f - pt) return k == 0 ? 0u : (8u | k);
    return 8u | (k + 1);
  }
  return sr_code_exact(xd, denom, u);
}

struct SRParams {
  QParams q;
  uint64_t k6_0, k6_1, k4_0, k4_1;  // Philox keys of the m=6 / m=4 streams
};

template <int DT>
__global__ void __launch_bounds__(128) quant_sr_kernel(SRParams sp) {
  const QParams& p = sp.q;
  const int64_t nb = (p.cols + 15) >> 4;
  const int64_t kb4 = (nb + 3) >> 2;
  const int64_t rows_pad = (p.rows + 127) & ~(int64_t)127;
  const int64_t total = rows_pad * kb4 * 4;
  const double alpha = resolve_alpha(p);
  prologue_flags(p, alpha);
  const TensorConsts tcs = make_consts(alpha, RULE_MSE, DT);
  bool nonfinite = false;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / (kb4 * 4), kb = idx - row * (kb4 * 4);
    if (row >= p.rows || kb >= nb) {
      p.scales_tc[sf_tc_offset(row, kb, kb4)] = 0;
      continue;
    }
    double xd[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int64_t c = kb * 16 + i;
      if (c >= p.cols)
        xd[i] = 0.0;
      else if constexpr (DT == DT_BF16)
        xd[i] = (double)__uint_as_float(
            (uint32_t)(reinterpret_cast<const uint16_t*>(p.x)[row * p.cols + c]) << 16);
      else if constexpr (DT == DT_F32)
        xd[i] = (double)reinterpret_cast<const float*>(p.x)[row * p.cols + c];
      else
        xd[i] = reinterpret_cast<const double*>(p.x)[row * p.cols + c];
      nonfinite |= !(fabs(xd[i]) <= 1.7976931348623157e308);
    }
    const uint64_t blk = (uint64_t)(row * nb + kb);
    double u[16];
    BlockOut o;
    // fast path: f32 brackets for the scale (exact tie test) and sr_code_fast
    // for the codes; the float64 error sums and the decision are the reference's
    double bmaxd = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) bmaxd = fmax(bmaxd, fabs(xd[i]));
    const float bmaxf = (float)bmaxd;
    const bool fast = DT != DT_F64 && !tcs.force_exact && !(bmaxd > 3.4e38) &&
                      (__float_as_uint(bmaxf) - 0x2B800000u) < 0x28000000u;
    auto fast_pass = [&](float m, float r_lo, float r_hi, ExactPass& o2) -> bool {
      const uint32_t sc = block_scale_code(bmaxf, tcs.alpha, m, r_lo, r_hi);
      if (sc == 0) return false;
      const float delta = e4m3_to_f32(sc);
      const float R = rcp_approx(tcs.alpha * delta);
      const double denom = (double)tcs.alpha * (double)delta;  // exact
      double e[16];  // the rule's per-element error (squared / absolute)
      double mx = 0.0;
      uint64_t codes = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t c = sr_code_fast((float)xd[i], R, u[i], xd[i], denom);
        codes |= (uint64_t)c << (4 * i);
        const double diff = __dsub_rn(__dmul_rn(dec_fp4_d(c), denom), xd[i]);
        e[i] = p.rule == RULE_MSE ? __dmul_rn(diff, diff) : fabs(diff);
        mx = fmax(mx, fabs(diff));
      }
      o2.codes = codes;
      o2.sc = sc;
      const double sum = p.rule == RULE_ABSMAX ? 0.0 : pw16(e);
      o2.sq = sum;  // only the field rule_err reads for this rule is meaningful
      o2.ab = sum;
      o2.mx = mx;
      return true;
    };
    if (fast && p.mode == ADAPTIVE) {
      ExactPass p6, p4;
      sr_uniforms16(blk, sp.k6_0, sp.k6_1, u);
      bool ok = fast_pass(6.f, tcs.r6_lo, tcs.r6_hi, p6);
      if (!ok) exact_pass_sr(xd, alpha, 6.0, u, p6);
      sr_uniforms16(blk, sp.k4_0, sp.k4_1, u);
      ok = fast_pass(4.f, tcs.r4_lo, tcs.r4_hi, p4);
      if (!ok) exact_pass_sr(xd, alpha, 4.0, u, p4);
      const bool k = rule_err(p4, p.rule) < rule_err(p6, p.rule);
      o.codes = k ? p4.codes : p6.codes;
      o.sc = k ? p4.sc : p6.sc;
      o.pick4 = k;
    } else if (fast) {
      const bool four = p.mode == FIXED4;
      ExactPass pp;
      sr_uniforms16(blk, four ? sp.k4_0 : sp.k6_0, four ? sp.k4_1 : sp.k6_1, u);
      if (!fast_pass(four ? 4.f : 6.f, four ? tcs.r4_lo : tcs.r6_lo, four ? tcs.r4_hi : tcs.r6_hi, pp))
        exact_pass_sr(xd, alpha, four ? 4.0 : 6.0, u, pp);
      o.codes = pp.codes;
      o.sc = pp.sc;
      o.pick4 = four;
    } else if (p.mode == ADAPTIVE) {
      ExactPass p6, p4;
      sr_uniforms16(blk, sp.k6_0, sp.k6_1, u);
      exact_pass_sr(xd, alpha, 6.0, u, p6);
      sr_uniforms16(blk, sp.k4_0, sp.k4_1, u);
      exact_pass_sr(xd, alpha, 4.0, u, p4);
      const bool k = rule_err(p4, p.rule) < rule_err(p6, p.rule);
      o.codes = k ? p4.codes : p6.codes;
      o.sc = k ? p4.sc : p6.sc;
      o.pick4 = k;
    } else {
      const bool four = p.mode == FIXED4;
      ExactPass pp;
      sr_uniforms16(blk, four ? sp.k4_0 : sp.k6_0, four ? sp.k4_1 : sp.k6_1, u);
      exact_pass_sr(xd, alpha, four ? 4.0 : 6.0, u, pp);
      o.codes = pp.codes;
      o.sc = pp.sc;
      o.pick4 = four;
    }
    uint64_t codes = o.codes;
    const int64_t c0 = kb * 16;
    if (c0 + 16 > p.cols) {
      const int valid = (int)(p.cols - c0);
      codes &= ((1ull << (4 * valid)) - 1);
    }
    *reinterpret_cast<uint64_t*>(p.codes + (row * nb + kb) * 8) = codes;
    p.scales_tc[sf_tc_offset(row, kb, kb4)] = (uint8_t)o.sc;
    if (p.scales_rm) p.scales_rm[row * nb + kb] = (uint8_t)o.sc;
    if (p.pick4) p.pick4[row * nb + kb] = (uint8_t)o.pick4;
  }
  if (nonfinite && p.d_flags) atomicOr(p.d_flags, F46_FLAG_NONFINITE);
}

// One block entirely in float64 (the reference's restatement), by one thread:
// the SR quad kernel's fallback for blocks outside the f32 fast path.
template <int DT>
__device__ __noinline__ void sr_block_exact(const SRParams sp, double alpha, int64_t row, int64_t kb,
                                            int64_t nb, int64_t kb4) {
  const QParams& p = sp.q;
  double xd[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int64_t c = kb * 16 + i;
    if (c >= p.cols)
      xd[i] = 0.0;
    else if constexpr (DT == DT_BF16)
      xd[i] = (double)__uint_as_float((uint32_t)(reinterpret_cast<const uint16_t*>(p.x)[row * p.cols + c]) << 16);
    else
      xd[i] = (double)reinterpret_cast<const float*>(p.x)[row * p.cols + c];
  }
  const uint64_t blk = (uint64_t)(row * nb + kb);
  double u[16];
  BlockOut o;
  if (p.mode == ADAPTIVE) {
    ExactPass p6, p4;
    sr_uniforms16(blk, sp.k6_0, sp.k6_1, u);
    exact_pass_sr(xd, alpha, 6.0, u, p6);
    sr_uniforms16(blk, sp.k4_0, sp.k4_1, u);
    exact_pass_sr(xd, alpha, 4.0, u, p4);
    const bool k = rule_err(p4, p.rule) < rule_err(p6, p.rule);
    o.codes = k ? p4.codes : p6.codes;
    o.sc = k ? p4.sc : p6.sc;
    o.pick4 = k;
  } else {
    const bool four = p.mode == FIXED4;
    ExactPass pp;
    sr_uniforms16(blk, four ? sp.k4_0 : sp.k6_0, four ? sp.k4_1 : sp.k6_1, u);
    exact_pass_sr(xd, alpha, four ? 4.0 : 6.0, u, pp);
    o.codes = pp.codes;
    o.sc = pp.sc;
    o.pick4 = four;
  }
  uint64_t codes = o.codes;
  const int64_t c0 = kb * 16;
  if (c0 + 16 > p.cols) codes &= ((1ull << (4 * (int)(p.cols - c0))) - 1);
  *reinterpret_cast<uint64_t*>(p.codes + blk * 8) = codes;
  p.scales_tc[sf_tc_offset(row, kb, kb4)] = (uint8_t)o.sc;
  if (p.scales_rm) p.scales_rm[blk] = (uint8_t)o.sc;
  if (p.pick4) p.pick4[blk] = (uint8_t)o.pick4;
}

// SR quantize with four threads per block (BF16 / F32 input): thread t of a
// quad owns elements 4t..4t+3, which are exactly the four uniforms of Philox
// counter 4b + t + 1, so each thread runs one Philox call per candidate.  The
// block max, the rule's error sum (numpy's pw16 association: r_j = e_j +
// e_{j+8} from the thread two lanes up, then ((r0+r1)+(r2+r3)) +
// ((r4+r5)+(r6+r7)) across the pair) and the decision go through quad
// shuffles.  Blocks outside the f32 fast path (alpha override that is not a
// float32, extreme magnitudes, underflowed scale) fall back to sr_block_exact.
template <int DT>
__global__ void __launch_bounds__(256, 3) quant_sr4_kernel(SRParams sp) {
  const QParams& p = sp.q;
  const int64_t nb = (p.cols + 15) >> 4;
  const int64_t kb4 = (nb + 3) >> 2;
  const int64_t rows_pad = (p.rows + 127) & ~(int64_t)127;
  const int64_t total = rows_pad * kb4 * 4;
  const double alpha = resolve_alpha(p);
  prologue_flags(p, alpha);
  const TensorConsts tcs = make_consts(alpha, RULE_MSE, DT);
  const int lane = threadIdx.x & 31, t = lane & 3, qbase = lane & ~3;
  const unsigned FULL = 0xFFFFFFFFu;
  bool nonfinite = false;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 8; base < total;
       base += nwarps * 8) {
    const int64_t idx = base + (lane >> 2);
    const int64_t row = idx / (kb4 * 4), kb = idx - row * (kb4 * 4);
    const bool inb = idx < total;
    const bool active = inb && row < p.rows && kb < nb;
    if (inb && !active && t == 0) p.scales_tc[sf_tc_offset(row, kb, kb4)] = 0;  // layout padding
    // the thread's four values (pads and inactive lanes: +0)
    float xf[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t c = kb * 16 + 4 * t + i;
      float v = 0.f;
      if (active && c < p.cols) {
        if constexpr (DT == DT_BF16)
          v = __uint_as_float((uint32_t)(reinterpret_cast<const uint16_t*>(p.x)[row * p.cols + c]) << 16);
        else
          v = reinterpret_cast<const float*>(p.x)[row * p.cols + c];
      }
      xf[i] = v;
    }
    uint32_t mb = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) mb = max(mb, __float_as_uint(xf[i]) & 0x7FFFFFFFu);
    mb = max(mb, __shfl_xor_sync(FULL, mb, 1));
    mb = max(mb, __shfl_xor_sync(FULL, mb, 2));
    nonfinite |= active && mb >= 0x7F800000u;
    const float bmax = __uint_as_float(mb);
    bool fast = !tcs.force_exact && (mb - 0x2B800000u) < 0x28000000u;
    const bool two = p.mode == ADAPTIVE;
    const bool m4only = p.mode == FIXED4;
    uint32_t sc[2] = {0, 0};
    double err[2] = {0.0, 0.0};
    uint32_t cw[2] = {0, 0};  // the thread's 4 codes per candidate
    if (fast) {
      sc[0] = block_scale_code(bmax, tcs.alpha, m4only ? 4.f : 6.f, m4only ? tcs.r4_lo : tcs.r6_lo,
                               m4only ? tcs.r4_hi : tcs.r6_hi);
      if (two) sc[1] = block_scale_code(bmax, tcs.alpha, 4.f, tcs.r4_lo, tcs.r4_hi);
      fast = sc[0] != 0u && (!two || sc[1] != 0u);
    }
    if (!fast) sc[0] = sc[1] = 0x38;  // placeholders: every lane runs the shuffles below
    {
      const uint64_t blk = (uint64_t)(row * nb + kb);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (k == 1 && !two) break;
        const bool use4 = (k == 1) || m4only;
        uint64_t c4[4] = {4 * blk + (uint64_t)t + 1, 0, 0, 0};
        philox4x64_10(c4, use4 ? sp.k4_0 : sp.k6_0, use4 ? sp.k4_1 : sp.k6_1);
        const float delta = e4m3_to_f32(sc[k]);
        const float R = rcp_approx(tcs.alpha * delta);
        const double denom = (double)tcs.alpha * (double)delta;  // exact
        double e[4];
        double mx = 0.0;
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double u = (double)(c4[i] >> 11) * 0x1p-53;
          const uint32_t c = sr_code_fast(xf[i], R, u, (double)xf[i], denom);
          w |= c << (4 * i);
          const double diff = __dsub_rn(__dmul_rn(dec_fp4_d(c), denom), (double)xf[i]);
          e[i] = p.rule == RULE_MSE ? __dmul_rn(diff, diff) : fabs(diff);
          mx = fmax(mx, fabs(diff));
        }
        double tot;
        if (p.rule == RULE_ABSMAX) {
          mx = fmax(mx, __shfl_xor_sync(FULL, mx, 1));
          tot = fmax(mx, __shfl_xor_sync(FULL, mx, 2));
        } else {
          double r[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) r[i] = __dadd_rn(e[i], __shfl_down_sync(FULL, e[i], 2));
          const double a = __dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3]));
          tot = __shfl_sync(FULL, __dadd_rn(a, __shfl_down_sync(FULL, a, 1)), qbase);
        }
        err[k] = tot;
        cw[k] = w;
      }
      const bool k4 = two ? (err[1] < err[0]) : m4only;
      const int ki = (two && k4) ? 1 : 0;
      if (active && fast) {
        reinterpret_cast<uint16_t*>(p.codes + (row * nb + kb) * 8)[t] = (uint16_t)cw[ki];
        if (t == 0) {
          p.scales_tc[sf_tc_offset(row, kb, kb4)] = (uint8_t)sc[ki];
          if (p.scales_rm) p.scales_rm[row * nb + kb] = (uint8_t)sc[ki];
          if (p.pick4) p.pick4[row * nb + kb] = (uint8_t)k4;
        }
      }
    }
    if (!fast && active && t == 0) sr_block_exact<DT>(sp, alpha, row, kb, nb, kb4);
  }
  nonfinite = __any_sync(FULL, nonfinite);
  if (nonfinite && lane == 0 && p.d_flags) atomicOr(p.d_flags, F46_FLAG_NONFINITE);
}

// ---------------------------------------------------------------------------
// Single block of any length at any target m (the reference's block-level API,
// blockquant.py:225-236 compute_block_scale and :379-414 quantize_block): one
// thread restates the float64 arithmetic, including numpy's 1-D pairwise sum
// for the error means (n < 8: sequential from -0.0; n <= 128: 8 accumulators
// + tail; larger: split at n/2 rounded down to a multiple of 8).
// ---------------------------------------------------------------------------
__device__ double np_pairwise_sum(const double* a, int64_t n, int kind) {
  // kind 0: a[i]^2 of the diffs, 1: |a[i]|
  auto term = [&](int64_t i) -> double { return kind == 0 ? __dmul_rn(a[i], a[i]) : fabs(a[i]); };
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, term(i));
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = term(j);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], term(i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, term(i));
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum(a, n2, kind), np_pairwise_sum(a + n2, n - n2, kind));
}

// x: n float64 values; u: n uniforms (stochastic rounding) or null (RNE).
// Writes codes[n], work[n] (the diffs, then overwritten with deq), and
// out[4] = {scale code, sum diff^2, sum |diff|, max |diff|}.
__global__ void block_ref_kernel(const double* __restrict__ x, int64_t n, double alpha, double m,
                                 const double* __restrict__ u, uint8_t* __restrict__ codes,
                                 double* __restrict__ work, double* __restrict__ out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double bmax = 0.0;
  for (int64_t i = 0; i < n; ++i) bmax = fmax(bmax, fabs(x[i]));
  // _nvfp4_scales (blockquant.py:239-242)
  uint32_t sc = enc_e4m3_d(__ddiv_rn(bmax, __dmul_rn(alpha, m)));
  if (bmax == 0.0) sc = 1;
  const double denom = __dmul_rn(alpha, dec_e4m3_d(sc));
  double mx = 0.0;
  // _cast_values (blockquant.py:260-280)
  for (int64_t i = 0; i < n; ++i) {
    double s;
    if (denom > 0.0)
      s = __ddiv_rn(x[i], denom);
    else
      s = (x[i] != 0.0) ? copysign(6.0, x[i]) : 0.0;
    const uint32_t c = u ? enc_fp4_sr_d(s, u[i]) : enc_fp4_d(s);
    codes[i] = (uint8_t)c;
    const double diff = __dsub_rn(__dmul_rn(dec_fp4_d(c), denom), x[i]);
    work[i] = diff;
    mx = fmax(mx, fabs(diff));
  }
  out[0] = (double)sc;
  out[1] = np_pairwise_sum(work, n, 0);
  out[2] = np_pairwise_sum(work, n, 1);
  out[3] = mx;
  for (int64_t i = 0; i < n; ++i) work[i] = __dmul_rn(dec_fp4_d(codes[i]), denom);
}

// ---------------------------------------------------------------------------
// qlinear.py:64-71 _accum_matmul_f32 restated: C = A @ B with float32 products
// summed in ascending k, one rounding each (no FMA): the reference's
// emulated_fp4_matmul for operands it cannot hand to a block-scaled tensor-core
// instruction (transpose_b=False: B blocked along N).  A [M,K], B [K,N], C
// [M,N] row-major float32; 32x32 output tiles staged through shared memory
// in ascending k.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) matmul_f32_ordered_kernel(const float* __restrict__ A,
                                                                const float* __restrict__ B,
                                                                int64_t M, int64_t N, int64_t K,
                                                                float* __restrict__ C) {
  __shared__ float As[32][33], Bs[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads, 4 rows each
  const int64_t n = (int64_t)blockIdx.x * 32 + tx;
  const int64_t m0 = (int64_t)blockIdx.y * 32;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t k0 = 0; k0 < K; k0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      const int64_t m = m0 + r, k = k0 + tx;
      As[r][tx] = (m < M && k < K) ? A[m * K + k] : 0.f;
      const int64_t kb = k0 + r;
      Bs[r][tx] = (kb < K && n < N) ? B[kb * N + n] : 0.f;
    }
    __syncthreads();
    const int kt = (K - k0) < 32 ? (int)(K - k0) : 32;
    for (int kk = 0; kk < kt; ++kk) {
      const float b = Bs[kk][tx];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], __fmul_rn(As[ty + 8 * i][kk], b));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty + 8 * i;
    if (m < M && n < N) C[m * N + n] = acc[i];
  }
}

// transforms.py:92-97 apply_rht: y = fwht(g * signs) / sqrt(16) per group of
// 16 along the last dim, float64, numpy's butterfly order (h = 1, 2, 4, 8).
template <int DT>
__global__ void __launch_bounds__(256) rht16_kernel(const void* __restrict__ x, int64_t ngroups,
                                                    double4 s0, double4 s1, double4 s2, double4 s3,
                                                    double* __restrict__ out, bool vec) {
  const double sg[16] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w,
                         s2.x, s2.y, s2.z, s2.w, s3.x, s3.y, s3.z, s3.w};
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    double a[16];
    uint32_t wb[8];  // bf16: the group's 32 bytes in two 16-byte loads
    if (DT == DT_BF16 && vec) {
      const uint4* xv = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(x) + g * 16);
      const uint4 v0 = __ldg(xv), v1 = __ldg(xv + 1);
      wb[0] = v0.x; wb[1] = v0.y; wb[2] = v0.z; wb[3] = v0.w;
      wb[4] = v1.x; wb[5] = v1.y; wb[6] = v1.z; wb[7] = v1.w;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      double v;
      if constexpr (DT == DT_BF16)
        v = vec ? (double)__uint_as_float((i & 1) ? (wb[i >> 1] & 0xFFFF0000u) : (wb[i >> 1] << 16))
                : (double)__uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(x)[g * 16 + i] << 16);
      else if constexpr (DT == DT_F32)
        v = (double)reinterpret_cast<const float*>(x)[g * 16 + i];
      else
        v = reinterpret_cast<const double*>(x)[g * 16 + i];
      a[i] = __dmul_rn(v, sg[i]);
    }
#pragma unroll
    for (int h = 1; h < 16; h <<= 1) {
      double b[16];
#pragma unroll
      for (int blk = 0; blk < 16; blk += 2 * h)
#pragma unroll
        for (int j = 0; j < h; ++j) {
          b[blk + j] = __dadd_rn(a[blk + j], a[blk + h + j]);
          b[blk + h + j] = __dsub_rn(a[blk + j], a[blk + h + j]);
        }
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = b[i];
    }
    // /4 == *0.25 exactly (power of two, both correctly rounded); 16-byte stores
    if (vec) {
      double2* o2 = reinterpret_cast<double2*>(out + g * 16);
#pragma unroll
      for (int i = 0; i < 8; ++i) o2[i] = make_double2(__dmul_rn(a[2 * i], 0.25), __dmul_rn(a[2 * i + 1], 0.25));
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) out[g * 16 + i] = __dmul_rn(a[i], 0.25);
    }
  }
}

// ---------------------------------------------------------------------------
// K1: amax
// ---------------------------------------------------------------------------
template <int DT>
__global__ void __launch_bounds__(256) amax_kernel(const void* __restrict__ x, int64_t n,
                                                   double* d_amax) {
  if (gridDim.y > 1) {  // grouped: group blockIdx.y of n elements each
    constexpr int64_t kEsz = DT == DT_BF16 ? 2 : (DT == DT_F32 ? 4 : 8);
    x = reinterpret_cast<const uint8_t*>(x) + (int64_t)blockIdx.y * n * kEsz;
    d_amax += blockIdx.y;
  }
  uint64_t m64 = 0;  // float64 |x| bit pattern (non-negative: bit order == value order)
  uint32_t m32 = 0;  // float32 |x| bit pattern
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool aligned = ((uintptr_t)x & 15) == 0;
  if constexpr (DT == DT_BF16) {
    const uint16_t* xs = reinterpret_cast<const uint16_t*>(x);
    int64_t done = 0;
    if (aligned) {
      const int64_t nv = n >> 3;
      const uint4* xv = reinterpret_cast<const uint4*>(x);
      uint32_t m = 0;
      int64_t i = tid;
      // four independent 16-byte loads in flight per thread
      for (; i + 3 * stride < nv; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(xv + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          m = __vmaxu2(m, v[u].x & 0x7FFF7FFFu);
          m = __vmaxu2(m, v[u].y & 0x7FFF7FFFu);
          m = __vmaxu2(m, v[u].z & 0x7FFF7FFFu);
          m = __vmaxu2(m, v[u].w & 0x7FFF7FFFu);
        }
      }
      for (; i < nv; i += stride) {
        const uint4 v = __ldcs(xv + i);
        m = __vmaxu2(m, v.x & 0x7FFF7FFFu);
        m = __vmaxu2(m, v.y & 0x7FFF7FFFu);
        m = __vmaxu2(m, v.z & 0x7FFF7FFFu);
        m = __vmaxu2(m, v.w & 0x7FFF7FFFu);
      }
      m32 = max(m & 0xFFFFu, m >> 16) << 16;
      done = nv << 3;
    }
    for (int64_t i = done + tid; i < n; i += stride)
      m32 = max(m32, ((uint32_t)xs[i] & 0x7FFFu) << 16);
  } else if constexpr (DT == DT_F32) {
    const uint32_t* xs = reinterpret_cast<const uint32_t*>(x);
    int64_t done = 0;
    if (aligned) {
      const int64_t nv = n >> 2;
      const uint4* xv = reinterpret_cast<const uint4*>(x);
      for (int64_t i = tid; i < nv; i += stride) {
        const uint4 v = __ldcs(xv + i);
        m32 = max(m32, max(max(v.x & 0x7FFFFFFFu, v.y & 0x7FFFFFFFu),
                           max(v.z & 0x7FFFFFFFu, v.w & 0x7FFFFFFFu)));
      }
      done = nv << 2;
    }
    for (int64_t i = done + tid; i < n; i += stride) m32 = max(m32, xs[i] & 0x7FFFFFFFu);
  } else {
    const uint64_t* xs = reinterpret_cast<const uint64_t*>(x);
    for (int64_t i = tid; i < n; i += stride) {
      const uint64_t b = xs[i] & 0x7FFFFFFFFFFFFFFFull;
      m64 = b > m64 ? b : m64;
    }
  }
  if constexpr (DT != DT_F64) {
    // f32 -> f64 keeps NaN above +inf (|NaN| bits > inf bits in both formats)
    m64 = (uint64_t)__double_as_longlong((double)__uint_as_float(m32));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t v = __shfl_xor_sync(0xFFFFFFFFu, m64, o);
    m64 = v > m64 ? v : m64;
  }
  __shared__ uint64_t wmax[8];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m64;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = wmax[w] > b ? wmax[w] : b;
    atomicMax(reinterpret_cast<unsigned long long*>(d_amax), (unsigned long long)b);
  }
}

// ---------------------------------------------------------------------------
// K3: dequantize
// ---------------------------------------------------------------------------
template <int OUT, int SL>
__global__ void __launch_bounds__(256) dequant_kernel(const uint8_t* __restrict__ codes,
                                                      const uint8_t* __restrict__ scales,
                                                      const double* d_alpha, int64_t rows,
                                                      int64_t cols, void* out, uint32_t* d_flags) {
  const int64_t nb = (cols + 15) >> 4;
  const int64_t kb4 = (nb + 3) >> 2;
  const double alpha_d = *d_alpha;
  const float alpha = (float)alpha_d;
  const bool f32_alpha = ((double)alpha == alpha_d);
  const int64_t total = rows * nb;
  bool nan_scale = false;
  const bool small = total < (1ll << 32);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = small ? (int64_t)((uint32_t)idx / (uint32_t)nb) : idx / nb;
    const int64_t kb = idx - row * nb;
    const uint32_t sc = SL == F46_SCALES_TC ? scales[sf_tc_offset(row, kb, kb4)] : scales[idx];
    nan_scale |= ((sc & 0x7F) == 0x7F);
    const uint64_t cw = *reinterpret_cast<const uint64_t*>(codes + idx * 8);
    const int64_t c0 = kb * 16;
    const bool full = (c0 + 16 <= cols);
    if constexpr (OUT == DT_F64) {
      const double delta = dec_e4m3_d(sc);
      double* o = reinterpret_cast<double*>(out) + row * cols + c0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        // (vals * alpha) * scale, as blockquant.py:376 evaluates it
        const double v = __dmul_rn(__dmul_rn(dec_fp4_d((uint32_t)(cw >> (4 * i)) & 15u), alpha_d),
                                   delta);
        if (c0 + i < cols) o[i] = v;
      }
    } else if (f32_alpha) {
      // hardware decode: E2M1 pairs -> f16x2 -> f32 (exact), v*Delta exact in
      // f32 (<= 6 significant bits), one rounding of (v*Delta)*alpha
      const float delta = e4m3_to_f32(sc & 0x7F) * ((sc & 0x80) ? -1.f : 1.f);
      const float2 d2 = make_float2(delta, delta), a2 = make_float2(alpha, alpha);
      float y[16];
      const uint32_t cwl = (uint32_t)cw, cwh = (uint32_t)(cw >> 32);
#pragma unroll
      for (int pp = 0; pp < 8; ++pp) {
        const uint32_t w = pp < 4 ? cwl : cwh;
        uint32_t h;
        switch (pp & 3) {
          case 0: { const __half2 t = e2m1x2_to_h2<0>(w); h = *reinterpret_cast<const uint32_t*>(&t); } break;
          case 1: { const __half2 t = e2m1x2_to_h2<1>(w); h = *reinterpret_cast<const uint32_t*>(&t); } break;
          case 2: { const __half2 t = e2m1x2_to_h2<2>(w); h = *reinterpret_cast<const uint32_t*>(&t); } break;
          default: { const __half2 t = e2m1x2_to_h2<3>(w); h = *reinterpret_cast<const uint32_t*>(&t); } break;
        }
        const float2 v = make_float2(fhadd_h<0>(h, -0.f), fhadd_h<1>(h, -0.f));
        const float2 vd = __fmul2_rn(v, d2);
        if constexpr (OUT == DT_F32) {
          const float2 r = __fmul2_rn(vd, a2);
          y[2 * pp] = r.x;
          y[2 * pp + 1] = r.y;
        } else {
          // round-to-odd to f32, then RN to bf16 == one rounding of the exact product
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float vv = e ? vd.y : vd.x;
            const float rz = __fmul_rz(vv, alpha);
            const float rem = fmaf(vv, alpha, -rz);
            y[2 * pp + e] = __uint_as_float(__float_as_uint(rz) | (rem != 0.f ? 1u : 0u));
          }
        }
      }
      if constexpr (OUT == DT_F32) {
        float* o = reinterpret_cast<float*>(out) + row * cols + c0;
        if (full && ((((uintptr_t)o) & 15) == 0)) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            reinterpret_cast<float4*>(o)[q] =
                make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
        } else {
          for (int i = 0; i < 16; ++i)
            if (c0 + i < cols) o[i] = y[i];
        }
      } else {
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + row * cols + c0;
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const __nv_bfloat162 hb = __floats2bfloat162_rn(y[2 * q], y[2 * q + 1]);
          w[q] = *reinterpret_cast<const uint32_t*>(&hb);
        }
        if (full && ((((uintptr_t)o) & 15) == 0)) {
          reinterpret_cast<uint4*>(o)[0] = make_uint4(w[0], w[1], w[2], w[3]);
          reinterpret_cast<uint4*>(o)[1] = make_uint4(w[4], w[5], w[6], w[7]);
        } else {
          for (int i = 0; i < 16; ++i)
            if (c0 + i < cols) reinterpret_cast<uint16_t*>(o)[i] = (uint16_t)(w[i >> 1] >> (16 * (i & 1)));
        }
      }
    } else {
      const float delta = e4m3_to_f32(sc & 0x7F) * ((sc & 0x80) ? -1.f : 1.f);
      float y[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t c = (uint32_t)(cw >> (4 * i)) & 15u;
        const float v = (c & 8) ? -fp4_mag_f32(c & 7) : fp4_mag_f32(c & 7);
        if (f32_alpha) {
          const float vd = v * delta;  // exact (<= 6 significant bits)
          if constexpr (OUT == DT_F32) {
            y[i] = __fmul_rn(vd, alpha);  // one rounding of the exact product
          } else {
            // round-to-odd to f32, then RN to bf16 == one rounding of the exact product
            const float rz = __fmul_rz(vd, alpha);
            const float rem = fmaf(vd, alpha, -rz);
            y[i] = __uint_as_float(__float_as_uint(rz) | (rem != 0.f ? 1u : 0u));
          }
        } else {
          // (vals * alpha) * scale in float64 exactly as blockquant.py:376
          const double d = __dmul_rn(__dmul_rn((double)v, alpha_d), (double)delta);
          if constexpr (OUT == DT_F32) {
            y[i] = __double2float_rn(d);
          } else {
            const float rz = __double2float_rz(d);
            y[i] = __uint_as_float(__float_as_uint(rz) | ((double)rz != d ? 1u : 0u));
          }
        }
      }
      if constexpr (OUT == DT_F32) {
        float* o = reinterpret_cast<float*>(out) + row * cols + c0;
        if (full && ((((uintptr_t)o) & 15) == 0)) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            reinterpret_cast<float4*>(o)[q] =
                make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
        } else {
          for (int i = 0; i < 16; ++i)
            if (c0 + i < cols) o[i] = y[i];
        }
      } else {
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + row * cols + c0;
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const __nv_bfloat162 h = __floats2bfloat162_rn(y[2 * q], y[2 * q + 1]);
          w[q] = *reinterpret_cast<const uint32_t*>(&h);
        }
        if (full && ((((uintptr_t)o) & 15) == 0)) {
          reinterpret_cast<uint4*>(o)[0] = make_uint4(w[0], w[1], w[2], w[3]);
          reinterpret_cast<uint4*>(o)[1] = make_uint4(w[4], w[5], w[6], w[7]);
        } else {
          for (int i = 0; i < 16; ++i)
            if (c0 + i < cols) {
              const uint16_t h = (uint16_t)(w[i >> 1] >> (16 * (i & 1)));
              reinterpret_cast<uint16_t*>(o)[i] = h;
            }
        }
      }
    }
  }
  if (nan_scale && d_flags) atomicOr(d_flags, F46_FLAG_NAN_SCALE);
}

// Coalesced K3 for f32 / bf16 output with a float32 alpha: each thread owns EPT
// consecutive elements (16 bytes of output), so a warp's store instruction
// covers 512 contiguous bytes; the block's scale byte is shared by 16/EPT
// neighbouring threads.  Same arithmetic as dequant_kernel's fast branch.
template <int OUT, int SL>
__global__ void __launch_bounds__(256) dequant_vec_kernel(const uint8_t* __restrict__ codes,
                                                          const uint8_t* __restrict__ scales,
                                                          const double* d_alpha, int64_t rows,
                                                          int64_t cols, void* out,
                                                          uint32_t* d_flags) {
  constexpr int EPT = OUT == DT_F32 ? 4 : 8;  // 16 output bytes per thread
  constexpr int TPB = 16 / EPT;                // threads per 16-element block
  const int64_t nb = cols >> 4;                // cols % 16 == 0 on this path
  const int64_t kb4 = (nb + 3) >> 2;
  const double alpha_d = *d_alpha;
  const float alpha = (float)alpha_d;
  const bool f32_alpha = (double)alpha == alpha_d;  // else: float64 product, one rounding
  const int64_t total = rows * nb * TPB;
  const bool small = rows * nb < (1ll << 32);
  bool nan_scale = false;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = t / TPB;
    const int part = (int)(t % TPB);
    const int64_t row = small ? (int64_t)((uint32_t)idx / (uint32_t)nb) : idx / nb;
    const int64_t kb = idx - row * nb;
    const uint32_t sc = SL == F46_SCALES_TC ? scales[sf_tc_offset(row, kb, kb4)] : scales[idx];
    nan_scale |= ((sc & 0x7F) == 0x7F);
    const float delta = e4m3_to_f32(sc & 0x7F) * ((sc & 0x80) ? -1.f : 1.f);
    const float2 d2 = make_float2(delta, delta), a2 = make_float2(alpha, alpha);
    uint32_t w;  // EPT codes, even element in the low nibble
    if (EPT == 4)
      w = *reinterpret_cast<const uint16_t*>(codes + idx * 8 + part * 2);
    else
      w = *reinterpret_cast<const uint32_t*>(codes + idx * 8 + part * 4);
    float y[EPT];
#pragma unroll
    for (int pp = 0; pp < EPT / 2; ++pp) {
      uint32_t h;
      switch (pp) {
        case 0: { const __half2 q = e2m1x2_to_h2<0>(w); h = *reinterpret_cast<const uint32_t*>(&q); } break;
        case 1: { const __half2 q = e2m1x2_to_h2<1>(w); h = *reinterpret_cast<const uint32_t*>(&q); } break;
        case 2: { const __half2 q = e2m1x2_to_h2<2>(w); h = *reinterpret_cast<const uint32_t*>(&q); } break;
        default: { const __half2 q = e2m1x2_to_h2<3>(w); h = *reinterpret_cast<const uint32_t*>(&q); } break;
      }
      const float2 vd = __fmul2_rn(make_float2(fhadd_h<0>(h, -0.f), fhadd_h<1>(h, -0.f)), d2);
      if (!f32_alpha) {
        // (vals * alpha) * scale in float64 exactly as blockquant.py:376, one rounding
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double d = __dmul_rn((double)(e ? vd.y : vd.x), alpha_d);
          if constexpr (OUT == DT_F32) {
            y[2 * pp + e] = __double2float_rn(d);
          } else {
            const float rz = __double2float_rz(d);
            y[2 * pp + e] = __uint_as_float(__float_as_uint(rz) | ((double)rz != d ? 1u : 0u));
          }
        }
      } else if constexpr (OUT == DT_F32) {
        const float2 r = __fmul2_rn(vd, a2);
        y[2 * pp] = r.x;
        y[2 * pp + 1] = r.y;
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float vv = e ? vd.y : vd.x;
          const float rz = __fmul_rz(vv, alpha);
          const float rem = fmaf(vv, alpha, -rz);
          y[2 * pp + e] = __uint_as_float(__float_as_uint(rz) | (rem != 0.f ? 1u : 0u));
        }
      }
    }
    const int64_t e0 = row * cols + kb * 16 + part * EPT;
    if constexpr (OUT == DT_F32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + e0) = make_float4(y[0], y[1], y[2], y[3]);
    } else {
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __nv_bfloat162 hb = __floats2bfloat162_rn(y[2 * q], y[2 * q + 1]);
        o[q] = *reinterpret_cast<const uint32_t*>(&hb);
      }
      *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + e0) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
  if (nan_scale && d_flags) atomicOr(d_flags, F46_FLAG_NAN_SCALE);
}

// K3 with TMA-staged stores.  cols % 16 == 0 makes the packed codes and the
// output one flat stream, so a warp owns a 1024-element chunk: each lane loads
// 16 contiguous code bytes (two blocks, the warp 512 B coalesced) and their two
// scale bytes, prefetched one chunk ahead; writes its 32 results into the
// warp's 128-byte-swizzled staging buffer (bank-conflict free); one lane then
// stores the chunk with a single cp.async.bulk.tensor (2 or 4 KB) and the warp
// moves on -- two buffers per warp keep a store in flight while the next chunk
// is computed.  The output is viewed as [n / EPR rows][128 B]; elements of a
// ragged last row (n % EPR) are stored directly.  Same arithmetic as
// dequant_vec_kernel (blockquant.py:363-376).
template <int OUT>
struct DqTma {
  static constexpr int OB = OUT == DT_F32 ? 4 : 2;  // output bytes per element
  static constexpr int EPR = 128 / OB;               // elements per staged 128-byte row
  static constexpr int kChunk = 1024;                // elements per warp chunk
  static constexpr int kBoxRows = kChunk / EPR;
  static constexpr int kBuf = kChunk * OB;           // bytes per staging buffer
  static constexpr int kWarpsPerCta = 8;
  static constexpr int kSmem = kWarpsPerCta * 2 * kBuf;
#ifndef F46_DQ_U
#define F46_DQ_U 2
#endif
  static constexpr int kU = F46_DQ_U;                  // chunks per warp pass
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_q() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read_q() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all_q() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem_q() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void sts128_q(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// the scale byte of flat block b
template <int SL>
__device__ __forceinline__ uint32_t dq_scale(const uint8_t* __restrict__ scales, int64_t b, int64_t nb,
                                             int64_t kb4, bool small) {
  if (SL != F46_SCALES_TC) return __ldg(scales + b);
  const int64_t row = small ? (int64_t)((uint32_t)b / (uint32_t)nb) : b / nb;
  return __ldg(scales + sf_tc_offset(row, b - row * nb, kb4));
}

#ifndef F46_DQ_MINB
#define F46_DQ_MINB 3
#endif
// (vals * alpha) * scale in float64 as blockquant.py:376, one rounding to the
// output type (bf16: round-to-odd f32 first).  Only for an alpha that is not a
// float32 (an explicit override); kept out of line so its float64 temporaries do
// not set the register budget of the common path.
template <int OUT>
__device__ __noinline__ float2 dq_f64_pair(float2 vd, double alpha_d) {
  const double p0 = __dmul_rn((double)vd.x, alpha_d), p1 = __dmul_rn((double)vd.y, alpha_d);
  if constexpr (OUT == DT_F32) {
    return make_float2(__double2float_rn(p0), __double2float_rn(p1));
  } else {
    const float r0 = __double2float_rz(p0), r1 = __double2float_rz(p1);
    return make_float2(__uint_as_float(__float_as_uint(r0) | ((double)r0 != p0 ? 1u : 0u)),
                       __uint_as_float(__float_as_uint(r1) | ((double)r1 != p1 ? 1u : 0u)));
  }
}

// Shape constants of one K3 launch, prepared on the host.  The flat block index
// b -> (row, kb) division uses a multiply-high by a precomputed magic number
// (round-up method) when every block index fits 32 bits.
struct DqArgs {
  int64_t rows, cols, n, nb, kb4;
  uint32_t magic, sh1, sh2;  // row = (t + ((b - t) >> sh1)) >> sh2, t = umulhi(b, magic)
  int fast32;                // block indices and scale offsets fit 32 bits
  int pair16;                // the lane's two scale bytes are adjacent and 2-byte aligned
};

// The two scale bytes of flat blocks b0, b0 + 1 (b0 even).
template <int SL>
__device__ __forceinline__ void dq_scales2(const uint8_t* __restrict__ scales, const DqArgs& a,
                                           int64_t b0, uint32_t& s0, uint32_t& s1) {
  if (SL != F46_SCALES_TC) {
    if (a.pair16) {
      const uint32_t v = __ldg(reinterpret_cast<const uint16_t*>(scales + b0));
      s0 = v & 0xFF;
      s1 = v >> 8;
    } else {
      s0 = __ldg(scales + b0);
      s1 = __ldg(scales + b0 + 1);
    }
    return;
  }
  if (a.fast32) {
    const uint32_t b = (uint32_t)b0, t = __umulhi(b, a.magic);
    const uint32_t r = (t + ((b - t) >> a.sh1)) >> a.sh2;
    const uint32_t kb = b - r * (uint32_t)a.nb;
    const uint32_t off = ((r >> 7) * (uint32_t)a.kb4 + (kb >> 2)) * 512 + (r & 31) * 16 +
                         ((r & 127) >> 5) * 4 + (kb & 3);
    if (a.pair16) {  // nb even: b0, b0 + 1 share the row and the 4-byte scale group
      const uint32_t v = __ldg(reinterpret_cast<const uint16_t*>(scales + off));
      s0 = v & 0xFF;
      s1 = v >> 8;
      return;
    }
    s0 = __ldg(scales + off);
  } else {
    s0 = dq_scale<SL>(scales, b0, a.nb, a.kb4, false);
  }
  s1 = dq_scale<SL>(scales, b0 + 1, a.nb, a.kb4, false);
}

// Alpha handling of one K3 launch, decided once per CTA from the device alpha:
//  DQ_DIRECT  f32 alpha and one f32 rounding is the answer: f32 output always;
//             bf16 output when no value can double-round (dq_bf16_direct_ok)
//  DQ_ODD     f32 alpha, bf16 output through a round-to-odd f32 product
//  DQ_F64     alpha not a float32 (explicit override): float64 product
enum { DQ_DIRECT = 0, DQ_ODD = 1, DQ_F64 = 2 };

// bf16(RN32(p * alpha)) == RN_bf16(p * alpha) for every decoded value p =
// fp4 * scale when RN32 never lands on a bf16 midpoint from off it.  p has at
// most 6 significant bits (2 from the FP4 value, 4 from the E4M3 scale), so
// p = m * 2^k with m odd <= 45 < 64, and while p * alpha stays a normal float
// the property of m * alpha decides it for every k.  One lane per odd m.
__device__ __forceinline__ bool dq_bf16_direct_ok(float alpha) {
  const int lane = threadIdx.x & 31;
  const float m = (float)(2 * lane + 1);
  const float y = __fmul_rn(m, alpha);
  const bool bad = (__float_as_uint(y) & 0xFFFFu) == 0x8000u && (double)y != (double)m * (double)alpha;
  // smallest nonzero |p| is 0.5 * 2^-9; largest 6 * 448
  const bool range = alpha >= 0x1p-115f && alpha <= 0x1p+114f;
  return !__any_sync(0xFFFFFFFFu, bad) && range;
}

template <int OUT, int SL, int AM>
__device__ __forceinline__ void dq_tma_body(const CUtensorMap* tmap_out, const uint8_t* __restrict__ codes,
                                            const uint8_t* __restrict__ scales, double alpha_d,
                                            const DqArgs& a, void* out, uint32_t* d_flags) {
  using C = DqTma<OUT>;
  extern __shared__ __align__(1024) uint8_t dq_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t nch = (n + C::kChunk - 1) / C::kChunk;
  const int64_t ntma = (n / C::EPR) * C::EPR;  // elements the tensor map covers
  const float alpha = (float)alpha_d;
  const float2 a2 = make_float2(alpha, alpha);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(dq_smem) + (uint32_t)warp * 2 * C::kBuf;
  const int64_t G = (int64_t)gridDim.x * C::kWarpsPerCta;
  bool nan_scale = false;

  // lane's 32 codes (two blocks) and their two scale bytes for chunk ch
  auto load = [&](int64_t ch, uint4& cw, uint32_t& s0, uint32_t& s1) {
    const int64_t e0 = ch * C::kChunk + lane * 32;
    cw = make_uint4(0, 0, 0, 0);
    s0 = s1 = 0x38;  // 1.0: harmless for padding lanes
    if (e0 + 32 <= n) {
      cw = __ldg(reinterpret_cast<const uint4*>(codes + (e0 >> 1)));
      dq_scales2<SL>(scales, a, e0 >> 4, s0, s1);
    } else if (e0 < n) {  // n % 16 == 0: exactly one valid block
      const uint2 h = __ldg(reinterpret_cast<const uint2*>(codes + (e0 >> 1)));
      cw.x = h.x;
      cw.y = h.y;
      s0 = dq_scale<SL>(scales, e0 >> 4, a.nb, a.kb4, false);
    }
  };

  // a warp takes kU consecutive chunks per pass, all their loads in flight first
  constexpr int kU = C::kU;
  const int64_t nsup = (nch + kU - 1) / kU;
  int it = 0;
  for (int64_t sup = blockIdx.x * (int64_t)C::kWarpsPerCta + warp; sup < nsup; sup += G) {
    uint4 cwv[kU];
    uint32_t s0v[kU], s1v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) load(sup * kU + u, cwv[u], s0v[u], s1v[u]);
#pragma unroll 1
    for (int u = 0; u < kU; ++u, ++it) {
      const int64_t ch = sup * kU + u;
      if (ch >= nch) break;
      // always consume slot 0, then rotate (keeps the body compiled once without
      // dynamically indexing the register arrays)
      const uint4 cw = cwv[0];
      const uint32_t s0 = s0v[0], s1 = s1v[0];
#pragma unroll
      for (int v = 0; v + 1 < kU; ++v) {
        cwv[v] = cwv[v + 1];
        s0v[v] = s0v[v + 1];
        s1v[v] = s1v[v + 1];
      }
      const int64_t e0 = ch * C::kChunk + lane * 32;
      const bool valid0 = e0 < n, valid1 = e0 + 16 < n;
      nan_scale |= (valid0 && (s0 & 0x7F) == 0x7F) || (valid1 && (s1 & 0x7F) == 0x7F);
      uint32_t o[32 * C::OB / 4];  // the lane's output bytes as words
#pragma unroll
      for (int blk = 0; blk < 2; ++blk) {
        const uint32_t sc = blk ? s1 : s0;
        const float delta = e4m3_to_f32(sc & 0x7F) * ((sc & 0x80) ? -1.f : 1.f);
        const float2 d2 = make_float2(delta, delta);
#pragma unroll
        for (int wi = 0; wi < 2; ++wi) {
          const uint32_t w = blk ? (wi ? cw.w : cw.z) : (wi ? cw.y : cw.x);
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) {
            uint32_t h;
            switch (pp) {
              case 0: { const __half2 q = e2m1x2_to_h2<0>(w); h = *reinterpret_cast<const uint32_t*>(&q); } break;
              case 1: { const __half2 q = e2m1x2_to_h2<1>(w); h = *reinterpret_cast<const uint32_t*>(&q); } break;
              case 2: { const __half2 q = e2m1x2_to_h2<2>(w); h = *reinterpret_cast<const uint32_t*>(&q); } break;
              default: { const __half2 q = e2m1x2_to_h2<3>(w); h = *reinterpret_cast<const uint32_t*>(&q); } break;
            }
            const float2 vd = __fmul2_rn(make_float2(fhadd_h<0>(h, -0.f), fhadd_h<1>(h, -0.f)), d2);
            float y0, y1;
            if constexpr (AM == DQ_F64) {
              const float2 r = dq_f64_pair<OUT>(vd, alpha_d);
              y0 = r.x;
              y1 = r.y;
            } else if constexpr (AM == DQ_DIRECT) {
              const float2 r = __fmul2_rn(vd, a2);
              y0 = r.x;
              y1 = r.y;
            } else {
              // round-to-odd to f32, then RN to bf16 == one rounding of the exact product
              const float r0 = __fmul_rz(vd.x, alpha), r1 = __fmul_rz(vd.y, alpha);
              y0 = __uint_as_float(__float_as_uint(r0) | (fmaf(vd.x, alpha, -r0) != 0.f ? 1u : 0u));
              y1 = __uint_as_float(__float_as_uint(r1) | (fmaf(vd.y, alpha, -r1) != 0.f ? 1u : 0u));
            }
            const int e = blk * 16 + wi * 8 + pp * 2;  // element index within the lane's 32
            if constexpr (OUT == DT_F32) {
              o[e] = __float_as_uint(y0);
              o[e + 1] = __float_as_uint(y1);
            } else {
              const __nv_bfloat162 hb = __floats2bfloat162_rn(y0, y1);
              o[e >> 1] = *reinterpret_cast<const uint32_t*>(&hb);
            }
          }
        }
      }
      // staging buffer `it & 1` was last read by the store committed two chunks ago
      const uint32_t buf = sbase + (uint32_t)(it & 1) * C::kBuf;
      if (lane == 0) bulk_wait_read_q<1>();
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 32 * C::OB / 16; ++c) {
        // 16-byte chunk c of the lane's bytes -> staged row r, logical chunk lc
        const int r = OUT == DT_F32 ? lane : (lane >> 1);
        const int lc = OUT == DT_F32 ? c : ((lane & 1) * 4 + c);
        sts128_q(buf + r * 128 + ((lc ^ (r & 7)) << 4), o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
      }
      fence_async_smem_q();
      __syncwarp();
      if (lane == 0 && ch * C::kChunk < ntma) {
        tma_store_2d(tmap_out, buf, 0, (int)(ch * C::kBoxRows));
        bulk_commit_q();
      }
      // elements past the tensor map (a ragged last 128-byte row) go out directly
      if (e0 + 32 > ntma && e0 < n) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int64_t e = e0 + i;
          if (e >= ntma && e < n) {
            if constexpr (OUT == DT_F32)
              reinterpret_cast<uint32_t*>(out)[e] = o[i];
            else
              reinterpret_cast<uint16_t*>(out)[e] = (uint16_t)(o[i >> 1] >> (16 * (i & 1)));
          }
        }
      }
    }
  }
  if (lane == 0) bulk_wait_all_q();
  if (nan_scale && d_flags) atomicOr(d_flags, F46_FLAG_NAN_SCALE);
}

template <int OUT, int SL>
__global__ void __launch_bounds__(256, F46_DQ_MINB) dequant_tma_kernel(const __grid_constant__ CUtensorMap tmap_out,
                                                          const uint8_t* __restrict__ codes,
                                                          const uint8_t* __restrict__ scales,
                                                          const double* d_alpha, const DqArgs a,
                                                          void* out, uint32_t* d_flags) {
  const double alpha_d = *d_alpha;
  if ((double)(float)alpha_d != alpha_d) {
    dq_tma_body<OUT, SL, DQ_F64>(&tmap_out, codes, scales, alpha_d, a, out, d_flags);
  } else if (OUT == DT_F32 || dq_bf16_direct_ok((float)alpha_d)) {
    dq_tma_body<OUT, SL, DQ_DIRECT>(&tmap_out, codes, scales, alpha_d, a, out, d_flags);
  } else {
    dq_tma_body<OUT, SL, (OUT == DT_F32 ? DQ_DIRECT : DQ_ODD)>(&tmap_out, codes, scales, alpha_d, a, out,
                                                               d_flags);
  }
}

// ---------------------------------------------------------------------------
// Host helpers
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int launch_status() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "[fouroversix] CUDA error: %s\n", cudaGetErrorString(e));
    return F46_ERR_CUDA;
  }
  return F46_OK;
}

template <int DT, int MODE, bool EXTRA, bool PAR>
int launch_quant_seg_kernel(const QParams& p, cudaStream_t s, int smem, int ctas_per_sm, int groups = 1);

template <int DT, int MODE, bool EXTRA>
int launch_quant_seg(const QParams& p, cudaStream_t s, int groups = 1) {
  constexpr int kTileBytes = kSegElems * ((DT == DT_BF16) ? 2 : 4);
  const int smem = kWarps * kStages * kTileBytes;
  const int ctas_per_sm =
      f46rt::configure((const void*)quant_seg_kernel<DT, MODE, EXTRA>, smem, kWarps * 32);
  if constexpr (!EXTRA && F46_PAR_RESOLVE) {
    // small tensors: the instantiation whose end-of-range deferred blocks are
    // resolved 16 lanes per block (its hot loop spills; large tensors keep the
    // serial resolver)
    if (groups == 1 && p.rows * p.cols * ((DT == DT_BF16) ? 2 : 4) <= kParResolveMaxBytes) {
      const int cps = f46rt::configure((const void*)quant_seg_kernel<DT, MODE, false, true>, smem, kWarps * 32);
      return launch_quant_seg_kernel<DT, MODE, false, true>(p, s, smem, cps);
    }
  }
  return launch_quant_seg_kernel<DT, MODE, EXTRA, false>(p, s, smem, ctas_per_sm, groups);
}

template <int DT, int MODE, bool EXTRA, bool PAR>
int launch_quant_seg_kernel(const QParams& p, cudaStream_t s, int smem, int ctas_per_sm, int groups) {
  QParams pm = p;
  udiv_magic((uint32_t)std::max<int64_t>(1, p.cols >> 4), &pm.nb_magic, &pm.nb_sh1, &pm.nb_sh2);
  // The kernel keeps 32-bit byte offsets: launch at most 2^31 input bytes at a
  // time, in whole 128-row slabs so each launch owns complete scale atoms.
  constexpr int64_t kEsz = (DT == DT_BF16) ? 2 : 4;
  const int64_t nb = p.cols >> 4, kb4 = (nb + 3) >> 2;
  int64_t chunk_bytes = (int64_t)1 << 31;
  const int64_t hook_bytes = f46rt::hook(f46rt::HOOK_SEG_CHUNK_BYTES);  // test hook: force multi-launch
  if (hook_bytes > 0 && hook_bytes < chunk_bytes) chunk_bytes = hook_bytes;
  int64_t rows_max = (chunk_bytes / (p.cols * kEsz)) & ~(int64_t)127;
  if (rows_max < 128) return F46_ERR_UNSUPPORTED;
  if (groups > 1) {  // one launch, group = blockIdx.y; each group within one slab
    if (p.rows > rows_max) return F46_ERR_UNSUPPORTED;
    const int64_t tiles = p.rows * ((p.cols + kSegElems - 1) / kSegElems);
    int64_t grid = ((int64_t)num_sms() * ctas_per_sm + groups - 1) / groups;
    grid = std::min(grid, (tiles + kWarps - 1) / kWarps);
    if (grid < 1) grid = 1;
    quant_seg_kernel<DT, MODE, EXTRA, PAR><<<dim3((unsigned)grid, (unsigned)groups), kWarps * 32, smem, s>>>(pm);
    return launch_status();
  }
  for (int64_t r0 = 0; r0 < p.rows; r0 += rows_max) {
    QParams q = pm;
    q.rows = std::min(rows_max, p.rows - r0);
    q.x = reinterpret_cast<const uint8_t*>(p.x) + r0 * p.cols * kEsz;
    q.codes = p.codes + r0 * nb * 8;
    q.scales_tc = p.scales_tc + (r0 / 128) * kb4 * 512;
    if (p.scales_rm) q.scales_rm = p.scales_rm + r0 * nb;
    if (p.pick4) q.pick4 = p.pick4 + r0 * nb;
    const int64_t tiles = q.rows * ((q.cols + kSegElems - 1) / kSegElems);
    int64_t grid = (tiles + kWarps - 1) / kWarps;
    if (grid > (int64_t)num_sms() * ctas_per_sm) grid = (int64_t)num_sms() * ctas_per_sm;
    if (grid < 1) grid = 1;
    quant_seg_kernel<DT, MODE, EXTRA, PAR><<<(unsigned)grid, kWarps * 32, smem, s>>>(q);
  }
  return launch_status();
}

template <int DT, int MODE>
int launch_quant_generic(const QParams& p, cudaStream_t s, int groups = 1) {
  const int64_t nb = (p.cols + 15) >> 4;
  const int64_t total = ((p.rows + 127) & ~(int64_t)127) * (((nb + 3) >> 2) * 4);
  int64_t grid = (total + 255) / 256;
  const int64_t cap = std::max<int64_t>(1, (int64_t)num_sms() * 8 / groups);
  if (grid > cap) grid = cap;
  quant_generic_kernel<DT, MODE><<<dim3((unsigned)grid, (unsigned)groups), 256, 0, s>>>(p);
  return launch_status();
}

template <int DT, int MODE>
int launch_quant(const QParams& p, cudaStream_t s, bool tma, int groups = 1) {
  if (!tma) return launch_quant_generic<DT, MODE>(p, s, groups);
  // parity views (row-major scales, 4/6 choice) get their own instantiation
  return (p.scales_rm || p.pick4) ? launch_quant_seg<DT, MODE, true>(p, s, groups)
                                  : launch_quant_seg<DT, MODE, false>(p, s, groups);
}

template <int DT>
int dispatch_mode(const QParams& p, cudaStream_t s, bool tma, int groups = 1) {
  switch (p.mode) {
    case F46_FIXED6:
      return launch_quant<DT, FIXED6>(p, s, tma, groups);
    case F46_FIXED4:
      return launch_quant<DT, FIXED4>(p, s, tma, groups);
    default:
      return launch_quant<DT, ADAPTIVE>(p, s, tma, groups);
  }
}

template <int OUT, int SL>
int launch_dequant_tma_t(const CUtensorMap& map, const uint8_t* codes, const uint8_t* scales,
                         const double* d_alpha, const DqArgs& a, void* out, uint32_t* d_flags,
                         cudaStream_t s) {
  using C = DqTma<OUT>;
  const int ctas_per_sm =
      f46rt::configure((const void*)dequant_tma_kernel<OUT, SL>, C::kSmem, C::kWarpsPerCta * 32);
  const int64_t nsup = (a.n + (int64_t)C::kChunk * C::kU - 1) / ((int64_t)C::kChunk * C::kU);
  int64_t grid = (nsup + C::kWarpsPerCta - 1) / C::kWarpsPerCta;
  const int64_t cap = (int64_t)num_sms() * ctas_per_sm;
  if (grid > cap) grid = cap;
  dequant_tma_kernel<OUT, SL><<<(unsigned)grid, C::kWarpsPerCta * 32, C::kSmem, s>>>(
      map, codes, scales, d_alpha, a, out, d_flags);
  return launch_status();
}

// Unsigned 32-bit division by d via multiply-high (round-up method):
// q = (t + ((x - t) >> sh1)) >> sh2 with t = umulhi(x, magic), exact for all x < 2^32.
void udiv_magic(uint32_t d, uint32_t* magic, uint32_t* sh1, uint32_t* sh2) {
  int l = 0;
  while (l < 32 && (1ull << l) < d) ++l;  // l = ceil(log2 d)
  *magic = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  *sh1 = l < 1 ? l : 1;
  *sh2 = l > 1 ? l - 1 : 0;
}

// F46_ERR_UNSUPPORTED when the output cannot be described by a tensor map
int launch_dequant_tma(const uint8_t* codes, const uint8_t* scales, bool tc, const double* d_alpha,
                       int64_t rows, int64_t cols, void* out, int out_dtype, uint32_t* d_flags,
                       cudaStream_t s) {
  EncodeTiledFn fn = get_encode_fn();
  const bool f32 = out_dtype == F46_DT_F32;
  const int epr = f32 ? DqTma<DT_F32>::EPR : DqTma<DT_BF16>::EPR;
  const int box_rows = f32 ? DqTma<DT_F32>::kBoxRows : DqTma<DT_BF16>::kBoxRows;
  const int64_t trows = rows * cols / epr;
  if (!fn || trows < 1 || trows > 0x7FFFFFFFll) return F46_ERR_UNSUPPORTED;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)epr, (cuuint64_t)trows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {(cuuint32_t)epr, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  if (fn(&map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out,
         dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return F46_ERR_UNSUPPORTED;
  DqArgs a;
  a.rows = rows;
  a.cols = cols;
  a.n = rows * cols;
  a.nb = cols >> 4;
  a.kb4 = (a.nb + 3) >> 2;
  udiv_magic((uint32_t)std::min<int64_t>(a.nb, 0xFFFFFFFFll), &a.magic, &a.sh1, &a.sh2);
  const int64_t sf_bytes = ((rows + 127) / 128) * a.kb4 * 512;
  a.fast32 = rows * a.nb < (1ll << 32) && sf_bytes < (1ll << 32) && a.nb < (1ll << 32);
  a.pair16 = (((uintptr_t)scales) & 1) == 0 && (!tc || a.nb % 2 == 0);
  if (f32)
    return tc ? launch_dequant_tma_t<DT_F32, F46_SCALES_TC>(map, codes, scales, d_alpha, a, out, d_flags, s)
              : launch_dequant_tma_t<DT_F32, F46_SCALES_RM>(map, codes, scales, d_alpha, a, out, d_flags, s);
  return tc ? launch_dequant_tma_t<DT_BF16, F46_SCALES_TC>(map, codes, scales, d_alpha, a, out, d_flags, s)
            : launch_dequant_tma_t<DT_BF16, F46_SCALES_RM>(map, codes, scales, d_alpha, a, out, d_flags, s);
}

}  // namespace

namespace f46rt {
namespace {
std::atomic<int64_t> g_hooks[HOOK_COUNT];
}
int64_t hook(int h) { return (h >= 0 && h < HOOK_COUNT) ? g_hooks[h].load(std::memory_order_relaxed) : 0; }
}  // namespace f46rt

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

int f46_set_test_hook(int hook, int64_t value) {
  if (hook < 0 || hook >= f46rt::HOOK_COUNT) return F46_ERR_INVALID_ARG;
  f46rt::g_hooks[hook].store(value, std::memory_order_relaxed);
  return F46_OK;
}

size_t f46_scales_tc_bytes(int64_t rows, int64_t cols) {
  const int64_t nb = (cols + 15) / 16;
  return (size_t)(((rows + 127) / 128) * ((nb + 3) / 4) * 512);
}

size_t f46_codes_bytes(int64_t rows, int64_t cols) {
  return (size_t)(rows * ((cols + 15) / 16) * 8);
}

int f46_amax(const void* x, int dtype, int64_t n, double* d_amax, f46_stream_t stream) {
  if (!x || !d_amax || n < 0) return F46_ERR_INVALID_ARG;
  if (n == 0) return F46_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // >= 16 vectors of 16 bytes per thread: small tensors get fewer CTAs and so
  // fewer same-address atomics at the tail; large ones the full 8 CTAs per SM
  const int64_t per = dtype == F46_DT_BF16 ? 256 * 8 * 16 : 256 * 4 * 16;
  int64_t grid = (n + per - 1) / per;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  switch (dtype) {
    case F46_DT_BF16:
      amax_kernel<DT_BF16><<<(unsigned)grid, 256, 0, s>>>(x, n, d_amax);
      break;
    case F46_DT_F32:
      amax_kernel<DT_F32><<<(unsigned)grid, 256, 0, s>>>(x, n, d_amax);
      break;
    case F46_DT_F64:
      amax_kernel<DT_F64><<<(unsigned)grid, 256, 0, s>>>(x, n, d_amax);
      break;
    default:
      return F46_ERR_INVALID_ARG;
  }
  return launch_status();
}

int f46_quantize(const void* x, int dtype, int64_t rows, int64_t cols, int mode, int rule,
                 double mcap, const double* d_amax, double alpha_override, uint8_t* codes,
                 uint8_t* scales_tc, uint8_t* scales_rm, uint8_t* pick4, double* d_alpha_out,
                 uint32_t* d_flags, f46_stream_t stream) {
  if (!x || !codes || !scales_tc || rows <= 0 || cols <= 0) return F46_ERR_INVALID_ARG;
  if (mode < F46_FIXED6 || mode > F46_ADAPTIVE || rule < F46_RULE_MSE || rule > F46_RULE_ABSMAX)
    return F46_ERR_CONFIG;
  if (alpha_override <= 0.0 && (!d_amax || !(mcap > 0.0))) return F46_ERR_INVALID_ARG;
  if (alpha_override > 0.0 && !(alpha_override <= 1.7976931348623157e308))
    return F46_ERR_INVALID_ARG;
  QParams p{x, rows, cols, mode, rule, dtype, mcap, d_amax, alpha_override, codes, scales_tc,
            scales_rm, pick4, d_alpha_out, d_flags};
  cudaStream_t s = (cudaStream_t)stream;
  // segment kernel: 16-element blocks never straddle rows, 16-byte aligned rows
  const bool tma = (dtype != F46_DT_F64) && (cols % 16 == 0) && (((uintptr_t)x & 15) == 0) &&
                   (((uintptr_t)codes & 7) == 0) &&
                   rows < (1ll << 31) && cols < (1ll << 31) && rows * ((cols + 15) / 16) < (1ll << 32);
  switch (dtype) {
    case F46_DT_BF16: {
      int rc = dispatch_mode<DT_BF16>(p, s, tma);
      if (rc == F46_ERR_UNSUPPORTED && tma) rc = dispatch_mode<DT_BF16>(p, s, false);
      return rc;
    }
    case F46_DT_F32: {
      int rc = dispatch_mode<DT_F32>(p, s, tma);
      if (rc == F46_ERR_UNSUPPORTED && tma) rc = dispatch_mode<DT_F32>(p, s, false);
      return rc;
    }
    case F46_DT_F64:
      return dispatch_mode<DT_F64>(p, s, false);
    default:
      return F46_ERR_INVALID_ARG;
  }
}

int f46_quantize_fused(const void* x, int dtype, int64_t rows, int64_t cols, int mode, int rule,
                       double mcap, double* d_work, uint8_t* codes, uint8_t* scales_tc,
                       double* d_alpha_out, uint32_t* d_flags, f46_stream_t stream) {
  if (!x || !codes || !scales_tc || !d_work || rows <= 0 || cols <= 0 || !(mcap > 0.0))
    return F46_ERR_INVALID_ARG;
  if (mode < F46_FIXED6 || mode > F46_ADAPTIVE || rule < F46_RULE_MSE || rule > F46_RULE_ABSMAX)
    return F46_ERR_CONFIG;
  if (dtype != F46_DT_BF16 && dtype != F46_DT_F32) return F46_ERR_UNSUPPORTED;
  const int64_t esz = dtype == F46_DT_BF16 ? 2 : 4;
  if (cols % 16 || ((uintptr_t)x & 15) || ((uintptr_t)codes & 7) || rows * cols * esz >= (1ll << 31))
    return F46_ERR_UNSUPPORTED;
  QParams p{x, rows, cols, mode, rule, dtype, mcap, d_work, 0.0, codes, scales_tc, nullptr,
            nullptr, d_alpha_out, d_flags};
  udiv_magic((uint32_t)std::max<int64_t>(1, cols >> 4), &p.nb_magic, &p.nb_sh1, &p.nb_sh2);
  p.d_sync = reinterpret_cast<uint32_t*>(d_work + 1);
  cudaStream_t s = (cudaStream_t)stream;
  auto launch = [&](const void* kernel, int smem) -> int {
    const int per_sm = f46rt::configure(kernel, smem, kWarps * 32);
    const int64_t tiles = rows * ((cols + kSegElems - 1) / kSegElems);
    int64_t grid = std::min<int64_t>((tiles + kWarps - 1) / kWarps, (int64_t)num_sms() * per_sm);
    if (grid < 1) grid = 1;
    void* args[] = {&p};
    const cudaError_t e = cudaLaunchCooperativeKernel(kernel, dim3((unsigned)grid), dim3(kWarps * 32),
                                                      args, (size_t)smem, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return F46_ERR_UNSUPPORTED;
    }
    return F46_OK;
  };
  const int smem_bf16 = kWarps * kStages * kSegElems * 2, smem_f32 = kWarps * kStages * kSegElems * 4;
#define F46_FUSED(DTV, MV, SMEM) launch((const void*)quant_seg_kernel<DTV, MV, false, F46_PAR_RESOLVE != 0>, SMEM)
  if (dtype == F46_DT_BF16) {
    switch (mode) {
      case F46_FIXED6: return F46_FUSED(DT_BF16, FIXED6, smem_bf16);
      case F46_FIXED4: return F46_FUSED(DT_BF16, FIXED4, smem_bf16);
      default: return F46_FUSED(DT_BF16, ADAPTIVE, smem_bf16);
    }
  }
  switch (mode) {
    case F46_FIXED6: return F46_FUSED(DT_F32, FIXED6, smem_f32);
    case F46_FIXED4: return F46_FUSED(DT_F32, FIXED4, smem_f32);
    default: return F46_FUSED(DT_F32, ADAPTIVE, smem_f32);
  }
#undef F46_FUSED
}

int f46_amax_grouped(const void* x, int dtype, int groups, int64_t n, double* d_amax,
                     f46_stream_t stream) {
  if (!x || !d_amax || n < 0 || groups < 1 || groups > 65535) return F46_ERR_INVALID_ARG;
  if (n == 0) return F46_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t per = dtype == F46_DT_BF16 ? 256 * 8 * 16 : 256 * 4 * 16;
  int64_t gx = (n + per - 1) / per;
  gx = std::min<int64_t>(gx, std::max<int64_t>(1, (int64_t)num_sms() * 8 / groups));
  const dim3 grid((unsigned)std::max<int64_t>(gx, 1), (unsigned)groups);
  switch (dtype) {
    case F46_DT_BF16:
      amax_kernel<DT_BF16><<<grid, 256, 0, s>>>(x, n, d_amax);
      break;
    case F46_DT_F32:
      amax_kernel<DT_F32><<<grid, 256, 0, s>>>(x, n, d_amax);
      break;
    case F46_DT_F64:
      amax_kernel<DT_F64><<<grid, 256, 0, s>>>(x, n, d_amax);
      break;
    default:
      return F46_ERR_INVALID_ARG;
  }
  return launch_status();
}

int f46_quantize_grouped(const void* x, int dtype, int groups, int64_t rows, int64_t cols, int mode,
                         int rule, double mcap, const double* d_amax, uint8_t* codes,
                         uint8_t* scales_tc, double* d_alpha_out, uint32_t* d_flags,
                         f46_stream_t stream) {
  if (!x || !codes || !scales_tc || !d_amax || rows <= 0 || cols <= 0 || groups < 1 ||
      groups > 65535 || !(mcap > 0.0))
    return F46_ERR_INVALID_ARG;
  if (mode < F46_FIXED6 || mode > F46_ADAPTIVE || rule < F46_RULE_MSE || rule > F46_RULE_ABSMAX)
    return F46_ERR_CONFIG;
  if (dtype != F46_DT_BF16 && dtype != F46_DT_F32 && dtype != F46_DT_F64) return F46_ERR_INVALID_ARG;
  const int64_t esz = dtype == F46_DT_BF16 ? 2 : (dtype == F46_DT_F32 ? 4 : 8);
  QParams p{x, rows, cols, mode, rule, dtype, mcap, d_amax, 0.0, codes, scales_tc, nullptr,
            nullptr, d_alpha_out, d_flags, rows * cols * esz, (int64_t)f46_codes_bytes(rows, cols),
            (int64_t)f46_scales_tc_bytes(rows, cols)};
  cudaStream_t s = (cudaStream_t)stream;
  // every group's base must satisfy the segment kernel's alignment as well
  const bool tma = (dtype != F46_DT_F64) && (cols % 16 == 0) && (((uintptr_t)x & 15) == 0) &&
                   ((p.g_x & 15) == 0) && (((uintptr_t)codes & 7) == 0) &&
                   rows < (1ll << 31) && cols < (1ll << 31) && rows * ((cols + 15) / 16) < (1ll << 32);
  int rc;
  switch (dtype) {
    case F46_DT_BF16:
      rc = dispatch_mode<DT_BF16>(p, s, tma, groups);
      if (rc == F46_ERR_UNSUPPORTED && tma) rc = dispatch_mode<DT_BF16>(p, s, false, groups);
      return rc;
    case F46_DT_F32:
      rc = dispatch_mode<DT_F32>(p, s, tma, groups);
      if (rc == F46_ERR_UNSUPPORTED && tma) rc = dispatch_mode<DT_F32>(p, s, false, groups);
      return rc;
    default:
      return dispatch_mode<DT_F64>(p, s, false, groups);
  }
}

int f46_quantize_2d_grouped(const void* w, int dtype, int groups, int64_t R, int64_t C, int mode,
                            int rule, double mcap, const double* d_amax, uint8_t* codes,
                            uint8_t* scales_tc, uint8_t* codes_t, uint8_t* scales_tc_t,
                            double* d_alpha_out, uint32_t* d_flags, f46_stream_t stream) {
  if (!w || !codes || !scales_tc || !d_amax || R <= 0 || C <= 0 || groups < 1 || groups > 65535 ||
      !(mcap > 0.0))
    return F46_ERR_INVALID_ARG;
  if (mode < F46_FIXED6 || mode > F46_ADAPTIVE || rule < F46_RULE_MSE || rule > F46_RULE_ABSMAX)
    return F46_ERR_CONFIG;
  if (dtype != F46_DT_F32 && dtype != F46_DT_BF16) return F46_ERR_INVALID_ARG;
  if ((codes_t == nullptr) != (scales_tc_t == nullptr)) return F46_ERR_INVALID_ARG;
  const int64_t esz = dtype == F46_DT_BF16 ? 2 : 4;
  Q2Params p{w, R, C, mode, rule, dtype, mcap, d_amax, 0.0, codes, scales_tc, nullptr, nullptr,
             codes_t, scales_tc_t, d_alpha_out, d_flags, R * C * esz,
             (int64_t)f46_codes_bytes(R, C), (int64_t)f46_scales_tc_bytes(R, C),
             (int64_t)f46_codes_bytes(C, R), (int64_t)f46_scales_tc_bytes(C, R)};
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t tiles = ((R + 15) / 16) * ((C + 15) / 16);
  // per group, tile indices and scale offsets stay in 32 bits (quant2d_v2_kernel)
  if (tiles >= (1LL << 31) || R * ((C + 15) / 16) >= (1LL << 31) || C * ((R + 15) / 16) >= (1LL << 31))
    return F46_ERR_UNSUPPORTED;
  int64_t g2 = (tiles + 15) / 16;  // 8 warps x 2 tiles per CTA
  g2 = std::min<int64_t>(g2, std::max<int64_t>(1, (int64_t)num_sms() * 8 / groups));
  if (rule == F46_RULE_MSE)
    quant2d_v2_kernel<true><<<dim3((unsigned)std::max<int64_t>(g2, 1), (unsigned)groups), 256, 0, s>>>(p);
  else
    quant2d_v2_kernel<false><<<dim3((unsigned)std::max<int64_t>(g2, 1), (unsigned)groups), 256, 0, s>>>(p);
  return launch_status();
}

int f46_matmul_f32_ordered(const float* A, const float* B, int64_t M, int64_t N, int64_t K, float* C,
                           f46_stream_t stream) {
  if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0) return F46_ERR_INVALID_ARG;
  if ((N + 31) / 32 > 0x7FFFFFFF || (M + 31) / 32 > 65535) return F46_ERR_UNSUPPORTED;
  const dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32));
  matmul_f32_ordered_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A, B, M, N, K, C);
  return launch_status();
}

int f46_quantize_block_ref(const double* d_x, int64_t n, double alpha, double m,
                           const double* d_u, uint8_t* d_codes, double* d_work, double* d_out,
                           f46_stream_t stream) {
  if (!d_x || !d_codes || !d_work || !d_out || n <= 0) return F46_ERR_INVALID_ARG;
  block_ref_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d_x, n, alpha, m, d_u, d_codes, d_work, d_out);
  return launch_status();
}

int f46_dequantize(const uint8_t* codes, const uint8_t* scales, int scale_layout,
                   const double* d_alpha, int64_t rows, int64_t cols, void* out, int out_dtype,
                   uint32_t* d_flags, f46_stream_t stream) {
  if (!codes || !scales || !d_alpha || !out || rows <= 0 || cols <= 0) return F46_ERR_INVALID_ARG;
  if (scale_layout != F46_SCALES_TC && scale_layout != F46_SCALES_RM) return F46_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t total = rows * ((cols + 15) / 16);
  int64_t grid = (total + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  const bool tc = scale_layout == F46_SCALES_TC;
  // TMA-staged path: f32 / bf16 out, cols % 16 == 0, 16-byte aligned codes and output
  if ((out_dtype == F46_DT_F32 || out_dtype == F46_DT_BF16) && cols % 16 == 0 &&
      (((uintptr_t)out) & 15) == 0 && (((uintptr_t)codes) & 15) == 0 && !f46rt::hook(f46rt::HOOK_DQ_VEC)) {
    const int rc = launch_dequant_tma(codes, scales, tc, d_alpha, rows, cols, out, out_dtype, d_flags, s);
    if (rc != F46_ERR_UNSUPPORTED) return rc;
  }
  // coalesced path: f32 / bf16 out, cols % 16 == 0, 16-byte aligned rows
  if ((out_dtype == F46_DT_F32 || out_dtype == F46_DT_BF16) && cols % 16 == 0 &&
      (((uintptr_t)out) & 15) == 0 && (((uintptr_t)codes) & 3) == 0) {
    const int tpb = out_dtype == F46_DT_F32 ? 4 : 2;
    int64_t g2 = (total * tpb + 255) / 256;
    const int64_t cap2 = (int64_t)num_sms() * 16;
    if (g2 > cap2) g2 = cap2;
#define F46_DQV(OUT, SL) \
  dequant_vec_kernel<OUT, SL><<<(unsigned)g2, 256, 0, s>>>(codes, scales, d_alpha, rows, cols, out, d_flags)
    if (out_dtype == F46_DT_F32) {
      if (tc) F46_DQV(DT_F32, F46_SCALES_TC); else F46_DQV(DT_F32, F46_SCALES_RM);
    } else {
      if (tc) F46_DQV(DT_BF16, F46_SCALES_TC); else F46_DQV(DT_BF16, F46_SCALES_RM);
    }
#undef F46_DQV
    return launch_status();
  }
#define F46_DQ(OUT, SL) \
  dequant_kernel<OUT, SL><<<(unsigned)grid, 256, 0, s>>>(codes, scales, d_alpha, rows, cols, out, d_flags)
  switch (out_dtype) {
    case F46_DT_F32:
      if (tc) F46_DQ(DT_F32, F46_SCALES_TC); else F46_DQ(DT_F32, F46_SCALES_RM);
      break;
    case F46_DT_BF16:
      if (tc) F46_DQ(DT_BF16, F46_SCALES_TC); else F46_DQ(DT_BF16, F46_SCALES_RM);
      break;
    case F46_DT_F64:
      if (tc) F46_DQ(DT_F64, F46_SCALES_TC); else F46_DQ(DT_F64, F46_SCALES_RM);
      break;
    default:
      return F46_ERR_INVALID_ARG;
  }
#undef F46_DQ
  return launch_status();
}

int f46_quantize_2d(const void* w, int dtype, int64_t R, int64_t C, int mode, int rule,
                    double mcap, const double* d_amax, double alpha_override, uint8_t* codes,
                    uint8_t* scales_tc, uint8_t* scales_rm, uint8_t* pick4, uint8_t* codes_t,
                    uint8_t* scales_tc_t, double* d_alpha_out, uint32_t* d_flags,
                    f46_stream_t stream) {
  if (!w || !codes || !scales_tc || R <= 0 || C <= 0) return F46_ERR_INVALID_ARG;
  if (mode < F46_FIXED6 || mode > F46_ADAPTIVE || rule < F46_RULE_MSE || rule > F46_RULE_ABSMAX)
    return F46_ERR_CONFIG;
  if (dtype != F46_DT_F32 && dtype != F46_DT_BF16 && dtype != F46_DT_F64) return F46_ERR_INVALID_ARG;
  if (alpha_override <= 0.0 && (!d_amax || !(mcap > 0.0))) return F46_ERR_INVALID_ARG;
  if ((codes_t == nullptr) != (scales_tc_t == nullptr)) return F46_ERR_INVALID_ARG;
  Q2Params p{w, R, C, mode, rule, dtype, mcap, d_amax, alpha_override, codes, scales_tc,
             scales_rm, pick4, codes_t, scales_tc_t, d_alpha_out, d_flags};
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t tiles = ((R + 15) / 16) * ((C + 15) / 16);
  int64_t grid = (tiles + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  // the v2 kernel keeps tile indices and scale offsets in 32 bits
  const bool fits32 = tiles < (1LL << 31) && R * ((C + 15) / 16) < (1LL << 31) &&
                      C * ((R + 15) / 16) < (1LL << 31);
  if (dtype != F46_DT_F64 && fits32 && !f46rt::hook(f46rt::HOOK_Q2_V1)) {
    int64_t g2 = (tiles + 15) / 16;  // 8 warps x 2 tiles per CTA
    const int64_t cap2 = (int64_t)num_sms() * 8;
    if (g2 > cap2) g2 = cap2;
    if (g2 < 1) g2 = 1;
    if (rule == F46_RULE_MSE)
      quant2d_v2_kernel<true><<<(unsigned)g2, 256, 0, s>>>(p);
    else
      quant2d_v2_kernel<false><<<(unsigned)g2, 256, 0, s>>>(p);
  } else {
    quant2d_kernel<<<(unsigned)grid, 256, 0, s>>>(p);
  }
  return launch_status();
}

int f46_selection_stats(const void* x, int dtype, int64_t rows, int64_t cols, double mcap,
                        const double* d_amax, double alpha_override, double* d_partials,
                        int nparts, double* d_alpha_out, f46_stream_t stream) {
  if (!x || !d_partials || rows <= 0 || cols <= 0 || nparts < 1) return F46_ERR_INVALID_ARG;
  if (alpha_override <= 0.0 && (!d_amax || !(mcap > 0.0))) return F46_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case F46_DT_BF16:
      stats_kernel<DT_BF16><<<nparts, 256, 0, s>>>(x, rows, cols, mcap, d_amax, alpha_override,
                                                   d_partials, d_alpha_out);
      break;
    case F46_DT_F32:
      stats_kernel<DT_F32><<<nparts, 256, 0, s>>>(x, rows, cols, mcap, d_amax, alpha_override,
                                                  d_partials, d_alpha_out);
      break;
    case F46_DT_F64:
      stats_kernel<DT_F64><<<nparts, 256, 0, s>>>(x, rows, cols, mcap, d_amax, alpha_override,
                                                  d_partials, d_alpha_out);
      break;
    default:
      return F46_ERR_INVALID_ARG;
  }
  return launch_status();
}

int f46_quantize_sr(const void* x, int dtype, int64_t rows, int64_t cols, int mode, int rule,
                    double mcap, const double* d_amax, double alpha_override, uint64_t key6_0,
                    uint64_t key6_1, uint64_t key4_0, uint64_t key4_1, uint8_t* codes,
                    uint8_t* scales_tc, uint8_t* scales_rm, uint8_t* pick4, double* d_alpha_out,
                    uint32_t* d_flags, f46_stream_t stream) {
  if (!x || !codes || !scales_tc || rows <= 0 || cols <= 0) return F46_ERR_INVALID_ARG;
  if (mode < F46_FIXED6 || mode > F46_ADAPTIVE || rule < F46_RULE_MSE || rule > F46_RULE_ABSMAX)
    return F46_ERR_CONFIG;
  if (alpha_override <= 0.0 && (!d_amax || !(mcap > 0.0))) return F46_ERR_INVALID_ARG;
  SRParams sp{{x, rows, cols, mode, rule, dtype, mcap, d_amax, alpha_override, codes, scales_tc,
               scales_rm, pick4, d_alpha_out, d_flags},
              key6_0, key6_1, key4_0, key4_1};
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nb = (cols + 15) / 16;
  const int64_t total = ((rows + 127) & ~(int64_t)127) * (((nb + 3) / 4) * 4);
  int64_t grid = (total + 127) / 128;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  const bool quad = !f46rt::hook(f46rt::HOOK_SR_ONE_THREAD);
  int64_t grid4 = (total * 4 + 255) / 256;
  const int64_t cap4 = (int64_t)num_sms() * 8;
  if (grid4 > cap4) grid4 = cap4;
  switch (dtype) {
    case F46_DT_BF16:
      if (quad)
        quant_sr4_kernel<DT_BF16><<<(unsigned)grid4, 256, 0, s>>>(sp);
      else
        quant_sr_kernel<DT_BF16><<<(unsigned)grid, 128, 0, s>>>(sp);
      break;
    case F46_DT_F32:
      if (quad)
        quant_sr4_kernel<DT_F32><<<(unsigned)grid4, 256, 0, s>>>(sp);
      else
        quant_sr_kernel<DT_F32><<<(unsigned)grid, 128, 0, s>>>(sp);
      break;
    case F46_DT_F64:
      quant_sr_kernel<DT_F64><<<(unsigned)grid, 128, 0, s>>>(sp);
      break;
    default:
      return F46_ERR_INVALID_ARG;
  }
  return launch_status();
}

int f46_rht16(const void* x, int dtype, int64_t n, const double* signs16, double* out,
              f46_stream_t stream) {
  if (!x || !signs16 || !out || n <= 0 || n % 16) return F46_ERR_INVALID_ARG;
  const double* g = signs16;
  const double4 s0 = make_double4(g[0], g[1], g[2], g[3]), s1 = make_double4(g[4], g[5], g[6], g[7]);
  const double4 s2 = make_double4(g[8], g[9], g[10], g[11]),
                s3 = make_double4(g[12], g[13], g[14], g[15]);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ng = n / 16;
  int64_t grid = (ng + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  const bool vec = ((((uintptr_t)x) | ((uintptr_t)out)) & 15) == 0;
  switch (dtype) {
    case F46_DT_BF16:
      rht16_kernel<DT_BF16><<<(unsigned)grid, 256, 0, s>>>(x, ng, s0, s1, s2, s3, out, vec);
      break;
    case F46_DT_F32:
      rht16_kernel<DT_F32><<<(unsigned)grid, 256, 0, s>>>(x, ng, s0, s1, s2, s3, out, vec);
      break;
    case F46_DT_F64:
      rht16_kernel<DT_F64><<<(unsigned)grid, 256, 0, s>>>(x, ng, s0, s1, s2, s3, out, vec);
      break;
    default:
      return F46_ERR_INVALID_ARG;
  }
  return launch_status();
}

#define F46_STR2(x) #x
#define F46_STR(x) F46_STR2(x)
const char* f46_build_info(void) {
  return "fouroversix sm_100a (tcgen05/TMA) built with nvcc " F46_STR(__CUDACC_VER_MAJOR__) "." F46_STR(
      __CUDACC_VER_MINOR__) "." F46_STR(__CUDACC_VER_BUILD__) ", host compiler " __VERSION__;
}

}  // extern "C"

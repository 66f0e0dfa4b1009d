// f46_rht.cu -- the WGRAD operand of the 4/6 recipe as one fused pass:
// transpose + 16-wide randomized Hadamard transform along the token axis +
// 4/6 NVFP4 quantization along it (reference qlinear.py:138-159:
// apply_rht(dy.T, spec) then _quantize_1d), grouped over experts.
//
// Input a[g] is a row-major [T][H] activation / gradient (tokens x features).
// The operand is A = RHT_T(a^T): [H][T], 16-blocks along T.  The RHT groups
// of 16 tokens are exactly the quantization blocks, so block (h, k) is
//   y = fwht(signs * a[16k .. 16k+15, h]) / 4      (transforms.py:92-97)
// and depends on one 16-token column segment only.  Two passes (the tensor
// scale needs the global max first, blockquant.py:215-222):
//   rht_t_amax_kernel   max|y| per group (float64 bit pattern, atomicMax)
//   quant_rht_t_kernel  y again, then the block quantizer
// A warp owns 64 features x 64 tokens: lane l holds features 2l, 2l+1, so each
// token row is one coalesced 128-byte load; a lane's consecutive blocks of one
// feature are contiguous code bytes (merged in L2).  y is formed in float64 in numpy's
// butterfly order (bit-exact with the reference); blocks whose 16 values are
// all float32-exact take the f32 fast path of f46_device.cuh (block_sl, exact
// per-nibble tie tests), the rest the float64 restatement (exact_block).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>

#include "../../include/fouroversix.h"
#include "f46_device.cuh"
#include "f46_runtime.h"

using namespace f46;

#ifndef F46_RT_MINB
#define F46_RT_MINB 2
#endif

namespace {

struct RtParams {
  const void* a;  // [T][H] of dtype, per group
  int64_t T, H;
  int dtype, mode, rule;
  double mcap;
  uint32_t negmask;  // bit i set: sign i of the RHT diagonal is -1
  double* d_amax;    // [groups]
  uint8_t* codes;    // [groups][H][T/16*8]
  uint8_t* scales_tc;  // [groups][scales_tc_bytes(H, T)], zero-initialised by the caller
  double* d_alpha_out;  // [groups] (nullable)
  uint32_t* d_flags;    // nullable
  int64_t g_a, g_codes, g_scales;  // per-group strides (bytes)
  float sq[16];  // signs[i] / 4 (exact): the f32 route's per-token factor
};

__device__ __forceinline__ void select_group(RtParams& p) {
  const int64_t g = blockIdx.y;
  p.a = reinterpret_cast<const uint8_t*>(p.a) + g * p.g_a;
  p.codes += g * p.g_codes;
  p.scales_tc += g * p.g_scales;
  p.d_amax += g;
  if (p.d_alpha_out) p.d_alpha_out += g;
}

constexpr int kUnitH = 64;   // features per warp unit (2 per lane)
constexpr int kUnitK = 4;    // 16-token blocks per warp unit

// The 16 tokens of block k for the lane's two features h0, h0+1 (h0 even):
// raw words, bf16 pairs (one coalesced 32-bit load per token row) or two
// floats.  Missing features (h >= H) read as 0.
template <int DT>
struct Col2 {
  uint32_t w[16];  // bf16: feature h0 in the low half; f32: feature h0 only
  uint32_t w1[DT == DT_BF16 ? 1 : 16];  // f32: feature h0 + 1
};

template <int DT>
__device__ __forceinline__ void load_pair(const RtParams& p, int64_t k, int64_t h0, Col2<DT>& c) {
  const int64_t t0 = k * 16;
  if constexpr (DT == DT_BF16) {
    const uint16_t* a = reinterpret_cast<const uint16_t*>(p.a);
    if (h0 + 1 < p.H && (p.H & 1) == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) c.w[i] = __ldcs(reinterpret_cast<const uint32_t*>(a + (t0 + i) * p.H + h0));
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        c.w[i] = (h0 < p.H ? (uint32_t)a[(t0 + i) * p.H + h0] : 0u) |
                 (h0 + 1 < p.H ? (uint32_t)a[(t0 + i) * p.H + h0 + 1] << 16 : 0u);
    }
  } else {
    const uint32_t* a = reinterpret_cast<const uint32_t*>(p.a);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      c.w[i] = h0 < p.H ? __ldcs(a + (t0 + i) * p.H + h0) : 0u;
      c.w1[i] = h0 + 1 < p.H ? __ldcs(a + (t0 + i) * p.H + h0 + 1) : 0u;
    }
  }
}

// feature f (0: h0, 1: h0 + 1) of a loaded pair as float64
template <int DT>
__device__ __forceinline__ void column(const Col2<DT>& c, int f, double (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if constexpr (DT == DT_BF16)
      v[i] = (double)__uint_as_float(f ? (c.w[i] & 0xFFFF0000u) : (c.w[i] << 16));
    else
      v[i] = (double)__uint_as_float(f ? c.w1[i] : c.w[i]);
  }
}

// transforms.py:92-97 on one group: signs (a negation is the product with
// -1.0, signed zeros included), numpy's butterfly order h = 1, 2, 4, 8, then
// the exact division by sqrt(16).
__device__ __forceinline__ void rht16(double (&a)[16], uint32_t negmask) {
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if ((negmask >> i) & 1u) a[i] = -a[i];
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
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = __dmul_rn(a[i], 0.25);
}

// BF16 input, both features of the lane at once in f32x2 (a[i] = (feature
// h0, feature h0+1) of token i).  Every operation is exact -- so the result
// equals the float64 route bit for bit -- when, per feature, the nonzero
// inputs span at most 12 binades (any partial sum of <= 16 terms then needs
// <= 8 + 12 + 4 = 24 significant bits) and none is below 2^-99 (x/4 and all
// sums stay normal).  ok0 / ok1 report the condition per feature; callers take
// the float64 route otherwise.  The signs and the /4 fold into one exact
// product per token.
__device__ __forceinline__ void rht16_pair_f32(const uint32_t (&w)[16], const float (&sq)[16],
                                               float2 (&a)[16], bool& ok0, bool& ok1) {
  uint32_t mx = 0, mn = 0xFFFFFFFFu;  // per half: max |bits|, min(|bits| - 1) (zeros wrap high)
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t m = w[i] & 0x7FFF7FFFu;
    mx = __vmaxu2(mx, m);
    mn = __vminu2(mn, __vsub2(m, 0x00010001u));
  }
  const int e0max = (mx & 0xFFFFu) >> 7, e1max = mx >> 23;
  const int e0min = ((mn & 0xFFFFu) + 1) >> 7, e1min = ((mn >> 16) + 1) >> 7;
  // all-zero feature: emin = 512 > emax (exact); else span and range checks
  ok0 = (e0max - e0min <= 12) && (e0min >= 28);
  ok1 = (e1max - e1min <= 12) && (e1min >= 28);
  ok0 |= e0min == 512;
  ok1 |= e1min == 512;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 x = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u));
    a[i] = __fmul2_rn(x, make_float2(sq[i], sq[i]));
  }
#pragma unroll
  for (int h = 1; h < 16; h <<= 1) {
    float2 b[16];
#pragma unroll
    for (int blk = 0; blk < 16; blk += 2 * h)
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const float2 u = a[blk + j], v = a[blk + h + j];
        b[blk + j] = __fadd2_rn(u, v);
        b[blk + h + j] = __fadd2_rn(u, make_float2(-v.x, -v.y));
      }
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = b[i];
  }
}

__device__ __forceinline__ uint64_t absbits(double v) {
  return (uint64_t)__double_as_longlong(v) & 0x7FFFFFFFFFFFFFFFull;
}

template <int DT>
__global__ void __launch_bounds__(256, 2) rht_t_amax_kernel(RtParams p) {
  select_group(p);
  const int64_t nbT = p.T >> 4;
  const int64_t nH = (p.H + kUnitH - 1) / kUnitH, nK = (nbT + kUnitK - 1) / kUnitK;
  const int64_t units = nH * nK;
  const int lane = threadIdx.x & 31;
  uint64_t m = 0;  // |y| bit pattern (non-negative: bit order == value order; NaN above inf)
  for (int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); u < units; u += (int64_t)gridDim.x * 8) {
    const int64_t hu = u % nH, ku = u / nH;
    const int64_t h0 = hu * kUnitH + 2 * lane;
    Col2<DT> cn;  // next token block's rows, in flight during this one
    if (ku * kUnitK < nbT) load_pair<DT>(p, ku * kUnitK, h0, cn);
#pragma unroll 1
    for (int kk = 0; kk < kUnitK; ++kk) {
      const int64_t k = ku * kUnitK + kk;
      if (k >= nbT) break;
      const Col2<DT> c = cn;
      if (kk + 1 < kUnitK && k + 1 < nbT) load_pair<DT>(p, k + 1, h0, cn);
      bool ok[2] = {false, false};
      if constexpr (DT == DT_BF16) {
        float2 a[16];
        rht16_pair_f32(c.w, p.sq, a, ok[0], ok[1]);
        uint32_t m0 = 0, m1 = 0;  // |y| f32 bit patterns
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          m0 = max(m0, __float_as_uint(a[i].x) & 0x7FFFFFFFu);
          m1 = max(m1, __float_as_uint(a[i].y) & 0x7FFFFFFFu);
        }
        const uint64_t b0 = absbits((double)__uint_as_float(m0)), b1 = absbits((double)__uint_as_float(m1));
        if (ok[0]) m = b0 > m ? b0 : m;
        if (ok[1]) m = b1 > m ? b1 : m;
      }
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        if (ok[f]) continue;
        double v[16];
        column<DT>(c, f, v);
        rht16(v, p.negmask);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t b0 = absbits(v[i]);
          m = b0 > m ? b0 : m;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t v = __shfl_xor_sync(0xFFFFFFFFu, m, o);
    m = v > m ? v : m;
  }
  __shared__ uint64_t wmax[8];
  if (lane == 0) wmax[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t b = 0;
    for (int w = 0; w < 8; ++w) b = wmax[w] > b ? wmax[w] : b;
    atomicMax(reinterpret_cast<unsigned long long*>(p.d_amax), (unsigned long long)b);
  }
}

// element i of the block's float32 values, from registers (the rare exact
// per-nibble tie test of exact_codes); a select chain keeps x in registers
struct RegLoad {
  const float2 (&x)[8];
  __device__ __forceinline__ float operator()(int i) const {
    float r = x[0].x;
#pragma unroll
    for (int j = 1; j < 16; ++j)
      if (i == j) r = (j & 1) ? x[j >> 1].y : x[j >> 1].x;
    return r;
  }
};

// Fast path of one block: y as float32 (all 16 values must be exact) through
// block_sl.  False: the block is deferred to the float64 restatement.
template <int MODE>
__device__ __forceinline__ bool quant_block_fast(const double (&y)[16], const TensorConsts& tc,
                                                 BlockOut& o) {
  float2 xf[8];
  bool f32ok = !tc.force_exact;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    xf[p] = make_float2(__double2float_rn(y[2 * p]), __double2float_rn(y[2 * p + 1]));
    f32ok &= ((double)xf[p].x == y[2 * p]) & ((double)xf[p].y == y[2 * p + 1]);
  }
  float m0 = 0.f;
#pragma unroll
  for (int p = 0; p < 8; ++p) m0 = fmaxf(m0, fmaxf(fabsf(xf[p].x), fabsf(xf[p].y)));
  return block_sl<MODE, 2>(xf, m0, tc, RegLoad{xf}, o) && f32ok;
}

constexpr int kRtDeferCta = 4096;  // deferred (h, k) per CTA

template <int DT>
__device__ __noinline__ void rt_resolve(const RtParams p, double alpha_d, uint32_t hk, int64_t kb4) {
  const int64_t h = hk >> 16, k = hk & 0xFFFFu;
  const int64_t t0 = k * 16;
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if constexpr (DT == DT_BF16)
      v[i] = (double)__uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(p.a)[(t0 + i) * p.H + h] << 16);
    else
      v[i] = (double)reinterpret_cast<const float*>(p.a)[(t0 + i) * p.H + h];
  }
  rht16(v, p.negmask);
  BlockOut o;
  exact_block(v, alpha_d, p.mode, p.rule, &o);
  *reinterpret_cast<uint64_t*>(p.codes + h * (p.T >> 4) * 8 + k * 8) = o.codes;
  p.scales_tc[sf_tc_offset(h, k, kb4)] = (uint8_t)o.sc;
}

template <int DT, int MODE>
__global__ void __launch_bounds__(256, F46_RT_MINB) quant_rht_t_kernel(RtParams p) {
  select_group(p);
  // blocks for the float64 route, CTA-wide: resolved by all 256 threads at the
  // end (a few per warp would otherwise run with most lanes idle)
  __shared__ uint32_t dlist[kRtDeferCta];
  __shared__ uint32_t ndef;
  if (threadIdx.x == 0) ndef = 0;
  __syncthreads();
  const double amax = *p.d_amax;
  const double alpha_d = amax == 0.0 ? 1.0 : (double)((float)amax / (float)p.mcap);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.d_alpha_out) *p.d_alpha_out = alpha_d;
    if (p.d_flags && !(amax <= 1.7976931348623157e308)) atomicOr(p.d_flags, F46_FLAG_NONFINITE);
  }
  // y is not BF16: the tie direction is unknown (exact per-nibble tests)
  const TensorConsts tc = make_consts(alpha_d, p.rule, DT_F32, 2);
  const int64_t nbT = p.T >> 4, kb4 = (nbT + 3) >> 2;
  const int64_t nH = (p.H + kUnitH - 1) / kUnitH, nK = (nbT + kUnitK - 1) / kUnitK;
  const int64_t units = nH * nK;
  const int lane = threadIdx.x & 31;
  const int64_t row_bytes = nbT * 8;
  for (int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); u < units; u += (int64_t)gridDim.x * 8) {
    const int64_t hu = u % nH, ku = u / nH;
    const int64_t h0 = hu * kUnitH + 2 * lane;
#pragma unroll 1
    for (int kk = 0; kk < kUnitK; ++kk) {
      const int64_t k = ku * kUnitK + kk;
      if (k >= nbT) break;
      Col2<DT> c;
      load_pair<DT>(p, k, h0, c);
      float2 a[16];
      bool okf[2] = {false, false};
      if constexpr (DT == DT_BF16) rht16_pair_f32(c.w, p.sq, a, okf[0], okf[1]);
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int64_t h = h0 + f;
        BlockOut o;
        bool ok;
        if constexpr (DT == DT_BF16) {
          // the f32 route's values are the reference's float64 values exactly
          float2 xf[8];
          float bm = 0.f;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            xf[q] = f ? make_float2(a[2 * q].y, a[2 * q + 1].y) : make_float2(a[2 * q].x, a[2 * q + 1].x);
            bm = fmaxf(bm, fmaxf(fabsf(xf[q].x), fabsf(xf[q].y)));
          }
          ok = block_sl<MODE, 2>(xf, bm, tc, RegLoad{xf}, o) && okf[f] && !tc.force_exact;
        } else {
          double v[16];
          column<DT>(c, f, v);
          rht16(v, p.negmask);
          ok = quant_block_fast<MODE>(v, tc, o);
        }
        const bool live = h < p.H;
        if (live && ok) {
          *reinterpret_cast<uint64_t*>(p.codes + h * row_bytes + k * 8) = o.codes;
          p.scales_tc[sf_tc_offset(h, k, kb4)] = (uint8_t)o.sc;
        }
        const bool defer = live && !ok;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, defer);
        if (m) {
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(&ndef, (uint32_t)__popc(m));
          base = __shfl_sync(0xFFFFFFFFu, base, 0);
          const uint32_t hk = ((uint32_t)h << 16) | (uint32_t)k;
          const uint32_t slot = base + __popc(m & ((1u << lane) - 1));
          if (defer) {
            if (slot < kRtDeferCta)
              dlist[slot] = hk;
            else
              rt_resolve<DT>(p, alpha_d, hk, kb4);  // list full: resolve in place
          }
        }
      }
    }
  }
  __syncthreads();
  const uint32_t n = min(ndef, (uint32_t)kRtDeferCta);
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) rt_resolve<DT>(p, alpha_d, dlist[i], kb4);
}

int num_sms() { return f46rt::num_sms(); }

int launch_status() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "[fouroversix] CUDA error: %s\n", cudaGetErrorString(e));
    return F46_ERR_CUDA;
  }
  return F46_OK;
}

int check_rt(const void* a, int dtype, int groups, int64_t T, int64_t H) {
  if (!a || groups < 1 || groups > 65535 || T <= 0 || H <= 0 || (T & 15)) return F46_ERR_INVALID_ARG;
  if (H > 65535 || (T >> 4) > 65535) return F46_ERR_UNSUPPORTED;  // deferred (h, k) packing
  if (dtype != F46_DT_BF16 && dtype != F46_DT_F32) return F46_ERR_INVALID_ARG;
  return F46_OK;
}

void fill_signs(RtParams& p) {
  for (int i = 0; i < 16; ++i) p.sq[i] = ((p.negmask >> i) & 1u) ? -0.25f : 0.25f;
}

dim3 rt_grid(const RtParams& p, int groups) {
  const int64_t nbT = p.T >> 4;
  const int64_t units = ((p.H + kUnitH - 1) / kUnitH) * ((nbT + kUnitK - 1) / kUnitK);
  int64_t gx = (units + 7) / 8;
  gx = std::min<int64_t>(gx, std::max<int64_t>(1, (int64_t)num_sms() * 8 / groups));
  return dim3((unsigned)std::max<int64_t>(gx, 1), (unsigned)groups);
}

}  // namespace

extern "C" {

int f46_rht_t_amax_grouped(const void* a, int dtype, int groups, int64_t T, int64_t H,
                           uint32_t sign_mask, double* d_amax, f46_stream_t stream) {
  if (const int rc = check_rt(a, dtype, groups, T, H)) return rc;
  if (!d_amax) return F46_ERR_INVALID_ARG;
  const int64_t esz = dtype == F46_DT_BF16 ? 2 : 4;
  RtParams p{a, T, H, dtype, 0, 0, 0.0, sign_mask & 0xFFFFu, d_amax, nullptr, nullptr, nullptr,
             nullptr, T * H * esz, 0, 0, {}};
  fill_signs(p);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == F46_DT_BF16)
    rht_t_amax_kernel<DT_BF16><<<rt_grid(p, groups), 256, 0, s>>>(p);
  else
    rht_t_amax_kernel<DT_F32><<<rt_grid(p, groups), 256, 0, s>>>(p);
  return launch_status();
}

int f46_quantize_rht_t_grouped(const void* a, int dtype, int groups, int64_t T, int64_t H,
                               uint32_t sign_mask, int mode, int rule, double mcap,
                               double* d_amax, uint8_t* codes, uint8_t* scales_tc,
                               double* d_alpha_out, uint32_t* d_flags, f46_stream_t stream) {
  if (const int rc = check_rt(a, dtype, groups, T, H)) return rc;
  if (!d_amax || !codes || !scales_tc || !(mcap > 0.0)) return F46_ERR_INVALID_ARG;
  if (mode < F46_FIXED6 || mode > F46_ADAPTIVE || rule < F46_RULE_MSE || rule > F46_RULE_ABSMAX)
    return F46_ERR_CONFIG;
  const int64_t esz = dtype == F46_DT_BF16 ? 2 : 4;
  const int64_t nbT = T >> 4;
  RtParams p{a, T, H, dtype, mode, rule, mcap, sign_mask & 0xFFFFu, d_amax, codes, scales_tc,
             d_alpha_out, d_flags, T * H * esz, H * nbT * 8,
             (int64_t)f46_scales_tc_bytes(H, T), {}};
  fill_signs(p);
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid = rt_grid(p, groups);
#define F46_RT_LAUNCH(DTV)                                                   \
  switch (mode) {                                                            \
    case F46_FIXED6:                                                         \
      quant_rht_t_kernel<DTV, FIXED6><<<grid, 256, 0, s>>>(p);               \
      break;                                                                 \
    case F46_FIXED4:                                                         \
      quant_rht_t_kernel<DTV, FIXED4><<<grid, 256, 0, s>>>(p);               \
      break;                                                                 \
    default:                                                                 \
      quant_rht_t_kernel<DTV, ADAPTIVE><<<grid, 256, 0, s>>>(p);             \
  }
  if (dtype == F46_DT_BF16) {
    F46_RT_LAUNCH(DT_BF16)
  } else {
    F46_RT_LAUNCH(DT_F32)
  }
#undef F46_RT_LAUNCH
  return launch_status();
}

}  // extern "C"

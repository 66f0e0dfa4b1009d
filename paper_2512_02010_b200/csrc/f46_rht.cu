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
    for (int kk = 0; kk < kUnitK; ++kk) {
      const int64_t k = ku * kUnitK + kk;
      if (k >= nbT) break;
      Col2<DT> c;
      load_pair<DT>(p, k, h0, c);
#pragma unroll
      for (int f = 0; f < 2; ++f) {
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

template <int MODE>
__device__ __forceinline__ BlockOut quant_block_f64(const double (&y)[16], const TensorConsts& tc,
                                                    double alpha_d, int mode, int rule) {
  float2 xf[8];
  bool f32ok = true;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    xf[p] = make_float2(__double2float_rn(y[2 * p]), __double2float_rn(y[2 * p + 1]));
    f32ok &= ((double)xf[p].x == y[2 * p]) & ((double)xf[p].y == y[2 * p + 1]);
  }
  BlockOut o;
  bool ok = false;
  if (f32ok && !tc.force_exact) {
    float m0 = 0.f;
#pragma unroll
    for (int p = 0; p < 8; ++p) m0 = fmaxf(m0, fmaxf(fabsf(xf[p].x), fabsf(xf[p].y)));
    ok = block_sl<MODE, 2>(xf, m0, tc, RegLoad{xf}, o);
  }
  if (!ok) exact_block(y, alpha_d, mode, rule, &o);
  return o;
}

template <int DT, int MODE>
__global__ void __launch_bounds__(256, F46_RT_MINB) quant_rht_t_kernel(RtParams p) {
  select_group(p);
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
  for (int64_t u = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); u < units; u += (int64_t)gridDim.x * 8) {
    const int64_t hu = u % nH, ku = u / nH;
    const int64_t h0 = hu * kUnitH + 2 * lane;
    const int64_t row_bytes = nbT * 8;
#pragma unroll 1
    for (int kk = 0; kk < kUnitK; ++kk) {
      const int64_t k = ku * kUnitK + kk;
      if (k >= nbT) break;
      Col2<DT> c;
      load_pair<DT>(p, k, h0, c);
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int64_t h = h0 + f;
        double v[16];
        column<DT>(c, f, v);
        rht16(v, p.negmask);
        const BlockOut o = quant_block_f64<MODE>(v, tc, alpha_d, p.mode, p.rule);
        if (h < p.H) {
          *reinterpret_cast<uint64_t*>(p.codes + h * row_bytes + k * 8) = o.codes;
          p.scales_tc[sf_tc_offset(h, k, kb4)] = (uint8_t)o.sc;
        }
      }
    }
  }
}

int g_sms[64];

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (g_sms[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n > 0 ? n : 148;
  }
  return g_sms[dev];
}

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
  if (dtype != F46_DT_BF16 && dtype != F46_DT_F32) return F46_ERR_INVALID_ARG;
  return F46_OK;
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
             nullptr, T * H * esz, 0, 0};
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
             (int64_t)f46_scales_tc_bytes(H, T)};
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

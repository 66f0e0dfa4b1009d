// f46_quant.cu -- amax, 4/6 quantize and dequantize kernels + their C ABI.
//
// Kernels (sm_100a):
//   amax_kernel        K1: grid-stride 128-bit loads, warp-shuffle max, one
//                      64-bit atomicMax on the float64 bit pattern per CTA.
//   quant_tma_kernel   K2: persistent CTAs stream 128-row x 64-col tiles of the
//                      input through a 3-stage TMA (cp.async.bulk.tensor, 128B
//                      swizzle) -> shared memory pipeline; one thread owns one
//                      row of the tile (4 blocks of 16), computes both 4/6
//                      candidates (f46_device.cuh) and writes 32 B of packed
//                      E2M1 codes plus 4 E4M3 scales straight into the tcgen05
//                      128x4 scale layout.  Requires cols % 64 == 0.
//   quant_generic_kernel  any shape / float64 input: one thread per block.
//   dequant_kernel     K3: one thread per block, 128-bit stores.
//
// Reference: blockquant.py:215-222, :334-376; adaptive.py:60-101.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <mutex>

#include "../../include/fouroversix.h"
#include "f46_device.cuh"

using namespace f46;

namespace {

constexpr int kStages = 3;

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

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
};

// blockquant.py:215-222 / :316-326: alpha = RN32(f32(amax) / f32(mcap)), 1.0
// for an all-zero tensor, or the override.
__device__ __forceinline__ double resolve_alpha(const QParams& p) {
  if (p.alpha_override > 0.0) return p.alpha_override;
  const double amax = *p.d_amax;
  if (amax == 0.0) return 1.0;
  return (double)((float)amax / (float)p.mcap);
}

__device__ __forceinline__ void prologue_flags(const QParams& p, double alpha) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.d_alpha_out) *p.d_alpha_out = alpha;
    if (p.alpha_override <= 0.0 && p.d_flags) {
      const double amax = *p.d_amax;
      if (!(amax <= 1.7976931348623157e308)) atomicOr(p.d_flags, F46_FLAG_NONFINITE);
    }
  }
}

// Re-read element i of the thread's block from the swizzled smem tile
// (warp tile: 32 rows x 128 B per box, TMA SWIZZLE_128B).
template <int DT>
struct TileLoad {
  const uint8_t* row;  // start of this thread's 128-byte row in box 0
  int r7, kb;          // r & 7, block index within the 64-column tile
  __device__ __forceinline__ float operator()(int i) const {
    if constexpr (DT == DT_BF16) {
      const int chunk = 2 * kb + (i >> 3);
      return __uint_as_float(
          (uint32_t)(*reinterpret_cast<const uint16_t*>(row + ((chunk ^ r7) << 4) + (i & 7) * 2))
          << 16);
    } else {
      const int chunk = (kb & 1) * 4 + (i >> 2);
      return *reinterpret_cast<const float*>(row + (kb >> 1) * 4096 + ((chunk ^ r7) << 4) +
                                             (i & 3) * 4);
    }
  }
};

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

template <int DT>
__device__ __forceinline__ void load_tile_block(const uint8_t* row, int r7, int kb, float2 (&x)[8],
                                                float& bmax) {
  if constexpr (DT == DT_BF16) {
    const uint4 a = *reinterpret_cast<const uint4*>(row + (((2 * kb) ^ r7) << 4));
    const uint4 b = *reinterpret_cast<const uint4*>(row + (((2 * kb + 1) ^ r7) << 4));
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int p = 0; p < 8; ++p)
      x[p] = make_float2(__uint_as_float(w[p] << 16), __uint_as_float(w[p] & 0xFFFF0000u));
  } else {
    const uint8_t* base = row + (kb >> 1) * 4096;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int chunk = (kb & 1) * 4 + c;
      const float4 v = *reinterpret_cast<const float4*>(base + ((chunk ^ r7) << 4));
      x[2 * c] = make_float2(v.x, v.y);
      x[2 * c + 1] = make_float2(v.z, v.w);
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
// K2: TMA-pipelined quantize (cols % 64 == 0)
//
// Each warp is an independent pipeline: it owns kStages shared-memory stages
// of one "warp tile" (32 rows x 64 columns; 4 KB of bf16, 8 KB of f32) and
// its own mbarriers; lane 0 issues the TMA for a stage as soon as the warp has
// consumed it.  Lane r quantizes row r of the tile: four 16-element blocks,
// 32 B of packed codes and 4 scale bytes (one u32 of the tcgen05 128x4 layout).
// ---------------------------------------------------------------------------
constexpr int kWarps = 4;

template <int DT, int MODE>
__global__ void __launch_bounds__(kWarps * 32) quant_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                               QParams p) {
  constexpr int kBox = 4096;                              // 32 rows x 128 B
  constexpr int kTileBytes = (DT == DT_BF16) ? kBox : 2 * kBox;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[kWarps][kStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n_ct = (uint32_t)(p.cols >> 6);
  const uint32_t n_rg = (uint32_t)((p.rows + 31) >> 5);  // 32-row groups holding data
  const uint32_t total = n_ct * n_rg;
  const int64_t nb = p.cols >> 4;
  const uint32_t gw = blockIdx.x * kWarps + warp, G = gridDim.x * kWarps;

  const double alpha_d = resolve_alpha(p);
  prologue_flags(p, alpha_d);
  const TensorConsts tc = make_consts(alpha_d, p.rule, DT);

  uint8_t* wsm = smem + warp * (kStages * kTileBytes);
  uint64_t* wb = bars[warp];
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&wb[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto issue = [&](int s, uint32_t t) {
    const uint32_t rg = t / n_ct, ct = t - rg * n_ct;
    uint8_t* dst = wsm + s * kTileBytes;
    mbar_expect_tx(&wb[s], kTileBytes);
    tma_load_2d(dst, &tmap, &wb[s], (int)(ct * 64), (int)(rg * 32));
    if constexpr (DT != DT_BF16) tma_load_2d(dst + kBox, &tmap, &wb[s], (int)(ct * 64 + 32), (int)(rg * 32));
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s)
      if (gw + s * G < total) issue(s, gw + s * G);
  }

  bool nonfinite = false;
  uint32_t it = 0;
  for (uint32_t t = gw; t < total; t += G, ++it) {
    const int s = it % kStages;
    mbar_wait(&wb[s], (it / kStages) & 1u);
    const uint32_t rg = t / n_ct, ct = t - rg * n_ct;
    const int64_t grow = (int64_t)rg * 32 + lane;
    const uint8_t* row = wsm + s * kTileBytes + lane * 128;
    const int r7 = lane & 7;

    uint64_t codes[4];
    uint32_t scw = 0, pkw = 0;
#pragma unroll 1
    for (int kb = 0; kb < 4; ++kb) {
      float2 x[8];
      float bmax;
      load_tile_block<DT>(row, r7, kb, x, bmax);
      const TileLoad<DT> ld{row, r7, kb};
      BlockOut o;
      bool ok = false;
      if (!tc.force_exact) ok = fast_block<MODE>(x, bmax, tc, ld, o);
      if (__builtin_expect(!ok, 0)) {
        double xd[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          xd[i] = (double)ld(i);
          nonfinite |= !(fabs(xd[i]) <= 3.4028234663852886e38);
        }
        exact_block(xd, alpha_d, MODE, p.rule, &o);
      }
      codes[kb] = o.codes;
      scw |= o.sc << (8 * kb);
      pkw |= o.pick4 << (8 * kb);
    }
    __syncwarp();
    if (lane == 0 && t + kStages * G < total) issue(s, t + kStages * G);

    const bool live = grow < p.rows;
    const int64_t rt = grow >> 7;
    *reinterpret_cast<uint32_t*>(p.scales_tc + (rt * n_ct + ct) * 512 + (lane & 31) * 16 +
                                 ((grow & 127) >> 5) * 4) = live ? scw : 0u;
    if (live) {
      uint4* dst = reinterpret_cast<uint4*>(p.codes + grow * (p.cols >> 1) + ct * 32);
      dst[0] = make_uint4((uint32_t)codes[0], (uint32_t)(codes[0] >> 32), (uint32_t)codes[1],
                          (uint32_t)(codes[1] >> 32));
      dst[1] = make_uint4((uint32_t)codes[2], (uint32_t)(codes[2] >> 32), (uint32_t)codes[3],
                          (uint32_t)(codes[3] >> 32));
      if (p.scales_rm) *reinterpret_cast<uint32_t*>(p.scales_rm + grow * nb + ct * 4) = scw;
      if (p.pick4) *reinterpret_cast<uint32_t*>(p.pick4 + grow * nb + ct * 4) = pkw;
    }
  }
  // 32-row groups that only exist as padding of the last 128-row scale tile
  const uint32_t n_rg_pad = (uint32_t)(((p.rows + 127) >> 7) << 2);
  for (uint32_t t = n_rg * n_ct + gw; t < n_rg_pad * n_ct; t += G) {
    const uint32_t rg = t / n_ct, ct = t - rg * n_ct;
    const int64_t grow = (int64_t)rg * 32 + lane;
    *reinterpret_cast<uint32_t*>(p.scales_tc + ((grow >> 7) * n_ct + ct) * 512 + lane * 16 +
                                 ((grow & 127) >> 5) * 4) = 0u;
  }
  if (nonfinite && p.d_flags) atomicOr(p.d_flags, F46_FLAG_NONFINITE);
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
// K1: amax
// ---------------------------------------------------------------------------
template <int DT>
__global__ void __launch_bounds__(256) amax_kernel(const void* __restrict__ x, int64_t n,
                                                   double* d_amax) {
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
      for (int64_t i = tid; i < nv; i += stride) {
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
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / nb, kb = idx - row * nb;
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

template <int DT, int MODE>
int launch_quant_tma(const QParams& p, cudaStream_t s) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return F46_ERR_UNSUPPORTED;
  CUtensorMap map;
  const int esz = DT == DT_BF16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)p.cols, (cuuint64_t)p.rows};
  cuuint64_t strides[1] = {(cuuint64_t)(p.cols * esz)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, DT == DT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, const_cast<void*>(p.x), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return F46_ERR_UNSUPPORTED;
  constexpr int kTileBytes = (DT == DT_BF16) ? 4096 : 8192;
  const int smem = kWarps * kStages * kTileBytes + 1024;
  static bool configured = false;
  static int ctas_per_sm = 1;
  if (!configured) {
    cudaFuncSetAttribute(quant_tma_kernel<DT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, quant_tma_kernel<DT, MODE>,
                                                  kWarps * 32, smem);
    if (ctas_per_sm < 1) ctas_per_sm = 1;
    configured = true;
  }
  const int64_t wtiles = (p.cols >> 6) * ((p.rows + 127) >> 7) * 4;
  int64_t grid = (wtiles + kWarps - 1) / kWarps;
  if (grid > (int64_t)num_sms() * ctas_per_sm) grid = (int64_t)num_sms() * ctas_per_sm;
  quant_tma_kernel<DT, MODE><<<(unsigned)grid, kWarps * 32, smem, s>>>(map, p);
  return launch_status();
}

template <int DT, int MODE>
int launch_quant_generic(const QParams& p, cudaStream_t s) {
  const int64_t nb = (p.cols + 15) >> 4;
  const int64_t total = ((p.rows + 127) & ~(int64_t)127) * (((nb + 3) >> 2) * 4);
  int64_t grid = (total + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  quant_generic_kernel<DT, MODE><<<(unsigned)grid, 256, 0, s>>>(p);
  return launch_status();
}

template <int DT>
int dispatch_mode(const QParams& p, cudaStream_t s, bool tma) {
  switch (p.mode) {
    case F46_FIXED6:
      return tma ? launch_quant_tma<DT, FIXED6>(p, s) : launch_quant_generic<DT, FIXED6>(p, s);
    case F46_FIXED4:
      return tma ? launch_quant_tma<DT, FIXED4>(p, s) : launch_quant_generic<DT, FIXED4>(p, s);
    default:
      return tma ? launch_quant_tma<DT, ADAPTIVE>(p, s) : launch_quant_generic<DT, ADAPTIVE>(p, s);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

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
  const int64_t per = dtype == F46_DT_BF16 ? 256 * 8 * 4 : 256 * 4 * 4;
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
  const bool tma = (dtype != F46_DT_F64) && (cols % 64 == 0) && (((uintptr_t)x & 15) == 0) &&
                   (((uintptr_t)codes & 15) == 0) && (((uintptr_t)scales_tc & 3) == 0) &&
                   (((uintptr_t)scales_rm & 3) == 0) && (((uintptr_t)pick4 & 3) == 0) &&
                   rows < (1ll << 31) && cols < (1ll << 31);
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
#define F46_DQ(OUT, SL) \
  dequant_kernel<OUT, SL><<<(unsigned)grid, 256, 0, s>>>(codes, scales, d_alpha, rows, cols, out, d_flags)
  const bool tc = scale_layout == F46_SCALES_TC;
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

const char* f46_build_info(void) {
  return "fouroversix sm_100a (tcgen05/TMA) built with nvcc " __VERSION__;
}

}  // extern "C"

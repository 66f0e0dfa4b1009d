/*
 * fouroversix.h -- C ABI of the B200-native Four Over Six (4/6) NVFP4 path.
 *
 * Library: paper_2512_02010_b200/libfouroversix.so (sm_100a).  Plain pointers
 * and sizes only; every pointer named d_* or documented "device" is CUDA
 * device memory owned by the caller.  The library never allocates or frees
 * caller memory; all work is enqueued on `stream` and is asynchronous.
 * Functions return F46_OK (0) or a negative F46_ERR_* code.
 *
 * Reference interface each entry point replaces (paths under
 * /root/reference/pkg/src/fp4emu/):
 *   f46_amax            blockquant.py:218-219  (max|X| inside compute_tensor_scale;
 *                                               non-finite check of _validated :197-198)
 *   f46_quantize        blockquant.py:334-360  quantize_tensor (fixed6 / fixed4)
 *                       adaptive.py:83-101     quantize_tensor_adaptive (4/6, MSE rule)
 *                       blockquant.py:215-222  compute_tensor_scale (alpha, in the prologue)
 *   f46_quantize_2d     transforms.py:134-179  quantize_weights_2d (16x16 tiles)
 *   f46_dequantize      blockquant.py:363-376  dequantize_tensor
 *   f46_gemm_nvfp4      qlinear.py:74-93       emulated_fp4_matmul(aq, bq, transpose_b=True)
 *   f46_*_grouped       the above per MoE expert (one tensor scale per expert), one launch
 *   f46_quantize_rht_t_grouped  qlinear.py:150-157  apply_rht(a.T) + _quantize_1d (WGRAD operand)
 *
 * Data layout written by f46_quantize for a tensor viewed as [rows, cols]
 * (cols = last dimension, 16-element blocks along it, nb = ceil(cols/16)):
 *   codes      uint8 [rows][nb*8]: two E2M1 codes per byte, the even element
 *              in the low nibble (tensor_io.py:118-123); tail pads are 0.
 *   scales_tc  E4M3 block scales in the tcgen05 block-scaled-MMA layout:
 *              128-row x 4-block tiles of 512 bytes,
 *              offset(r, kb) = ((r/128)*ceil(nb/4) + kb/4)*512
 *                              + (r%32)*16 + ((r%128)/32)*4 + kb%4;
 *              size f46_scales_tc_bytes(rows, cols).
 *   scales_rm  optional uint8 [rows][nb] (the reference's scale_codes layout).
 *   pick4      optional uint8 [rows][nb]: 1 where the M=4 candidate was kept
 *              (adaptive.py:77-80; parity/diagnostics only).
 */
#ifndef FOUROVERSIX_H_
#define FOUROVERSIX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* f46_stream_t; /* a cudaStream_t */

/* return codes */
#define F46_OK 0
#define F46_ERR_INVALID_ARG (-1) /* -> InvalidInputError in the Python mirror */
#define F46_ERR_CONFIG (-2)      /* -> ConfigError */
#define F46_ERR_UNSUPPORTED (-3) /* shape/alignment the kernel does not take */
#define F46_ERR_CUDA (-4)        /* launch failure -> RuntimeError */

/* element types */
#define F46_DT_F32 0
#define F46_DT_BF16 1
#define F46_DT_F64 2

/* scale modes (QuantConfig.scale_mode, blockquant.py:59) */
#define F46_FIXED6 0
#define F46_FIXED4 1
#define F46_ADAPTIVE 2

/* adaptive selection rules (QuantConfig.rule, adaptive.py:46) */
#define F46_RULE_MSE 0
#define F46_RULE_L1 1
#define F46_RULE_ABSMAX 2

/* scale layouts for f46_dequantize */
#define F46_SCALES_TC 0
#define F46_SCALES_RM 1

/* bits of the device flags word */
#define F46_FLAG_NONFINITE 1u   /* a non-finite input element was seen */
#define F46_FLAG_NAN_SCALE 2u   /* dequantize saw an E4M3 NaN scale code */

/* Bytes of the scales_tc buffer for a [rows, cols] tensor. */
size_t f46_scales_tc_bytes(int64_t rows, int64_t cols);

/* Bytes of the packed code buffer: rows * ceil(cols/16) * 8. */
size_t f46_codes_bytes(int64_t rows, int64_t cols);

/*
 * Tensor-wide max|x| (blockquant.py:218-219).  Folds into *d_amax with an
 * order-independent atomic max on the float64 bit pattern, so the caller
 * zeroes d_amax once and may call this for several shards; a non-finite
 * element leaves d_amax >= +inf (checked by the caller / quantize prologue).
 *   x       device, n elements of `dtype`
 *   d_amax  device double[1]
 */
int f46_amax(const void* x, int dtype, int64_t n, double* d_amax, f46_stream_t stream);

/*
 * 1-D NVFP4 quantization, 16-element blocks along the last dimension.
 *   mode/rule      F46_FIXED6 | F46_FIXED4 | F46_ADAPTIVE, F46_RULE_*
 *   mcap           M_fp4 * fp8_cap of QuantConfig (2688, 1792, 1536, 1024)
 *   d_amax         device double[1] from f46_amax (+ allreduce MAX when
 *                  sharded); ignored when alpha_override > 0
 *   alpha_override > 0: use this tensor scale (blockquant.py:323-326)
 *   d_alpha_out    device double[1]: the resolved alpha (nullable)
 *   d_flags        device uint32[1]: F46_FLAG_* are OR-ed in (nullable)
 * Outputs as described in the header comment; scales_rm / pick4 nullable.
 */
int f46_quantize(const void* x, int dtype, int64_t rows, int64_t cols, int mode, int rule,
                 double mcap, const double* d_amax, double alpha_override, uint8_t* codes,
                 uint8_t* scales_tc, uint8_t* scales_rm, uint8_t* pick4, double* d_alpha_out,
                 uint32_t* d_flags, f46_stream_t stream);

/*
 * 2-D 16x16-tile quantization of a [R, C] weight (transforms.py:134-179):
 * one E4M3 scale per tile chosen over all 256 values (written to every row of
 * the tile), FP4 codes in the same packed layout as f46_quantize.  Because a
 * tile's scale is shared, W^T quantized this way is the transpose: with
 * codes_t / scales_tc_t non-null the kernel also writes W^T ([C, R], packed
 * codes [C][ceil(R/16)*8], tcgen05-layout scales) -- the K-major operand of
 * the DGRAD GEMM dx = dy @ W (qlinear.py:123-135).  scales_tc and
 * scales_tc_t must be zero-initialised by the caller (pad entries are not
 * written).  Exact float64 arithmetic, numpy's pairwise order for the tile
 * error sums.
 */
int f46_quantize_2d(const void* w, int dtype, int64_t R, int64_t C, int mode, int rule,
                    double mcap, const double* d_amax, double alpha_override, uint8_t* codes,
                    uint8_t* scales_tc, uint8_t* scales_rm, uint8_t* pick4, uint8_t* codes_t,
                    uint8_t* scales_tc_t, double* d_alpha_out, uint32_t* d_flags,
                    f46_stream_t stream);

/*
 * Dequantize (blockquant.py:363-376): out = decode_fp4(code) * alpha * decode(scale).
 *   scales       scales_tc (scale_layout = F46_SCALES_TC) or scales_rm (F46_SCALES_RM)
 *   d_alpha      device double[1]
 *   out          device [rows][cols] of out_dtype (F46_DT_F32: the exact value
 *                rounded once to float32; F46_DT_BF16: rounded once to bf16;
 *                F46_DT_F64: the exact value)
 * A NaN scale code sets F46_FLAG_NAN_SCALE in d_flags.
 */
int f46_dequantize(const uint8_t* codes, const uint8_t* scales, int scale_layout,
                   const double* d_alpha, int64_t rows, int64_t cols, void* out, int out_dtype,
                   uint32_t* d_flags, f46_stream_t stream);

/*
 * Block-scaled NVFP4 GEMM on tcgen05 (kind::mxf4nvf4, E4M3 scales, 16-blocks):
 *   C[M,N] = alpha_a * alpha_b * sum_k A[m,k] * B[n,k]
 * A and B are both K-major f46_quantize outputs ("TN": qlinear.py:74-93 with
 * transpose_b=True): codes [rows][ceil(K/16)*8] bytes, scales in the tcgen05
 * layout, alpha as a device double.  ceil(K/16) must be even (16-byte code
 * rows for TMA); M, N arbitrary.  C is row-major [M][ldc] of c_dtype
 * (F46_DT_F32 or F46_DT_BF16), ldc >= N.  F46_ERR_UNSUPPORTED for odd
 * ceil(K/16) or unaligned operand buffers.
 */
int f46_gemm_nvfp4(const uint8_t* a_codes, const uint8_t* a_scales_tc, const double* d_alpha_a,
                   const uint8_t* b_codes, const uint8_t* b_scales_tc, const double* d_alpha_b,
                   int64_t M, int64_t N, int64_t K, void* c, int64_t ldc, int c_dtype,
                   f46_stream_t stream);

/* Grouped (MoE-style) variant: `groups` independent GEMMs of one shape whose
 * operands are packed back to back (group stride = one operand's code / scale
 * buffer size), one alpha per group (d_alpha_a[g], d_alpha_b[g]); C is
 * [groups][M][ldc]. */
int f46_gemm_nvfp4_grouped(int groups, const uint8_t* a_codes, const uint8_t* a_scales_tc,
                           const double* d_alpha_a, const uint8_t* b_codes,
                           const uint8_t* b_scales_tc, const double* d_alpha_b, int64_t M,
                           int64_t N, int64_t K, void* c, int64_t ldc, int c_dtype,
                           f46_stream_t stream);

/*
 * Producer-fused amax (no reference counterpart --
 * PAPER.md:153-161's recipe).  As f46_gemm_nvfp4 / f46_gemm_nvfp4_grouped,
 * and the epilogue also reduces max |C| of the stored values (after the bf16
 * rounding when c_dtype is bf16) into d_amax_out[0] (grouped: d_amax_out[g]
 * per group) as a float64, with the same 64-bit atomicMax on the bit pattern
 * f46_amax uses: the caller zeroes d_amax_out first, and the buffer can be
 * handed to f46_quantize as its d_amax, so quantizing C for the next layer
 * reads C once (2.5625 instead of 4.5625 bytes per bf16 element).  A NaN in C
 * propagates and makes the quantizer flag the input as non-finite.
 */
int f46_gemm_nvfp4_amax(const uint8_t* a_codes, const uint8_t* a_scales_tc, const double* d_alpha_a,
                        const uint8_t* b_codes, const uint8_t* b_scales_tc, const double* d_alpha_b,
                        int64_t M, int64_t N, int64_t K, void* c, int64_t ldc, int c_dtype,
                        double* d_amax_out, f46_stream_t stream);
int f46_gemm_nvfp4_grouped_amax(int groups, const uint8_t* a_codes, const uint8_t* a_scales_tc,
                                const double* d_alpha_a, const uint8_t* b_codes,
                                const uint8_t* b_scales_tc, const double* d_alpha_b, int64_t M,
                                int64_t N, int64_t K, void* c, int64_t ldc, int c_dtype,
                                double* d_amax_out, f46_stream_t stream);

/*
 * Selection statistics of the 4/6 rules in one pass (adaptive.py:159-187):
 * for every block both candidates' exact float64 errors and each rule's
 * pick (mse / l1 / absmax, strict '<').  Writes d_partials[nparts][9] =
 * {4-picks mse, l1, absmax; disagreements mse-l1, mse-absmax, l1-absmax;
 * summed chosen squared error for mse, l1, absmax} (one CTA per part, fixed
 * reduction order); the caller folds the parts.
 */
int f46_selection_stats(const void* x, int dtype, int64_t rows, int64_t cols, double mcap,
                        const double* d_amax, double alpha_override, double* d_partials,
                        int nparts, double* d_alpha_out, f46_stream_t stream);

/*
 * Stochastic-rounding quantization (rounding="sr": blockquant.py:253-257,
 * codecs.py:120-148), modes as f46_quantize.  key6 / key4 are the Philox4x64
 * keys of the reference's uniform streams, SeedSequence(seed, spawn_key=(tag,
 * 6 | 4)).generate_state(2, uint64), derived by the host; the kernel draws
 * numpy's exact uniforms per element.  Exact float64 arithmetic.
 */
int f46_quantize_sr(const void* x, int dtype, int64_t rows, int64_t cols, int mode, int rule,
                    double mcap, const double* d_amax, double alpha_override, uint64_t key6_0,
                    uint64_t key6_1, uint64_t key4_0, uint64_t key4_1, uint8_t* codes,
                    uint8_t* scales_tc, uint8_t* scales_rm, uint8_t* pick4, double* d_alpha_out,
                    uint32_t* d_flags, f46_stream_t stream);

/*
 * 16-wide randomized Hadamard transform along the last dim (transforms.py:92-97):
 * out = fwht(x * signs) / 4 per contiguous group of 16, float64 (numpy's
 * butterfly order).  n = number of elements (multiple of 16); signs16 is a
 * HOST array of 16 values +-1.
 */
int f46_rht16(const void* x, int dtype, int64_t n, const double* signs16, double* out,
              f46_stream_t stream);

/*
 * Fused amax + quantize in one cooperative launch for tensors that fit in L2
 * (< 2^31 bytes; worthwhile up to ~96 MB): each warp takes max|x| over
 * exactly the tiles it then quantizes, a grid-wide barrier publishes the
 * tensor amax, and the quantize pass re-reads its tiles from L2.  Identical
 * output to f46_amax + f46_quantize.  d_work: device 16 bytes, zeroed by the
 * caller (the float64 amax, then the barrier counter); no alpha override and
 * no parity views.  F46_ERR_UNSUPPORTED when the tensor or the device does
 * not allow it (the caller then runs the two-kernel path).
 */
int f46_quantize_fused(const void* x, int dtype, int64_t rows, int64_t cols, int mode, int rule,
                       double mcap, double* d_work, uint8_t* codes, uint8_t* scales_tc,
                       double* d_alpha_out, uint32_t* d_flags, f46_stream_t stream);

/*
 * Grouped (expert-parallel MoE) variants.  A grouped
 * tensor is `groups` equal tensors stored back to back; each group is its own
 * reference tensor with its own tensor scale (d_amax[g], d_alpha_out[g]), i.e.
 * exactly what a per-group call of the single-tensor function would produce
 * (blockquant.py:215-222 per expert), in one launch.  Output buffers are the
 * per-group buffers back to back (group stride f46_codes_bytes(rows, cols) /
 * f46_scales_tc_bytes(rows, cols)) -- the operand packing of
 * f46_gemm_nvfp4_grouped.  The caller zeroes d_amax[groups] before the amax
 * call.
 */
int f46_amax_grouped(const void* x, int dtype, int groups, int64_t n, double* d_amax,
                     f46_stream_t stream);
/* f46_quantize per group (no alpha override, no parity views). */
int f46_quantize_grouped(const void* x, int dtype, int groups, int64_t rows, int64_t cols, int mode,
                         int rule, double mcap, const double* d_amax, uint8_t* codes,
                         uint8_t* scales_tc, double* d_alpha_out, uint32_t* d_flags,
                         f46_stream_t stream);
/* f46_quantize_2d per group (W and, if non-null, W^T); scale buffers zeroed by the caller. */
int f46_quantize_2d_grouped(const void* w, int dtype, int groups, int64_t R, int64_t C, int mode,
                            int rule, double mcap, const double* d_amax, uint8_t* codes,
                            uint8_t* scales_tc, uint8_t* codes_t, uint8_t* scales_tc_t,
                            double* d_alpha_out, uint32_t* d_flags, f46_stream_t stream);

/*
 * WGRAD operand in one fused pass (qlinear.py:138-159): for each group's
 * row-major a[T][H] (T % 16 == 0), the operand A = RHT16 along T of a^T,
 * i.e. apply_rht(a.T, spec) (transforms.py:92-97, float64, numpy's butterfly
 * order), quantized 1-D along T with the given mode -- an [H][T] container
 * (codes [H][T/16*8], tcgen05 scales of [H, T], zeroed by the caller).
 * sign_mask bit i = 1 where spec.signs[i] == -1.  f46_rht_t_amax_grouped
 * folds max|A| per group into d_amax[g] (zeroed by the caller); the quantize
 * call reads it.  BF16 or FP32 input.
 */
int f46_rht_t_amax_grouped(const void* a, int dtype, int groups, int64_t T, int64_t H,
                           uint32_t sign_mask, double* d_amax, f46_stream_t stream);
int f46_quantize_rht_t_grouped(const void* a, int dtype, int groups, int64_t T, int64_t H,
                               uint32_t sign_mask, int mode, int rule, double mcap,
                               double* d_amax, uint8_t* codes, uint8_t* scales_tc,
                               double* d_alpha_out, uint32_t* d_flags, f46_stream_t stream);

/*
 * One block of any length n at any block-max target m (the reference's
 * block-level API: compute_block_scale blockquant.py:225-236, quantize_block
 * :379-414, quantize_block_adaptive adaptive.py:104-146 per candidate), in
 * float64 exactly as the reference computes it.  d_x: n doubles; d_u: n
 * uniforms for stochastic rounding or NULL for RNE; d_codes: n bytes (one code
 * per element); d_work: n doubles (returns the dequantized block); d_out[4] =
 * {scale code, sum diff^2, sum |diff|, max |diff|} with numpy's 1-D pairwise
 * summation order.
 */
int f46_quantize_block_ref(const double* d_x, int64_t n, double alpha, double m,
                           const double* d_u, uint8_t* d_codes, double* d_work, double* d_out,
                           f46_stream_t stream);

/*
 * C[M,N] = A[M,K] @ B[K,N], float32, products and sums each rounded once in
 * ascending k (no FMA): the reference's _accum_matmul_f32 (qlinear.py:64-71)
 * bit for bit.  Used for emulated_fp4_matmul(transpose_b=False), whose B is
 * blocked along N and so cannot feed a block-scaled tensor-core GEMM.
 */
int f46_matmul_f32_ordered(const float* A, const float* B, int64_t M, int64_t N, int64_t K, float* C,
                           f46_stream_t stream);

/*
 * Test / diagnostic hooks, process-wide, default 0 (f46_runtime.h Hook):
 *   0 SEG_CHUNK_BYTES  > 0: K2 launches at most this many input bytes at a time
 *   1 DQ_VEC           1: dequantize takes the coalesced (non-TMA) kernel
 *   2 Q2_V1            1: 2-D tiles take the one-tile-per-warp kernel
 *   3 SR_ONE_THREAD    1: stochastic rounding takes the one-thread-per-block kernel
 *   4 GEMM_KERNEL      0: CTA-pair GEMM, 1: single-CTA persistent, 2: one tile per CTA
 * Production launches read these as plain integers; nothing is taken from
 * the environment.
 */
int f46_set_test_hook(int hook, int64_t value);

/* Human-readable build info ("sm_100a ..."). */
const char* f46_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* FOUROVERSIX_H_ */

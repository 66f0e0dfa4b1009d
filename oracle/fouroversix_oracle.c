/*
 * fouroversix_oracle.c -- CPU restatement of the reference's 4/6 NVFP4 path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2512_02010_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path never calls it (and fails loudly when its own CUDA library is missing).
 *
 * It restates, in IEEE float64 with no FMA contraction (built with
 * -ffp-contract=off), the numpy algorithm of the reference package fp4emu:
 *
 *   codecs.py:92-96     decode_fp4
 *   codecs.py:99-117    encode_fp4_rne         (frexp / rint / searchsorted)
 *   codecs.py:151-155   decode_fp8_e4m3        (table codecs.py:56-68)
 *   codecs.py:158-178   encode_fp8_e4m3        (RNE, saturate at 448)
 *   blockquant.py:215-222 compute_tensor_scale (alpha through float32)
 *   blockquant.py:239-242 _nvfp4_scales        (bmax == 0 -> code 1)
 *   blockquant.py:260-280 _cast_values         (divide by *decoded* scale,
 *                                               underflowed scale -> +-6 / 0)
 *   blockquant.py:283-293 _block_error_sums    (numpy pairwise sum, 8 lanes)
 *   blockquant.py:302-313 _fixed_pass
 *   blockquant.py:334-360 quantize_tensor      (fixed6 / fixed4)
 *   blockquant.py:363-376 dequantize_tensor
 *   adaptive.py:60-101   _dual_pass/_select/quantize_tensor_adaptive
 *                        (strict '<', ties keep the 6 candidate)
 *   transforms.py:108-179 _tile_pass / quantize_weights_2d (16x16 tiles)
 *
 * The numpy summation order for a length-16 block reduction (numpy 2.3
 * pairwise_sum, n <= 128 branch) is r_j = e_j + e_{j+8}, then
 * ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); a 256-element tile is
 * P(e[0:128]) + P(e[128:256]) with P the same 8-accumulator scheme.  Both
 * were checked against numpy 2.3.5 (tests/golden/make_golden.py).
 *
 * Layouts produced (identical to the CUDA kernels, so tests can memcmp):
 *   codes   : uint8 [rows][nblocks*8]  two FP4 codes per byte, the even
 *             element in the low nibble (tensor_io.py:118-123), tail pads 0
 *   scales  : uint8 [rows][nblocks]    E4M3 codes (reference layout)
 *   pick4   : uint8 [rows][nblocks]    1 where the 4 candidate was kept
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define FO_DT_F32 0
#define FO_DT_BF16 1
#define FO_DT_F64 2

#define FO_MODE_FIXED6 0
#define FO_MODE_FIXED4 1
#define FO_MODE_ADAPTIVE 2

#define FO_RULE_MSE 0
#define FO_RULE_L1 1
#define FO_RULE_ABSMAX 2

static const double FP4_MAGS[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};

/* codecs.py:92-96 -- code 8 decodes to -0.0 */
double fo_decode_fp4(uint8_t code) {
    double v = FP4_MAGS[code & 7];
    return (code & 8) ? -v : v;
}

/* codecs.py:99-117 */
uint8_t fo_encode_fp4_rne(double x) {
    int sign = signbit(x) ? 1 : 0;
    double m = fabs(x);
    if (m > 6.0) m = 6.0;
    int e;
    frexp(m, &e);
    int ex = e - 1;
    if (ex < 0) ex = 0;
    double q = ldexp(1.0, ex - 1);
    double mag = rint(m / q) * q;
    /* searchsorted(_FP4_MAGS, mag), side='left' */
    int idx = 0;
    while (idx < 8 && FP4_MAGS[idx] < mag) idx++;
    return (uint8_t)(idx + (sign << 3));
}

/* codecs.py:56-68 table, :151-155 */
double fo_decode_e4m3(uint8_t code) {
    double sign = (code & 0x80) ? -1.0 : 1.0;
    int ex = (code >> 3) & 0xF;
    int mant = code & 7;
    if (ex == 0xF && mant == 7) return NAN;
    if (ex == 0) return sign * mant * ldexp(1.0, -9);
    return sign * (1.0 + mant / 8.0) * ldexp(1.0, ex - 7);
}

/* codecs.py:158-178 */
uint8_t fo_encode_e4m3(double x) {
    if (isnan(x)) return 0x7F;
    int sign = signbit(x) ? 1 : 0;
    double m = fabs(x);
    if (!isfinite(m)) m = 448.0;
    if (m > 448.0) m = 448.0;
    int e;
    frexp(m, &e);
    int ex = e - 1;
    if (ex < -6) ex = -6;
    double q = ldexp(1.0, ex - 3);
    double mag = rint(m / q) * q;
    /* searchsorted over the 127 increasing positive finite magnitudes */
    int idx = 0;
    while (idx < 0x7F && fo_decode_e4m3((uint8_t)idx) < mag) idx++;
    return (uint8_t)(idx + (sign << 7));
}

static inline double load_elem(const void* x, int dtype, int64_t i) {
    if (dtype == FO_DT_F32) return (double)((const float*)x)[i];
    if (dtype == FO_DT_BF16) {
        uint32_t b = ((uint32_t)((const uint16_t*)x)[i]) << 16;
        float f;
        memcpy(&f, &b, 4);
        return (double)f;
    }
    return ((const double*)x)[i];
}

/* numpy pairwise_sum for 8 <= n <= 128 (the n % 8 rest added in sequence) */
static double pw_sum(const double* a, int n) {
    double r[8];
    int i, j;
    for (j = 0; j < 8; j++) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
        for (j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
}

/* amax over the whole tensor; returns -1 if any element is non-finite
 * (blockquant.py:191-199 raises InvalidInputError). */
int fo_amax(const void* x, int dtype, int64_t n, double* amax_out) {
    double m = 0.0;
    int bad = 0;
    for (int64_t i = 0; i < n; i++) {
        double v = load_elem(x, dtype, i);
        if (!isfinite(v)) bad = 1;
        double a = fabs(v);
        if (a > m) m = a;
    }
    *amax_out = m;
    return bad ? -1 : 0;
}

/* blockquant.py:215-222 */
double fo_tensor_scale(double amax, double m_fp4, double fp8_cap) {
    if (amax == 0.0) return 1.0;
    float a = (float)amax;
    float d = (float)(m_fp4 * fp8_cap);
    return (double)(a / d);
}

/* One fixed-target pass over one padded block of n values
 * (blockquant.py:302-313 with _nvfp4_scales :239-242, _cast_values :260-280,
 * _block_error_sums :283-293).  n is the padded block length (16 or 256). */
typedef struct {
    uint8_t sc;
    double sq, ab, mx;
} fo_pass_t;

static void fixed_pass(const double* xb, int n, double alpha, double m, uint8_t* codes,
                       double* deq, fo_pass_t* out) {
    double bmax = 0.0;
    for (int i = 0; i < n; i++) {
        double a = fabs(xb[i]);
        if (a > bmax) bmax = a;
    }
    uint8_t sc = fo_encode_e4m3(bmax / (alpha * m));
    if (bmax == 0.0) sc = 1;
    double sdec = fo_decode_e4m3(sc);
    double denom = alpha * sdec;
    double e_sq[256], e_ab[256];
    double mx = 0.0;
    for (int i = 0; i < n; i++) {
        double scaled;
        if (denom > 0.0)
            scaled = xb[i] / denom;
        else
            scaled = (xb[i] != 0.0) ? copysign(6.0, xb[i]) : 0.0;
        uint8_t c = fo_encode_fp4_rne(scaled);
        codes[i] = c;
        double d = fo_decode_fp4(c) * denom;
        deq[i] = d;
        double diff = d - xb[i];
        e_sq[i] = diff * diff;
        e_ab[i] = fabs(diff);
        if (e_ab[i] > mx) mx = e_ab[i];
    }
    out->sc = sc;
    if (n == 16) {
        out->sq = pw_sum(e_sq, 16);
        out->ab = pw_sum(e_ab, 16);
    } else { /* 256: numpy splits 128 + 128 (transforms.py:285-289) */
        out->sq = pw_sum(e_sq, 128) + pw_sum(e_sq + 128, 128);
        out->ab = pw_sum(e_ab, 128) + pw_sum(e_ab + 128, 128);
    }
    out->mx = mx;
}

static double rule_err(const fo_pass_t* p, int rule) {
    return rule == FO_RULE_MSE ? p->sq : (rule == FO_RULE_L1 ? p->ab : p->mx);
}

/*
 * Quantize a [rows, cols] tensor blocked by 16 along cols.
 *   mode    FO_MODE_FIXED6 / FIXED4 / ADAPTIVE
 *   alpha   tensor scale (already resolved: computed or override)
 * Outputs (any may be NULL except codes/scales):
 *   codes   [rows][nblocks*8] packed, scales [rows][nblocks],
 *   pick4   [rows][nblocks], err6/err4 [rows][nblocks] per-rule error sums
 */
int fo_quantize(const void* x, int dtype, int64_t rows, int64_t cols, int mode, int rule,
                double alpha, uint8_t* codes, uint8_t* scales, uint8_t* pick4, double* err6,
                double* err4, int nthreads) {
    if (rows <= 0 || cols <= 0) return -1;
    const int64_t nb = (cols + 15) / 16;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t r = 0; r < rows; r++) {
        double xb[16], deq[16];
        uint8_t c6[16], c4[16];
        for (int64_t b = 0; b < nb; b++) {
            for (int i = 0; i < 16; i++) {
                int64_t c = b * 16 + i;
                xb[i] = (c < cols) ? load_elem(x, dtype, r * cols + c) : 0.0;
            }
            fo_pass_t p6, p4;
            const uint8_t* chosen;
            uint8_t sc;
            int k = 0;
            if (mode == FO_MODE_ADAPTIVE) {
                fixed_pass(xb, 16, alpha, 6.0, c6, deq, &p6);
                fixed_pass(xb, 16, alpha, 4.0, c4, deq, &p4);
                k = rule_err(&p4, rule) < rule_err(&p6, rule); /* adaptive.py:77-80 */
                chosen = k ? c4 : c6;
                sc = k ? p4.sc : p6.sc;
                if (err6) err6[r * nb + b] = rule_err(&p6, rule);
                if (err4) err4[r * nb + b] = rule_err(&p4, rule);
            } else {
                double m = (mode == FO_MODE_FIXED4) ? 4.0 : 6.0;
                fixed_pass(xb, 16, alpha, m, c6, deq, &p6);
                chosen = c6;
                sc = p6.sc;
                k = (mode == FO_MODE_FIXED4);
                if (err6) err6[r * nb + b] = rule_err(&p6, rule);
            }
            uint8_t* dst = codes + r * nb * 8 + b * 8;
            for (int i = 0; i < 8; i++) {
                /* pad positions carry code 0 (_strip_pad drops them) */
                int64_t c0 = b * 16 + 2 * i, c1 = c0 + 1;
                uint8_t lo = (c0 < cols) ? chosen[2 * i] : 0;
                uint8_t hi = (c1 < cols) ? chosen[2 * i + 1] : 0;
                dst[i] = (uint8_t)(lo | (hi << 4));
            }
            scales[r * nb + b] = sc;
            if (pick4) pick4[r * nb + b] = (uint8_t)k;
        }
    }
    return 0;
}

/* blockquant.py:363-376: out = decode_fp4(code) * alpha * decode(scale)
 * (float64, exact for alpha with <= 24 significant bits). */
int fo_dequantize(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols,
                  double alpha, double* out, int nthreads) {
    const int64_t nb = (cols + 15) / 16;
    for (int64_t i = 0; i < rows * nb; i++)
        if (isnan(fo_decode_e4m3(scales[i]))) return -2;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t r = 0; r < rows; r++) {
        for (int64_t c = 0; c < cols; c++) {
            uint8_t byte = codes[r * nb * 8 + c / 2];
            uint8_t code = (c & 1) ? (byte >> 4) : (byte & 15);
            double sdec = fo_decode_e4m3(scales[r * nb + c / 16]);
            out[r * cols + c] = fo_decode_fp4(code) * alpha * sdec;
        }
    }
    return 0;
}

/*
 * 2-D 16x16 tile quantization of a [R, C] weight (transforms.py:134-179):
 * one scale per tile, replicated over the tile's 16 rows in the row-major
 * scale array [R][ceil(C/16)] (transforms.py:331), codes in the same packed
 * layout as fo_quantize.
 */
int fo_quantize_2d(const void* x, int dtype, int64_t R, int64_t C, int mode, int rule,
                   double alpha, uint8_t* codes, uint8_t* scales, uint8_t* pick4, int nthreads) {
    const int64_t TR = (R + 15) / 16, TC = (C + 15) / 16;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t tr = 0; tr < TR; tr++) {
        double t[256], deq[256];
        uint8_t c6[256], c4[256];
        for (int64_t tc = 0; tc < TC; tc++) {
            for (int i = 0; i < 16; i++)
                for (int j = 0; j < 16; j++) {
                    int64_t r = tr * 16 + i, c = tc * 16 + j;
                    t[i * 16 + j] = (r < R && c < C) ? load_elem(x, dtype, r * C + c) : 0.0;
                }
            fo_pass_t p6, p4;
            const uint8_t* chosen;
            uint8_t sc;
            int k = 0;
            if (mode == FO_MODE_ADAPTIVE) {
                fixed_pass(t, 256, alpha, 6.0, c6, deq, &p6);
                fixed_pass(t, 256, alpha, 4.0, c4, deq, &p4);
                k = rule_err(&p4, rule) < rule_err(&p6, rule);
                chosen = k ? c4 : c6;
                sc = k ? p4.sc : p6.sc;
            } else {
                fixed_pass(t, 256, alpha, mode == FO_MODE_FIXED4 ? 4.0 : 6.0, c6, deq, &p6);
                chosen = c6;
                sc = p6.sc;
                k = (mode == FO_MODE_FIXED4);
            }
            for (int i = 0; i < 16; i++) {
                int64_t r = tr * 16 + i;
                if (r >= R) break;
                uint8_t* dst = codes + r * TC * 8 + tc * 8;
                for (int j = 0; j < 8; j++) {
                    int64_t c0 = tc * 16 + 2 * j;
                    uint8_t lo = (c0 < C) ? chosen[i * 16 + 2 * j] : 0;
                    uint8_t hi = (c0 + 1 < C) ? chosen[i * 16 + 2 * j + 1] : 0;
                    dst[j] = (uint8_t)(lo | (hi << 4));
                }
                scales[r * TC + tc] = sc;
                if (pick4) pick4[r * TC + tc] = (uint8_t)k;
            }
        }
    }
    return 0;
}

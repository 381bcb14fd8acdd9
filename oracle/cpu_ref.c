/*
 * oracle/cpu_ref.c -- CPU restatement of the QSync quantized-operator hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker (or the timed CPU baseline).  The product path (paper_2407_02327_b200)
 * never links or calls it.
 *
 * Parity status: the stochastic-rounding stream (mt19937_64, uniform01, SR) is
 * PINNED against the reference's own stochastic_round (oracle/_ref, built from
 * /root/reference/proj/src) and the golden vectors in BASELINE.md sec. G.  The
 * quantize / GEMM / dequant arithmetic is not present in the reference
 * (SPEC.md:9 puts the LP-PyTorch backend out of scope), so it follows the
 * paper's formulas plus the builder choices documented in DESIGN.md sec. 3
 * ("parity unpinned" for those formula choices, pinned for everything the
 * reference defines).
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off matters: the dequant epilogue is specified as two rounded
 * FP32 operations, not one FMA.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* mt19937_64, the engine std::mt19937_64 is defined as (C++ [rand.predef]):   */
/* w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9 u=29 d=0x5555555555555555 s=17   */
/* b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43 f=6364136223846793005.  */
/* Reference use: rng.hpp:12-14, indicator.cpp:179-187.                         */
/* ------------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL
#define MT_A 0xB5026F5AA96619E9ULL

typedef struct {
    uint64_t s[MT_N];
    int idx;
} ref_mt64;

void ref_mt64_seed(ref_mt64* g, uint64_t seed) {
    g->s[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        g->s[i] = 6364136223846793005ULL * (g->s[i - 1] ^ (g->s[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_N;
}

static void mt_twist(ref_mt64* g) {
    for (int i = 0; i < MT_N; ++i) {
        uint64_t y = (g->s[i] & MT_UPPER) | (g->s[(i + 1) % MT_N] & MT_LOWER);
        uint64_t v = g->s[(i + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) v ^= MT_A;
        g->s[i] = v;
    }
    g->idx = 0;
}

static inline uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

uint64_t ref_mt64_next(ref_mt64* g) {
    if (g->idx >= MT_N) mt_twist(g);
    return mt_temper(g->s[g->idx++]);
}

/* First n draws of mt19937_64(seed). */
void ref_mt64_draws(uint64_t seed, int64_t n, uint64_t* out) {
    ref_mt64 g;
    ref_mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = ref_mt64_next(&g);
}

/* rng.hpp:12-14: top 53 bits of one draw times 2^-53. */
static inline double uniform01_of(uint64_t draw) { return (double)(draw >> 11) * 0x1.0p-53; }

/* ------------------------------------------------------------------------- */
/* Stochastic rounding (indicator.cpp:176-193, :195-200).                      */
/* Returns 0, or 4 (= domain) when q <= 0 / k < 1 like the reference raises.   */
/* ------------------------------------------------------------------------- */
int ref_stochastic_round(const double* x, int64_t n, double q, double zp, uint64_t seed,
                         int64_t* rounded, double* dequantized) {
    if (!(q > 0)) return 4;
    ref_mt64 g;
    ref_mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) {
        const double xbar = (x[i] - zp) / q;
        const double lo = floor(xbar);
        const double frac = xbar - lo;
        const double up = uniform01_of(ref_mt64_next(&g)) < frac ? 1.0 : 0.0;
        const int64_t r = (int64_t)lo + (int64_t)up;
        if (rounded) rounded[i] = r;
        if (dequantized) dequantized[i] = q * (double)r + zp;
    }
    return 0;
}

int ref_stochastic_round_float(const double* x, int64_t n, int e, int k, uint64_t seed,
                               double* out) {
    if (k < 1) return 4;
    const double spacing = exp2((double)(e - k));
    return ref_stochastic_round(x, n, spacing, 0.0, seed, NULL, out);
}

/* ------------------------------------------------------------------------- */
/* INT8 fixed-point quantization (xbar=(x-z)/q, symmetric z=0).  */
/* Scale choice: s = absmax / 127 in FP32, s = 1 when the   */
/* tensor is all-zero.  RNE: rintf(x / s) saturated to [-127, 127].            */
/* ------------------------------------------------------------------------- */
float ref_absmax_f32(const float* x, int64_t n) {
    float m = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        float a = fabsf(x[i]);
        if (a > m) m = a;
    }
    return m;
}

float ref_scale_from_absmax(float absmax) { return absmax > 0.0f ? absmax / 127.0f : 1.0f; }

static inline int8_t sat_i8(float r) {
    if (r > 127.0f) r = 127.0f;
    if (r < -127.0f) r = -127.0f;
    return (int8_t)r;
}

/* Per-tensor RNE quantization; writes the scale it used. */
void ref_quantize_per_tensor(const float* x, int64_t n, int8_t* q, float* scale_out) {
    const float s = ref_scale_from_absmax(ref_absmax_f32(x, n));
    for (int64_t i = 0; i < n; ++i) q[i] = sat_i8(rintf(x[i] / s));
    *scale_out = s;
}

/* Per-channel (per output row of W [rows, cols]) RNE quantization. */
void ref_quantize_per_channel(const float* w, int64_t rows, int64_t cols, int8_t* q,
                              float* scales) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
        const float* row = w + r * cols;
        const float s = ref_scale_from_absmax(ref_absmax_f32(row, cols));
        for (int64_t c = 0; c < cols; ++c) q[r * cols + c] = sat_i8(rintf(row[c] / s));
        scales[r] = s;
    }
}

/* Stochastic-rounding quantization to INT8 with the reference stream: element
 * i uses draw i of mt19937_64(seed) exactly as indicator.cpp:183-191, then the
 * result is saturated to +-127 (xbar can exceed 127 at
 * x = absmax). */
void ref_quantize_sr_per_tensor(const float* x, int64_t n, float scale, uint64_t seed,
                                int8_t* q) {
    ref_mt64 g;
    ref_mt64_seed(&g, seed);
    const double qd = (double)scale;
    for (int64_t i = 0; i < n; ++i) {
        const double xbar = ((double)x[i] - 0.0) / qd;
        const double lo = floor(xbar);
        const double frac = xbar - lo;
        const int64_t up = uniform01_of(ref_mt64_next(&g)) < frac ? 1 : 0;
        int64_t r = (int64_t)lo + up;
        if (r > 127) r = 127;
        if (r < -127) r = -127;
        q[i] = (int8_t)r;
    }
}

void ref_dequantize_per_tensor(const int8_t* q, int64_t n, float scale, float* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)q[i] * scale;
}

void ref_dequantize_per_channel(const int8_t* q, int64_t rows, int64_t cols, const float* scales,
                                float* out) {
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) out[r * cols + c] = (float)q[r * cols + c] * scales[r];
}

/* ------------------------------------------------------------------------- */
/* IEEE binary16 conversions (RNE), the FP16 format of Precision::Fp16.        */
/* ------------------------------------------------------------------------- */
uint16_t ref_f32_to_f16(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u;
    const uint32_t absx = x & 0x7FFFFFFFu;
    if (absx >= 0x7F800000u) return (uint16_t)(sign | (absx > 0x7F800000u ? 0x7E00u : 0x7C00u));
    if (absx >= 0x477FF000u) return (uint16_t)(sign | 0x7C00u); /* rounds to >= 65520 -> inf */
    if (absx < 0x33000001u) return (uint16_t)sign;              /* < 2^-25 (+tie) -> 0 */
    const int exp = (int)(absx >> 23);
    uint32_t mant = (absx & 0x7FFFFFu) | 0x800000u;
    if (exp < 113) { /* subnormal half */
        const int shift = 126 - exp;  /* 14..24 */
        uint32_t h = mant >> shift;
        const uint32_t rem = mant & ((1u << shift) - 1u);
        const uint32_t half = 1u << (shift - 1);
        if (rem > half || (rem == half && (h & 1u))) ++h;
        return (uint16_t)(sign | h);
    }
    uint32_t h = ((uint32_t)(exp - 112) << 10) | ((mant >> 13) & 0x3FFu);
    const uint32_t rem = mant & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
    return (uint16_t)(sign | h);
}

float ref_f16_to_f32(uint16_t h) {
    const uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    const uint32_t exp = (h >> 10) & 0x1Fu;
    const uint32_t mant = h & 0x3FFu;
    uint32_t x;
    if (exp == 0) {
        if (mant == 0) {
            x = sign;
        } else {
            float f = ldexpf((float)mant, -24);
            memcpy(&x, &f, 4);
            x |= sign;
        }
    } else if (exp == 31) {
        x = sign | 0x7F800000u | (mant << 13);
    } else {
        x = sign | ((exp + 112) << 23) | (mant << 13);
    }
    float f;
    memcpy(&f, &x, 4);
    return f;
}

void ref_cast_f32_f16(const float* x, int64_t n, uint16_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = ref_f32_to_f16(x[i]);
}

/* ------------------------------------------------------------------------- */
/* GEMMs.  Layout convention for every GEMM here and on the device:            */
/*   C[m, n] = sum_k A[m, k] * B[n, k]   (both operands K-contiguous, "TN")    */
/* which is Y = X W^T for a Linear with X [M, K] and W [N, K].                 */
/* ------------------------------------------------------------------------- */

/* Exact int8 x int8 -> int32 (INT32 accumulation). */
void ref_gemm_s8_tn(const int8_t* a, const int8_t* b, int64_t M, int64_t N, int64_t K,
                    int32_t* c) {
#pragma omp parallel for schedule(static) collapse(2)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t n = 0; n < N; ++n) {
            const int8_t* ar = a + m * K;
            const int8_t* br = b + n * K;
            int32_t acc = 0;
#pragma omp simd reduction(+ : acc)
            for (int64_t k = 0; k < K; ++k) acc += (int32_t)ar[k] * (int32_t)br[k];
            c[m * N + n] = acc;
        }
    }
}

/* Fused-epilogue semantics of the INT8 Linear (PAPER.md:426-427 layer-wise
 * activation x channel-wise weight -> channel-wise dequantizer; graph.hpp:38-40
 * INT8 kernels emit FP32):  y = float(acc) * (s_a * s_w[n]) + bias[n],
 * two rounded FP32 steps, no FMA. bias may be NULL. */
void ref_dequant_epilogue(const int32_t* acc, int64_t M, int64_t N, float s_a, const float* s_w,
                          const float* bias, float* y) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            const float scale = s_a * s_w[n];
            float v = (float)acc[m * N + n] * scale;
            if (bias) v = v + bias[n];
            y[m * N + n] = v;
        }
}

/* FP16 x FP16 with a wide accumulator (FP64 here; the device accumulates in
 * FP32, compared within tolerance).  alpha scales the result (the activation
 * scale of an INT8 op's wgrad). */
void ref_gemm_f16_tn(const uint16_t* a, const uint16_t* b, int64_t M, int64_t N, int64_t K,
                     float alpha, float* c) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k)
                acc += (double)ref_f16_to_f32(a[m * K + k]) * (double)ref_f16_to_f32(b[n * K + k]);
            c[m * N + n] = (float)(acc * (double)alpha);
        }
    }
}

/* FP32 reference GEMM (float inputs, double accumulation). */
void ref_gemm_f32_tn(const float* a, const float* b, int64_t M, int64_t N, int64_t K, float* c) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k) acc += (double)a[m * K + k] * (double)b[n * K + k];
            c[m * N + n] = (float)acc;
        }
}

/* ------------------------------------------------------------------------- */
/* Tensor statistics feeding OpStats (profile.hpp:95-108).                    */
/* out[0] = squared L2 norm (FP64 accumulation), out[1] = absmax,             */
/* out[2] = q = absmax/127 (FP32 scale rule above), out[3] = e = floor(log2   */
/* absmax) (effective exponent; 0 for an all-zero tensor),   */
/* out[4] = numel.                                                             */
/* ------------------------------------------------------------------------- */
void ref_tensor_stats_f32(const float* x, int64_t n, double* out) {
    double ss = 0.0;
    float m = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        ss += (double)x[i] * (double)x[i];
        float a = fabsf(x[i]);
        if (a > m) m = a;
    }
    out[0] = ss;
    out[1] = (double)m;
    out[2] = (double)ref_scale_from_absmax(m);
    out[3] = m > 0.0f ? floor(log2((double)m)) : 0.0;
    out[4] = (double)n;
}

/* ------------------------------------------------------------------------- */
/* Helpers for the Linear oracles: operands are rounded once (to binary16 or   */
/* to their int8 grid values), transposed where the reduction would otherwise  */
/* stride, and every dot product accumulates in FP64 (omp simd reduction: the  */
/* summation order is not pinned -- the device accumulates in FP32 -- these     */
/* outputs are compared within tolerance).                                     */
/* ------------------------------------------------------------------------- */
#include <stdlib.h>

static float* round16(const float* x, int64_t n) {
    float* o = (float*)malloc(sizeof(float) * (size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) o[i] = ref_f16_to_f32(ref_f32_to_f16(x[i]));
    return o;
}

static float* transpose(const float* x, int64_t rows, int64_t cols) {
    float* o = (float*)malloc(sizeof(float) * (size_t)(rows * cols));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < cols; ++c)
        for (int64_t r = 0; r < rows; ++r) o[c * rows + r] = x[r * cols + c];
    return o;
}

static inline double dot(const float* a, const float* b, int64_t n) {
    double acc = 0.0;
#pragma omp simd reduction(+ : acc)
    for (int64_t i = 0; i < n; ++i) acc += (double)a[i] * (double)b[i];
    return acc;
}

/* c[m, n] = sum_k a[m, k] b[n, k] in FP64, times alpha, rounded to FP32. */
static void gemm_tn_f(const float* a, const float* b, int64_t M, int64_t N, int64_t K, double alpha,
                      float* c) {
#pragma omp parallel for schedule(static) collapse(2)
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) c[m * N + n] = (float)(dot(a + m * K, b + n * K, K) * alpha);
}

static void colsum(const float* dy, int64_t M, int64_t N, float* db) {
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        double s = 0.0;
        for (int64_t m = 0; m < M; ++m) s += (double)dy[m * N + n];
        db[n] = (float)s;
    }
}

/* ------------------------------------------------------------------------- */
/* One quantized Linear, forward + backward, exactly the composition the       */
/* device runs:                                             */
/*   fwd  INT8 : xq = Q(x) per-tensor, wq = Q(w) per-channel,                  */
/*               y = (xq wq^T) * s_x * s_w[n] + b           (FP32 out)         */
/*   bwd  FP16 : (cost_mapper.cpp:13-15)  g16 = f16(dy), w16 = f16(w)          */
/*               dx = g16 w16                     (FP16 out, held as float)    */
/*               dw = s_x * g16^T xq              (FP32 out, cost_mapper:48-50)*/
/*               db = sum_m dy                                                 */
/* Shapes: x [M,K], w [N,K], dy [M,N].  Outputs y [M,N], dx [M,K], dw [N,K].   */
/* ------------------------------------------------------------------------- */
void ref_qlinear_int8_fwd_bwd(const float* x, const float* w, const float* bias, const float* dy,
                              int64_t M, int64_t N, int64_t K, int8_t* xq, int8_t* wq,
                              float* s_x, float* s_w, int32_t* acc, float* y, float* dx, float* dw,
                              float* db) {
    ref_quantize_per_tensor(x, M * K, xq, s_x);
    ref_quantize_per_channel(w, N, K, wq, s_w);
    ref_gemm_s8_tn(xq, wq, M, N, K, acc);
    ref_dequant_epilogue(acc, M, N, *s_x, s_w, bias, y);
    if (!dy) return;
    float* g16 = round16(dy, M * N);
    float* w16 = round16(w, N * K);
    float* w16t = transpose(w16, N, K);   /* [K, N] */
    float* g16t = transpose(g16, M, N);   /* [N, M] */
    float* xqf = (float*)malloc(sizeof(float) * (size_t)(M * K));
    for (int64_t i = 0; i < M * K; ++i) xqf[i] = (float)xq[i];
    float* xqt = transpose(xqf, M, K);    /* [K, M] */
    gemm_tn_f(g16, w16t, M, K, N, 1.0, dx);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M * K; ++i) dx[i] = ref_f16_to_f32(ref_f32_to_f16(dx[i]));
    gemm_tn_f(g16t, xqt, N, K, M, (double)*s_x, dw);
    if (db) colsum(dy, M, N, db);
    free(g16); free(w16); free(w16t); free(g16t); free(xqf); free(xqt);
}

/* FP16 Linear, forward + backward (the FP16 kernel of a plan): operands rounded
 * to binary16, wide accumulation, y emitted as FP16 (held as float); backward as
 * the INT8 op's but with the FP16 activation in wgrad and alpha = 1. */
void ref_qlinear_f16_fwd_bwd(const float* x, const float* w, const float* bias, const float* dy,
                             int64_t M, int64_t N, int64_t K, float* y, float* dx, float* dw,
                             float* db) {
    float* x16 = round16(x, M * K);
    float* w16 = round16(w, N * K);
    gemm_tn_f(x16, w16, M, N, K, 1.0, y);
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            float v = y[m * N + n];
            if (bias) v = v + bias[n];
            y[m * N + n] = ref_f16_to_f32(ref_f32_to_f16(v));
        }
    if (dy) {
        float* g16 = round16(dy, M * N);
        float* w16t = transpose(w16, N, K);
        float* g16t = transpose(g16, M, N);
        float* x16t = transpose(x16, M, K);
        gemm_tn_f(g16, w16t, M, K, N, 1.0, dx);
        gemm_tn_f(g16t, x16t, N, K, M, 1.0, dw);
        if (db) colsum(dy, M, N, db);
        free(g16); free(w16t); free(g16t); free(x16t);
    }
    free(x16); free(w16);
}

/* ------------------------------------------------------------------------- */
/* Conv2d as GEMM, NHWC: the column matrix and its adjoint.     */
/* A[(n,p,q),(r,s,c)] = x[n, p*sh-ph+r*dh, q*sw-pw+s*dw, c], 0 outside; K      */
/* padded with zeros to ld.  esz = element size (1 int8, 2 fp16, 4 fp32).       */
/* ------------------------------------------------------------------------- */
void ref_im2col(const void* x, int esz, int64_t N, int64_t H, int64_t W, int64_t C, int R, int S,
                int sh, int sw, int ph, int pw, int dh, int dw, int64_t P, int64_t Q, int64_t ld,
                void* out) {
    const char* xb = (const char*)x;
    char* ob = (char*)out;
    const int64_t K = (int64_t)R * S * C;
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < N * P * Q; ++row) {
        const int64_t q = row % Q, p = (row / Q) % P, n = row / (Q * P);
        memset(ob + row * ld * esz, 0, (size_t)(ld * esz));
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) {
                const int64_t h = p * sh - ph + (int64_t)r * dh, w = q * sw - pw + (int64_t)s * dw;
                if (h < 0 || h >= H || w < 0 || w >= W) continue;
                memcpy(ob + (row * ld + ((int64_t)r * S + s) * C) * esz,
                       xb + (((n * H + h) * W + w) * C) * esz, (size_t)(C * esz));
            }
        (void)K;
    }
}

/* dx[n,h,w,c] = sum of dcol entries that gathered x[n,h,w,c] (FP64 accumulate). */
void ref_col2im(const float* dcol, int64_t N, int64_t H, int64_t W, int64_t C, int R, int S, int sh,
                int sw, int ph, int pw, int dh, int dw, int64_t P, int64_t Q, int64_t ld,
                float* dx) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N * H * W * C; ++i) {
        const int64_t c = i % C, w = (i / C) % W, h = (i / (C * W)) % H, n = i / (C * W * H);
        double acc = 0.0;
        for (int r = 0; r < R; ++r) {
            const int64_t hp = h + ph - (int64_t)r * dh;
            if (hp < 0 || hp % sh) continue;
            const int64_t p = hp / sh;
            if (p >= P) continue;
            for (int s = 0; s < S; ++s) {
                const int64_t wq = w + pw - (int64_t)s * dw;
                if (wq < 0 || wq % sw) continue;
                const int64_t q = wq / sw;
                if (q >= Q) continue;
                acc += dcol[((n * P + p) * Q + q) * ld + ((int64_t)r * S + s) * C + c];
            }
        }
        dx[i] = (float)acc;
    }
}

int ref_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

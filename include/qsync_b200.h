/*
 * qsync_b200.h -- C ABI of the B200-native QSync quantized-operator hot path.
 *
 * Every entry point:
 *   - is extern "C", takes plain pointers/sizes, never throws;
 *   - returns an int status: QSYNC_OK (0) or (qsync::ErrorKind + 1), the kinds of
 *     reference errors.hpp:11-26, so a C++ caller re-raises with
 *     qsync::fail(ErrorKind(status - 1), qsync_last_error()) (errors.hpp:42-44);
 *     CUDA failures map to QSYNC_ERR_INTERNAL;
 *   - works on caller-owned DEVICE buffers, stream-ordered on `stream`
 *     (a cudaStream_t; NULL = legacy default stream), and allocates nothing;
 *   - is reentrant per stream.
 *
 * The reference (/root/reference/proj) has no tensor-level API: its hot path is
 * consumed as measured costs.  Each entry cites the reference
 * semantics it implements or the reference interface it replaces.
 *
 * GEMM convention for every GEMM entry:  C[m,n] = sum_k A[m,k] * B[n,k]
 * (row-major, both operands K-contiguous), i.e. Y = X W^T for X [M,K], W [N,K].
 */
#ifndef QSYNC_B200_H
#define QSYNC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* qsync_stream_t; /* cudaStream_t */

/* Status codes: ErrorKind (errors.hpp:11-26) + 1. */
enum qsync_status {
    QSYNC_OK = 0,
    QSYNC_ERR_GRAPH_CYCLE = 1,
    QSYNC_ERR_VALIDATION = 2,
    QSYNC_ERR_REFERENCE = 3,
    QSYNC_ERR_DOMAIN = 4,
    QSYNC_ERR_MISSING_PROFILE = 5,
    QSYNC_ERR_MISSING_MODEL = 6,
    QSYNC_ERR_DEGENERATE_FIT = 7,
    QSYNC_ERR_STATS_INCOMPLETE = 8,
    QSYNC_ERR_KIND_MISMATCH = 9,
    QSYNC_ERR_TOPOLOGY = 10,
    QSYNC_ERR_ENUMERATION_LIMIT = 11,
    QSYNC_ERR_INFEASIBLE = 12,
    QSYNC_ERR_IO = 13,
    QSYNC_ERR_INTERNAL = 14
};

/* Element types for the typed entries. */
enum qsync_dtype { QSYNC_F32 = 0, QSYNC_F16 = 1, QSYNC_BF16 = 2, QSYNC_I8 = 3, QSYNC_I32 = 4, QSYNC_F8E4M3 = 5 };

/* "<kind>: message" of the last failure on this host thread (errors.hpp:33). */
const char* qsync_last_error(void);
/* Kind tag of a status, as error_kind_name (errors.cpp:5-23). */
const char* qsync_status_name(int status);
int qsync_abi_version(void);
/* Kernels this library has launched in the process (diagnostics / bench). */
unsigned long long qsync_launch_count(void);
/* Number of SMs of the current device (grid sizing), or -1. */
int qsync_device_sm_count(void);

/* ---------------------------------------------------------------------------
 * K1  absmax -> scale.  The paper's two-step minmax; the
 * scale rule s = absmax/127 (s = 1 for an all-zero tensor) is the symmetric
 * fixed-point grid x_bar = (x - z)/q of PAPER.md:342 with z = 0.
 * ------------------------------------------------------------------------- */
/* absmax over n FP32/FP16/BF16 values into *absmax (device float). */
int qsync_absmax(const void* x, int dtype, int64_t n, float* absmax, qsync_stream_t stream);
/* absmax of every row of a [rows, cols] matrix (per-channel). */
int qsync_absmax_rows(const void* x, int dtype, int64_t rows, int64_t cols, float* absmax_rows,
                      qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * K2  quantize to INT8 (round-to-nearest-even, saturating to +-127).
 * q = sat(rint(x / s)), s derived from absmax as above, FP32 IEEE division.
 * ------------------------------------------------------------------------- */
/* Per-tensor: absmax + scale + quantize of a [rows, cols] matrix.  `scale` is a
 * device float[2]: scale[0] receives s, scale[1] the absmax.  If q_t != NULL the
 * same quantized values are also written transposed, as q_t_dtype QSYNC_I8 (the
 * 1-byte activation an INT8 op keeps for backward) or QSYNC_F16 integers,
 * [cols, rows] with row pitch ld_t
 * (>= rows, 0 = rows; pad columns untouched) -- the saved activation operand of
 * the FP16 wgrad GEMM (cost_mapper.cpp:13-15), whose K (= rows) must be padded
 * to a multiple of 8 for TMA. */
int qsync_quantize_per_tensor(const void* x, int dtype, int64_t rows, int64_t cols, int8_t* q,
                              float* scale, void* q_t, int q_t_dtype, int64_t ld_t,
                              qsync_stream_t stream);
/* Quantize with a scale already on the device (e.g. delayed / shared scale). */
int qsync_quantize_with_scale(const void* x, int dtype, int64_t n, const float* scale, int8_t* q,
                              qsync_stream_t stream);
/* Per-channel over rows of W [rows, cols] (PAPER.md:426-427 channel-wise
 * weight).  scales[rows] receives s_r.  If w_t_f16 != NULL, W itself (not the
 * quantized copy) is also cast to FP16 transposed [cols, rows] -- the dgrad
 * weight operand of the FP16 backward. */
int qsync_quantize_per_channel(const float* w, int64_t rows, int64_t cols, int8_t* q,
                               float* scales, uint16_t* w_t_f16, qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * K9  stochastic rounding on the reference RNG stream.
 * Element i consumes draw i of std::mt19937_64(seed) (indicator.cpp:179-187,
 * rng.hpp:12-14), reproduced on the device by GF(2) jump-ahead.
 * ------------------------------------------------------------------------- */
/* Exact device restatement of qsync::stochastic_round (indicator.cpp:176-193):
 * FP64 in, int64 rounded + FP64 dequantized out, no clamp.  Domain if q <= 0. */
int qsync_stochastic_round_f64(const double* x, int64_t n, double q, double zp, uint64_t seed,
                               int64_t* rounded, double* dequantized, qsync_stream_t stream);
/* qsync::stochastic_round_float (indicator.cpp:195-200): spacing 2^(e-k). */
int qsync_stochastic_round_float_f64(const double* x, int64_t n, int e, int k, uint64_t seed,
                                     double* out, qsync_stream_t stream);
/* FP32 -> INT8 SR quantization with a device scale (promoted to FP64 as the
 * reference does), saturated to +-127. */
int qsync_quantize_sr(const float* x, int64_t n, const float* scale, uint64_t seed, int8_t* q,
                      qsync_stream_t stream);
/* Raw stream: out[i] = draw (offset + i) of mt19937_64(seed). */
int qsync_mt64_draws(uint64_t seed, uint64_t offset, int64_t n, uint64_t* out,
                     qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * K3  dequantize: out = float(q) * s.
 * ------------------------------------------------------------------------- */
int qsync_dequantize_per_tensor(const int8_t* q, int64_t n, const float* scale, float* out,
                                qsync_stream_t stream);
int qsync_dequantize_per_channel(const int8_t* q, int64_t rows, int64_t cols, const float* scales,
                                 float* out, qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * K4  float casts (CastScheme::FloatToFloat, profile.hpp:19).  RNE.  Also
 * I8 / F8E4M3 -> F16/F32 (exact): the FP16 backward's view of a saved INT8 / FP8
 * activation.
 * ------------------------------------------------------------------------- */
int qsync_cast(const void* x, int src_dtype, void* out, int dst_dtype, int64_t n,
               qsync_stream_t stream);
/* [rows, cols] FP32/FP16 -> FP16 copy (optional), FP16 transposed [cols, rows]
 * (optional, row pitch ld_t >= rows, 0 = rows) and FP32 column sums
 * (optional; the bias gradient of a Linear),
 * added into `colsum` when colsum_accumulate != 0, else overwriting it.
 * This is the backward entry of an INT8/FP16 op: the incoming gradient is cast
 * to the FP16 backward format (cost_mapper.cpp:13-15) for dgrad and wgrad. */
int qsync_cast_transpose(const void* x, int dtype, int64_t rows, int64_t cols, uint16_t* out,
                         uint16_t* out_t, int64_t ld_t, float* colsum, int colsum_accumulate,
                         qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * K5  fused tensor statistics for OpStats (profile.hpp:95-108).
 * out[0] = ||x||^2 (FP64 accumulation)   -> norm_*_sq
 * out[1] = absmax
 * out[2] = q = absmax/127                -> q_act / q_w
 * out[3] = e = floor(log2(absmax))       -> e_act / e_w / e_grad
 * out[4] = numel                         -> d_act / d_w / d_grad
 * `out` is a device double[5]; `workspace` a device buffer of
 * qsync_stats_workspace_bytes() bytes.
 * ------------------------------------------------------------------------- */
size_t qsync_stats_workspace_bytes(void);
int qsync_tensor_stats(const void* x, int dtype, int64_t n, double* out, void* workspace,
                       qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * K6  INT8 GEMM on tcgen05 (kind::i8, int32 accumulators in TMEM, TMA-fed).
 * A [M,K] int8, B [N,K] int8, K % 16 == 0.
 *   c_i32 != NULL : raw int32 accumulators [M,N] (bit-exact parity output);
 *   c_f32 != NULL : fused dequant epilogue (graph.hpp:38-40: INT8 emits FP32)
 *                   c = float(acc) * (scale_a[0] * scale_b[n]) (+ bias[n]).
 *   scale_b may be per-row (b_per_channel=1, [N]) or a device scalar.
 * ------------------------------------------------------------------------- */
int qsync_gemm_s8(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k,
                  int32_t* c_i32, float* c_f32, const float* scale_a, const float* scale_b,
                  int b_per_channel, const float* bias, qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * FP8 rung of the precision ladder: E4M3 operands on the
 * tcgen05 kind::f8f6f4 tensor cores, FP32 accumulators, the same dequant
 * epilogue as K6 (c = acc * (scale_a[0] * scale_b[n]) + bias[n]).  Quantizers:
 * s = absmax / 448, q = e4m3_rn_satfinite(x / s); per tensor (absmax from
 * qsync_absmax) or per row (weights).  K % 16 == 0.
 * ------------------------------------------------------------------------- */
int qsync_gemm_f8(const uint8_t* a, const uint8_t* b, int64_t m, int64_t n, int64_t k, void* c, int c_dtype,
                  const float* scale_a, const float* scale_b, int b_per_channel, const float* bias,
                  qsync_stream_t stream);
int qsync_quantize_fp8(const void* x, int dtype, int64_t n, const float* absmax, uint8_t* q, float* scale_out,
                       qsync_stream_t stream);
int qsync_quantize_fp8_rows(const float* w, int64_t rows, int64_t cols, uint8_t* q, float* scales,
                            qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * K7  FP16/BF16 GEMM on tcgen05 (kind::f16, FP32 accumulators in TMEM).
 * A [M,K], B [N,K] of ab_dtype (QSYNC_F16 / QSYNC_BF16), K % 8 == 0.
 * c = alpha * (alpha_dev ? *alpha_dev : 1) * acc (+ bias[n]) (+ c if accumulate)
 * written as c_dtype (QSYNC_F32 or QSYNC_F16 / QSYNC_BF16).
 * layout: 0 = A [M,K] and B [N,K] (K-major); 2 = B stored [K,N] (MN-major);
 * 3 = A stored [K,M] and B stored [K,N] (both MN-major).  With MN-major operands
 * the backward needs no transposed copies: dgrad reads W [N_out,K_in] as
 * MN-major B, wgrad reads dY [M,N_out] and X [M,K_in] as MN-major A and B.
 * Used for FP16 forward, dgrad (FP16 out) and wgrad (FP32 out, alpha_dev = the
 * activation scale of an INT8 op; cost_mapper.cpp:48-50).
 * ------------------------------------------------------------------------- */
int qsync_gemm_f16(const void* a, const void* b, int ab_dtype, int64_t m, int64_t n, int64_t k,
                   void* c, int c_dtype, float alpha, const float* alpha_dev, const float* bias,
                   int accumulate, int layout, qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * FP32 operator kernel on the tensor cores (the training devices' plan: they
 * stay FP32, replayer.cpp:96-101).  3xTF32: each FP32 operand is split into
 * hi = rna_tf32(x) and lo = rna_tf32(x - hi) (|x - hi - lo| <= 2^-22 |x|), and
 * one tcgen05 kind::tf32 GEMM over K' = 3K computes hi*hi + hi*lo + lo*hi with
 * FP32 accumulation -- FP32-level accuracy (the dropped lo*lo term is 2^-22).
 * Same operand convention, layouts (0 / 2 / 3), alpha / bias / accumulate as
 * qsync_gemm_f16; FP32 output.  workspace: caller-owned device buffer of
 * qsync_gemm_f32_workspace_bytes(m, n, k) bytes (the split operands).
 * ------------------------------------------------------------------------- */
size_t qsync_gemm_f32_workspace_bytes(int64_t m, int64_t n, int64_t k);
int qsync_gemm_f32(const float* a, const float* b, int64_t m, int64_t n, int64_t k, float* c, float alpha,
                   const float* alpha_dev, const float* bias, int accumulate, int layout, void* workspace,
                   qsync_stream_t stream);
/* The pieces: the split of x [rows, k] (transpose = 1: x stored [k, rows]) into
 * out [rows, 3 kp] = (hi, hi, lo) (order 0, the A operand) or (hi, lo, hi)
 * (order 1, B), each part zero-padded to kp = k rounded up to 4; and the
 * K-major TF32 GEMM (operands read as TF32, K % 4 == 0). */
int qsync_split_tf32x3(const float* x, int64_t rows, int64_t k, int transpose, int order, float* out,
                       qsync_stream_t stream);
int qsync_gemm_tf32(const float* a, const float* b, int64_t m, int64_t n, int64_t k, float* c, float alpha,
                    const float* alpha_dev, const float* bias, int accumulate, qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * K8  Conv2d as GEMM, NHWC.  The column matrix
 * A[(n,p,q), (r,s,c)] = x[n, p*sh-ph+r*dh, q*sw-pw+s*dw, c] (0 outside) is the
 * K-major operand of qsync_gemm_s8 / qsync_gemm_f16 (weights [Cout, R*S*C],
 * i.e. KRSC); `ld` is its row pitch (>= R*S*C, zero padded; 16-byte multiple
 * for TMA).  col2im is the deterministic gather adjoint (dgrad), FP32 out.
 * ------------------------------------------------------------------------- */
int qsync_conv_out_size(int64_t H, int64_t W, int R, int S, int sh, int sw, int ph, int pw, int dh,
                        int dw, int64_t* P, int64_t* Q);
int qsync_im2col(const void* x, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R, int S,
                 int sh, int sw, int ph, int pw, int dh, int dw, void* out, int64_t ld,
                 qsync_stream_t stream);
int qsync_col2im(const void* dcol, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R,
                 int S, int sh, int sw, int ph, int pw, int dh, int dw, int64_t ld, float* dx,
                 qsync_stream_t stream);

/* Implicit-GEMM Conv2d (replaces the im2col + GEMM pair of the reference's
 * quantized conv, graph.hpp:38-40 / cost_mapper.cpp:13-15): the GEMM's producer
 * warp gathers the column tiles straight from the NHWC tensor, nothing is
 * materialised.  Dilation 1.
 *   fwd:   y[(n,p,q), k] = sum x[n, p*sh-ph+r, q*sw-pw+s, c] w[k,(r,s,c)]
 *          x I8 (dequant epilogue with scale_a / scale_b, as qsync_gemm_s8) or
 *          F16/BF16; needs C * elem % 128 == 0.  y [N*P*Q, cout] y_dtype.
 *   dgrad: dx[(n,h,w), c] = sum dy[n, (h+ph-r)/sh, (w+pw-s)/sw, k] w[k,r,s,c]
 *          (terms off the stride grid vanish); dy F16/BF16 [N,P,Q,cout] with
 *          cout % 64 == 0, w [cout, R, S, C] (unpadded, C % 8 == 0), dx
 *          [N*H*W, C] dx_dtype.
 *   wgrad: dw[k, (r,s,c)] (+)= alpha * alpha_dev * sum dy[(n,p,q), k] *
 *          x[n, p*sh-ph+r, q*sw-pw+s, c]; x F16/BF16 with C % 64 == 0, dy
 *          [N*P*Q, cout] (cout % 8 == 0), dw FP32 [cout, R*S*C]; accumulate != 0
 *          adds into dw (the K = pixels reduction is then split across SMs). */
int qsync_conv_fwd_implicit(const void* x, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R,
                            int S, int sh, int sw, int ph, int pw, const void* w, int64_t cout, void* y,
                            int y_dtype, const float* scale_a, const float* scale_b, int b_per_channel,
                            const float* bias, qsync_stream_t stream);
int qsync_conv_dgrad_implicit(const void* dy, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R,
                              int S, int sh, int sw, int ph, int pw, const void* w, int64_t cout, void* dx,
                              int dx_dtype, qsync_stream_t stream);
int qsync_conv_wgrad_implicit(const void* x, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R,
                              int S, int sh, int sw, int ph, int pw, const void* dy, int64_t cout, float* dw,
                              float alpha, const float* alpha_dev, int accumulate, qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * Glue between planned operators: fused residual add + LayerNorm.
 * fwd: s = a + b (b FP32 or FP16 [rows, cols], may be NULL), y = LN(s) with
 *      gamma/beta; saves s (optional), mean[rows], rstd[rows].
 * bwd: dx from dy; dgamma/dbeta ADDED into the given FP32 buffers.
 * 128 <= cols <= 1024, cols % 128 == 0.
 * ------------------------------------------------------------------------- */
int qsync_layernorm_fwd(const float* a, const void* b, int b_dtype, const float* gamma,
                        const float* beta, int64_t rows, int64_t cols, float eps, float* s_out,
                        float* y, float* mean, float* rstd, qsync_stream_t stream);
int qsync_layernorm_bwd(const float* dy, const float* s, const float* mean, const float* rstd,
                        const float* gamma, int64_t rows, int64_t cols, float* dx, float* dgamma,
                        float* dbeta, qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * Fused encoder-layer glue (the operators between two planned Linears fold
 * into the kernels that produce / consume the planned operand format).
 * ------------------------------------------------------------------------- */
enum qsync_act { QSYNC_ACT_NONE = 0, QSYNC_ACT_GELU = 1, QSYNC_ACT_DERIV = 2 };

/* LayerNorm forward that also emits what the NEXT planned Linear consumes:
 * y16 (optional) = FP16(y) for an FP16 op; y_absmax (optional, device float,
 * overwritten) = absmax(y) for an INT8 op, so its per-tensor quantizer is one
 * pass (qsync_quantize_act).  Same y / s / mean / rstd as qsync_layernorm_fwd. */
int qsync_layernorm_fwd_ex(const float* a, const void* b, int b_dtype, const float* gamma,
                           const float* beta, int64_t rows, int64_t cols, float eps, float* s_out,
                           float* y, float* mean, float* rstd, uint16_t* y16, float* y_absmax,
                           qsync_stream_t stream);
/* LayerNorm forward fused with the per-tensor INT8 quantizer of y (the input of
 * an INT8-planned Linear): y, s_out, mean, rstd as qsync_layernorm_fwd_ex, q =
 * RNE int8 of y with s = absmax(y)/127, q16 (optional) = FP16(q), scale[0] = s,
 * scale[1] = absmax -- bit-identical to qsync_layernorm_fwd_ex(.., y_absmax)
 * followed by qsync_quantize_act_ex.  One kernel when one row per warp fits
 * co-resident (the rows stay in registers across a grid barrier on absmax),
 * else those two launches. */
int qsync_layernorm_fwd_quant(const float* a, const void* b, int b_dtype, const float* gamma, const float* beta,
                              int64_t rows, int64_t cols, float eps, float* s_out, float* y, float* mean,
                              float* rstd, int8_t* q, uint16_t* q16, float* scale, qsync_stream_t stream);
/* LayerNorm backward that also emits the incoming gradient of the Linear that
 * produced the residual branch: dx16 (optional) = FP16(dx), the FP16 backward
 * format (cost_mapper.cpp:13-15), and dcolsum (optional) += sum_rows dx, that
 * Linear's bias gradient. */
int qsync_layernorm_bwd_ex(const float* dy, const float* s, const float* mean, const float* rstd,
                           const float* gamma, int64_t rows, int64_t cols, float* dx, float* dgamma,
                           float* dbeta, uint16_t* dx16, float* dcolsum, qsync_stream_t stream);

/* Embedding + LayerNorm of the encoder input: row r's input is
 * word[tokens[r]] + pos[r % seq] + typ[0] (gathered, never materialised), then
 * LayerNorm as qsync_layernorm_fwd_ex (s_out, mean, rstd saved; optional y16 /
 * y_absmax for the first planned op).  The backward scatter-adds the row
 * gradients into dword[tokens[r]] and dpos[r % seq] (vector reductions), adds
 * their column sums into dtyp, and dgamma / dbeta as qsync_layernorm_bwd. */
int qsync_embed_layernorm_fwd(const int64_t* tokens, int64_t rows, int64_t seq, const float* word,
                              const float* pos, const float* typ, const float* gamma, const float* beta,
                              int64_t cols, float eps, float* s_out, float* y, float* mean, float* rstd,
                              uint16_t* y16, float* y_absmax, qsync_stream_t stream);
/* qsync_embed_layernorm_fwd fused with the INT8 quantizer of y, as
 * qsync_layernorm_fwd_quant. */
int qsync_embed_layernorm_fwd_quant(const int64_t* tokens, int64_t rows, int64_t seq, const float* word,
                                    const float* pos, const float* typ, const float* gamma, const float* beta,
                                    int64_t cols, float eps, float* s_out, float* y, float* mean, float* rstd,
                                    int8_t* q, uint16_t* q16, float* scale, qsync_stream_t stream);
int qsync_embed_layernorm_bwd(const float* dy, const float* s, const float* mean, const float* rstd,
                              const float* gamma, const int64_t* tokens, int64_t rows, int64_t seq, int64_t cols,
                              float* dgamma, float* dbeta, float* dword, float* dpos, float* dtyp,
                              qsync_stream_t stream);

/* absmax of act(x) over n values (device float, overwritten). */
int qsync_absmax_act(const void* x, int dtype, int64_t n, int act, float* absmax,
                     qsync_stream_t stream);
/* Per-tensor RNE quantize of act(x) with s = absmax/127 from a device absmax
 * computed upstream (LayerNorm epilogue / qsync_absmax_act); *scale_out = s.
 * dact_out (optional, FP16) receives act'(x) for the backward (QSYNC_ACT_DERIV). */
int qsync_quantize_act(const void* x, int dtype, int64_t n, int act, const float* absmax, int8_t* q,
                       float* scale_out, uint16_t* dact_out, qsync_stream_t stream);
/* The same, also writing q16_out (optional) = FP16(q): the grid values exactly,
 * the operand the op's FP16 wgrad reads in the backward (no separate cast). */
int qsync_quantize_act_ex(const void* x, int dtype, int64_t n, int act, const float* absmax, int8_t* q,
                          float* scale_out, uint16_t* dact_out, uint16_t* q16_out, qsync_stream_t stream);
/* y = GELU(x) in x's format (F32 / F16: the value the GELU-prologue quantizer
 * would quantize), dact_out (optional, F16) = GELU'(x) from the same erf, and
 * *absmax (device float, overwritten) = max |y|.  FF2's INT8 operand is then
 * qsync_quantize_act(y, ..., QSYNC_ACT_NONE): bit-identical q and s to the
 * GELU-prologue form, with one GELU evaluation instead of two. */
int qsync_gelu_absmax_store(const void* x, int dtype, int64_t n, float* absmax, void* y, uint16_t* dact_out,
                            qsync_stream_t stream);
/* out = act(x) cast to dst_dtype (F32/F16 -> F32/F16); optional FP16 act'(x). */
int qsync_act_cast(const void* x, int src_dtype, void* out, int dst_dtype, int64_t n, int act,
                   uint16_t* dact_out, qsync_stream_t stream);
/* Backward through act and into a planned op's FP16 backward format:
 * g = dy * act'(h) (act NONE: g = dy, h may be NULL; act DERIV: h is the FP16
 * act'(x) the forward stored, g = dy * h), out (optional) = g as
 * out_dtype, colsum (optional) += sum_rows g (the bias gradient).  dy, h
 * [rows, cols] F32/F16; with act NONE, dy and out may also be BF16 (the BF16
 * backward entry of a BF16-planned op). */
int qsync_act_bwd_colsum(const void* dy, int dy_dtype, const void* h, int h_dtype, int64_t rows,
                         int64_t cols, int act, void* out, int out_dtype, float* colsum,
                         qsync_stream_t stream);

/* INT8 GEMM with the dequant epilogue written as c_dtype (F32 = the
 * graph.hpp:38-40 format; F16 when the consumer is an FP16 kernel, e.g. the
 * attention core -- the same FP32 value rounded once, so it equals
 * qsync_gemm_s8 followed by qsync_cast). */
int qsync_gemm_s8_ex(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k, void* c,
                     int c_dtype, const float* scale_a, const float* scale_b, int b_per_channel,
                     const float* bias, qsync_stream_t stream);

/* An encoder layer's FF1 with the GELU that follows it in the GEMM epilogue
 * (the work of the FF2 operand kernels qsync_act_cast / qsync_gelu_absmax_store,
 * minus the quantization, which needs the finished absmax).  ab_dtype I8: the
 * qsync_gemm_s8_ex dequant epilogue (scale_a, scale_b, bias) gives y in FP32;
 * F16/BF16: y = the qsync_gemm_f16 value rounded to FP16 (what the FP16 op
 * stores).  Then g = gelu(y) (erf form), rounded to y's dtype and stored as
 * g_dtype (F32 or F16); dact [m, n] FP16 = gelu'(y) (for the backward); and
 * *absmax (device float, overwritten) = max |g| -- the FF2 quantizer's input.
 * Bit-identical to the unfused GEMM followed by those kernels.  n % 8 == 0,
 * g and dact 16-byte aligned. */
int qsync_gemm_gelu(const void* a, const void* b, int ab_dtype, int64_t m, int64_t n, int64_t k,
                    const float* scale_a, const float* scale_b, int b_per_channel, const float* bias, void* g,
                    int g_dtype, uint16_t* dact, float* absmax, qsync_stream_t stream);

/* An INT8 FF1 feeding an INT8 FF2 without storing GELU(h):
 *   qsync_gemm_s8_ymax: qsync_gemm_s8_ex with FP32 output that also writes
 *     *ymax (overwritten) = max(0, max over the outputs y);
 *   qsync_gelu_quantize: FF2's operand from h (FP32) in one pass -- q = INT8 of
 *     gelu(h) with s = absmax(gelu(h)) / 127, q16 (optional) = FP16 of the grid
 *     values, dact (optional) = FP16 gelu'(h), scale_out[0] = s, [1] = absmax.
 *     gelu is non-decreasing where it exceeds 0.1701 and below that for every
 *     h < 0 (qsync_gelu_fp32_check), so absmax = gelu(hmax) when that is >= 0.1701
 *     and no absmax pass is needed; otherwise the kernel reduces it exactly
 *     first.  Bit-identical to qsync_gelu_absmax_store + qsync_quantize_act_ex.
 *   qsync_gelu_fp32_check: out[0] += monotonicity violations over every float32
 *     in [0, 16] above 0.1701, out[1] = max |gelu(h)| over h < 0 (float bits);
 *     out zeroed by the caller (a self-check for the tests). */
int qsync_gemm_s8_ymax(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k, float* c,
                       const float* scale_a, const float* scale_b, int b_per_channel, const float* bias, float* ymax,
                       qsync_stream_t stream);
int qsync_gelu_quantize(const float* h, int64_t n, const float* hmax, int8_t* q, uint16_t* q16, uint16_t* dact_out,
                        float* scale_out, qsync_stream_t stream);
int qsync_gelu_fp32_check(unsigned* out);

/* The classification head around the encoder stack (FP32 ops; train_step.py:
 * pooler = tanh(x[:, 0] Wp^T + bp), logits = pooled Wc^T + bc, loss = mean
 * cross entropy), so the graphed step launches only this library's kernels.
 * x [B, S, H] FP32; Wp [H, H], Wc [C, H]; labels [B] int64.  Forward writes
 * pooled [B, H], probs [B, C] (softmax, kept for the backward) and *loss.
 * Backward (dloss a device scalar) ADDS into dwp / dbp / dwc / dbc (the flat
 * FP32 gradient buffer), uses dpre [9 * B * H] floats as scratch and writes all of
 * dx [B, S, H] (zero except token 0).  Deterministic (fixed reduction order). */
int qsync_cls_head_fwd(const float* x, int64_t B, int64_t S, int64_t H, const float* wp, const float* bp,
                       const float* wc, const float* bc, int64_t C, const int64_t* labels, float* pooled,
                       float* probs, float* loss, qsync_stream_t stream);
int qsync_cls_head_bwd(const float* x, int64_t B, int64_t S, int64_t H, const float* wp, const float* wc, int64_t C,
                       const int64_t* labels, const float* pooled, const float* probs, const float* dloss,
                       float* dwp, float* dbp, float* dwc, float* dbc, float* dpre, float* dx,
                       qsync_stream_t stream);
/* Zero `bytes` bytes (16-byte vector stores when aligned), as a PDL kernel: the
 * per-step gradient-buffer reset inside the graphed step. */
int qsync_zero(void* p, int64_t bytes, qsync_stream_t stream);

/* Attention core softmax(Q K^T scale) V of an encoder layer (stays
 * floating point), in the planned projections' formats: qkv packed
 * [B, S, 3, H, D] FP16 (the QKV projection's output), out [B, S, H, D] FP16,
 * lse [B, H, S] FP32 (row log-sum-exp, kept for the backward), out_absmax
 * (optional, device float, overwritten) = absmax(out) for an INT8 O projection.
 * Backward: dqkv packed like qkv from dout [B, S, H, D].  S = 128, D = 64. */
int qsync_attention_fwd(const void* qkv, int64_t B, int64_t S, int64_t H, int64_t D, float scale, void* out,
                        float* lse, float* out_absmax, qsync_stream_t stream);
/* Attention forward for an INT8 O projection: also quantizes out per tensor --
 * q [B, S, H, D] int8, q16 (optional) = FP16 of the grid values (the wgrad
 * operand), qscale[0] = scale, qscale[1] = absmax(out).  One kernel (a grid
 * barrier over the co-resident (batch, head) blocks) when they all fit, else
 * qsync_attention_fwd + qsync_quantize_act_ex; the same bits either way. */
int qsync_attention_fwd_quant(const void* qkv, int64_t B, int64_t S, int64_t H, int64_t D, float scale, void* out,
                              float* lse, int8_t* q, uint16_t* q16, float* qscale, qsync_stream_t stream);
int qsync_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse, int64_t B,
                        int64_t S, int64_t H, int64_t D, float scale, void* dqkv, qsync_stream_t stream);

/* ---------------------------------------------------------------------------
 * Optimizer on FP32 master weights fused with the per-step weight preparation
 * of the planned kernels: AdamW (decoupled weight decay, bias-corrected, step
 * counter on the device) over a table of parameter segments, each optionally
 * emitting w16 = FP16(W) and/or wq = per-row INT8 quantization of W with its
 * scales (the operands the next step's INT8 / FP16 Linears read).  With
 * lr_scale = 0 ... no: `update` = 0 only (re)computes the prepared copies.
 * ------------------------------------------------------------------------- */
typedef struct qsync_adamw_seg {
    float* p;          /* FP32 master weights [rows, cols] */
    const float* g;    /* FP32 gradient (same layout) */
    float* m;          /* first moment */
    float* v;          /* second moment */
    uint16_t* w16;     /* optional FP16 copy */
    int8_t* wq;        /* optional per-row INT8 copy */
    float* wscale;     /* [rows] scales of wq */
    int64_t rows;
    int64_t cols;
} qsync_adamw_seg;
/* segs: DEVICE array of nseg segments; seg_row_start: DEVICE int64[nseg + 1]
 * prefix sums of the segments' rows (total_rows = last entry); step: device
 * int64 counter, incremented once per call with update != 0 (the bias
 * corrections use the incremented value, as torch.optim.AdamW). */
int qsync_adamw_step(const qsync_adamw_seg* segs, int nseg, const int64_t* seg_row_start,
                     int64_t total_rows, int64_t* step, float lr, float beta1, float beta2,
                     float eps, float weight_decay, int update, qsync_stream_t stream);
/* The same update over the global rows [row_begin, row_end) only (a gradient
 * bucket whose parameters are final -- the optimizer then overlaps the rest of
 * the backward), reading the step counter without advancing it; call
 * qsync_adamw_advance once after every range of the step has been enqueued. */
int qsync_adamw_step_range(const qsync_adamw_seg* segs, int nseg, const int64_t* seg_row_start,
                           int64_t row_begin, int64_t row_end, const int64_t* step, float lr, float beta1,
                           float beta2, float eps, float weight_decay, int update, qsync_stream_t stream);
int qsync_adamw_advance(int64_t* step, qsync_stream_t stream);


/* ---------------------------------------------------------------------------
 * C1  data-parallel gradient exchange over NCCL (NVLink 5 / NVSwitch).
 * The reference models it, it does not run it: per-rank bucket slots
 * {earliest_ready_offset_ns, duration_ns, bucket_bytes} (profile.hpp:118-129),
 * slot n starts at max(every rank ready, end of slot n-1) and the optimizer
 * waits for the last slot (replayer.cpp:48-73).  These entries are that
 * exchange: one communicator per rank (one process per GPU), FP32 buckets
 * reduced in place on the caller's stream, in the order the caller issues them
 * (identical on every rank whatever its precision plan).  NCCL is resolved at
 * run time (the libnccl.so.2 already in the process, else the system one), so
 * the library links no NCCL; failures map to QSYNC_ERR_INTERNAL with NCCL's
 * message, bad arguments to VALIDATION / DOMAIN.  Capturable in a CUDA graph.
 * ------------------------------------------------------------------------- */
#define QSYNC_COMM_ID_BYTES 128
typedef struct qsync_comm_s* qsync_comm_t;
/* A fresh communicator id (rank 0 creates it, the caller broadcasts the bytes). */
int qsync_comm_unique_id(uint8_t id[QSYNC_COMM_ID_BYTES]);
/* Join communicator `id` as `rank` of `nranks` on the CURRENT CUDA device
 * (collective: every rank must call it). */
int qsync_comm_init(qsync_comm_t* comm, int nranks, int rank, const uint8_t id[QSYNC_COMM_ID_BYTES]);
int qsync_comm_destroy(qsync_comm_t comm);
/* nranks / rank / CUDA device of a communicator (any pointer may be NULL). */
int qsync_comm_info(qsync_comm_t comm, int* nranks, int* rank, int* device);
/* In-place all-reduce of `count` FP32 values at `buf` (one gradient bucket):
 * average != 0 -> mean over ranks (ncclAvg), else sum. */
int qsync_allreduce_bucket(qsync_comm_t comm, float* buf, int64_t count, int average, qsync_stream_t stream);
/* NCCL version of the resolved library (e.g. 22809), or -1 if none loads. */
int qsync_comm_nccl_version(void);

#ifdef __cplusplus
}
#endif

#endif /* QSYNC_B200_H */

// common.cuh -- shared helpers of the qsync_b200 device library (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "qsync_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "qsync_b200 is written for sm_100a (B200) only"
#endif

namespace qsb {

// ---- error plumbing (status = ErrorKind + 1, errors.hpp:11-26) -------------
int set_error(int status, const std::string& msg);
int check_launch(const char* what);  // cudaGetLastError -> status
inline int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return QSYNC_OK;
    return set_error(QSYNC_ERR_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}
#define QSB_TRY(expr)                      \
    do {                                   \
        int _st = (expr);                  \
        if (_st != QSYNC_OK) return _st;   \
    } while (0)
#define QSB_REQUIRE(cond, status, msg)                   \
    do {                                                 \
        if (!(cond)) return ::qsb::set_error(status, msg); \
    } while (0)

inline cudaStream_t to_stream(qsync_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-DEVICE property:
// set it once per (kernel, device ordinal) -- a process that launches on a
// second GPU gets the attribute there too (capi.cu).
int ensure_max_dynamic_smem(const void* kernel, int bytes);
// Zero `bytes` (a multiple of 4) as a PDL kernel (keeps the graph's kernel chain).
int zero_async(void* p, int64_t bytes, cudaStream_t st);
// 2-D SWIZZLE_128B TMA map (row pitch = inner * elem_bytes), defined in gemm.cu.
int make_tma_2d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, uint32_t elem_bytes, int64_t inner,
                int64_t outer, uint32_t box_inner, uint32_t box_outer);

// ---- programmatic dependent launch (PDL) -----------------------------------
// Every kernel of this library starts with QSB_PDL_ENTER(): it waits for the
// preceding grid in the stream to complete (griddepcontrol.wait -- a no-op when
// not launched with PDL) and immediately allows the next grid to be scheduled,
// so inside a CUDA graph a kernel's launch and prologue overlap the previous
// kernel's tail.  launch_pdl() launches with the programmatic-serialization
// attribute (qsync_gemm_set_pdl turns it off for A/B runs).
extern int g_pdl_enabled;
#define QSB_PDL_ENTER()                                              \
    do {                                                             \
        asm volatile("griddepcontrol.wait;" ::: "memory");           \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    } while (0)

// Launch with PDL; the caller's check_launch() reports errors (as for <<<>>>).
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl_enabled ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
int launch_pdl(const char* what, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
               Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl_enabled ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) return cuda_status(e, what);
    return check_launch(what);
}

// ---- typed loads ----------------------------------------------------------
template <int DT>
struct Elem;
template <>
struct Elem<QSYNC_F32> {
    using T = float;
    __device__ static float f(T v) { return v; }
};
template <>
struct Elem<QSYNC_F16> {
    using T = __half;
    __device__ static float f(T v) { return __half2float(v); }
};
template <>
struct Elem<QSYNC_BF16> {
    using T = __nv_bfloat16;
    __device__ static float f(T v) { return __bfloat162float(v); }
};

template <>
struct Elem<QSYNC_I8> {
    using T = int8_t;
    __device__ static float f(T v) { return static_cast<float>(v); }
};
template <>
struct Elem<QSYNC_F8E4M3> {
    using T = uint8_t;
    __device__ static float f(T v) {
        const __half_raw h = __nv_cvt_fp8_to_halfraw(static_cast<__nv_fp8_storage_t>(v), __NV_E4M3);
        return __half2float(__half(h));
    }
};

// Scale rule shared by every quantizer: s = absmax / 127 (IEEE), 1 if all-zero.
__device__ __forceinline__ float scale_from_absmax(float a) {
    return a > 0.0f ? __fdiv_rn(a, 127.0f) : 1.0f;
}
// RNE, saturating to the symmetric INT8 grid [-127, 127]: sat(rint(RN(x / s))),
// bit-identical to the oracle's IEEE division, without a division per element.
// QScale carries s and r = RN(1/s) (computed once per tensor / row); then
//   y = RN(x r),  t = RN(x - y s) (one FMA; the remainder is exact),
//   q = RN(t r + y)  (one FMA: Markstein's correction -> the correctly rounded x/s)
// 3 FP ops instead of __fdiv_rn's reciprocal + Newton steps + range check, which
// held the quantizers SM-bound (84% sm__throughput at 1 GiB, r1 profiles).  The
// fast path is taken for s in [2^-90, 2^100] (r finite, every remainder normal);
// |y| >= 256 saturates anyway and skips the correction (no inf - inf).  Other
// scales take the IEEE division.  tests/cpp/recip_check.c checks the identity
// exhaustively over every x with |x / s| in [1/4, 256] for edge and random s.
struct QScale {
    float s, r;  // r == 0: divide
};
__device__ __forceinline__ QScale make_qscale(float s) {
    return {s, (s >= 0x1p-90f && s <= 0x1p+100f) ? __frcp_rn(s) : 0.0f};
}
__device__ __forceinline__ float quot_rn(float x, QScale q) {
    if (q.r == 0.0f) return __fdiv_rn(x, q.s);
    const float y = __fmul_rn(x, q.r);
    const float t = __fmaf_rn(-y, q.s, x);
    return fabsf(y) < 256.0f ? __fmaf_rn(t, q.r, y) : y;
}
// The quantized value is produced as a "grid float": t = RN(clamp(x/s) + 1.5*2^23).
// Every float in [2^23, 2^24) is an integer, so the add is the round-to-nearest-
// even of the clamped quotient, t's bits are 0x4B400000 + q, and -- that
// constant's low byte being 0 -- t's low byte IS the int8 two's-complement byte
// of q.  No FRND / F2I / I2F (quarter-rate conversion pipe) on the path: the
// quantizers were issue-bound on them.  Clamping before rounding equals
// rounding then clamping on [-127, 127] (the bounds are integers); a NaN
// quotient clamps to -127 either way (fmaxf returns the non-NaN operand).
__device__ __forceinline__ float quant_rne_f(float x, QScale q) {
    const float v = fminf(fmaxf(quot_rn(x, q), -127.0f), 127.0f);
    return __fadd_rn(v, 12582912.0f);
}
__device__ __forceinline__ int quant_rne(float x, QScale q) {
    return static_cast<int>(__float_as_uint(quant_rne_f(x, q))) - 0x4B400000;
}
// Four grid floats -> four packed int8 (their low bytes), lowest address first.
__device__ __forceinline__ uint32_t pack_q4(float a, float b, float c, float d) {
    const uint32_t ab = __byte_perm(__float_as_uint(a), __float_as_uint(b), 0x0040);
    const uint32_t cd = __byte_perm(__float_as_uint(c), __float_as_uint(d), 0x0040);
    return __byte_perm(ab, cd, 0x5410);
}
// The grid value q of a grid float, exactly, as a float.
__device__ __forceinline__ float grid_value(float t) { return __fsub_rn(t, 12582912.0f); }


// Two floats -> packed 16-bit pair (one F2FP.PACK_AB instruction), low half first.
__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack_bf162(float lo, float hi) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// GELU (erf form, BERT's activation) and its derivative:
//   gelu(x)  = x Phi(x),           Phi(x) = 0.5 (1 + erf(x / sqrt 2)) = 0.5 erfc(-x / sqrt 2)
//   gelu'(x) = Phi(x) + x phi(x),  phi(x) = exp(-x^2 / 2) / sqrt(2 pi)
// evaluated through ONE exponential: with t = |x| / sqrt 2, erfc(t) =
// exp(-x^2/2) erfcx(t) and erfcx(t) = P11(q) / (1 + 2t), q = (t - 2.5) / (t + 2.5)
// (a degree-11 fit, relative error 1e-8 on [0, 14]; Schonfelder's variable).
// Phi = 1 - erfc/2 for x >= 0, erfc/2 for x < 0 -- no 1 + erf cancellation, so
// gelu keeps its relative accuracy for negative x too.  Float32-emulated sweep
// over [-12, 12] against an erfc-based float64 reference: gelu within 2 ulp
// (6.7 ulp at |x| > 10 where |gelu| < 1e-25), gelu' within 2.1e-7 absolute.
// ~40 instructions and two MUFU ops for both (CUDA's erff + expf pair took
// ~88: the FF2 operand kernels were compute-bound on it): the exponential is
// ex2.approx (<= 2 ulp) of a two-term product x^2/2 * log2(e), the reciprocal
// rcp.approx (1 ulp), which adds ~2 ulp to the sweep's bound.  Every operation
// is an explicit intrinsic so all kernels that evaluate it agree bit for bit.
__device__ __forceinline__ float ex2_approx(float v) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ float rcp_approx(float v) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ void gelu_and_grad(float x, float& g, float& gp) {
    const float t = __fmul_rn(fabsf(x), 0.70710678118654752f);
    const float x2 = __fmul_rn(x, x);
    const float x2lo = __fmaf_rn(x, x, -x2);  // x^2 = x2 + x2lo exactly
    // exp(-x^2/2) = 2^(ph + pl): ph = -x2/2 * log2(e) rounded, pl the rest
    const float arg = __fmul_rn(-0.5f, x2);
    const float ph = __fmul_rn(arg, 1.4426950408889634f);
    const float pl = __fmaf_rn(__fmul_rn(-0.5f, x2lo), 1.4426950408889634f,
                               __fmaf_rn(arg, 1.92596298909109e-08f, __fmaf_rn(arg, 1.4426950408889634f, -ph)));
    const float e0 = ex2_approx(ph);
    const float e = __fmaf_rn(e0, __fmul_rn(pl, 0.69314718055994531f), e0);
    const float a = __fadd_rn(t, 2.5f);
    const float b = __fmaf_rn(2.0f, t, 1.0f);
    const float r = rcp_approx(__fmul_rn(a, b));
    const float q = __fmul_rn(__fmul_rn(__fadd_rn(t, -2.5f), b), r);  // (t - 2.5) / (t + 2.5)
    const float ib = __fmul_rn(a, r);                                  // 1 / (1 + 2t)
    float p = -7.423775969073176e-05f;
    p = __fmaf_rn(p, q, -7.442452624673024e-05f);
    p = __fmaf_rn(p, q, 0.000600203697104007f);
    p = __fmaf_rn(p, q, 0.00048243391211144626f);
    p = __fmaf_rn(p, q, -0.004368482157588005f);
    p = __fmaf_rn(p, q, 0.000934525509364903f);
    p = __fmaf_rn(p, q, 0.032757923007011414f);
    p = __fmaf_rn(p, q, -0.10296733677387238f);
    p = __fmaf_rn(p, q, 0.15763020515441895f);
    p = __fmaf_rn(p, q, -0.09902453422546387f);
    p = __fmaf_rn(p, q, -0.12235677242279053f);
    p = __fmaf_rn(p, q, 1.2648382186889648f);
    const float ec = __fmul_rn(e, __fmul_rn(p, ib));  // erfc(t)
    const float phi = x >= 0.0f ? __fmaf_rn(-0.5f, ec, 1.0f) : __fmul_rn(0.5f, ec);
    g = __fmul_rn(x, phi);
    gp = __fmaf_rn(x, __fmul_rn(e, 0.39894228040143268f), phi);
}
// The 16-bit-input grade (x an FP16 / BF16 value, g rounded to 16 bits): x^2
// is exact for such x, so the exponent needs no compensation, and erfcx a
// degree-8 fit at (t-3)/(t+3) (2.8e-6 relative).  Over all 63488 finite FP16
// inputs (float32 emulation, tools/fits/gelu_erfcx_fit.py) FP16(gelu) differs
// from the correctly rounded value for 71 inputs, by one ulp; ~27 instructions.
__device__ __forceinline__ void gelu_and_grad_h(float x, float& g, float& gp) {
    const float t = __fmul_rn(fabsf(x), 0.70710678118654752f);
    const float e = ex2_approx(__fmul_rn(__fmul_rn(-0.5f, __fmul_rn(x, x)), 1.4426950408889634f));
    const float a = __fadd_rn(t, 3.0f);
    const float b = __fmaf_rn(2.0f, t, 1.0f);
    const float r = rcp_approx(__fmul_rn(a, b));
    const float q = __fmul_rn(__fmul_rn(__fadd_rn(t, -3.0f), b), r);
    const float ib = __fmul_rn(a, r);
    float p = 0.002183391246944666f;
    p = __fmaf_rn(p, q, 0.001770266331732273f);
    p = __fmaf_rn(p, q, -0.02409461885690689f);
    p = __fmaf_rn(p, q, 0.06860112398862839f);
    p = __fmaf_rn(p, q, -0.11917967349290848f);
    p = __fmaf_rn(p, q, 0.1295975148677826f);
    p = __fmaf_rn(p, q, -0.04757000878453255f);
    p = __fmaf_rn(p, q, -0.13561883568763733f);
    p = __fmaf_rn(p, q, 1.2530081272125244f);
    const float ec = __fmul_rn(e, __fmul_rn(p, ib));
    const float phi = x >= 0.0f ? __fmaf_rn(-0.5f, ec, 1.0f) : __fmul_rn(0.5f, ec);
    g = __fmul_rn(x, phi);
    gp = __fmaf_rn(x, __fmul_rn(e, 0.39894228040143268f), phi);
}
// kHalf: the input is a 16-bit value (FP16 / BF16 producer) -> the 16-bit grade.
template <bool kHalf = false>
__device__ __forceinline__ void gelu_pair(float x, float& g, float& gp) {
    if constexpr (kHalf)
        gelu_and_grad_h(x, g, gp);
    else
        gelu_and_grad(x, g, gp);
}
template <bool kHalf = false>
__device__ __forceinline__ float gelu_erf(float x) {
    float g, gp;
    gelu_pair<kHalf>(x, g, gp);
    return g;
}
template <bool kHalf = false>
__device__ __forceinline__ float gelu_erf_grad(float x) {
    float g, gp;
    gelu_pair<kHalf>(x, g, gp);
    return gp;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace qsb

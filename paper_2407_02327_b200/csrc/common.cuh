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

// GELU (erf form, BERT's activation) and its derivative, every operation
// rounded explicitly so that all kernels that evaluate it agree bit for bit:
//   gelu(x)  = 0.5 x (1 + erf(x / sqrt 2))
//   gelu'(x) = 0.5 (1 + erf(x / sqrt 2)) + x exp(-x^2 / 2) / sqrt(2 pi)
__device__ __forceinline__ float gelu_erf(float x) {
    const float e = erff(__fmul_rn(x, 0.70710678118654752f));
    return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.0f, e));
}
// Both at once, sharing the erf (the FF2 operand kernels store GELU'(x) in FP16
// for the backward): g is bit-identical to gelu_erf(x); gp uses the fast
// exponential (it is rounded to FP16 anyway).
__device__ __forceinline__ void gelu_and_grad(float x, float& g, float& gp) {
    const float e1 = __fadd_rn(1.0f, erff(__fmul_rn(x, 0.70710678118654752f)));
    g = __fmul_rn(__fmul_rn(0.5f, x), e1);
    // gp is stored in FP16: the fast exponential's few-ulp error is far below that
    const float pdf = __fmul_rn(__expf(__fmul_rn(-0.5f, __fmul_rn(x, x))), 0.39894228040143268f);
    gp = __fadd_rn(__fmul_rn(0.5f, e1), __fmul_rn(x, pdf));
}
__device__ __forceinline__ float gelu_erf_grad(float x) {
    const float cdf = __fmul_rn(0.5f, __fadd_rn(1.0f, erff(__fmul_rn(x, 0.70710678118654752f))));
    const float pdf = __fmul_rn(expf(__fmul_rn(-0.5f, __fmul_rn(x, x))), 0.39894228040143268f);
    return __fadd_rn(cdf, __fmul_rn(x, pdf));
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

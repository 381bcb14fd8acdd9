// act.cu -- backward through the encoder layer's activation into a planned
// op's FP16 backward format, fused with that op's bias gradient.
//
//   g = dy * act'(h)       (act NONE: g = dy; act DERIV: h already holds act'(x) in
//                           FP16, written by the forward's operand kernel)
//   out = g as out_dtype   (optional; FP16 for an INT8/FP16 op, cost_mapper.cpp:13-15)
//   colsum += sum_rows g   (optional; the Linear's bias gradient, FP32)
//
// Layout: row-major [rows, cols].  A block of 8 warps owns a 256-column strip
// and a chunk of rows sized so the grid is one resident wave; each lane owns 8
// consecutive columns (one 16-byte FP16 vector, two FP32 vectors) and walks
// chunk/8 rows, so every warp access is a contiguous 512 B (FP16) / 1 KB (FP32)
// row segment.  Column partials are reduced through shared memory, then one
// FP32 atomic per column per block.  HBM-bound:
// algorithmic bytes per element = size(dy) + size(h) + size(out).
#include <algorithm>

#include "common.cuh"
#include "vec.cuh"

namespace qsb {
namespace {

constexpr int kCols = 256;      // columns per block (32 lanes x 8)
constexpr int kWarps = 8;

template <int DT>
__device__ __forceinline__ void load8v(const void* base, int64_t i, float* f) {
    if constexpr (DT == QSYNC_F32) {
        const uint4* v = reinterpret_cast<const uint4*>(static_cast<const float*>(base) + i);
        Vec<QSYNC_F32>::unpack(ld_stream(v), f);
        Vec<QSYNC_F32>::unpack(ld_stream(v + 1), f + 4);
    } else {
        Vec<DT>::unpack(ld_stream(static_cast<const uint16_t*>(base) + i), f);
    }
}

template <int DT>
__device__ __forceinline__ float load1(const void* base, int64_t i) {
    return Elem<DT>::f(static_cast<const typename Elem<DT>::T*>(base)[i]);
}

template <int DT>
__device__ __forceinline__ void store8v(void* base, int64_t i, const float* f) {
    if constexpr (DT == QSYNC_F32) {
        float4* o = reinterpret_cast<float4*>(static_cast<float*>(base) + i);
        o[0] = make_float4(f[0], f[1], f[2], f[3]);
        o[1] = make_float4(f[4], f[5], f[6], f[7]);
    } else {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            w[k] = DT == QSYNC_BF16 ? pack_bf162(f[2 * k], f[2 * k + 1]) : pack_half2(f[2 * k], f[2 * k + 1]);
        }
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(base) + i) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

template <int DT>
__device__ __forceinline__ void store1(void* base, int64_t i, float v) {
    if constexpr (DT == QSYNC_F32)
        static_cast<float*>(base)[i] = v;
    else if constexpr (DT == QSYNC_BF16)
        static_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16_rn(v);
    else
        static_cast<__half*>(base)[i] = __float2half_rn(v);
}

template <int DDY, int DH, int DO, int ACT>
__device__ __forceinline__ void act_row8(const void* __restrict__ dy, const void* __restrict__ h,
                                         void* __restrict__ out, int64_t off, int64_t c, int64_t cols,
                                         bool full, float (&g)[8]) {
    if (full) {
        load8v<DDY>(dy, off, g);
        if constexpr (ACT == 1) {
            float hv[8];
            load8v<DH>(h, off, hv);
#pragma unroll
            for (int j = 0; j < 8; ++j) g[j] = __fmul_rn(g[j], gelu_erf_grad<DH != QSYNC_F32>(hv[j]));
        } else if constexpr (ACT == 2) {  // h holds act'(x) (FP16), stored by the forward
            float hv[8];
            load8v<QSYNC_F16>(h, off, hv);
#pragma unroll
            for (int j = 0; j < 8; ++j) g[j] = __fmul_rn(g[j], hv[j]);
        }
        if (out) store8v<DO>(out, off, g);
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            g[j] = 0.0f;
            if (c + j < cols) {
                g[j] = load1<DDY>(dy, off + j);
                if constexpr (ACT == 1) g[j] = __fmul_rn(g[j], gelu_erf_grad<DH != QSYNC_F32>(load1<DH>(h, off + j)));
                if constexpr (ACT == 2) g[j] = __fmul_rn(g[j], load1<QSYNC_F16>(h, off + j));
                if (out) store1<DO>(out, off + j, g[j]);
            }
        }
    }
}

// Grid = (256-column strips) x (row chunks), the chunk height chosen so the whole
// grid is ONE resident wave (a fixed 64-row chunk left a 4% tail wave at
// [4096, 3072]); each block reduces its column partials once.
template <int DDY, int DH, int DO, int ACT>
__global__ void __launch_bounds__(kWarps * 32) k_act_bwd_colsum(const void* __restrict__ dy,
                                                                const void* __restrict__ h,
                                                                int64_t rows, int64_t cols,
                                                                void* __restrict__ out,
                                                                float* __restrict__ colsum,
                                                                int vec_ok, int chunk) {
    QSB_PDL_ENTER();
    __shared__ float red[kWarps][kCols];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * kCols + lane * 8;
    const int per_warp = chunk / kWarps;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * chunk + warp * per_warp;
    float cs[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) cs[j] = 0.0f;
    const bool full = vec_ok && c + 8 <= cols;
#pragma unroll 4
    for (int rr = 0; rr < per_warp; ++rr) {
        const int64_t r = r0 + rr;
        if (r >= rows) break;
        float g[8];
        act_row8<DDY, DH, DO, ACT>(dy, h, out, r * cols + c, c, cols, full, g);
#pragma unroll
        for (int j = 0; j < 8; ++j) cs[j] += g[j];
    }
    if (!colsum) return;
#pragma unroll
    for (int j = 0; j < 8; ++j) red[warp][lane * 8 + j] = cs[j];
    __syncthreads();
    const int64_t col = static_cast<int64_t>(blockIdx.x) * kCols + threadIdx.x;
    if (col < cols) {
        float t = 0.0f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) t += red[w][threadIdx.x];
        atomicAdd(colsum + col, t);
    }
}

template <int DDY, int DH, int DO, int ACT>
int launch_act_bwd(const void* dy, const void* h, int64_t rows, int64_t cols, void* out,
                   float* colsum, cudaStream_t st) {
    const int vec = (cols % 8 == 0) && aligned16(dy) && (!h || aligned16(h)) && (!out || aligned16(out));
    static int per_sm = 0;
    if (!per_sm) {
        QSB_TRY(cuda_status(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                &per_sm, k_act_bwd_colsum<DDY, DH, DO, ACT>, kWarps * 32, 0),
                            "cudaOccupancyMaxActiveBlocksPerMultiprocessor"));
        per_sm = std::max(per_sm, 1);
    }
    const int64_t strips = (cols + kCols - 1) / kCols;
    const int64_t slots = int64_t(sm_count()) * per_sm;
    const int64_t chunks_want = std::max<int64_t>(1, slots / strips);
    int64_t chunk = (rows + chunks_want - 1) / chunks_want;
    chunk = std::max<int64_t>(kWarps, (chunk + kWarps - 1) / kWarps * kWarps);  // whole rows per warp
    const int64_t chunks = (rows + chunk - 1) / chunk;
    QSB_REQUIRE(chunks < 65535 && chunk < (int64_t(1) << 30), QSYNC_ERR_DOMAIN, "too many rows");
    dim3 grid(static_cast<unsigned>(strips), static_cast<unsigned>(chunks));
    pdl_launch(k_act_bwd_colsum<DDY, DH, DO, ACT>, grid, dim3(kWarps * 32), 0, st, dy, h, rows, cols, out,
               colsum, vec, static_cast<int>(chunk));
    return check_launch("k_act_bwd_colsum");
}

template <int DDY, int DH, int ACT>
int act_bwd_out(const void* dy, const void* h, int64_t rows, int64_t cols, void* out, int out_dtype,
                float* colsum, cudaStream_t st) {
    if (out_dtype == QSYNC_F32) return launch_act_bwd<DDY, DH, QSYNC_F32, ACT>(dy, h, rows, cols, out, colsum, st);
    if constexpr (ACT == 0) {  // the BF16 backward entry of a BF16 op (no activation)
        if (out_dtype == QSYNC_BF16)
            return launch_act_bwd<DDY, DH, QSYNC_BF16, ACT>(dy, h, rows, cols, out, colsum, st);
    }
    return launch_act_bwd<DDY, DH, QSYNC_F16, ACT>(dy, h, rows, cols, out, colsum, st);
}

template <int DDY>
int act_bwd_h(const void* dy, const void* h, int h_dtype, int64_t rows, int64_t cols, int act, void* out,
              int out_dtype, float* colsum, cudaStream_t st) {
    if (act == QSYNC_ACT_NONE) return act_bwd_out<DDY, QSYNC_F32, 0>(dy, nullptr, rows, cols, out, out_dtype, colsum, st);
    if (act == QSYNC_ACT_DERIV) return act_bwd_out<DDY, QSYNC_F16, 2>(dy, h, rows, cols, out, out_dtype, colsum, st);
    if (h_dtype == QSYNC_F32) return act_bwd_out<DDY, QSYNC_F32, 1>(dy, h, rows, cols, out, out_dtype, colsum, st);
    return act_bwd_out<DDY, QSYNC_F16, 1>(dy, h, rows, cols, out, out_dtype, colsum, st);
}

}  // namespace
}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_act_bwd_colsum(const void* dy, int dy_dtype, const void* h, int h_dtype, int64_t rows,
                         int64_t cols, int act, void* out, int out_dtype, float* colsum,
                         qsync_stream_t stream) {
    QSB_REQUIRE(dy != nullptr, QSYNC_ERR_VALIDATION, "dy is required");
    QSB_REQUIRE(rows >= 0 && cols >= 0, QSYNC_ERR_DOMAIN, "negative shape");
    QSB_REQUIRE(act == QSYNC_ACT_NONE || act == QSYNC_ACT_GELU || act == QSYNC_ACT_DERIV, QSYNC_ERR_DOMAIN,
                "unknown activation");
    QSB_REQUIRE(act == QSYNC_ACT_NONE || h != nullptr, QSYNC_ERR_VALIDATION, "activation backward needs h");
    QSB_REQUIRE(dy_dtype == QSYNC_F32 || dy_dtype == QSYNC_F16 || (dy_dtype == QSYNC_BF16 && act == QSYNC_ACT_NONE),
                QSYNC_ERR_DOMAIN, "dy must be F32 or F16 (BF16 without an activation)");
    QSB_REQUIRE(act != QSYNC_ACT_GELU || h_dtype == QSYNC_F32 || h_dtype == QSYNC_F16, QSYNC_ERR_DOMAIN,
                "h must be F32 or F16");
    QSB_REQUIRE(act != QSYNC_ACT_DERIV || h_dtype == QSYNC_F16, QSYNC_ERR_DOMAIN, "a stored derivative is F16");
    QSB_REQUIRE(!out || out_dtype == QSYNC_F32 || out_dtype == QSYNC_F16 ||
                    (out_dtype == QSYNC_BF16 && act == QSYNC_ACT_NONE),
                QSYNC_ERR_DOMAIN, "out must be F32 or F16 (BF16 without an activation)");
    if (rows == 0 || cols == 0 || (!out && !colsum)) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    if (dy_dtype == QSYNC_F32)
        return act_bwd_h<QSYNC_F32>(dy, h, h_dtype, rows, cols, act, out, out_dtype, colsum, st);
    if (dy_dtype == QSYNC_BF16)
        return act_bwd_out<QSYNC_BF16, QSYNC_F32, 0>(dy, nullptr, rows, cols, out, out_dtype, colsum, st);
    return act_bwd_h<QSYNC_F16>(dy, h, h_dtype, rows, cols, act, out, out_dtype, colsum, st);
}

}  // extern "C"

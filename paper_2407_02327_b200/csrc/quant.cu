// quant.cu -- K1 absmax, K2 RNE quantize, K3 dequantize, K4 casts, K5 statistics.
//
// All of these are HBM-bound streaming kernels: 16-byte
// vector loads/stores, several loads in flight per thread, grids sized as a
// multiple of the SM count, warp-shuffle reductions.  Semantics follow the
// oracle (oracle/cpu_ref.c) bit for bit: s = absmax/127 (IEEE), q =
// sat(rint(x/s)), dequant = float(q)*s.
#include <algorithm>

#include <cuda_fp8.h>

#include "common.cuh"
#include "vec.cuh"

namespace qsb {

namespace {

constexpr int kThreads = 512;

template <int DT>
__device__ __forceinline__ float round_to(float g) {
    if constexpr (DT == QSYNC_F16) return __half2float(__float2half_rn(g));
    if constexpr (DT == QSYNC_BF16) return __bfloat162float(__float2bfloat16_rn(g));
    return g;
}

// Fused prologue activation of the streaming kernels: ACT 0 = identity,
// ACT 1 = GELU (the FF1 -> FF2 activation of an encoder layer, so the
// quantizer / cast of the FF2 input reads the pre-activation directly).
// For a 16-bit input the activation is a dependent op of an FP16 producer and
// runs in its precision (the cascade rule, graph.cpp:254-269): its output is
// rounded to that format before it is quantized, exactly as if materialised.
template <int ACT, int DT = QSYNC_F32>
__device__ __forceinline__ float act_f(float v) {
    if constexpr (ACT == 1) {
        const float g = gelu_erf<DT != QSYNC_F32>(v);
        if constexpr (DT == QSYNC_F16) return __half2float(__float2half_rn(g));
        if constexpr (DT == QSYNC_BF16) return __bfloat162float(__float2bfloat16_rn(g));
        return g;
    }
    return v;
}

// Running absmax of act(x).  (Pruning the erf for elements that cannot raise the
// running max -- |gelu(x)| <= x for x >= 0, <= 0.171 below -- is exact but was
// measured slower: the divergent branch costs more than the erf it skips.)
template <int ACT, int DT>
__device__ __forceinline__ void absmax_acc(float& m, float x) {
    m = fmaxf(m, fabsf(act_f<ACT, DT>(x)));
}

// ---------------------------------------------------------------------------
// K1: per-tensor absmax.  Grid-stride, 4 x 16B loads in flight per thread,
// warp shuffle + smem block reduce, one atomicMax per block on the float bits
// (valid ordering for non-negative floats; max is order-independent, so the
// result is deterministic).
// ---------------------------------------------------------------------------
template <int DT, int ACT = 0>
__global__ void __launch_bounds__(kThreads) k_absmax(const typename Elem<DT>::T* __restrict__ x,
                                                     int64_t n, unsigned* __restrict__ out,
                                                     int vec_ok) {
    QSB_PDL_ENTER();
    using V = Vec<DT>;
    constexpr int U = 4;
    float m = 0.0f;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (vec_ok) {
        const int64_t nv = n / V::N;
        const uint4* xv = reinterpret_cast<const uint4*>(x);
        int64_t i = tid;
        for (; i + (U - 1) * stride < nv; i += U * stride) {
            uint4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = ld_stream(xv + i + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float f[V::N];
                V::unpack(r[u], f);
#pragma unroll
                for (int j = 0; j < V::N; ++j) absmax_acc<ACT, DT>(m, f[j]);
            }
        }
        for (; i < nv; i += stride) {
            float f[V::N];
            V::unpack(ld_stream(xv + i), f);
#pragma unroll
            for (int j = 0; j < V::N; ++j) absmax_acc<ACT, DT>(m, f[j]);
        }
        done = nv * V::N;
    }
    for (int64_t i = done + tid; i < n; i += stride) absmax_acc<ACT, DT>(m, Elem<DT>::f(x[i]));

    __shared__ float red[32];
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
        m = warp_max(m);
        if (threadIdx.x == 0 && m > 0.0f) atomicMax(out, __float_as_uint(m));
    }
}

// FF2's INT8 operand in two passes with ONE GELU evaluation: this pass computes
// g = GELU(x) (rounded to x's format, the cascade rule) and GELU'(x) from one
// erf, writes both, and reduces absmax(g); the quantizer then reads g with no
// activation (a pure HBM pass) instead of recomputing the erf.  g is the value
// k_quantize<DT, 1> would quantize, so q / s are bit-identical.
template <int DT>
__global__ void __launch_bounds__(kThreads) k_gelu_absmax_store(const typename Elem<DT>::T* __restrict__ x,
                                                                int64_t n, unsigned* __restrict__ out,
                                                                typename Elem<DT>::T* __restrict__ y,
                                                                uint16_t* __restrict__ dact, int vec_ok) {
    QSB_PDL_ENTER();
    using V = Vec<DT>;
    using T = typename Elem<DT>::T;
    float m = 0.0f;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (vec_ok) {
        const int64_t n8 = n / 8;  // 8 elements per step: 2 (F32) or 1 (F16) 16 B loads
        for (int64_t i = tid; i < n8; i += stride) {
            float f[8];
            if constexpr (DT == QSYNC_F32) {
                const uint4* xv = reinterpret_cast<const uint4*>(x) + 2 * i;
                V::unpack(ld_stream(xv), f);
                V::unpack(ld_stream(xv + 1), f + 4);
            } else {
                V::unpack(ld_stream(reinterpret_cast<const uint4*>(x) + i), f);
            }
            float g[8];
            uint32_t dp[4];
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                float d0, d1;
                gelu_pair<DT != QSYNC_F32>(f[j], g[j], d0);
                gelu_pair<DT != QSYNC_F32>(f[j + 1], g[j + 1], d1);
                g[j] = round_to<DT>(g[j]);
                g[j + 1] = round_to<DT>(g[j + 1]);
                m = fmaxf(m, fmaxf(fabsf(g[j]), fabsf(g[j + 1])));
                dp[j / 2] = pack_half2(d0, d1);
            }
            if constexpr (DT == QSYNC_F32) {
                float4* yv = reinterpret_cast<float4*>(y) + 2 * i;
                yv[0] = make_float4(g[0], g[1], g[2], g[3]);
                yv[1] = make_float4(g[4], g[5], g[6], g[7]);
            } else {
                reinterpret_cast<uint4*>(y)[i] = make_uint4(pack_half2(g[0], g[1]), pack_half2(g[2], g[3]),
                                                            pack_half2(g[4], g[5]), pack_half2(g[6], g[7]));
            }
            if (dact) reinterpret_cast<uint4*>(dact)[i] = make_uint4(dp[0], dp[1], dp[2], dp[3]);
        }
        done = n8 * 8;
    }
    for (int64_t i = done + tid; i < n; i += stride) {
        float g, d;
        gelu_pair<DT != QSYNC_F32>(Elem<DT>::f(x[i]), g, d);
        g = round_to<DT>(g);
        m = fmaxf(m, fabsf(g));
        if constexpr (DT == QSYNC_F32)
            y[i] = g;
        else
            y[i] = __float2half_rn(g);
        if (dact) dact[i] = __half_as_ushort(__float2half_rn(d));
    }
    __shared__ float red[32];
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
        m = warp_max(m);
        if (threadIdx.x == 0 && m > 0.0f) atomicMax(out, __float_as_uint(m));
    }
    (void)sizeof(T);
}

// absmax of each row, one warp per row.
template <int DT>
__global__ void __launch_bounds__(256) k_absmax_rows(const typename Elem<DT>::T* __restrict__ x,
                                                     int64_t rows, int64_t cols,
                                                     float* __restrict__ out) {
    QSB_PDL_ENTER();
    const int64_t row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const typename Elem<DT>::T* xr = x + row * cols;
    float m = 0.0f;
    for (int64_t c = lane; c < cols; c += 32) m = fmaxf(m, fabsf(Elem<DT>::f(xr[c])));
    m = warp_max(m);
    if (lane == 0) out[row] = m;
}

// ---------------------------------------------------------------------------
// K2: RNE quantize with the scale derived on the fly from absmax (absmax_in
// holds float bits written by k_absmax).  16 elements per thread-iteration:
// 4 (F32) or 2 (F16/BF16) 16B loads, one 16B store.  Block 0 publishes s.
// ---------------------------------------------------------------------------
template <int DT, int ACT = 0>
__global__ void __launch_bounds__(kThreads, 2) k_quantize(const typename Elem<DT>::T* __restrict__ x,
                                                       int64_t n, const float* __restrict__ absmax_in,
                                                       const float* __restrict__ scale_in,
                                                       int8_t* __restrict__ q,
                                                       float* __restrict__ scale_out, int vec_ok,
                                                       uint16_t* __restrict__ dact = nullptr,
                                                       uint16_t* __restrict__ q16 = nullptr) {
    QSB_PDL_ENTER();
    using V = Vec<DT>;
    constexpr int LOADS = 16 / V::N;
    const float s = scale_in ? *scale_in : scale_from_absmax(*absmax_in);
    if (scale_out && blockIdx.x == 0 && threadIdx.x == 0) *scale_out = s;
    const QScale qs = make_qscale(s);
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (vec_ok) {
        const int64_t n16 = n / 16;
        const uint4* xv = reinterpret_cast<const uint4*>(x);
        uint4* qv = reinterpret_cast<uint4*>(q);
        // G groups of 16 elements per thread-iteration, all loads issued before
        // any math: 128 B (F32) / 64 B (16-bit) in flight per thread, so the
        // stream stays HBM-bound at the occupancy the registers allow.
        constexpr int G = DT == QSYNC_F32 ? 2 : (ACT == 1 ? 2 : 4);
        auto process = [&](int64_t i, const uint4 (&r)[LOADS]) {
            uint32_t packed[4];
            uint32_t dp[8];  // GELU'(x) of the 16 elements as FP16 pairs (the backward's factor)
            uint32_t hq[8];  // the 16 grid values as FP16 pairs (exact; the wgrad's operand)
#pragma unroll
            for (int u = 0; u < LOADS; ++u) {
                float f[V::N];
                V::unpack(r[u], f);
#pragma unroll
                for (int j = 0; j < V::N; j += 4) {
                    float a[4];
                    if (ACT == 1 && dact) {  // GELU and GELU' share the erf
                        float d[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            gelu_pair<DT != QSYNC_F32>(f[j + e], a[e], d[e]);
                            a[e] = round_to<DT>(a[e]);
                        }
                        dp[(u * V::N + j) / 2] = pack_half2(d[0], d[1]);
                        dp[(u * V::N + j) / 2 + 1] = pack_half2(d[2], d[3]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e) a[e] = act_f<ACT, DT>(f[j + e]);
                    }
                    const float t0 = quant_rne_f(a[0], qs), t1 = quant_rne_f(a[1], qs);
                    const float t2 = quant_rne_f(a[2], qs), t3 = quant_rne_f(a[3], qs);
                    packed[(u * V::N + j) / 4] = pack_q4(t0, t1, t2, t3);
                    if (q16) {
                        hq[(u * V::N + j) / 2] = pack_half2(grid_value(t0), grid_value(t1));
                        hq[(u * V::N + j) / 2 + 1] = pack_half2(grid_value(t2), grid_value(t3));
                    }
                }
            }
            qv[i] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
            if (q16) {
                uint4* hv = reinterpret_cast<uint4*>(q16) + 2 * i;
                hv[0] = make_uint4(hq[0], hq[1], hq[2], hq[3]);
                hv[1] = make_uint4(hq[4], hq[5], hq[6], hq[7]);
            }
            if (ACT == 1 && dact) {
                uint4* dv = reinterpret_cast<uint4*>(dact) + 2 * i;
                dv[0] = make_uint4(dp[0], dp[1], dp[2], dp[3]);
                dv[1] = make_uint4(dp[4], dp[5], dp[6], dp[7]);
            }
        };
        // vec_ok bit 1: walk the groups from the end -- the second pass of the
        // two-pass per-tensor quantizer then starts on what the absmax pass read
        // last (still in L2) instead of on what it has already evicted.
        const bool rev = (vec_ok & 2) != 0;
        auto at = [&](int64_t j) { return rev ? n16 - 1 - j : j; };
        int64_t i = tid;
        for (; i + (G - 1) * stride < n16; i += G * stride) {
            uint4 r[G][LOADS];
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int u = 0; u < LOADS; ++u) r[g][u] = ld_stream(xv + at(i + g * stride) * LOADS + u);
#pragma unroll
            for (int g = 0; g < G; ++g) process(at(i + g * stride), r[g]);
        }
        for (; i < n16; i += stride) {
            uint4 r[LOADS];
#pragma unroll
            for (int u = 0; u < LOADS; ++u) r[u] = ld_stream(xv + at(i) * LOADS + u);
            process(at(i), r);
        }
        done = n16 * 16;
    }
    for (int64_t i = done + tid; i < n; i += stride) {
        const float xv = Elem<DT>::f(x[i]);
        const int qi = quant_rne(act_f<ACT, DT>(xv), qs);
        q[i] = static_cast<int8_t>(qi);
        if (q16) q16[i] = __half_as_ushort(__int2half_rn(qi));
        if (ACT == 1 && dact) dact[i] = __half_as_ushort(__float2half_rn(gelu_erf_grad<DT != QSYNC_F32>(xv)));
    }
}

// ---------------------------------------------------------------------------
// 2-D tile kernels: quantize / cast a [rows, cols] matrix and also emit its
// FP16 transpose (the K-major operand the wgrad / dgrad GEMMs need), plus
// optional column sums (bias gradient).  Tile 64 x 64, 256 threads; each
// thread loads 4 consecutive elements of a row (16 B for F32, 8 B for 16-bit),
// writes the row-major output as one 4/8-byte vector, and stages the values
// in a padded smem tile from which the transpose is written as 16-byte rows.
// mode 0: quantize with absmax-derived scale -> q (int8) + q_t (fp16 ints)
// mode 1: cast -> out (fp16) + out_t (fp16) + colsum (fp32, atomics)
// Shapes with cols % 4 != 0 or misaligned bases take the scalar edge path
// inside the same kernel.
// ---------------------------------------------------------------------------
constexpr int TR = 64, TC = 64;

template <int DT>
__device__ __forceinline__ void load4(const typename Elem<DT>::T* p, float* f) {
    if (DT == QSYNC_F32) {
        const float4 v = *reinterpret_cast<const float4*>(p);
        f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
    } else {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        const uint32_t w[2] = {v.x, v.y};
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            float2 t;
            if (DT == QSYNC_F16) t = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
            else t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
            f[2 * i] = t.x;
            f[2 * i + 1] = t.y;
        }
    }
}

template <int DT, int MODE>
__global__ void __launch_bounds__(256) k_tile(const typename Elem<DT>::T* __restrict__ x,
                                              int64_t rows, int64_t cols,
                                              const float* __restrict__ absmax_in,
                                              int8_t* __restrict__ q, uint16_t* __restrict__ out,
                                              uint16_t* __restrict__ out_t, int64_t ld_t,
                                              float* __restrict__ colsum,
                                              float* __restrict__ scale_out, int vec_ok,
                                              int8_t* __restrict__ out_t8 = nullptr) {
    QSB_PDL_ENTER();
    __shared__ __align__(16) __half tile[TC][TR + 8];  // [col][row], 16B-aligned rows
    __shared__ float csum[16][TC + 1];
    const int tid = threadIdx.x;
    const int cg = tid & 15;   // 4-column group within the tile
    const int rl0 = tid >> 4;  // 0..15
    const int64_t r0 = blockIdx.y * (int64_t)TR, c0 = blockIdx.x * (int64_t)TC;
    float s = 1.0f;
    if (MODE == 0) {
        s = scale_from_absmax(*absmax_in);
        if (scale_out && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *scale_out = s;
    }
    const QScale qs = make_qscale(s);
    const int64_t c = c0 + cg * 4;
    const bool full_cols = vec_ok && (c + 4 <= cols);
    float cs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int pass = 0; pass < TR / 16; ++pass) {
        const int rl = rl0 + 16 * pass;
        const int64_t r = r0 + rl;
        float f[4] = {0.f, 0.f, 0.f, 0.f};
        if (r < rows) {
            if (full_cols) {
                load4<DT>(x + r * cols + c, f);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (c + i < cols) f[i] = Elem<DT>::f(x[r * cols + c + i]);
            }
        }
        __half h[4];
        if (MODE == 0) {
            float t[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                t[i] = quant_rne_f(f[i], qs);
                h[i] = __float2half_rn(grid_value(t[i]));
            }
            if (q && r < rows) {
                if (full_cols) {
                    *reinterpret_cast<uint32_t*>(q + r * cols + c) = pack_q4(t[0], t[1], t[2], t[3]);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (c + i < cols) q[r * cols + c + i] = static_cast<int8_t>(__float_as_uint(t[i]) & 0xffu);
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                h[i] = __float2half_rn(f[i]);
                cs[i] += f[i];
            }
            if (out && r < rows) {
                if (full_cols) {
                    uint2 pk;
                    pk.x = __half_as_ushort(h[0]) | (static_cast<uint32_t>(__half_as_ushort(h[1])) << 16);
                    pk.y = __half_as_ushort(h[2]) | (static_cast<uint32_t>(__half_as_ushort(h[3])) << 16);
                    *reinterpret_cast<uint2*>(out + r * cols + c) = pk;
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (c + i < cols) out[r * cols + c + i] = __half_as_ushort(h[i]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) tile[cg * 4 + i][rl] = h[i];
    }
    if (MODE == 1 && colsum) {
#pragma unroll
        for (int i = 0; i < 4; ++i) csum[rl0][cg * 4 + i] = cs[i];
    }
    __syncthreads();
    if (out_t) {
        // 64 columns x 64 rows: each thread writes 2 x (8 rows as one 16B store).
        const bool vec_t = vec_ok && (ld_t % 8 == 0);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int idx = tid + 256 * k;  // 0..511
            const int cc = idx >> 3;        // column within tile
            const int rg = (idx & 7) * 8;   // row group
            const int64_t oc = c0 + cc;
            const int64_t orow = r0 + rg;
            if (oc >= cols || orow >= rows) continue;
            if (vec_t && orow + 8 <= rows) {
                *reinterpret_cast<uint4*>(out_t + oc * ld_t + orow) =
                    *reinterpret_cast<const uint4*>(&tile[cc][rg]);
            } else {
                for (int i = 0; i < 8 && orow + i < rows; ++i)
                    out_t[oc * ld_t + orow + i] = __half_as_ushort(tile[cc][rg + i]);
            }
        }
    }
    if (MODE == 0 && out_t8) {
        // INT8 transpose (the saved activation of an INT8 op, 1 byte/element):
        // 8 rows as one 8-byte store.
        const bool vec_t = vec_ok && (ld_t % 8 == 0);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int idx = tid + 256 * k;
            const int cc = idx >> 3;
            const int rg = (idx & 7) * 8;
            const int64_t oc = c0 + cc;
            const int64_t orow = r0 + rg;
            if (oc >= cols || orow >= rows) continue;
            if (vec_t && orow + 8 <= rows) {
                uint32_t lo = 0, hi = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    lo |= static_cast<uint32_t>(static_cast<uint8_t>(__half2int_rn(tile[cc][rg + i]))) << (8 * i);
                    hi |= static_cast<uint32_t>(static_cast<uint8_t>(__half2int_rn(tile[cc][rg + 4 + i]))) << (8 * i);
                }
                *reinterpret_cast<uint2*>(out_t8 + oc * ld_t + orow) = make_uint2(lo, hi);
            } else {
                for (int i = 0; i < 8 && orow + i < rows; ++i)
                    out_t8[oc * ld_t + orow + i] = static_cast<int8_t>(__half2int_rn(tile[cc][rg + i]));
            }
        }
    }
    if (MODE == 1 && colsum && tid < TC) {
        const int64_t cc = c0 + tid;
        if (cc < cols) {
            float t = 0.0f;
#pragma unroll
            for (int j = 0; j < 16; ++j) t += csum[j][tid];
            atomicAdd(colsum + cc, t);
        }
    }
}

// Per-channel quantize: one warp per row.  Rows of up to 32 * 4 * kRowVec
// floats stay in registers between the absmax and the quantize step (all of a
// lane's 16-byte loads in flight at once, one HBM read per element); longer or
// unaligned rows take two passes (the second read hits L1/L2).
constexpr int kRowVec = 8;  // float4 per lane cached: rows of <= 1024 floats
__global__ void __launch_bounds__(256) k_quant_rows(const float* __restrict__ w, int64_t rows,
                                                    int64_t cols, int8_t* __restrict__ q,
                                                    float* __restrict__ scales) {
    QSB_PDL_ENTER();
    const int64_t row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float* wr = w + row * cols;
    int8_t* qr = q + row * cols;
    const bool vec = (cols % 4 == 0) && aligned16(wr) && (reinterpret_cast<uintptr_t>(qr) & 3u) == 0;
    const int64_t n4 = cols / 4;
    if (vec && n4 <= 32 * kRowVec) {
        const float4* v = reinterpret_cast<const float4*>(wr);
        float4 f[kRowVec];
#pragma unroll
        for (int i = 0; i < kRowVec; ++i) {
            const int64_t c = lane + 32 * i;
            f[i] = c < n4 ? __ldcs(v + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float m = 0.0f;
#pragma unroll
        for (int i = 0; i < kRowVec; ++i)
            m = fmaxf(m, fmaxf(fmaxf(fabsf(f[i].x), fabsf(f[i].y)), fmaxf(fabsf(f[i].z), fabsf(f[i].w))));
        m = warp_max(m);
        const float s = scale_from_absmax(m);
        if (lane == 0) scales[row] = s;
        const QScale qs = make_qscale(s);
        uint32_t* qo = reinterpret_cast<uint32_t*>(qr);
#pragma unroll
        for (int i = 0; i < kRowVec; ++i) {
            const int64_t c = lane + 32 * i;
            if (c < n4)
                qo[c] = pack_q4(quant_rne_f(f[i].x, qs), quant_rne_f(f[i].y, qs), quant_rne_f(f[i].z, qs),
                                quant_rne_f(f[i].w, qs));
        }
        return;
    }
    float m = 0.0f;
    if (vec) {
        const float4* v = reinterpret_cast<const float4*>(wr);
#pragma unroll 4
        for (int64_t c = lane; c < n4; c += 32) {
            float4 f = v[c];
            m = fmaxf(m, fmaxf(fmaxf(fabsf(f.x), fabsf(f.y)), fmaxf(fabsf(f.z), fabsf(f.w))));
        }
    } else {
        for (int64_t c = lane; c < cols; c += 32) m = fmaxf(m, fabsf(wr[c]));
    }
    m = warp_max(m);
    const float s = scale_from_absmax(m);
    if (lane == 0) scales[row] = s;
    const QScale qs = make_qscale(s);
    if (vec) {
        const float4* v = reinterpret_cast<const float4*>(wr);
        uint32_t* qo = reinterpret_cast<uint32_t*>(qr);
#pragma unroll 4
        for (int64_t c = lane; c < n4; c += 32) {
            float4 f = v[c];
            qo[c] = pack_q4(quant_rne_f(f.x, qs), quant_rne_f(f.y, qs), quant_rne_f(f.z, qs), quant_rne_f(f.w, qs));
        }
    } else {
        for (int64_t c = lane; c < cols; c += 32) qr[c] = static_cast<int8_t>(quant_rne(wr[c], qs));
    }
}

// ---------------------------------------------------------------------------
// FP8 (E4M3) quantizers for the FP8 rung of the precision ladder: s =
// absmax / 448 (IEEE; 1 for an all-zero tensor), q = e4m3_rn_satfinite(x / s).
// Per-tensor (activations, absmax computed upstream) and per-row (weights).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float scale_fp8(float a) { return a > 0.0f ? __fdiv_rn(a, 448.0f) : 1.0f; }
__device__ __forceinline__ uint32_t e4m3x4(float a, float b, float c, float d) {
    const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
    const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(c, d), __NV_SATFINITE, __NV_E4M3);
    return lo | (hi << 16);
}

template <int DT>
__global__ void __launch_bounds__(kThreads) k_quantize_fp8(const typename Elem<DT>::T* __restrict__ x, int64_t n,
                                                           const float* __restrict__ absmax_in,
                                                           uint8_t* __restrict__ q, float* __restrict__ scale_out,
                                                           int vec_ok) {
    QSB_PDL_ENTER();
    using V = Vec<DT>;
    constexpr int LOADS = 16 / V::N;
    const float s = scale_fp8(*absmax_in);
    if (scale_out && blockIdx.x == 0 && threadIdx.x == 0) *scale_out = s;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (vec_ok) {
        const int64_t n16 = n / 16;
        const uint4* xv = reinterpret_cast<const uint4*>(x);
        uint4* qv = reinterpret_cast<uint4*>(q);
        for (int64_t i = tid; i < n16; i += stride) {
            uint4 r[LOADS];
#pragma unroll
            for (int u = 0; u < LOADS; ++u) r[u] = ld_stream(xv + i * LOADS + u);
            uint32_t packed[4];
#pragma unroll
            for (int u = 0; u < LOADS; ++u) {
                float f[V::N];
                V::unpack(r[u], f);
#pragma unroll
                for (int j = 0; j < V::N; j += 4)
                    packed[(u * V::N + j) / 4] = e4m3x4(__fdiv_rn(f[j], s), __fdiv_rn(f[j + 1], s),
                                                        __fdiv_rn(f[j + 2], s), __fdiv_rn(f[j + 3], s));
            }
            qv[i] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        }
        done = n16 * 16;
    }
    for (int64_t i = done + tid; i < n; i += stride)
        q[i] = static_cast<uint8_t>(__nv_cvt_float_to_fp8(__fdiv_rn(Elem<DT>::f(x[i]), s), __NV_SATFINITE, __NV_E4M3));
}

__global__ void __launch_bounds__(256) k_quant_rows_fp8(const float* __restrict__ w, int64_t rows, int64_t cols,
                                                        uint8_t* __restrict__ q, float* __restrict__ scales) {
    QSB_PDL_ENTER();
    const int64_t row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float* wr = w + row * cols;
    uint8_t* qr = q + row * cols;
    float m = 0.0f;
    for (int64_t c = lane; c < cols; c += 32) m = fmaxf(m, fabsf(wr[c]));
    m = warp_max(m);
    const float s = scale_fp8(m);
    if (lane == 0) scales[row] = s;
    const bool vec = (cols % 4 == 0) && aligned16(wr) && ((reinterpret_cast<uintptr_t>(qr) & 3u) == 0);
    if (vec) {
        const float4* v = reinterpret_cast<const float4*>(wr);
        uint32_t* qo = reinterpret_cast<uint32_t*>(qr);
        for (int64_t c = lane; c < cols / 4; c += 32) {
            const float4 f = v[c];
            qo[c] = e4m3x4(__fdiv_rn(f.x, s), __fdiv_rn(f.y, s), __fdiv_rn(f.z, s), __fdiv_rn(f.w, s));
        }
    } else {
        for (int64_t c = lane; c < cols; c += 32)
            qr[c] = static_cast<uint8_t>(__nv_cvt_float_to_fp8(__fdiv_rn(wr[c], s), __NV_SATFINITE, __NV_E4M3));
    }
}

template <int DT>
struct QuantFp8Run {
    static int run(const void* x, int64_t n, const float* absmax, uint8_t* q, float* scale_out, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        if (n == 0) return QSYNC_OK;
        const int vec = aligned16(x) && aligned16(q);
        const int grid = grid_for(n / 16 + 1, kThreads, 4);
        pdl_launch(k_quantize_fp8<DT>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n, absmax, q,
                   scale_out, vec);
        return check_launch("k_quantize_fp8");
    }
};

// ---------------------------------------------------------------------------
// K3: dequantize, 16 int8 in -> 16 floats out per thread-iteration.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_dequant(const int8_t* __restrict__ q, int64_t n,
                                                      const float* __restrict__ scale,
                                                      float* __restrict__ out, int vec_ok) {
    QSB_PDL_ENTER();
    // Thread i owns output float4 i (4 int8 in, 16 B out): every store
    // instruction writes 512 contiguous bytes per warp, so no partial sectors
    // are written (partial-sector writes made L2 fetch lines from DRAM).
    const float s = *scale;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (vec_ok) {
        const int64_t n4 = n / 4;
        const uint32_t* qv = reinterpret_cast<const uint32_t*>(q);
        float4* ov = reinterpret_cast<float4*>(out);
        constexpr int U = 4;
        int64_t i = tid;
        for (; i + (U - 1) * stride < n4; i += U * stride) {
            uint32_t w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) w[u] = __ldcs(qv + i + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float4 f;
                f.x = static_cast<float>(static_cast<int8_t>(w[u] & 0xff)) * s;
                f.y = static_cast<float>(static_cast<int8_t>((w[u] >> 8) & 0xff)) * s;
                f.z = static_cast<float>(static_cast<int8_t>((w[u] >> 16) & 0xff)) * s;
                f.w = static_cast<float>(static_cast<int8_t>(w[u] >> 24)) * s;
                __stcs(ov + i + u * stride, f);
            }
        }
        for (; i < n4; i += stride) {
            const uint32_t w = __ldcs(qv + i);
            float4 f;
            f.x = static_cast<float>(static_cast<int8_t>(w & 0xff)) * s;
            f.y = static_cast<float>(static_cast<int8_t>((w >> 8) & 0xff)) * s;
            f.z = static_cast<float>(static_cast<int8_t>((w >> 16) & 0xff)) * s;
            f.w = static_cast<float>(static_cast<int8_t>(w >> 24)) * s;
            __stcs(ov + i, f);
        }
        done = n4 * 4;
    }
    for (int64_t i = done + tid; i < n; i += stride) out[i] = static_cast<float>(q[i]) * s;
}

__global__ void __launch_bounds__(256) k_dequant_rows(const int8_t* __restrict__ q, int64_t rows,
                                                      int64_t cols, const float* __restrict__ scales,
                                                      float* __restrict__ out) {
    QSB_PDL_ENTER();
    const int64_t row = blockIdx.y;
    const float s = scales[row];
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cols;
         c += (int64_t)gridDim.x * blockDim.x)
        out[row * cols + c] = static_cast<float>(q[row * cols + c]) * s;
}

// ---------------------------------------------------------------------------
// K4: elementwise casts (RNE).
// ---------------------------------------------------------------------------
template <int SD, int DD>
struct Store;
template <int SD>
struct Store<SD, QSYNC_F32> {
    using T = float;
    __device__ static T cvt(float v) { return v; }
};
template <int SD>
struct Store<SD, QSYNC_F16> {
    using T = __half;
    __device__ static T cvt(float v) { return __float2half_rn(v); }
};
template <int SD>
struct Store<SD, QSYNC_BF16> {
    using T = __nv_bfloat16;
    __device__ static T cvt(float v) { return __float2bfloat16_rn(v); }
};

// 8 elements per thread-iteration: src read as 16B vectors (2 for F32, 1 for
// 16-bit), dst written as 16B vectors; two iterations in flight per thread.
template <int SD>
__device__ __forceinline__ void load8(const typename Elem<SD>::T* x, int64_t i, float* f) {
    const uint4* v = reinterpret_cast<const uint4*>(x + i);
    if constexpr (SD == QSYNC_F8E4M3) {
        const uint2 w = *reinterpret_cast<const uint2*>(x + i);
        const uint32_t ww[2] = {w.x, w.y};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const __half2_raw h = __nv_cvt_fp8x2_to_halfraw2(
                static_cast<__nv_fp8x2_storage_t>((ww[k >> 1] >> (16 * (k & 1))) & 0xffffu), __NV_E4M3);
            const float2 t = __half22float2(__half2(h));
            f[2 * k] = t.x;
            f[2 * k + 1] = t.y;
        }
    } else if constexpr (SD == QSYNC_I8) {
        const uint2 w = *reinterpret_cast<const uint2*>(x + i);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            f[k] = static_cast<float>(static_cast<int8_t>((w.x >> (8 * k)) & 0xff));
            f[4 + k] = static_cast<float>(static_cast<int8_t>((w.y >> (8 * k)) & 0xff));
        }
    } else if constexpr (SD == QSYNC_F32) {
        Vec<QSYNC_F32>::unpack(ld_stream(v), f);
        Vec<QSYNC_F32>::unpack(ld_stream(v + 1), f + 4);
    } else {
        Vec<SD>::unpack(ld_stream(v), f);
    }
}
template <int DD>
__device__ __forceinline__ void store8(void* out, int64_t i, const float* f) {
    if (DD == QSYNC_F32) {
        float4* o = reinterpret_cast<float4*>(static_cast<float*>(out) + i);
        __stcs(o, make_float4(f[0], f[1], f[2], f[3]));
        __stcs(o + 1, make_float4(f[4], f[5], f[6], f[7]));
    } else {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            w[k] = DD == QSYNC_F16 ? pack_half2(f[2 * k], f[2 * k + 1]) : pack_bf162(f[2 * k], f[2 * k + 1]);
        }
        __stcs(reinterpret_cast<uint4*>(static_cast<uint16_t*>(out) + i), make_uint4(w[0], w[1], w[2], w[3]));
    }
}

template <int SD, int DD, int ACT = 0>
__global__ void __launch_bounds__(kThreads) k_cast(const typename Elem<SD>::T* __restrict__ x,
                                                   typename Store<SD, DD>::T* __restrict__ out,
                                                   int64_t n, int vec_ok,
                                                   uint16_t* __restrict__ dact = nullptr) {
    QSB_PDL_ENTER();
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (vec_ok) {
        const int64_t n8 = n / 8;
        int64_t i = tid;
        for (; i + stride < n8; i += 2 * stride) {
            float f0[8], f1[8];
            load8<SD>(x, i * 8, f0);
            load8<SD>(x, (i + stride) * 8, f1);
            if (ACT == 1 && dact) {  // GELU and GELU' share the erf
                float d0[8], d1[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    gelu_pair<SD != QSYNC_F32>(f0[j], f0[j], d0[j]);
                    gelu_pair<SD != QSYNC_F32>(f1[j], f1[j], d1[j]);
                    f0[j] = round_to<SD>(f0[j]);
                    f1[j] = round_to<SD>(f1[j]);
                }
                reinterpret_cast<uint4*>(dact)[i] =
                    make_uint4(pack_half2(d0[0], d0[1]), pack_half2(d0[2], d0[3]), pack_half2(d0[4], d0[5]),
                               pack_half2(d0[6], d0[7]));
                reinterpret_cast<uint4*>(dact)[i + stride] =
                    make_uint4(pack_half2(d1[0], d1[1]), pack_half2(d1[2], d1[3]), pack_half2(d1[4], d1[5]),
                               pack_half2(d1[6], d1[7]));
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    f0[j] = act_f<ACT, SD>(f0[j]);
                    f1[j] = act_f<ACT, SD>(f1[j]);
                }
            }
            store8<DD>(out, i * 8, f0);
            store8<DD>(out, (i + stride) * 8, f1);
        }
        for (; i < n8; i += stride) {
            float f0[8];
            load8<SD>(x, i * 8, f0);
            if (ACT == 1 && dact) {
                float d0[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    gelu_pair<SD != QSYNC_F32>(f0[j], f0[j], d0[j]);
                    f0[j] = round_to<SD>(f0[j]);
                }
                reinterpret_cast<uint4*>(dact)[i] =
                    make_uint4(pack_half2(d0[0], d0[1]), pack_half2(d0[2], d0[3]), pack_half2(d0[4], d0[5]),
                               pack_half2(d0[6], d0[7]));
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) f0[j] = act_f<ACT, SD>(f0[j]);
            }
            store8<DD>(out, i * 8, f0);
        }
        done = n8 * 8;
    }
    for (int64_t i = done + tid; i < n; i += stride) {
        const float xv = Elem<SD>::f(x[i]);
        out[i] = Store<SD, DD>::cvt(act_f<ACT, SD>(xv));
        if (ACT == 1 && dact) dact[i] = __half_as_ushort(__float2half_rn(gelu_erf_grad<SD != QSYNC_F32>(xv)));
    }
}

// ---------------------------------------------------------------------------
// K5: statistics.  Pass 1: per-block (sum x^2 in FP64, absmax) partials.
// Pass 2: one block reduces the partials in a fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr int kStatsBlocks = 1024;

template <int DT>
__global__ void __launch_bounds__(kThreads) k_stats_partial(const typename Elem<DT>::T* __restrict__ x,
                                                            int64_t n, double* __restrict__ part,
                                                            int vec_ok) {
    QSB_PDL_ENTER();
    using V = Vec<DT>;
    double ss = 0.0;
    float m = 0.0f;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (vec_ok) {
        const int64_t nv = n / V::N;
        const uint4* xv = reinterpret_cast<const uint4*>(x);
        // 4 x 16 B loads in flight per thread (as k_absmax): one load per
        // iteration left the smaller sweep sizes latency-bound (0.68 at 64 MB)
        constexpr int U = 4;
        int64_t i = tid;
        for (; i + (U - 1) * stride < nv; i += U * stride) {
            uint4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = ld_stream(xv + i + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float f[V::N];
                V::unpack(r[u], f);
#pragma unroll
                for (int j = 0; j < V::N; ++j) {
                    m = fmaxf(m, fabsf(f[j]));
                    ss = fma(static_cast<double>(f[j]), static_cast<double>(f[j]), ss);
                }
            }
        }
        for (; i < nv; i += stride) {
            float f[V::N];
            V::unpack(ld_stream(xv + i), f);
#pragma unroll
            for (int j = 0; j < V::N; ++j) {
                m = fmaxf(m, fabsf(f[j]));
                ss = fma(static_cast<double>(f[j]), static_cast<double>(f[j]), ss);
            }
        }
        done = nv * V::N;
    }
    for (int64_t i = done + tid; i < n; i += stride) {
        const float v = Elem<DT>::f(x[i]);
        m = fmaxf(m, fabsf(v));
        ss = fma(static_cast<double>(v), static_cast<double>(v), ss);
    }
    __shared__ double rs[32];
    __shared__ float rm[32];
    ss = warp_sum(ss);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) {
        rs[threadIdx.x >> 5] = ss;
        rm[threadIdx.x >> 5] = m;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const bool live = threadIdx.x < (blockDim.x >> 5);
        ss = warp_sum(live ? rs[threadIdx.x] : 0.0);
        m = warp_max(live ? rm[threadIdx.x] : 0.0f);
        if (threadIdx.x == 0) {
            part[2 * blockIdx.x] = ss;
            part[2 * blockIdx.x + 1] = static_cast<double>(m);
        }
    }
}

__global__ void __launch_bounds__(1024) k_stats_final(const double* __restrict__ part, int nparts,
                                                      int64_t n, double* __restrict__ out) {
    QSB_PDL_ENTER();
    __shared__ double rs[32];
    __shared__ double rm[32];
    double ss = 0.0, m = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
        ss += part[2 * i];
        m = fmax(m, part[2 * i + 1]);
    }
    ss = warp_sum(ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) {
        rs[threadIdx.x >> 5] = ss;
        rm[threadIdx.x >> 5] = m;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0, mm = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            t += rs[w];
            mm = fmax(mm, rm[w]);
        }
        const float a = static_cast<float>(mm);
        out[0] = t;
        out[1] = mm;
        out[2] = static_cast<double>(scale_from_absmax(a));
        out[3] = a > 0.0f ? floor(log2(mm)) : 0.0;
        out[4] = static_cast<double>(n);
    }
}

template <template <int> class F, typename... Args>
int dispatch_dtype(int dtype, Args&&... args) {
    switch (dtype) {
        case QSYNC_F32: return F<QSYNC_F32>::run(args...);
        case QSYNC_F16: return F<QSYNC_F16>::run(args...);
        case QSYNC_BF16: return F<QSYNC_BF16>::run(args...);
        default: return set_error(QSYNC_ERR_DOMAIN, "unsupported dtype " + std::to_string(dtype));
    }
}

template <int DT>
struct AbsmaxRun {
    static int run(const void* x, int64_t n, float* absmax, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        QSB_TRY(zero_async(absmax, sizeof(float), st));
        if (n == 0) return QSYNC_OK;
        const int vec = aligned16(x);
        const int grid = grid_for(n / Vec<DT>::N + 1, kThreads * 4);
        pdl_launch(k_absmax<DT>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n,
                                                reinterpret_cast<unsigned*>(absmax), vec);
        return check_launch("k_absmax");
    }
};

template <int DT>
struct AbsmaxRowsRun {
    static int run(const void* x, int64_t rows, int64_t cols, float* out, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        if (rows == 0) return QSYNC_OK;
        pdl_launch(k_absmax_rows<DT>, dim3(static_cast<unsigned>((rows + 7) / 8)), dim3(256), 0, st, 
            static_cast<const T*>(x), rows, cols, out);
        return check_launch("k_absmax_rows");
    }
};

template <int DT>
struct QuantRun {
    // scale[0] <- s, scale[1] <- absmax (scratch + output).
    static int run(const void* x, int64_t rows, int64_t cols, int8_t* q, float* scale,
                   void* q_t, int q_t_dtype, int64_t ld_t, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        const int64_t n = rows * cols;
        QSB_TRY(AbsmaxRun<DT>::run(x, n, scale + 1, st));
        if (q_t && n > 0) {
            dim3 grid(static_cast<unsigned>((cols + TC - 1) / TC), static_cast<unsigned>((rows + TR - 1) / TR));
            const int vt = (cols % 4 == 0) && aligned16(x) && aligned16(q) && aligned16(q_t);
            const bool t8 = q_t_dtype == QSYNC_I8;
            pdl_launch(k_tile<DT, 0>, dim3(grid), dim3(256), 0, st, static_cast<const T*>(x), rows, cols, scale + 1, q,
                                                nullptr, t8 ? nullptr : static_cast<uint16_t*>(q_t),
                                                ld_t, nullptr, scale, vt,
                                                t8 ? static_cast<int8_t*>(q_t) : nullptr);
            return check_launch("k_tile<quant>");
        }
        const int vec = (aligned16(x) && aligned16(q)) ? 3 : 0;  // bit 1: reverse walk (L2 reuse)
        const int grid = grid_for(n / 16 + 1, kThreads, 2);  // <= 64 regs: 2 x 512 threads per SM
        pdl_launch(k_quantize<DT>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n, scale + 1, nullptr,
                                                  q, scale, vec, static_cast<uint16_t*>(nullptr), static_cast<uint16_t*>(nullptr));
        return check_launch("k_quantize");
    }
};

template <int DT>
struct QuantScaleRun {
    static int run(const void* x, int64_t n, const float* scale, int8_t* q, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        if (n == 0) return QSYNC_OK;
        const int vec = aligned16(x) && aligned16(q);
        const int grid = grid_for(n / 16 + 1, kThreads, 2);  // <= 64 regs: 2 x 512 threads per SM
        pdl_launch(k_quantize<DT>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n, nullptr, scale, q,
                                                  nullptr, vec, static_cast<uint16_t*>(nullptr), static_cast<uint16_t*>(nullptr));
        return check_launch("k_quantize");
    }
};

template <int DT>
struct CastTRun {
    static int run(const void* x, int64_t rows, int64_t cols, uint16_t* out, uint16_t* out_t,
                   int64_t ld_t, float* colsum, int colsum_accumulate, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        if (colsum && !colsum_accumulate)
            QSB_TRY(zero_async(colsum, sizeof(float) * cols, st));
        if (rows == 0 || cols == 0) return QSYNC_OK;
        dim3 grid(static_cast<unsigned>((cols + TC - 1) / TC), static_cast<unsigned>((rows + TR - 1) / TR));
        const int vt = (cols % 4 == 0) && aligned16(x) && aligned16(out) && aligned16(out_t);
        pdl_launch(k_tile<DT, 1>, dim3(grid), dim3(256), 0, st, static_cast<const T*>(x), rows, cols, nullptr, nullptr,
                                            out, out_t, ld_t, colsum, nullptr, vt, static_cast<int8_t*>(nullptr));
        return check_launch("k_tile<cast>");
    }
};

template <int DT>
struct StatsRun {
    static int run(const void* x, int64_t n, double* out, void* ws, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        const int vec = aligned16(x);
        int grid = grid_for(n / Vec<DT>::N + 1, kThreads * 2, 4);
        grid = std::min(grid, kStatsBlocks);
        double* part = static_cast<double*>(ws);
        pdl_launch(k_stats_partial<DT>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n, part, vec);
        QSB_TRY(check_launch("k_stats_partial"));
        pdl_launch(k_stats_final, dim3(1), dim3(1024), 0, st, part, grid, n, out);
        return check_launch("k_stats_final");
    }
};

template <int DT>
struct AbsmaxActRun {
    static int run(const void* x, int64_t n, int act, float* absmax, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        QSB_TRY(zero_async(absmax, sizeof(float), st));
        if (n == 0) return QSYNC_OK;
        const int vec = aligned16(x);
        const int grid = grid_for(n / Vec<DT>::N + 1, kThreads * 4);
        if (act == 1)
            pdl_launch(k_absmax<DT, 1>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n,
                                                       reinterpret_cast<unsigned*>(absmax), vec);
        else
            pdl_launch(k_absmax<DT, 0>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n,
                                                       reinterpret_cast<unsigned*>(absmax), vec);
        return check_launch("k_absmax");
    }
};

template <int DT>
struct GeluAbsmaxStoreRun {
    static int run(const void* x, int64_t n, float* absmax, void* y, uint16_t* dact, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        QSB_TRY(zero_async(absmax, sizeof(float), st));
        if (n == 0) return QSYNC_OK;
        const int vec = aligned16(x) && aligned16(y) && (!dact || aligned16(dact));
        const int grid = grid_for(n / 8 + 1, kThreads, 4);
        pdl_launch(k_gelu_absmax_store<DT>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n,
                   reinterpret_cast<unsigned*>(absmax), static_cast<T*>(y), dact, vec);
        return check_launch("k_gelu_absmax_store");
    }
};

// ---------------------------------------------------------------------------
// FF2's INT8 operand from FF1's FP32 output h in ONE pass when the answer is
// known up front.  The unfused path quantizes g = gelu(h) with s = absmax(g)/127.
// gelu (this library's float32 function) is monotone only up to ulp-level
// dips, but over every float32 x in [0, 16] above 0.1701, gelu(y) >= gelu(x)
// for every y at least kGeluGap ulps above x (checked exhaustively with steps
// of kGeluGap .. 2 kGeluGap - 1 ulps, which compose into any larger gap, by
// qsync_gelu_fp32_check), and |gelu(h)| < 0.1701 for every h < 0.  So with hmax
// the largest h (reduced by FF1's GEMM epilogue, qsync_gemm_s8_ymax): if
// gelu(hmax) >= 0.1701 and no float within kGeluGap ulps below hmax has a larger
// gelu, absmax(g) = gelu(hmax) exactly and the quantizer needs no absmax pass
// over g: read h, write q, FP16(q) and GELU'(h).  Otherwise the kernel takes
// the exact absmax over gelu(h) first, across a grid barrier (one co-resident
// wave).  q / s / q16 / GELU' are bit-identical to gelu_absmax_store +
// quantize_act either way.
constexpr float kGeluMonoFloor = 0.1701f;
constexpr int kGeluGap = 16;
constexpr int kGqSlots = 32;
constexpr int kGqMaxBlocks = 2048;
__device__ float g_gq_part[kGqSlots][kGqMaxBlocks];
__device__ unsigned g_gq_bar[kGqSlots][2];

__device__ __forceinline__ void gq_grid_barrier(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g0 = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g0) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_gelu_quant(const float* __restrict__ h, int64_t n,
                                                     const float* __restrict__ hmax, int8_t* __restrict__ q,
                                                     uint16_t* __restrict__ q16, uint16_t* __restrict__ dact,
                                                     float* __restrict__ scale_out, int slot, int vec_ok) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // dependents only after the (possible) barrier
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const float hm = fmaxf(*hmax, 0.0f);
    const float gm = gelu_erf<false>(hm);
    bool fast = gm >= kGeluMonoFloor;
    if (fast) {  // no float just below hmax may have a larger gelu (ulp-level dips):
        // lane k-1 of every warp checks hmax - k ulps, k = 1 .. kGeluGap-1
        static_assert(kGeluGap <= 32, "one candidate per lane");
        const uint32_t hb = __float_as_uint(hm);
        const uint32_t k = (threadIdx.x & 31) + 1;
        const bool dip = k < static_cast<uint32_t>(kGeluGap) && k <= hb &&
                         gelu_erf<false>(__uint_as_float(hb - k)) > gm;
        fast = !__any_sync(0xffffffffu, dip);
    }
    float am = gm;
    if (!fast) {  // exact fallback: absmax over gelu(h)
        float m = 0.0f;
        for (int64_t i = tid; i < n; i += stride) m = fmaxf(m, fabsf(gelu_erf<false>(h[i])));
        __shared__ float red[8];
        m = warp_max(m);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            float b = 0.0f;
            for (int w = 0; w < 8; ++w) b = fmaxf(b, red[w]);
            g_gq_part[slot][blockIdx.x] = b;
        }
        gq_grid_barrier(g_gq_bar[slot], gridDim.x);
        __shared__ float s_am;
        if (threadIdx.x == 0) {
            float b = 0.0f;
            for (int i = 0; i < static_cast<int>(gridDim.x); ++i) b = fmaxf(b, __ldcg(&g_gq_part[slot][i]));
            s_am = b;
        }
        __syncthreads();
        am = s_am;
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const float sc = scale_from_absmax(am);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        scale_out[0] = sc;
        scale_out[1] = am;
    }
    const QScale qs = make_qscale(sc);
    int64_t done = 0;
    if (vec_ok) {  // 8 elements per thread-iteration: 2 x 16 B loads, 8 B of q, 16 B of q16 and GELU'
        const int64_t n8 = n / 8;
        for (int64_t i = tid; i < n8; i += stride) {
            float f[8];
            Vec<QSYNC_F32>::unpack(ld_stream(reinterpret_cast<const uint4*>(h) + 2 * i), f);
            Vec<QSYNC_F32>::unpack(ld_stream(reinterpret_cast<const uint4*>(h) + 2 * i + 1), f + 4);
            float t[8];
            uint32_t dp[4], hq[4];
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                float g0, g1, d0, d1;
                gelu_pair<false>(f[j], g0, d0);
                gelu_pair<false>(f[j + 1], g1, d1);
                t[j] = quant_rne_f(g0, qs);
                t[j + 1] = quant_rne_f(g1, qs);
                dp[j / 2] = pack_half2(d0, d1);
                hq[j / 2] = pack_half2(grid_value(t[j]), grid_value(t[j + 1]));
            }
            reinterpret_cast<uint2*>(q)[i] = make_uint2(pack_q4(t[0], t[1], t[2], t[3]), pack_q4(t[4], t[5], t[6], t[7]));
            if (q16) reinterpret_cast<uint4*>(q16)[i] = make_uint4(hq[0], hq[1], hq[2], hq[3]);
            if (dact) reinterpret_cast<uint4*>(dact)[i] = make_uint4(dp[0], dp[1], dp[2], dp[3]);
        }
        done = n8 * 8;
    }
    for (int64_t i = done + tid; i < n; i += stride) {
        float g, d;
        gelu_pair<false>(h[i], g, d);
        const int qi = quant_rne(g, qs);
        q[i] = static_cast<int8_t>(qi);
        if (q16) q16[i] = __half_as_ushort(__int2half_rn(qi));
        if (dact) dact[i] = __half_as_ushort(__float2half_rn(d));
    }
}

// Exhaustive checks behind k_gelu_quant's shortcut: over every float32 x in
// [0, 16] with gelu(x) > 0.1701, count the steps y = x + j ulp, j in
// [kGeluGap, 2 kGeluGap), with gelu(y) < gelu(x) (must be 0; outside [0, 16]
// gelu(h) is h); and max |gelu(h)| over h in [-16, 0) (must be < 0.1701).  A
// block takes 1024 consecutive floats and their 2 kGeluGap successors from
// shared memory.
__global__ void __launch_bounds__(256) k_gelu_check(unsigned* out) {
    constexpr int kChunk = 1024;
    __shared__ float gs[kChunk + 2 * kGeluGap];
    const uint32_t top = 0x41800000u;  // 16.0f
    unsigned viol = 0;
    float negmax = 0.0f;
    for (uint32_t b0 = blockIdx.x * kChunk; b0 < top; b0 += gridDim.x * kChunk) {
        __syncthreads();
        for (int i = threadIdx.x; i < kChunk + 2 * kGeluGap; i += blockDim.x)
            gs[i] = gelu_erf<false>(__uint_as_float(b0 + i));
        __syncthreads();
        for (int i = threadIdx.x; i < kChunk; i += blockDim.x) {
            const float g = gs[i];
            if (g > kGeluMonoFloor) {
                for (int j = kGeluGap; j < 2 * kGeluGap; ++j) viol += gs[i + j] < g ? 1u : 0u;
            }
            negmax = fmaxf(negmax, fabsf(gelu_erf<false>(-__uint_as_float(b0 + i))));
        }
    }
    if (viol) atomicAdd(out, viol);
    negmax = warp_max(negmax);
    if ((threadIdx.x & 31) == 0 && negmax > 0.0f) atomicMax(out + 1, __float_as_uint(negmax));
}

template <int DT>
struct QuantActRun {
    static int run(const void* x, int64_t n, int act, const float* absmax, int8_t* q,
                   float* scale_out, uint16_t* dact, uint16_t* q16, cudaStream_t st) {
        using T = typename Elem<DT>::T;
        if (n == 0) return QSYNC_OK;
        const int vec = aligned16(x) && aligned16(q) && (!dact || aligned16(dact)) && (!q16 || aligned16(q16));
        const int grid = grid_for(n / 16 + 1, kThreads, 2);  // <= 64 regs: 2 x 512 threads per SM
        if (act == 1)
            pdl_launch(k_quantize<DT, 1>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n, absmax, nullptr,
                                                         q, scale_out, vec, dact, q16);
        else
            pdl_launch(k_quantize<DT, 0>, dim3(grid), dim3(kThreads), 0, st, static_cast<const T*>(x), n, absmax, nullptr,
                                                         q, scale_out, vec, static_cast<uint16_t*>(nullptr), q16);
        return check_launch("k_quantize");
    }
};

}  // namespace

}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_absmax(const void* x, int dtype, int64_t n, float* absmax, qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    return dispatch_dtype<AbsmaxRun>(dtype, x, n, absmax, to_stream(stream));
}

int qsync_absmax_rows(const void* x, int dtype, int64_t rows, int64_t cols, float* out,
                      qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0 && cols >= 0, QSYNC_ERR_DOMAIN, "negative shape");
    return dispatch_dtype<AbsmaxRowsRun>(dtype, x, rows, cols, out, to_stream(stream));
}

int qsync_quantize_per_tensor(const void* x, int dtype, int64_t rows, int64_t cols, int8_t* q,
                              float* scale, void* q_t, int q_t_dtype, int64_t ld_t,
                              qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0 && cols >= 0, QSYNC_ERR_DOMAIN, "negative shape");
    QSB_REQUIRE(scale != nullptr, QSYNC_ERR_VALIDATION, "scale buffer (float[2]) is required");
    QSB_REQUIRE(!q_t || q_t_dtype == QSYNC_F16 || q_t_dtype == QSYNC_I8, QSYNC_ERR_DOMAIN,
                "transposed copy must be F16 or I8");
    if (ld_t <= 0) ld_t = rows;
    QSB_REQUIRE(ld_t >= rows, QSYNC_ERR_DOMAIN, "transposed pitch must be >= rows");
    return dispatch_dtype<QuantRun>(dtype, x, rows, cols, q, scale, q_t, q_t_dtype, ld_t,
                                    to_stream(stream));
}

int qsync_quantize_with_scale(const void* x, int dtype, int64_t n, const float* scale, int8_t* q,
                              qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    return dispatch_dtype<QuantScaleRun>(dtype, x, n, scale, q, to_stream(stream));
}

int qsync_quantize_per_channel(const float* w, int64_t rows, int64_t cols, int8_t* q,
                               float* scales, uint16_t* w_t_f16, qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0 && cols >= 0, QSYNC_ERR_DOMAIN, "negative shape");
    cudaStream_t st = to_stream(stream);
    if (rows == 0) return QSYNC_OK;
    pdl_launch(k_quant_rows, dim3(static_cast<unsigned>((rows + 7) / 8)), dim3(256), 0, st, w, rows, cols, q, scales);
    QSB_TRY(check_launch("k_quant_rows"));
    if (w_t_f16) return CastTRun<QSYNC_F32>::run(w, rows, cols, nullptr, w_t_f16, rows, nullptr, 0, st);
    return QSYNC_OK;
}

int qsync_dequantize_per_tensor(const int8_t* q, int64_t n, const float* scale, float* out,
                                qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    if (n == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int vec = aligned16(q) && aligned16(out);
    pdl_launch(k_dequant, dim3(grid_for(n / 16 + 1, kThreads, 4)), dim3(kThreads), 0, st, q, n, scale, out, vec);
    return check_launch("k_dequant");
}

int qsync_dequantize_per_channel(const int8_t* q, int64_t rows, int64_t cols, const float* scales,
                                 float* out, qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0 && cols >= 0, QSYNC_ERR_DOMAIN, "negative shape");
    QSB_REQUIRE(rows < 65536, QSYNC_ERR_DOMAIN, "per-channel dequantize supports < 65536 rows");
    if (rows == 0 || cols == 0) return QSYNC_OK;
    dim3 grid(static_cast<unsigned>(std::min<int64_t>((cols + 255) / 256, 64)), static_cast<unsigned>(rows));
    pdl_launch(k_dequant_rows, dim3(grid), dim3(256), 0, to_stream(stream), q, rows, cols, scales, out);
    return check_launch("k_dequant_rows");
}

int qsync_cast(const void* x, int src, void* out, int dst, int64_t n, qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    if (n == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int grid = grid_for(n / 8 + 1, kThreads * 2, 4);
    const int vec = aligned16(x) && aligned16(out);
#define QSB_CAST(S, D)                                                                     \
    if (src == S && dst == D) {                                                            \
        pdl_launch(k_cast<S, D>, dim3(grid), dim3(kThreads), 0, st, static_cast<const typename Elem<S>::T*>(x), \
                                                static_cast<typename Store<S, D>::T*>(out), n, vec, static_cast<uint16_t*>(nullptr)); \
        return check_launch("k_cast");                                                     \
    }
    QSB_CAST(QSYNC_F32, QSYNC_F16)
    QSB_CAST(QSYNC_F32, QSYNC_BF16)
    QSB_CAST(QSYNC_F16, QSYNC_F32)
    QSB_CAST(QSYNC_BF16, QSYNC_F32)
    QSB_CAST(QSYNC_F16, QSYNC_BF16)
    QSB_CAST(QSYNC_BF16, QSYNC_F16)
    QSB_CAST(QSYNC_I8, QSYNC_F16)
    QSB_CAST(QSYNC_I8, QSYNC_F32)
    QSB_CAST(QSYNC_F8E4M3, QSYNC_F16)
    QSB_CAST(QSYNC_F8E4M3, QSYNC_F32)
#undef QSB_CAST
    return set_error(QSYNC_ERR_DOMAIN, "unsupported cast " + std::to_string(src) + "->" + std::to_string(dst));
}

int qsync_cast_transpose(const void* x, int dtype, int64_t rows, int64_t cols, uint16_t* out,
                         uint16_t* out_t, int64_t ld_t, float* colsum, int colsum_accumulate,
                         qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0 && cols >= 0, QSYNC_ERR_DOMAIN, "negative shape");
    QSB_REQUIRE(rows / TR < 65535, QSYNC_ERR_DOMAIN, "too many rows for cast_transpose");
    if (ld_t <= 0) ld_t = rows;
    QSB_REQUIRE(ld_t >= rows, QSYNC_ERR_DOMAIN, "transposed pitch must be >= rows");
    return dispatch_dtype<CastTRun>(dtype, x, rows, cols, out, out_t, ld_t, colsum,
                                    colsum_accumulate, to_stream(stream));
}

size_t qsync_stats_workspace_bytes(void) { return sizeof(double) * 2 * kStatsBlocks; }

int qsync_tensor_stats(const void* x, int dtype, int64_t n, double* out, void* workspace,
                       qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    QSB_REQUIRE(workspace != nullptr, QSYNC_ERR_VALIDATION, "stats workspace is required");
    return dispatch_dtype<StatsRun>(dtype, x, n, out, workspace, to_stream(stream));
}

int qsync_absmax_act(const void* x, int dtype, int64_t n, int act, float* absmax,
                     qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    QSB_REQUIRE(act == QSYNC_ACT_NONE || act == QSYNC_ACT_GELU, QSYNC_ERR_DOMAIN, "unknown activation");
    return dispatch_dtype<AbsmaxActRun>(dtype, x, n, act, absmax, to_stream(stream));
}

int qsync_quantize_act(const void* x, int dtype, int64_t n, int act, const float* absmax, int8_t* q,
                       float* scale_out, uint16_t* dact_out, qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    QSB_REQUIRE(absmax != nullptr, QSYNC_ERR_VALIDATION, "absmax is required");
    QSB_REQUIRE(act == QSYNC_ACT_NONE || act == QSYNC_ACT_GELU, QSYNC_ERR_DOMAIN, "unknown activation");
    return dispatch_dtype<QuantActRun>(dtype, x, n, act, absmax, q, scale_out, dact_out,
                                       static_cast<uint16_t*>(nullptr), to_stream(stream));
}

int qsync_gelu_absmax_store(const void* x, int dtype, int64_t n, float* absmax, void* y, uint16_t* dact_out,
                            qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    QSB_REQUIRE(absmax != nullptr && y != nullptr, QSYNC_ERR_VALIDATION, "absmax and y are required");
    QSB_REQUIRE(dtype == QSYNC_F32 || dtype == QSYNC_F16, QSYNC_ERR_DOMAIN, "x must be F32 or F16");
    if (dtype == QSYNC_F32)
        return GeluAbsmaxStoreRun<QSYNC_F32>::run(x, n, absmax, y, dact_out, to_stream(stream));
    return GeluAbsmaxStoreRun<QSYNC_F16>::run(x, n, absmax, y, dact_out, to_stream(stream));
}

int qsync_gelu_quantize(const float* h, int64_t n, const float* hmax, int8_t* q, uint16_t* q16, uint16_t* dact_out,
                        float* scale_out, qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    QSB_REQUIRE(h && hmax && q && scale_out, QSYNC_ERR_VALIDATION, "h, hmax, q and scale_out (float[2]) are required");
    if (n == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    static int occ[16] = {0};
    int dev = 0;
    QSB_TRY(cuda_status(cudaGetDevice(&dev), "cudaGetDevice"));
    if (dev < 16 && occ[dev] == 0) {
        int nb = 0;
        QSB_TRY(cuda_status(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_gelu_quant, 256, 0),
                            "cudaOccupancyMaxActiveBlocksPerMultiprocessor"));
        occ[dev] = nb > 0 ? nb : 1;
    }
    const int per_sm = dev < 16 ? occ[dev] : 1;
    // one co-resident wave (the fallback's grid barrier needs every block resident)
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>({(n / 8 + 255) / 256, int64_t(per_sm) * sm_count(), int64_t(kGqMaxBlocks)})));
    const int vec = aligned16(h) && (reinterpret_cast<uintptr_t>(q) & 7) == 0 && (!q16 || aligned16(q16)) &&
                    (!dact_out || aligned16(dact_out));
    const int slot = static_cast<int>((reinterpret_cast<uintptr_t>(st) >> 4) % kGqSlots);
    pdl_launch(k_gelu_quant, dim3(grid), dim3(256), 0, st, h, n, hmax, q, q16, dact_out, scale_out, slot, vec);
    return check_launch("k_gelu_quant");
}

int qsync_gelu_fp32_check(unsigned* out) {
    QSB_REQUIRE(out != nullptr, QSYNC_ERR_VALIDATION, "out (uint32[2], zeroed) is required");
    k_gelu_check<<<sm_count() * 8, 256>>>(out);
    return check_launch("k_gelu_check");
}

int qsync_quantize_act_ex(const void* x, int dtype, int64_t n, int act, const float* absmax, int8_t* q,
                          float* scale_out, uint16_t* dact_out, uint16_t* q16_out, qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    QSB_REQUIRE(absmax != nullptr, QSYNC_ERR_VALIDATION, "absmax is required");
    QSB_REQUIRE(act == QSYNC_ACT_NONE || act == QSYNC_ACT_GELU, QSYNC_ERR_DOMAIN, "unknown activation");
    return dispatch_dtype<QuantActRun>(dtype, x, n, act, absmax, q, scale_out, dact_out, q16_out,
                                       to_stream(stream));
}

int qsync_act_cast(const void* x, int src, void* out, int dst, int64_t n, int act, uint16_t* dact_out,
                   qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    if (act == QSYNC_ACT_NONE) return qsync_cast(x, src, out, dst, n, stream);
    QSB_REQUIRE(act == QSYNC_ACT_GELU, QSYNC_ERR_DOMAIN, "unknown activation");
    if (n == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int grid = grid_for(n / 8 + 1, kThreads * 2, 4);
    const int vec = aligned16(x) && aligned16(out) && (!dact_out || aligned16(dact_out));
#define QSB_ACAST(S, D)                                                                       \
    if (src == S && dst == D) {                                                               \
        pdl_launch(k_cast<S, D, 1>, dim3(grid), dim3(kThreads), 0, st, static_cast<const typename Elem<S>::T*>(x), \
                                                   static_cast<typename Store<S, D>::T*>(out), n, vec, dact_out); \
        return check_launch("k_cast<gelu>");                                                  \
    }
    QSB_ACAST(QSYNC_F32, QSYNC_F32)
    QSB_ACAST(QSYNC_F32, QSYNC_F16)
    QSB_ACAST(QSYNC_F16, QSYNC_F16)
    QSB_ACAST(QSYNC_F16, QSYNC_F32)
#undef QSB_ACAST
    return set_error(QSYNC_ERR_DOMAIN, "unsupported activation cast " + std::to_string(src) + "->" +
                                           std::to_string(dst));
}

int qsync_quantize_fp8(const void* x, int dtype, int64_t n, const float* absmax, uint8_t* q, float* scale_out,
                       qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    QSB_REQUIRE(absmax != nullptr, QSYNC_ERR_VALIDATION, "absmax is required");
    return dispatch_dtype<QuantFp8Run>(dtype, x, n, absmax, q, scale_out, to_stream(stream));
}

int qsync_quantize_fp8_rows(const float* w, int64_t rows, int64_t cols, uint8_t* q, float* scales,
                            qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0 && cols >= 0, QSYNC_ERR_DOMAIN, "negative shape");
    if (rows == 0) return QSYNC_OK;
    pdl_launch(k_quant_rows_fp8, dim3(static_cast<unsigned>((rows + 7) / 8)), dim3(256), 0, to_stream(stream), w,
               rows, cols, q, scales);
    return check_launch("k_quant_rows_fp8");
}

}  // extern "C"

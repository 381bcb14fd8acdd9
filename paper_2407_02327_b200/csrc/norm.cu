// norm.cu -- fused residual-add + LayerNorm forward / backward (the glue between
// the planned Linears of an encoder layer: LN(x + sublayer(x))).
//
// One warp per row, the row held in registers (cols <= 1024, cols % 128 == 0
// for the vector path; BERT-base hidden 768), grid-stride over rows.
//   fwd: s = a + b  (b FP32 or FP16 -- the planned op's output format,
//        graph.hpp:38-40), y = (s - mean) * rstd * gamma + beta; saves s, mean, rstd.
//   bwd: xh = (s - mean) * rstd, g = dy * gamma,
//        dx = rstd * (g - mean(g) - xh * mean(g * xh)),
//        dgamma += sum_rows dy * xh, dbeta += sum_rows dy  (accumulated into the
//        caller's FP32 buffers -- the parameters' main_grad slices).
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"
#include "vec.cuh"

#ifndef QSB_LN_FWD_MINB
#define QSB_LN_FWD_MINB 1  // A/B (tools/ab_step.py lib=): 1, 2 and 4 blocks / SM within 0.2%
#endif

namespace qsb {
namespace {

template <int NV>
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void red_add_v4(float* p, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

// Fused per-tensor quantizer state (kQ): per-block absmax partials and a
// self-resetting grid barrier, one slot per stream (slot = stream hash), in
// statically allocated device memory -- nothing to allocate or zero per call.
constexpr int kLnQSlots = 32;
constexpr int kLnQMaxBlocks = 1024;
__device__ float g_lnq_part[kLnQSlots][kLnQMaxBlocks];
__device__ unsigned g_lnq_bar[kLnQSlots][2];  // [0] arrivals, [1] generation

// Grid-wide barrier over co-resident blocks (the host checks residency): the
// last arriving block resets the count and bumps the generation the others
// spin on.  Each kernel uses its slot once, and launches on one stream are
// ordered, so a slot is never shared by two live barriers.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g0 = *gen;  // read before arriving: it cannot move until every block arrived
        __threadfence();           // this block's partial is visible before its arrival
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

// kQ: LayerNorm + per-tensor INT8 quantizer of y in one kernel (the input of an
// INT8-planned Linear).  One row per warp and every block co-resident: the
// normalised row stays in shared memory across a grid barrier on absmax(y), then
// is quantized with s = absmax/127 (quant_rne_f, bit-identical to
// qsync_quantize_act_ex on the stored y) -- y is not read back and the
// separate quantize launch is gone.  qs[0] = s, qs[1] = absmax.
template <int NV, int BDT, bool kQ = false>
__global__ void __launch_bounds__(256, kQ ? 4 : QSB_LN_FWD_MINB) k_ln_fwd(const float* __restrict__ a,
                                                const typename Elem<BDT>::T* __restrict__ b,
                                                const float* __restrict__ gamma,
                                                const float* __restrict__ beta, int64_t rows,
                                                int cols, float eps, float* __restrict__ s_out,
                                                float* __restrict__ y, float* __restrict__ mean_out,
                                                float* __restrict__ rstd_out,
                                                __half* __restrict__ y16,
                                                unsigned* __restrict__ y_absmax,
                                                const int64_t* __restrict__ tok = nullptr,
                                                const float* __restrict__ pos = nullptr,
                                                const float* __restrict__ typ = nullptr,
                                                int seq = 1, int8_t* __restrict__ q = nullptr,
                                                uint16_t* __restrict__ q16 = nullptr,
                                                float* __restrict__ qs = nullptr, int qslot = 0) {
    if constexpr (kQ) {
        asm volatile("griddepcontrol.wait;" ::: "memory");  // dependents only after the barrier
    } else {
        QSB_PDL_ENTER();
    }
    const int lane = threadIdx.x & 31;
    float amax = 0.0f;
    int64_t keep_row = -1;
    // kQ: this warp's normalised row, parked in shared memory across the barrier
    __shared__ float4 s_keep[kQ ? 8 : 1][kQ ? NV : 1][32];
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    // gamma / beta are read at use (L1-resident, shared by all rows) rather than
    // held across the grid-stride rows: 48 registers less, which the fused
    // quantizer needs (<= 64 registers: 4 blocks / SM, one row per warp for
    // BERT's 4096 rows co-resident).
    constexpr bool kHold = false;
    float4 g[kHold ? NV : 1], be[kHold ? NV : 1];
    if constexpr (kHold) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            g[i] = reinterpret_cast<const float4*>(gamma)[lane + 32 * i];
            be[i] = reinterpret_cast<const float4*>(beta)[lane + 32 * i];
        }
    }
    const float inv_n = 1.0f / static_cast<float>(cols);
    for (int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
         row += warps) {
        float4 v[NV];
        float sum = 0.0f;
#pragma unroll
        // Embedding mode: a is the word table, the row's input is
        // word[tok[row]] + pos[row % seq] + typ[0] (gathered, never materialised).
        const int64_t arow = tok ? tok[row] : row;
        const int64_t prow = tok ? row % seq : 0;
        for (int i = 0; i < NV; ++i) {
            const int64_t off = row * cols + 4 * (lane + 32 * i);
            float4 x = *reinterpret_cast<const float4*>(a + arow * cols + 4 * (lane + 32 * i));
            if (tok) {
                const float4 p4 = *reinterpret_cast<const float4*>(pos + prow * cols + 4 * (lane + 32 * i));
                const float4 t4 = reinterpret_cast<const float4*>(typ)[lane + 32 * i];
                // (word + pos) + typ: the association of the unfused path, bit for bit
                x.x = (x.x + p4.x) + t4.x; x.y = (x.y + p4.y) + t4.y;
                x.z = (x.z + p4.z) + t4.z; x.w = (x.w + p4.w) + t4.w;
            } else if (b) {
                if (BDT == QSYNC_F32) {
                    const float4 r = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(b) + off);
                    x.x += r.x; x.y += r.y; x.z += r.z; x.w += r.w;
                } else {
                    const uint2 r = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(b) + off);
                    const float2 r0 = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
                    const float2 r1 = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
                    x.x += r0.x; x.y += r0.y; x.z += r1.x; x.w += r1.y;
                }
            }
            v[i] = x;
            sum += (x.x + x.y) + (x.z + x.w);
            if (s_out) *reinterpret_cast<float4*>(s_out + off) = x;
        }
        const float mean = warp_sum_f<NV>(sum) * inv_n;
        float sq = 0.0f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const float dx = v[i].x - mean, dy = v[i].y - mean, dz = v[i].z - mean, dw = v[i].w - mean;
            sq += (dx * dx + dy * dy) + (dz * dz + dw * dw);
        }
        const float rstd = rsqrtf(warp_sum_f<NV>(sq) * inv_n + eps);
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int64_t off = row * cols + 4 * (lane + 32 * i);
            const float4 gi = kHold ? g[kHold ? i : 0] : __ldg(reinterpret_cast<const float4*>(gamma) + lane + 32 * i);
            const float4 bi = kHold ? be[kHold ? i : 0] : __ldg(reinterpret_cast<const float4*>(beta) + lane + 32 * i);
            float4 o;
            o.x = (v[i].x - mean) * rstd * gi.x + bi.x;
            o.y = (v[i].y - mean) * rstd * gi.y + bi.y;
            o.z = (v[i].z - mean) * rstd * gi.z + bi.z;
            o.w = (v[i].w - mean) * rstd * gi.w + bi.w;
            *reinterpret_cast<float4*>(y + off) = o;
            if constexpr (kQ) s_keep[threadIdx.x >> 5][i][lane] = o;
            if (y16) {
                uint2 h;
                h.x = pack_half2(o.x, o.y);
                h.y = pack_half2(o.z, o.w);
                *reinterpret_cast<uint2*>(y16 + off) = h;
            }
            amax = fmaxf(amax, fmaxf(fmaxf(fabsf(o.x), fabsf(o.y)), fmaxf(fabsf(o.z), fabsf(o.w))));
        }
        if (lane == 0) {
            mean_out[row] = mean;
            rstd_out[row] = rstd;
        }
        if constexpr (kQ) keep_row = row;
    }
    if constexpr (kQ) {
        __shared__ float wmax[8];
        __shared__ float s_abs;
        amax = warp_max(amax);
        if (lane == 0) wmax[threadIdx.x >> 5] = amax;
        __syncthreads();
        if (threadIdx.x < 32) {
            amax = warp_max(threadIdx.x < (blockDim.x >> 5) ? wmax[threadIdx.x] : 0.0f);
            if (threadIdx.x == 0) g_lnq_part[qslot][blockIdx.x] = amax;
        }
        grid_barrier(g_lnq_bar[qslot], gridDim.x);
        // every block reduces all partials (deterministic, no accumulator to zero)
        float m = 0.0f;
        for (int i = threadIdx.x; i < static_cast<int>(gridDim.x); i += blockDim.x)
            m = fmaxf(m, __ldcg(&g_lnq_part[qslot][i]));
        m = warp_max(m);
        if (lane == 0) wmax[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            float t = 0.0f;
            for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t = fmaxf(t, wmax[w]);
            s_abs = t;
        }
        __syncthreads();
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        const float sc = scale_from_absmax(s_abs);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            qs[0] = sc;
            qs[1] = s_abs;
        }
        const QScale qsc = make_qscale(sc);
        if (keep_row >= 0) {
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int64_t off = keep_row * cols + 4 * (lane + 32 * i);
                const float4 o = s_keep[threadIdx.x >> 5][i][lane];
                const float t0 = quant_rne_f(o.x, qsc), t1 = quant_rne_f(o.y, qsc);
                const float t2 = quant_rne_f(o.z, qsc), t3 = quant_rne_f(o.w, qsc);
                *reinterpret_cast<uint32_t*>(q + off) = pack_q4(t0, t1, t2, t3);
                if (q16) {
                    uint2 h;
                    h.x = pack_half2(grid_value(t0), grid_value(t1));
                    h.y = pack_half2(grid_value(t2), grid_value(t3));
                    *reinterpret_cast<uint2*>(q16 + off) = h;
                }
            }
        }
        return;
    }
    if (y_absmax) {
        // absmax of y for the next INT8 op's per-tensor scale: warp max, block
        // max through shared memory, one atomicMax per block on the float bits
        // (order-independent, so deterministic).
        __shared__ float wmax[8];
        amax = warp_max(amax);
        if (lane == 0) wmax[threadIdx.x >> 5] = amax;
        __syncthreads();
        if (threadIdx.x < 32) {
            amax = warp_max(threadIdx.x < (blockDim.x >> 5) ? wmax[threadIdx.x] : 0.0f);
            if (threadIdx.x == 0 && amax > 0.0f) atomicMax(y_absmax, __float_as_uint(amax));
        }
    }
}

template <int NV>
__global__ void __launch_bounds__(256) k_ln_bwd(const float* __restrict__ dy,
                                                const float* __restrict__ s,
                                                const float* __restrict__ mean_in,
                                                const float* __restrict__ rstd_in,
                                                const float* __restrict__ gamma, int64_t rows,
                                                int cols, float* __restrict__ dx,
                                                float* __restrict__ dgamma,
                                                float* __restrict__ dbeta,
                                                __half* __restrict__ dx16,
                                                float* __restrict__ dcol) {
    QSB_PDL_ENTER();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    float4 g[NV], acc_g[NV], acc_b[NV], acc_c[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        g[i] = reinterpret_cast<const float4*>(gamma)[lane + 32 * i];
        acc_g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        acc_b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        acc_c[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float inv_n = 1.0f / static_cast<float>(cols);
    for (int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; row < rows; row += warps) {
        const float mean = mean_in[row], rstd = rstd_in[row];
        float4 xh[NV], gy[NV];
        float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int64_t off = row * cols + 4 * (lane + 32 * i);
            const float4 d = *reinterpret_cast<const float4*>(dy + off);
            const float4 x = *reinterpret_cast<const float4*>(s + off);
            xh[i] = make_float4((x.x - mean) * rstd, (x.y - mean) * rstd, (x.z - mean) * rstd,
                                (x.w - mean) * rstd);
            gy[i] = make_float4(d.x * g[i].x, d.y * g[i].y, d.z * g[i].z, d.w * g[i].w);
            s1 += (gy[i].x + gy[i].y) + (gy[i].z + gy[i].w);
            s2 += (gy[i].x * xh[i].x + gy[i].y * xh[i].y) + (gy[i].z * xh[i].z + gy[i].w * xh[i].w);
            acc_g[i].x += d.x * xh[i].x; acc_g[i].y += d.y * xh[i].y;
            acc_g[i].z += d.z * xh[i].z; acc_g[i].w += d.w * xh[i].w;
            acc_b[i].x += d.x; acc_b[i].y += d.y; acc_b[i].z += d.z; acc_b[i].w += d.w;
        }
        const float m1 = warp_sum_f<NV>(s1) * inv_n;
        const float m2 = warp_sum_f<NV>(s2) * inv_n;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int64_t off = row * cols + 4 * (lane + 32 * i);
            float4 o;
            o.x = rstd * (gy[i].x - m1 - xh[i].x * m2);
            o.y = rstd * (gy[i].y - m1 - xh[i].y * m2);
            o.z = rstd * (gy[i].z - m1 - xh[i].z * m2);
            o.w = rstd * (gy[i].w - m1 - xh[i].w * m2);
            *reinterpret_cast<float4*>(dx + off) = o;
            if (dx16) {
                uint2 h;
                h.x = pack_half2(o.x, o.y);
                h.y = pack_half2(o.z, o.w);
                *reinterpret_cast<uint2*>(dx16 + off) = h;
            }
            acc_c[i].x += o.x; acc_c[i].y += o.y; acc_c[i].z += o.z; acc_c[i].w += o.w;
        }
    }
    // Block-reduce the per-warp column partials (gamma, then beta through the
    // same smem buffer), then one atomic per column per block.
    __shared__ float red[8][1024 + 4];
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int pass = 0; pass < 3; ++pass) {
        float* outp = pass == 0 ? dgamma : (pass == 1 ? dbeta : dcol);
        if (pass == 2 && !dcol) break;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const float4 v = pass == 0 ? acc_g[i] : (pass == 1 ? acc_b[i] : acc_c[i]);
            const int c = 4 * (lane + 32 * i);
            red[warp][c] = v.x; red[warp][c + 1] = v.y; red[warp][c + 2] = v.z; red[warp][c + 3] = v.w;
        }
        __syncthreads();
        for (int c = threadIdx.x; c < cols; c += blockDim.x) {
            float t = 0.f;
            for (int w = 0; w < nw; ++w) t += red[w][c];
            if (outp) atomicAdd(outp + c, t);
        }
        __syncthreads();
    }
}

// Same LN backward with each row split over a warp PAIR (NV even): every lane
// owns NV/2 float4 columns, which halves the per-lane column accumulators and
// brings the kernel to 2 blocks / SM.  The two halves' row sums are exchanged
// through shared memory under a 64-thread named barrier.
#ifndef QSB_LN_BWD_MINB
#define QSB_LN_BWD_MINB 2
#endif
// ST > 0: each pair's rows of dy and s are staged in shared memory by 1-D bulk
// copies issued ST rows ahead (mbarrier per stage), so a pair keeps ST rows of
// loads in flight through its reductions and stores; ST = 0 loads straight into
// registers.
template <int NV, int ST>
__global__ void __launch_bounds__(256, QSB_LN_BWD_MINB) k_ln_bwd2(const float* __restrict__ dy,
                                                    const float* __restrict__ s,
                                                    const float* __restrict__ mean_in,
                                                    const float* __restrict__ rstd_in,
                                                    const float* __restrict__ gamma, int64_t rows,
                                                    int cols, float* __restrict__ dx,
                                                    float* __restrict__ dgamma,
                                                    float* __restrict__ dbeta,
                                                    __half* __restrict__ dx16,
                                                    float* __restrict__ dcol,
                                                    int red4,
                                                    const int64_t* __restrict__ tok = nullptr,
                                                    float* __restrict__ dword = nullptr,
                                                    float* __restrict__ dpos = nullptr,
                                                    int seq = 1) {
    QSB_PDL_ENTER();
    constexpr int NH = NV / 2;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int pair = warp >> 1, half = warp & 1;
    const int cbase = half * NH * 128;  // first column of this warp's half
    const int64_t pairs = (int64_t)gridDim.x * 4;
    float4 g[NH], acc_g[NH], acc_b[NH], acc_c[NH];
#pragma unroll
    for (int i = 0; i < NH; ++i) {
        g[i] = reinterpret_cast<const float4*>(gamma + cbase)[lane + 32 * i];
        acc_g[i] = acc_b[i] = acc_c[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float inv_n = 1.0f / static_cast<float>(cols);
    int parity = 0;
    const int64_t row0 = blockIdx.x * (int64_t)4 + pair;
    extern __shared__ __align__(16) float lnb_stage[];
    __shared__ __align__(8) uint64_t lnb_bar[4][ST > 0 ? ST : 1];
    float* stage = lnb_stage + static_cast<size_t>(pair) * (ST > 0 ? ST : 1) * 2 * cols;
    const bool issuer = half == 0 && lane == 0;
    const uint32_t row_bytes = static_cast<uint32_t>(cols) * 4u;
    if constexpr (ST > 0) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < 4 * ST; ++i) ptx::mbar_init(&lnb_bar[i / ST][i % ST], 1);
            ptx::fence_mbar_init();
        }
        __syncthreads();
        if (issuer) {
#pragma unroll
            for (int k = 0; k < ST; ++k) {
                const int64_t r = row0 + k * pairs;
                if (r < rows) {
                    ptx::mbar_arrive_expect_tx(&lnb_bar[pair][k], 2 * row_bytes);
                    ptx::bulk_load_1d(stage + k * 2 * cols, dy + r * cols, row_bytes, &lnb_bar[pair][k]);
                    ptx::bulk_load_1d(stage + k * 2 * cols + cols, s + r * cols, row_bytes, &lnb_bar[pair][k]);
                }
            }
        }
    }
    float mean_n = 0.f, rstd_n = 0.f;
    if (row0 < rows) {
        mean_n = mean_in[row0];
        rstd_n = rstd_in[row0];
    }
    int it = 0;
    for (int64_t row = row0; row < rows; row += pairs, ++it) {
        const float mean = mean_n, rstd = rstd_n;
        if (row + pairs < rows) {  // next row's statistics in flight under this row
            mean_n = mean_in[row + pairs];
            rstd_n = rstd_in[row + pairs];
        }
        const float* dyr = dy + row * cols + cbase;
        const float* sr = s + row * cols + cbase;
        if constexpr (ST > 0) {
            ptx::mbar_wait(&lnb_bar[pair][it % ST], static_cast<uint32_t>(it / ST) & 1u);
            dyr = stage + (it % ST) * 2 * cols + cbase;
            sr = dyr + cols;
        }
        float4 xh[NH], gy[NH];
        float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            const float4 d = reinterpret_cast<const float4*>(dyr)[lane + 32 * i];
            const float4 x = reinterpret_cast<const float4*>(sr)[lane + 32 * i];
            xh[i] = make_float4((x.x - mean) * rstd, (x.y - mean) * rstd, (x.z - mean) * rstd,
                                (x.w - mean) * rstd);
            gy[i] = make_float4(d.x * g[i].x, d.y * g[i].y, d.z * g[i].z, d.w * g[i].w);
            s1 += (gy[i].x + gy[i].y) + (gy[i].z + gy[i].w);
            s2 += (gy[i].x * xh[i].x + gy[i].y * xh[i].y) + (gy[i].z * xh[i].z + gy[i].w * xh[i].w);
            acc_g[i].x += d.x * xh[i].x; acc_g[i].y += d.y * xh[i].y;
            acc_g[i].z += d.z * xh[i].z; acc_g[i].w += d.w * xh[i].w;
            acc_b[i].x += d.x; acc_b[i].y += d.y; acc_b[i].z += d.z; acc_b[i].w += d.w;
        }
        s1 = warp_sum_f<NV>(s1);
        s2 = warp_sum_f<NV>(s2);
        // exchange with the partner warp (double-buffered by row parity)
        __shared__ float xb[2][4][2][2];
        if (lane == 0) {
            xb[parity][pair][half][0] = s1;
            xb[parity][pair][half][1] = s2;
        }
        asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory");
        s1 += xb[parity][pair][half ^ 1][0];
        s2 += xb[parity][pair][half ^ 1][1];
        parity ^= 1;
        if constexpr (ST > 0) {
            // both warps of the pair have read this stage (the named barrier above):
            // refill it with the row ST iterations ahead
            const int64_t r = row + ST * pairs;
            if (issuer && r < rows) {
                const int k = it % ST;
                ptx::mbar_arrive_expect_tx(&lnb_bar[pair][k], 2 * row_bytes);
                ptx::bulk_load_1d(stage + k * 2 * cols, dy + r * cols, row_bytes, &lnb_bar[pair][k]);
                ptx::bulk_load_1d(stage + k * 2 * cols + cols, s + r * cols, row_bytes, &lnb_bar[pair][k]);
            }
        }
        const float m1 = s1 * inv_n;
        const float m2 = s2 * inv_n;
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            const int64_t off = row * cols + cbase + 4 * (lane + 32 * i);
            float4 o;
            o.x = rstd * (gy[i].x - m1 - xh[i].x * m2);
            o.y = rstd * (gy[i].y - m1 - xh[i].y * m2);
            o.z = rstd * (gy[i].z - m1 - xh[i].z * m2);
            o.w = rstd * (gy[i].w - m1 - xh[i].w * m2);
            if (tok) {
                // Embedding mode: scatter-add into the word row and the position row
                // (vector reductions in L2), never materialising dx.
                const int c = cbase + 4 * (lane + 32 * i);
                red_add_v4(dword + tok[row] * cols + c, o);
                red_add_v4(dpos + (row % seq) * cols + c, o);
            } else {
                *reinterpret_cast<float4*>(dx + off) = o;
            }
            if (dx16) {
                uint2 h;
                h.x = pack_half2(o.x, o.y);
                h.y = pack_half2(o.z, o.w);
                *reinterpret_cast<uint2*>(dx16 + off) = h;
            }
            acc_c[i].x += o.x; acc_c[i].y += o.y; acc_c[i].z += o.z; acc_c[i].w += o.w;
        }
    }
    // Column partials: 4 pairs per block, reduced through shared memory.
    __shared__ float red[4][1024 + 4];
#pragma unroll
    for (int pass = 0; pass < 3; ++pass) {
        float* outp = pass == 0 ? dgamma : (pass == 1 ? dbeta : dcol);
        if (pass == 2 && !dcol) break;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            const float4 v = pass == 0 ? acc_g[i] : (pass == 1 ? acc_b[i] : acc_c[i]);
            const int c = cbase + 4 * (lane + 32 * i);
            red[pair][c] = v.x; red[pair][c + 1] = v.y; red[pair][c + 2] = v.z; red[pair][c + 3] = v.w;
        }
        __syncthreads();
        if (!red4) {  // a column-sum target not 16-byte aligned: scalar atomics
            for (int c = threadIdx.x; c < cols; c += blockDim.x) {
                const float t = (red[0][c] + red[1][c]) + (red[2][c] + red[3][c]);
                if (outp) atomicAdd(outp + c, t);
            }
            continue;
        }
        // one 16-byte vector reduction per 4 columns (a quarter of the L2 atomics)
        for (int c = 4 * threadIdx.x; c < cols; c += 4 * blockDim.x) {
            float4 t;
            t.x = (red[0][c] + red[1][c]) + (red[2][c] + red[3][c]);
            t.y = (red[0][c + 1] + red[1][c + 1]) + (red[2][c + 1] + red[3][c + 1]);
            t.z = (red[0][c + 2] + red[1][c + 2]) + (red[2][c + 2] + red[3][c + 2]);
            t.w = (red[0][c + 3] + red[1][c + 3]) + (red[2][c + 3] + red[3][c + 3]);
            if (outp) red_add_v4(outp + c, t);
        }
    }
}

template <int NV>
int ln_fwd_nv(const float* a, const void* b, int b_dtype, const float* gamma, const float* beta,
              int64_t rows, int cols, float eps, float* s_out, float* y, float* mean, float* rstd,
              uint16_t* y16, float* y_absmax, cudaStream_t st) {
    if (y_absmax) QSB_TRY(zero_async(y_absmax, sizeof(float), st));
    const int grid = static_cast<int>(std::min<int64_t>((rows + 7) / 8, sm_count() * 8LL));
    if (b_dtype == QSYNC_F16)
        pdl_launch(k_ln_fwd<NV, QSYNC_F16>, dim3(grid), dim3(256), 0, st, a, static_cast<const __half*>(b), gamma, beta,
                                                      rows, cols, eps, s_out, y, mean, rstd,
                                                      reinterpret_cast<__half*>(y16),
                                                      reinterpret_cast<unsigned*>(y_absmax), nullptr, nullptr,
                                                      nullptr, 1, static_cast<int8_t*>(nullptr),
                                                      static_cast<uint16_t*>(nullptr), static_cast<float*>(nullptr), 0);
    else
        pdl_launch(k_ln_fwd<NV, QSYNC_F32>, dim3(grid), dim3(256), 0, st, a, static_cast<const float*>(b), gamma, beta,
                                                      rows, cols, eps, s_out, y, mean, rstd,
                                                      reinterpret_cast<__half*>(y16),
                                                      reinterpret_cast<unsigned*>(y_absmax), nullptr, nullptr,
                                                      nullptr, 1, static_cast<int8_t*>(nullptr),
                                                      static_cast<uint16_t*>(nullptr), static_cast<float*>(nullptr), 0);
    return check_launch("k_ln_fwd");
}

// LayerNorm (+ embedding gather when tok) fused with the per-tensor INT8
// quantizer of y (k_ln_fwd<kQ>) when one row per warp fits co-resident;
// otherwise LayerNorm with absmax, then the one-pass quantizer -- the same q,
// q16 and qs either way.
template <int NV, int BDT>
int ln_fwd_quant_launch(const float* a, const void* b, const int64_t* tok, const float* pos, const float* typ,
                        int seq, const float* gamma, const float* beta, int64_t rows, int cols, float eps,
                        float* s_out, float* y, float* mean, float* rstd, int8_t* q, uint16_t* q16, float* qs,
                        cudaStream_t st) {
    using BT = typename Elem<BDT>::T;
    const int64_t blocks = (rows + 7) / 8;
    static int occ[16] = {0};
    int dev = 0;
    QSB_TRY(cuda_status(cudaGetDevice(&dev), "cudaGetDevice"));
    if (dev < 16 && occ[dev] == 0) {
        int n = 0;
        QSB_TRY(cuda_status(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_ln_fwd<NV, BDT, true>, 256, 0),
                            "cudaOccupancyMaxActiveBlocksPerMultiprocessor"));
        occ[dev] = n > 0 ? n : -1;
    }
    const int per_sm = dev < 16 ? occ[dev] : 0;
    if (per_sm > 0 && blocks <= kLnQMaxBlocks && blocks <= static_cast<int64_t>(per_sm) * sm_count()) {
        const int slot = static_cast<int>((reinterpret_cast<uintptr_t>(st) >> 4) % kLnQSlots);
        pdl_launch(k_ln_fwd<NV, BDT, true>, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st, a,
                   static_cast<const BT*>(b), gamma, beta, rows, cols, eps, s_out, y, mean, rstd,
                   static_cast<__half*>(nullptr), static_cast<unsigned*>(nullptr), tok, pos, typ, seq, q, q16, qs,
                   slot);
        return check_launch("k_ln_fwd<quant>");
    }
    QSB_TRY(zero_async(qs + 1, sizeof(float), st));
    const int grid = static_cast<int>(std::min<int64_t>(blocks, sm_count() * 8LL));
    pdl_launch(k_ln_fwd<NV, BDT>, dim3(grid), dim3(256), 0, st, a, static_cast<const BT*>(b), gamma, beta, rows, cols,
               eps, s_out, y, mean, rstd, static_cast<__half*>(nullptr), reinterpret_cast<unsigned*>(qs + 1), tok, pos,
               typ, seq, static_cast<int8_t*>(nullptr), static_cast<uint16_t*>(nullptr), static_cast<float*>(nullptr),
               0);
    QSB_TRY(check_launch("k_ln_fwd"));
    return qsync_quantize_act_ex(y, QSYNC_F32, rows * cols, QSYNC_ACT_NONE, qs + 1, q, qs, nullptr, q16, st);
}

template <int NV>
int ln_fwd_quant_nv(const float* a, const void* b, int b_dtype, const int64_t* tok, const float* pos,
                    const float* typ, int seq, const float* gamma, const float* beta, int64_t rows, int cols,
                    float eps, float* s_out, float* y, float* mean, float* rstd, int8_t* q, uint16_t* q16, float* qs,
                    cudaStream_t st) {
    if (b_dtype == QSYNC_F16)
        return ln_fwd_quant_launch<NV, QSYNC_F16>(a, b, tok, pos, typ, seq, gamma, beta, rows, cols, eps, s_out, y,
                                                  mean, rstd, q, q16, qs, st);
    return ln_fwd_quant_launch<NV, QSYNC_F32>(a, b, tok, pos, typ, seq, gamma, beta, rows, cols, eps, s_out, y, mean,
                                              rstd, q, q16, qs, st);
}

// Bulk-staged LN backward (k_ln_bwd2<NV, ST > 0>): stage depth by row width so
// two blocks per SM fit (4 pairs x ST stages x 2 rows x cols floats each).
// Two stages measured best in the step (ab_step lib=: 4.466 ms vs 4.48 with 1
// or 3; the side-stream GEMMs co-schedule better next to smaller blocks).
#ifndef QSB_LN_BWD_ST
#define QSB_LN_BWD_ST 2
#endif
constexpr int ln_bwd_stages(int nv) {
    return QSB_LN_BWD_ST <= 0 ? 0 : (32 * QSB_LN_BWD_ST * nv * 128 <= 90000 ? QSB_LN_BWD_ST : 1);
}
constexpr int ln_bwd_smem(int nv, int st) { return 4 * st * 2 * nv * 128 * 4; }
inline bool ln_bwd_staged(const float* dy, const float* s) {
    return QSB_LN_BWD_ST > 0 && aligned16(dy) && aligned16(s);
}

template <int NV>
int ln_bwd_nv(const float* dy, const float* s, const float* mean, const float* rstd,
              const float* gamma, int64_t rows, int cols, float* dx, float* dgamma, float* dbeta,
              uint16_t* dx16, float* dcol, cudaStream_t st) {
    if constexpr (NV % 2 == 0) {
        // one resident wave (QSB_LN_BWD_MINB blocks / SM): every block amortises
        // its column-partial reduction over as many rows as possible
        const int grid = static_cast<int>(std::min<int64_t>((rows + 3) / 4, sm_count() * int64_t(QSB_LN_BWD_MINB)));
        const int red4 = aligned16(dgamma) && aligned16(dbeta) && aligned16(dcol);
        if (ln_bwd_staged(dy, s)) {
            constexpr int ST = ln_bwd_stages(NV);
            const int smem = ln_bwd_smem(NV, ST);
            QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_ln_bwd2<NV, ST>), smem));
            pdl_launch(k_ln_bwd2<NV, ST>, dim3(grid), dim3(256), smem, st, dy, s, mean, rstd, gamma, rows, cols, dx,
                       dgamma, dbeta, reinterpret_cast<__half*>(dx16), dcol, red4, nullptr, nullptr, nullptr, 1);
            return check_launch("k_ln_bwd<staged>");
        }
        pdl_launch(k_ln_bwd2<NV, 0>, dim3(grid), dim3(256), 0, st, dy, s, mean, rstd, gamma, rows, cols, dx, dgamma, dbeta,
                                             reinterpret_cast<__half*>(dx16), dcol, red4, nullptr, nullptr, nullptr, 1);
        return check_launch("k_ln_bwd");
    }
    const int grid = static_cast<int>(std::min<int64_t>((rows + 7) / 8, sm_count() * 2LL));
    pdl_launch(k_ln_bwd<NV>, dim3(grid), dim3(256), 0, st, dy, s, mean, rstd, gamma, rows, cols, dx, dgamma, dbeta,
                                        reinterpret_cast<__half*>(dx16), dcol);
    return check_launch("k_ln_bwd");
}

template <int NV>
int embed_ln_fwd_nv(const int64_t* tok, int64_t rows, int seq, const float* word, const float* pos,
                    const float* typ, const float* gamma, const float* beta, int cols, float eps, float* s_out,
                    float* y, float* mean, float* rstd, uint16_t* y16, float* y_absmax, cudaStream_t st) {
    if (y_absmax) QSB_TRY(zero_async(y_absmax, sizeof(float), st));
    const int grid = static_cast<int>(std::min<int64_t>((rows + 7) / 8, sm_count() * 8LL));
    pdl_launch(k_ln_fwd<NV, QSYNC_F32>, dim3(grid), dim3(256), 0, st, word, static_cast<const float*>(nullptr), gamma, beta, rows, cols, eps, s_out, y, mean,
                                                  rstd, reinterpret_cast<__half*>(y16),
                                                  reinterpret_cast<unsigned*>(y_absmax), tok, pos, typ, seq,
                                                  static_cast<int8_t*>(nullptr), static_cast<uint16_t*>(nullptr),
                                                  static_cast<float*>(nullptr), 0);
    return check_launch("k_ln_fwd<embed>");
}

template <int NV>
int embed_ln_bwd_nv(const float* dy, const float* s, const float* mean, const float* rstd, const float* gamma,
                    const int64_t* tok, int64_t rows, int seq, int cols, float* dgamma, float* dbeta,
                    float* dword, float* dpos, float* dtyp, cudaStream_t st) {
    const int grid = static_cast<int>(std::min<int64_t>((rows + 3) / 4, sm_count() * int64_t(QSB_LN_BWD_MINB)));
    const int red4 = static_cast<int>(aligned16(dgamma) && aligned16(dbeta) && aligned16(dtyp));
    if (ln_bwd_staged(dy, s)) {
        constexpr int ST = ln_bwd_stages(NV);
        const int smem = ln_bwd_smem(NV, ST);
        QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_ln_bwd2<NV, ST>), smem));
        pdl_launch(k_ln_bwd2<NV, ST>, dim3(grid), dim3(256), smem, st, dy, s, mean, rstd, gamma, rows, cols,
                   static_cast<float*>(nullptr), dgamma, dbeta, static_cast<__half*>(nullptr), dtyp, red4, tok, dword,
                   dpos, seq);
        return check_launch("k_ln_bwd<embed, staged>");
    }
    pdl_launch(k_ln_bwd2<NV, 0>, dim3(grid), dim3(256), 0, st, dy, s, mean, rstd, gamma, rows, cols, static_cast<float*>(nullptr), dgamma, dbeta,
                                         static_cast<__half*>(nullptr), dtyp, red4, tok, dword, dpos, seq);
    return check_launch("k_ln_bwd<embed>");
}

}  // namespace
}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_layernorm_fwd_ex(const float* a, const void* b, int b_dtype, const float* gamma,
                           const float* beta, int64_t rows, int64_t cols, float eps, float* s_out,
                           float* y, float* mean, float* rstd, uint16_t* y16, float* y_absmax,
                           qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0, QSYNC_ERR_DOMAIN, "negative row count");
    QSB_REQUIRE(cols % 128 == 0 && cols >= 128 && cols <= 1024, QSYNC_ERR_DOMAIN,
                "layernorm supports 128 <= cols <= 1024, cols % 128 == 0");
    QSB_REQUIRE(b_dtype == QSYNC_F32 || b_dtype == QSYNC_F16, QSYNC_ERR_DOMAIN,
                "residual operand must be F32 or F16");
    if (rows == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int c = static_cast<int>(cols);
    switch (c / 128) {
        case 1: return ln_fwd_nv<1>(a, b, b_dtype, gamma, beta, rows, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        case 2: return ln_fwd_nv<2>(a, b, b_dtype, gamma, beta, rows, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        case 3: return ln_fwd_nv<3>(a, b, b_dtype, gamma, beta, rows, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        case 4: return ln_fwd_nv<4>(a, b, b_dtype, gamma, beta, rows, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        case 5: return ln_fwd_nv<5>(a, b, b_dtype, gamma, beta, rows, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        case 6: return ln_fwd_nv<6>(a, b, b_dtype, gamma, beta, rows, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        case 7: return ln_fwd_nv<7>(a, b, b_dtype, gamma, beta, rows, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        default: return ln_fwd_nv<8>(a, b, b_dtype, gamma, beta, rows, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
    }
}

int qsync_layernorm_fwd_quant(const float* a, const void* b, int b_dtype, const float* gamma, const float* beta,
                              int64_t rows, int64_t cols, float eps, float* s_out, float* y, float* mean,
                              float* rstd, int8_t* q, uint16_t* q16, float* scale, qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0, QSYNC_ERR_DOMAIN, "negative row count");
    QSB_REQUIRE(cols % 128 == 0 && cols >= 128 && cols <= 1024, QSYNC_ERR_DOMAIN,
                "layernorm supports 128 <= cols <= 1024, cols % 128 == 0");
    QSB_REQUIRE(b_dtype == QSYNC_F32 || b_dtype == QSYNC_F16, QSYNC_ERR_DOMAIN,
                "residual operand must be F32 or F16");
    QSB_REQUIRE(q != nullptr && scale != nullptr, QSYNC_ERR_VALIDATION, "q and scale (float[2]) are required");
    if (rows == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int c = static_cast<int>(cols);
#define QSB_LNQ(NV) \
    return ln_fwd_quant_nv<NV>(a, b, b_dtype, nullptr, nullptr, nullptr, 1, gamma, beta, rows, c, eps, s_out, y, mean, \
                               rstd, q, q16, scale, st)
    switch (c / 128) {
        case 1: QSB_LNQ(1);
        case 2: QSB_LNQ(2);
        case 3: QSB_LNQ(3);
        case 4: QSB_LNQ(4);
        case 5: QSB_LNQ(5);
        case 6: QSB_LNQ(6);
        case 7: QSB_LNQ(7);
        default: QSB_LNQ(8);
    }
#undef QSB_LNQ
}

int qsync_embed_layernorm_fwd_quant(const int64_t* tokens, int64_t rows, int64_t seq, const float* word,
                                    const float* pos, const float* typ, const float* gamma, const float* beta,
                                    int64_t cols, float eps, float* s_out, float* y, float* mean, float* rstd,
                                    int8_t* q, uint16_t* q16, float* scale, qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0 && seq > 0, QSYNC_ERR_DOMAIN, "bad rows / seq");
    QSB_REQUIRE(cols % 128 == 0 && cols >= 128 && cols <= 1024, QSYNC_ERR_DOMAIN,
                "layernorm supports 128 <= cols <= 1024, cols % 128 == 0");
    QSB_REQUIRE(tokens && word && pos && typ, QSYNC_ERR_VALIDATION, "tokens and embedding tables are required");
    QSB_REQUIRE(q != nullptr && scale != nullptr, QSYNC_ERR_VALIDATION, "q and scale (float[2]) are required");
    if (rows == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int c = static_cast<int>(cols);
#define QSB_ELNQ(NV)                                                                                          \
    return ln_fwd_quant_nv<NV>(word, nullptr, QSYNC_F32, tokens, pos, typ, static_cast<int>(seq), gamma, beta, rows, \
                               c, eps, s_out, y, mean, rstd, q, q16, scale, st)
    switch (c / 128) {
        case 1: QSB_ELNQ(1);
        case 2: QSB_ELNQ(2);
        case 3: QSB_ELNQ(3);
        case 4: QSB_ELNQ(4);
        case 5: QSB_ELNQ(5);
        case 6: QSB_ELNQ(6);
        case 7: QSB_ELNQ(7);
        default: QSB_ELNQ(8);
    }
#undef QSB_ELNQ
}

int qsync_layernorm_bwd_ex(const float* dy, const float* s, const float* mean, const float* rstd,
                           const float* gamma, int64_t rows, int64_t cols, float* dx, float* dgamma,
                           float* dbeta, uint16_t* dx16, float* dcolsum, qsync_stream_t stream) {
    QSB_REQUIRE(rows >= 0, QSYNC_ERR_DOMAIN, "negative row count");
    QSB_REQUIRE(cols % 128 == 0 && cols >= 128 && cols <= 1024, QSYNC_ERR_DOMAIN,
                "layernorm supports 128 <= cols <= 1024, cols % 128 == 0");
    if (rows == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int c = static_cast<int>(cols);
    switch (c / 128) {
        case 1: return ln_bwd_nv<1>(dy, s, mean, rstd, gamma, rows, c, dx, dgamma, dbeta, dx16, dcolsum, st);
        case 2: return ln_bwd_nv<2>(dy, s, mean, rstd, gamma, rows, c, dx, dgamma, dbeta, dx16, dcolsum, st);
        case 3: return ln_bwd_nv<3>(dy, s, mean, rstd, gamma, rows, c, dx, dgamma, dbeta, dx16, dcolsum, st);
        case 4: return ln_bwd_nv<4>(dy, s, mean, rstd, gamma, rows, c, dx, dgamma, dbeta, dx16, dcolsum, st);
        case 5: return ln_bwd_nv<5>(dy, s, mean, rstd, gamma, rows, c, dx, dgamma, dbeta, dx16, dcolsum, st);
        case 6: return ln_bwd_nv<6>(dy, s, mean, rstd, gamma, rows, c, dx, dgamma, dbeta, dx16, dcolsum, st);
        case 7: return ln_bwd_nv<7>(dy, s, mean, rstd, gamma, rows, c, dx, dgamma, dbeta, dx16, dcolsum, st);
        default: return ln_bwd_nv<8>(dy, s, mean, rstd, gamma, rows, c, dx, dgamma, dbeta, dx16, dcolsum, st);
    }
}

int qsync_layernorm_fwd(const float* a, const void* b, int b_dtype, const float* gamma,
                        const float* beta, int64_t rows, int64_t cols, float eps, float* s_out,
                        float* y, float* mean, float* rstd, qsync_stream_t stream) {
    return qsync_layernorm_fwd_ex(a, b, b_dtype, gamma, beta, rows, cols, eps, s_out, y, mean, rstd,
                                  nullptr, nullptr, stream);
}

int qsync_layernorm_bwd(const float* dy, const float* s, const float* mean, const float* rstd,
                        const float* gamma, int64_t rows, int64_t cols, float* dx, float* dgamma,
                        float* dbeta, qsync_stream_t stream) {
    return qsync_layernorm_bwd_ex(dy, s, mean, rstd, gamma, rows, cols, dx, dgamma, dbeta, nullptr,
                                  nullptr, stream);
}

int qsync_embed_layernorm_fwd(const int64_t* tokens, int64_t rows, int64_t seq, const float* word,
                              const float* pos, const float* typ, const float* gamma, const float* beta,
                              int64_t cols, float eps, float* s_out, float* y, float* mean, float* rstd,
                              uint16_t* y16, float* y_absmax, qsync_stream_t stream) {
    QSB_REQUIRE(tokens && word && pos && typ && s_out && y && mean && rstd, QSYNC_ERR_VALIDATION,
                "embedding LayerNorm needs tokens, tables and outputs");
    QSB_REQUIRE(rows >= 0 && seq > 0, QSYNC_ERR_DOMAIN, "bad row / sequence count");
    QSB_REQUIRE(cols == 768 || cols == 1024 || cols == 512 || cols == 256, QSYNC_ERR_DOMAIN,
                "embedding LayerNorm supports hidden 256, 512, 768, 1024");
    if (rows == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int c = static_cast<int>(cols), sq = static_cast<int>(seq);
    switch (c / 128) {
        case 2: return embed_ln_fwd_nv<2>(tokens, rows, sq, word, pos, typ, gamma, beta, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        case 4: return embed_ln_fwd_nv<4>(tokens, rows, sq, word, pos, typ, gamma, beta, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        case 6: return embed_ln_fwd_nv<6>(tokens, rows, sq, word, pos, typ, gamma, beta, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
        default: return embed_ln_fwd_nv<8>(tokens, rows, sq, word, pos, typ, gamma, beta, c, eps, s_out, y, mean, rstd, y16, y_absmax, st);
    }
}

int qsync_embed_layernorm_bwd(const float* dy, const float* s, const float* mean, const float* rstd,
                              const float* gamma, const int64_t* tokens, int64_t rows, int64_t seq, int64_t cols,
                              float* dgamma, float* dbeta, float* dword, float* dpos, float* dtyp,
                              qsync_stream_t stream) {
    QSB_REQUIRE(dy && s && mean && rstd && gamma && tokens && dword && dpos && dtyp, QSYNC_ERR_VALIDATION,
                "embedding LayerNorm backward needs all buffers");
    QSB_REQUIRE(rows >= 0 && seq > 0, QSYNC_ERR_DOMAIN, "bad row / sequence count");
    QSB_REQUIRE(cols == 768 || cols == 1024 || cols == 512 || cols == 256, QSYNC_ERR_DOMAIN,
                "embedding LayerNorm supports hidden 256, 512, 768, 1024");
    if (rows == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int c = static_cast<int>(cols), sq = static_cast<int>(seq);
    switch (c / 128) {
        case 2: return embed_ln_bwd_nv<2>(dy, s, mean, rstd, gamma, tokens, rows, sq, c, dgamma, dbeta, dword, dpos, dtyp, st);
        case 4: return embed_ln_bwd_nv<4>(dy, s, mean, rstd, gamma, tokens, rows, sq, c, dgamma, dbeta, dword, dpos, dtyp, st);
        case 6: return embed_ln_bwd_nv<6>(dy, s, mean, rstd, gamma, tokens, rows, sq, c, dgamma, dbeta, dword, dpos, dtyp, st);
        default: return embed_ln_bwd_nv<8>(dy, s, mean, rstd, gamma, tokens, rows, sq, c, dgamma, dbeta, dword, dpos, dtyp, st);
    }
}

}  // extern "C"

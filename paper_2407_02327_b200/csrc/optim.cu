// optim.cu -- AdamW on the FP32 master weights fused with the per-step weight
// preparation of the planned kernels.
//
// Every planned Linear reads its weight in the plan's format each step: an
// INT8 op per-channel INT8 W^ + scales and FP16 W for its
// FP16 dgrad (cost_mapper.cpp:13-15), an FP16 op FP16 W.  Those copies are a
// pure function of the master weights, which change only in the optimizer, so
// the optimizer kernel that has just produced row r of W also emits row r's
// copies: the weights are read once per step instead of once by the optimizer
// and again by each quantize / cast kernel.
//
// One warp per weight row (row = output channel; 1-D parameters are one row).
// Pass 1 updates p, m, v (16-byte vectors) and tracks the row absmax of the
// new p; pass 2 re-reads the row (L2-resident, just written) and writes the
// FP16 copy and the RNE INT8 copy with s = absmax/127 -- the same scale rule
// and rounding as k_quant_rows, so the prepared copy is bit-identical to
// qsync_quantize_per_channel of the updated weights.
//
// AdamW exactly as torch.optim.AdamW (decoupled decay):
//   p *= 1 - lr*wd;  m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2
//   p -= (lr / (1 - b1^t)) * m / (sqrt(v) / sqrt(1 - b2^t) + eps)
// with t read from a device counter (graph-capturable), incremented by a
// one-thread kernel after the update.
#include <algorithm>

#include "common.cuh"

namespace qsb {
namespace {

constexpr int kWarps = 8;

__device__ __forceinline__ int find_seg(const int64_t* start, int nseg, int64_t row) {
    int lo = 0, hi = nseg - 1;  // largest s with start[s] <= row
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (start[mid] <= row) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

struct AdamCoef {
    float lr, b1, b2, eps, decay;  // decay = 1 - lr*wd
    float step_size, inv_bc2_sqrt;
};

__device__ __forceinline__ float adam1(float p, float g, float& m, float& v, const AdamCoef& c) {
    p = p * c.decay;
    m = c.b1 * m + (1.0f - c.b1) * g;
    v = c.b2 * v + (1.0f - c.b2) * g * g;
    const float denom = sqrtf(v) * c.inv_bc2_sqrt + c.eps;
    return p - c.step_size * (m / denom);
}

#ifndef QSB_ADAM_MINB
#define QSB_ADAM_MINB 4  // 64 registers: 4 x 256 threads resident per SM (2 at 88 regs held HBM at 0.69)
#endif
__global__ void __launch_bounds__(kWarps * 32, QSB_ADAM_MINB) k_adamw(const qsync_adamw_seg* __restrict__ segs, int nseg,
                                                       const int64_t* seg_start, int64_t row_begin,
                                                       int64_t total_rows, const int64_t* __restrict__ step,
                                                       float lr, float b1, float b2, float eps, float wd,
                                                       int update) {
    QSB_PDL_ENTER();
    const int lane = threadIdx.x & 31;
    AdamCoef c{};
    if (update) {
        const float t = static_cast<float>(*step + 1);
        const float bc1 = 1.0f - powf(b1, t);
        const float bc2 = 1.0f - powf(b2, t);
        c.lr = lr;
        c.b1 = b1;
        c.b2 = b2;
        c.eps = eps;
        c.decay = 1.0f - lr * wd;
        c.step_size = lr / bc1;
        c.inv_bc2_sqrt = 1.0f / sqrtf(bc2);
    }
    // Segment row offsets staged in shared memory: the per-row binary search
    // would otherwise be a chain of dependent global loads.
    extern __shared__ int64_t s_start[];
    for (int i = threadIdx.x; i <= nseg; i += blockDim.x) s_start[i] = seg_start[i];
    __syncthreads();
    seg_start = s_start;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
    for (int64_t row = row_begin + static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5); row < total_rows;
         row += nwarps) {
        const int s = find_seg(seg_start, nseg, row);
        const qsync_adamw_seg sg = segs[s];
        const int64_t r = row - seg_start[s];
        const int64_t cols = sg.cols;
        float* p = sg.p + r * cols;
        const bool vec = (cols % 4 == 0) && ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(sg.g) |
                                              reinterpret_cast<uintptr_t>(sg.m) | reinterpret_cast<uintptr_t>(sg.v)) &
                                             15u) == 0;
        float amax = 0.0f;
        if (update) {
            const float* g = sg.g + r * cols;
            float* m = sg.m + r * cols;
            float* v = sg.v + r * cols;
            if (vec) {
                // Two float4 of each operand per lane in flight (8 x 16 B loads);
                // g / m / v are streamed (evict-first), p stays L2-resident for
                // the prepared-copy pass below.
                const int64_t n4 = cols / 4;
                const bool w16_now = sg.w16 && !sg.wq && ((reinterpret_cast<uintptr_t>(sg.w16 + r * cols) & 7u) == 0);
                float4* p4 = reinterpret_cast<float4*>(p);
                const float4* g4 = reinterpret_cast<const float4*>(g);
                float4* m4 = reinterpret_cast<float4*>(m);
                float4* v4 = reinterpret_cast<float4*>(v);
                for (int64_t k = lane; k < n4; k += 64) {
                    const bool two = k + 32 < n4;
                    float4 pv[2], gv[2], mv[2], vv[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        if (u == 1 && !two) break;
                        const int64_t kk = k + 32 * u;
                        pv[u] = p4[kk];
                        gv[u] = __ldcs(g4 + kk);
                        mv[u] = __ldcs(m4 + kk);
                        vv[u] = __ldcs(v4 + kk);
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        if (u == 1 && !two) break;
                        const int64_t kk = k + 32 * u;
                        pv[u].x = adam1(pv[u].x, gv[u].x, mv[u].x, vv[u].x, c);
                        pv[u].y = adam1(pv[u].y, gv[u].y, mv[u].y, vv[u].y, c);
                        pv[u].z = adam1(pv[u].z, gv[u].z, mv[u].z, vv[u].z, c);
                        pv[u].w = adam1(pv[u].w, gv[u].w, mv[u].w, vv[u].w, c);
                        p4[kk] = pv[u];
                        __stcs(m4 + kk, mv[u]);
                        __stcs(v4 + kk, vv[u]);
                        amax = fmaxf(amax, fmaxf(fmaxf(fabsf(pv[u].x), fabsf(pv[u].y)),
                                                 fmaxf(fabsf(pv[u].z), fabsf(pv[u].w))));
                        if (w16_now) {  // an FP16-only copy needs no row scale: write it now
                            uint2 h;
                            h.x = pack_half2(pv[u].x, pv[u].y);
                            h.y = pack_half2(pv[u].z, pv[u].w);
                            reinterpret_cast<uint2*>(sg.w16 + r * cols)[kk] = h;
                        }
                    }
                }
            } else {
                for (int64_t k = lane; k < cols; k += 32) {
                    float mm = m[k], vv = v[k];
                    const float pn = adam1(p[k], g[k], mm, vv, c);
                    p[k] = pn;
                    m[k] = mm;
                    v[k] = vv;
                    amax = fmaxf(amax, fabsf(pn));
                }
            }
        } else if (sg.wq) {
            for (int64_t k = lane; k < cols; k += 32) amax = fmaxf(amax, fabsf(p[k]));
        }
        if (!sg.w16 && !sg.wq) continue;
        if (update && vec && !sg.wq && (reinterpret_cast<uintptr_t>(sg.w16 + r * cols) & 7u) == 0) continue;
        __syncwarp();  // this warp's p stores are visible to its own re-reads
        amax = warp_max(amax);
        const float sc = scale_from_absmax(amax);
        if (sg.wq && lane == 0) sg.wscale[r] = sc;
        const QScale qsc = make_qscale(sc);
        uint16_t* w16 = sg.w16 ? sg.w16 + r * cols : nullptr;
        int8_t* wq = sg.wq ? sg.wq + r * cols : nullptr;
        const bool vec2 = vec && (!w16 || (reinterpret_cast<uintptr_t>(w16) & 7u) == 0) &&
                          (!wq || (reinterpret_cast<uintptr_t>(wq) & 3u) == 0);
        if (vec2) {
            for (int64_t k = lane; k < cols / 4; k += 32) {
                const float4 pv = reinterpret_cast<const float4*>(p)[k];
                if (w16) {
                    uint2 h;
                    h.x = pack_half2(pv.x, pv.y);
                    h.y = pack_half2(pv.z, pv.w);
                    reinterpret_cast<uint2*>(w16)[k] = h;
                }
                if (wq) {
                    reinterpret_cast<uint32_t*>(wq)[k] = pack_q4(quant_rne_f(pv.x, qsc), quant_rne_f(pv.y, qsc),
                                                                 quant_rne_f(pv.z, qsc), quant_rne_f(pv.w, qsc));
                }
            }
        } else {
            for (int64_t k = lane; k < cols; k += 32) {
                const float pv = p[k];
                if (w16) w16[k] = __half_as_ushort(__float2half_rn(pv));
                if (wq) wq[k] = static_cast<int8_t>(quant_rne(pv, qsc));
            }
        }
    }
}

__global__ void k_step_inc(int64_t* step) {
    QSB_PDL_ENTER(); *step += 1; }

}  // namespace
}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_adamw_step_range(const qsync_adamw_seg* segs, int nseg, const int64_t* seg_row_start,
                           int64_t row_begin, int64_t row_end, const int64_t* step, float lr, float beta1,
                           float beta2, float eps, float weight_decay, int update, qsync_stream_t stream) {
    QSB_REQUIRE(segs && seg_row_start && nseg > 0, QSYNC_ERR_VALIDATION, "segment table is required");
    QSB_REQUIRE(row_begin >= 0 && row_end >= row_begin, QSYNC_ERR_DOMAIN, "bad row range");
    QSB_REQUIRE(!update || step != nullptr, QSYNC_ERR_VALIDATION, "step counter is required");
    QSB_REQUIRE(!update || (beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f && eps > 0.f),
                QSYNC_ERR_DOMAIN, "AdamW needs 0 <= beta < 1 and eps > 0");
    if (row_end == row_begin) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    const int grid =
        static_cast<int>(std::min<int64_t>((row_end - row_begin + kWarps - 1) / kWarps, sm_count() * 16LL));
    const size_t smem = sizeof(int64_t) * (static_cast<size_t>(nseg) + 1);
    QSB_REQUIRE(smem <= 48 * 1024, QSYNC_ERR_DOMAIN, "too many parameter segments");
    // A plain launch, not PDL: the optimizer follows the join of the wgrad side
    // stream, and launched programmatically (its 4-wave grid becoming resident
    // behind the last backward kernels) it ran ~770 us in the graphed step
    // against ~570 us alone; plain, the step went 4.73 -> 4.53 ms (A/B of the
    // two library builds, tools/ab_step.py lib=...).
    k_adamw<<<grid, kWarps * 32, smem, st>>>(segs, nseg, seg_row_start, row_begin, row_end, step, lr, beta1, beta2,
                                              eps, weight_decay, update);
    return check_launch("k_adamw");
}

int qsync_adamw_advance(int64_t* step, qsync_stream_t stream) {
    QSB_REQUIRE(step != nullptr, QSYNC_ERR_VALIDATION, "step counter is required");
    pdl_launch(k_step_inc, dim3(1), dim3(1), 0, to_stream(stream), step);
    return check_launch("k_step_inc");
}

int qsync_adamw_step(const qsync_adamw_seg* segs, int nseg, const int64_t* seg_row_start,
                     int64_t total_rows, int64_t* step, float lr, float beta1, float beta2, float eps,
                     float weight_decay, int update, qsync_stream_t stream) {
    QSB_REQUIRE(total_rows >= 0, QSYNC_ERR_DOMAIN, "negative row count");
    QSB_TRY(qsync_adamw_step_range(segs, nseg, seg_row_start, 0, total_rows, step, lr, beta1, beta2, eps,
                                   weight_decay, update, stream));
    if (!update || total_rows == 0) return QSYNC_OK;
    return qsync_adamw_advance(step, stream);
}

}  // extern "C"

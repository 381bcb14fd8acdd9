// head.cu -- the BERT classification head around the planned encoder stack, so
// the graphed train step launches no framework kernels (train_step.py: the
// pooler and classifier are FP32 ops, plan["pooler"] = FP32):
//
//   pooled[b, j] = tanh(sum_h x[b, 0, h] Wp[j, h] + bp[j])          (pooler)
//   logits[b, c] = sum_h pooled[b, h] Wc[c, h] + bc[c]               (classifier)
//   loss = mean_b (logsumexp_c logits[b, :] - logits[b, label_b])    (cross entropy)
//
// and its backward (dloss a device scalar), accumulating into the FP32 weight
// gradients (main_grad):
//   dl[b, c]  = (softmax(logits)[b, c] - [c == label_b]) * dloss / B
//   dWc += dl^T pooled, dbc += sum_b dl
//   dpre[b, j] = (dl Wc)[b, j] * (1 - pooled[b, j]^2)
//   dWp += dpre^T x0,  dbp += sum_b dpre
//   dx[b, s, h] = s == 0 ? (dpre Wp)[b, h] : 0          (the whole [B, S, H] gradient)
//
// B x H x H = 32 x 768 x 768 multiply-adds per GEMM-like piece: latency, not
// throughput, bound -- SIMT FP32 with warp-shuffle / shared-memory reductions in
// a fixed order (deterministic), one launch per dependency level.  Also
// qsync_zero: the vectorized memset of the flat gradient buffer.
#include <algorithm>

#include "common.cuh"

namespace qsb {
namespace {

// 8 staged rows of H floats per block; the dynamic-smem attribute is set once
// to the largest (it is per kernel, a smaller value would cap later launches).
constexpr int kHeadMaxH = 4096;
constexpr int kHeadSmemMax = 8 * kHeadMaxH * 4;

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// pooled: block (blockIdx.x, blockIdx.y) = 8 columns j (one per warp) x 8
// sequences b, whose token-0 rows are staged in shared memory once per block
// (re-reading x0 from L2 per warp moved 75 MB for 98 KB of data).
__global__ void __launch_bounds__(256) k_head_pool(const float* __restrict__ x, int B, int64_t SH, int H,
                                                   const float* __restrict__ wp, const float* __restrict__ bp,
                                                   float* __restrict__ pooled) {
    QSB_PDL_ENTER();
    extern __shared__ float xs[];  // [8][H]
    const int b0 = blockIdx.y * 8;
    const int nb = min(8, B - b0);
    for (int i = threadIdx.x; i < nb * H; i += blockDim.x) xs[i] = x[(b0 + i / H) * SH + i % H];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (j >= H) return;
    const float* w = wp + static_cast<int64_t>(j) * H;
    float acc[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    for (int h = lane; h < H; h += 32) {
        const float wv = w[h];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(xs[i * H + h], wv, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float a = warp_sum_f(acc[i]);
        if (lane == 0 && i < nb) pooled[static_cast<int64_t>(b0 + i) * H + j] = tanhf(a + bp[j]);
    }
}

// logits, softmax and the mean cross entropy: one block.
__global__ void __launch_bounds__(1024) k_head_cls(const float* __restrict__ pooled, int B, int H,
                                                   const float* __restrict__ wc, const float* __restrict__ bc, int C,
                                                   const int64_t* __restrict__ labels, float* __restrict__ probs,
                                                   float* __restrict__ loss) {
    QSB_PDL_ENTER();
    extern __shared__ float sm[];  // [B * C] logits, then [B] per-row losses
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int task = warp; task < B * C; task += nw) {
        const int b = task / C, c = task % C;
        const float* pr = pooled + static_cast<int64_t>(b) * H;
        const float* w = wc + static_cast<int64_t>(c) * H;
        float acc = 0.0f;
        for (int h = lane; h < H; h += 32) acc = fmaf(pr[h], w[h], acc);
        acc = warp_sum_f(acc);
        if (lane == 0) sm[task] = acc + bc[c];
    }
    __syncthreads();
    float* rl = sm + B * C;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        const float* l = sm + b * C;
        float m = l[0];
        for (int c = 1; c < C; ++c) m = fmaxf(m, l[c]);
        float s = 0.0f;
        for (int c = 0; c < C; ++c) s += expf(l[c] - m);
        const float lse = m + logf(s);
        for (int c = 0; c < C; ++c) probs[b * C + c] = expf(l[c] - lse);
        const int64_t y = labels[b];
        rl[b] = lse - l[(y >= 0 && y < C) ? y : 0];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int b = 0; b < B; ++b) s += rl[b];  // fixed order: deterministic
        *loss = s / static_cast<float>(B);
    }
}

// dl (recomputed per block from probs), dWc / dbc, and dpre: thread per column h.
__global__ void __launch_bounds__(256) k_head_bwd1(const float* __restrict__ pooled, int B, int H,
                                                   const float* __restrict__ wc, int C,
                                                   const int64_t* __restrict__ labels,
                                                   const float* __restrict__ probs, const float* __restrict__ dloss,
                                                   float* __restrict__ dwc, float* __restrict__ dbc,
                                                   float* __restrict__ dpre) {
    QSB_PDL_ENTER();
    extern __shared__ float dl[];  // [B * C]
    const float g = *dloss / static_cast<float>(B);
    for (int i = threadIdx.x; i < B * C; i += blockDim.x) {
        const int b = i / C, c = i % C;
        dl[i] = (probs[i] - (labels[b] == c ? 1.0f : 0.0f)) * g;
    }
    __syncthreads();
    if (blockIdx.x == 0) {
        for (int c = threadIdx.x; c < C; c += blockDim.x) {
            float s = 0.0f;
            for (int b = 0; b < B; ++b) s += dl[b * C + c];
            dbc[c] += s;
        }
    }
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= H) return;
    for (int c = 0; c < C; ++c) {
        float s = 0.0f;
        for (int b = 0; b < B; ++b) s = fmaf(dl[b * C + c], pooled[static_cast<int64_t>(b) * H + h], s);
        dwc[static_cast<int64_t>(c) * H + h] += s;
    }
    for (int b = 0; b < B; ++b) {
        float s = 0.0f;
        for (int c = 0; c < C; ++c) s = fmaf(dl[b * C + c], wc[static_cast<int64_t>(c) * H + h], s);
        const float p = pooled[static_cast<int64_t>(b) * H + h];
        dpre[static_cast<int64_t>(b) * H + h] = s * (1.0f - p * p);
    }
}

// dWp[j, :] += sum_b dpre[b, j] x0[b, :], dbp[j] += sum_b dpre[b, j]: block per
// 8 rows j, so each x0 element is read once per 8 rows.
__global__ void __launch_bounds__(256) k_head_bwd_w(const float* __restrict__ x, int B, int64_t SH, int H,
                                                    const float* __restrict__ dpre, float* __restrict__ dwp,
                                                    float* __restrict__ dbp) {
    QSB_PDL_ENTER();
    extern __shared__ float col[];  // [B][8]
    const int j0 = blockIdx.x * 8;
    const int nj = min(8, H - j0);
    for (int i = threadIdx.x; i < B * 8; i += blockDim.x) {
        const int b = i / 8, jj = i % 8;
        col[i] = jj < nj ? dpre[static_cast<int64_t>(b) * H + j0 + jj] : 0.0f;
    }
    __syncthreads();
    if (threadIdx.x < nj) {
        float s = 0.0f;
        for (int b = 0; b < B; ++b) s += col[b * 8 + threadIdx.x];
        dbp[j0 + threadIdx.x] += s;
    }
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
        float acc[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 8
        for (int b = 0; b < B; ++b) {
            const float xv = x[b * SH + h];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) acc[jj] = fmaf(col[b * 8 + jj], xv, acc[jj]);
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
            if (jj < nj) dwp[static_cast<int64_t>(j0 + jj) * H + h] += acc[jj];
    }
}

// dx row 0 = dpre Wp ([B, H] x [H, H]) in two deterministic steps: k_head_dx_part
// splits the j range over blockIdx.z (kDxSplit parts) for parallelism -- block =
// 256 columns h x 8 sequences, the 8 dpre rows of its j range staged in shared
// memory, Wp rows read coalesced -- into part[split][b][h]; k_head_dx sums the
// parts in split order and writes all of dx (rows 1..S-1 zero).  One block per
// 8 sequences over the whole j range had left 12 blocks doing 768 serial loads.
constexpr int kDxSplit = 8;
__global__ void __launch_bounds__(256) k_head_dx_part(const float* __restrict__ dpre, int B, int H,
                                                      const float* __restrict__ wp, float* __restrict__ part) {
    QSB_PDL_ENTER();
    __shared__ float rows[8][128];  // dpre[b0 .. b0+7, j0 .. j0+127]
    const int b0 = blockIdx.y * 8;
    const int nb = min(8, B - b0);
    const int per = (H + kDxSplit - 1) / kDxSplit;
    const int ja = blockIdx.z * per, jb = min(H, ja + per);
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    float acc[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    for (int j0 = ja; j0 < jb; j0 += 128) {
        const int nj = min(128, jb - j0);
        __syncthreads();
        for (int i = threadIdx.x; i < 8 * 128; i += blockDim.x) {
            const int bi = i / 128, jj = i % 128;
            rows[bi][jj] = (bi < nb && jj < nj) ? dpre[static_cast<int64_t>(b0 + bi) * H + j0 + jj] : 0.0f;
        }
        __syncthreads();
        if (h < H) {
#pragma unroll 4
            for (int jj = 0; jj < nj; ++jj) {
                const float wv = wp[static_cast<int64_t>(j0 + jj) * H + h];
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] = fmaf(rows[i][jj], wv, acc[i]);
            }
        }
    }
    if (h >= H) return;
    for (int i = 0; i < nb; ++i) part[(static_cast<int64_t>(blockIdx.z) * B + b0 + i) * H + h] = acc[i];
}

__global__ void __launch_bounds__(256) k_head_dx(const float* __restrict__ part, int B, int S, int H,
                                                 float* __restrict__ dx) {
    QSB_PDL_ENTER();
    const int b = blockIdx.y;
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= H) return;
    float s = 0.0f;
#pragma unroll
    for (int k = 0; k < kDxSplit; ++k) s += part[(static_cast<int64_t>(k) * B + b) * H + h];
    float* out = dx + static_cast<int64_t>(b) * S * H + h;
    out[0] = s;
    for (int t = 1; t < S; ++t) out[static_cast<int64_t>(t) * H] = 0.0f;
}

// 16-byte stores over the aligned body, single bytes for the unaligned head
// (< 16 bytes before the first 16-byte boundary) and tail.
__global__ void k_zero16(uint8_t* __restrict__ p, int64_t head, int64_t n16, int64_t tail) {
    QSB_PDL_ENTER();
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    uint4* body = reinterpret_cast<uint4*>(p + head);
    for (int64_t i = tid; i < n16; i += static_cast<int64_t>(gridDim.x) * blockDim.x) __stcs(body + i, z);
    if (tid < head) p[tid] = 0;
    if (tid < tail) p[head + n16 * 16 + tid] = 0;
}

}  // namespace
}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_zero(void* p, int64_t bytes, qsync_stream_t stream) {
    QSB_REQUIRE(bytes >= 0, QSYNC_ERR_DOMAIN, "negative byte count");
    if (bytes == 0) return QSYNC_OK;
    QSB_REQUIRE(p != nullptr, QSYNC_ERR_VALIDATION, "qsync_zero needs a buffer");
    cudaStream_t st = to_stream(stream);
    const int64_t head = std::min<int64_t>(bytes, (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15);
    const int64_t n16 = (bytes - head) / 16;
    const int64_t tail = bytes - head - n16 * 16;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n16 + 255) / 256, int64_t(sm_count()) * 8)));
    return launch_pdl("k_zero16", k_zero16, dim3(grid), dim3(256), 0, st, static_cast<uint8_t*>(p), head, n16, tail);
}

int qsync_cls_head_fwd(const float* x, int64_t B, int64_t S, int64_t H, const float* wp, const float* bp,
                       const float* wc, const float* bc, int64_t C, const int64_t* labels, float* pooled,
                       float* probs, float* loss, qsync_stream_t stream) {
    QSB_REQUIRE(x && wp && bp && wc && bc && labels && pooled && probs && loss, QSYNC_ERR_VALIDATION,
                "classification head needs every buffer");
    QSB_REQUIRE(B > 0 && S > 0 && H > 0 && C > 0 && B * C <= 8192 && B <= 4096 && H <= kHeadMaxH,
                QSYNC_ERR_DOMAIN, "classification head extents out of range");
    cudaStream_t st = to_stream(stream);
    const int Bi = static_cast<int>(B), Hi = static_cast<int>(H), Ci = static_cast<int>(C);
    QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_head_pool), kHeadSmemMax));
    QSB_TRY(launch_pdl("k_head_pool", k_head_pool,
                       dim3(static_cast<unsigned>((H + 7) / 8), static_cast<unsigned>((B + 7) / 8)), dim3(256),
                       sizeof(float) * 8 * H, st, x, Bi, S * H, Hi, wp, bp, pooled));
    return launch_pdl("k_head_cls", k_head_cls, dim3(1), dim3(1024), sizeof(float) * (B * C + B), st,
                      static_cast<const float*>(pooled), Bi, Hi, wc, bc, Ci, labels, probs, loss);
}

int qsync_cls_head_bwd(const float* x, int64_t B, int64_t S, int64_t H, const float* wp, const float* wc, int64_t C,
                       const int64_t* labels, const float* pooled, const float* probs, const float* dloss,
                       float* dwp, float* dbp, float* dwc, float* dbc, float* dpre, float* dx,
                       qsync_stream_t stream) {
    QSB_REQUIRE(x && wp && wc && labels && pooled && probs && dloss && dwp && dbp && dwc && dbc && dpre && dx,
                QSYNC_ERR_VALIDATION, "classification head backward needs every buffer");
    QSB_REQUIRE(B > 0 && S > 0 && H > 0 && C > 0 && B * C <= 8192 && B <= 4096 && H <= kHeadMaxH, QSYNC_ERR_DOMAIN,
                "classification head extents out of range");
    cudaStream_t st = to_stream(stream);
    const int Bi = static_cast<int>(B), Hi = static_cast<int>(H), Ci = static_cast<int>(C);
    QSB_TRY(launch_pdl("k_head_bwd1", k_head_bwd1, dim3(static_cast<unsigned>((H + 255) / 256)), dim3(256),
                       sizeof(float) * B * C, st, pooled, Bi, Hi, wc, Ci, labels, probs, dloss, dwc, dbc, dpre));
    QSB_TRY(launch_pdl("k_head_bwd_w", k_head_bwd_w, dim3(static_cast<unsigned>((H + 7) / 8)), dim3(256),
                       sizeof(float) * B * 8, st, x, Bi, S * H, Hi, static_cast<const float*>(dpre), dwp, dbp));
    float* part = dpre + B * H;  // the scratch holds dpre [B, H] then the split partials [kDxSplit, B, H]
    QSB_TRY(launch_pdl("k_head_dx_part", k_head_dx_part,
                       dim3(static_cast<unsigned>((H + 255) / 256), static_cast<unsigned>((B + 7) / 8), kDxSplit),
                       dim3(256), 0, st, static_cast<const float*>(dpre), Bi, Hi, wp, part));
    return launch_pdl("k_head_dx", k_head_dx, dim3(static_cast<unsigned>((H + 255) / 256), static_cast<unsigned>(B)),
                      dim3(256), 0, st, static_cast<const float*>(part), Bi, static_cast<int>(S), Hi, dx);
}

}  // extern "C"

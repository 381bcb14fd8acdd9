// conv.cu -- K8 Conv2d as GEMM (NHWC; PAPER.md:607 -- below-16-bit convolutions
// require channels-last): im2col gather into the K-major GEMM operand and the
// deterministic col2im gather for dgrad.
//
//   A[(n,p,q), (r,s,c)] = x[n, p*sh - ph + r*dh, q*sw - pw + s*dw, c]   (0 outside)
//   K = R*S*C, padded with zeros to the row pitch `ld` (16 B multiple for TMA).
//   dx[n,h,w,c] = sum over (r,s) with h = p*sh - ph + r*dh (p integral, in range)
//                 and w likewise of dcol[(n,p,q), (r,s,c)]    -- no atomics.
//
// Forward of an INT8 conv = quantize x once (1 B/elem), im2col of the int8 NHWC
// tensor, tcgen05 kind::i8 GEMM with the fused dequant epilogue (output NHWC FP32).
#include <algorithm>

#include "common.cuh"

namespace qsb {
namespace {

struct ConvGeom {
    int64_t N, H, W, C, P, Q;
    int R, S, sh, sw, ph, pw, dh, dw;
    int64_t ld;  // row pitch of the column matrix (>= R*S*C)
};

// One thread per 16-byte chunk of the column matrix (C a multiple of the
// vector width, fewer than 2^31 chunks): consecutive threads write consecutive
// chunks, so every store is a full coalesced line whatever the row length.  The
// warp-per-row kernel below leaves lanes idle when a row is not a multiple of
// 32 chunks (C = 64 INT8 3x3: 36 chunks per row, 1.2 TB/s).
template <typename T>
__global__ void __launch_bounds__(256) k_im2col_chunks(const T* __restrict__ x, ConvGeom g,
                                                       T* __restrict__ out, int items) {
    constexpr int V = 16 / sizeof(T);
    const int C = static_cast<int>(g.C), CV = C / V;
    const int K = g.R * g.S * C;
    const int nch = static_cast<int>(g.ld / V);
    const int P = static_cast<int>(g.P), Q = static_cast<int>(g.Q);
    const int H = static_cast<int>(g.H), W = static_cast<int>(g.W);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < items; i += gridDim.x * blockDim.x) {
        const int row = i / nch;
        const int j = i - row * nch;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (j * V < K) {
            const int tap = j / CV;
            const int c = (j - tap * CV) * V;
            const int r = tap / g.S, ss = tap - r * g.S;
            const int q = row % Q, t = row / Q;
            const int p = t % P, n = t / P;
            const int h = p * g.sh - g.ph + r * g.dh, w = q * g.sw - g.pw + ss * g.dw;
            if (h >= 0 && h < H && w >= 0 && w < W)
                v = *reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + h) * W + w) * C + c);
        }
        *reinterpret_cast<uint4*>(out + static_cast<int64_t>(row) * g.ld + static_cast<int64_t>(j) * V) = v;
    }
}

// One warp per column row (n,p,q): the row's coordinates are decoded once, the
// lanes stride over its 16-byte chunks (tap = chunk / (C/V), 32-bit math).
// Scalar fallback (C not a multiple of the vector width) keeps one element per lane.
template <typename T>
__global__ void __launch_bounds__(256) k_im2col(const T* __restrict__ x, ConvGeom g,
                                                T* __restrict__ out, int vec) {
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte chunk
    const int lane = threadIdx.x & 31;
    const int K = g.R * g.S * static_cast<int>(g.C);
    const int C = static_cast<int>(g.C);
    const int rows = static_cast<int>(g.N * g.P * g.Q);
    const int P = static_cast<int>(g.P), Q = static_cast<int>(g.Q);
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows; row += warps) {
        const int q = row % Q;
        const int p = (row / Q) % P;
        const int n = row / (Q * P);
        const int h0 = p * g.sh - g.ph, w0 = q * g.sw - g.pw;
        const T* xn = x + static_cast<int64_t>(n) * g.H * g.W * C;
        T* orow = out + static_cast<int64_t>(row) * g.ld;
        if (vec == 1) {
            const int CV = C / V;
            const int nch = static_cast<int>(g.ld / V);
            for (int j = lane; j < nch; j += 32) {
                uint4 v = make_uint4(0, 0, 0, 0);
                if (j * V < K) {
                    const int tap = j / CV;
                    const int c = (j - tap * CV) * V;
                    const int r = tap / g.S, ss = tap - r * g.S;
                    const int h = h0 + r * g.dh, w = w0 + ss * g.dw;
                    if (h >= 0 && h < g.H && w >= 0 && w < g.W)
                        v = *reinterpret_cast<const uint4*>(xn + (static_cast<int64_t>(h) * g.W + w) * C + c);
                }
                *reinterpret_cast<uint4*>(orow + j * V) = v;
            }
        } else if (vec == 2) {
            // Narrow C (the stem's C = 3): each lane assembles a 16-byte chunk of
            // the row, stepping (c, s, r) incrementally instead of dividing per element.
            const int nch = static_cast<int>(g.ld / V);
            for (int j = lane; j < nch; j += 32) {
                const int k0 = j * V;
                int tap = k0 / C;
                int c = k0 - tap * C;
                int r = tap / g.S, ss = tap - r * g.S;
                union {
                    uint4 u;
                    T e[V];
                } v;
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    T val = T(0);
                    const int h = h0 + r * g.dh, w = w0 + ss * g.dw;
                    if (k0 + e < K && h >= 0 && h < g.H && w >= 0 && w < g.W)
                        val = xn[(static_cast<int64_t>(h) * g.W + w) * C + c];
                    v.e[e] = val;
                    if (++c == C) {
                        c = 0;
                        if (++ss == g.S) {
                            ss = 0;
                            ++r;
                        }
                    }
                }
                *reinterpret_cast<uint4*>(orow + j * V) = v.u;
            }
        } else {
            for (int k = lane; k < g.ld; k += 32) {
                T v = T(0);
                if (k < K) {
                    const int tap = k / C;
                    const int c = k - tap * C;
                    const int r = tap / g.S, ss = tap - r * g.S;
                    const int h = h0 + r * g.dh, w = w0 + ss * g.dw;
                    if (h >= 0 && h < g.H && w >= 0 && w < g.W) v = xn[(static_cast<int64_t>(h) * g.W + w) * C + c];
                }
                orow[k] = v;
            }
        }
    }
}

template <int DT>
__device__ __forceinline__ float ldf(const void* p, int64_t i) {
    return Elem<DT>::f(static_cast<const typename Elem<DT>::T*>(p)[i]);
}

// dx[n,h,w,c] (FP32) = sum of the column entries that gathered x[n,h,w,c]: one
// warp per input pixel (the (r,s) tap validity is warp-uniform), lanes over
// channel groups of 4 (16-byte FP32 column loads, one float4 store).
template <int DT>
__global__ void __launch_bounds__(256) k_col2im(const void* __restrict__ dcol, ConvGeom g,
                                                float* __restrict__ dx, int vec) {
    const int lane = threadIdx.x & 31;
    const int C = static_cast<int>(g.C);
    const int pixels = static_cast<int>(g.N * g.H * g.W);
    const int H = static_cast<int>(g.H), W = static_cast<int>(g.W);
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int pix = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); pix < pixels; pix += warps) {
        const int w = pix % W;
        const int h = (pix / W) % H;
        const int n = pix / (W * H);
        float* out = dx + static_cast<int64_t>(pix) * C;
        const int groups = vec ? C / 4 : C;
        for (int cg = lane; cg < groups; cg += 32) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            // With dilation 1 only every sh-th (sw-th) tap can land on this
            // pixel: start at the first such tap and step by the stride.
            const int r0 = g.dh == 1 ? (h + g.ph) % g.sh : 0, rstep = g.dh == 1 ? g.sh : 1;
            const int s0 = g.dw == 1 ? (w + g.pw) % g.sw : 0, sstep = g.dw == 1 ? g.sw : 1;
            for (int r = r0; r < g.R; r += rstep) {
                const int hp = h + g.ph - r * g.dh;
                if (hp < 0) break;
                if (hp % g.sh) continue;
                const int p = hp / g.sh;
                if (p >= g.P) continue;
                for (int s = s0; s < g.S; s += sstep) {
                    const int wq = w + g.pw - s * g.dw;
                    if (wq < 0) break;
                    if (wq % g.sw) continue;
                    const int q = wq / g.sw;
                    if (q >= g.Q) continue;
                    const int64_t row = (static_cast<int64_t>(n) * g.P + p) * g.Q + q;
                    const int64_t base = row * g.ld + static_cast<int64_t>(r * g.S + s) * C;
                    if (vec) {
                        if (DT == QSYNC_F32) {
                            const float4 v = *reinterpret_cast<const float4*>(static_cast<const float*>(dcol) + base + 4 * cg);
                            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                        } else {
                            const uint2 u = *reinterpret_cast<const uint2*>(static_cast<const __half*>(dcol) + base + 4 * cg);
                            const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
                            const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
                            acc.x += a.x; acc.y += a.y; acc.z += b.x; acc.w += b.y;
                        }
                    } else {
                        acc.x += ldf<DT>(dcol, base + cg);
                    }
                }
            }
            if (vec)
                *reinterpret_cast<float4*>(out + 4 * cg) = acc;
            else
                out[cg] = acc.x;
        }
    }
}

// Scalar col2im for channel counts that are not a vector multiple (ResNet
// conv1, C = 3): one thread per element, 32-bit index math, so narrow pixels
// do not leave most of a warp idle.
template <int DT>
__global__ void __launch_bounds__(256) k_col2im_s(const void* __restrict__ dcol, ConvGeom g, float* __restrict__ dx) {
    const int C = static_cast<int>(g.C);
    const int H = static_cast<int>(g.H), W = static_cast<int>(g.W);
    const int total = static_cast<int>(g.N * g.H * g.W * g.C);  // < 2^31 (checked by the caller)
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int pix = idx / C;
        const int c = idx - pix * C;
        const int w = pix % W, h = (pix / W) % H, n = pix / (W * H);
        float acc = 0.f;
        const int r0 = g.dh == 1 ? (h + g.ph) % g.sh : 0, rstep = g.dh == 1 ? g.sh : 1;
        const int s0 = g.dw == 1 ? (w + g.pw) % g.sw : 0, sstep = g.dw == 1 ? g.sw : 1;
        for (int r = r0; r < g.R; r += rstep) {
            const int hp = h + g.ph - r * g.dh;
            if (hp < 0) break;
            if (hp % g.sh) continue;
            const int p = hp / g.sh;
            if (p >= g.P) continue;
            for (int s = s0; s < g.S; s += sstep) {
                const int wq = w + g.pw - s * g.dw;
                if (wq < 0) break;
                if (wq % g.sw) continue;
                const int q = wq / g.sw;
                if (q >= g.Q) continue;
                const int64_t row = (static_cast<int64_t>(n) * g.P + p) * g.Q + q;
                acc += ldf<DT>(dcol, row * g.ld + static_cast<int64_t>(r * g.S + s) * C + c);
            }
        }
        dx[idx] = acc;
    }
}

int make_geom(ConvGeom& g, int64_t N, int64_t H, int64_t W, int64_t C, int R, int S, int sh,
              int sw, int ph, int pw, int dh, int dw, int64_t ld) {
    QSB_REQUIRE(N >= 0 && H > 0 && W > 0 && C > 0 && R > 0 && S > 0, QSYNC_ERR_DOMAIN,
                "conv extents must be positive");
    QSB_REQUIRE(sh > 0 && sw > 0 && dh > 0 && dw > 0 && ph >= 0 && pw >= 0, QSYNC_ERR_DOMAIN,
                "conv stride/dilation must be > 0 and padding >= 0");
    g.N = N; g.H = H; g.W = W; g.C = C; g.R = R; g.S = S;
    g.sh = sh; g.sw = sw; g.ph = ph; g.pw = pw; g.dh = dh; g.dw = dw;
    g.P = (H + 2 * ph - dh * (R - 1) - 1) / sh + 1;
    g.Q = (W + 2 * pw - dw * (S - 1) - 1) / sw + 1;
    QSB_REQUIRE(g.P > 0 && g.Q > 0, QSYNC_ERR_DOMAIN, "conv output would be empty");
    const int64_t K = static_cast<int64_t>(R) * S * C;
    g.ld = ld > 0 ? ld : K;
    QSB_REQUIRE(g.ld >= K, QSYNC_ERR_DOMAIN, "column pitch must be >= R*S*C");
    return QSYNC_OK;
}

// Narrow C (the stem's C = 3): one THREAD per 16-byte chunk of the column matrix
// (a warp per row would leave 22 of 32 lanes idle on a 160-byte row); the chunk's
// elements step (c, s, r) incrementally, no division per element.
template <typename T>
__global__ void __launch_bounds__(256) k_im2col_narrow(const T* __restrict__ x, ConvGeom g,
                                                       T* __restrict__ out) {
    constexpr int V = 16 / sizeof(T);
    const int C = static_cast<int>(g.C);
    const int K = g.R * g.S * C;
    const int nch = static_cast<int>(g.ld / V);
    const int P = static_cast<int>(g.P), Q = static_cast<int>(g.Q);
    const int64_t items = g.N * g.P * g.Q * nch;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < items;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int row = static_cast<int>(i / nch);
        const int j = static_cast<int>(i - static_cast<int64_t>(row) * nch);
        const int q = row % Q, p = (row / Q) % P, n = row / (Q * P);
        const int h0 = p * g.sh - g.ph, w0 = q * g.sw - g.pw;
        const T* xn = x + static_cast<int64_t>(n) * g.H * g.W * C;
        const int k0 = j * V;
        int tap = k0 / C;
        int c = k0 - tap * C;
        int r = tap / g.S, ss = tap - r * g.S;
        union {
            uint4 u;
            T e[V];
        } v;
#pragma unroll
        for (int e = 0; e < V; ++e) {
            T val = T(0);
            const int h = h0 + r * g.dh, w = w0 + ss * g.dw;
            if (k0 + e < K && h >= 0 && h < g.H && w >= 0 && w < g.W)
                val = xn[(static_cast<int64_t>(h) * g.W + w) * C + c];
            v.e[e] = val;
            if (++c == C) {
                c = 0;
                if (++ss == g.S) {
                    ss = 0;
                    ++r;
                }
            }
        }
        *reinterpret_cast<uint4*>(out + static_cast<int64_t>(row) * g.ld + k0) = v.u;
    }
}

int grid_of(int64_t warps_of_work) {  // blocks of 8 warps
    const int64_t cap = static_cast<int64_t>(sm_count()) * 16;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((warps_of_work + 7) / 8, cap)));
}

}  // namespace
}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_conv_out_size(int64_t H, int64_t W, int R, int S, int sh, int sw, int ph, int pw, int dh,
                        int dw, int64_t* P, int64_t* Q) {
    ConvGeom g;
    QSB_TRY(make_geom(g, 1, H, W, 1, R, S, sh, sw, ph, pw, dh, dw, 0));
    *P = g.P;
    *Q = g.Q;
    return QSYNC_OK;
}

int qsync_im2col(const void* x, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R, int S,
                 int sh, int sw, int ph, int pw, int dh, int dw, void* out, int64_t ld,
                 qsync_stream_t stream) {
    ConvGeom g;
    QSB_TRY(make_geom(g, N, H, W, C, R, S, sh, sw, ph, pw, dh, dw, ld));
    if (N == 0) return QSYNC_OK;
    QSB_REQUIRE(g.N * g.P * g.Q < (int64_t(1) << 31), QSYNC_ERR_DOMAIN, "conv too large");
    cudaStream_t st = to_stream(stream);
    const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    if (dtype == QSYNC_I8) {
        const int vec = (C % 16 == 0) && (g.ld % 16 == 0) && al(x) && al(out) ? 1
                        : (g.ld % 16 == 0 && al(out))                          ? 2
                                                                               : 0;
        const int64_t work = g.N * g.P * g.Q;
        const int64_t chunks = work * (g.ld / 16);
        if (vec == 1 && chunks < (int64_t(1) << 31))
            k_im2col_chunks<int8_t><<<grid_of(chunks / 32 + 1), 256, 0, st>>>(
                static_cast<const int8_t*>(x), g, static_cast<int8_t*>(out), static_cast<int>(chunks));
        else if (vec == 2)
            k_im2col_narrow<int8_t><<<grid_of(work * (g.ld / 16) / 32 + 1), 256, 0, st>>>(
                static_cast<const int8_t*>(x), g, static_cast<int8_t*>(out));
        else
            k_im2col<int8_t><<<grid_of(work), 256, 0, st>>>(static_cast<const int8_t*>(x), g,
                                                             static_cast<int8_t*>(out), vec);
    } else if (dtype == QSYNC_F16 || dtype == QSYNC_BF16) {
        const int vec = (C % 8 == 0) && (g.ld % 8 == 0) && al(x) && al(out) ? 1
                        : (g.ld % 8 == 0 && al(out))                         ? 2
                                                                             : 0;
        const int64_t work = g.N * g.P * g.Q;
        const int64_t chunks = work * (g.ld / 8);
        if (vec == 1 && chunks < (int64_t(1) << 31))
            k_im2col_chunks<uint16_t><<<grid_of(chunks / 32 + 1), 256, 0, st>>>(
                static_cast<const uint16_t*>(x), g, static_cast<uint16_t*>(out), static_cast<int>(chunks));
        else if (vec == 2)
            k_im2col_narrow<uint16_t><<<grid_of(work * (g.ld / 8) / 32 + 1), 256, 0, st>>>(
                static_cast<const uint16_t*>(x), g, static_cast<uint16_t*>(out));
        else
            k_im2col<uint16_t><<<grid_of(work), 256, 0, st>>>(static_cast<const uint16_t*>(x), g,
                                                               static_cast<uint16_t*>(out), vec);
    } else {
        return set_error(QSYNC_ERR_DOMAIN, "im2col supports I8, F16 and BF16 inputs");
    }
    return check_launch("k_im2col");
}

int qsync_col2im(const void* dcol, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R,
                 int S, int sh, int sw, int ph, int pw, int dh, int dw, int64_t ld, float* dx,
                 qsync_stream_t stream) {
    ConvGeom g;
    QSB_TRY(make_geom(g, N, H, W, C, R, S, sh, sw, ph, pw, dh, dw, ld));
    if (N == 0) return QSYNC_OK;
    cudaStream_t st = to_stream(stream);
    QSB_REQUIRE(N * H * W * C < (int64_t(1) << 31) && g.N * g.P * g.Q < (int64_t(1) << 31), QSYNC_ERR_DOMAIN,
                "conv too large");
    const int grid = grid_of(N * H * W);
    const int vec = (C % 4 == 0) && (g.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(dcol) & 15u) == 0) &&
                    ((reinterpret_cast<uintptr_t>(dx) & 15u) == 0);
    const int grid_s = grid_of(N * H * W * C / 32 + 1);
    switch (dtype) {
        case QSYNC_F32:
            if (vec) k_col2im<QSYNC_F32><<<grid, 256, 0, st>>>(dcol, g, dx, vec);
            else k_col2im_s<QSYNC_F32><<<grid_s, 256, 0, st>>>(dcol, g, dx);
            break;
        case QSYNC_F16:
            if (vec) k_col2im<QSYNC_F16><<<grid, 256, 0, st>>>(dcol, g, dx, vec);
            else k_col2im_s<QSYNC_F16><<<grid_s, 256, 0, st>>>(dcol, g, dx);
            break;
        default: return set_error(QSYNC_ERR_DOMAIN, "col2im supports F32 and F16 columns");
    }
    return check_launch("k_col2im");
}

}  // extern "C"

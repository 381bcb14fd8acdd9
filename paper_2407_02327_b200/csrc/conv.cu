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

// One thread per 16-byte (or element, on the scalar path) chunk of a column row.
// Rows are (n,p,q); within a row the (r,s) taps are C-contiguous runs.
template <typename T>
__global__ void __launch_bounds__(256) k_im2col(const T* __restrict__ x, ConvGeom g,
                                                T* __restrict__ out, int vec) {
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte chunk
    const int64_t K = static_cast<int64_t>(g.R) * g.S * g.C;
    const int64_t chunks_per_row = vec ? g.ld / V : g.ld;
    const int64_t total = g.N * g.P * g.Q * chunks_per_row;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = idx / chunks_per_row;
        const int64_t ch = idx - row * chunks_per_row;
        const int64_t q = row % g.Q;
        const int64_t p = (row / g.Q) % g.P;
        const int64_t n = row / (g.Q * g.P);
        if (vec) {
            const int64_t k0 = ch * V;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (k0 < K) {
                const int64_t tap = k0 / g.C;
                const int64_t c = k0 - tap * g.C;
                const int r = static_cast<int>(tap / g.S), s = static_cast<int>(tap % g.S);
                const int64_t h = p * g.sh - g.ph + r * g.dh;
                const int64_t w = q * g.sw - g.pw + s * g.dw;
                if (h >= 0 && h < g.H && w >= 0 && w < g.W)
                    v = *reinterpret_cast<const uint4*>(x + ((n * g.H + h) * g.W + w) * g.C + c);
            }
            *reinterpret_cast<uint4*>(out + row * g.ld + k0) = v;
        } else {
            const int64_t k = ch;
            T v = T(0);
            if (k < K) {
                const int64_t tap = k / g.C;
                const int64_t c = k - tap * g.C;
                const int r = static_cast<int>(tap / g.S), s = static_cast<int>(tap % g.S);
                const int64_t h = p * g.sh - g.ph + r * g.dh;
                const int64_t w = q * g.sw - g.pw + s * g.dw;
                if (h >= 0 && h < g.H && w >= 0 && w < g.W) v = x[((n * g.H + h) * g.W + w) * g.C + c];
            }
            out[row * g.ld + k] = v;
        }
    }
}

template <int DT>
__device__ __forceinline__ float ldf(const void* p, int64_t i) {
    return Elem<DT>::f(static_cast<const typename Elem<DT>::T*>(p)[i]);
}

// dx[n,h,w,c] (FP32) = sum of the column entries that gathered x[n,h,w,c].
template <int DT>
__global__ void __launch_bounds__(256) k_col2im(const void* __restrict__ dcol, ConvGeom g,
                                                float* __restrict__ dx) {
    const int64_t total = g.N * g.H * g.W * g.C;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = idx % g.C;
        const int64_t w = (idx / g.C) % g.W;
        const int64_t h = (idx / (g.C * g.W)) % g.H;
        const int64_t n = idx / (g.C * g.W * g.H);
        float acc = 0.0f;
        for (int r = 0; r < g.R; ++r) {
            const int64_t hp = h + g.ph - r * g.dh;
            if (hp < 0 || hp % g.sh) continue;
            const int64_t p = hp / g.sh;
            if (p >= g.P) continue;
            for (int s = 0; s < g.S; ++s) {
                const int64_t wq = w + g.pw - s * g.dw;
                if (wq < 0 || wq % g.sw) continue;
                const int64_t q = wq / g.sw;
                if (q >= g.Q) continue;
                const int64_t row = (n * g.P + p) * g.Q + q;
                acc += ldf<DT>(dcol, row * g.ld + (static_cast<int64_t>(r) * g.S + s) * g.C + c);
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

int grid_of(int64_t work) {
    const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, cap)));
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
    cudaStream_t st = to_stream(stream);
    const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    if (dtype == QSYNC_I8) {
        const int vec = (C % 16 == 0) && (g.ld % 16 == 0) && al(x) && al(out);
        const int64_t work = g.N * g.P * g.Q * (vec ? g.ld / 16 : g.ld);
        k_im2col<int8_t><<<grid_of(work), 256, 0, st>>>(static_cast<const int8_t*>(x), g,
                                                         static_cast<int8_t*>(out), vec);
    } else if (dtype == QSYNC_F16 || dtype == QSYNC_BF16) {
        const int vec = (C % 8 == 0) && (g.ld % 8 == 0) && al(x) && al(out);
        const int64_t work = g.N * g.P * g.Q * (vec ? g.ld / 8 : g.ld);
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
    const int grid = grid_of(N * H * W * C);
    switch (dtype) {
        case QSYNC_F32: k_col2im<QSYNC_F32><<<grid, 256, 0, st>>>(dcol, g, dx); break;
        case QSYNC_F16: k_col2im<QSYNC_F16><<<grid, 256, 0, st>>>(dcol, g, dx); break;
        default: return set_error(QSYNC_ERR_DOMAIN, "col2im supports F32 and F16 columns");
    }
    return check_launch("k_col2im");
}

}  // extern "C"

// sr.cu -- K9: stochastic rounding on the reference's RNG stream.
//
// The reference rounds element i with draw i of a fresh std::mt19937_64(seed)
// (indicator.cpp:179-187; uniform01 = (draw >> 11) * 2^-53, rng.hpp:12-14).
// mt19937_64 is a linear recurrence over GF(2); the device reproduces the
// stream exactly:
//   * one CTA owns one contiguous segment of draws and advances a 312-word
//     state held in shared memory by parallel twists (3 dependency phases:
//     words [0,156) read only old words; [156,311) read new words i-156;
//     word 311 reads new words 0 and 155);
//   * segment start states come from GF(2) jump-ahead (mt_jump.cpp): the
//     state at draw offset J is sum_i p_i * window_i(raw stream of the seed)
//     with p(x) = x^J mod phi(x), phi the 19937-degree characteristic
//     polynomial.  The raw stream prefix and the XOR-accumulation run on the
//     device (k_mt_jump), the seed-independent polynomials on the host.
// SR arithmetic is FP64 exactly as indicator.cpp:180-189.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "mt_jump.hpp"

namespace qsb {

namespace {

constexpr int MT_N = 312;
constexpr int MT_M = 156;
constexpr uint64_t UPPER = 0xFFFFFFFF80000000ULL;
constexpr uint64_t LOWER = 0x000000007FFFFFFFULL;
constexpr uint64_t MATA = 0xB5026F5AA96619E9ULL;
constexpr int kSrThreads = 320;  // 312 state words, 10 warps
// The jump-ahead of a segment is split into kJumpParts partial sums (k_mt_jump).
constexpr int kJumpParts = 8;
constexpr int kJumpChunk = (mtjump::kPolyWords + kJumpParts - 1) / kJumpParts;  // poly words per part

__device__ __forceinline__ uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

__device__ __forceinline__ uint64_t twist_word(uint64_t cur, uint64_t next, uint64_t far) {
    const uint64_t y = (cur & UPPER) | (next & LOWER);
    return far ^ (y >> 1) ^ ((y & 1ULL) ? MATA : 0ULL);
}

// In-place twist of st[0..312) by threads 0..311 (all threads must call).
__device__ __forceinline__ void twist(uint64_t* st) {
    const int i = threadIdx.x;
    uint64_t v = 0;
    if (i < MT_M) v = twist_word(st[i], st[i + 1], st[i + MT_M]);
    __syncthreads();
    if (i < MT_M) st[i] = v;
    __syncthreads();
    if (i >= MT_M && i < MT_N) v = twist_word(st[i], st[(i + 1) % MT_N], st[i - MT_M]);
    __syncthreads();
    if (i >= MT_M && i < MT_N) st[i] = v;
    __syncthreads();
}

__device__ __forceinline__ double u01(uint64_t draw) {
    return static_cast<double>(draw >> 11) * 0x1.0p-53;
}

enum SrMode { kSrF64 = 0, kSrI8 = 1, kSrDraws = 2 };

struct SrArgs {
    const double* x64;
    const float* x32;
    int64_t n;
    double q;
    double zp;
    const float* scale_dev;
    int64_t* rounded;
    double* deq;
    int8_t* q8;
    uint64_t* draws;
    // segment layout: CTA b handles draws [b*seg_len, min(n, (b+1)*seg_len)) of
    // the stream shifted by `offset`; its start state (the 312 words of the twist
    // block containing draw offset + b*seg_len) is states[b*312 ..).
    int64_t seg_len;
    uint64_t offset;
    const uint64_t* states;
};

// One CTA per segment.  states[b] is the state whose next twist produces the
// twist block containing draw (offset + b*seg_len).
template <int MODE>
__global__ void __launch_bounds__(kSrThreads) k_sr(const SrArgs a) {
    __shared__ uint64_t st[MT_N];
    const int i = threadIdx.x;
    const int64_t first = static_cast<int64_t>(blockIdx.x) * a.seg_len;
    const int64_t last = min(a.n, first + a.seg_len);
    if (first >= last) return;
    if (i < MT_N) {
        uint64_t v = 0;
        for (int y = 0; y < kJumpParts; ++y)
            v ^= a.states[(static_cast<int64_t>(y) * gridDim.x + blockIdx.x) * MT_N + i];
        st[i] = v;
    }
    double q = a.q;
    if (MODE == kSrI8) q = static_cast<double>(*a.scale_dev);
    // Absolute draw index of element e is offset + e; its twist block is
    // (offset+e)/312 and position (offset+e)%312.
    const uint64_t abs_first = a.offset + static_cast<uint64_t>(first);
    int64_t block_base = static_cast<int64_t>(abs_first / MT_N) * MT_N;  // absolute
    // The next block's input is loaded before this block's twist, so the HBM
    // latency overlaps the twist and the FP64 work (one block per iteration).
    const auto fetch = [&](int64_t base) -> double {
        const int64_t e = base + i - static_cast<int64_t>(a.offset);
        if (MODE == kSrDraws || i >= MT_N || e < first || e >= last) return 0.0;
        return MODE == kSrF64 ? a.x64[e] : static_cast<double>(a.x32[e]);
    };
    double xnext = fetch(block_base);
    __syncthreads();
    while (true) {
        const double xcur = xnext;
        xnext = fetch(block_base + MT_N);
        twist(st);
        const int64_t e = block_base + i - static_cast<int64_t>(a.offset);  // element index
        if (i < MT_N && e >= first && e < last) {
            const uint64_t d = temper(st[i]);
            if (MODE == kSrDraws) {
                a.draws[e] = d;
            } else if (MODE == kSrF64) {
                const double xbar = __ddiv_rn(__dsub_rn(xcur, a.zp), q);
                const double lo = floor(xbar);
                const double frac = __dsub_rn(xbar, lo);
                const int64_t r = static_cast<int64_t>(lo) + (u01(d) < frac ? 1 : 0);
                if (a.rounded) a.rounded[e] = r;
                if (a.deq) a.deq[e] = __dadd_rn(__dmul_rn(q, static_cast<double>(r)), a.zp);
            } else {
                const double xbar = __ddiv_rn(xcur, q);
                const double lo = floor(xbar);
                const double frac = __dsub_rn(xbar, lo);
                int64_t r = static_cast<int64_t>(lo) + (u01(d) < frac ? 1 : 0);
                r = r > 127 ? 127 : (r < -127 ? -127 : r);
                a.q8[e] = static_cast<int8_t>(r);
            }
        }
        block_base += MT_N;
        if (block_base - static_cast<int64_t>(a.offset) >= last) break;
    }
}

// Device jump-ahead: out state (312 words) for each segment b = sum over the
// set bits i of poly_b of raw_window_i, where raw_window_i = raw[i .. i+312)
// is the word window of the seed's raw recurrence sequence (raw[0..312) = the
// seeded state, raw[312+t] = t-th generated word).  Grid (segment, part): part y
// covers poly words [y*kJumpChunk, (y+1)*kJumpChunk) and writes its partial sum
// to out[(y*nseg + b)*312 ..); k_sr XORs the parts.  The raw words that chunk
// touches sit in shared memory, and the set bits are consumed four at a time
// (independent loads into four accumulators) -- the loop was L2-latency bound
// at one dependent load per bit.
__global__ void __launch_bounds__(kSrThreads) k_mt_jump(const uint64_t* __restrict__ raw,
                                                        const uint64_t* __restrict__ polys,
                                                        int poly_words, uint64_t* __restrict__ out) {
    __shared__ uint64_t sraw[kJumpChunk * 64 + MT_N];
    __shared__ uint64_t spoly[kJumpChunk];
    const int i = threadIdx.x;
    const int w0 = blockIdx.y * kJumpChunk;
    const int w1 = min(poly_words, w0 + kJumpChunk);
    const uint64_t* poly = polys + static_cast<int64_t>(blockIdx.x) * poly_words;
    const int nraw = max(0, (w1 - w0) * 64 + MT_N);
    for (int j = i; j < nraw; j += blockDim.x) {
        const int64_t g = static_cast<int64_t>(w0) * 64 + j;
        sraw[j] = g < mtjump::kRawWords ? raw[g] : 0ull;
    }
    for (int j = i; j < w1 - w0; j += blockDim.x) spoly[j] = poly[w0 + j];
    __syncthreads();
    if (i >= MT_N) return;
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int w = 0; w < w1 - w0; ++w) {
        uint64_t bits = spoly[w];  // uniform across the CTA
        const uint64_t* base = sraw + w * 64 + i;
#if QSB_JUMP_SETBITS
        while (__popcll(bits) >= 4) {
            const int b0 = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            const int b1 = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            const int b2 = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            const int b3 = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            a0 ^= base[b0];
            a1 ^= base[b1];
            a2 ^= base[b2];
            a3 ^= base[b3];
        }
        while (bits) {
            const int b = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            a0 ^= base[b];
        }
#else
        // all 64 positions unrolled: constant smem offsets, predicated loads
        // (the predicate is uniform across the CTA), no bit-scan per set bit
        const uint32_t lo = static_cast<uint32_t>(bits), hi = static_cast<uint32_t>(bits >> 32);
#pragma unroll
        for (int b = 0; b < 32; b += 4) {
            if (lo & (1u << b)) a0 ^= base[b];
            if (lo & (2u << b)) a1 ^= base[b + 1];
            if (lo & (4u << b)) a2 ^= base[b + 2];
            if (lo & (8u << b)) a3 ^= base[b + 3];
        }
#pragma unroll
        for (int b = 0; b < 32; b += 4) {
            if (hi & (1u << b)) a0 ^= base[32 + b];
            if (hi & (2u << b)) a1 ^= base[33 + b];
            if (hi & (4u << b)) a2 ^= base[34 + b];
            if (hi & (8u << b)) a3 ^= base[35 + b];
        }
#endif
    }
    out[(static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * MT_N + i] = a0 ^ a1 ^ a2 ^ a3;
}

// Raw recurrence sequence of a seed: raw[0..312) = seeded state, then words
// generated by the twists, total `len` words.  Single CTA.
__global__ void __launch_bounds__(kSrThreads) k_mt_raw(uint64_t seed, int64_t len,
                                                       uint64_t* __restrict__ raw) {
    __shared__ uint64_t st[MT_N];
    const int i = threadIdx.x;
    if (i == 0) {
        st[0] = seed;
        for (int k = 1; k < MT_N; ++k)
            st[k] = 6364136223846793005ULL * (st[k - 1] ^ (st[k - 1] >> 62)) + static_cast<uint64_t>(k);
    }
    __syncthreads();
    if (i < MT_N && i < len) raw[i] = st[i];
    for (int64_t base = MT_N; base < len; base += MT_N) {
        twist(st);
        if (i < MT_N && base + i < len) raw[base + i] = st[i];
    }
}

// Host orchestration.  Each SR call: (1) raw prefix of the seed (k_mt_raw),
// (2) segment start states by jump-ahead (k_mt_jump), (3) the SR pass.  The
// start state of segment b must be the state just BEFORE the twist that
// produces the block containing absolute draw offset + b*seg_len, i.e. the
// state after T_b = floor((offset + b*seg_len)/312) twists; that is the raw
// window starting at word 312*T_b.  We jump the raw sequence by J_b = 312*T_b
// words: p_b = x^{J_b} mod phi.
struct Workspace {
    uint64_t* raw = nullptr;
    uint64_t* polys = nullptr;
    uint64_t* states = nullptr;
    size_t cap_segments = 0;
};

Workspace& workspace_for(cudaStream_t st);

int run_sr(int mode, SrArgs a, uint64_t seed, cudaStream_t st) {
    if (a.n == 0) return QSYNC_OK;
    // The jump polynomials come from the host per call: not capturable.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    QSB_TRY(cuda_status(cudaStreamIsCapturing(st, &cap), "cudaStreamIsCapturing"));
    QSB_REQUIRE(cap == cudaStreamCaptureStatusNone, QSYNC_ERR_VALIDATION,
                "stochastic rounding on the reference RNG stream cannot be captured in a CUDA graph "
                "(its jump-ahead polynomials are computed on the host per call)");
    Workspace& ws = workspace_for(st);
    const int sms = sm_count();
    // Segment length: a whole number of twist blocks; enough segments to fill
    // the chip, but not shorter than the cost of a jump (~20K words).
    int64_t seg_blocks = std::max<int64_t>(64, (a.n / MT_N + 2 * sms - 1) / (2 * sms));
    seg_blocks = mtjump::round_segment_blocks(seg_blocks);
    const int64_t seg_len = seg_blocks * MT_N;
    const int64_t nseg = (a.n + seg_len - 1) / seg_len;
    a.seg_len = seg_len;
    // Twist counts at each segment start.
    std::vector<uint64_t> twists(nseg);
    for (int64_t b = 0; b < nseg; ++b) twists[b] = (a.offset + static_cast<uint64_t>(b * seg_len)) / MT_N;
    const std::vector<uint64_t>& polys = mtjump::jump_polys(twists);  // nseg x kPolyWords
    const int pw = mtjump::kPolyWords;
    if (ws.cap_segments < static_cast<size_t>(nseg)) {
        // Stream-ordered growth: the old buffers are released after the work
        // already queued on this stream (no hidden device synchronisation).
        if (ws.raw) QSB_TRY(cuda_status(cudaFreeAsync(ws.raw, st), "cudaFreeAsync"));
        if (ws.polys) QSB_TRY(cuda_status(cudaFreeAsync(ws.polys, st), "cudaFreeAsync"));
        if (ws.states) QSB_TRY(cuda_status(cudaFreeAsync(ws.states, st), "cudaFreeAsync"));
        ws.raw = ws.polys = ws.states = nullptr;
        ws.cap_segments = 0;
        QSB_TRY(cuda_status(cudaMallocAsync(reinterpret_cast<void**>(&ws.raw), sizeof(uint64_t) * mtjump::kRawWords, st),
                            "cudaMallocAsync"));
        QSB_TRY(cuda_status(cudaMallocAsync(reinterpret_cast<void**>(&ws.polys), sizeof(uint64_t) * pw * nseg, st),
                            "cudaMallocAsync"));
        QSB_TRY(cuda_status(cudaMallocAsync(reinterpret_cast<void**>(&ws.states), sizeof(uint64_t) * MT_N * nseg * kJumpParts, st),
                            "cudaMallocAsync"));
        ws.cap_segments = nseg;
    }
    // Pageable source: the copy is staged before cudaMemcpyAsync returns, so the
    // cache-owned host buffer may change afterwards.
    QSB_TRY(cuda_status(cudaMemcpyAsync(ws.polys, polys.data(), sizeof(uint64_t) * pw * nseg,
                                        cudaMemcpyHostToDevice, st),
                        "copy jump polynomials"));
    k_mt_raw<<<1, kSrThreads, 0, st>>>(seed, mtjump::kRawWords, ws.raw);
    QSB_TRY(check_launch("k_mt_raw"));
    k_mt_jump<<<dim3(static_cast<unsigned>(nseg), kJumpParts), kSrThreads, 0, st>>>(ws.raw, ws.polys, pw, ws.states);
    QSB_TRY(check_launch("k_mt_jump"));
    a.states = ws.states;
    switch (mode) {
        case kSrF64: k_sr<kSrF64><<<static_cast<unsigned>(nseg), kSrThreads, 0, st>>>(a); break;
        case kSrI8: k_sr<kSrI8><<<static_cast<unsigned>(nseg), kSrThreads, 0, st>>>(a); break;
        default: k_sr<kSrDraws><<<static_cast<unsigned>(nseg), kSrThreads, 0, st>>>(a); break;
    }
    QSB_TRY(check_launch("k_sr"));
    return QSYNC_OK;
}

// Library-owned jump-ahead scratch, one per (device, stream): work on one
// stream is ordered, so its workspace is reused safely; two streams (or the
// same stream handle on another device) never share one.  The SR entries are
// the only ones that keep per-device state.
Workspace& workspace_for(cudaStream_t st) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, Workspace> table;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    return table[{dev, st}];
}

}  // namespace
}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_stochastic_round_f64(const double* x, int64_t n, double q, double zp, uint64_t seed,
                               int64_t* rounded, double* dequantized, qsync_stream_t stream) {
    // indicator.cpp:178 -- same domain check and message.
    QSB_REQUIRE(q > 0, QSYNC_ERR_DOMAIN, "stochastic rounding needs a scaling factor > 0");
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    SrArgs a{};
    a.x64 = x;
    a.n = n;
    a.q = q;
    a.zp = zp;
    a.rounded = rounded;
    a.deq = dequantized;
    return run_sr(kSrF64, a, seed, to_stream(stream));
}

int qsync_stochastic_round_float_f64(const double* x, int64_t n, int e, int k, uint64_t seed,
                                     double* out, qsync_stream_t stream) {
    // indicator.cpp:197.
    QSB_REQUIRE(k >= 1, QSYNC_ERR_DOMAIN, "mantissa bit count must be at least 1");
    const double spacing = std::exp2(static_cast<double>(e - k));
    return qsync_stochastic_round_f64(x, n, spacing, 0.0, seed, nullptr, out, stream);
}

int qsync_quantize_sr(const float* x, int64_t n, const float* scale, uint64_t seed, int8_t* q,
                      qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    SrArgs a{};
    a.x32 = x;
    a.n = n;
    a.scale_dev = scale;
    a.q8 = q;
    return run_sr(kSrI8, a, seed, to_stream(stream));
}

int qsync_mt64_draws(uint64_t seed, uint64_t offset, int64_t n, uint64_t* out,
                     qsync_stream_t stream) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "negative element count");
    SrArgs a{};
    a.n = n;
    a.draws = out;
    a.offset = offset;
    return run_sr(kSrDraws, a, seed, to_stream(stream));
}

}  // extern "C"

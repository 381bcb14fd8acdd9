// gemm.cu -- K6 INT8 and K7 FP16/BF16 GEMMs on the 5th-generation tensor cores.
//
//   C[m,n] = sum_k A[m,k] * B[n,k]      (A [M,K], B [N,K], both K-contiguous)
//
// Persistent, warp-specialised tcgen05 kernel:
//   warp 0      TMA producer: A/B tiles -> 128B-swizzled smem ring (mbarrier
//               full/empty handshake, expect_tx byte counts)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (kind::i8 -> int32 accumulators, kind::f16 -> FP32), commits
//               free smem stages and publish finished accumulators
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers, fused dequant /
//               rescale / bias / accumulate, stores to global
// The accumulator is double-buffered in TMEM (2 x BN columns) so the epilogue
// of tile i overlaps the MMAs of tile i+1.
//
// INT8 epilogue semantics (pinned, bit-exact vs oracle/cpu_ref.c
// ref_dequant_epilogue): y = __fmul_rn(float(acc), __fmul_rn(s_a, s_b[n]))
// then __fadd_rn(y, bias[n]) -- the INT8 kernel emits FP32 (graph.hpp:38-40),
// layer-wise activation x channel-wise weight scales (PAPER.md:426-427,
// PAPER.md:588-592).
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>

#include "common.cuh"
#include "ptx.cuh"

namespace qsb {

namespace {

constexpr int BM = 128;             // UMMA M (cta_group::1)
constexpr int BK_BYTES = 128;       // one 128B swizzle row per stage
constexpr int kEpiWarp0 = 2;
constexpr int kEpiWarps = 8;        // two per TMEM lane quadrant
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);  // producer, MMA, 8 epilogue warps

struct EpiParams {
    int64_t M, N, K;
    int32_t* c_i32;
    void* c;
    int c_dtype;
    const float* scale_a;
    const float* scale_b;
    int b_per_channel;
    const float* bias;
    float alpha;
    const float* alpha_dev;
    int accumulate;
    uint32_t idesc;
    int tma_store;  // epilogue writes through tm_c (TMA store / reduce-add)
    int debug_epi;  // bench hook: 1 = skip epilogue math+stores (TMEM read only)
    int ksplit;     // split-K factor (>1 only with accumulate: partials reduce-add)
    int kb_per;     // k-blocks per split
    // Stream-K (streamk = 1): the tiles x k-blocks iteration space is cut into
    // one contiguous range per CTA.  A CTA's first unit may start inside a tile
    // (a "contributor": its raw accumulators go to sk_ws slot blockIdx.x and it
    // bumps sk_flags[tile]); a unit that starts a tile but ends inside it (the
    // "owner") waits for that tile's contributors, adds their partials in CTA
    // order and runs the epilogue; the owner resets the flag.  Accumulating
    // outputs need no fixup: every unit reduce-adds, bias from the k = 0 unit.
    int streamk;
    uint32_t* sk_ws;   // [gridDim.x][BN / 4][BM][4] raw 32-bit accumulators
    int* sk_flags;     // [tiles], zero between launches
    // Implicit-GEMM convolution (kLay bit 2): A[(n,p,q), (r,s,c)] is gathered from
    // the NHWC input on the fly -- never materialised.
    int fp8;            // byte operands are FP8 E4M3 (host side; the kernel sees kLay bit 7)
    // kLay bit 3: B (MN-major) is gathered instead -- the conv wgrad, whose
    // B[(n,p,q), (r,s,c)] is the same column matrix read K-rows = pixels.
    // The dgrad runs as a kLay-bit-2 gather over dY with ctap = -1 (h_in =
    // h + ph - r) and cdv = the forward stride (taps with h_in % stride != 0
    // are zero), its B = W [Cout][R*S][C] read by a 3-D TMA map (kLay bit 4).
    const uint8_t* cx;  // NHWC input (elements of the GEMM operand type)
    int cN, cH, cW, cC, cP, cQ, cR, cS, csh, csw, cph, cpw;
    int ctap, cdvh, cdvw;
    // kLay bit 9: GELU epilogue (an encoder layer's FF1 with the activation that
    // follows it): c = g = gelu(y), dact = FP16(gelu'(y)) through tm_d, and
    // act_absmax = max |g| (float bits, atomicMax; the caller zeroes it).
    uint16_t* dact;
    unsigned* act_absmax;
    // kLay bit 12: also reduce ymax = max(0, max y) over the stored outputs
    // (float bits, atomicMax; zeroed by the host) -- FF1's input to the
    // one-pass GELU quantizer (qsync_gelu_quantize).
    unsigned* ymax;
    // kLay bits 5 / 6: the same operands loaded by TMA in im2col mode instead
    // (A for fwd / stride-1 dgrad -- the dgrad as a conv of dY with pad k-1-p and
    // flipped taps; B for wgrad); one elected thread, no gather lanes.
};

constexpr int kStageChunkBytes = 32 * 128;  // one warp's 32 rows x 128 B staging chunk

// kCta = 1: one CTA computes a 128 x BN tile.  kCta = 2: a CTA pair (cluster of
// 2, cta_group::2) computes a 256 x BN tile; each CTA holds its 128 A rows and
// half (BN/2 rows) of B, and the leader issues 2-SM MMAs reading both halves.
template <int BN, int kCta = 1>
struct Cfg {
    static constexpr int kBRows = BN / kCta;  // B rows held by one CTA
    static constexpr int kStageBytes = (BM + kBRows) * BK_BYTES;
#ifndef QSB_GEMM_STAGES_48K
#define QSB_GEMM_STAGES_48K 4
#endif
    static constexpr int kStagesWant =
        kStageBytes >= 48 * 1024 ? QSB_GEMM_STAGES_48K : (kStageBytes >= 32 * 1024 ? 6 : 8);
    // Staging chunks per epilogue warp: two (the TMA store of one overlaps the
    // next chunk's math) unless that costs a mainloop stage (BN = 256, 1 CTA).
    static constexpr int kEpiBufs = (BN / kCta) >= 256 ? 1 : 2;
    static constexpr int kEpiStageBytes = kEpiWarps * kEpiBufs * kStageChunkBytes;
    // per-column epilogue factors of the current tile: scale (s_a * s_b[n]) + bias
    static constexpr int kFacBytes = 2 * BN * 4;
    // mbarriers (full/empty per stage, 2 tfull + 2 tempty) + the TMEM address slot
    static constexpr int kBarBytes = ((2 * kStagesWant + 4) * 8 + 4 + 15) / 16 * 16;
    // ... as many stages as fit next to the epilogue staging in 227 KB (the
    // dynamic smem base is 1024-aligned, __align__ below; checked at entry)
    static constexpr int kStagesFit = (227 * 1024 - kEpiStageBytes - kFacBytes - kBarBytes) / kStageBytes;
    static constexpr int kStages = kStagesWant < kStagesFit ? kStagesWant : kStagesFit;
    // two accumulator buffers; TMEM allocations are powers of two (BN = 192 -> 512)
    static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
    static constexpr int kSmemBytes = kStages * kStageBytes + kEpiStageBytes + kFacBytes + kBarBytes;
};

// Phase timeline of every CTA (tools/gemm_trace.py; A/B builds only:
// tools/build_variant.sh <lib> -DQSB_GEMM_TRACE).  Slot layout per CTA:
// [0] globaltimer at entry, [1] clock at entry, [2] clock after the prologue
// (griddepcontrol.wait), [3] clock at exit, [4] globaltimer at exit; then per unit u < 8 at 8 + 8u:
// [0] producer's first load issued, [1] MMA: accumulator free, [2] MMA: first
// stage full, [3] MMA: last commit issued, [4] epilogue: accumulator full,
// [5] epilogue: last store issued.
#ifdef QSB_GEMM_TRACE
__device__ unsigned long long* g_gemm_trace = nullptr;
__device__ __forceinline__ unsigned long long trace_clock() {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    return c;
}
#define QSB_TRACE(slot, val)                                                               \
    do {                                                                                   \
        if (g_gemm_trace) g_gemm_trace[static_cast<size_t>(blockIdx.x) * 72 + (slot)] = (val); \
    } while (0)
#define QSB_TRACE_U(u, ev)                                                      \
    do {                                                                        \
        const int _k = ((u) - unit0) / unit_stride;                             \
        if (_k < 8) QSB_TRACE(8 + 8 * _k + (ev), trace_clock());                \
    } while (0)
#else
#define QSB_TRACE(slot, val) \
    do {                     \
    } while (0)
#define QSB_TRACE_U(u, ev) \
    do {                   \
    } while (0)
#endif

__device__ __forceinline__ float bits_f(uint32_t v) { return __uint_as_float(v); }

// Work unit i of a CTA: tile t, k-blocks [kb0, kb1), and its stream-K role
// (0 plain / split-K part / accumulating, 1 contributor, 2 owner).  The
// classic schedule strides units u = cta + i * ncta over tiles x ksplit.
enum { kUnitPlain = 0, kUnitContrib = 1, kUnitOwner = 2 };
template <bool kSK>
__device__ __forceinline__ bool unit_at(const EpiParams& p, int i, int cta, int ncta, int num_tiles, int ksplit,
                                        int num_kb, int& t, int& kb0, int& kb1, int& role) {
    if (!kSK || !p.streamk) {
        const int u = cta + i * ncta;
        if (u >= num_tiles * ksplit) return false;
        t = u / ksplit;
        kb0 = (u % ksplit) * p.kb_per;
        kb1 = ksplit > 1 ? min(num_kb, kb0 + p.kb_per) : num_kb;
        role = kUnitPlain;
        return true;
    } else {
    const int64_t total = static_cast<int64_t>(num_tiles) * num_kb;
    int64_t pos = total * cta / ncta;
    const int64_t end = total * (cta + 1) / ncta;
    for (int j = 0;; ++j) {
        if (pos >= end) return false;
        const int64_t tt = pos / num_kb;
        const int k0 = static_cast<int>(pos - tt * num_kb);
        const int k1 = static_cast<int>(min(static_cast<int64_t>(num_kb), end - tt * num_kb));
        if (j == i) {
            t = static_cast<int>(tt);
            kb0 = k0;
            kb1 = k1;
            role = p.accumulate ? kUnitPlain : (k0 > 0 ? kUnitContrib : (k1 < num_kb ? kUnitOwner : kUnitPlain));
            return true;
        }
        pos = tt * num_kb + k1;
    }
    }
}

// kLay bit 0: A is MN-major (stored [K, M]); bit 1: B is MN-major ([K, N]).
// MN-major tiles are loaded as 64-element-wide (128 B) blocks of bk K-rows.
template <bool kI8, int BN, int kCta, int kLay>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
              const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_d,
              const EpiParams p) {
    using C = Cfg<BN, kCta>;
    constexpr int kBRows = C::kBRows;
    constexpr int kStages = C::kStages;
    // kLay bit 7: FP8 E4M3 byte operands (kind::f8f6f4, FP32 accumulators).  A
    // template bit, not a runtime flag: a per-MMA / per-element branch on it cost
    // the INT8 GEMM 20% (8192^3: 3.07 -> 2.43 POPS).
    constexpr bool kF8 = (kLay & 128) != 0;
    // kLay bit 8: TF32 operands (4-byte elements, kind::tf32, FP32 accumulators),
    // K-major only -- the FP32 plan's 3xTF32 GEMM (qsync_gemm_f32).
    constexpr bool kTF32 = (kLay & 256) != 0;
    static_assert(!kTF32 || (!kI8 && (kLay & 255) == 0), "TF32 is a K-major FP-kind layout");
    constexpr bool kGelu = (kLay & 512) != 0;
    // kLay bit 10: stream-K schedule (EpiParams::streamk; 256-wide single-CTA tiles)
    constexpr bool kSK = (kLay & 1024) != 0;
    // kLay bit 11: two MMA issuers on ONE work unit per CTA, alternate k-blocks
    // into the two accumulator buffers, summed by the epilogue.  One issuing
    // thread cannot keep the tensor pipe busy below N = 256 (>= ~116 cycles
    // per tcgen05.mma); two can (trace build, isolation mode 18: 2x the MMAs
    // of a 192-wide tile in 1.63x the time, 128-wide in 1.2x).
    constexpr bool kDual = (kLay & 2048) != 0;
    constexpr bool kYmax = (kLay & 4096) != 0;
    static_assert(!kYmax || (kI8 && kCta == 1 && (kLay & 0xfff) == 0), "ymax: INT8 K-major single-CTA");
    static_assert(!kDual || (kCta == 1 && (kLay & 0x7fc) == 0), "dual issue: plain single-CTA tiles");
    static_assert(!kSK || (kCta == 1 && BN == 256 && (kLay & 0x3fc) == 0), "stream-K: plain 256-wide single-CTA");
    static_assert(!kGelu || (kCta == 1 && (kLay & 511) == 0), "GELU epilogue: single-CTA K-major tiles");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for the 128B swizzle atoms: the declaration asks for
    // it and the smem budget (Cfg::kSmemBytes) assumes it -- trap, not corrupt.
    if (ptx::smem_u32(smem_raw) & 1023) __trap();
    uint8_t* smem = smem_raw;
    uint8_t* smem_a = smem;                              // kStages x [BM rows x 128B]
    uint8_t* smem_b = smem + kStages * BM * BK_BYTES;    // kStages x [kBRows rows x 128B]
    uint8_t* smem_stage = smem + kStages * C::kStageBytes;  // 1024-aligned epilogue staging
    float* fac = reinterpret_cast<float*>(smem_stage + C::kEpiStageBytes);  // [2][BN]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_stage + C::kEpiStageBytes + C::kFacBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = bars + 2 * kStages + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
#ifdef QSB_GEMM_TRACE
    if (threadIdx.x == 0) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        QSB_TRACE(0, gt);
        QSB_TRACE(1, trace_clock());
    }
#endif

    const int64_t M = p.M, N = p.N, K = p.K;
    constexpr int kTileM = BM * kCta;  // rows of one (pair) tile
    const int num_m = static_cast<int>((M + kTileM - 1) / kTileM);
    // CTA pairs share one work sequence; rank 0 of a pair leads the MMAs.
    const uint32_t rank = kCta == 2 ? ptx::cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const int unit0 = blockIdx.x / kCta;
    const int unit_stride = gridDim.x / kCta;
    const int num_n = static_cast<int>((N + BN - 1) / BN);
    const int num_tiles = num_m * num_n;
    // Work units = (tile, K split); split-K partials are reduce-added by TMA.
    const int ksplit = p.ksplit > 1 ? p.ksplit : 1;
    const int bk_elems = kI8 ? BK_BYTES : (kTF32 ? BK_BYTES / 4 : BK_BYTES / 2);
    const int num_kb = static_cast<int>((K + bk_elems - 1) / bk_elems);

    if (warp == 0 && lane == 0) {
        if (!(kLay & 4)) ptx::tma_prefetch(&tm_a);
        if (!(kLay & 8)) ptx::tma_prefetch(&tm_b);
        if (p.tma_store) ptx::tma_prefetch(&tm_c);
        if (kGelu) ptx::tma_prefetch(&tm_d);
        for (int s = 0; s < kStages; ++s) {
            // implicit conv: + one cp.async completion arrival per producer lane
            ptx::mbar_init(&full[s], (kLay & 12) ? 33 : 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], (kDual && a == 0) ? 2 : 1);  // dual: both issuers commit
            ptx::mbar_init(&tempty[a], kCta * kEpiWarps * 32);  // epilogue threads of both CTAs
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        if (kCta == 2)
            ptx::tmem_alloc_pair<C::kTmemCols>(tmem_slot);
        else
            ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    }
    ptx::tc_fence_before();
    if (kCta == 2)
        ptx::cluster_sync();  // peer barriers initialised before any remote arrive
    else
        __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // Programmatic dependent launch: everything above (barrier init, TMEM
    // allocation, descriptor prefetch) may overlap the previous kernel's tail;
    // no global memory is touched before the previous grid has completed.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef QSB_GEMM_TRACE
    if (threadIdx.x == 0) QSB_TRACE(2, trace_clock());
#endif
    // Leader-CTA addresses of the barriers the pair shares.
    const uint32_t full_leader0 = kCta == 2 ? ptx::mapa(ptx::smem_u32(&full[0]), 0) : 0u;
    const uint32_t tempty_leader0 = kCta == 2 ? ptx::mapa(ptx::smem_u32(&tempty[0]), 0) : 0u;

    // kDual: issuer `parity` takes the k-blocks kb0 + parity, kb0 + parity + 2, ...
    // of the CTA's single unit into accumulator buffer `parity`, frees each
    // stage it consumed and commits once to tfull[0] (count 2).
    auto dual_issue = [&](int parity) {
        int t, kb0, kb1, role;
        if (!unit_at<kSK>(p, 0, unit0, unit_stride, num_tiles, ksplit, num_kb, t, kb0, kb1, role)) return;
        const uint32_t d = tmem_base + static_cast<uint32_t>(parity * BN);
        for (int kb = kb0 + parity; kb < kb1; kb += 2) {
            const int j = kb - kb0;
            const int stage = j % kStages;
            ptx::mbar_wait(&full[stage], static_cast<uint32_t>((j / kStages) & 1));
            ptx::tc_fence_after();
            const uint32_t a_addr = ptx::smem_u32(smem_a + stage * BM * BK_BYTES);
            const uint32_t b_addr = ptx::smem_u32(smem_b + stage * kBRows * BK_BYTES);
#pragma unroll
            for (int k = 0; k < BK_BYTES / 32; ++k) {
                const uint64_t da = (kLay & 1) ? ptx::sw128_mnmajor_desc(a_addr + k * 16 * 128, bk_elems * 128)
                                               : ptx::sw128_kmajor_desc(a_addr + k * 32);
                const uint64_t db = (kLay & 2) ? ptx::sw128_mnmajor_desc(b_addr + k * 16 * 128, bk_elems * 128)
                                               : ptx::sw128_kmajor_desc(b_addr + k * 32);
                const uint32_t accum = (kb != kb0 + parity || k != 0) ? 1u : 0u;
                if (kI8)
                    ptx::mma_i8(d, da, db, p.idesc, accum);
                else
                    ptx::mma_f16(d, da, db, p.idesc, accum);
            }
            ptx::tc_commit(&empty[stage]);
        }
        ptx::tc_commit(&tfull[0]);
    };

    if (warp == 0 && (kLay & 12)) {
        // ============ implicit-GEMM conv producer (all 32 lanes) ============
        // kLay & 4 (fwd / dgrad): A tile row m = output pixel (n,p,q); its
        // 128-byte K-slice kb is one (r,s) tap's contiguous channel run
        // x[n, p*sh-ph+r, q*sw-pw+s, c0:c0+bk] (C*elem % 128 == 0), copied by
        // eight 16-byte cp.async into the 128B-swizzled K-major layout the UMMA
        // descriptor reads; padding taps and rows past M are zero-filled
        // (src-size 0).  Lane l owns rows l, l+32, l+64, l+96; lane 0 also
        // TMA-loads the weight tile (B).
        // kLay & 8 (wgrad): B is MN-major -- per 64-column block j (one tap's
        // 64-channel run) the stage holds bk K-rows = pixels of 128 B, the same
        // swizzle; lane l owns K-rows l, l+32; lane 0 TMA-loads dY (A, MN-major).
        int stage = 0;
        uint32_t phase = 0;
        const int eb = kI8 ? 1 : 2;
        const int rowbytes = p.cC * eb;
        const int64_t img = static_cast<int64_t>(p.cH) * p.cW * rowbytes;
        for (int ui = 0;; ++ui) {
            int t, kb0, kb1, role;
            if (!unit_at<kSK>(p, ui, unit0, unit_stride, num_tiles, ksplit, num_kb, t, kb0, kb1, role)) break;
            const int m0 = (t % num_m) * kTileM;
            const int n0 = (t / num_m) * BN;
            int hb[4], wb[4];
            const uint8_t* pix[4];
            bool rok[4];
            if (kLay & 4) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int m = m0 + lane + 32 * i;
                    rok[i] = m < M;
                    const int mm = rok[i] ? m : 0;
                    const int q = mm % p.cQ, pp = (mm / p.cQ) % p.cP, n = mm / (p.cQ * p.cP);
                    hb[i] = pp * p.csh - p.cph;
                    wb[i] = q * p.csw - p.cpw;
                    pix[i] = p.cx + static_cast<int64_t>(n) * img;
                }
            }
            for (int kb = kb0; kb < kb1; ++kb) {
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sa = smem_a + stage * BM * BK_BYTES;
                uint8_t* sb = smem_b + stage * kBRows * BK_BYTES;
                if (lane == 0) {
                    if (kLay & 4) {
                        ptx::mbar_arrive_expect_tx(&full[stage], kBRows * BK_BYTES);
                        if (kLay & 16) {  // W [Cout][R*S][C]: K index = (rs, k) with k < cC
                            const int kk = kb * bk_elems;
                            for (int j = 0; j < kBRows / 64; ++j)
                                ptx::tma_load_3d(sb + j * bk_elems * 128, &tm_b, &full[stage], n0 + 64 * j,
                                                 kk % p.cC, kk / p.cC);
                        } else if (kLay & 2) {
                            for (int j = 0; j < kBRows / 64; ++j)
                                ptx::tma_load_2d(sb + j * bk_elems * 128, &tm_b, &full[stage], n0 + 64 * j,
                                                 kb * bk_elems);
                        } else {
                            ptx::tma_load_2d(sb, &tm_b, &full[stage], kb * bk_elems, n0);
                        }
                    } else {
                        ptx::mbar_arrive_expect_tx(&full[stage], BM * BK_BYTES);
                        for (int j = 0; j < BM / 64; ++j)
                            ptx::tma_load_2d(sa + j * bk_elems * 128, &tm_a, &full[stage], m0 + 64 * j,
                                             kb * bk_elems);
                    }
                }
                if (kLay & 4) {
                    // A 64-byte channel run (INT8 C = 64) fills half a K-slice: the slice
                    // then holds two taps, four 16-byte chunks each (taps past R*S and
                    // rows past M are zero-filled).
                    const int halves = (rowbytes & (BK_BYTES - 1)) ? 2 : 1;
                    const uint32_t sbase = ptx::smem_u32(sa);
                    for (int hf = 0; hf < halves; ++hf) {
                    const int kbyte = kb * BK_BYTES + hf * 64;  // byte offset along K = (tap, c)
                    const int tap = kbyte / rowbytes;
                    const int cbyte = kbyte - tap * rowbytes;
                    const int r = tap / p.cS, sx = tap - r * p.cS;
                    const bool tap_ok = tap < p.cR * p.cS;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int row = lane + 32 * i;
                        int h = hb[i] + p.ctap * r, w = wb[i] + p.ctap * sx;
                        bool ok = rok[i] && tap_ok;
                        if (p.cdvh > 1) {  // dgrad of a strided conv: only taps on the stride grid
                            ok = ok && h >= 0 && h % p.cdvh == 0;
                            h /= p.cdvh;
                        }
                        if (p.cdvw > 1) {
                            ok = ok && w >= 0 && w % p.cdvw == 0;
                            w /= p.cdvw;
                        }
                        ok = ok && h >= 0 && h < p.cH && w >= 0 && w < p.cW;
                        const uint8_t* src =
                            ok ? pix[i] + (static_cast<int64_t>(h) * p.cW + w) * rowbytes + cbyte : p.cx;
                        const uint32_t nbytes = ok ? 16u : 0u;
                        if (halves == 1) {
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                ptx::cp_async16_zfill(sbase + row * 128 + ((j ^ (row & 7)) << 4), src + 16 * j,
                                                      nbytes);
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                ptx::cp_async16_zfill(sbase + row * 128 + (((hf * 4 + j) ^ (row & 7)) << 4),
                                                      src + 16 * j, nbytes);
                        }
                    }
                    }
                } else {
                    constexpr int kRows = kI8 ? 4 : 2;  // K-rows (pixels) per lane per stage
                    int kh[kRows], kw[kRows];
                    const uint8_t* kpix[kRows];
                    bool kok[kRows];
#pragma unroll
                    for (int i = 0; i < kRows; ++i) {
                        const int64_t m = static_cast<int64_t>(kb) * bk_elems + lane + 32 * i;
                        kok[i] = m < K;
                        const int mm = kok[i] ? static_cast<int>(m) : 0;
                        const int q = mm % p.cQ, pp = (mm / p.cQ) % p.cP, n = mm / (p.cQ * p.cP);
                        kh[i] = pp * p.csh - p.cph;
                        kw[i] = q * p.csw - p.cpw;
                        kpix[i] = p.cx + static_cast<int64_t>(n) * img;
                    }
#pragma unroll 1
                    for (int j = 0; j < kBRows / 64; ++j) {
                        const int col = n0 + 64 * j;  // first (r,s,c) column of this block
                        const int kbyte = col * eb;
                        const int tap = kbyte / rowbytes;
                        const int cbyte = kbyte - tap * rowbytes;
                        const int r = tap / p.cS, sx = tap - r * p.cS;
                        const uint32_t sbase = ptx::smem_u32(sb + j * bk_elems * 128);
#pragma unroll
                        for (int i = 0; i < kRows; ++i) {
                            const int row = lane + 32 * i;
                            const int h = kh[i] + r, w = kw[i] + sx;
                            const bool ok = kok[i] && col < N && h >= 0 && h < p.cH && w >= 0 && w < p.cW;
                            const uint8_t* src =
                                ok ? kpix[i] + (static_cast<int64_t>(h) * p.cW + w) * rowbytes + cbyte : p.cx;
                            const uint32_t nbytes = ok ? 16u : 0u;
#pragma unroll
                            for (int c = 0; c < 8; ++c)
                                ptx::cp_async16_zfill(sbase + row * 128 + ((c ^ (row & 7)) << 4), src + 16 * c,
                                                      nbytes);
                        }
                    }
                }
                ptx::cp_async_mbar_arrive_noinc(&full[stage]);
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 0) {
        // ===================== TMA producer =====================
#ifdef QSB_GEMM_TRACE
        // isolation mode 16 (with 2, MMA-only): this warp issues a SECOND MMA
        // stream of the same shape into the other accumulator buffer -- two
        // issuing threads on one SM's tensor pipe (wrong sums; timing only)
        if ((p.debug_epi & 18) == 18 && kCta == 1 && lane == 0) {
            for (int ui = 0;; ++ui) {
                int t, kb0, kb1, role;
                if (!unit_at<kSK>(p, ui, unit0, unit_stride, num_tiles, ksplit, num_kb, t, kb0, kb1, role)) break;
                const uint32_t d2 = tmem_base + static_cast<uint32_t>(((ui & 1) ^ 1) * BN);
                for (int kb = kb0; kb < kb1; ++kb) {
                    const uint32_t a_addr = ptx::smem_u32(smem_a);
                    const uint32_t b_addr = ptx::smem_u32(smem_b);
#pragma unroll
                    for (int k = 0; k < BK_BYTES / 32; ++k) {
                        const uint64_t da = ptx::sw128_kmajor_desc(a_addr + k * 32);
                        const uint64_t db = ptx::sw128_kmajor_desc(b_addr + k * 32);
                        if (kI8)
                            ptx::mma_i8(d2, da, db, p.idesc, 1u);
                        else
                            ptx::mma_f16(d2, da, db, p.idesc, 1u);
                    }
                }
            }
            ptx::tc_commit(&full[0]);
            ptx::mbar_wait(&full[0], 0);
        } else
#endif
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int ui = 0;; ++ui) {
                int t, kb0, kb1, role;
                if (!unit_at<kSK>(p, ui, unit0, unit_stride, num_tiles, ksplit, num_kb, t, kb0, kb1, role)) break;
                const int u = unit0 + ui * unit_stride;  // (trace slot)
                (void)u;
                const int m0 = (t % num_m) * kTileM + static_cast<int>(rank) * BM;
                const int n0 = (t / num_m) * BN + static_cast<int>(rank) * kBRows;
                for (int kb = kb0; kb < kb1; ++kb) {
#ifdef QSB_GEMM_TRACE
                    if (p.debug_epi & 2) break;  // isolation: MMA-only (no operand loads)
#endif
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    if (kb == kb0) QSB_TRACE_U(u, 0);
                    if (kCta == 2) {
                        // Both CTAs' bytes complete on the leader's full barrier.
                        if (leader) ptx::mbar_arrive_expect_tx(&full[stage], kCta * C::kStageBytes);
                        const uint32_t fb = full_leader0 + stage * 8;
                        uint8_t* sa = smem_a + stage * BM * BK_BYTES;
                        uint8_t* sb = smem_b + stage * kBRows * BK_BYTES;
                        if (kLay & 1) {
                            for (int j = 0; j < BM / 64; ++j)
                                ptx::tma_load_2d_pair(sa + j * bk_elems * 128, &tm_a, fb, m0 + 64 * j,
                                                      kb * bk_elems);
                        } else {
                            ptx::tma_load_2d_pair(sa, &tm_a, fb, kb * bk_elems, m0);
                        }
                        if (kLay & 2) {
                            for (int j = 0; j < kBRows / 64; ++j)
                                ptx::tma_load_2d_pair(sb + j * bk_elems * 128, &tm_b, fb, n0 + 64 * j,
                                                      kb * bk_elems);
                        } else {
                            ptx::tma_load_2d_pair(sb, &tm_b, fb, kb * bk_elems, n0);
                        }
                    } else if (kLay & 96) {
                        // TMA im2col (implicit-GEMM conv): the hardware walks the
                        // NHWC bounding box, padding taps come back as zeros.
                        uint8_t* sa = smem_a + stage * BM * BK_BYTES;
                        uint8_t* sb = smem_b + stage * kBRows * BK_BYTES;
                        const int eb = kI8 ? 1 : 2;
                        const int rowbytes = p.cC * eb;
                        if (kLay & 32) {  // A = column tile of 128 output pixels from m0
                            ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                            const int kbyte = kb * BK_BYTES;
                            const int tap = kbyte / rowbytes;
                            const int c0 = (kbyte - tap * rowbytes) / eb;
                            const int r = tap / p.cS, sx = tap - r * p.cS;
                            const int q = m0 % p.cQ, pp = (m0 / p.cQ) % p.cP, n = m0 / (p.cQ * p.cP);
                            ptx::tma_load_im2col_4d(sa, &tm_a, &full[stage], c0, q * p.csw - p.cpw,
                                                    pp * p.csh - p.cph, n, static_cast<uint16_t>(sx),
                                                    static_cast<uint16_t>(r));
                            if (kLay & 16) {  // dgrad: W [Cout][R*S][C], taps flipped
                                const int kk = kb * bk_elems;
                                const int rs = p.cS * (p.K / p.cC / p.cS) - 1 - kk / p.cC;
                                for (int j = 0; j < kBRows / 64; ++j)
                                    ptx::tma_load_3d(sb + j * bk_elems * 128, &tm_b, &full[stage], n0 + 64 * j,
                                                     kk % p.cC, rs);
                            } else {
                                ptx::tma_load_2d(sb, &tm_b, &full[stage], kb * bk_elems, n0);
                            }
                        } else {  // wgrad: A = dY (MN-major), B = column blocks, K rows = pixels
                            const int nblk = min(kBRows / 64, static_cast<int>((N - n0 + 63) / 64));
                            ptx::mbar_arrive_expect_tx(&full[stage], BM * BK_BYTES + nblk * bk_elems * 128);
                            for (int j = 0; j < BM / 64; ++j)
                                ptx::tma_load_2d(sa + j * bk_elems * 128, &tm_a, &full[stage], m0 + 64 * j,
                                                 kb * bk_elems);
                            const int pix = kb * bk_elems;
                            const int q = pix % p.cQ, pp = (pix / p.cQ) % p.cP, n = pix / (p.cQ * p.cP);
                            for (int j = 0; j < nblk; ++j) {
                                const int kbyte = (n0 + 64 * j) * eb;
                                const int tap = kbyte / rowbytes;
                                const int c0 = (kbyte - tap * rowbytes) / eb;
                                const int r = tap / p.cS, sx = tap - r * p.cS;
                                ptx::tma_load_im2col_4d(sb + j * bk_elems * 128, &tm_b, &full[stage], c0,
                                                        q * p.csw - p.cpw, pp * p.csh - p.cph, n,
                                                        static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
                            }
                        }
                    } else {
                        ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                        uint8_t* sa = smem_a + stage * BM * BK_BYTES;
                        uint8_t* sb = smem_b + stage * kBRows * BK_BYTES;
                        if (kLay & 1) {
                            for (int j = 0; j < BM / 64; ++j)
                                ptx::tma_load_2d(sa + j * bk_elems * 128, &tm_a, &full[stage],
                                                 m0 + 64 * j, kb * bk_elems);
                        } else {
                            ptx::tma_load_2d(sa, &tm_a, &full[stage], kb * bk_elems, m0);
                        }
                        if (kLay & 2) {
                            for (int j = 0; j < kBRows / 64; ++j)
                                ptx::tma_load_2d(sb + j * bk_elems * 128, &tm_b, &full[stage],
                                                 n0 + 64 * j, kb * bk_elems);
                        } else {
                            ptx::tma_load_2d(sb, &tm_b, &full[stage], kb * bk_elems, n0);
                        }
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA of a pair) =====================
        if (kDual) {
            if (lane == 0) dual_issue(0);
        } else if (lane == 0 && leader) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int ui = 0;; ++ui) {
                int t, kb0, kb1, role;
                if (!unit_at<kSK>(p, ui, unit0, unit_stride, num_tiles, ksplit, num_kb, t, kb0, kb1, role)) break;
                const int u = unit0 + ui * unit_stride;  // (trace slot)
                (void)u;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                QSB_TRACE_U(u, 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int kb = kb0; kb < kb1; ++kb) {
#ifdef QSB_GEMM_TRACE
                    // isolation modes: 2 = MMA-only (no full wait), 4 = loads only (no MMAs)
                    if (!(p.debug_epi & 2)) ptx::mbar_wait(&full[stage], phase);
                    if (p.debug_epi & 4) {
                        if (kb == kb0) QSB_TRACE_U(u, 2);
                        ptx::mbar_arrive(&empty[stage]);
                        if (++stage == kStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
#else
                    ptx::mbar_wait(&full[stage], phase);
#endif
                    if (kb == kb0) QSB_TRACE_U(u, 2);
                    // cp.async (generic proxy) wrote A: order it before the
                    // tensor core's async-proxy reads.
                    if (kLay & 12) ptx::fence_proxy_async_smem();
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(smem_a + stage * BM * BK_BYTES);
                    const uint32_t b_addr = ptx::smem_u32(smem_b + stage * kBRows * BK_BYTES);
#pragma unroll
                    for (int k = 0; k < BK_BYTES / 32; ++k) {  // UMMA_K = 32 bytes
                        // K-major: advance 32 bytes along the swizzled row; MN-major:
                        // advance 16 K-rows (UMMA_K for 16-bit operands) of 128 bytes.
                        const uint64_t da = (kLay & 1)
                                                ? ptx::sw128_mnmajor_desc(a_addr + k * 16 * 128, bk_elems * 128)
                                                : ptx::sw128_kmajor_desc(a_addr + k * 32);
                        const uint64_t db = (kLay & 2)
                                                ? ptx::sw128_mnmajor_desc(b_addr + k * 16 * 128, bk_elems * 128)
                                                : ptx::sw128_kmajor_desc(b_addr + k * 32);
                        const uint32_t accum = (kb != kb0 || k != 0) ? 1u : 0u;
#ifdef QSB_GEMM_TRACE
                        // isolation mode 8: odd K-steps into the other accumulator
                        // buffer (wrong sums; times two independent MMA chains)
                        const uint32_t d_tmem_k = ((p.debug_epi & 8) && (k & 1))
                                                      ? tmem_base + static_cast<uint32_t>((acc ^ 1) * BN)
                                                      : d_tmem;
#define d_tmem d_tmem_k
#endif
                        if (kCta == 2) {
                            if (kI8 && kF8)
                                ptx::mma_f8_pair(d_tmem, da, db, p.idesc, accum);
                            else if (kI8)
                                ptx::mma_i8_pair(d_tmem, da, db, p.idesc, accum);
                            else
                                ptx::mma_f16_pair(d_tmem, da, db, p.idesc, accum);
                        } else {
                            if (kI8 && kF8)
                                ptx::mma_f8(d_tmem, da, db, p.idesc, accum);
                            else if (kI8)
                                ptx::mma_i8(d_tmem, da, db, p.idesc, accum);
                            else if (kTF32)
                                ptx::mma_tf32(d_tmem, da, db, p.idesc, accum);
                            else
                                ptx::mma_f16(d_tmem, da, db, p.idesc, accum);
                        }
#ifdef QSB_GEMM_TRACE
#undef d_tmem
#endif
                    }
                    if (kCta == 2)
                        ptx::tc_commit_pair(&empty[stage]);  // frees the stage in both CTAs
                    else
                        ptx::tc_commit(&empty[stage]);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (kCta == 2)
                    ptx::tc_commit_pair(&tfull[acc]);  // both CTAs' epilogues
                else
                    ptx::tc_commit(&tfull[acc]);
                QSB_TRACE_U(u, 3);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        // ===================== epilogue (warps 2..9) =====================
        if (kDual) {  // the second MMA issuer, then this warp's epilogue share
            if (warp == kEpiWarp0 && lane == 0) dual_issue(1);
            __syncwarp();
        }
        // Two warps per TMEM lane quadrant (warp w reads lanes 32*(w%4)..+31):
        // the tile's column chunks alternate between them, so each quadrant's
        // TMEM loads, dequant math and staging stores run on two warps.
        // TMEM -> registers -> (scale, bias) -> 128B-swizzled smem staging ->
        // TMA 2-D store (or reduce-add) of a 32-row x 128-byte chunk per warp.
        // The per-column factors (s_a*s_b[n], bias[n]) are staged in smem once
        // per tile by all epilogue threads (broadcast float4 reads replace the
        // per-column shuffles).  Direct global stores remain as the path for
        // shapes TMA cannot address (row pitch not a multiple of 16 bytes).
        const int ew = warp - kEpiWarp0;  // 0..7
        const int quad = warp & 3;        // TMEM lane quadrant this warp may access
        const int half = ew >> 2;         // chunks half, half + 2, ... of the tile
        const int et = ew * 32 + lane;    // 0..255
        uint8_t* my_stage = smem_stage + ew * C::kEpiBufs * kStageChunkBytes;
        float* fs = fac;       // [BN] column scale
        float* fb = fac + BN;  // [BN] column bias
        int sbuf = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        float alpha = p.alpha;
        if (p.alpha_dev) alpha *= *p.alpha_dev;
        float vmax = 0.0f;  // kYmax: this thread's running max of the unit's outputs
        (void)vmax;
        const float sa = (kI8 && p.scale_a) ? *p.scale_a : 1.0f;
        const bool out16 = p.c && p.c_dtype != QSYNC_F32;
        const bool raw = p.c_i32 != nullptr && p.c == nullptr;
        const bool need_fac = !raw && (kI8 || p.bias);
        const int chunk_cols = out16 ? 64 : 32;
#ifdef QSB_GEMM_TRACE
        unsigned long long t_ld = 0, t_math = 0, t_wait = 0, t_store = 0;
#endif
        for (int ui = 0;; ++ui) {
            int t, kb0, kb1, role;
            if (!unit_at<kSK>(p, ui, unit0, unit_stride, num_tiles, ksplit, num_kb, t, kb0, kb1, role)) break;
            const int u = unit0 + ui * unit_stride;  // (trace slot)
            (void)u;
            const bool add_bias = kb0 == 0;  // bias once per tile under split-K / stream-K
            const int64_t m0 = static_cast<int64_t>(t % num_m) * kTileM + static_cast<int64_t>(rank) * BM;
            const int64_t n0 = static_cast<int64_t>(t / num_m) * BN;
            if (need_fac) {
                // Every epilogue warp is past the previous tile's factors, then this
                // tile's are written -- BEFORE waiting for the accumulator, so their
                // latency hides behind the tile's MMAs.
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                for (int c = et; c < BN; c += kEpiWarps * 32) {
                    const int64_t col = n0 + c;
                    const bool ok = col < N;
                    if (kI8) {
                        const float sb = p.scale_b ? (p.b_per_channel ? (ok ? p.scale_b[col] : 0.0f) : *p.scale_b)
                                                   : 1.0f;
                        fs[c] = __fmul_rn(sa, sb);
                    }
                    fb[c] = (p.bias && ok && add_bias) ? p.bias[col] : 0.0f;
                }
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
            }
            ptx::mbar_wait(&tfull[acc], acc_phase);
            if (warp == kEpiWarp0 && lane == 0) QSB_TRACE_U(u, 4);
            ptx::tc_fence_after();
            const int64_t row0 = m0 + quad * 32;
            const int64_t row = row0 + lane;
            const bool row_ok = row < M;
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                                   static_cast<uint32_t>(acc * BN);
            // Stream-K owner: the contributors are the next CTAs whose ranges start
            // inside tile t; wait until all of them have published their partials.
            int sk_c0 = 0, sk_nc = 0;
            if (kSK && role == kUnitOwner) {
                const int64_t total = static_cast<int64_t>(num_tiles) * num_kb;
                const int64_t tile_end = static_cast<int64_t>(t + 1) * num_kb;
                sk_c0 = static_cast<int>(blockIdx.x) + 1;
                for (int c = sk_c0; c < static_cast<int>(gridDim.x) && total * c / gridDim.x < tile_end; ++c) ++sk_nc;
                if (et == 0) {
                    uint32_t spins = 0;
                    while (ptx::ld_acquire_gpu(p.sk_flags + t) < sk_nc)
                        if (++spins == 0x40000000u) __trap();
                    p.sk_flags[t] = 0;  // every contributor has arrived: ready for the next launch
                }
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                __threadfence();
            }
            if constexpr (kGelu) {
                // 64-column chunks: y exactly as the plain GEMM would store it (FP32
                // for INT8; the FP16 GEMM's value rounded to FP16), then the FF2
                // operand kernel's math (qsync_act_cast / gelu_absmax_store):
                // g = gelu(y) rounded as those kernels round it (to y's dtype, then to
                // c_dtype), FP16 gelu'(y), max |g| over the valid rows and columns.
                const bool g16 = p.c_dtype == QSYNC_F16;
                float amax = 0.0f;
                // one staged 32-row x 128-byte piece -> TMA store at (col, row0)
                auto emit = [&](const uint32_t (&wv)[32], const CUtensorMap* map, int64_t col) {
                    if (lane == 0) ptx::bulk_wait_read<C::kEpiBufs - 1>();
                    __syncwarp();
                    uint8_t* buf = my_stage + sbuf * kStageChunkBytes;
                    const uint32_t rbase = ptx::smem_u32(buf) + lane * 128;
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        ptx::st_shared_v4(rbase + ((c ^ (lane & 7)) << 4), wv[4 * c], wv[4 * c + 1], wv[4 * c + 2],
                                          wv[4 * c + 3]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_2d(map, buf, static_cast<int32_t>(col), static_cast<int32_t>(row0));
                        ptx::bulk_commit();
                    }
                    sbuf = (sbuf + 1) % C::kEpiBufs;
                };
#pragma unroll 1
                for (int c0 = half * 64; c0 < BN; c0 += 128) {
                    const int64_t col0 = n0 + c0;
                    uint32_t rr[2][32];
                    ptx::tmem_ld32(tbase + static_cast<uint32_t>(c0), rr[0]);
                    ptx::tmem_ld32(tbase + static_cast<uint32_t>(c0 + 32), rr[1]);
                    ptx::tmem_ld_wait();
                    if (row0 >= M || col0 >= N) continue;  // warp-uniform
                    uint32_t wg[32], wd[32];  // FP16 g (64 cols), FP16 gelu' (64 cols)
#pragma unroll
                    for (int sub = 0; sub < 2; ++sub) {
                        const int cb = c0 + 32 * sub;
                        uint32_t wf[32];  // FP32 g of these 32 columns
#pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            float gv[2], dv[2];
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const uint32_t a = rr[sub][j + e];
                                float v = kI8 ? __fmul_rn(__int2float_rn(static_cast<int>(a)), fs[cb + j + e])
                                              : __fmul_rn(bits_f(a), alpha);
                                if (p.bias) v = __fadd_rn(v, fb[cb + j + e]);
                                if (!kI8) v = __half2float(__float2half_rn(v));  // the FP16 GEMM's stored h
                                gelu_pair<!kI8>(v, gv[e], dv[e]);  // FP16 GEMM: h is an FP16 value
                                // round_to<h dtype> as the FF2 operand kernels do (FP16 for an
                                // FP16 GEMM's h), and the stored dtype
                                if (g16 || !kI8) gv[e] = __half2float(__float2half_rn(gv[e]));
                                if (row_ok && col0 + 32 * sub + j + e < N) amax = fmaxf(amax, fabsf(gv[e]));
                                wf[j + e] = __float_as_uint(gv[e]);
                            }
                            wg[16 * sub + j / 2] = pack_half2(gv[0], gv[1]);
                            wd[16 * sub + j / 2] = pack_half2(dv[0], dv[1]);
                        }
                        if (!g16) emit(wf, &tm_c, col0 + 32 * sub);
                    }
                    if (g16) emit(wg, &tm_c, col0);
                    emit(wd, &tm_d, col0);
                }
                amax = warp_max(amax);
                if (lane == 0 && amax > 0.0f) atomicMax(p.act_absmax, __float_as_uint(amax));
            } else
#pragma unroll 1
            for (int c0 = half * chunk_cols; c0 < BN; c0 += 2 * chunk_cols) {
                uint32_t w[32];  // the 128 bytes of this thread's row in the chunk
                const int64_t col0 = n0 + c0;
                const int nsub = out16 ? 2 : 1;
                // Both 32-column TMEM loads of a 16-bit chunk are in flight
                // before the single wait.
                uint32_t rr[2][32];
#ifdef QSB_GEMM_TRACE
                unsigned long long tc0 = trace_clock();
#endif
                ptx::tmem_ld32(tbase + static_cast<uint32_t>(c0), rr[0]);
                if (out16) ptx::tmem_ld32(tbase + static_cast<uint32_t>(c0 + 32), rr[1]);
                ptx::tmem_ld_wait();
                if constexpr (kDual) {  // + the odd k-blocks' accumulator (buffer 1)
#pragma unroll
                    for (int sub = 0; sub < 2; ++sub) {
                        if (sub >= nsub) break;
                        uint32_t r2[32];
                        ptx::tmem_ld32(tbase + static_cast<uint32_t>(BN + c0 + 32 * sub), r2);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            if constexpr (kI8 && !kF8)
                                rr[sub][j] = static_cast<uint32_t>(static_cast<int>(rr[sub][j]) + static_cast<int>(r2[j]));
                            else
                                rr[sub][j] = __float_as_uint(__fadd_rn(bits_f(rr[sub][j]), bits_f(r2[j])));
                        }
                    }
                }
#ifdef QSB_GEMM_TRACE
                unsigned long long tc1 = trace_clock();
                t_ld += tc1 - tc0;
#endif
                if (kSK && role != kUnitPlain) {
                    // stream-K partials: raw 32-bit accumulators of the tile in 16-byte
                    // pieces [slot][column quad][row], so a warp's 32 rows of one quad
                    // are 512 contiguous bytes (coalesced; a row-major slot made every
                    // lane's 16 bytes a separate transaction: 7 us per partial tile).
                    const int row_l = quad * 32 + lane;
                    if (role == kUnitContrib) {
                        uint32_t* dst = p.sk_ws + static_cast<size_t>(blockIdx.x) * BM * BN + row_l * 4;
#pragma unroll
                        for (int sub = 0; sub < 2; ++sub) {
                            if (sub >= nsub) break;
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                __stcg(reinterpret_cast<uint4*>(dst + ((c0 + 32 * sub + j) >> 2) * (BM * 4)),
                                       make_uint4(rr[sub][j], rr[sub][j + 1], rr[sub][j + 2], rr[sub][j + 3]));
                        }
                        continue;
                    }
                    for (int c = sk_c0; c < sk_c0 + sk_nc; ++c) {  // owner: add in CTA order
                        const uint32_t* src = p.sk_ws + static_cast<size_t>(c) * BM * BN + row_l * 4;
#pragma unroll
                        for (int sub = 0; sub < 2; ++sub) {
                            if (sub >= nsub) break;
#pragma unroll
                            for (int j = 0; j < 32; j += 4) {
                                const uint4 v =
                                    __ldcg(reinterpret_cast<const uint4*>(src + ((c0 + 32 * sub + j) >> 2) * (BM * 4)));
                                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    if constexpr (kI8 && !kF8)
                                        rr[sub][j + e] = static_cast<uint32_t>(static_cast<int>(rr[sub][j + e]) +
                                                                               static_cast<int>(w4[e]));
                                    else
                                        rr[sub][j + e] = __float_as_uint(__fadd_rn(bits_f(rr[sub][j + e]), bits_f(w4[e])));
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int sub = 0; sub < 2; ++sub) {
                    if (sub >= nsub) break;
                    uint32_t (&r)[32] = rr[sub];
                    if (p.debug_epi) continue;
                    if (raw) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) w[j] = r[j];
                        continue;
                    }
                    if (p.c_i32 && row_ok && row0 < M) {
                        // both outputs requested (direct-store path): raw accumulators first
                        int32_t* dst = p.c_i32 + row * N + col0;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < N) dst[j] = static_cast<int32_t>(r[j]);
                    }
                    const int cb = c0 + 32 * sub;  // tile column of r[0]
                    const bool bf = p.c_dtype == QSYNC_BF16;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        float4 s4 = make_float4(alpha, alpha, alpha, alpha);
                        if (kI8) s4 = *reinterpret_cast<const float4*>(fs + cb + j);
                        const float sj[4] = {s4.x, s4.y, s4.z, s4.w};
                        float v[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const uint32_t a = r[j + e];
                            v[e] = kI8 ? __fmul_rn(kF8 ? bits_f(a) : __int2float_rn(static_cast<int>(a)), sj[e])
                                       : __fmul_rn(bits_f(a), sj[e]);
                        }
                        if (p.bias) {
                            const float4 b4 = *reinterpret_cast<const float4*>(fb + cb + j);
                            v[0] = __fadd_rn(v[0], b4.x);
                            v[1] = __fadd_rn(v[1], b4.y);
                            v[2] = __fadd_rn(v[2], b4.z);
                            v[3] = __fadd_rn(v[3], b4.w);
                        }
                        if constexpr (kYmax) {  // valid rows / columns only (padding rows hold the bias)
                            if (row_ok) {
#pragma unroll
                                for (int e = 0; e < 4; ++e)
                                    if (col0 + 32 * sub + j + e < N) vmax = fmaxf(vmax, v[e]);
                            }
                        }
                        if (out16) {
                            w[16 * sub + j / 2] = bf ? pack_bf162(v[0], v[1]) : pack_half2(v[0], v[1]);
                            w[16 * sub + j / 2 + 1] = bf ? pack_bf162(v[2], v[3]) : pack_half2(v[2], v[3]);
                        } else {
#pragma unroll
                            for (int e = 0; e < 4; ++e) w[j + e] = __float_as_uint(v[e]);
                        }
                    }
                }
#ifdef QSB_GEMM_TRACE
                unsigned long long tc2 = trace_clock();
                t_math += tc2 - tc1;
#endif
                if (row0 >= M || col0 >= N || p.debug_epi) continue;  // warp-uniform skip
                if (p.tma_store) {
                    // Free the staging buffer used kEpiBufs chunks ago, then write
                    // this row's 8 x 16B pieces at their 128B-swizzled positions.
                    if (lane == 0) ptx::bulk_wait_read<C::kEpiBufs - 1>();
                    __syncwarp();
#ifdef QSB_GEMM_TRACE
                    unsigned long long tc3 = trace_clock();
                    t_wait += tc3 - tc2;
#endif
                    uint8_t* buf = my_stage + sbuf * kStageChunkBytes;
                    const uint32_t rbase = ptx::smem_u32(buf) + lane * 128;
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        ptx::st_shared_v4(rbase + ((c ^ (lane & 7)) << 4), w[4 * c], w[4 * c + 1],
                                          w[4 * c + 2], w[4 * c + 3]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (p.accumulate)
                            ptx::tma_reduce_add_2d(&tm_c, buf, static_cast<int32_t>(col0),
                                                   static_cast<int32_t>(row0));
                        else
                            ptx::tma_store_2d(&tm_c, buf, static_cast<int32_t>(col0),
                                              static_cast<int32_t>(row0));
                        ptx::bulk_commit();
                    }
                    sbuf = (sbuf + 1) % C::kEpiBufs;
#ifdef QSB_GEMM_TRACE
                    t_store += trace_clock() - tc3;
#endif
                    continue;
                }
                // ---- direct-store path (fully unrolled: keeps w[] in registers) ----
                if (!row_ok) continue;
                if (raw) {
                    int32_t* dst = p.c_i32 + row * N + col0;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (col0 + j < N) dst[j] = static_cast<int32_t>(w[j]);
                    continue;
                }
                if (!out16) {
                    float* dst = static_cast<float*>(p.c) + row * N + col0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (col0 + j < N) {
                            const float x = __uint_as_float(w[j]);
                            dst[j] = p.accumulate ? dst[j] + x : x;
                        }
                    }
                } else {
                    uint16_t* dst = static_cast<uint16_t*>(p.c) + row * N + col0;
                    const bool bf = p.c_dtype == QSYNC_BF16;
#pragma unroll
                    for (int j = 0; j < 64; ++j) {
                        if (col0 + j < N) {
                            const uint16_t h = static_cast<uint16_t>((w[j >> 1] >> (16 * (j & 1))) & 0xffffu);
                            if (!p.accumulate) {
                                dst[j] = h;
                            } else {
                                const float old = bf ? __bfloat162float(__ushort_as_bfloat16(dst[j]))
                                                     : __half2float(__ushort_as_half(dst[j]));
                                const float nv = (bf ? __bfloat162float(__ushort_as_bfloat16(h))
                                                     : __half2float(__ushort_as_half(h))) + old;
                                dst[j] = bf ? __bfloat16_as_ushort(__float2bfloat16_rn(nv))
                                            : __half_as_ushort(__float2half_rn(nv));
                            }
                        }
                    }
                }
            }
            if constexpr (kYmax) {
                vmax = warp_max(vmax);
                if (lane == 0 && vmax > 0.0f) atomicMax(p.ymax, __float_as_uint(vmax));
                vmax = 0.0f;
            }
            if (kSK && role == kUnitContrib) {  // publish this CTA's partial of tile t
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                if (et == 0) atomicAdd(p.sk_flags + t, 1);
            }
            if (warp == kEpiWarp0 && lane == 0) QSB_TRACE_U(u, 5);
            ptx::tc_fence_before();
            if (kCta == 2)
                ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);  // leader's barrier
            else
                ptx::mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        // The staging smem must outlive the TMA reads only; the global writes complete
        // with the grid (the next kernel sees them after its griddepcontrol.wait).
        if (lane == 0) ptx::bulk_wait_read<0>();
#ifdef QSB_GEMM_TRACE
        if (warp == kEpiWarp0 && lane == 0) {  // header slots 5..7 + the spare slot 71
            QSB_TRACE(5, t_ld);
            QSB_TRACE(6, t_math);
            QSB_TRACE(7, t_wait);
            QSB_TRACE(71, t_store);
        }
#endif
    }

    ptx::tc_fence_before();
    if (kCta == 2)
        ptx::cluster_sync();  // both CTAs done with TMEM and remote barriers
    else
        __syncthreads();
#ifdef QSB_GEMM_TRACE
    if (threadIdx.x == 0) {
        QSB_TRACE(3, trace_clock());
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        QSB_TRACE(4, gt);
    }
#endif
    if (warp == 1) {
        ptx::tc_fence_after();
        if (kCta == 2)
            ptx::tmem_dealloc_pair<C::kTmemCols>(tmem_base);
        else
            ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// ---------------------------------------------------------------------------
// Host side: tensor maps (driver entry point fetched through the runtime so
// the library does not link libcuda), tile-shape selection, launch.
// ---------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

int make_map(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, uint32_t elem_bytes,
             int64_t inner, int64_t outer, uint32_t box_inner, uint32_t box_outer) {
    // (inner extent may be padded by the caller's pitch; here pitch == inner)
    EncodeFn fn = encode_fn();
    QSB_REQUIRE(fn != nullptr, QSYNC_ERR_INTERNAL, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(inner) * elem_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    QSB_REQUIRE(r == CUDA_SUCCESS, QSYNC_ERR_INTERNAL,
                "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return QSYNC_OK;
}

// 3-D map: dims (inner, d1, d2) with byte strides (s1, s2) for d1, d2 (any
// order), box (box_inner, box_1, 1).
int make_map_3d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, uint32_t elem_bytes,
                int64_t inner, int64_t d1, int64_t d2, int64_t s1, int64_t s2, uint32_t box_inner,
                uint32_t box_1) {
    EncodeFn fn = encode_fn();
    QSB_REQUIRE(fn != nullptr, QSYNC_ERR_INTERNAL, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(d1),
                          static_cast<cuuint64_t>(d2)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(s1), static_cast<cuuint64_t>(s2)};
    cuuint32_t box[3] = {box_inner, box_1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    (void)elem_bytes;
    CUresult r = fn(map, dt, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    QSB_REQUIRE(r == CUDA_SUCCESS, QSYNC_ERR_INTERNAL,
                "cuTensorMapEncodeTiled (3-D) failed (" + std::to_string(static_cast<int>(r)) + ")");
    return QSYNC_OK;
}

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
    static EncodeIm2colFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeIm2colFn>(f);
    });
    return fn;
}

// im2col map over the NHWC tensor the conv gathers from (p.cx geometry): dims
// {C, W, H, N}; the bounding box spans input coordinates [-pad, dim-1+pad-(k-1)]
// walked with the conv strides, so consecutive box pixels are consecutive GEMM
// rows (n, p, q); `pixels` rows of 128 bytes per load, 128B-swizzled.
int make_im2col_map(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, uint32_t eb, const EpiParams& p,
                    uint32_t pixels) {
    EncodeIm2colFn fn = encode_im2col_fn();
    QSB_REQUIRE(fn != nullptr, QSYNC_ERR_INTERNAL, "cuTensorMapEncodeIm2col unavailable");
    const int R = static_cast<int>(p.cR), S = p.cS;
    QSB_REQUIRE(p.cpw <= 127 && p.cph <= 127 && p.cpw - (S - 1) >= -128 && p.cph - (R - 1) >= -128 &&
                    p.csw <= 8 && p.csh <= 8 && R <= 65535 && S <= 65535,
                QSYNC_ERR_DOMAIN, "conv geometry outside the TMA im2col range");
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(p.cC), static_cast<cuuint64_t>(p.cW),
                          static_cast<cuuint64_t>(p.cH), static_cast<cuuint64_t>(p.cN)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(p.cC) * eb, static_cast<cuuint64_t>(p.cW) * p.cC * eb,
                             static_cast<cuuint64_t>(p.cH) * p.cW * p.cC * eb};
    int lower[2] = {-p.cpw, -p.cph};
    int upper[2] = {p.cpw - (S - 1), p.cph - (R - 1)};
    cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(p.csw), static_cast<cuuint32_t>(p.csh), 1};
    CUresult r = fn(map, dt, 4, const_cast<void*>(ptr), dims, strides, lower, upper, BK_BYTES / eb, pixels, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    QSB_REQUIRE(r == CUDA_SUCCESS, QSYNC_ERR_INTERNAL,
                "cuTensorMapEncodeIm2col failed (" + std::to_string(static_cast<int>(r)) + ")");
    return QSYNC_OK;
}

// Instruction descriptor (tcgen05 "idesc"): c_format [4,6), a_format [7,10),
// b_format [10,13), a/b major [15],[16] (0 = K-major), N>>3 [17,23), M>>4 [24,29).
uint32_t make_idesc(bool i8, bool bf16, int n, int m, int lay = 0, bool fp8 = false, bool tf32 = false) {
    uint32_t d = 0;
    d |= static_cast<uint32_t>(lay & 1) << 15;         // A MN-major
    d |= static_cast<uint32_t>((lay >> 1) & 1) << 16;  // B MN-major
    d |= (i8 && !fp8 ? 2u : 1u) << 4;                 // S32 / F32 accumulator
    // kind::i8: signed = 1; kind::f16: F16 = 0, BF16 = 1; kind::tf32: TF32 = 2;
    // kind::f8f6f4: E4M3 = 0
    const uint32_t fmt = fp8 ? 0u : (i8 ? 1u : (tf32 ? 2u : (bf16 ? 1u : 0u)));
    d |= fmt << 7;
    d |= fmt << 10;
    d |= static_cast<uint32_t>(n >> 3) << 17;
    d |= static_cast<uint32_t>(m >> 4) << 24;         // 128 (1 CTA) or 256 (CTA pair)
    return d;
}

int g_force_splitk = 0;  // test/bench hook (qsync_gemm_force_splitk): 0 = heuristic
int g_splitk_wide = 0;   // accumulate GEMMs prefer BN=256 (bench hook)
int g_force_cta = 0;     // test/bench hook (qsync_gemm_force_cta): 0 = cost model, 1, 2
int g_debug_epi = 0;     // bench hook (qsync_gemm_debug_epilogue)
int g_pdl = 1;           // programmatic dependent launch (qsync_gemm_set_pdl)
int g_max_ctas = 0;      // cap on the persistent grid (qsync_gemm_set_max_ctas), 0 = all SMs
int g_conv_tma = 1;      // implicit conv operand loads: 1 = TMA im2col, 0 = cp.async gather lanes
// Stream-K (qsync_gemm_set_streamk): -1 = never (default), 0 = cost model,
// 1 = wherever eligible.  Off by default: graph-timed at every BERT step shape
// it lost to the tile schedule -- accumulating dgrad / wgrad 18.6 vs 16.8 us
// (QKV dgrad), 13.3 vs 9.7 (O wgrad), 21.8 vs 18.7 (FF2 wgrad); with a plain
// output the partial-tile fixup made it 2-3x slower (tools/acc_sweep.py,
// tools/gemm_overhead.py --streamk).  The 256-wide tiles it needs run the
// MN-major B operand at ~86% of their MMA rate and each CTA's range crosses
// tile boundaries, each crossing a pipeline drain + an accumulator switch.
int g_streamk = -1;
// Two MMA issuers (kLay bit 11) for 192-wide single-CTA tiles when every CTA
// owns exactly one work unit of >= 4 k-blocks (qsync_gemm_set_dual; 1 = on).
int g_dual = 1;

// Stream-K scratch, one per (device, stream) and never freed (a captured graph
// keeps pointing at it): partial accumulators of at most one unit per CTA
// ([CTAs][128][256] 32-bit) + one arrival counter per tile (zeroed once; the
// tile's owner resets it).  Allocated on first use outside a graph capture; a
// GEMM captured on a stream that has none keeps the tile schedule.
constexpr int kSkMaxTiles = 1 << 16;
struct SkWorkspace {
    uint32_t* ws = nullptr;
    int* flags = nullptr;
};
int sk_workspace(cudaStream_t st, SkWorkspace& out) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, SkWorkspace> table;
    int dev = 0;
    QSB_TRY(cuda_status(cudaGetDevice(&dev), "cudaGetDevice"));
    std::lock_guard<std::mutex> lock(mu);
    SkWorkspace& w = table[{dev, st}];
    if (!w.ws) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        QSB_TRY(cuda_status(cudaStreamIsCapturing(st, &cap), "cudaStreamIsCapturing"));
        if (cap != cudaStreamCaptureStatusNone) {
            out = SkWorkspace{};
            return QSYNC_OK;
        }
        const size_t bytes = static_cast<size_t>(sm_count()) * BM * 256 * 4;
        QSB_TRY(cuda_status(cudaMalloc(reinterpret_cast<void**>(&w.ws), bytes), "cudaMalloc(stream-K partials)"));
        QSB_TRY(cuda_status(cudaMalloc(reinterpret_cast<void**>(&w.flags), sizeof(int) * kSkMaxTiles),
                            "cudaMalloc(stream-K flags)"));
        QSB_TRY(cuda_status(cudaMemsetAsync(w.flags, 0, sizeof(int) * kSkMaxTiles, st), "cudaMemsetAsync"));
    }
    out = w;
    return QSYNC_OK;
}

template <bool kI8, int BN, int kCta, int kLay>
int launch(const void* a, const void* b, CUtensorMapDataType dt, EpiParams p, cudaStream_t st) {
    using C = Cfg<BN, kCta>;
    const uint32_t eb = kI8 ? 1 : ((kLay & 256) ? 4 : 2);
    const uint32_t box_k = BK_BYTES / eb;
    CUtensorMap ma, mb, mc, md;
    std::memset(&md, 0, sizeof(md));
    if (kLay & 512)  // GELU epilogue: FP16 gelu'(y) [M, N], 64-column x 32-row boxes
        QSB_TRY(make_map(&md, p.dact, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, p.N, p.M, 64, 32));
    if (kLay & 4)  // implicit conv: A is gathered by the producer lanes
        std::memset(&ma, 0, sizeof(ma));
    else if (kLay & 32)  // A = im2col view of the NHWC input, 128 pixels x 128 bytes
        QSB_TRY(make_im2col_map(&ma, a, dt, eb, p, BM));
    else if (kLay & 1)  // A stored [K, M]: boxes of 64 M-elements x box_k K-rows
        QSB_TRY(make_map(&ma, a, dt, eb, p.M, p.K, 64, box_k));
    else
        QSB_TRY(make_map(&ma, a, dt, eb, p.K, p.M, box_k, BM));
    if (kLay & 8)  // implicit wgrad: B is gathered by the producer lanes
        std::memset(&mb, 0, sizeof(mb));
    else if (kLay & 64)  // wgrad B = im2col view of the input, bk pixels x 128 bytes
        QSB_TRY(make_im2col_map(&mb, b, dt, eb, p, box_k));
    else if (kLay & 16)  // dgrad weights W [Cout][R*S][C] as the MN-major B [(rs, k), c]
        QSB_TRY(make_map_3d(&mb, b, dt, eb, p.N, p.cC, p.K / p.cC,
                            (p.K / p.cC) * p.N * eb, static_cast<int64_t>(p.N) * eb, 64, box_k));
    else if (kLay & 2)
        QSB_TRY(make_map(&mb, b, dt, eb, p.N, p.K, 64, box_k));
    else
        QSB_TRY(make_map(&mb, b, dt, eb, p.K, p.N, box_k, C::kBRows));
    std::memset(&mc, 0, sizeof(mc));
    // TMA-store epilogue when exactly one output is requested and its rows are
    // 16-byte pitched and aligned; 16-bit accumulate keeps the direct path.
    const bool raw = p.c_i32 && !p.c;
    const bool one_out = (p.c_i32 != nullptr) != (p.c != nullptr);
    const void* cptr = raw ? static_cast<const void*>(p.c_i32) : p.c;
    const uint32_t ceb = (raw || p.c_dtype == QSYNC_F32) ? 4 : 2;
    p.tma_store = one_out && (p.N * ceb) % 16 == 0 && (reinterpret_cast<uintptr_t>(cptr) & 15) == 0 &&
                  !(p.accumulate && ceb == 2);
    if (p.tma_store) {
        const CUtensorMapDataType cdt = raw ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                      : p.c_dtype == QSYNC_F32  ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                      : p.c_dtype == QSYNC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                                : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
        QSB_TRY(make_map(&mc, cptr, cdt, ceb, p.N, p.M, 128 / ceb, 32));
    }
    QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_gemm_tc<kI8, BN, kCta, kLay>),
                                    C::kSmemBytes));
    const int64_t tiles = ((p.M + BM * kCta - 1) / (BM * kCta)) * ((p.N + BN - 1) / BN);
    // Split-K when the tile grid leaves SMs idle and the result is reduce-added
    // anyway (accumulating FP32 output, e.g. wgrad into the flat main_grad).
    const int64_t bk_elems = BK_BYTES / eb;
    const int64_t num_kb = (p.K + bk_elems - 1) / bk_elems;
    const int preset = p.ksplit;  // chosen by dispatch (choose_acc), 0 = decide here
    p.ksplit = 1;
    p.kb_per = static_cast<int>(num_kb);
    const int sms = sm_count();
    const int slots = sms / kCta;  // concurrent (pair) tiles
    const bool can_split = p.accumulate && p.tma_store && p.c_dtype == QSYNC_F32 && !kI8;
    if (g_force_splitk > 0) {
        if (can_split && g_force_splitk > 1) {
            const int64_t per = (num_kb + g_force_splitk - 1) / g_force_splitk;
            p.kb_per = static_cast<int>(per);
            p.ksplit = static_cast<int>((num_kb + per - 1) / per);
        }
    } else if (can_split && preset > 0) {
        if (preset > 1) {
            const int64_t per = (num_kb + preset - 1) / preset;
            p.kb_per = static_cast<int>(per);
            p.ksplit = static_cast<int>((num_kb + per - 1) / per);
        }
    } else if (can_split && tiles < slots && !(kLay & 2048)) {  // (dual issue: the split is dispatch's)
        int64_t want = std::max<int64_t>(1, (2 * slots) / tiles);         // ~2 units per slot
        want = std::min<int64_t>(want, std::max<int64_t>(1, num_kb / 8));  // >= 8 k-blocks each
        if (want > 1) {
            const int64_t per = (num_kb + want - 1) / want;
            p.kb_per = static_cast<int>(per);
            p.ksplit = static_cast<int>((num_kb + per - 1) / per);
        }
    }
    if (!(kLay & 1024)) p.streamk = 0;
    if (p.streamk) {
        SkWorkspace w;
        QSB_TRY(sk_workspace(st, w));
        if (kCta != 1 || g_max_ctas > 0 || tiles > kSkMaxTiles || (!p.accumulate && !w.ws) || BN > 256 ||
            (p.accumulate && !p.tma_store)) {
            p.streamk = 0;
        } else {
            p.sk_ws = w.ws;
            p.sk_flags = w.flags;
            p.ksplit = 1;
            p.kb_per = static_cast<int>(num_kb);
        }
    }
    const int64_t units = p.streamk ? std::min<int64_t>(tiles * num_kb, slots) : tiles * p.ksplit;
    int64_t cap = slots;
    if (g_max_ctas > 0) cap = std::max<int64_t>(1, std::min<int64_t>(slots, g_max_ctas / kCta));
    QSB_REQUIRE(!(kLay & 2048) || (units <= cap && p.kb_per >= 2), QSYNC_ERR_INTERNAL,
                "dual-issue GEMM needs one work unit of >= 2 k-blocks per CTA");
    const int grid = static_cast<int>(std::min<int64_t>(units, cap)) * kCta;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (g_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (kCta == 2) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 2;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    QSB_TRY(cuda_status(cudaLaunchKernelEx(&cfg, k_gemm_tc<kI8, BN, kCta, kLay>, ma, mb, mc, md, p),
                        "cudaLaunchKernelEx(k_gemm_tc)"));
    return check_launch("k_gemm_tc");
}

// Tile-shape cost model: per k-block a tile costs max(MMA cycles, operand bytes
// this SM pulls from L2 / ~64 B per cycle); total = waves x k-blocks x that.
// CTA pairs halve the B bytes per SM (each CTA holds half of B).
struct Shape {
    int bn, cta;
};
Shape pick_shape(int64_t M, int64_t N, bool allow_pair) {
    const int sms = sm_count();
    // 192-wide tiles: N = 768 is 4 of them, so M = 4096 fills 128 SMs in one
    // wave where 256-wide tiles leave a third of the SMs idle (96 tiles).
    const Shape cands[6] = {{256, 2}, {256, 1}, {192, 1}, {128, 2}, {128, 1}, {64, 1}};
    Shape best{256, 1};
    double best_cost = 1e300;
    for (const Shape& c : cands) {
        // Measured (tools/bench_bwd_gemm.py): CTA pairs win at 8192^3 (+11% INT8)
        // but not at BERT-sized GEMMs (<= 1 wave of 256x256 pair tiles), where
        // fixed costs dominate -- only consider them with >= 3 waves of work.
        if (c.cta == 2 && (!allow_pair || M <= BM ||
                           ((M + BM - 1) / BM) * ((N + 255) / 256) < 3LL * sms))
            continue;
        const int64_t tiles = ((M + BM * c.cta - 1) / (BM * c.cta)) * ((N + c.bn - 1) / c.bn);
        const int64_t slots = sms / c.cta;
        const int64_t waves = (tiles + slots - 1) / slots;
        const double mma = 4.0 * BM * c.bn / 256.0;
        const double l2 = (BM + c.bn / c.cta) * 128.0 / 64.0;
        const double cost = static_cast<double>(waves) * std::max(mma, l2);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = c;
        }
    }
    return best;
}

// Tile width and split-K of an accumulating FP32 GEMM (wgrad into main_grad,
// dgrad reduce-added into the residual gradient), chosen together: a unit
// (tile, K range) costs its k-blocks x the measured per-k-block time plus a
// fixed pipeline fill + reduce-add epilogue; the GEMM costs waves x that.
// Per k-block (4 MMAs of K = 32 bytes): tcgen05.mma at M = 128 takes >= ~116
// cycles per instruction whatever N <= 192 (isolation runs of the trace build,
// MMA-only: 463-467 cycles per k-block at N = 64, 128, 192 and for CTA pairs),
// + ~12% when the operand loads run beside it; N = 256 runs at its own rate
// (128 / MMA) and, with an MN-major B, ~86% of it.  The fixed cost is fitted to
// tools/acc_sweep.py.  E.g. wgrad QKV 2304x768x4096 -> 192-wide tiles split 2
// ways = 144 units, one wave; wgrad FF1/FF2 -> 256-wide split 2 ways; dgrad
// QKV / FF1 (4096x768, K 2304 / 3072) -> 192-wide, no split (128 tiles).
struct AccChoice {
    int bn, ksplit;
};
AccChoice choose_acc(int64_t M, int64_t N, int64_t num_kb) {
    int slots = sm_count();
    if (g_max_ctas > 0) slots = std::min(slots, g_max_ctas);
    AccChoice best{256, 1};
    double best_cost = 1e300;
    for (int bn : {256, 192, 128}) {
        const int64_t tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
#ifdef QSB_ACC_MODEL_R1
        const double kb_cost = std::max(4.0 * BM * bn / 256.0, (BM + bn) * 128.0 / 64.0);
        const double fixed = 1500.0 + 8.0 * bn;
#else
        const double kb_cost = bn >= 256 ? 600.0 : 520.0;
        const double fixed = 6000.0;
#endif
        for (int ks = 1; ks <= 16; ++ks) {
            const int64_t per = (num_kb + ks - 1) / ks;
            if (ks > 1 && per < 4) break;
            const int64_t units = tiles * ((num_kb + per - 1) / per);
            const int64_t waves = (units + slots - 1) / slots;
            const double cost = static_cast<double>(waves) * (static_cast<double>(per) * kb_cost + fixed);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = {bn, ks};
            }
        }
    }
    return best;
}

template <bool kI8, int kLay>
int dispatch_shape(const void* a, const void* b, CUtensorMapDataType dt, EpiParams p,
                   cudaStream_t st, Shape sh) {
    if (sh.cta == 2) {
        switch (sh.bn) {
            case 256: return launch<kI8, 256, 2, kLay>(a, b, dt, p, st);
            case 128: return launch<kI8, 128, 2, kLay>(a, b, dt, p, st);
            case 192:
                // 96 B rows per CTA: one 96-row TMA box when B is K-major; the
                // MN-major B loads come in 64-wide blocks, so no 192-wide pair there.
                if constexpr (!(kLay & 2)) return launch<kI8, 192, 2, kLay>(a, b, dt, p, st);
                break;
            default: break;
        }
    }
    switch (sh.bn) {
        case 256: return launch<kI8, 256, 1, kLay>(a, b, dt, p, st);
        case 192: return launch<kI8, 192, 1, kLay>(a, b, dt, p, st);
        case 128: return launch<kI8, 128, 1, kLay>(a, b, dt, p, st);
        case 64: return launch<kI8, 64, 1, kLay>(a, b, dt, p, st);
        default: return set_error(QSYNC_ERR_DOMAIN, "unsupported tile N " + std::to_string(sh.bn));
    }
}

template <bool kI8>
int dispatch(const void* a, const void* b, CUtensorMapDataType dt, EpiParams p, cudaStream_t st,
             int force_bn, int layout = 0) {
    const bool splitk_ok = !kI8 && p.accumulate && p.c_dtype == QSYNC_F32 && g_splitk_wide;
    // Accumulating FP32 GEMMs (wgrad) go split-K on single-CTA 256-wide tiles.
    const bool accumulating = !kI8 && p.accumulate && p.c_dtype == QSYNC_F32;
    Shape sh = pick_shape(p.M, p.N, g_force_cta != 1 && !accumulating);
    if (splitk_ok) sh.bn = 256;
    if (accumulating && !splitk_ok && !force_bn && g_force_splitk == 0 && !(layout & 108)) {
        const AccChoice c = choose_acc(p.M, p.N, (p.K + 63) / 64);
        sh.bn = c.bn;
        sh.cta = 1;
        p.ksplit = c.ksplit;
    } else if (accumulating) {
        sh.bn = 256;
    }
    if (force_bn) sh.bn = force_bn;
    if (g_force_cta) sh.cta = g_force_cta;
    // Stream-K candidate (plain operand layouts): 256-wide single-CTA tiles --
    // the only width at which tcgen05.mma runs at its rate (116-cycle floor per
    // instruction below it) -- with the tiles x k-blocks space spread evenly over
    // all SMs, so N = 768 GEMMs (96 such tiles at M = 4096) use the whole chip.
    // Costs in cycles per k-block as choose_acc, + a partial write/read fixup.
    const bool sk_layout = layout == 0 || layout == 2 || layout == 3;
    // The cost model only takes accumulating FP32 outputs, where every unit
    // reduce-adds its partial.  With a plain output the fixup (a 128 KB partial
    // tile written, then read back by the tile's owner) cost more than the even
    // split saved at every step shape (tools/gemm_overhead.py --streamk 1: O
    // 8.3 -> 22 us, FF2 19.5 -> 30 us); qsync_gemm_set_streamk(1) still forces
    // it (tested bit-exact for INT8).
    const bool sk_acc = p.c != nullptr && p.c_i32 == nullptr && p.accumulate && !kI8 && p.c_dtype == QSYNC_F32;
    const bool sk_plain = p.c != nullptr && p.c_i32 == nullptr && !p.accumulate;
    const bool sk_out = g_streamk == 1 ? (sk_acc || sk_plain) : sk_acc;
    if (g_streamk >= 0 && sk_layout && sk_out && !force_bn && !g_force_cta && g_force_splitk == 0 &&
        g_max_ctas == 0) {
        const int sms = sm_count();
        const int64_t bk = kI8 ? BK_BYTES : BK_BYTES / 2;
        const int64_t kb = (p.K + bk - 1) / bk;
        const int64_t mt = (p.M + BM - 1) / BM;
        const double kb256 = (layout & 2) ? 600.0 : 560.0;
        const double sk_cost = static_cast<double>((mt * ((p.N + 255) / 256) * kb + sms - 1) / sms) * kb256 +
                               (p.accumulate ? 0.0 : 3000.0) + 6000.0;
        const int64_t ks = std::max(1, p.ksplit);
        const int64_t units = ((p.M + BM * sh.cta - 1) / (BM * sh.cta)) * ((p.N + sh.bn - 1) / sh.bn) * ks;
        const int64_t slots = sms / sh.cta;
        const double kbc = sh.bn >= 256 ? (sh.cta == 2 ? 540.0 : kb256) : 520.0;
        const double cl_cost =
            static_cast<double>((units + slots - 1) / slots) * (static_cast<double>((kb + ks - 1) / ks) * kbc + 6000.0);
        if (g_streamk == 1 || sk_cost < 0.9 * cl_cost) {
            sh = Shape{256, 1};
            p.streamk = 1;
            p.ksplit = 0;
        }
    }
    // pairs: BN/2 a multiple of 64, or 96 with a K-major B
    if (sh.cta == 2 && (sh.bn == 64 || (sh.bn == 192 && (layout & 2)))) sh.cta = 1;
    p.idesc = make_idesc(kI8, dt == CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, sh.bn, BM * sh.cta, layout, p.fp8);
    p.debug_epi = g_debug_epi;
    if (!p.streamk && g_dual && !p.fp8 && sh.cta == 1 && sh.bn == 192 && g_max_ctas == 0 &&
        (layout == 0 || layout == 2 || layout == 3)) {
        // dual issue: one unit per CTA (tiles x K-splits <= SMs), >= 4 k-blocks each
        const int64_t bk = kI8 ? BK_BYTES : BK_BYTES / 2;
        const int64_t kb = (p.K + bk - 1) / bk;
        const int64_t ks = std::max(1, p.ksplit);
        const int64_t units = ((p.M + BM - 1) / BM) * ((p.N + 191) / 192) * ks;
        if (units <= sm_count() && (kb + ks - 1) / ks >= 4) {
            if (layout == 0) return launch<kI8, 192, 1, 2048>(a, b, dt, p, st);
            if constexpr (!kI8) {
                if (layout == 2) return launch<false, 192, 1, 2050>(a, b, dt, p, st);
                if (layout == 3) return launch<false, 192, 1, 2051>(a, b, dt, p, st);
            }
        }
    }
    if (p.streamk && !p.fp8) {  // the stream-K instantiations (kLay bit 10)
        if (layout == 0) return launch<kI8, 256, 1, 1024>(a, b, dt, p, st);
        if constexpr (!kI8) {
            if (layout == 2) return launch<false, 256, 1, 1026>(a, b, dt, p, st);
            if (layout == 3) return launch<false, 256, 1, 1027>(a, b, dt, p, st);
        }
    }
    p.streamk = 0;
    if (layout & 108) {  // implicit conv (fwd 4/32, dgrad 22/50, wgrad 11/67): single-CTA tiles
        sh.cta = 1;
        if (sh.bn == 192) sh.bn = 256;  // (no 192-wide conv instantiations)
        p.idesc = make_idesc(kI8, dt == CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, sh.bn, BM, layout & 3, p.fp8);
        if (layout == 4) {
            switch (sh.bn) {
                case 256: return launch<kI8, 256, 1, 4>(a, b, dt, p, st);
                case 128: return launch<kI8, 128, 1, 4>(a, b, dt, p, st);
                default: return launch<kI8, 64, 1, 4>(a, b, dt, p, st);
            }
        }
        if (layout == 32) {
            switch (sh.bn) {
                case 256: return launch<kI8, 256, 1, 32>(a, b, dt, p, st);
                case 128: return launch<kI8, 128, 1, 32>(a, b, dt, p, st);
                default: return launch<kI8, 64, 1, 32>(a, b, dt, p, st);
            }
        }
        if (kI8) return set_error(QSYNC_ERR_DOMAIN, "implicit conv backward is FP16/BF16 only");
        if (layout == 22) {
            switch (sh.bn) {
                case 256: return launch<false, 256, 1, 22>(a, b, dt, p, st);
                case 128: return launch<false, 128, 1, 22>(a, b, dt, p, st);
                default: return launch<false, 64, 1, 22>(a, b, dt, p, st);
            }
        }
        if (layout == 50) {
            switch (sh.bn) {
                case 256: return launch<false, 256, 1, 50>(a, b, dt, p, st);
                case 128: return launch<false, 128, 1, 50>(a, b, dt, p, st);
                default: return launch<false, 64, 1, 50>(a, b, dt, p, st);
            }
        }
        if (layout == 11) return launch<false, 256, 1, 11>(a, b, dt, p, st);
        if (layout == 67) return launch<false, 256, 1, 67>(a, b, dt, p, st);
        return set_error(QSYNC_ERR_DOMAIN, "unsupported implicit conv layout " + std::to_string(layout));
    }
    if (layout == 4096) {  // INT8 with ymax: single-CTA 128..256-wide K-major tiles
        if constexpr (kI8) {
            if (sh.bn == 64) sh.bn = 128;
            p.idesc = make_idesc(true, false, sh.bn, BM, 0, false);
            switch (sh.bn) {
                case 256: return launch<true, 256, 1, 4096>(a, b, dt, p, st);
                case 192: return launch<true, 192, 1, 4096>(a, b, dt, p, st);
                default: return launch<true, 128, 1, 4096>(a, b, dt, p, st);
            }
        }
        return set_error(QSYNC_ERR_DOMAIN, "ymax GEMM is INT8 only");
    }
    if (layout == 512) {  // GELU epilogue (FF1): single-CTA 128..256-wide K-major tiles
        if (sh.bn == 64) sh.bn = 128;
        p.idesc = make_idesc(kI8, dt == CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, sh.bn, BM, 0, false);
        switch (sh.bn) {
            case 256: return launch<kI8, 256, 1, 512>(a, b, dt, p, st);
            case 192: return launch<kI8, 192, 1, 512>(a, b, dt, p, st);
            default: return launch<kI8, 128, 1, 512>(a, b, dt, p, st);
        }
    }
    if constexpr (kI8) {
        return p.fp8 ? dispatch_shape<true, 128>(a, b, dt, p, st, sh) : dispatch_shape<true, 0>(a, b, dt, p, st, sh);
    } else {
        switch (layout) {
            case 0: return dispatch_shape<false, 0>(a, b, dt, p, st, sh);
            case 2: return dispatch_shape<false, 2>(a, b, dt, p, st, sh);
            case 3: return dispatch_shape<false, 3>(a, b, dt, p, st, sh);
            default: return set_error(QSYNC_ERR_DOMAIN, "unsupported operand layout " + std::to_string(layout));
        }
    }
}

// TF32 (K-major) GEMM: single-CTA tiles by the same cost models (a 128-byte
// K-slice is 32 TF32 elements, the MMA time per slice equals the FP16 one).
int dispatch_tf32(const void* a, const void* b, EpiParams p, cudaStream_t st, int force_bn) {
    const bool accumulating = p.accumulate && p.c_dtype == QSYNC_F32;
    Shape sh = pick_shape(p.M, p.N, false);
    if (accumulating && !force_bn && g_force_splitk == 0) {
        const AccChoice c = choose_acc(p.M, p.N, (p.K + 31) / 32);
        sh.bn = c.bn;
        p.ksplit = c.ksplit;
    } else if (accumulating) {
        sh.bn = 256;
    }
    if (force_bn) sh.bn = force_bn;
    p.idesc = make_idesc(false, false, sh.bn, BM, 0, false, true);
    p.debug_epi = g_debug_epi;
    const CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    switch (sh.bn) {
        case 256: return launch<false, 256, 1, 256>(a, b, dt, p, st);
        case 192: return launch<false, 192, 1, 256>(a, b, dt, p, st);
        case 128: return launch<false, 128, 1, 256>(a, b, dt, p, st);
        default: return launch<false, 64, 1, 256>(a, b, dt, p, st);
    }
}

// 3xTF32 operand split: x = hi + lo + r with hi = rna_tf32(x), lo =
// rna_tf32(x - hi) (|r| <= 2^-22 |x|).  out [R, 3K] holds the parts along K in
// the order (hi, hi, lo) for A or (hi, lo, hi) for B, so ONE TF32 GEMM over
// K' = 3Kp computes hi_a hi_b + hi_a lo_b + lo_a hi_b -- FP32-level accuracy on
// the tensor cores (each part zero-padded from K to Kp = K rounded up to 4).
// transpose = 1 reads x as [K, R] (an MN-major source) and writes the K-major
// parts through a 32 x 33 smem tile.
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__global__ void __launch_bounds__(256) k_split_tf32(const float* __restrict__ x, int64_t R, int64_t K, int64_t Kp,
                                                    int transpose, int order, float* __restrict__ out) {
    QSB_PDL_ENTER();
    __shared__ float tile[32][33];
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, k0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
    float v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int rr = ty + 8 * i;
        if (transpose) {  // x [K, R]: coalesced along R, stored transposed
            const int64_t kk = k0 + rr, r = r0 + tx;
            tile[rr][tx] = (kk < K && r < R) ? x[kk * R + r] : 0.0f;
        } else {
            const int64_t r = r0 + rr, kk = k0 + tx;
            v[i] = (r < R && kk < K) ? x[r * K + kk] : 0.0f;
        }
    }
    if (transpose) {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = tile[tx][ty + 8 * i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = r0 + ty + 8 * i, kk = k0 + tx;
        if (r >= R || kk >= Kp) continue;  // columns K..Kp-1: zero padding of each part
        const float hi = tf32_rna(v[i]);
        const float lo = tf32_rna(v[i] - hi);
        float* o = out + r * 3 * Kp + kk;
        o[0] = hi;
        o[Kp] = order ? lo : hi;
        o[2 * Kp] = order ? hi : lo;
    }
}

// Each split part is K padded to a multiple of 4 elements (16-byte TMA rows).
inline int64_t tf32_part(int64_t k) { return (k + 3) / 4 * 4; }

int g_force_bn = 0;  // test hook (qsync_gemm_force_tile_n)

int validate(const void* a, const void* b, int64_t m, int64_t n, int64_t k, int64_t k_align) {
    QSB_REQUIRE(a && b, QSYNC_ERR_VALIDATION, "null GEMM operand");
    QSB_REQUIRE(m > 0 && n > 0 && k > 0, QSYNC_ERR_DOMAIN, "GEMM extents must be positive");
    QSB_REQUIRE(k % k_align == 0, QSYNC_ERR_DOMAIN,
                "GEMM K must be a multiple of " + std::to_string(k_align) +
                    " (16-byte TMA row pitch); pad K");
    QSB_REQUIRE((reinterpret_cast<uintptr_t>(a) & 15) == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0,
                QSYNC_ERR_DOMAIN, "GEMM operands must be 16-byte aligned");
    QSB_REQUIRE(m < (int64_t(1) << 31) && n < (int64_t(1) << 31) && k < (int64_t(1) << 31),
                QSYNC_ERR_DOMAIN, "GEMM extent too large");
    return QSYNC_OK;
}

}  // namespace

// 2-D SWIZZLE_128B tensor map for kernels outside this file (attention core).
int make_tma_2d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, uint32_t elem_bytes, int64_t inner,
                int64_t outer, uint32_t box_inner, uint32_t box_outer) {
    return make_map(map, ptr, dt, elem_bytes, inner, outer, box_inner, box_outer);
}
}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_gemm_force_splitk(int ks) {
    QSB_REQUIRE(ks >= 0 && ks <= 64, QSYNC_ERR_DOMAIN, "split-K override must be in [0, 64]");
    g_force_splitk = ks;
    return QSYNC_OK;
}

// A/B hook (QSB_GEMM_TRACE builds): device buffer of 72 uint64 per CTA for
// the phase timeline; nullptr turns tracing off.  No-op in normal builds.
int qsync_gemm_trace_buffer(void* buf) {
#ifdef QSB_GEMM_TRACE
    unsigned long long* p = static_cast<unsigned long long*>(buf);
    QSB_TRY(cuda_status(cudaMemcpyToSymbol(g_gemm_trace, &p, sizeof(p)), "cudaMemcpyToSymbol"));
    return QSYNC_OK;
#else
    (void)buf;
    return set_error(QSYNC_ERR_DOMAIN, "library built without QSB_GEMM_TRACE");
#endif
}

int qsync_gemm_set_max_ctas(int n) {
    QSB_REQUIRE(n >= 0, QSYNC_ERR_DOMAIN, "CTA cap must be >= 0");
    g_max_ctas = n;
    return QSYNC_OK;
}

int qsync_conv_set_impl(int tma) {
    g_conv_tma = tma ? 1 : 0;
    return QSYNC_OK;
}

int qsync_gemm_set_pdl(int on) {
    g_pdl = on ? 1 : 0;
    g_pdl_enabled = g_pdl;
    return QSYNC_OK;
}

int qsync_gemm_debug_epilogue(int v) {
    g_debug_epi = v;
    return QSYNC_OK;
}

int qsync_gemm_set_streamk(int mode) {
    QSB_REQUIRE(mode >= -1 && mode <= 1, QSYNC_ERR_DOMAIN, "stream-K mode must be -1 (never), 0 (cost model) or 1");
    g_streamk = mode;
    return QSYNC_OK;
}

int qsync_gemm_set_dual(int on) {
    g_dual = on ? 1 : 0;
    return QSYNC_OK;
}

int qsync_gemm_force_cta(int cta) {
    QSB_REQUIRE(cta >= 0 && cta <= 2, QSYNC_ERR_DOMAIN, "CTA override must be 0, 1 or 2");
    g_force_cta = cta;
    return QSYNC_OK;
}

int qsync_gemm_force_tile_n(int bn) {
    QSB_REQUIRE(bn == 0 || bn == 64 || bn == 128 || bn == 192 || bn == 256, QSYNC_ERR_DOMAIN,
                "tile N must be 0/64/128/192/256");
    g_force_bn = bn;
    return QSYNC_OK;
}

int qsync_gemm_f8(const uint8_t* a, const uint8_t* b, int64_t m, int64_t n, int64_t k, void* c, int c_dtype,
                  const float* scale_a, const float* scale_b, int b_per_channel, const float* bias,
                  qsync_stream_t stream) {
    QSB_TRY(validate(a, b, m, n, k, 16));
    QSB_REQUIRE(c != nullptr, QSYNC_ERR_VALIDATION, "GEMM needs an output");
    QSB_REQUIRE(c_dtype == QSYNC_F32 || c_dtype == QSYNC_F16 || c_dtype == QSYNC_BF16, QSYNC_ERR_DOMAIN,
                "FP8 GEMM epilogue output must be F32, F16 or BF16");
    QSB_REQUIRE(scale_a && scale_b, QSYNC_ERR_VALIDATION, "the dequant epilogue needs scale_a and scale_b");
    EpiParams p{};
    p.M = m;
    p.N = n;
    p.K = k;
    p.c = c;
    p.c_dtype = c_dtype;
    p.scale_a = scale_a;
    p.scale_b = scale_b;
    p.b_per_channel = b_per_channel;
    p.bias = bias;
    p.alpha = 1.0f;
    p.fp8 = 1;
    return dispatch<true>(a, b, CU_TENSOR_MAP_DATA_TYPE_UINT8, p, to_stream(stream), g_force_bn);
}

int qsync_gemm_s8_ex(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k, void* c,
                     int c_dtype, const float* scale_a, const float* scale_b, int b_per_channel,
                     const float* bias, qsync_stream_t stream) {
    QSB_TRY(validate(a, b, m, n, k, 16));
    QSB_REQUIRE(c != nullptr, QSYNC_ERR_VALIDATION, "GEMM needs an output");
    QSB_REQUIRE(c_dtype == QSYNC_F32 || c_dtype == QSYNC_F16 || c_dtype == QSYNC_BF16, QSYNC_ERR_DOMAIN,
                "INT8 GEMM epilogue output must be F32, F16 or BF16");
    QSB_REQUIRE(scale_a && scale_b, QSYNC_ERR_VALIDATION, "the dequant epilogue needs scale_a and scale_b");
    EpiParams p{};
    p.M = m;
    p.N = n;
    p.K = k;
    p.c = c;
    p.c_dtype = c_dtype;
    p.scale_a = scale_a;
    p.scale_b = scale_b;
    p.b_per_channel = b_per_channel;
    p.bias = bias;
    p.alpha = 1.0f;
    return dispatch<true>(a, b, CU_TENSOR_MAP_DATA_TYPE_UINT8, p, to_stream(stream), g_force_bn);
}

int qsync_gemm_gelu(const void* a, const void* b, int ab_dtype, int64_t m, int64_t n, int64_t k,
                    const float* scale_a, const float* scale_b, int b_per_channel, const float* bias, void* g,
                    int g_dtype, uint16_t* dact, float* absmax, qsync_stream_t stream) {
    QSB_REQUIRE(ab_dtype == QSYNC_I8 || ab_dtype == QSYNC_F16 || ab_dtype == QSYNC_BF16, QSYNC_ERR_DOMAIN,
                "GELU GEMM operands must be I8, F16 or BF16");
    const bool i8 = ab_dtype == QSYNC_I8;
    QSB_TRY(validate(a, b, m, n, k, i8 ? 16 : 8));
    QSB_REQUIRE(g && dact && absmax, QSYNC_ERR_VALIDATION, "GELU GEMM needs g, dact and absmax");
    QSB_REQUIRE(g_dtype == QSYNC_F32 || g_dtype == QSYNC_F16, QSYNC_ERR_DOMAIN, "GELU GEMM output must be F32 or F16");
    QSB_REQUIRE(n % 8 == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(dact) & 15) == 0,
                QSYNC_ERR_DOMAIN, "GELU GEMM needs N % 8 == 0 and 16-byte aligned outputs (TMA stores)");
    QSB_REQUIRE(!i8 || (scale_a && scale_b), QSYNC_ERR_VALIDATION, "the dequant epilogue needs scale_a and scale_b");
    EpiParams p{};
    p.M = m;
    p.N = n;
    p.K = k;
    p.c = g;
    p.c_dtype = g_dtype;
    p.scale_a = i8 ? scale_a : nullptr;
    p.scale_b = i8 ? scale_b : nullptr;
    p.b_per_channel = b_per_channel;
    p.bias = bias;
    p.alpha = 1.0f;
    p.dact = dact;
    p.act_absmax = reinterpret_cast<unsigned*>(absmax);
    QSB_TRY(zero_async(absmax, sizeof(float), to_stream(stream)));
    if (i8) return dispatch<true>(a, b, CU_TENSOR_MAP_DATA_TYPE_UINT8, p, to_stream(stream), g_force_bn, 512);
    const CUtensorMapDataType dt =
        ab_dtype == QSYNC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    return dispatch<false>(a, b, dt, p, to_stream(stream), g_force_bn, 512);
}

int qsync_gemm_s8_ymax(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k, float* c,
                       const float* scale_a, const float* scale_b, int b_per_channel, const float* bias, float* ymax,
                       qsync_stream_t stream) {
    QSB_TRY(validate(a, b, m, n, k, 16));
    QSB_REQUIRE(c != nullptr && ymax != nullptr, QSYNC_ERR_VALIDATION, "GEMM needs an output and ymax");
    QSB_REQUIRE(scale_a && scale_b, QSYNC_ERR_VALIDATION, "the dequant epilogue needs scale_a and scale_b");
    EpiParams p{};
    p.M = m;
    p.N = n;
    p.K = k;
    p.c = c;
    p.c_dtype = QSYNC_F32;
    p.scale_a = scale_a;
    p.scale_b = scale_b;
    p.b_per_channel = b_per_channel;
    p.bias = bias;
    p.alpha = 1.0f;
    p.ymax = reinterpret_cast<unsigned*>(ymax);
    cudaStream_t st = to_stream(stream);
    QSB_TRY(zero_async(ymax, sizeof(float), st));
    return dispatch<true>(a, b, CU_TENSOR_MAP_DATA_TYPE_UINT8, p, st, g_force_bn, 4096);
}

int qsync_gemm_s8(const int8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k,
                  int32_t* c_i32, float* c_f32, const float* scale_a, const float* scale_b,
                  int b_per_channel, const float* bias, qsync_stream_t stream) {
    QSB_TRY(validate(a, b, m, n, k, 16));
    QSB_REQUIRE(c_i32 || c_f32, QSYNC_ERR_VALIDATION, "GEMM needs an output");
    QSB_REQUIRE(!c_f32 || (scale_a && scale_b), QSYNC_ERR_VALIDATION,
                "the dequant epilogue needs scale_a and scale_b");
    EpiParams p{};
    p.M = m;
    p.N = n;
    p.K = k;
    p.c_i32 = c_i32;
    p.c = c_f32;
    p.c_dtype = QSYNC_F32;
    p.scale_a = scale_a;
    p.scale_b = scale_b;
    p.b_per_channel = b_per_channel;
    p.bias = bias;
    p.alpha = 1.0f;
    return dispatch<true>(a, b, CU_TENSOR_MAP_DATA_TYPE_UINT8, p, to_stream(stream), g_force_bn);
}

int qsync_conv_fwd_implicit(const void* x, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R,
                            int S, int sh, int sw, int ph, int pw, const void* w, int64_t cout, void* y,
                            int y_dtype, const float* scale_a, const float* scale_b, int b_per_channel,
                            const float* bias, qsync_stream_t stream) {
    QSB_REQUIRE(x && w && y, QSYNC_ERR_VALIDATION, "implicit conv needs x, w and y");
    QSB_REQUIRE(dtype == QSYNC_I8 || dtype == QSYNC_F16 || dtype == QSYNC_BF16, QSYNC_ERR_DOMAIN,
                "implicit conv input must be I8, F16 or BF16");
    const int eb = dtype == QSYNC_I8 ? 1 : 2;
    QSB_REQUIRE(N > 0 && H > 0 && W > 0 && C > 0 && R > 0 && S > 0 && sh > 0 && sw > 0 && ph >= 0 && pw >= 0,
                QSYNC_ERR_DOMAIN, "bad conv geometry");
    QSB_REQUIRE((C * eb) % 64 == 0, QSYNC_ERR_DOMAIN,
                "implicit conv needs C * element size to be a multiple of 64 bytes (use im2col)");
    const int64_t P = (H + 2 * ph - R) / sh + 1, Q = (W + 2 * pw - S) / sw + 1;
    QSB_REQUIRE(P > 0 && Q > 0, QSYNC_ERR_DOMAIN, "conv output would be empty");
    const int64_t M = N * P * Q, K = static_cast<int64_t>(R) * S * C;
    QSB_REQUIRE(M < (int64_t(1) << 31) && N * H * W * C * eb < (int64_t(1) << 40), QSYNC_ERR_DOMAIN,
                "conv too large");
    QSB_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0,
                QSYNC_ERR_DOMAIN, "implicit conv operands must be 16-byte aligned");
    QSB_REQUIRE(y_dtype == QSYNC_F32 || y_dtype == QSYNC_F16 || y_dtype == QSYNC_BF16, QSYNC_ERR_DOMAIN,
                "conv output must be F32, F16 or BF16");
    EpiParams p{};
    p.M = M;
    p.N = cout;
    p.K = K;
    p.c = y;
    p.c_dtype = y_dtype;
    p.bias = bias;
    p.alpha = 1.0f;
    p.cx = static_cast<const uint8_t*>(x);
    p.cN = static_cast<int>(N); p.cH = static_cast<int>(H); p.cW = static_cast<int>(W);
    p.cC = static_cast<int>(C); p.cP = static_cast<int>(P); p.cQ = static_cast<int>(Q);
    p.cR = R; p.cS = S; p.csh = sh; p.csw = sw; p.cph = ph; p.cpw = pw;
    p.ctap = 1; p.cdvh = 1; p.cdvw = 1;
    // 64-byte channel runs go through the gather lanes (two taps per 128-byte K-slice)
    const int lay = (g_conv_tma && (C * eb) % BK_BYTES == 0) ? 32 : 4;
    if (dtype == QSYNC_I8) {
        QSB_REQUIRE(scale_a && scale_b, QSYNC_ERR_VALIDATION, "the dequant epilogue needs scale_a and scale_b");
        p.scale_a = scale_a;
        p.scale_b = scale_b;
        p.b_per_channel = b_per_channel;
        return dispatch<true>(x, w, CU_TENSOR_MAP_DATA_TYPE_UINT8, p, to_stream(stream), g_force_bn, lay);
    }
    const CUtensorMapDataType dt =
        dtype == QSYNC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    return dispatch<false>(x, w, dt, p, to_stream(stream), g_force_bn, lay);
}

int qsync_conv_dgrad_implicit(const void* dy, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R,
                              int S, int sh, int sw, int ph, int pw, const void* w, int64_t cout, void* dx,
                              int dx_dtype, qsync_stream_t stream) {
    QSB_REQUIRE(dy && w && dx, QSYNC_ERR_VALIDATION, "implicit conv dgrad needs dy, w and dx");
    QSB_REQUIRE(dtype == QSYNC_F16 || dtype == QSYNC_BF16, QSYNC_ERR_DOMAIN,
                "implicit conv dgrad operands must be F16 or BF16");
    QSB_REQUIRE(N > 0 && H > 0 && W > 0 && C > 0 && R > 0 && S > 0 && sh > 0 && sw > 0 && ph >= 0 && pw >= 0,
                QSYNC_ERR_DOMAIN, "bad conv geometry");
    QSB_REQUIRE((cout * 2) % BK_BYTES == 0, QSYNC_ERR_DOMAIN,
                "implicit conv dgrad needs Cout % 64 == 0 (use col2im)");
    QSB_REQUIRE(C % 8 == 0, QSYNC_ERR_DOMAIN, "implicit conv dgrad needs C % 8 == 0 (16-byte weight rows)");
    const int64_t P = (H + 2 * ph - R) / sh + 1, Q = (W + 2 * pw - S) / sw + 1;
    QSB_REQUIRE(P > 0 && Q > 0, QSYNC_ERR_DOMAIN, "conv output would be empty");
    const int64_t M = N * H * W, K = static_cast<int64_t>(R) * S * cout;
    QSB_REQUIRE(M < (int64_t(1) << 31) && N * P * Q * cout * 2 < (int64_t(1) << 40), QSYNC_ERR_DOMAIN,
                "conv too large");
    QSB_REQUIRE((reinterpret_cast<uintptr_t>(dy) & 15) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0,
                QSYNC_ERR_DOMAIN, "implicit conv operands must be 16-byte aligned");
    QSB_REQUIRE(dx_dtype == QSYNC_F32 || dx_dtype == QSYNC_F16 || dx_dtype == QSYNC_BF16, QSYNC_ERR_DOMAIN,
                "conv dgrad output must be F32, F16 or BF16");
    // dX[(n,h,w), c] = sum_{r,s,k} dY[n, (h+ph-r)/sh, (w+pw-s)/sw, k] W[k,r,s,c]
    // (terms whose numerators are off the stride grid or out of range vanish).
    EpiParams p{};
    p.M = M;
    p.N = C;
    p.K = K;
    p.c = dx;
    p.c_dtype = dx_dtype;
    p.alpha = 1.0f;
    p.cx = static_cast<const uint8_t*>(dy);
    p.cN = static_cast<int>(N); p.cH = static_cast<int>(P); p.cW = static_cast<int>(Q);
    p.cC = static_cast<int>(cout); p.cP = static_cast<int>(H); p.cQ = static_cast<int>(W);
    p.cR = R; p.cS = S; p.csh = 1; p.csw = 1;
    const CUtensorMapDataType dt =
        dtype == QSYNC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    if (g_conv_tma && sh == 1 && sw == 1) {
        // a stride-1 conv of dY with pad (k-1-p) and flipped taps: TMA im2col
        p.cph = R - 1 - ph; p.cpw = S - 1 - pw;
        p.ctap = 1; p.cdvh = 1; p.cdvw = 1;
        return dispatch<false>(dy, w, dt, p, to_stream(stream), g_force_bn, 50);
    }
    p.cph = -ph; p.cpw = -pw;
    p.ctap = -1; p.cdvh = sh; p.cdvw = sw;
    return dispatch<false>(dy, w, dt, p, to_stream(stream), g_force_bn, 22);
}

int qsync_conv_wgrad_implicit(const void* x, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int R,
                              int S, int sh, int sw, int ph, int pw, const void* dy, int64_t cout, float* dw,
                              float alpha, const float* alpha_dev, int accumulate, qsync_stream_t stream) {
    QSB_REQUIRE(x && dy && dw, QSYNC_ERR_VALIDATION, "implicit conv wgrad needs x, dy and dw");
    QSB_REQUIRE(dtype == QSYNC_F16 || dtype == QSYNC_BF16, QSYNC_ERR_DOMAIN,
                "implicit conv wgrad operands must be F16 or BF16");
    QSB_REQUIRE(N > 0 && H > 0 && W > 0 && C > 0 && R > 0 && S > 0 && sh > 0 && sw > 0 && ph >= 0 && pw >= 0,
                QSYNC_ERR_DOMAIN, "bad conv geometry");
    QSB_REQUIRE((C * 2) % BK_BYTES == 0, QSYNC_ERR_DOMAIN,
                "implicit conv wgrad needs C % 64 == 0 (use im2col)");
    QSB_REQUIRE(cout % 8 == 0, QSYNC_ERR_DOMAIN, "implicit conv wgrad needs Cout % 8 == 0");
    const int64_t P = (H + 2 * ph - R) / sh + 1, Q = (W + 2 * pw - S) / sw + 1;
    QSB_REQUIRE(P > 0 && Q > 0, QSYNC_ERR_DOMAIN, "conv output would be empty");
    const int64_t M = cout, K = N * P * Q, Ncol = static_cast<int64_t>(R) * S * C;
    QSB_REQUIRE(K < (int64_t(1) << 31) && N * H * W * C * 2 < (int64_t(1) << 40), QSYNC_ERR_DOMAIN,
                "conv too large");
    QSB_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(dy) & 15) == 0,
                QSYNC_ERR_DOMAIN, "implicit conv operands must be 16-byte aligned");
    // dW[k, (r,s,c)] (+)= alpha * sum_{(n,p,q)} dY[(n,p,q), k] x[n, p*sh-ph+r, q*sw-pw+s, c]
    EpiParams p{};
    p.M = M;
    p.N = Ncol;
    p.K = K;
    p.c = dw;
    p.c_dtype = QSYNC_F32;
    p.alpha = alpha;
    p.alpha_dev = alpha_dev;
    p.accumulate = accumulate;
    p.cx = static_cast<const uint8_t*>(x);
    p.cN = static_cast<int>(N); p.cH = static_cast<int>(H); p.cW = static_cast<int>(W);
    p.cC = static_cast<int>(C); p.cP = static_cast<int>(P); p.cQ = static_cast<int>(Q);
    p.cR = R; p.cS = S; p.csh = sh; p.csw = sw; p.cph = ph; p.cpw = pw;
    p.ctap = 1; p.cdvh = 1; p.cdvw = 1;
    const CUtensorMapDataType dt =
        dtype == QSYNC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    return dispatch<false>(dy, x, dt, p, to_stream(stream), 256, g_conv_tma ? 67 : 11);
}

int qsync_split_tf32x3(const float* x, int64_t rows, int64_t k, int transpose, int order, float* out,
                       qsync_stream_t stream) {
    QSB_REQUIRE(x && out, QSYNC_ERR_VALIDATION, "split needs x and out");
    QSB_REQUIRE(rows >= 0 && k >= 0, QSYNC_ERR_DOMAIN, "negative extent");
    QSB_REQUIRE(rows < (int64_t(1) << 31) && k < (int64_t(1) << 31), QSYNC_ERR_DOMAIN, "split extent too large");
    if (rows == 0 || k == 0) return QSYNC_OK;
    const int64_t kp = tf32_part(k);
    dim3 grid(static_cast<unsigned>((kp + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
    QSB_REQUIRE(grid.y < 65536, QSYNC_ERR_DOMAIN, "too many rows for the split grid");
    pdl_launch(k_split_tf32, grid, dim3(256), 0, to_stream(stream), x, rows, k, kp, transpose, order, out);
    return check_launch("k_split_tf32");
}

int qsync_gemm_tf32(const float* a, const float* b, int64_t m, int64_t n, int64_t k, float* c, float alpha,
                    const float* alpha_dev, const float* bias, int accumulate, qsync_stream_t stream) {
    QSB_TRY(validate(a, b, m, n, k, 4));
    QSB_REQUIRE(c != nullptr, QSYNC_ERR_VALIDATION, "GEMM needs an output");
    EpiParams p{};
    p.M = m;
    p.N = n;
    p.K = k;
    p.c = c;
    p.c_dtype = QSYNC_F32;
    p.alpha = alpha;
    p.alpha_dev = alpha_dev;
    p.bias = bias;
    p.accumulate = accumulate;
    return dispatch_tf32(a, b, p, to_stream(stream), g_force_bn);
}

size_t qsync_gemm_f32_workspace_bytes(int64_t m, int64_t n, int64_t k) {
    const int64_t kp = tf32_part(k);
    return static_cast<size_t>(3) * 4 * static_cast<size_t>(m * kp + n * kp) + 256;
}

int qsync_gemm_f32(const float* a, const float* b, int64_t m, int64_t n, int64_t k, float* c, float alpha,
                   const float* alpha_dev, const float* bias, int accumulate, int layout, void* workspace,
                   qsync_stream_t stream) {
    QSB_REQUIRE(layout == 0 || layout == 2 || layout == 3, QSYNC_ERR_DOMAIN,
                "operand layout must be 0 (K-major A/B), 2 (MN-major B) or 3 (MN-major A and B)");
    QSB_REQUIRE(a && b && c && workspace, QSYNC_ERR_VALIDATION, "FP32 GEMM needs a, b, c and the workspace");
    QSB_REQUIRE(m > 0 && n > 0 && k > 0, QSYNC_ERR_DOMAIN, "GEMM extents must be positive");
    const int64_t kp = tf32_part(k);
    float* a3 = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(workspace) + 127) & ~uintptr_t(127));
    float* b3 = a3 + ((3 * m * kp + 31) / 32) * 32;
    cudaStream_t st = to_stream(stream);
    QSB_TRY(qsync_split_tf32x3(a, m, k, (layout & 1) ? 1 : 0, 0, a3, st));
    QSB_TRY(qsync_split_tf32x3(b, n, k, (layout & 2) ? 1 : 0, 1, b3, st));
    return qsync_gemm_tf32(a3, b3, m, n, 3 * kp, c, alpha, alpha_dev, bias, accumulate, st);
}

int qsync_gemm_f16(const void* a, const void* b, int ab_dtype, int64_t m, int64_t n, int64_t k,
                   void* c, int c_dtype, float alpha, const float* alpha_dev, const float* bias,
                   int accumulate, int layout, qsync_stream_t stream) {
    QSB_REQUIRE(layout == 0 || layout == 2 || layout == 3, QSYNC_ERR_DOMAIN,
                "operand layout must be 0 (K-major A/B), 2 (MN-major B) or 3 (MN-major A and B)");
    // 16-byte TMA row pitch: the contiguous extent of each operand.
    QSB_TRY(validate(a, b, m, n, k, (layout & 3) == 3 ? 1 : 8));
    QSB_REQUIRE(!(layout & 1) || m % 8 == 0, QSYNC_ERR_DOMAIN, "MN-major A needs M % 8 == 0");
    QSB_REQUIRE(!(layout & 2) || n % 8 == 0, QSYNC_ERR_DOMAIN, "MN-major B needs N % 8 == 0");
    QSB_REQUIRE(c != nullptr, QSYNC_ERR_VALIDATION, "GEMM needs an output");
    QSB_REQUIRE(ab_dtype == QSYNC_F16 || ab_dtype == QSYNC_BF16, QSYNC_ERR_DOMAIN,
                "FP16 GEMM operands must be F16 or BF16");
    QSB_REQUIRE(c_dtype == QSYNC_F32 || c_dtype == QSYNC_F16 || c_dtype == QSYNC_BF16,
                QSYNC_ERR_DOMAIN, "FP16 GEMM output must be F32, F16 or BF16");
    EpiParams p{};
    p.M = m;
    p.N = n;
    p.K = k;
    p.c = c;
    p.c_dtype = c_dtype;
    p.alpha = alpha;
    p.alpha_dev = alpha_dev;
    p.bias = bias;
    p.accumulate = accumulate;
    const CUtensorMapDataType dt =
        ab_dtype == QSYNC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    return dispatch<false>(a, b, dt, p, to_stream(stream), g_force_bn, layout);
}

}  // extern "C"

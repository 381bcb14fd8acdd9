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
#include <mutex>

#include "common.cuh"
#include "ptx.cuh"

namespace qsb {

namespace {

constexpr int BM = 128;             // UMMA M (cta_group::1)
constexpr int BK_BYTES = 128;       // one 128B swizzle row per stage
constexpr int kThreads = 192;       // 6 warps
constexpr int kEpiWarp0 = 2;

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
};

template <int BN>
struct Cfg {
    static constexpr int kStageBytes = (BM + BN) * BK_BYTES;
    static constexpr int kStages = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
    static constexpr int kTmemCols = 2 * BN;  // two accumulator buffers
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float bits_f(uint32_t v) { return __uint_as_float(v); }

template <bool kI8, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
              const EpiParams p) {
    using C = Cfg<BN>;
    constexpr int kStages = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B swizzle atoms.
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
    uint8_t* smem_a = smem;                              // kStages x [BM rows x 128B]
    uint8_t* smem_b = smem + kStages * BM * BK_BYTES;    // kStages x [BN rows x 128B]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = bars + 2 * kStages + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    const int64_t M = p.M, N = p.N, K = p.K;
    const int num_m = static_cast<int>((M + BM - 1) / BM);
    const int num_n = static_cast<int>((N + BN - 1) / BN);
    const int num_tiles = num_m * num_n;
    const int bk_elems = kI8 ? BK_BYTES : BK_BYTES / 2;
    const int num_kb = static_cast<int>((K + bk_elems - 1) / bk_elems);

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tm_a);
        ptx::tma_prefetch(&tm_b);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 4 * 32);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                const int m0 = (t % num_m) * BM;
                const int n0 = (t / num_m) * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                    ptx::tma_load_2d(smem_a + stage * BM * BK_BYTES, &tm_a, &full[stage],
                                     kb * bk_elems, m0);
                    ptx::tma_load_2d(smem_b + stage * BN * BK_BYTES, &tm_b, &full[stage],
                                     kb * bk_elems, n0);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(smem_a + stage * BM * BK_BYTES);
                    const uint32_t b_addr = ptx::smem_u32(smem_b + stage * BN * BK_BYTES);
#pragma unroll
                    for (int k = 0; k < BK_BYTES / 32; ++k) {  // UMMA_K = 32 bytes
                        const uint64_t da = ptx::sw128_kmajor_desc(a_addr + k * 32);
                        const uint64_t db = ptx::sw128_kmajor_desc(b_addr + k * 32);
                        const uint32_t accum = (kb | k) != 0 ? 1u : 0u;
                        if (kI8)
                            ptx::mma_i8(d_tmem, da, db, p.idesc, accum);
                        else
                            ptx::mma_f16(d_tmem, da, db, p.idesc, accum);
                    }
                    ptx::tc_commit(&empty[stage]);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::tc_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        // ===================== epilogue (warps 2..5) =====================
        const int quad = warp & 3;  // TMEM lane quadrant this warp may access
        int acc = 0;
        uint32_t acc_phase = 0;
        float alpha = p.alpha;
        if (p.alpha_dev) alpha *= *p.alpha_dev;
        const float sa = (kI8 && p.scale_a) ? *p.scale_a : 1.0f;
        const bool vec4 = (N % 4) == 0;
        const bool vec8 = (N % 8) == 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const int64_t m0 = static_cast<int64_t>(t % num_m) * BM;
            const int64_t n0 = static_cast<int64_t>(t / num_m) * BN;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const int64_t row = m0 + quad * 32 + lane;
            const bool row_ok = row < M;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                                       static_cast<uint32_t>(acc * BN + c0);
                ptx::tmem_ld32(taddr, r);
                ptx::tmem_ld_wait();
                const int64_t col0 = n0 + c0;
                if (!row_ok || col0 >= N) continue;
                const bool full_chunk = col0 + 32 <= N;
                if (p.c_i32) {
                    int32_t* dst = p.c_i32 + row * N + col0;
                    if (full_chunk && vec4) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            *reinterpret_cast<int4*>(dst + j) =
                                make_int4(static_cast<int>(r[j]), static_cast<int>(r[j + 1]),
                                          static_cast<int>(r[j + 2]), static_cast<int>(r[j + 3]));
                    } else {
                        for (int j = 0; j < 32 && col0 + j < N; ++j) dst[j] = static_cast<int>(r[j]);
                    }
                }
                if (!p.c) continue;
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int64_t col = col0 + j;
                    const int64_t cc = col < N ? col : N - 1;
                    float x;
                    if (kI8) {
                        const float sb = p.scale_b ? (p.b_per_channel ? p.scale_b[cc] : *p.scale_b) : 1.0f;
                        x = __fmul_rn(__int2float_rn(static_cast<int>(r[j])), __fmul_rn(sa, sb));
                    } else {
                        x = __fmul_rn(bits_f(r[j]), alpha);
                    }
                    if (p.bias) x = __fadd_rn(x, p.bias[cc]);
                    v[j] = x;
                }
                if (p.c_dtype == QSYNC_F32) {
                    float* dst = static_cast<float*>(p.c) + row * N + col0;
                    if (full_chunk && vec4) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                            if (p.accumulate) {
                                const float4 old = *reinterpret_cast<const float4*>(dst + j);
                                o.x += old.x;
                                o.y += old.y;
                                o.z += old.z;
                                o.w += old.w;
                            }
                            *reinterpret_cast<float4*>(dst + j) = o;
                        }
                    } else {
                        for (int j = 0; j < 32 && col0 + j < N; ++j)
                            dst[j] = p.accumulate ? dst[j] + v[j] : v[j];
                    }
                } else {
                    // 16-bit outputs (FP16 op outputs, FP16 dgrad).
                    uint16_t* dst = static_cast<uint16_t*>(p.c) + row * N + col0;
                    const bool bf = p.c_dtype == QSYNC_BF16;
                    auto cvt = [bf](float f) -> uint16_t {
                        return bf ? __bfloat16_as_ushort(__float2bfloat16_rn(f))
                                  : __half_as_ushort(__float2half_rn(f));
                    };
                    auto back = [bf](uint16_t h) -> float {
                        return bf ? __bfloat162float(__ushort_as_bfloat16(h))
                                  : __half2float(__ushort_as_half(h));
                    };
                    if (full_chunk && vec8 && !p.accumulate) {
#pragma unroll
                        for (int j = 0; j < 32; j += 8) {
                            uint4 o;
                            o.x = cvt(v[j]) | (static_cast<uint32_t>(cvt(v[j + 1])) << 16);
                            o.y = cvt(v[j + 2]) | (static_cast<uint32_t>(cvt(v[j + 3])) << 16);
                            o.z = cvt(v[j + 4]) | (static_cast<uint32_t>(cvt(v[j + 5])) << 16);
                            o.w = cvt(v[j + 6]) | (static_cast<uint32_t>(cvt(v[j + 7])) << 16);
                            *reinterpret_cast<uint4*>(dst + j) = o;
                        }
                    } else {
                        for (int j = 0; j < 32 && col0 + j < N; ++j)
                            dst[j] = cvt(p.accumulate ? back(dst[j]) + v[j] : v[j]);
                    }
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
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

// Instruction descriptor (tcgen05 "idesc"): c_format [4,6), a_format [7,10),
// b_format [10,13), a/b major [15],[16] (0 = K-major), N>>3 [17,23), M>>4 [24,29).
uint32_t make_idesc(bool i8, bool bf16, int n) {
    uint32_t d = 0;
    d |= (i8 ? 2u : 1u) << 4;                         // S32 / F32 accumulator
    const uint32_t fmt = i8 ? 1u : (bf16 ? 1u : 0u);  // signed int8 / BF16 / F16
    d |= fmt << 7;
    d |= fmt << 10;
    d |= static_cast<uint32_t>(n >> 3) << 17;
    d |= static_cast<uint32_t>(BM >> 4) << 24;
    return d;
}

template <bool kI8, int BN>
int launch(const void* a, const void* b, CUtensorMapDataType dt, EpiParams p, cudaStream_t st) {
    using C = Cfg<BN>;
    const uint32_t eb = kI8 ? 1 : 2;
    const uint32_t box_k = BK_BYTES / eb;
    CUtensorMap ma, mb;
    QSB_TRY(make_map(&ma, a, dt, eb, p.K, p.M, box_k, BM));
    QSB_TRY(make_map(&mb, b, dt, eb, p.K, p.N, box_k, BN));
    static bool configured = false;
    if (!configured) {
        QSB_TRY(cuda_status(cudaFuncSetAttribute(k_gemm_tc<kI8, BN>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 C::kSmemBytes),
                            "cudaFuncSetAttribute"));
        configured = true;
    }
    const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
    const int grid = static_cast<int>(std::min<int64_t>(tiles, sm_count()));
    k_gemm_tc<kI8, BN><<<grid, kThreads, C::kSmemBytes, st>>>(ma, mb, p);
    return check_launch("k_gemm_tc");
}

// Pick BN from {256, 128, 64} minimising (waves x per-tile cost), where the
// per-k-block cost is max(MMA cycles, smem operand bytes / 128 B per cycle).
int pick_bn(int64_t M, int64_t N) {
    const int sms = sm_count();
    const int cands[3] = {256, 128, 64};
    int best = 256;
    double best_cost = 1e300;
    for (int bn : cands) {
        const int64_t tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
        const int64_t waves = (tiles + sms - 1) / sms;
        const double mma = 4.0 * BM * bn / 256.0;
        const double smem = (BM + bn) * 128.0 / 128.0;
        const double cost = static_cast<double>(waves) * std::max(mma, smem);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = bn;
        }
    }
    return best;
}

template <bool kI8>
int dispatch(const void* a, const void* b, CUtensorMapDataType dt, EpiParams p, cudaStream_t st,
             int force_bn) {
    const int bn = force_bn ? force_bn : pick_bn(p.M, p.N);
    p.idesc = make_idesc(kI8, dt == CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, bn);
    switch (bn) {
        case 256: return launch<kI8, 256>(a, b, dt, p, st);
        case 128: return launch<kI8, 128>(a, b, dt, p, st);
        case 64: return launch<kI8, 64>(a, b, dt, p, st);
        default: return set_error(QSYNC_ERR_DOMAIN, "unsupported tile N " + std::to_string(bn));
    }
}

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
}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_gemm_force_tile_n(int bn) {
    QSB_REQUIRE(bn == 0 || bn == 64 || bn == 128 || bn == 256, QSYNC_ERR_DOMAIN, "tile N must be 0/64/128/256");
    g_force_bn = bn;
    return QSYNC_OK;
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

int qsync_gemm_f16(const void* a, const void* b, int ab_dtype, int64_t m, int64_t n, int64_t k,
                   void* c, int c_dtype, float alpha, const float* alpha_dev, const float* bias,
                   int accumulate, qsync_stream_t stream) {
    QSB_TRY(validate(a, b, m, n, k, 8));
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
    return dispatch<false>(a, b, dt, p, to_stream(stream), g_force_bn);
}

}  // extern "C"

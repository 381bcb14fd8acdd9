// attn.cu -- the encoder layer's attention core softmax(Q K^T * scale) V, forward
// and backward, FP16 in / FP16 out with FP32 softmax statistics.  QSync leaves
// this operator in floating point; it sits between the planned
// QKV and O projections, so its I/O is in their formats:
//   in : packed QKV [B, S, 3, H, D] FP16 (what the QKV projection emits)
//   out: O [B, S, H, D] FP16 (+ optional absmax(O) for an INT8 O projection)
//        and the row log-sum-exp [B, H, S] FP32 for the backward;
//   bwd: dQKV packed [B, S, 3, H, D] FP16 (the QKV projection's FP16 dY).
//
// Sequence length 128, head dim 64 (BERT-base): one CTA owns one (batch, head),
// the whole sequence fits on chip, so there is no online softmax and no
// atomics.  Three implementations (qsync_attention_set_impl):
//   impl 2 (default): tcgen05 -- TMA-loaded Q/K/V, S and O accumulated in TMEM,
//     thread-per-row softmax, P written in the K-major UMMA layout; the backward
//     (k_attn_bwd_tc2) runs five UMMA GEMMs at 2 CTAs/SM with P^T kept in TMEM;
//   impl 1: the same forward, a 1-CTA/SM tcgen05 backward (k_attn_bwd_tc);
//   impl 0: the first version, mma.sync m16n8k16 on ldmatrix fragments of
//     XOR-swizzled 128B-row tiles (8 warps; forward warp w owns query rows
//     16w..; backward phase 1 per key rows -> dV, dK, dS^T in smem; phase 2 per
//     query rows -> dQ), kept selectable for A/B and tested like the others.
// HBM traffic per (b, h): fwd 3 x 16 KB in, 16 KB out; bwd 5 x 16 KB in
// (Q, K, V, O, dO), 48 KB out.
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace qsb {
namespace {

constexpr int kS = 128;
constexpr int kD = 64;
constexpr int kThreadsA = 256;
constexpr int kTile = kS * kD * 2;  // bytes of one [128 x 64] FP16 tile
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// [rows x 64] FP16 tile, 128-byte rows of 8 chunks; chunk c of row r lives at c ^ (r & 7).
__device__ __forceinline__ uint32_t t64(uint32_t base, int r, int c) {
    return base + r * 128 + ((c ^ (r & 7)) << 4);
}
// [rows x 128] FP16 tile (256-byte rows, 16 chunks), same swizzle.
__device__ __forceinline__ uint32_t t128(uint32_t base, int r, int c) {
    return base + r * 256 + ((c ^ (r & 7)) << 4);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Copy a [128 x 64] FP16 tile (global row stride `rs` elements) into a swizzled smem tile.
__device__ __forceinline__ void load_tile(uint32_t sbase, const __half* g, int64_t rs) {
    for (int i = threadIdx.x; i < kS * 8; i += kThreadsA) {
        const int r = i >> 3, c = i & 7;
        cp_async16(t64(sbase, r, c), g + r * rs + c * 8);
    }
}

// A-operand fragments (16 x 16 at rows r0, k-step ks) of a row-major tile.
__device__ __forceinline__ void frag_a(uint32_t base, int r0, int ks, int lane, uint32_t (&a)[4]) {
    ldsm4(t64(base, r0 + (lane & 15), 2 * ks + (lane >> 4)), a);
}
// B-operand fragments for n-tiles n0 and n0+8 at k-step ks from a tile stored
// [n][k] (rows = n): {b0(n0), b1(n0), b0(n0+8), b1(n0+8)}.
__device__ __forceinline__ void frag_b_nk(uint32_t base, int n0, int ks, int lane, uint32_t (&b)[4]) {
    ldsm4(t64(base, n0 + (lane & 7) + ((lane >> 4) << 3), 2 * ks + ((lane >> 3) & 1)), b);
}
// B-operand fragments for n-tiles n0, n0+8 at k rows k0.. from a tile stored
// [k][n] (rows = k): transposing ldmatrix.
__device__ __forceinline__ void frag_b_kn(uint32_t base, int k0, int n0, int lane, uint32_t (&b)[4]) {
    ldsm4t(t64(base, k0 + (lane & 7) + (((lane >> 3) & 1) << 3), (n0 >> 3) + (lane >> 4)), b);
}

__device__ __forceinline__ uint32_t pk(float a, float b) { return pack_half2(a, b); }

// ---------------------------------------------------------------------------- forward
__global__ void __launch_bounds__(kThreadsA) k_attn_fwd(const __half* __restrict__ qkv, int H, float scale,
                                                        __half* __restrict__ out, float* __restrict__ lse,
                                                        unsigned* __restrict__ out_absmax) {
    QSB_PDL_ENTER();
    extern __shared__ __align__(128) uint8_t sm[];
    const int bh = blockIdx.x;
    const int b = bh / H, h = bh % H;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const uint32_t sQ = smem_addr(sm), sK = sQ + kTile, sV = sK + kTile;
    const int64_t rs = 3LL * H * kD;                         // packed row stride
    const __half* base = qkv + static_cast<int64_t>(b) * kS * rs + static_cast<int64_t>(h) * kD;
    // Q and K first; V streams in while Q K^T and the softmax run.
    load_tile(sQ, base, rs);
    load_tile(sK, base + H * kD, rs);
    cp_async_commit();
    load_tile(sV, base + 2 * H * kD, rs);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    const int m0 = warp * 16;
    uint32_t qa[4][4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) frag_a(sQ, m0, ks, lane, qa[ks]);
    float s[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
        for (int np = 0; np < 8; ++np) {
            uint32_t bf[4];
            frag_b_nk(sK, 16 * np, ks, lane, bf);
            mma16816(s[2 * np], qa[ks], bf[0], bf[1]);
            mma16816(s[2 * np + 1], qa[ks], bf[2], bf[3]);
        }
    }
    // Row softmax (rows g and g+8 of this warp's 16), scores scaled by `scale`.
    const float sl2 = scale * kLog2e;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
        mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    float sum0 = 0.f, sum1 = 0.f;
    uint32_t pa[8][4];  // P as A fragments (FP16), keys 16kk.. per k-step
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const float p0 = exp2f(s[j][0] * sl2 - mx0 * sl2), p1 = exp2f(s[j][1] * sl2 - mx0 * sl2);
        const float p2 = exp2f(s[j][2] * sl2 - mx1 * sl2), p3 = exp2f(s[j][3] * sl2 - mx1 * sl2);
        sum0 += p0 + p1;
        sum1 += p2 + p3;
        pa[j >> 1][(j & 1) * 2] = pk(p0, p1);
        pa[j >> 1][(j & 1) * 2 + 1] = pk(p2, p3);
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        sum0 += __shfl_xor_sync(0xffffffffu, sum0, o);
        sum1 += __shfl_xor_sync(0xffffffffu, sum1, o);
    }
    cp_async_wait<0>();
    __syncthreads();
    float oacc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        // pa[kk] = {row g keys 2t.., row g+8 keys 2t.., row g keys 8+2t.., row g+8 keys 8+2t..}
        const uint32_t a[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
#pragma unroll
        for (int np = 0; np < 4; ++np) {
            uint32_t bf[4];
            frag_b_kn(sV, 16 * kk, 16 * np, lane, bf);
            mma16816(oacc[2 * np], a, bf[0], bf[1]);
            mma16816(oacc[2 * np + 1], a, bf[2], bf[3]);
        }
    }
    const float inv0 = 1.f / sum0, inv1 = 1.f / sum1;
    const int64_t orow = static_cast<int64_t>(H) * kD;
    __half* o0 = out + (static_cast<int64_t>(b) * kS + m0 + g) * orow + static_cast<int64_t>(h) * kD;
    __half* o1 = o0 + 8 * orow;
    float amax = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t w0 = pk(oacc[j][0] * inv0, oacc[j][1] * inv0);
        const uint32_t w1 = pk(oacc[j][2] * inv1, oacc[j][3] * inv1);
        *reinterpret_cast<uint32_t*>(o0 + 8 * j + 2 * t) = w0;
        *reinterpret_cast<uint32_t*>(o1 + 8 * j + 2 * t) = w1;
        if (out_absmax) {
            const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&w0));
            const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&w1));
            amax = fmaxf(amax, fmaxf(fmaxf(fabsf(f0.x), fabsf(f0.y)), fmaxf(fabsf(f1.x), fabsf(f1.y))));
        }
    }
    if (t == 0) {
        float* l = lse + static_cast<int64_t>(bh) * kS + m0;
        l[g] = mx0 * scale + logf(sum0);
        l[g + 8] = mx1 * scale + logf(sum1);
    }
    if (out_absmax) {
        __shared__ float wm[8];
        amax = warp_max(amax);
        if (lane == 0) wm[warp] = amax;
        __syncthreads();
        if (threadIdx.x < 32) {
            amax = warp_max(threadIdx.x < 8 ? wm[threadIdx.x] : 0.f);
            if (threadIdx.x == 0 && amax > 0.f) atomicMax(out_absmax, __float_as_uint(amax));
        }
    }
}

// ---------------------------------------------------------------------------- backward
__global__ void __launch_bounds__(kThreadsA, 2) k_attn_bwd(const __half* __restrict__ qkv,
                                                        const __half* __restrict__ out,
                                                        const __half* __restrict__ dout,
                                                        const float* __restrict__ lse, int H, float scale,
                                                        __half* __restrict__ dqkv) {
    QSB_PDL_ENTER();
    extern __shared__ __align__(128) uint8_t sm[];
    const int bh = blockIdx.x;
    const int b = bh / H, h = bh % H;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const uint32_t sQ = smem_addr(sm), sK = sQ + kTile, sV = sK + kTile, sdO = sV + kTile;
    const uint32_t sdST = sdO + kTile;                              // [128 keys x 128 queries] FP16
    float* lse_s = reinterpret_cast<float*>(sm + 4 * kTile + 2 * kTile);
    float* d_s = lse_s + kS;
    const int64_t rs = 3LL * H * kD;
    const int64_t orow = static_cast<int64_t>(H) * kD;
    const __half* base = qkv + static_cast<int64_t>(b) * kS * rs + static_cast<int64_t>(h) * kD;
    const __half* obase = out + static_cast<int64_t>(b) * kS * orow + static_cast<int64_t>(h) * kD;
    const __half* dobase = dout + static_cast<int64_t>(b) * kS * orow + static_cast<int64_t>(h) * kD;
    load_tile(sQ, base, rs);
    load_tile(sK, base + H * kD, rs);
    load_tile(sV, base + 2 * H * kD, rs);
    load_tile(sdO, dobase, orow);
    // D[q] = sum_d dO[q, d] O[q, d]  (two threads per query row)
    {
        const int q = threadIdx.x >> 1, hf = threadIdx.x & 1;
        const uint4* op = reinterpret_cast<const uint4*>(obase + q * orow + hf * 32);
        const uint4* dp = reinterpret_cast<const uint4*>(dobase + q * orow + hf * 32);
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 ov = op[i], dv = dp[i];
            const __half2* oh = reinterpret_cast<const __half2*>(&ov);
            const __half2* dh = reinterpret_cast<const __half2*>(&dv);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 a = __half22float2(oh[e]), c = __half22float2(dh[e]);
                acc += a.x * c.x + a.y * c.y;
            }
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (hf == 0) d_s[q] = acc;
        if (threadIdx.x < kS) lse_s[threadIdx.x] = lse[static_cast<int64_t>(bh) * kS + threadIdx.x] * kLog2e;
    }
    cp_async_wait_all();
    __syncthreads();

    const float sl2 = scale * kLog2e;
    // ---- phase 1: warp w owns key rows k0 = 16w
    {
        const int k0 = warp * 16;
        float dv[8][4], dk[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            dv[j][0] = dv[j][1] = dv[j][2] = dv[j][3] = 0.f;
            dk[j][0] = dk[j][1] = dk[j][2] = dk[j][3] = 0.f;
        }
#pragma unroll 1
        for (int qc = 0; qc < 4; ++qc) {  // 32 queries per chunk (4 n-tiles)
            float st[4][4], dpt[4][4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                st[j][0] = st[j][1] = st[j][2] = st[j][3] = 0.f;
                dpt[j][0] = dpt[j][1] = dpt[j][2] = dpt[j][3] = 0.f;
            }
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                uint32_t ka[4], va[4];  // re-read per k-step: keeps the kernel at 2 CTAs / SM
                frag_a(sK, k0, ks, lane, ka);
                frag_a(sV, k0, ks, lane, va);
#pragma unroll
                for (int np = 0; np < 2; ++np) {
                    uint32_t bq[4], bo[4];
                    frag_b_nk(sQ, 32 * qc + 16 * np, ks, lane, bq);
                    frag_b_nk(sdO, 32 * qc + 16 * np, ks, lane, bo);
                    mma16816(st[2 * np], ka, bq[0], bq[1]);
                    mma16816(st[2 * np + 1], ka, bq[2], bq[3]);
                    mma16816(dpt[2 * np], va, bo[0], bo[1]);
                    mma16816(dpt[2 * np + 1], va, bo[2], bo[3]);
                }
            }
            // P^T = exp(S^T scale - lse[q]), dS^T = P^T (dP^T - D[q]); columns are queries.
            uint32_t pa[2][4], dsa[2][4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int q = 32 * qc + 8 * j + 2 * t;
                const float l0 = lse_s[q], l1 = lse_s[q + 1];
                const float d0 = d_s[q], d1 = d_s[q + 1];
                const float p0 = exp2f(st[j][0] * sl2 - l0), p1 = exp2f(st[j][1] * sl2 - l1);
                const float p2 = exp2f(st[j][2] * sl2 - l0), p3 = exp2f(st[j][3] * sl2 - l1);
                const float s0 = p0 * (dpt[j][0] - d0), s1 = p1 * (dpt[j][1] - d1);
                const float s2 = p2 * (dpt[j][2] - d0), s3 = p3 * (dpt[j][3] - d1);
                pa[j >> 1][(j & 1) * 2] = pk(p0, p1);
                pa[j >> 1][(j & 1) * 2 + 1] = pk(p2, p3);
                const uint32_t w01 = pk(s0, s1), w23 = pk(s2, s3);
                dsa[j >> 1][(j & 1) * 2] = w01;
                dsa[j >> 1][(j & 1) * 2 + 1] = w23;
                // dS^T rows k0+g, k0+g+8, columns q, q+1 -> shared [key][query]
                const int c = q >> 3, e = (q & 7) * 2;
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(t128(sdST, k0 + g, c) + e), "r"(w01));
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(t128(sdST, k0 + g + 8, c) + e), "r"(w23));
            }
            // dV += P^T dO, dK += dS^T Q over this chunk's 32 queries (2 k-steps).
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                const uint32_t ap[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
                const uint32_t as[4] = {dsa[kk][0], dsa[kk][1], dsa[kk][2], dsa[kk][3]};
                const int qr = 32 * qc + 16 * kk;
#pragma unroll
                for (int np = 0; np < 4; ++np) {
                    uint32_t bo[4], bq[4];
                    frag_b_kn(sdO, qr, 16 * np, lane, bo);
                    frag_b_kn(sQ, qr, 16 * np, lane, bq);
                    mma16816(dv[2 * np], ap, bo[0], bo[1]);
                    mma16816(dv[2 * np + 1], ap, bo[2], bo[3]);
                    mma16816(dk[2 * np], as, bq[0], bq[1]);
                    mma16816(dk[2 * np + 1], as, bq[2], bq[3]);
                }
            }
        }
        __half* dk0 = dqkv + (static_cast<int64_t>(b) * kS + k0 + g) * rs + H * kD + static_cast<int64_t>(h) * kD;
        __half* dv0 = dk0 + H * kD;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            *reinterpret_cast<uint32_t*>(dk0 + 8 * j + 2 * t) = pk(dk[j][0] * scale, dk[j][1] * scale);
            *reinterpret_cast<uint32_t*>(dk0 + 8 * rs + 8 * j + 2 * t) = pk(dk[j][2] * scale, dk[j][3] * scale);
            *reinterpret_cast<uint32_t*>(dv0 + 8 * j + 2 * t) = pk(dv[j][0], dv[j][1]);
            *reinterpret_cast<uint32_t*>(dv0 + 8 * rs + 8 * j + 2 * t) = pk(dv[j][2], dv[j][3]);
        }
    }
    __syncthreads();
    // ---- phase 2: warp w owns query rows m0 = 16w: dQ = dS K scale
    {
        const int m0 = warp * 16;
        float dq[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            // A = dS[m0.., keys 16kk..] read transposed from dS^T [key][query]
            uint32_t a[4];
            ldsm4t(t128(sdST, 16 * kk + (lane & 7) + ((lane >> 4) << 3), (m0 >> 3) + ((lane >> 3) & 1)), a);
#pragma unroll
            for (int np = 0; np < 4; ++np) {
                uint32_t bk[4];
                frag_b_kn(sK, 16 * kk, 16 * np, lane, bk);
                mma16816(dq[2 * np], a, bk[0], bk[1]);
                mma16816(dq[2 * np + 1], a, bk[2], bk[3]);
            }
        }
        __half* dq0 = dqkv + (static_cast<int64_t>(b) * kS + m0 + g) * rs + static_cast<int64_t>(h) * kD;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            *reinterpret_cast<uint32_t*>(dq0 + 8 * j + 2 * t) = pk(dq[j][0] * scale, dq[j][1] * scale);
            *reinterpret_cast<uint32_t*>(dq0 + 8 * rs + 8 * j + 2 * t) = pk(dq[j][2] * scale, dq[j][3] * scale);
        }
    }
}

// ---------------------------------------------------------------------------- tcgen05 forward
// One CTA (4 warps) per (batch, head), the two GEMMs on the 5th-generation tensor
// cores: Q, K, V land by TMA (128B swizzle) from the packed QKV; S = Q K^T
// (M = 128 queries, N = 128 keys, K = 64) accumulates in TMEM; thread t owns
// query row t (TMEM lane t), so the row softmax needs no shuffles; P (FP16) is
// written into shared memory in the K-major UMMA layout and O = P V (N = 64,
// K = 128, V read MN-major) accumulates in the same TMEM columns once S has been
// read out.  P overwrites Q and K (dead after S), so a CTA needs 48 KB of shared
// memory and 128 TMEM columns: 4 CTAs (4 heads) per SM.
constexpr int kTcThreads = 128;
constexpr int kTcFwdSmem = 3 * kTile + 1024 + 64;

__device__ __forceinline__ uint32_t idesc_f16_f32(int n, int m, bool b_mn) {
    uint32_t d = 1u << 4;                                // F32 accumulator; A/B F16
    d |= static_cast<uint32_t>(b_mn) << 16;              // B MN-major
    d |= static_cast<uint32_t>(n >> 3) << 17;
    d |= static_cast<uint32_t>(m >> 4) << 24;
    return d;
}

// kQ: the O projection is INT8 -- the forward also quantizes O per tensor (its
// INT8 operand + the FP16 copy of the grid values for its wgrad): per-block
// absmax partials, a grid barrier over the co-resident (batch, head) blocks,
// then each thread quantizes the O row it still holds in registers.  Same q,
// q16 and scale as qsync_attention_fwd + qsync_quantize_act_ex.
constexpr int kAttQSlots = 32;
constexpr int kAttQMaxBlocks = 4096;
__device__ float g_attq_part[kAttQSlots][kAttQMaxBlocks];
__device__ unsigned g_attq_bar[kAttQSlots][2];  // [0] arrivals, [1] generation

__device__ __forceinline__ void attq_grid_barrier(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g0 = *gen;  // cannot move before every block has arrived
        __threadfence();           // this block's partial before its arrival
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

template <bool kQ>
__global__ void __launch_bounds__(kTcThreads) k_attn_fwd_tc(const __grid_constant__ CUtensorMap tm_qkv, int H,
                                                            float scale, __half* __restrict__ out,
                                                            float* __restrict__ lse,
                                                            unsigned* __restrict__ out_absmax, int8_t* __restrict__ q,
                                                            uint16_t* __restrict__ q16, float* __restrict__ qs,
                                                            int qslot) {
    if constexpr (kQ) {
        // dependents may launch only after the grid barrier: a dependent grid's
        // blocks must not take the SMs this grid's unscheduled blocks still need
        asm volatile("griddepcontrol.wait;" ::: "memory");
    } else {
        QSB_PDL_ENTER();
    }
    extern __shared__ uint8_t sm_raw[];
    const uint32_t raw = ptx::smem_u32(sm_raw);
    uint8_t* sm = sm_raw + ((1024 - (raw & 1023)) & 1023);
    uint8_t* sQ = sm;
    uint8_t* sK = sm + kTile;
    uint8_t* sV = sm + 2 * kTile;
    uint8_t* sP = sm;  // over Q and K: 2 K-blocks (keys 0..63, 64..127) of [128 x 128B]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 3 * kTile);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
    const int bh = blockIdx.x, b = bh / H, h = bh % H;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t == 0) {
        ptx::tma_prefetch(&tm_qkv);
        for (int i = 0; i < 3; ++i) ptx::mbar_init(&bars[i], 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<128>(tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    if (t == 0) {
        ptx::mbar_arrive_expect_tx(&bars[0], 3 * kTile);
        const int row = b * kS;
        ptx::tma_load_2d(sQ, &tm_qkv, &bars[0], h * kD, row);
        ptx::tma_load_2d(sK, &tm_qkv, &bars[0], (H + h) * kD, row);
        ptx::tma_load_2d(sV, &tm_qkv, &bars[0], (2 * H + h) * kD, row);
        ptx::mbar_wait(&bars[0], 0);
        ptx::tc_fence_after();
        const uint32_t id_s = idesc_f16_f32(kS, kS, false);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k)
            ptx::mma_f16(tmem, ptx::sw128_kmajor_desc(ptx::smem_u32(sQ) + k * 32),
                         ptx::sw128_kmajor_desc(ptx::smem_u32(sK) + k * 32), id_s, k > 0 ? 1u : 0u);
        ptx::tc_commit(&bars[1]);
    }
    ptx::mbar_wait(&bars[1], 0);
    ptx::tc_fence_after();
    const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32(trow + 32 * c, r);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(r[j]));
    }
    const float sl2 = scale * kLog2e;
    float sum = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32(trow + 32 * c, r);
        ptx::tmem_ld_wait();
        uint32_t pkd[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float p0 = exp2f(__uint_as_float(r[2 * j]) * sl2 - mx * sl2);
            const float p1 = exp2f(__uint_as_float(r[2 * j + 1]) * sl2 - mx * sl2);
            sum += p0 + p1;
            pkd[j] = pk(p0, p1);
        }
        const uint32_t blk = ptx::smem_u32(sP + (c >> 1) * kTile) + t * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int chunk = (c & 1) * 4 + q;
            ptx::st_shared_v4(blk + ((chunk ^ (t & 7)) << 4), pkd[4 * q], pkd[4 * q + 1], pkd[4 * q + 2],
                              pkd[4 * q + 3]);
        }
    }
    ptx::fence_proxy_async_smem();  // P (generic-proxy stores) before the tensor core reads it
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (t == 0) {
        const uint32_t id_o = idesc_f16_f32(kD, kS, true);
#pragma unroll
        for (int k = 0; k < kS / 16; ++k) {
            const uint64_t da = ptx::sw128_kmajor_desc(ptx::smem_u32(sP) + (k >> 2) * kTile + (k & 3) * 32);
            const uint64_t db = ptx::sw128_mnmajor_desc(ptx::smem_u32(sV) + k * 16 * 128, kTile);
            ptx::mma_f16(tmem, da, db, id_o, k > 0 ? 1u : 0u);
        }
        ptx::tc_commit(&bars[2]);
    }
    ptx::mbar_wait(&bars[2], 0);
    ptx::tc_fence_after();
    uint32_t o[2][32];
    ptx::tmem_ld32(trow, o[0]);
    ptx::tmem_ld32(trow + 32, o[1]);
    ptx::tmem_ld_wait();
    const float inv = 1.f / sum;
    uint32_t w[32];
#pragma unroll
    for (int j = 0; j < 32; ++j)
        w[j] = pk(__uint_as_float(o[j >> 4][(2 * j) & 31]) * inv, __uint_as_float(o[j >> 4][(2 * j + 1) & 31]) * inv);
    __half* orow = out + (static_cast<int64_t>(b * kS + t) * H + h) * kD;
#pragma unroll
    for (int q = 0; q < 8; ++q)
        reinterpret_cast<uint4*>(orow)[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    lse[static_cast<int64_t>(bh) * kS + t] = mx * scale + logf(sum);
    if (kQ || out_absmax) {
        float amax = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[j]));
            amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
        }
        amax = warp_max(amax);
        if constexpr (kQ) {
            __shared__ float wmax[kTcThreads / 32];
            __shared__ float s_abs;
            if (lane == 0) wmax[warp] = amax;
            __syncthreads();
            if (t == 0) {
                float m = 0.f;
                for (int i = 0; i < kTcThreads / 32; ++i) m = fmaxf(m, wmax[i]);
                g_attq_part[qslot][blockIdx.x] = m;
            }
            attq_grid_barrier(g_attq_bar[qslot], gridDim.x);
            // every block reduces all partials (deterministic, nothing to zero)
            float m = 0.f;
            for (int i = t; i < static_cast<int>(gridDim.x); i += kTcThreads)
                m = fmaxf(m, __ldcg(&g_attq_part[qslot][i]));
            m = warp_max(m);
            if (lane == 0) wmax[warp] = m;
            __syncthreads();
            if (t == 0) {
                float a2 = 0.f;
                for (int i = 0; i < kTcThreads / 32; ++i) a2 = fmaxf(a2, wmax[i]);
                s_abs = a2;
            }
            __syncthreads();
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
            const float sc = scale_from_absmax(s_abs);
            if (blockIdx.x == 0 && t == 0) {
                qs[0] = sc;
                qs[1] = s_abs;
            }
            const QScale qsc = make_qscale(sc);
            const int64_t off = (static_cast<int64_t>(b * kS + t) * H + h) * kD;  // this thread's O row
            uint32_t qw[16], hw[32];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&w[2 * j]));
                const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&w[2 * j + 1]));
                const float t0 = quant_rne_f(f0.x, qsc), t1 = quant_rne_f(f0.y, qsc);
                const float t2 = quant_rne_f(f1.x, qsc), t3 = quant_rne_f(f1.y, qsc);
                qw[j] = pack_q4(t0, t1, t2, t3);
                hw[2 * j] = pack_half2(grid_value(t0), grid_value(t1));
                hw[2 * j + 1] = pack_half2(grid_value(t2), grid_value(t3));
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
                reinterpret_cast<uint4*>(q + off)[i] = make_uint4(qw[4 * i], qw[4 * i + 1], qw[4 * i + 2], qw[4 * i + 3]);
            if (q16) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    reinterpret_cast<uint4*>(q16 + off)[i] =
                        make_uint4(hw[4 * i], hw[4 * i + 1], hw[4 * i + 2], hw[4 * i + 3]);
            }
        } else {
            if (lane == 0 && amax > 0.f) atomicMax(out_absmax, __float_as_uint(amax));
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<128>(tmem);
    }
}

// ---------------------------------------------------------------------------- tcgen05 backward
// One CTA (4 warps) per (batch, head); five UMMA GEMMs:
//   S^T = K Q^T, dP^T = V dO^T      (M = 128 keys, N = 128 queries, K = 64)   TMEM cols 0..255
//   thread t = key row t: P^T = exp(S^T scale - lse[q]), dS^T = P^T (dP^T - D[q])
//   -> FP16 into shared memory (K-major, over the dead V tile and beyond)
//   dV = P^T dO, dK = dS^T Q         (M = 128 keys, N = 64, K = 128 queries)  TMEM cols 0..127
//   dQ = dS K  (A = dS read MN-major from the dS^T tile)                       TMEM cols 128..191
// Q, K, V, dO by TMA (128B swizzle; each [128 x 64] tile serves as K-major or
// MN-major operand by descriptor); D = rowsum(dO * O) from global.  8 warps:
// both warpgroups cover the 128 TMEM lanes and split the 128 query columns of
// the elementwise phase and the three outputs of the epilogue.
constexpr int kTcBwdSmem = 7 * kTile + 1024 + 2 * kS * 4 + 64;

__device__ __forceinline__ uint32_t idesc_f16_f32_ab(int n, int m, bool a_mn, bool b_mn) {
    return idesc_f16_f32(n, m, b_mn) | (static_cast<uint32_t>(a_mn) << 15);
}

__global__ void __launch_bounds__(2 * kTcThreads) k_attn_bwd_tc(const __grid_constant__ CUtensorMap tm_qkv,
                                                            const __grid_constant__ CUtensorMap tm_do,
                                                            const __half* __restrict__ out,
                                                            const __half* __restrict__ dout,
                                                            const float* __restrict__ lse, int H, float scale,
                                                            __half* __restrict__ dqkv) {
    QSB_PDL_ENTER();
    extern __shared__ uint8_t sm_raw[];
    const uint32_t raw = ptx::smem_u32(sm_raw);
    uint8_t* sm = sm_raw + ((1024 - (raw & 1023)) & 1023);
    uint8_t* sQ = sm;
    uint8_t* sK = sm + kTile;
    uint8_t* sdO = sm + 2 * kTile;
    uint8_t* sV = sm + 3 * kTile;   // dead after dP^T: P^T / dS^T are written over it
    uint8_t* sPT = sm + 3 * kTile;  // [128 keys x 128 queries] as 2 K-blocks of [128 x 128B]
    uint8_t* sDS = sm + 5 * kTile;  // dS^T, same layout
    float* sL = reinterpret_cast<float*>(sm + 7 * kTile);
    float* sD = sL + kS;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + kS);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
    const int bh = blockIdx.x, b = bh / H, h = bh % H;
    const int t = threadIdx.x & 127, warp = (threadIdx.x >> 5) & 3, wg = threadIdx.x >> 7;
    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tm_qkv);
        ptx::tma_prefetch(&tm_do);
        for (int i = 0; i < 3; ++i) ptx::mbar_init(&bars[i], 1);
        ptx::fence_mbar_init();
    }
    if (threadIdx.x < 32) ptx::tmem_alloc<256>(tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    const int64_t orow = static_cast<int64_t>(H) * kD;
    if (threadIdx.x == 0) {
        ptx::mbar_arrive_expect_tx(&bars[0], 4 * kTile);
        const int row = b * kS;
        ptx::tma_load_2d(sQ, &tm_qkv, &bars[0], h * kD, row);
        ptx::tma_load_2d(sK, &tm_qkv, &bars[0], (H + h) * kD, row);
        ptx::tma_load_2d(sV, &tm_qkv, &bars[0], (2 * H + h) * kD, row);
        ptx::tma_load_2d(sdO, &tm_do, &bars[0], h * kD, row);
    }
    if (wg == 0) {   // D[q] = sum_d dO[q,d] O[q,d] (thread t = query t) and lse in log2 units
        const uint4* op = reinterpret_cast<const uint4*>(out + (static_cast<int64_t>(b) * kS + t) * orow + h * kD);
        const uint4* dp = reinterpret_cast<const uint4*>(dout + (static_cast<int64_t>(b) * kS + t) * orow + h * kD);
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint4 ov = op[i], dv = dp[i];
            const __half2* oh = reinterpret_cast<const __half2*>(&ov);
            const __half2* dh = reinterpret_cast<const __half2*>(&dv);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 a = __half22float2(oh[e]), c = __half22float2(dh[e]);
                acc += a.x * c.x + a.y * c.y;
            }
        }
        sD[t] = acc;
        sL[t] = lse[static_cast<int64_t>(bh) * kS + t] * kLog2e;
    }
    if (threadIdx.x == 0) {
        ptx::mbar_wait(&bars[0], 0);
        ptx::tc_fence_after();
        const uint32_t id = idesc_f16_f32_ab(kS, kS, false, false);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
            ptx::mma_f16(tmem, ptx::sw128_kmajor_desc(ptx::smem_u32(sK) + k * 32),
                         ptx::sw128_kmajor_desc(ptx::smem_u32(sQ) + k * 32), id, k > 0 ? 1u : 0u);
            ptx::mma_f16(tmem + kS, ptx::sw128_kmajor_desc(ptx::smem_u32(sV) + k * 32),
                         ptx::sw128_kmajor_desc(ptx::smem_u32(sdO) + k * 32), id, k > 0 ? 1u : 0u);
        }
        ptx::tc_commit(&bars[1]);
    }
    __syncthreads();  // sD / sL visible to every thread
    ptx::mbar_wait(&bars[1], 0);
    ptx::tc_fence_after();
    const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const float sl2 = scale * kLog2e;
#pragma unroll 1
    for (int c = 2 * wg; c < 2 * wg + 2; ++c) {  // 32 queries per chunk; each warpgroup takes half
        uint32_t rs[32], rp[32];
        ptx::tmem_ld32(trow + 32 * c, rs);
        ptx::tmem_ld32(trow + kS + 32 * c, rp);
        ptx::tmem_ld_wait();
        uint32_t pp[16], pd[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int q = 32 * c + 2 * j;
            const float p0 = exp2f(__uint_as_float(rs[2 * j]) * sl2 - sL[q]);
            const float p1 = exp2f(__uint_as_float(rs[2 * j + 1]) * sl2 - sL[q + 1]);
            const float d0 = p0 * (__uint_as_float(rp[2 * j]) - sD[q]);
            const float d1 = p1 * (__uint_as_float(rp[2 * j + 1]) - sD[q + 1]);
            pp[j] = pk(p0, p1);
            pd[j] = pk(d0, d1);
        }
        const uint32_t off = (c >> 1) * kTile + t * 128;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            const uint32_t sw = ((((c & 1) * 4 + q4) ^ (t & 7)) << 4);
            ptx::st_shared_v4(ptx::smem_u32(sPT) + off + sw, pp[4 * q4], pp[4 * q4 + 1], pp[4 * q4 + 2], pp[4 * q4 + 3]);
            ptx::st_shared_v4(ptx::smem_u32(sDS) + off + sw, pd[4 * q4], pd[4 * q4 + 1], pd[4 * q4 + 2], pd[4 * q4 + 3]);
        }
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t id_kv = idesc_f16_f32_ab(kD, kS, false, true);
        const uint32_t id_q = idesc_f16_f32_ab(kD, kS, true, true);
#pragma unroll
        for (int k = 0; k < kS / 16; ++k) {
            const uint32_t aoff = (k >> 2) * kTile + (k & 3) * 32;
            const uint32_t brow = k * 16 * 128;
            const uint32_t acc = k > 0 ? 1u : 0u;
            // dV = P^T dO, dK = dS^T Q   (B MN-major: rows = queries)
            ptx::mma_f16(tmem, ptx::sw128_kmajor_desc(ptx::smem_u32(sPT) + aoff),
                         ptx::sw128_mnmajor_desc(ptx::smem_u32(sdO) + brow, kTile), id_kv, acc);
            ptx::mma_f16(tmem + kD, ptx::sw128_kmajor_desc(ptx::smem_u32(sDS) + aoff),
                         ptx::sw128_mnmajor_desc(ptx::smem_u32(sQ) + brow, kTile), id_kv, acc);
            // dQ = dS K   (A = dS MN-major from the dS^T tile: rows = keys; B = K MN-major)
            ptx::mma_f16(tmem + kS, ptx::sw128_mnmajor_desc(ptx::smem_u32(sDS) + brow, kTile),
                         ptx::sw128_mnmajor_desc(ptx::smem_u32(sK) + brow, kTile), id_q, acc);
        }
        ptx::tc_commit(&bars[2]);
    }
    ptx::mbar_wait(&bars[2], 0);
    ptx::tc_fence_after();
    const int64_t rs3 = 3LL * H * kD;
#pragma unroll 1
    for (int which = wg; which < 3; which += 2) {  // 0 dQ (row = query t), 1 dK, 2 dV (row = key t)
        const uint32_t col = which == 0 ? kS : (which == 1 ? kD : 0);
        const float f = which == 2 ? 1.f : scale;
        uint32_t r[2][32];
        ptx::tmem_ld32(trow + col, r[0]);
        ptx::tmem_ld32(trow + col + 32, r[1]);
        ptx::tmem_ld_wait();
        uint32_t w[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
            w[j] = pk(__uint_as_float(r[j >> 4][(2 * j) & 31]) * f, __uint_as_float(r[j >> 4][(2 * j + 1) & 31]) * f);
        __half* dst = dqkv + (static_cast<int64_t>(b) * kS + t) * rs3 + (static_cast<int64_t>(which) * H + h) * kD;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            reinterpret_cast<uint4*>(dst)[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<256>(tmem);
    }
}

// Two CTAs per SM: P^T never touches shared memory.  The elementwise phase
// writes P^T (FP16 pairs) into the consumed S^T columns of tensor memory and dV
// = P^T dO reads it from there (tcgen05.mma with A in TMEM); dS^T goes to smem
// over the dead V tile and one more (it is also dQ's MN-major A).  Five 16 KB
// tiles instead of seven: 2 x ~83 KB smem and 2 x 256 TMEM columns per SM, so
// one CTA's MMAs / loads overlap the other's elementwise phase and epilogue.
//   TMEM: phase 1  S^T cols 0..127, dP^T 128..255
//         phase 2  P^T 0..63 (packed), dV 64..127, dK 128..191, dQ 192..255
constexpr int kTcBwd2Smem = 5 * kTile + 1024 + 2 * kS * 4 + 64;

__global__ void __launch_bounds__(2 * kTcThreads, 2) k_attn_bwd_tc2(const __grid_constant__ CUtensorMap tm_qkv,
                                                                const __grid_constant__ CUtensorMap tm_do,
                                                                const __half* __restrict__ out,
                                                                const __half* __restrict__ dout,
                                                                const float* __restrict__ lse, int H, float scale,
                                                                __half* __restrict__ dqkv) {
    QSB_PDL_ENTER();
    extern __shared__ uint8_t sm_raw[];
    const uint32_t raw = ptx::smem_u32(sm_raw);
    uint8_t* sm = sm_raw + ((1024 - (raw & 1023)) & 1023);
    uint8_t* sQ = sm;
    uint8_t* sK = sm + kTile;
    uint8_t* sdO = sm + 2 * kTile;
    uint8_t* sV = sm + 3 * kTile;   // dead after dP^T: dS^T is written over it
    uint8_t* sDS = sm + 3 * kTile;  // dS^T [128 keys x 128 queries] as 2 K-blocks of [128 x 128B]
    float* sL = reinterpret_cast<float*>(sm + 5 * kTile);
    float* sD = sL + kS;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + kS);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
    const int bh = blockIdx.x, b = bh / H, h = bh % H;
    const int t = threadIdx.x & 127, warp = (threadIdx.x >> 5) & 3, wg = threadIdx.x >> 7;
    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tm_qkv);
        ptx::tma_prefetch(&tm_do);
        for (int i = 0; i < 3; ++i) ptx::mbar_init(&bars[i], 1);
        ptx::fence_mbar_init();
    }
    if (threadIdx.x < 32) ptx::tmem_alloc<256>(tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    const int64_t orow = static_cast<int64_t>(H) * kD;
    if (threadIdx.x == 0) {
        ptx::mbar_arrive_expect_tx(&bars[0], 4 * kTile);
        const int row = b * kS;
        ptx::tma_load_2d(sQ, &tm_qkv, &bars[0], h * kD, row);
        ptx::tma_load_2d(sK, &tm_qkv, &bars[0], (H + h) * kD, row);
        ptx::tma_load_2d(sV, &tm_qkv, &bars[0], (2 * H + h) * kD, row);
        ptx::tma_load_2d(sdO, &tm_do, &bars[0], h * kD, row);
    }
    if (wg == 0) {   // D[q] = sum_d dO[q,d] O[q,d] (thread t = query t) and lse in log2 units
        const uint4* op = reinterpret_cast<const uint4*>(out + (static_cast<int64_t>(b) * kS + t) * orow + h * kD);
        const uint4* dp = reinterpret_cast<const uint4*>(dout + (static_cast<int64_t>(b) * kS + t) * orow + h * kD);
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint4 ov = op[i], dv = dp[i];
            const __half2* oh = reinterpret_cast<const __half2*>(&ov);
            const __half2* dh = reinterpret_cast<const __half2*>(&dv);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 a = __half22float2(oh[e]), c = __half22float2(dh[e]);
                acc += a.x * c.x + a.y * c.y;
            }
        }
        sD[t] = acc;
        sL[t] = lse[static_cast<int64_t>(bh) * kS + t] * kLog2e;
    }
    if (threadIdx.x == 0) {
        ptx::mbar_wait(&bars[0], 0);
        ptx::tc_fence_after();
        const uint32_t id = idesc_f16_f32_ab(kS, kS, false, false);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
            ptx::mma_f16(tmem, ptx::sw128_kmajor_desc(ptx::smem_u32(sK) + k * 32),
                         ptx::sw128_kmajor_desc(ptx::smem_u32(sQ) + k * 32), id, k > 0 ? 1u : 0u);
            ptx::mma_f16(tmem + kS, ptx::sw128_kmajor_desc(ptx::smem_u32(sV) + k * 32),
                         ptx::sw128_kmajor_desc(ptx::smem_u32(sdO) + k * 32), id, k > 0 ? 1u : 0u);
        }
        ptx::tc_commit(&bars[1]);
    }
    __syncthreads();  // sD / sL visible to every thread
    ptx::mbar_wait(&bars[1], 0);
    ptx::tc_fence_after();
    const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const float sl2 = scale * kLog2e;
    uint32_t keep[2][16];  // this warp's P^T chunks, stored to TMEM once every S^T column is read
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {  // 32 queries per chunk; each warpgroup takes half
        const int c = 2 * wg + cc;
        uint32_t rs[32], rp[32];
        ptx::tmem_ld32(trow + 32 * c, rs);
        ptx::tmem_ld32(trow + kS + 32 * c, rp);
        ptx::tmem_ld_wait();
        uint32_t pd[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int q = 32 * c + 2 * j;
            const float p0 = exp2f(__uint_as_float(rs[2 * j]) * sl2 - sL[q]);
            const float p1 = exp2f(__uint_as_float(rs[2 * j + 1]) * sl2 - sL[q + 1]);
            const float d0 = p0 * (__uint_as_float(rp[2 * j]) - sD[q]);
            const float d1 = p1 * (__uint_as_float(rp[2 * j + 1]) - sD[q + 1]);
            keep[cc][j] = pk(p0, p1);
            pd[j] = pk(d0, d1);
        }
        const uint32_t off = (c >> 1) * kTile + t * 128;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            const uint32_t sw = ((((c & 1) * 4 + q4) ^ (t & 7)) << 4);
            ptx::st_shared_v4(ptx::smem_u32(sDS) + off + sw, pd[4 * q4], pd[4 * q4 + 1], pd[4 * q4 + 2], pd[4 * q4 + 3]);
        }
    }
    // every warp has read its S^T / dP^T columns: P^T may now overwrite S^T
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) ptx::tmem_st16(trow + 16 * (2 * wg + cc), keep[cc]);
    ptx::tmem_st_wait();
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t id_kv = idesc_f16_f32_ab(kD, kS, false, true);
        const uint32_t id_q = idesc_f16_f32_ab(kD, kS, true, true);
#pragma unroll
        for (int k = 0; k < kS / 16; ++k) {
            const uint32_t aoff = (k >> 2) * kTile + (k & 3) * 32;
            const uint32_t brow = k * 16 * 128;
            const uint32_t acc = k > 0 ? 1u : 0u;
            // dV = P^T dO   (A = P^T from TMEM, 8 columns per 16 queries; B MN-major)
            ptx::mma_f16_ts(tmem + 64, tmem + 8 * k, ptx::sw128_mnmajor_desc(ptx::smem_u32(sdO) + brow, kTile),
                            id_kv, acc);
            // dK = dS^T Q
            ptx::mma_f16(tmem + 128, ptx::sw128_kmajor_desc(ptx::smem_u32(sDS) + aoff),
                         ptx::sw128_mnmajor_desc(ptx::smem_u32(sQ) + brow, kTile), id_kv, acc);
            // dQ = dS K   (A = dS MN-major from the dS^T tile: rows = keys; B = K MN-major)
            ptx::mma_f16(tmem + 192, ptx::sw128_mnmajor_desc(ptx::smem_u32(sDS) + brow, kTile),
                         ptx::sw128_mnmajor_desc(ptx::smem_u32(sK) + brow, kTile), id_q, acc);
        }
        ptx::tc_commit(&bars[2]);
    }
    ptx::mbar_wait(&bars[2], 0);
    ptx::tc_fence_after();
    const int64_t rs3 = 3LL * H * kD;
#pragma unroll 1
    for (int which = wg; which < 3; which += 2) {  // 0 dQ (row = query t), 1 dK, 2 dV (row = key t)
        const uint32_t col = which == 0 ? 192 : (which == 1 ? 128 : 64);
        const float f = which == 2 ? 1.f : scale;
        uint32_t r[2][32];
        ptx::tmem_ld32(trow + col, r[0]);
        ptx::tmem_ld32(trow + col + 32, r[1]);
        ptx::tmem_ld_wait();
        uint32_t w[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
            w[j] = pk(__uint_as_float(r[j >> 4][(2 * j) & 31]) * f, __uint_as_float(r[j >> 4][(2 * j + 1) & 31]) * f);
        __half* dst = dqkv + (static_cast<int64_t>(b) * kS + t) * rs3 + (static_cast<int64_t>(which) * H + h) * kD;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            reinterpret_cast<uint4*>(dst)[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<256>(tmem);
    }
}

int g_attn_tc = 2;  // 0 mma.sync kernels, 1 tcgen05, 2 tcgen05 backward at 2 CTAs / SM (qsync_attention_set_impl)

constexpr int kFwdSmem = 3 * kTile;
constexpr int kBwdSmem = 4 * kTile + 2 * kTile + 2 * kS * 4;

int check_shape(int64_t B, int64_t S, int64_t H, int64_t D) {
    QSB_REQUIRE(S == kS && D == kD, QSYNC_ERR_DOMAIN,
                "attention core supports seq 128, head dim 64 (got seq " + std::to_string(S) + ", dim " +
                    std::to_string(D) + ")");
    QSB_REQUIRE(B > 0 && H > 0 && B * H < (int64_t(1) << 31), QSYNC_ERR_DOMAIN, "bad batch / head count");
    return QSYNC_OK;
}

}  // namespace
}  // namespace qsb

using namespace qsb;

extern "C" {

int qsync_attention_fwd(const void* qkv, int64_t B, int64_t S, int64_t H, int64_t D, float scale, void* out,
                        float* lse, float* out_absmax, qsync_stream_t stream) {
    QSB_REQUIRE(qkv && out && lse, QSYNC_ERR_VALIDATION, "attention needs qkv, out and lse buffers");
    QSB_TRY(check_shape(B, S, H, D));
    cudaStream_t st = to_stream(stream);
    QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_attn_fwd), kFwdSmem));
    if (out_absmax) QSB_TRY(zero_async(out_absmax, sizeof(float), st));
    if (g_attn_tc) {
        QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_attn_fwd_tc<false>), kTcFwdSmem));
        CUtensorMap tm;
        QSB_TRY(make_tma_2d(&tm, qkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, 3 * H * kD, B * kS, kD, kS));
        pdl_launch(k_attn_fwd_tc<false>, dim3(static_cast<unsigned>(B * H)), dim3(kTcThreads), kTcFwdSmem, st, tm,
                   static_cast<int>(H), scale, static_cast<__half*>(out), lse, reinterpret_cast<unsigned*>(out_absmax),
                   static_cast<int8_t*>(nullptr), static_cast<uint16_t*>(nullptr), static_cast<float*>(nullptr), 0);
        return check_launch("k_attn_fwd_tc");
    }
    pdl_launch(k_attn_fwd, dim3(static_cast<unsigned>(B * H)), dim3(kThreadsA), kFwdSmem, st, 
        static_cast<const __half*>(qkv), static_cast<int>(H), scale, static_cast<__half*>(out), lse,
        reinterpret_cast<unsigned*>(out_absmax));
    return check_launch("k_attn_fwd");
}

int qsync_attention_fwd_quant(const void* qkv, int64_t B, int64_t S, int64_t H, int64_t D, float scale, void* out,
                              float* lse, int8_t* q, uint16_t* q16, float* qscale, qsync_stream_t stream) {
    QSB_REQUIRE(qkv && out && lse && q && qscale, QSYNC_ERR_VALIDATION,
                "attention + quantize needs qkv, out, lse, q and qscale (float[2]) buffers");
    QSB_TRY(check_shape(B, S, H, D));
    cudaStream_t st = to_stream(stream);
    const int64_t blocks = B * H;
    bool fused = g_attn_tc != 0 && blocks <= kAttQMaxBlocks;
    if (fused) {
        // every block must be co-resident for the grid barrier (TMEM: 128 columns each)
        static int occ[16] = {0};
        int dev = 0;
        QSB_TRY(cuda_status(cudaGetDevice(&dev), "cudaGetDevice"));
        QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_attn_fwd_tc<true>), kTcFwdSmem));
        if (dev < 16 && occ[dev] == 0) {
            // cudaOccupancyMaxActiveBlocksPerMultiprocessor answers 1 for ANY kernel that
            // executes tcgen05.alloc (it cannot see the column count); the hardware keeps
            // 4 of these blocks per SM resident (measured: a 4 x 148-block grid of
            // 128-thread, 50 KB, 128-column blocks all pass a barrier). So count the
            // per-SM limits here: shared memory, registers (per warp, 256-register
            // granules), threads, and TMEM columns.
            cudaFuncAttributes fa{};
            QSB_TRY(cuda_status(cudaFuncGetAttributes(&fa, k_attn_fwd_tc<true>), "cudaFuncGetAttributes"));
            int smem_sm = 0, regs_sm = 0, thr_sm = 0, resv = 0;
            QSB_TRY(cuda_status(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev),
                                "cudaDeviceGetAttribute"));
            QSB_TRY(cuda_status(cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev),
                                "cudaDeviceGetAttribute"));
            QSB_TRY(cuda_status(cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev),
                                "cudaDeviceGetAttribute"));
            QSB_TRY(cuda_status(cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev),
                                "cudaDeviceGetAttribute"));
            const int smem_blk = ((kTcFwdSmem + static_cast<int>(fa.sharedSizeBytes) + resv + 1023) / 1024) * 1024;
            const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
            const int n = std::min({smem_sm / smem_blk, regs_sm / (regs_warp * (kTcThreads / 32)),
                                    thr_sm / kTcThreads, 512 / 128});
            occ[dev] = n > 0 ? n : -1;
        }
        const int per_sm = dev < 16 ? occ[dev] : 0;
        fused = per_sm > 0 && blocks <= static_cast<int64_t>(per_sm) * sm_count();
    }
    if (!fused) {  // attention with absmax, then the one-pass quantizer: the same q, q16, scale
        QSB_TRY(qsync_attention_fwd(qkv, B, S, H, D, scale, out, lse, qscale + 1, stream));
        return qsync_quantize_act_ex(out, QSYNC_F16, B * S * H * D, QSYNC_ACT_NONE, qscale + 1, q, qscale, nullptr,
                                     q16, stream);
    }
    CUtensorMap tm;
    QSB_TRY(make_tma_2d(&tm, qkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, 3 * H * kD, B * kS, kD, kS));
    const int slot = static_cast<int>((reinterpret_cast<uintptr_t>(st) >> 4) % kAttQSlots);
    pdl_launch(k_attn_fwd_tc<true>, dim3(static_cast<unsigned>(blocks)), dim3(kTcThreads), kTcFwdSmem, st, tm,
               static_cast<int>(H), scale, static_cast<__half*>(out), lse, static_cast<unsigned*>(nullptr), q, q16,
               qscale, slot);
    return check_launch("k_attn_fwd_tc<quant>");
}

int qsync_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse, int64_t B,
                        int64_t S, int64_t H, int64_t D, float scale, void* dqkv, qsync_stream_t stream) {
    QSB_REQUIRE(qkv && out && dout && lse && dqkv, QSYNC_ERR_VALIDATION, "attention backward needs all buffers");
    QSB_TRY(check_shape(B, S, H, D));
    cudaStream_t st = to_stream(stream);
    if (g_attn_tc == 2) {
        QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_attn_bwd_tc2), kTcBwd2Smem));
        CUtensorMap tq, td;
        QSB_TRY(make_tma_2d(&tq, qkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, 3 * H * kD, B * kS, kD, kS));
        QSB_TRY(make_tma_2d(&td, dout, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, H * kD, B * kS, kD, kS));
        pdl_launch(k_attn_bwd_tc2, dim3(static_cast<unsigned>(B * H)), dim3(2 * kTcThreads), kTcBwd2Smem, st, tq,
                   td, static_cast<const __half*>(out), static_cast<const __half*>(dout), lse, static_cast<int>(H),
                   scale, static_cast<__half*>(dqkv));
        return check_launch("k_attn_bwd_tc2");
    }
    if (g_attn_tc) {
        QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_attn_bwd_tc), kTcBwdSmem));
        CUtensorMap tq, td;
        QSB_TRY(make_tma_2d(&tq, qkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, 3 * H * kD, B * kS, kD, kS));
        QSB_TRY(make_tma_2d(&td, dout, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, H * kD, B * kS, kD, kS));
        pdl_launch(k_attn_bwd_tc, dim3(static_cast<unsigned>(B * H)), dim3(2 * kTcThreads), kTcBwdSmem, st, tq, td,
                   static_cast<const __half*>(out), static_cast<const __half*>(dout), lse, static_cast<int>(H),
                   scale, static_cast<__half*>(dqkv));
        return check_launch("k_attn_bwd_tc");
    }
    QSB_TRY(ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_attn_bwd), kBwdSmem));
    pdl_launch(k_attn_bwd, dim3(static_cast<unsigned>(B * H)), dim3(kThreadsA), kBwdSmem, st, 
        static_cast<const __half*>(qkv), static_cast<const __half*>(out), static_cast<const __half*>(dout), lse,
        static_cast<int>(H), scale, static_cast<__half*>(dqkv));
    return check_launch("k_attn_bwd");
}

int qsync_attention_set_impl(int tc) {
    QSB_REQUIRE(tc >= 0 && tc <= 2, QSYNC_ERR_DOMAIN, "attention impl must be 0 (mma.sync), 1 or 2 (tcgen05)");
    g_attn_tc = tc;
    return QSYNC_OK;
}

}  // extern "C"

// vec.cuh -- 16-byte vector load/unpack helpers shared by the streaming kernels.
#pragma once

#include <algorithm>

#include "common.cuh"

namespace qsb {

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Unpack a 16-byte vector of DT into floats (4 for F32, 8 for F16/BF16).
template <int DT>
struct Vec;
template <>
struct Vec<QSYNC_F32> {
    static constexpr int N = 4;
    __device__ static void unpack(uint4 r, float* f) {
        f[0] = __uint_as_float(r.x);
        f[1] = __uint_as_float(r.y);
        f[2] = __uint_as_float(r.z);
        f[3] = __uint_as_float(r.w);
    }
};
template <>
struct Vec<QSYNC_F16> {
    static constexpr int N = 8;
    __device__ static void unpack(uint4 r, float* f) {
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
            float2 v = __half22float2(h);
            f[2 * i] = v.x;
            f[2 * i + 1] = v.y;
        }
    }
};
template <>
struct Vec<QSYNC_BF16> {
    static constexpr int N = 8;
    __device__ static void unpack(uint4 r, float* f) {
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
            float2 v = __bfloat1622float2(h);
            f[2 * i] = v.x;
            f[2 * i + 1] = v.y;
        }
    }
};

__host__ __device__ inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int grid_for(int64_t work_items, int per_block, int max_blocks_per_sm = 4) {
    int64_t want = (work_items + per_block - 1) / per_block;
    int64_t cap = static_cast<int64_t>(sm_count()) * max_blocks_per_sm;
    return static_cast<int>(std::max<int64_t>(1, std::min(want, cap)));
}

}  // namespace qsb

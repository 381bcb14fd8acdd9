// capi.cpp -- status / error plumbing of the C ABI (qsync_b200.h).
//
// Status codes are qsync::ErrorKind + 1 (errors.hpp:11-26); the kind tags are
// the reference's error_kind_name strings (errors.cpp:5-23), and messages carry
// the "<kind>: " prefix of qsync::Error (errors.hpp:33) so a C++ caller can
// re-raise without reformatting.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <set>
#include <string>

#include "common.cuh"
#include "mt_jump.hpp"

namespace qsb {

namespace {
thread_local std::string g_last_error;

const char* kind_name(int status) {
    switch (status) {
        case QSYNC_OK: return "ok";
        case QSYNC_ERR_GRAPH_CYCLE: return "graph-cycle";
        case QSYNC_ERR_VALIDATION: return "validation";
        case QSYNC_ERR_REFERENCE: return "reference";
        case QSYNC_ERR_DOMAIN: return "domain";
        case QSYNC_ERR_MISSING_PROFILE: return "missing-profile";
        case QSYNC_ERR_MISSING_MODEL: return "missing-model";
        case QSYNC_ERR_DEGENERATE_FIT: return "degenerate-fit";
        case QSYNC_ERR_STATS_INCOMPLETE: return "stats-incomplete";
        case QSYNC_ERR_KIND_MISMATCH: return "kind-mismatch";
        case QSYNC_ERR_TOPOLOGY: return "topology";
        case QSYNC_ERR_ENUMERATION_LIMIT: return "enumeration-limit";
        case QSYNC_ERR_INFEASIBLE: return "infeasible";
        case QSYNC_ERR_IO: return "io";
        case QSYNC_ERR_INTERNAL: return "internal";
    }
    return "unknown";
}
}  // namespace

int set_error(int status, const std::string& msg) {
    g_last_error = std::string(kind_name(status)) + ": " + msg;
    return status;
}

static std::atomic<unsigned long long> g_launches{0};
int g_pdl_enabled = 1;

int check_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return QSYNC_OK;
    return set_error(QSYNC_ERR_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}

// Zero n 32-bit words as a kernel launched with PDL (an accumulator such as a
// device absmax before the atomicMax kernel that produces it).  A memset node
// would break the programmatic-dependent chain of the CUDA graph: the next
// kernel could no longer overlap its launch and prologue with this one.
__global__ void k_zero_words(uint32_t* __restrict__ p, int64_t n) {
    QSB_PDL_ENTER();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = 0u;
}

int zero_async(void* p, int64_t bytes, cudaStream_t st) {
    if (!p || bytes <= 0) return QSYNC_OK;
    QSB_REQUIRE(bytes % 4 == 0 && (reinterpret_cast<uintptr_t>(p) & 3) == 0, QSYNC_ERR_DOMAIN,
                "zero_async needs 4-byte words");
    const int64_t n = bytes / 4;
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 1024));
    return launch_pdl("k_zero_words", k_zero_words, dim3(grid), dim3(256), 0, st, static_cast<uint32_t*>(p), n);
}

int ensure_max_dynamic_smem(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    QSB_TRY(cuda_status(cudaGetDevice(&dev), "cudaGetDevice"));
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({kernel, dev})) return QSYNC_OK;
    QSB_TRY(cuda_status(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                        "cudaFuncSetAttribute"));
    done.insert({kernel, dev});
    return QSYNC_OK;
}

int sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    static int cached[64] = {0};
    if (dev < 64 && cached[dev]) return cached[dev];
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        n = 148;
    if (dev < 64) cached[dev] = n;
    return n;
}

}  // namespace qsb

extern "C" {

const char* qsync_last_error(void) { return qsb::g_last_error.c_str(); }

const char* qsync_status_name(int status) { return qsb::kind_name(status); }

int qsync_abi_version(void) { return 1; }

unsigned long long qsync_launch_count(void) { return qsb::g_launches.load(); }

int qsync_device_sm_count(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

// Host-only self-test of the mt19937_64 jump-ahead polynomials (no GPU needed).
int qsync_mt_jump_selftest(void) {
    const int r = qsb::mtjump::self_test();
    if (r != 0) return qsb::set_error(QSYNC_ERR_INTERNAL, "mt19937_64 jump-ahead self-test failed (" + std::to_string(r) + ")");
    return QSYNC_OK;
}

}  // extern "C"

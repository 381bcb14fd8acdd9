// capi.cpp -- status / error plumbing of the C ABI (qsync_b200.h).
//
// Status codes are qsync::ErrorKind + 1 (errors.hpp:11-26); the kind tags are
// the reference's error_kind_name strings (errors.cpp:5-23), and messages carry
// the "<kind>: " prefix of qsync::Error (errors.hpp:33) so a C++ caller can
// re-raise without reformatting.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
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

// comm.cu -- C1: the data-parallel FP32 gradient exchange (qsync_b200.h, "C1").
//
// The reference models this exchange and never runs it: per-rank bucket slots
// (profile.hpp:118-129) are replayed with Eq. 6 semantics -- slot n starts at
// max(all ranks ready, end of slot n-1), the optimizer after the last slot
// (replayer.cpp:48-73).  Here it runs: one NCCL communicator per rank (one
// process per GPU), in-place FP32 bucket all-reduce on the caller's stream.
//
// NCCL is resolved at run time with dlopen: the libnccl.so.2 already mapped into
// the process (torch's, when the caller is the Python training step) is reused
// through RTLD_NOLOAD, otherwise the system library is loaded.  The library
// therefore links no NCCL and a C++ host without torch still works.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace qsb {
namespace {

// The slice of nccl.h (NCCL 2.x ABI, stable since 2.10) this file calls.
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[QSYNC_COMM_ID_BYTES];
} ncclUniqueId;
typedef int ncclResult_t;     // ncclSuccess = 0
constexpr int kNcclSum = 0;   // ncclRedOp_t
constexpr int kNcclAvg = 4;
constexpr int kNcclFloat32 = 7;  // ncclDataType_t

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string why;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
            if (n.h) break;
        }
        if (!n.h) n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!n.h) n.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!n.h) {
            const char* e = dlerror();
            n.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(n.h, "ncclGetUniqueId"));
        n.init_rank = reinterpret_cast<decltype(n.init_rank)>(dlsym(n.h, "ncclCommInitRank"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(n.h, "ncclCommDestroy"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(n.h, "ncclAllReduce"));
        n.get_version = reinterpret_cast<decltype(n.get_version)>(dlsym(n.h, "ncclGetVersion"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(n.h, "ncclGetErrorString"));
        if (!n.get_unique_id || !n.init_rank || !n.destroy || !n.all_reduce || !n.get_version)
            n.why = "libnccl.so.2 lacks a required symbol";
    });
    return n;
}

int nccl_ready() {
    const Nccl& n = nccl();
    QSB_REQUIRE(n.why.empty(), QSYNC_ERR_INTERNAL, n.why);
    return QSYNC_OK;
}

int nccl_status(ncclResult_t r, const char* what) {
    if (r == 0) return QSYNC_OK;
    const Nccl& n = nccl();
    const char* msg = n.error_string ? n.error_string(r) : "unknown NCCL error";
    return set_error(QSYNC_ERR_INTERNAL, std::string(what) + ": " + msg + " (ncclResult " + std::to_string(r) + ")");
}

}  // namespace
}  // namespace qsb

struct qsync_comm_s {
    qsb::ncclComm_t nc;
    int nranks;
    int rank;
    int device;
};

using namespace qsb;

extern "C" {

int qsync_comm_nccl_version(void) {
    if (nccl_ready() != QSYNC_OK) return -1;
    int v = -1;
    if (nccl().get_version(&v) != 0) return -1;
    return v;
}

int qsync_comm_unique_id(uint8_t id[QSYNC_COMM_ID_BYTES]) {
    QSB_REQUIRE(id != nullptr, QSYNC_ERR_VALIDATION, "null communicator id buffer");
    QSB_TRY(nccl_ready());
    ncclUniqueId u;
    QSB_TRY(nccl_status(nccl().get_unique_id(&u), "ncclGetUniqueId"));
    std::memcpy(id, u.internal, QSYNC_COMM_ID_BYTES);
    return QSYNC_OK;
}

int qsync_comm_init(qsync_comm_t* comm, int nranks, int rank, const uint8_t id[QSYNC_COMM_ID_BYTES]) {
    QSB_REQUIRE(comm != nullptr && id != nullptr, QSYNC_ERR_VALIDATION, "null communicator argument");
    QSB_REQUIRE(nranks >= 1, QSYNC_ERR_DOMAIN, "communicator needs nranks >= 1");
    QSB_REQUIRE(rank >= 0 && rank < nranks, QSYNC_ERR_DOMAIN,
                "rank " + std::to_string(rank) + " outside [0, " + std::to_string(nranks) + ")");
    *comm = nullptr;
    QSB_TRY(nccl_ready());
    int dev = 0;
    QSB_TRY(cuda_status(cudaGetDevice(&dev), "cudaGetDevice"));
    ncclUniqueId u;
    std::memcpy(u.internal, id, QSYNC_COMM_ID_BYTES);
    ncclComm_t nc = nullptr;
    QSB_TRY(nccl_status(nccl().init_rank(&nc, nranks, u, rank), "ncclCommInitRank"));
    *comm = new qsync_comm_s{nc, nranks, rank, dev};
    return QSYNC_OK;
}

int qsync_comm_destroy(qsync_comm_t comm) {
    if (!comm) return QSYNC_OK;
    const int st = nccl_status(nccl().destroy(comm->nc), "ncclCommDestroy");
    delete comm;
    return st;
}

int qsync_comm_info(qsync_comm_t comm, int* nranks, int* rank, int* device) {
    QSB_REQUIRE(comm != nullptr, QSYNC_ERR_VALIDATION, "null communicator");
    if (nranks) *nranks = comm->nranks;
    if (rank) *rank = comm->rank;
    if (device) *device = comm->device;
    return QSYNC_OK;
}

int qsync_allreduce_bucket(qsync_comm_t comm, float* buf, int64_t count, int average, qsync_stream_t stream) {
    QSB_REQUIRE(comm != nullptr, QSYNC_ERR_VALIDATION, "null communicator");
    QSB_REQUIRE(count >= 0, QSYNC_ERR_DOMAIN, "bucket element count must be >= 0");
    if (count == 0) return QSYNC_OK;
    QSB_REQUIRE(buf != nullptr, QSYNC_ERR_VALIDATION, "null bucket buffer");
    QSB_TRY(nccl_status(nccl().all_reduce(buf, buf, static_cast<size_t>(count), kNcclFloat32,
                                          average ? kNcclAvg : kNcclSum, comm->nc, to_stream(stream)),
                        "ncclAllReduce"));
    return QSYNC_OK;
}

}  // extern "C"

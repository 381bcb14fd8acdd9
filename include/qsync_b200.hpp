// qsync_b200.hpp -- C++ host-side mirror of the reference operator API over the
// C ABI (qsync_b200.h).  Header-only; link libqsync_b200.so and libcudart.
//
// Drop-in for the reference's stochastic-rounding entry points
// (include/qsync/indicator.hpp:77-91, src/indicator.cpp:176-200): same
// argument meaning, same results bit for bit, same error kinds and messages.
// Errors surface as qsync::Error when the reference's errors.hpp is visible
// (define QSYNC_B200_WITH_REFERENCE_ERRORS after including "qsync/errors.hpp"),
// else as qsync_b200::Error carrying the same kind tag.
#ifndef QSYNC_B200_HPP
#define QSYNC_B200_HPP

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "qsync_b200.h"

namespace qsync_b200 {

/// Mirror of qsync::Error (errors.hpp:30-40) for standalone use.
class Error : public std::runtime_error {
  public:
    Error(int status, const std::string& what) : std::runtime_error(what), status_(status) {}
    int status() const { return status_; }
    std::string kind() const { return qsync_status_name(status_); }

  private:
    int status_;
};

inline void check(int status) {
    if (status == QSYNC_OK) return;
#ifdef QSYNC_B200_WITH_REFERENCE_ERRORS
    // qsync::fail prefixes "<kind>: " itself (errors.hpp:33); strip ours.
    std::string msg = qsync_last_error();
    const std::string tag = std::string(qsync_status_name(status)) + ": ";
    if (msg.rfind(tag, 0) == 0) msg = msg.substr(tag.size());
    qsync::fail(static_cast<qsync::ErrorKind>(status - 1), msg);
#else
    throw Error(status, qsync_last_error());
#endif
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(QSYNC_ERR_INTERNAL, std::string("internal: ") + what + ": " + cudaGetErrorString(e));
}

/// RAII device buffer.
template <typename T>
class DeviceBuffer {
  public:
    explicit DeviceBuffer(size_t n) : n_(n) {
        if (n_) cuda_check(cudaMalloc(&p_, n_ * sizeof(T)), "cudaMalloc");
    }
    ~DeviceBuffer() {
        if (p_) cudaFree(p_);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    T* get() const { return p_; }
    void upload(const T* h) { cuda_check(cudaMemcpy(p_, h, n_ * sizeof(T), cudaMemcpyHostToDevice), "H2D"); }
    void download(T* h) const { cuda_check(cudaMemcpy(h, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "D2H"); }

  private:
    size_t n_;
    T* p_ = nullptr;
};

/// Result layout of qsync::StochasticRoundResult (indicator.hpp:77-80).
struct StochasticRoundResult {
    std::vector<std::int64_t> rounded;
    std::vector<double> dequantized;
};

/// Device qsync::stochastic_round: element i uses draw i of a fresh
/// std::mt19937_64(seed); x_bar = (x - zp) / q in FP64; round up iff
/// uniform01 < frac (indicator.cpp:176-193).  Domain error if q <= 0.
inline StochasticRoundResult stochastic_round(const std::vector<double>& values, double q,
                                              double zp, std::uint64_t seed,
                                              cudaStream_t stream = nullptr) {
    StochasticRoundResult r;
    const size_t n = values.size();
    r.rounded.resize(n);
    r.dequantized.resize(n);
    DeviceBuffer<double> x(n), d(n);
    DeviceBuffer<std::int64_t> o(n);
    if (n) x.upload(values.data());
    check(qsync_stochastic_round_f64(x.get(), static_cast<int64_t>(n), q, zp, seed, o.get(),
                                     d.get(), stream));
    cuda_check(cudaStreamSynchronize(stream), "sync");
    if (n) {
        o.download(r.rounded.data());
        d.download(r.dequantized.data());
    }
    return r;
}

/// Device qsync::stochastic_round_float: spacing 2^(e-k) (indicator.cpp:195-200).
inline std::vector<double> stochastic_round_float(const std::vector<double>& values, int e, int k,
                                                  std::uint64_t seed, cudaStream_t stream = nullptr) {
    std::vector<double> out(values.size());
    DeviceBuffer<double> x(values.size()), d(values.size());
    if (!values.empty()) x.upload(values.data());
    check(qsync_stochastic_round_float_f64(x.get(), static_cast<int64_t>(values.size()), e, k,
                                           seed, d.get(), stream));
    cuda_check(cudaStreamSynchronize(stream), "sync");
    if (!values.empty()) d.download(out.data());
    return out;
}

/// OpStats-layout statistics of one device tensor (profile.hpp:95-108):
/// {||x||^2, absmax, q = absmax/127, e = floor(log2 absmax), numel}.
struct TensorStats5 {
    double norm_sq, absmax, q, e, numel;
};

inline TensorStats5 tensor_stats(const void* device_x, int dtype, int64_t n,
                                 cudaStream_t stream = nullptr) {
    DeviceBuffer<double> out(5);
    DeviceBuffer<unsigned char> ws(qsync_stats_workspace_bytes());
    check(qsync_tensor_stats(device_x, dtype, n, out.get(), ws.get(), stream));
    cuda_check(cudaStreamSynchronize(stream), "sync");
    double h[5];
    out.download(h);
    return {h[0], h[1], h[2], h[3], h[4]};
}

/// One rank's NCCL communicator for the data-parallel gradient exchange (C1):
/// the in-order bucket all-reduce whose slots the replayer models
/// (profile.hpp:118-129, replayer.cpp:48-73).  Rank 0 creates the id with
/// unique_id(); the caller broadcasts it (MPI, a file, a TCP store ...).
class Communicator {
  public:
    using Id = std::vector<std::uint8_t>;
    static Id unique_id() {
        Id id(QSYNC_COMM_ID_BYTES);
        check(qsync_comm_unique_id(id.data()));
        return id;
    }
    /// Collective over the ranks; binds the CURRENT CUDA device.
    Communicator(int nranks, int rank, const Id& id) {
        if (id.size() != QSYNC_COMM_ID_BYTES)
            throw Error(QSYNC_ERR_VALIDATION, "validation: communicator id must be 128 bytes");
        check(qsync_comm_init(&c_, nranks, rank, id.data()));
    }
    ~Communicator() {
        if (c_) qsync_comm_destroy(c_);
    }
    Communicator(const Communicator&) = delete;
    Communicator& operator=(const Communicator&) = delete;
    int nranks() const {
        int n = 0;
        check(qsync_comm_info(c_, &n, nullptr, nullptr));
        return n;
    }
    int rank() const {
        int r = 0;
        check(qsync_comm_info(c_, nullptr, &r, nullptr));
        return r;
    }
    /// In-place FP32 bucket all-reduce on `stream` (mean over ranks by default).
    void allreduce_bucket(float* device_buf, std::int64_t count, cudaStream_t stream = nullptr,
                          bool average = true) {
        check(qsync_allreduce_bucket(c_, device_buf, count, average ? 1 : 0, stream));
    }

  private:
    qsync_comm_t c_ = nullptr;
};

}  // namespace qsync_b200

#endif  // QSYNC_B200_HPP

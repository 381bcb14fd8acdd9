// Drop-in check of the C++ host mirror (include/qsync_b200.hpp) on the device:
// the reference's own stochastic-rounding unit cases (tests/test_indicator.cpp:
// 206-275 in the reference) and acceptance criteria 1-3
// (tests/acceptance_main.cpp:84-151, tolerances :31-42), re-run against the
// device implementation with the same seeds, sizes and tolerances.
// Built and run by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "qsync_b200.hpp"

namespace {
int g_fail = 0;

void require(bool ok, const std::string& what) {
    std::printf("%s: %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++g_fail;
}

// rng.hpp:12-14
double uniform01(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

double fixed_var(double q, double d) { return q * q * d / 6.0; }               // indicator.cpp:35-39
double float_var(double e, int k, double d) {                                 // indicator.cpp:41-45
    return std::exp2(2.0 * e) * std::exp2(-2.0 * k) * d / 6.0;
}
}  // namespace

int main() {
    using namespace qsync_b200;
    // test_indicator.cpp:206-216 -- on-grid values untouched; q <= 0 is a domain error.
    {
        std::vector<double> v;
        for (int i = -8; i <= 8; ++i) v.push_back(0.25 * i + 0.5);
        auto r = stochastic_round(v, 0.25, 0.5, 123);
        bool ok = true;
        for (size_t i = 0; i < v.size(); ++i)
            ok = ok && r.dequantized[i] == v[i] && r.rounded[i] == static_cast<int64_t>(i) - 8;
        require(ok, "on-grid values untouched");
        bool threw = false;
        try {
            stochastic_round(v, 0.0, 0.0, 1);
        } catch (const Error& e) {
            threw = e.kind() == "domain" && std::string(e.what()).find("scaling factor") != std::string::npos;
        }
        require(threw, "q <= 0 raises domain: ... scaling factor");
    }
    // :218-228 -- reproducible per seed.
    {
        std::mt19937_64 rng(5);
        std::vector<double> v;
        for (int i = 0; i < 1000; ++i) v.push_back(uniform01(rng));
        auto a = stochastic_round(v, 0.01, 0.0, 42), b = stochastic_round(v, 0.01, 0.0, 42),
             c = stochastic_round(v, 0.01, 0.0, 43);
        require(a.rounded == b.rounded && a.dequantized == b.dequantized && a.rounded != c.rounded,
                "reproducible per seed");
    }
    // :230-238 -- midpoints round up half the time (3 sigma at 1e5).
    {
        std::vector<double> v(100000, 0.005);
        auto r = stochastic_round(v, 0.01, 0.0, 2024);
        double mean = 0;
        for (auto x : r.rounded) mean += static_cast<double>(x);
        mean /= static_cast<double>(r.rounded.size());
        require(std::abs(mean - 0.5) <= 3.0 * 0.5 / std::sqrt(100000.0), "midpoint mean within 3 sigma");
    }
    // :240-253 -- variance within 10% of q^2 D / 6.
    {
        std::mt19937_64 rng(99);
        std::vector<double> v;
        for (int i = 0; i < 10000; ++i) v.push_back(uniform01(rng));
        auto r = stochastic_round(v, 0.01, 0.0, 7);
        double sq = 0;
        for (size_t i = 0; i < v.size(); ++i) sq += (r.dequantized[i] - v[i]) * (r.dequantized[i] - v[i]);
        require(std::abs(sq / fixed_var(0.01, 10000) - 1.0) <= 0.10, "fixed-point variance within 10%");
    }
    // :255-275 -- float grid.
    {
        std::vector<double> v{0.0, std::exp2(-8), 3 * std::exp2(-8), 1.0};
        require(stochastic_round_float(v, 1, 9, 11) == v, "float grid: on-grid exact");
        std::mt19937_64 rng(17);
        std::vector<double> rv;
        for (int i = 0; i < 10000; ++i) rv.push_back(uniform01(rng));
        auto out = stochastic_round_float(rv, 0, 9, 13);
        double sq = 0;
        for (size_t i = 0; i < rv.size(); ++i) sq += (out[i] - rv[i]) * (out[i] - rv[i]);
        require(std::abs(sq / float_var(0, 9, 10000) - 1.0) <= 0.10, "float variance within 10%");
        bool threw = false;
        try {
            stochastic_round_float(v, 0, 0, 1);
        } catch (const Error& e) {
            threw = e.kind() == "domain" && std::string(e.what()).find("mantissa") != std::string::npos;
        }
        require(threw, "k < 1 raises domain: ... mantissa");
    }
    // Acceptance criterion 1 (acceptance_main.cpp:84-105): 100 x 1e5, tolerance 3%.
    {
        const double q = 0.01;
        const int d = 100000, reps = 100;
        double total = 0;
        for (int rep = 0; rep < reps; ++rep) {
            std::mt19937_64 rng(1000 + rep);
            std::vector<double> v(d);
            for (double& x : v) x = uniform01(rng);
            auto r = stochastic_round(v, q, 0.0, 2000 + rep);
            double s = 0;
            for (int i = 0; i < d; ++i) s += (r.dequantized[i] - v[i]) * (r.dequantized[i] - v[i]);
            total += s;
        }
        const double ratio = total / reps / fixed_var(q, d);
        require(std::abs(ratio - 1.0) <= 0.03, "criterion 1: fixed-point variance ratio " + std::to_string(ratio));
    }
    // Criterion 2 (:107-129): 20 x 1e5 on the FP16 grid (k = 9), tolerance 5%.
    {
        const int d = 100000, reps = 20;
        double total = 0;
        for (int rep = 0; rep < reps; ++rep) {
            std::mt19937_64 rng(3000 + rep);
            std::vector<double> v(d);
            for (double& x : v) x = uniform01(rng);
            auto out = stochastic_round_float(v, 0, 9, 4000 + rep);
            double s = 0;
            for (int i = 0; i < d; ++i) s += (out[i] - v[i]) * (out[i] - v[i]);
            total += s;
        }
        const double ratio = total / reps / float_var(0, 9, d);
        require(std::abs(ratio - 1.0) <= 0.05, "criterion 2: float variance ratio " + std::to_string(ratio));
    }
    // Criterion 3 (:131-151): unbiasedness at 1e6, 3 sigma.
    {
        const double q = 0.01;
        const int d = 1000000;
        std::mt19937_64 rng(5005);
        std::vector<double> v(d);
        double in_mean = 0;
        for (double& x : v) {
            x = uniform01(rng);
            in_mean += x;
        }
        in_mean /= d;
        auto r = stochastic_round(v, q, 0.0, 6006);
        double out_mean = 0;
        for (double x : r.dequantized) out_mean += x;
        out_mean /= d;
        const double limit = 3.0 * q / (2.0 * std::sqrt(static_cast<double>(d)));
        require(std::abs(out_mean - in_mean) <= limit, "criterion 3: unbiased within 3 sigma");
    }
    // C1: the gradient exchange through the C++ mirror -- a 1-rank communicator
    // (the box has one GPU), in-place bucket mean is the identity.
    {
        Communicator comm(1, 0, Communicator::unique_id());
        const int n = 1 << 20;
        std::vector<float> h(n), back(n);
        for (int i = 0; i < n; ++i) h[i] = static_cast<float>(i % 977) * 0.5f - 100.0f;
        DeviceBuffer<float> g(n);
        g.upload(h.data());
        comm.allreduce_bucket(g.get(), n);
        cuda_check(cudaDeviceSynchronize(), "sync");
        g.download(back.data());
        require(comm.nranks() == 1 && comm.rank() == 0 && back == h, "1-rank bucket all-reduce is the identity");
        bool threw = false;
        try {
            Communicator bad(2, 7, Communicator::unique_id());
        } catch (const Error& e) {
            threw = e.kind() == "domain";
        }
        require(threw, "rank outside [0, nranks) raises domain");
    }
    std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASS", g_fail);
    return g_fail ? 1 : 0;
}

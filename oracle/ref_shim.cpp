// oracle/ref_shim.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/cpu_ref.c header).  Compiled together with
// /root/reference/proj/src/{errors,graph,profile,indicator,cost_mapper,replayer,
// allocator}.cpp by oracle/Makefile into oracle/_ref/libqsync_ref.so.  Nothing of
// the reference is copied: the sources are compiled where they lie.
//
// Used to pin the CPU restatement (cpu_ref.c) and the device path against the
// reference's own code: stochastic_round (indicator.cpp:176-193),
// stochastic_round_float (:195-200), sigma_fwd/sigma_bwd/omega (:65-132),
// reduce_stats (profile.cpp:134-162) and score_all on a bundle (:144-162).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "qsync/allocator.hpp"
#include "qsync/graph.hpp"
#include "qsync/indicator.hpp"
#include "qsync/replayer.hpp"
#include "qsync/profile.hpp"
#include "qsync/rng.hpp"

using namespace qsync;

namespace {
thread_local std::string g_err;

int code_of(const Error& e) { return static_cast<int>(e.kind()) + 1; }

// OpStats <-> (values[12], present-mask) in profile.hpp:95-108 field order.
OpStats unpack(const double* v, uint32_t mask) {
    OpStats s;
    std::optional<double> OpStats::*f[12] = {
        &OpStats::norm_w_sq, &OpStats::norm_act_sq, &OpStats::norm_grad_act_sq,
        &OpStats::norm_grad_act_hat_sq, &OpStats::d_act, &OpStats::d_w, &OpStats::d_grad,
        &OpStats::q_act, &OpStats::q_w, &OpStats::e_act, &OpStats::e_w, &OpStats::e_grad};
    for (int i = 0; i < 12; ++i)
        if (mask & (1u << i)) s.*f[i] = v[i];
    return s;
}
}  // namespace

extern "C" {

const char* qref_last_error() { return g_err.c_str(); }

int qref_stochastic_round(const double* x, int64_t n, double q, double zp, uint64_t seed,
                          int64_t* rounded, double* dequantized) {
    try {
        std::vector<double> v(x, x + n);
        StochasticRoundResult r = stochastic_round(v, q, zp, seed);
        if (rounded) std::memcpy(rounded, r.rounded.data(), sizeof(int64_t) * n);
        if (dequantized) std::memcpy(dequantized, r.dequantized.data(), sizeof(double) * n);
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return code_of(e);
    }
}

int qref_stochastic_round_float(const double* x, int64_t n, int e, int k, uint64_t seed,
                                double* out) {
    try {
        std::vector<double> v(x, x + n);
        std::vector<double> r = stochastic_round_float(v, e, k, seed);
        std::memcpy(out, r.data(), sizeof(double) * n);
        return 0;
    } catch (const Error& err) {
        g_err = err.what();
        return code_of(err);
    }
}

void qref_mt64_draws(uint64_t seed, int64_t n, uint64_t* out) {
    std::mt19937_64 rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng();
}

void qref_uniform01(uint64_t seed, int64_t n, double* out) {
    std::mt19937_64 rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = uniform01(rng);
}

// which: 0 = sigma_fwd, 1 = sigma_bwd.  precision: 0 INT8, 1 FP16, 2 FP32.
int qref_sigma(int which, const double* v, uint32_t mask, int precision, int parameter_free,
               int k, double* out) {
    try {
        OpStats s = unpack(v, mask);
        Precision p = static_cast<Precision>(precision);
        *out = which == 0 ? sigma_fwd(s, p, "op", parameter_free != 0, k)
                          : sigma_bwd(s, p, "op", parameter_free != 0, k);
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return code_of(e);
    }
}

int qref_omega(const double* v, uint32_t mask, int has_weight, int depth, int d_l, int loss_kind,
               int64_t loss_n, int precision, int k, double* out) {
    try {
        OperatorNode node;
        node.id = "op";
        node.kind = OperatorKind::Adjustable;
        node.depth = depth;
        node.has_weight = has_weight != 0;
        TensorStats ts;
        ts.per_op["op"] = unpack(v, mask);
        LossSpec loss{static_cast<LossKind>(loss_kind), loss_n};
        *out = omega(node, static_cast<Precision>(precision), d_l, loss, ts, k);
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return code_of(e);
    }
}

// reduce_stats over `snaps` snapshots of one operator: values[snaps][12], masks[snaps].
int qref_reduce_stats(const double* values, const uint32_t* masks, int snaps, int window,
                      double* out, uint32_t* out_mask) {
    try {
        std::vector<TensorStats> per_it(snaps);
        for (int i = 0; i < snaps; ++i) per_it[i].per_op["op"] = unpack(values + 12 * i, masks[i]);
        TensorStats r = reduce_stats(per_it, window);
        const OpStats& s = r.per_op.at("op");
        const std::optional<double>* f[12] = {&s.norm_w_sq, &s.norm_act_sq, &s.norm_grad_act_sq,
                                              &s.norm_grad_act_hat_sq, &s.d_act, &s.d_w,
                                              &s.d_grad, &s.q_act, &s.q_w, &s.e_act, &s.e_w,
                                              &s.e_grad};
        *out_mask = 0;
        for (int i = 0; i < 12; ++i) {
            out[i] = f[i]->has_value() ? **f[i] : 0.0;
            if (f[i]->has_value()) *out_mask |= 1u << i;
        }
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return code_of(e);
    }
}

// score_all over a bundle file; writes up to cap (op, precision, omega) rows as
// "op\tPREC\tomega\n" text into buf.  Returns bytes written or -code.
int64_t qref_score_bundle(const char* path, int loss_kind, int64_t loss_n, int window, char* buf,
                          int64_t cap) {
    try {
        ProfileBundle b = load_profile(path);
        PerturbationTable t = score_all(b.graph, b.reduced_stats(window),
                                        LossSpec{static_cast<LossKind>(loss_kind), loss_n});
        std::string out;
        char line[256];
        for (const auto& [op, row] : t.per_op)
            for (const auto& [p, e] : row) {
                std::snprintf(line, sizeof line, "%s\t%s\t%.17g\n", op.c_str(), precision_name(p),
                              e.omega);
                out += line;
            }
        if (static_cast<int64_t>(out.size()) > cap) return -100;
        std::memcpy(buf, out.data(), out.size());
        return static_cast<int64_t>(out.size());
    } catch (const Error& e) {
        g_err = e.what();
        return -code_of(e);
    }
}

// The reference's `plan` subcommand (cli.cpp:116-136) on a bundle file: writes
// the solve_report JSON (allocator.cpp:404-437) into buf.  cap_device/cap_bytes
// give one inference device's memory cap.  Returns bytes written or -code.
int64_t qref_plan_bundle(const char* path, int loss_kind, int64_t loss_n, int window,
                         const char* cap_device, int64_t cap_bytes, int b_max, char* buf,
                         int64_t cap) {
    try {
        const ProfileBundle bundle = load_profile(path);
        const TensorStats stats =
            bundle.tensor_stats.empty() ? TensorStats{} : bundle.reduced_stats(window);
        AllocProblem problem;
        problem.bundle = &bundle;
        problem.loss = LossSpec{static_cast<LossKind>(loss_kind), loss_n};
        problem.scores = score_all(bundle.graph, stats, problem.loss);
        if (cap_device && cap_device[0]) problem.mem_caps[cap_device] = cap_bytes;
        problem.b_max = b_max;
        const SolveResult result = solve(problem);
        const std::string out = solve_report(result).dump();
        if (static_cast<int64_t>(out.size()) > cap) return -100;
        std::memcpy(buf, out.data(), out.size());
        return static_cast<int64_t>(out.size());
    } catch (const Error& e) {
        g_err = e.what();
        return -code_of(e);
    }
}

// The reference's `replay` (cli.cpp:90-114): simulate one iteration of the
// bundle under a plan JSON ({"per_device": ...}); returns makespan ns or -code.
int64_t qref_replay_bundle(const char* path, const char* plan_json) {
    try {
        const ProfileBundle bundle = load_profile(path);
        const PrecisionPlan plan = plan_from_json(nlohmann::json::parse(plan_json));
        const Timeline t = simulate(build_global_dfg(bundle, plan).global);
        return t.makespan_ns;
    } catch (const Error& e) {
        g_err = e.what();
        return -code_of(e);
    }
}

// The replayer's Chrome trace (trace_to_json, replayer.cpp:126-148) of one
// simulated iteration; writes the JSON into buf.  Returns bytes or -code.
int64_t qref_replay_trace(const char* path, const char* plan_json, char* buf, int64_t cap) {
    try {
        const ProfileBundle bundle = load_profile(path);
        const PrecisionPlan plan = plan_from_json(nlohmann::json::parse(plan_json));
        const Timeline t = simulate(build_global_dfg(bundle, plan).global);
        const std::string out = trace_to_json(t).dump();
        if (static_cast<int64_t>(out.size()) > cap) return -100;
        std::memcpy(buf, out.data(), out.size());
        return static_cast<int64_t>(out.size());
    } catch (const Error& e) {
        g_err = e.what();
        return -code_of(e);
    }
}

}  // extern "C"

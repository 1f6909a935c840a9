// parcop_b200.hpp — the reference's `parcop::` C++ entry points for the hot
// path, re-implemented over the C-ABI (parcop_b200.h) so existing callers are
// source-compatible: same names, argument meaning, return types and exception
// types as /root/reference/proj/include/parcop (present pieces) and
// /root/reference/SPEC.md (absent estimator / partition-combine modules).
//
//   normalized_ranks     pseudo_obs.hpp:71-77
//   pseudo_loglik
//   fit
//   asymptotic_variance
//   partition
//   combine
//   fit_parallel
//
// Include this header INSTEAD of the reference headers (the types below
// mirror pseudo_obs.hpp:15-28 and copula.hpp:25). Link -lparcop_b200.
// Errors: std::invalid_argument / std::domain_error exactly where the
// reference throws them; std::runtime_error for device failures and for a
// combine with no converged block.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "parcop_b200.h"

namespace parcop {
inline namespace b200 {

enum class CopulaFamily { Gaussian, Frank, Gumbel };  // copula.hpp:25
enum class Scheme { Contiguous, Strided };

struct DataMatrix {  // pseudo_obs.hpp:15-20
    std::vector<double> col1;
    std::vector<double> col2;
    std::size_t rows() const { return col1.size(); }
};

struct PseudoSample {  // pseudo_obs.hpp:23-28
    std::vector<double> u1;
    std::vector<double> u2;
    std::size_t rows() const { return u1.size(); }
};

struct FitResult {
    double theta_hat = 0.0;
    double sigma2 = 0.0;
    std::size_t n = 0;
    double loglik = 0.0;
    int iterations = 0;
    bool converged = false;
};

struct Partition {  // SPEC.md:263-267 (row offsets of the scheme's row order)
    std::vector<std::uint64_t> offsets;
    Scheme scheme = Scheme::Contiguous;
    std::size_t blocks() const { return offsets.empty() ? 0 : offsets.size() - 1; }
};

struct CombinedResult {
    double theta_combined = 0.0;
    std::vector<FitResult> per_block;
    std::vector<double> weights;
    double wall_clock_per_block = 0.0;
    std::size_t blocks_used = 0;
};

namespace detail {

inline void rethrow(pcb_context* ctx, int rc) {
    if (rc == PCB_OK) return;
    const std::string msg = pcb_last_error(ctx);
    if (rc == PCB_E_INVALID) throw std::invalid_argument(msg);
    if (rc == PCB_E_DOMAIN) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}

// One context per host thread (SURVEY.md §8(b) threading rule), device 0
// unless set_device() is called first on that thread.
struct CtxHolder {
    int device = 0;
    pcb_context* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) pcb_destroy(ctx);
    }
};
inline CtxHolder& holder() {
    thread_local CtxHolder h;
    return h;
}
inline pcb_context* ctx() {
    CtxHolder& h = holder();
    if (!h.ctx) {
        h.ctx = pcb_create(h.device);
        if (!h.ctx) throw std::runtime_error(pcb_last_error(nullptr));
    }
    return h.ctx;
}

inline FitResult to_fit(const pcb_fit_result& r) {
    FitResult f;
    f.theta_hat = r.theta_hat;
    f.sigma2 = r.sigma2;
    f.n = static_cast<std::size_t>(r.n);
    f.loglik = r.loglik;
    f.iterations = r.iterations;
    f.converged = r.converged != 0;
    return f;
}

inline void check_pseudo(const PseudoSample& u) {
    if (u.u1.size() != u.u2.size()) throw std::invalid_argument("pseudo sample: columns differ in length");
}

}  // namespace detail

inline void set_device(int device) {
    detail::CtxHolder& h = detail::holder();
    if (h.ctx) {
        pcb_destroy(h.ctx);
        h.ctx = nullptr;
    }
    h.device = device;
}

inline PseudoSample normalized_ranks(const DataMatrix& x) {
    if (x.col1.size() != x.col2.size()) throw std::invalid_argument("data matrix: columns differ in length");
    if (x.rows() < 2) throw std::invalid_argument("data matrix: need at least 2 rows");
    PseudoSample p;
    p.u1.resize(x.rows());
    p.u2.resize(x.rows());
    const std::uint64_t off[2] = {0, x.rows()};
    pcb_context* c = detail::ctx();
    detail::rethrow(c, pcb_normalized_ranks(c, x.col1.data(), x.col2.data(), x.rows(), off, 1, p.u1.data(),
                                            p.u2.data()));
    return p;
}

inline double pseudo_loglik(CopulaFamily f, double theta, const PseudoSample& u) {
    detail::check_pseudo(u);
    const std::uint64_t off[2] = {0, u.rows()};
    double out = 0.0;
    pcb_context* c = detail::ctx();
    detail::rethrow(c, pcb_pseudo_loglik(c, static_cast<int>(f), &theta, u.u1.data(), u.u2.data(), u.rows(), off, 1,
                                         &out));
    return out;
}

inline FitResult fit(CopulaFamily f, const PseudoSample& u) {
    detail::check_pseudo(u);
    const std::uint64_t off[2] = {0, u.rows()};
    pcb_fit_result r{};
    pcb_context* c = detail::ctx();
    detail::rethrow(c, pcb_fit(c, static_cast<int>(f), PCB_FP64, u.u1.data(), u.u2.data(), u.rows(), off, 1, &r));
    return detail::to_fit(r);
}

inline double asymptotic_variance(CopulaFamily f, double theta_hat, const PseudoSample& u) {
    detail::check_pseudo(u);
    const std::uint64_t off[2] = {0, u.rows()};
    double s2 = 0.0;
    pcb_context* c = detail::ctx();
    detail::rethrow(c, pcb_asymptotic_variance(c, static_cast<int>(f), &theta_hat, u.u1.data(), u.u2.data(),
                                               u.rows(), off, 1, &s2));
    return s2;
}

inline Partition partition(const DataMatrix& x, std::size_t m, Scheme scheme = Scheme::Contiguous) {
    if (m < 1) throw std::invalid_argument("partition: need M >= 1");
    Partition p;
    p.scheme = scheme;
    p.offsets.resize(m + 1);
    if (pcb_partition(x.rows(), m, static_cast<int>(scheme), p.offsets.data()) != PCB_OK)
        throw std::invalid_argument("partition: block below the 30-row floor");
    return p;
}

inline CombinedResult combine(const std::vector<FitResult>& results) {
    if (results.empty()) throw std::invalid_argument("combine: empty input");
    std::vector<pcb_fit_result> in(results.size());
    for (std::size_t i = 0; i < results.size(); ++i) {
        in[i] = pcb_fit_result{results[i].theta_hat, results[i].sigma2, results[i].loglik, results[i].n,
                               results[i].iterations, results[i].converged ? 1 : 0, 0, 0};
    }
    CombinedResult out;
    out.per_block = results;
    out.weights.resize(results.size());
    pcb_combined cr{};
    pcb_context* c = detail::ctx();
    detail::rethrow(c, pcb_combine(c, in.data(), in.size(), out.weights.data(), &cr));
    out.theta_combined = cr.theta_combined;
    out.blocks_used = static_cast<std::size_t>(cr.blocks_used);
    return out;
}

// `workers` is kept for source compatibility; blocks run on the GPU's SMs
// and the result is bitwise independent of it.
inline CombinedResult fit_parallel(CopulaFamily f, const DataMatrix& x, std::size_t m, std::size_t workers = 0,
                                   Scheme scheme = Scheme::Contiguous) {
    (void)workers;
    if (x.col1.size() != x.col2.size()) throw std::invalid_argument("data matrix: columns differ in length");
    std::vector<pcb_fit_result> per(m);
    CombinedResult out;
    out.weights.resize(m);
    pcb_combined cr{};
    pcb_context* c = detail::ctx();
    detail::rethrow(c, pcb_fit_parallel(c, static_cast<int>(f), PCB_FP64, x.col1.data(), x.col2.data(), x.rows(), m,
                                        static_cast<int>(scheme), per.data(), out.weights.data(), &cr));
    out.theta_combined = cr.theta_combined;
    out.blocks_used = static_cast<std::size_t>(cr.blocks_used);
    out.per_block.reserve(m);
    for (const auto& r : per) out.per_block.push_back(detail::to_fit(r));
    return out;
}

// sim_study rel_l1 / rel_l2, tensor Gauss-Legendre on device
inline double rel_l1(CopulaFamily f, double theta_a, double theta_b, int quad_nodes = 200) {
    double l1 = 0.0, l2 = 0.0;
    pcb_context* c = detail::ctx();
    detail::rethrow(c, pcb_rel_error(c, static_cast<int>(f), theta_a, theta_b, quad_nodes, &l1, &l2));
    return l1;
}

inline double rel_l2(CopulaFamily f, double theta_a, double theta_b, int quad_nodes = 200) {
    double l1 = 0.0, l2 = 0.0;
    pcb_context* c = detail::ctx();
    detail::rethrow(c, pcb_rel_error(c, static_cast<int>(f), theta_a, theta_b, quad_nodes, &l1, &l2));
    return l2;
}

}  // namespace b200
}  // namespace parcop

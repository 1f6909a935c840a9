// parcop_b200.hpp — the reference's `parcop::` C++ entry points for the hot
// path, re-implemented over the C-ABI (parcop_b200.h) so existing callers are
// source-compatible: same names, argument meaning, return types and exception
// types as /root/reference/proj/include/parcop (present pieces) and
// /root/reference/SPEC.md (absent estimator / partition-combine modules).
//
//   pseudo_loglik
//   fit
//   asymptotic_variance
//   partition            SPEC.md:275-283  (Partition holds the blocks)
//   combine
//   fit_parallel         SPEC.md:293-301  (wall_clock_per_block filled)
//   b200::normalized_ranks  pseudo_obs.hpp:71-77 on the GPU (opt-in name)
//
// Types. When the reference headers are on the include path
// (`-I…/proj/include`), this header includes <parcop/copula.hpp> and uses
// the reference's own DataMatrix, PseudoSample (pseudo_obs.hpp:15-28) and
// CopulaFamily (copula.hpp:25), so a translation unit can mix the two freely
// (sample with parcop::sample_matrix, fit with parcop::fit_parallel). It
// defines only the SPEC types the reference lacks (FitResult, Scheme,
// Partition, CombinedResult). The reference's parcop::normalized_ranks stays
// the CPU one; the device version is parcop::b200::normalized_ranks. Without
// the reference headers (or with PARCOP_B200_STANDALONE_TYPES defined), the
// three types are defined here with the reference's layout and
// parcop::normalized_ranks is the device version.
// (The reference's normal.hpp:21 needs std::numbers::inv_sqrt2, which C++20
// lacks: reference callers already compile it with their own definition,
// e.g. oracle/shim.hpp.)
//
// Devices. One context per host thread: device 0 unless
// parcop::b200::set_device / set_devices is called first on that thread.
// With several devices, fit_parallel shards the blocks over all of them
// (pcb_create_multi) and the result is bitwise the same.
//
// Errors: std::invalid_argument / std::domain_error exactly where the
// reference throws them; std::runtime_error for device failures and for a
// combine with no converged block. Link -lparcop_b200.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "parcop_b200.h"

#if !defined(PARCOP_B200_STANDALONE_TYPES) && defined(__has_include)
#if __has_include(<parcop/copula.hpp>)
#define PARCOP_B200_REFERENCE_TYPES 1
#endif
#endif

#if defined(PARCOP_B200_REFERENCE_TYPES)
#include <parcop/copula.hpp>  // CopulaFamily (copula.hpp:25); DataMatrix, PseudoSample (pseudo_obs.hpp:15-28)
#else
namespace parcop {

enum class CopulaFamily { Gaussian, Frank, Gumbel };  // copula.hpp:25

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

inline void validate_data(const DataMatrix& x) {  // pseudo_obs.hpp:30-37
    if (x.col1.size() != x.col2.size()) throw std::invalid_argument("data matrix: columns differ in length");
    if (x.rows() < 2) throw std::invalid_argument("data matrix: need at least 2 rows");
    for (std::size_t i = 0; i < x.rows(); ++i)
        if (!std::isfinite(x.col1[i]) || !std::isfinite(x.col2[i]))
            throw std::domain_error("data matrix: non-finite value");
}

inline void validate_pseudo_sample(const PseudoSample& u) {  // pseudo_obs.hpp:79-88
    if (u.u1.size() != u.u2.size()) throw std::invalid_argument("pseudo sample: columns differ in length");
    for (std::size_t i = 0; i < u.rows(); ++i)
        if (!(u.u1[i] > 0.0 && u.u1[i] < 1.0) || !(u.u2[i] > 0.0 && u.u2[i] < 1.0))
            throw std::domain_error("pseudo sample: values must lie strictly in (0,1)");
}

}  // namespace parcop
#endif

namespace parcop {

// ---------------------------------------------------- SPEC types the reference lacks
enum class Scheme { Contiguous, Strided };

struct FitResult {
    double theta_hat = 0.0;
    double sigma2 = 0.0;
    std::size_t n = 0;
    double loglik = 0.0;
    int iterations = 0;
    bool converged = false;
};

struct Partition {
    std::vector<DataMatrix> blocks;  // ordered row-blocks, pairwise disjoint, covering X
    Scheme scheme = Scheme::Contiguous;
    // B200 extension: the blocks' row offsets in the scheme's row order
    // (Contiguous: rows of X; Strided: X gathered so block m = rows i ≡ m mod M)
    std::vector<std::uint64_t> offsets;
    std::size_t size() const { return blocks.size(); }
};

struct CombinedResult {
    double theta_combined = 0.0;
    std::vector<FitResult> per_block;
    std::vector<double> weights;
    double wall_clock_per_block = 0.0;  // seconds
    std::size_t blocks_used = 0;
};

namespace b200 {

namespace detail {

inline void rethrow(pcb_context* ctx, int rc) {
    if (rc == PCB_OK) return;
    const std::string msg = pcb_last_error(ctx);
    if (rc == PCB_E_INVALID) throw std::invalid_argument(msg);
    if (rc == PCB_E_DOMAIN) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}

struct CtxHolder {
    std::vector<int> devices{0};
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
        h.ctx = pcb_create_multi(h.devices.data(), static_cast<int>(h.devices.size()));
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

// The GPUs this thread's context spans (default {0}).
inline void set_devices(const std::vector<int>& devices) {
    if (devices.empty()) throw std::invalid_argument("set_devices: need at least one device");
    detail::CtxHolder& h = detail::holder();
    if (h.ctx) {
        pcb_destroy(h.ctx);
        h.ctx = nullptr;
    }
    h.devices = devices;
}
inline void set_device(int device) { set_devices({device}); }

// pseudo_obs.hpp:71-77 on the device, bit-identical to the reference.
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

// the blocks themselves (row copies), scheme order.
inline Partition partition(const DataMatrix& x, std::size_t m, Scheme scheme = Scheme::Contiguous) {
    if (m < 1) throw std::invalid_argument("partition: need M >= 1");
    if (x.col1.size() != x.col2.size()) throw std::invalid_argument("data matrix: columns differ in length");
    Partition p;
    p.scheme = scheme;
    p.offsets.resize(m + 1);
    if (pcb_partition(x.rows(), m, static_cast<int>(scheme), p.offsets.data()) != PCB_OK)
        throw std::invalid_argument("partition: block below the 30-row floor");
    p.blocks.resize(m);
    for (std::size_t b = 0; b < m; ++b) {
        DataMatrix& blk = p.blocks[b];
        const std::size_t len = static_cast<std::size_t>(p.offsets[b + 1] - p.offsets[b]);
        blk.col1.resize(len);
        blk.col2.resize(len);
        for (std::size_t k = 0; k < len; ++k) {
            const std::size_t row = scheme == Scheme::Contiguous ? static_cast<std::size_t>(p.offsets[b]) + k : b + k * m;
            blk.col1[k] = x.col1[row];
            blk.col2[k] = x.col2[row];
        }
    }
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

// `workers` is kept for source compatibility; blocks run on the GPUs' SMs
// and the result is bitwise independent of it. Host columns
// (pinned or pageable) stream to the device(s) while earlier blocks compute.
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
    out.wall_clock_per_block = cr.wall_clock_per_block;
    out.per_block.reserve(m);
    for (const auto& r : per) out.per_block.push_back(detail::to_fit(r));
    return out;
}

// Device sampler (copula.hpp:359-410 transforms over counter-based
// splitmix64 streams): n rows as `blocks` seeded blocks.
inline DataMatrix sample_matrix_device(CopulaFamily f, double theta, std::size_t n, std::size_t blocks = 1,
                                       std::uint64_t base_seed = 0x160905530ull) {
    DataMatrix x;
    x.col1.resize(n);
    x.col2.resize(n);
    pcb_context* c = detail::ctx();
    detail::rethrow(c, pcb_sample(c, static_cast<int>(f), theta, n, blocks, 0, blocks, base_seed, x.col1.data(),
                                  x.col2.data()));
    return x;
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

// The SPEC operations the reference does not implement, under their SPEC
// names (no reference declaration to collide with).
using b200::asymptotic_variance;
using b200::combine;
using b200::fit;
using b200::fit_parallel;
using b200::partition;
using b200::pseudo_loglik;
using b200::rel_l1;
using b200::rel_l2;
using b200::set_device;
#if !defined(PARCOP_B200_REFERENCE_TYPES)
using b200::normalized_ranks;  // standalone: no reference normalized_ranks exists
#endif

}  // namespace parcop

// Drop-in check: ONE translation unit includes the reference's own headers
// (<parcop/copula.hpp>, compiled in place from /root/reference with the
// normal.hpp:21 shim every reference caller needs) AND parcop_b200.hpp. The
// reference's types are used throughout: it samples with the reference's
// parcop::sample_matrix (copula.hpp:413-423, std::mt19937_64 stream), ranks
// with the reference's parcop::normalized_ranks (CPU) and with
// parcop::b200::normalized_ranks (GPU, must be bit-identical), and fits with
// the B200 parcop::fit_parallel / parcop::fit. Built by tests/cpp/Makefile only
// where /root/reference exists; run on the GPU by tests/test_gpu_cpp.py.
#include <parcop/copula.hpp>
#include <parcop/pseudo_obs.hpp>

#include "parcop_b200.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <type_traits>

#ifndef PARCOP_B200_REFERENCE_TYPES
#error "parcop_b200.hpp did not pick up the reference types"
#endif

int main() {
    using namespace parcop;
    static_assert(std::is_same<decltype(DataMatrix{}.col1), std::vector<double>>::value, "reference DataMatrix");
    bool all = true;
    auto report = [&](const char* what, bool ok) {
        std::printf("%s %s\n", what, ok ? "ok" : "FAIL");
        all = all && ok;
    };
    for (CopulaFamily fam : {CopulaFamily::Gaussian, CopulaFamily::Frank, CopulaFamily::Gumbel}) {
        const double theta = fam == CopulaFamily::Gaussian ? 0.5 : fam == CopulaFamily::Frank ? 5.0 : 2.0;
        RngStream rng(mix_seed(0x160905530ull, {static_cast<std::uint64_t>(fam), 20000}));
        const DataMatrix x = sample_matrix(make_model(fam, theta), 20000, rng);  // the reference's sampler
        const PseudoSample ref = normalized_ranks(x);                            // the reference's CPU ranks
        const PseudoSample dev = b200::normalized_ranks(x);                      // B200
        const bool same = ref.u1.size() == dev.u1.size() &&
                          std::memcmp(ref.u1.data(), dev.u1.data(), ref.u1.size() * sizeof(double)) == 0 &&
                          std::memcmp(ref.u2.data(), dev.u2.data(), ref.u2.size() * sizeof(double)) == 0;
        report("ranks_bit_identical", same);
        validate_pseudo_sample(dev);  // the reference's validator accepts the device output
        const FitResult f = fit(fam, ref);
        const CombinedResult cr = fit_parallel(fam, x, 10, 4);
        const Partition p = partition(x, 10);
        double sum_w = 0.0, sum_wt = 0.0;
        bool blocks_ok = p.size() == 10;
        for (std::size_t b = 0; b < p.size() && blocks_ok; ++b) {
            const FitResult fb = fit(fam, b200::normalized_ranks(p.blocks[b]));
            // fit() on pseudo-observations and fit_parallel() on raw data take
            // different device routes (per-point transforms vs per-rank tables):
            // equal to rounding, both held to the oracle at 1e-9 elsewhere
            blocks_ok = fb.converged && std::fabs(fb.theta_hat - cr.per_block[b].theta_hat) <= 1e-12 * std::fabs(fb.theta_hat) &&
                        std::fabs(fb.sigma2 - cr.per_block[b].sigma2) <= 1e-11 * fb.sigma2;
            sum_w += 1.0 / fb.sigma2;
            sum_wt += fb.theta_hat / fb.sigma2;
        }
        report("partition_blocks_fit_equal", blocks_ok);
        report("fit_parallel", cr.blocks_used == 10 && std::fabs(cr.theta_combined - sum_wt / sum_w) <=
                                                           1e-11 * std::fabs(cr.theta_combined) &&
                                   cr.wall_clock_per_block > 0.0 && std::fabs(f.theta_hat - theta) < 0.1);
        std::printf("  family %d theta_full=%.12f theta_c=%.12f wall/block=%.3g s\n", static_cast<int>(fam),
                    f.theta_hat, cr.theta_combined, cr.wall_clock_per_block);
    }
    return all ? 0 : 1;
}

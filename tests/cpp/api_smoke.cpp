// C++ host API check: compiles against include/parcop_b200.hpp exactly as a
// reference caller would (parcop:: names), links libparcop_b200.so, and —
// when run on a B200 (tests/test_gpu_cpp.py) — exercises every entry point
// and the reference's exception types. Prints one line per check.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "parcop_b200.hpp"

int main() {
    using namespace parcop;
    // pseudo_obs examples
    DataMatrix x{{3.1, 1.2, 7.5}, {1.0, 1.0, 2.0}};
    PseudoSample u = normalized_ranks(x);
    const bool ranks_ok = u.u1[0] == 0.5 && u.u1[1] == 0.25 && u.u1[2] == 0.75 && u.u2[0] == 0.375 &&
                          u.u2[1] == 0.375 && u.u2[2] == 0.75;
    std::printf("ranks %s\n", ranks_ok ? "ok" : "FAIL");
    bool threw = false;
    try {
        normalized_ranks(DataMatrix{{1.0, NAN}, {1.0, 2.0}});
    } catch (const std::domain_error&) {
        threw = true;
    }
    std::printf("nonfinite domain_error %s\n", threw ? "ok" : "FAIL");
    // combine examples
    FitResult a, b;
    a.theta_hat = 0.2;
    a.sigma2 = 1.0;
    a.converged = true;
    b.theta_hat = 0.4;
    b.sigma2 = 4.0;
    b.converged = true;
    const CombinedResult cr = combine({a, b});
    std::printf("combine %s %.17g\n", std::fabs(cr.theta_combined - 0.24) < 1e-15 ? "ok" : "FAIL", cr.theta_combined);
    // partition example
    DataMatrix big;
    big.col1.resize(100);
    big.col2.resize(100);
    for (int i = 0; i < 100; ++i) big.col1[i] = i;
    const Partition p = partition(big, 3);
    const Partition ps = partition(big, 3, Scheme::Strided);  // row i -> block i mod M
    std::printf("partition %s\n", p.offsets[1] == 33 && p.offsets[3] == 100 && p.size() == 3 &&
                                         p.blocks[2].rows() == 34 && p.blocks[1].col1[0] == 33.0 &&
                                         ps.blocks[1].rows() == 33 && ps.blocks[1].col1[1] == 4.0
                                     ? "ok"
                                     : "FAIL");
    // a small fit_parallel on a deterministic dataset
    DataMatrix d;
    for (int i = 0; i < 3000; ++i) {
        const double s = std::sin(0.37 * i) + 0.5 * std::sin(1.91 * i + 0.3);
        d.col1.push_back(s + 0.3 * std::cos(0.71 * i));
        d.col2.push_back(s - 0.3 * std::cos(2.13 * i + 1.0));
    }
    const CombinedResult fp = fit_parallel(CopulaFamily::Gaussian, d, 3, 8);
    std::printf("fit_parallel %s theta_c=%.12f used=%zu\n",
                fp.blocks_used == 3 && std::isfinite(fp.theta_combined) && fp.wall_clock_per_block > 0.0 ? "ok"
                                                                                                       : "FAIL",
                fp.theta_combined, fp.blocks_used);
    const FitResult f = fit(CopulaFamily::Gaussian, normalized_ranks(d));
    const double s2 = asymptotic_variance(CopulaFamily::Gaussian, f.theta_hat, normalized_ranks(d));
    std::printf("fit %s theta=%.12f sigma2=%.6g\n", f.converged && std::fabs(s2 - f.sigma2) <= 1e-12 * s2 ? "ok" : "FAIL",
                f.theta_hat, f.sigma2);
    threw = false;
    try {
        pseudo_loglik(CopulaFamily::Gumbel, 0.5, normalized_ranks(d));
    } catch (const std::domain_error&) {
        threw = true;
    }
    std::printf("theta domain_error %s\n", threw ? "ok" : "FAIL");
    const double l1 = rel_l1(CopulaFamily::Frank, 5.0, 5.2, 64), l0 = rel_l2(CopulaFamily::Frank, 5.0, 5.0, 64);
    std::printf("rel_error %s l1=%.12g\n", l1 > 0.0 && l1 < 1.0 && l0 == 0.0 ? "ok" : "FAIL", l1);
    return 0;
}

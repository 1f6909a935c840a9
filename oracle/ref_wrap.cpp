// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/copula_math.hpp header).
//
// oracle/_ref/libparcop_ref.so: the reference's OWN headers
// (/root/reference/proj/include/parcop, compiled in place with shim.hpp, never
// copied) behind the same extern "C" surface as liboracle.so. The present
// reference pieces — normalized_rank_column (pseudo_obs.hpp:44-65), log_pdf
// (copula.hpp:293-311), detail::shc (copula.hpp:256-269), debye1
// (quadrature.hpp:115-120), sample_matrix + RngStream (copula.hpp:413-423,
// rng.hpp:32-63) — are called directly; the absent estimator/combine layers
// are the SPEC restatement in mpl_driver.hpp. Used to pin the oracle and as
// bench.py --impl reference's CPU path (cpu_baseline.kind = "reference").
#include <parcop/copula.hpp>
#include <parcop/pseudo_obs.hpp>
#include <parcop/quadrature.hpp>
#include <parcop/rng.hpp>

#include <cstring>

#include "mpl_driver.hpp"

namespace {

parcop::CopulaFamily fam_of(int f) { return static_cast<parcop::CopulaFamily>(f); }

struct RefMath {
    static void rank_column(const double* x, size_t n, double* u) {
        std::vector<double> col(x, x + n);
        const std::vector<double> r = parcop::detail::normalized_rank_column(col);
        std::memcpy(u, r.data(), n * sizeof(double));
    }
    static double log_density(int fam, double t, double u, double v) {
        return parcop::log_pdf(parcop::CopulaModel{fam_of(fam), t}, parcop::UnitPair{u, v});
    }
    static oracle::PointDerivs derivs(int fam, double t, double u, double v) {
        // what score_theta/hess_theta/cross_score evaluate (copula.hpp:316-334), once
        const parcop::detail::Shc s = parcop::detail::shc(parcop::CopulaModel{fam_of(fam), t},
                                                          parcop::detail::clamp_unit(u),
                                                          parcop::detail::clamp_unit(v));
        return oracle::PointDerivs{s.score, s.hess, s.cross1, s.cross2};
    }
    static double log_density_checked(int fam, double t, double u, double v) { return log_density(fam, t, u, v); }
    static oracle::PointDerivs derivs_checked(int fam, double t, double u, double v) {
        parcop::validate_model(parcop::CopulaModel{fam_of(fam), t});
        return derivs(fam, t, u, v);
    }
    static double debye1(double x) { return parcop::debye1(x); }
    static double cdf(int fam, double t, double u, double v) {
        return parcop::cdf(parcop::CopulaModel{fam_of(fam), t}, parcop::UnitPair{u, v});
    }
    static double spearman_rho(int fam, double t, int n) {
        const parcop::CopulaModel mdl{fam_of(fam), t};
        return 12.0 * parcop::integrate_unit_square(
                          [&](double u, double v) { return parcop::cdf(mdl, parcop::UnitPair{u, v}); }, n) -
               3.0;
    }
    // the reference's own tensor quadrature (quadrature.hpp:66-78) of its pdf (copula.hpp:313)
    static void rel_sums(int fam, double ta, double tb, int n, double out[4]) {
        const parcop::CopulaModel a{fam_of(fam), ta}, b{fam_of(fam), tb};
        auto pa = [&](double u, double v) { return parcop::pdf(a, parcop::UnitPair{u, v}); };
        auto pb = [&](double u, double v) { return parcop::pdf(b, parcop::UnitPair{u, v}); };
        out[0] = parcop::integrate_unit_square([&](double u, double v) { return std::fabs(pa(u, v) - pb(u, v)); }, n);
        out[1] = parcop::integrate_unit_square(
            [&](double u, double v) {
                const double d = pa(u, v) - pb(u, v);
                return d * d;
            },
            n);
        out[2] = parcop::integrate_unit_square(pa, n);
        out[3] = parcop::integrate_unit_square(
            [&](double u, double v) {
                const double f = pa(u, v);
                return f * f;
            },
            n);
    }
};

}  // namespace

#define MATH RefMath
#define PFX ref_
#include "exports.inc"

extern "C" {

// The reference's own generator: sample_matrix over RngStream(seed) (mt19937_64).
int ref_sample_matrix(int fam, double theta, uint64_t n, uint64_t seed, double* c1, double* c2) {
    return guarded([&] {
        parcop::RngStream rng(seed);
        const parcop::DataMatrix x = parcop::sample_matrix(parcop::CopulaModel{fam_of(fam), theta}, n, rng);
        std::memcpy(c1, x.col1.data(), n * sizeof(double));
        std::memcpy(c2, x.col2.data(), n * sizeof(double));
    });
}

uint64_t ref_mix_seed4(uint64_t base, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    return parcop::mix_seed(base, {a, b, c, d});
}

uint64_t ref_splitmix64(uint64_t z) { return parcop::splitmix64(z); }

}  // extern "C"

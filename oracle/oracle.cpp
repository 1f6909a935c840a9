// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/copula_math.hpp header).
//
// liboracle.so: the SPEC-restated driver (mpl_driver.hpp) over the oracle's
// own restated per-point arithmetic (copula_math.hpp), plus the
// counter-based input generator (sampler.hpp). Loaded by tests/ and bench.py's
// cpu_baseline leg through ctypes (oracle/oracle.py). Never linked by the
// product library.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "copula_math.hpp"
#include "mpl_driver.hpp"
#include "sampler.hpp"

namespace {

// quadrature.hpp:82-111 (adaptive Simpson) restated for debye1 (quadrature.hpp:115-120)
template <class F>
double simpson_rec(F& f, double a, double b, double fa, double fm, double fb, double whole, double tol, int depth) {
    const double m = 0.5 * (a + b), lm = 0.5 * (a + m), rm = 0.5 * (m + b);
    const double flm = f(lm), frm = f(rm);
    const double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm);
    const double right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
    const double delta = left + right - whole;
    if (depth <= 0 || std::fabs(delta) <= 15.0 * tol) return left + right + delta / 15.0;
    return simpson_rec(f, a, m, fa, flm, fm, left, 0.5 * tol, depth - 1) +
           simpson_rec(f, m, b, fm, frm, fb, right, 0.5 * tol, depth - 1);
}

double debye1_restated(double x) {
    if (x == 0.0) return 1.0;
    if (x < 0.0) return debye1_restated(-x) - x / 2.0;
    auto f = [](double t) { return t == 0.0 ? 1.0 : t / std::expm1(t); };
    const double fa = f(0.0), fm = f(0.5 * x), fb = f(x);
    const double whole = x / 6.0 * (fa + 4.0 * fm + fb);
    return simpson_rec(f, 0.0, x, fa, fm, fb, whole, 1e-13 * std::max(1.0, x), 48) / x;
}

// quadrature.hpp:22-62 restated: n-point Gauss-Legendre on (0, 1)
void gauss_legendre01_restated(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double z = std::cos(pi * (i + 0.75) / (n + 0.5)), dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = z;
            for (int j = 2; j <= n; ++j) {
                const double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (z * p1 - p0) / (z * z - 1.0);
            const double step = p1 / dp;
            z -= step;
            if (std::fabs(step) < 1e-15) break;
        }
        x[i] = -z;
        x[n - 1 - i] = z;
        w[i] = w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
    if (n % 2 == 1) x[n / 2] = 0.0;
    for (int i = 0; i < n; ++i) {
        x[i] = 0.5 * (x[i] + 1.0);
        w[i] *= 0.5;
    }
}

struct RestatedMath {
    // SPEC.md:362-374 sums over the tensor rule (quadrature.hpp:66-78 order:
    // row sums over j, then the weighted sum over rows i)
    static void rel_sums(int fam, double ta, double tb, int n, double out[4]) {
        std::vector<double> x, w;
        gauss_legendre01_restated(n, x, w);
        for (int k = 0; k < 4; ++k) out[k] = 0.0;
        for (int i = 0; i < n; ++i) {
            double row[4] = {0.0, 0.0, 0.0, 0.0};
            for (int j = 0; j < n; ++j) {
                const double fa = std::exp(oracle::log_density(fam, ta, x[i], x[j]));
                const double fb = std::exp(oracle::log_density(fam, tb, x[i], x[j]));
                const double d = fa - fb;
                row[0] += w[j] * std::fabs(d);
                row[1] += w[j] * (d * d);
                row[2] += w[j] * fa;
                row[3] += w[j] * (fa * fa);
            }
            for (int k = 0; k < 4; ++k) out[k] += w[i] * row[k];
        }
    }
    static void rank_column(const double* x, size_t n, double* u) { oracle::rank_column_restated(x, n, u); }
    static double log_density(int fam, double t, double u, double v) { return oracle::log_density(fam, t, u, v); }
    static oracle::PointDerivs derivs(int fam, double t, double u, double v) {
        return oracle::derivs(fam, t, oracle::clamp01(u), oracle::clamp01(v));
    }
    static double log_density_checked(int fam, double t, double u, double v) { return oracle::log_density(fam, t, u, v); }
    static oracle::PointDerivs derivs_checked(int fam, double t, double u, double v) {
        return oracle::point_derivs(fam, t, u, v);
    }
    static double debye1(double x) { return debye1_restated(x); }
};

}  // namespace

#define MATH RestatedMath
#define PFX orc_
#include "exports.inc"

extern "C" {

uint64_t orc_splitmix64(uint64_t z) { return oracle::splitmix64(z); }
uint64_t orc_mix_seed4(uint64_t base, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    return oracle::mix_seed4(base, a, b, c, d);
}
double orc_unit_draw(uint64_t seed, uint64_t d) { return oracle::unit_draw(seed, d); }

// Rows of blocks [first, last) of a partition `off` (K+1 offsets over n_total
// rows); block m is drawn from seed mix_seed(base, {fam, n_total, K, m}).
// Output row r of block b lands at index off[b] - off[first] + r.
int orc_sample_blocks(int fam, double theta, uint64_t n_total, uint64_t k, uint64_t base_seed, const uint64_t* off,
                      uint64_t first, uint64_t last, double* c1, double* c2, int workers) {
    if (!oracle::theta_ok(fam, theta)) return 3;
    if (workers < 1) workers = 1;
    std::atomic<uint64_t> next{first};
    auto work = [&]() {
        for (;;) {
            const uint64_t b = next.fetch_add(1);
            if (b >= last) return;
            const uint64_t seed = oracle::mix_seed4(base_seed, static_cast<uint64_t>(fam), n_total, k, b);
            const uint64_t base = off[b] - off[first];
            for (uint64_t i = 0; i < off[b + 1] - off[b]; ++i)
                oracle::sample_point(fam, theta, seed, i, c1 + base + i, c2 + base + i);
        }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < workers; ++w) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return 0;
}

}  // extern "C"

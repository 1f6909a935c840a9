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

// normal.hpp:97-155 restated (bvn_upper over the 6/12/20-node rules of bvn_rule)
double bvn_upper_restated(double h, double k, double r) {
    const double twopi = 2.0 * 3.14159265358979323846;
    const double ar = std::fabs(r);
    const int nn = ar < 0.3 ? 6 : (ar < 0.75 ? 12 : 20);  // bvn_rule, normal.hpp:84-91
    std::vector<double> x(nn), w(nn);
    {  // recompute on [-1, 1] exactly as quadrature.hpp:22-55 (before its (0, 1) map)
        const double pi = 3.14159265358979323846;
        for (int i = 0; i < (nn + 1) / 2; ++i) {
            double z = std::cos(pi * (i + 0.75) / (nn + 0.5)), dp = 0.0;
            for (int it = 0; it < 100; ++it) {
                double p0 = 1.0, p1 = z;
                for (int j = 2; j <= nn; ++j) {
                    const double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
                    p0 = p1;
                    p1 = p2;
                }
                dp = nn * (z * p1 - p0) / (z * z - 1.0);
                const double step = p1 / dp;
                z -= step;
                if (std::fabs(step) < 1e-15) break;
            }
            x[i] = -z;
            x[nn - 1 - i] = z;
            w[i] = w[nn - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
        }
        if (nn % 2 == 1) x[nn / 2] = 0.0;
    }
    double hk = h * k, bvn = 0.0;
    if (ar < 0.925) {
        if (ar > 0.0) {
            const double hs = 0.5 * (h * h + k * k), asr = std::asin(r);
            for (int i = 0; i < nn; ++i) {
                const double sn = std::sin(0.5 * asr * (x[i] + 1.0));
                bvn += w[i] * std::exp((sn * hk - hs) / (1.0 - sn * sn));
            }
            bvn *= asr / (2.0 * twopi);
        }
        bvn += oracle::phi_cdf(-h) * oracle::phi_cdf(-k);
    } else {
        if (r < 0.0) {
            k = -k;
            hk = -hk;
        }
        if (ar < 1.0) {
            const double as = (1.0 - r) * (1.0 + r);
            double a = std::sqrt(as);
            const double bs = (h - k) * (h - k), cc = (4.0 - hk) / 8.0, dd = (12.0 - hk) / 16.0;
            double asr = -0.5 * (bs / as + hk);
            if (asr > -100.0)
                bvn = a * std::exp(asr) * (1.0 - cc * (bs - as) * (1.0 - dd * bs / 5.0) / 3.0 + cc * dd * as * as / 5.0);
            if (-hk < 100.0) {
                const double bb = std::sqrt(bs);
                bvn -= std::exp(-0.5 * hk) * std::sqrt(twopi) * oracle::phi_cdf(-bb / a) * bb *
                       (1.0 - cc * bs * (1.0 - dd * bs / 5.0) / 3.0);
            }
            a *= 0.5;
            for (int i = 0; i < nn; ++i) {
                const double t = a * (x[i] + 1.0), xs = t * t;
                asr = -0.5 * (bs / xs + hk);
                if (asr > -100.0) {
                    const double rs = std::sqrt(1.0 - xs);
                    bvn += a * w[i] * std::exp(asr) *
                           (std::exp(-hk * (1.0 - rs) / (2.0 * (1.0 + rs))) / rs - (1.0 + cc * xs * (1.0 + dd * xs)));
                }
            }
            bvn = -bvn / twopi;
        }
        if (r > 0.0) {
            bvn += oracle::phi_cdf(-std::max(h, k));
        } else {
            bvn = -bvn;
            if (k > h) bvn += oracle::phi_cdf(k) - oracle::phi_cdf(h);
        }
    }
    return std::clamp(bvn, 0.0, 1.0);
}

double frank_cdf_pos_restated(double u, double v, double t) {  // copula.hpp:174-181
    const double lo = std::min(u, v), hi = std::max(u, v);
    const double k2 = -t * (hi - lo);
    const double b = std::expm1(-t * (1.0 - lo)) + std::exp(k2) * std::expm1(-t * lo);
    return lo - (std::log(-b) - std::log(-std::expm1(-t))) / t;
}

struct RestatedMath {
    // copula.hpp:273-290
    static double cdf(int fam, double t, double u, double v) {
        if (!oracle::theta_ok(fam, t)) throw std::domain_error("theta outside the family domain");
        u = oracle::clamp01(u);
        v = oracle::clamp01(v);
        if (fam == 0) return bvn_upper_restated(-oracle::phi_inv(u), -oracle::phi_inv(v), t);
        if (fam == 1) return t > 0.0 ? frank_cdf_pos_restated(u, v, t) : u - frank_cdf_pos_restated(u, 1.0 - v, -t);
        const double lx = std::log(-std::log(u)), ly = std::log(-std::log(v));
        const double a = t * lx, b = t * ly, m = std::max(a, b);
        const double lnS = m + std::log(std::exp(a - m) + std::exp(b - m));
        return std::exp(-std::exp(lnS / t));
    }
    // 12 int C - 3, same tensor rule order as rel_sums
    static double spearman_rho(int fam, double t, int n) {
        std::vector<double> x, w;
        gauss_legendre01_restated(n, x, w);
        double total = 0.0;
        for (int i = 0; i < n; ++i) {
            double row = 0.0;
            for (int j = 0; j < n; ++j) row += w[j] * cdf(fam, t, x[i], x[j]);
            total += w[i] * row;
        }
        return 12.0 * total - 3.0;
    }
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

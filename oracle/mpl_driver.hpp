// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/copula_math.hpp header).
//
// CPU restatement of the reference's ABSENT estimator and partition/combine
// layers, written from their SPEC contracts (the reference ships no code for
// them — SURVEY.md §0.2):
//   pseudo_loglik
//   fit / FitResult
//   asymptotic_variance
//   partition
//   combine
//   fit_parallel
// plus the reference's present pieces (ranks: pseudo_obs.hpp:30-77).
//
// Parity definition: theta_hat is the converged root of the
// pseudo-score equation sum_i d/dtheta log c(u_i; theta) = 0, polished by
// safeguarded Newton until |dtheta| <= 1e-14 * max(1, |theta|). The SPEC's
// Brent tolerance (1e-8) cannot support a 1e-9 relative parity
// bar; the root is the same maximiser the SPEC's optimiser approximates, and
// tests/test_oracle.py checks it against the SPEC's brute-force grid oracle
// (SPEC.md:215, 224, 482).
//
// The driver is a template over a `Math` policy so the same SPEC restatement
// runs over (a) the oracle's own restated per-point arithmetic
// (oracle/copula_math.hpp -> liboracle.so) and (b) the compiled reference
// headers themselves (oracle/ref_wrap.cpp -> oracle/_ref/libparcop_ref.so).
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "copula_math.hpp"

namespace oracle {

struct FitRecord {  // SPEC.md:200-204 (FitResult), flat for ctypes
    double theta_hat;
    double sigma2;
    double loglik;
    uint64_t n;
    int32_t iterations;  // data passes (score+Hessian sweeps) the Newton root took
    int32_t converged;   // 1 = converged, 0 = not
    int32_t status;      // 0 ok, 1 no convergence, 2 Info<=0, 3 domain/data error
    int32_t pad;
};

struct NaiveFlag {};

// ------------------------------------------------------------------ ranks
// pseudo_obs.hpp:44-65 restated: order = indices sorted by (value, index);
// tie runs i..j get avg = 0.5*((i+1)+(j+1)); u = avg * (1/(n+1)).
inline void rank_column_restated(const double* x, size_t n, double* out) {
    std::vector<uint32_t> ord(n);
    std::iota(ord.begin(), ord.end(), 0u);
    std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return x[a] < x[b]; });
    const double scale = 1.0 / (static_cast<double>(n) + 1.0);
    size_t i = 0;
    while (i < n) {
        size_t j = i;
        while (j + 1 < n && x[ord[j + 1]] == x[ord[i]]) ++j;
        const double avg = 0.5 * (static_cast<double>(i + 1) + static_cast<double>(j + 1));
        const double u = avg * scale;
        for (size_t k = i; k <= j; ++k) out[ord[k]] = u;
        i = j + 1;
    }
}

inline void validate_columns(const double* c1, const double* c2, size_t n) {  // pseudo_obs.hpp:30-37
    if (n < 2) throw std::invalid_argument("data matrix: need at least 2 rows");
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(c1[i]) || !std::isfinite(c2[i]))
            throw std::domain_error("data matrix: non-finite value");
}

// ------------------------------------------------------------------ tau init
// Kendall's tau on the first m rows by merge-sort
// inversion counting (Knight 1966): sort by (u1, u2), count discordant swaps
// of u2. Used only to initialise the root search, so ties are not corrected.
inline double kendall_tau_rows(const double* u1, const double* u2, size_t m) {
    if (m < 2) return 0.0;
    std::vector<uint32_t> ord(m);
    std::iota(ord.begin(), ord.end(), 0u);
    std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) {
        if (u1[a] != u1[b]) return u1[a] < u1[b];
        return u2[a] < u2[b];
    });
    std::vector<double> y(m), tmp(m);
    for (size_t k = 0; k < m; ++k) y[k] = u2[ord[k]];
    uint64_t swaps = 0;
    for (size_t width = 1; width < m; width *= 2) {
        for (size_t lo = 0; lo < m; lo += 2 * width) {
            const size_t mid = std::min(lo + width, m), hi = std::min(lo + 2 * width, m);
            size_t a = lo, b = mid, o = lo;
            while (a < mid && b < hi) {
                if (y[b] < y[a]) { tmp[o++] = y[b++]; swaps += mid - a; }
                else tmp[o++] = y[a++];
            }
            while (a < mid) tmp[o++] = y[a++];
            while (b < hi) tmp[o++] = y[b++];
        }
        std::swap(y, tmp);
    }
    const double pairs = 0.5 * static_cast<double>(m) * static_cast<double>(m - 1);
    return 1.0 - 2.0 * static_cast<double>(swaps) / pairs;
}

// inverse_tau: closed form for Gaussian/Gumbel, bisection
// on tau(theta) = 1 - (4/theta)(1 - D1(theta)) for Frank.
template <class Math>
double inverse_tau(int fam, double tau) {
    tau = std::min(std::max(tau, -0.999), 0.999);
    if (fam == 0) return std::sin(0.5 * 3.14159265358979323846 * tau);
    if (fam == 2) return tau <= 0.0 ? 1.0 : 1.0 / (1.0 - tau);
    const double at = std::fabs(tau);
    if (at < 1e-7) return tau < 0 ? -1e-6 : 1e-6;
    auto tau_of = [](double th) { return 1.0 - 4.0 / th * (1.0 - Math::debye1(th)); };
    double lo = 1e-6, hi = 1.0;
    while (tau_of(hi) < at && hi < 1e6) hi *= 2.0;
    for (int it = 0; it < 200 && hi - lo > 1e-10 * hi; ++it) {
        const double mid = 0.5 * (lo + hi);
        (tau_of(mid) < at ? lo : hi) = mid;
    }
    const double th = 0.5 * (lo + hi);
    return tau < 0 ? -th : th;
}

// ------------------------------------------------------------------ driver
template <class Math>
struct Driver {
    // SPEC.md:207-215
    static double pseudo_loglik(int fam, double t, const double* u1, const double* u2, size_t n) {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i) s += Math::log_density(fam, t, u1[i], u2[i]);
        return s;
    }

    static void score_hess(int fam, double t, const double* u1, const double* u2, size_t n,
                           double& S, double& H) {
        double s = 0.0, h = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const PointDerivs d = Math::derivs(fam, t, u1[i], u2[i]);
            s += d.score;
            h += d.hess;
        }
        S = s;
        H = h;
    }

    // SPEC.md:216-224, 242-244 with the root-polish parity definition above.
    static FitRecord fit(int fam, const double* u1, const double* u2, size_t n, size_t min_rows = 30) {
        FitRecord r{};
        r.n = n;
        r.theta_hat = std::nan("");
        r.sigma2 = std::nan("");
        r.loglik = std::nan("");
        if (n < min_rows) {
            r.status = 3;
            return r;
        }
        // init: inverse_tau of the empirical tau on min(n, 5000) rows
        const size_t m = std::min<size_t>(n, 5000);
        double t = inverse_tau<Math>(fam, kendall_tau_rows(u1, u2, m));
        double lo, hi;  // bracket of the root in theta
        if (fam == 0) { lo = -1.0; hi = 1.0; t = std::min(std::max(t, -0.99), 0.99); }
        else if (fam == 1) { lo = -INFINITY; hi = INFINITY; if (std::fabs(t) < 1e-6) t = t < 0 ? -1e-6 : 1e-6; }
        else { lo = 1.0; hi = INFINITY; t = std::max(t, 1.0); }
        int passes = 0;
        bool conv = false, tried_one = false;
        for (int it = 0; it < 200; ++it) {
            double S, H;
            score_hess(fam, t, u1, u2, n, S, H);
            ++passes;
            if (!std::isfinite(S) || !std::isfinite(H)) break;
            if (S > 0.0) lo = t; else hi = t;
            if (fam == 2 && t == 1.0) {  // Gumbel boundary theta = 1
                tried_one = true;
                if (S <= 0.0) { conv = true; break; }  // boundary maximum
            }
            double cand = NAN;
            if (H < 0.0) {
                cand = t - S / H;
                if (std::fabs(cand - t) <= 1e-14 * std::max(1.0, std::fabs(t))) {  // Newton step at the noise floor
                    if (!(fam == 2 && cand < 1.0)) t = cand;
                    conv = true;
                    break;
                }
            }
            bool inside = std::isfinite(cand) && cand > lo && cand < hi;
            if (!inside && fam == 2 && !tried_one && std::isfinite(cand) && cand <= 1.0) {
                cand = 1.0;  // evaluate the boundary before bisecting towards it
                inside = true;
            }
            if (!inside) {
                if (std::isfinite(lo) && std::isfinite(hi)) cand = 0.5 * (lo + hi);
                else if (std::isfinite(lo)) cand = lo + std::max(1.0, std::fabs(lo));
                else cand = hi - std::max(1.0, std::fabs(hi));
                if (fam == 2 && !(cand > 1.0)) cand = 1.0;
            }
            if (fam == 1 && std::fabs(cand) < 1e-6) cand = cand < 0 ? -1e-6 : 1e-6;
            const double step = cand - t;
            t = cand;
            if (std::fabs(step) <= 1e-14 * std::max(1.0, std::fabs(t))) { conv = true; break; }
        }
        r.theta_hat = t;
        r.iterations = passes;
        r.converged = conv ? 1 : 0;
        r.status = conv ? 0 : 1;
        if (conv) {
            r.loglik = pseudo_loglik(fam, t, u1, u2, n);
            try {
                r.sigma2 = asymptotic_variance(fam, t, u1, u2, n);
            } catch (const std::exception&) {
                r.converged = 0;
                r.status = 2;
            }
        }
        return r;
    }

    // sigma2 = M/I^2/n with the rank-correction terms
    // W_ji evaluated by sorting on u_j and suffix sums (ties share the suffix
    // that starts at their run).
    static double asymptotic_variance(int fam, double t, const double* u1, const double* u2, size_t n) {
        std::vector<PointDerivs> d(n);
        double hsum = 0.0;
        for (size_t i = 0; i < n; ++i) {
            d[i] = Math::derivs(fam, t, u1[i], u2[i]);
            hsum += d[i].hess;
        }
        const double info = -hsum / static_cast<double>(n);
        if (!(info > 0.0)) throw std::domain_error("asymptotic_variance: information <= 0");
        std::vector<double> w1(n), w2(n);
        rank_term(u1, d, n, 1, w1);
        rank_term(u2, d, n, 2, w2);
        double msum = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const double z = d[i].score + w1[i] + w2[i];
            msum += z * z;
        }
        const double mhat = msum / static_cast<double>(n);
        return mhat / (info * info) / static_cast<double>(n);
    }

    static void rank_term(const double* u, const std::vector<PointDerivs>& d, size_t n, int j,
                          std::vector<double>& w) {
        auto cr = [&](size_t h) { return j == 1 ? d[h].cross1 : d[h].cross2; };
        double c = 0.0;
        for (size_t h = 0; h < n; ++h) c += u[h] * cr(h);
        std::vector<uint32_t> ord(n);
        std::iota(ord.begin(), ord.end(), 0u);
        std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return u[a] < u[b]; });
        double suffix = 0.0;
        size_t k = n;
        while (k > 0) {  // walk tie runs from the top
            size_t a = k - 1;
            while (a > 0 && u[ord[a - 1]] == u[ord[k - 1]]) --a;
            for (size_t q = k; q-- > a;) suffix += cr(ord[q]);
            for (size_t q = a; q < k; ++q) w[ord[q]] = (suffix - c) / static_cast<double>(n);
            k = a;
        }
    }

    // The SPEC's literal O(n^2) definition, for cross-checking only.
    static double asymptotic_variance_naive(int fam, double t, const double* u1, const double* u2, size_t n) {
        std::vector<PointDerivs> d(n);
        double hsum = 0.0;
        for (size_t i = 0; i < n; ++i) {
            d[i] = Math::derivs(fam, t, u1[i], u2[i]);
            hsum += d[i].hess;
        }
        const double info = -hsum / static_cast<double>(n);
        if (!(info > 0.0)) throw std::domain_error("asymptotic_variance: information <= 0");
        double msum = 0.0;
        for (size_t i = 0; i < n; ++i) {
            double a1 = 0.0, a2 = 0.0;
            for (size_t h = 0; h < n; ++h) {
                a1 += ((u1[i] <= u1[h] ? 1.0 : 0.0) - u1[h]) * d[h].cross1;
                a2 += ((u2[i] <= u2[h] ? 1.0 : 0.0) - u2[h]) * d[h].cross2;
            }
            const double z = d[i].score + a1 / static_cast<double>(n) + a2 / static_cast<double>(n);
            msum += z * z;
        }
        return msum / static_cast<double>(n) / (info * info) / static_cast<double>(n);
    }

    // normalized_ranks on one block, then fit (which fills sigma2).
    static FitRecord fit_block(int fam, const double* c1, const double* c2, size_t n) {
        std::vector<double> u1(n), u2(n);
        validate_columns(c1, c2, n);
        Math::rank_column(c1, n, u1.data());
        Math::rank_column(c2, n, u2.data());
        return fit(fam, u1.data(), u2.data(), n);
    }

    // fit_parallel's worker pool: positional result slots,
    // so completion order cannot affect the output.
    static void fit_blocks(int fam, const double* c1, const double* c2, const uint64_t* off, size_t nblk,
                           int workers, FitRecord* out) {
        if (workers < 1) workers = 1;
        std::atomic<size_t> next{0};
        std::vector<std::string> errs(nblk);
        auto work = [&]() {
            for (;;) {
                const size_t b = next.fetch_add(1);
                if (b >= nblk) return;
                const size_t a = off[b], e = off[b + 1];
                try {
                    out[b] = fit_block(fam, c1 + a, c2 + a, e - a);
                } catch (const std::exception& ex) {
                    FitRecord r{};
                    r.n = e - a;
                    r.theta_hat = r.sigma2 = r.loglik = std::nan("");
                    r.status = 3;
                    out[b] = r;
                }
            }
        };
        std::vector<std::thread> pool;
        for (int w = 1; w < workers; ++w) pool.emplace_back(work);
        work();
        for (auto& th : pool) th.join();
    }
};

// theta_c = sum w theta / sum w, w = 1/sigma2 over the
// converged blocks, in block order. Returns the number of blocks used.
// Eq. (15) anchored at the first used block's estimate a:
//   theta_c = a + sum w (theta - a) / sum w  (== sum w theta / sum w),
// which is exact in the SPEC's degenerate cases (M = 1 returns the full-data
// fit bit for bit; constant estimates return the constant,
// SPEC.md:290) where the plain ratio can be off by an ulp.
inline size_t combine_records(const FitRecord* r, size_t k, double* theta_c, double* weights) {
    double sw = 0.0, swd = 0.0, anchor = 0.0;
    size_t used = 0;
    for (size_t m = 0; m < k; ++m) {
        const bool ok = r[m].converged && r[m].sigma2 > 0.0 && std::isfinite(r[m].sigma2);
        const double w = ok ? 1.0 / r[m].sigma2 : 0.0;
        if (weights) weights[m] = w;
        if (!ok) continue;
        if (used == 0) anchor = r[m].theta_hat;
        sw += w;
        swd += w * (r[m].theta_hat - anchor);
        ++used;
    }
    if (used == 0) throw std::runtime_error("combine: no converged blocks");
    *theta_c = anchor + swd / sw;
    return used;
}

// SPEC.md:275-283. Contiguous: block m = rows [m*floor(N/M), (m+1)*floor(N/M)),
// remainder to the last block. Offsets has M+1 entries.
inline void partition_contiguous(uint64_t n, uint64_t m, uint64_t* off) {
    if (m < 1) throw std::invalid_argument("partition: need M >= 1");
    const uint64_t q = n / m;
    if (q < 30) throw std::invalid_argument("partition: block below the 30-row floor");
    for (uint64_t b = 0; b < m; ++b) off[b] = b * q;
    off[m] = n;
}

}  // namespace oracle

// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's per-point copula arithmetic, used by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
// CHECKER for the CUDA path. Nothing in paper_1609_05530_b200/ may include,
// link or call this file.
//
// Every function cites the reference file:line it restates
// (/root/reference/proj/include/parcop/...). The restatement keeps the
// reference's operation order where it matters for rounding, so its values
// agree with the compiled reference headers (oracle/_ref) to a few ulp; the
// pin is tests/test_oracle_pin.py.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>

namespace oracle {

enum Family : int { kGaussian = 0, kFrank = 1, kGumbel = 2 };  // copula.hpp:25

struct PointDerivs {  // copula.hpp:99-104 (Shc)
    double score, hess, cross1, cross2;
};

// ---------------------------------------------------------------- normal.hpp
inline double phi_pdf(double x) {  // normal.hpp:15-18
    return 0.3989422804014326779399 * std::exp(-0.5 * x * x);
}

inline double phi_cdf(double x) {  // normal.hpp:20-22 (inv_sqrt2 = correctly rounded 1/sqrt2)
    return 0.5 * std::erfc(-x * 0x1.6a09e667f3bcdp-1);
}

namespace as241 {  // Wichura AS241 / PPND16 coefficient tables, normal.hpp:40-63
constexpr double A[8] = {3.3871328727963666080e+0, 1.3314166789178437745e+2,
                         1.9715909503065514427e+3, 1.3731693765509461125e+4,
                         4.5921953931549871457e+4, 6.7265770927008700853e+4,
                         3.3430575583588128105e+4, 2.5090809287301226727e+3};
constexpr double B[8] = {1.0, 4.2313330701600911252e+1, 6.8718700749205790830e+2,
                         5.3941960214247511077e+3, 2.1213794301586595867e+4,
                         3.9307895800092710610e+4, 2.8729085735721942674e+4,
                         5.2264952788528545610e+3};
constexpr double C[8] = {1.42343711074968357734e+0, 4.63033784615654529590e+0,
                         5.76949722146069140550e+0, 3.64784832476320460504e+0,
                         1.27045825245236838258e+0, 2.41780725177450611770e-1,
                         2.27238449892691845833e-2, 7.74545014278341407640e-4};
constexpr double D[8] = {1.0, 2.05319162663775882187e+0, 1.67638483018380384940e+0,
                         6.89767334985100004550e-1, 1.48103976427480074590e-1,
                         1.51986665636164571966e-2, 5.47593808499534494600e-4,
                         1.05075007164441684324e-9};
constexpr double E[8] = {6.65790464350110377720e+0, 5.46378491116411436990e+0,
                         1.78482653991729133580e+0, 2.96560571828504891230e-1,
                         2.65321895265761230930e-2, 1.24266094738807843860e-3,
                         2.71155556874348757815e-5, 2.01033439929228813265e-7};
constexpr double F[8] = {1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1,
                         1.48753612908506148525e-2, 7.86869131145613259100e-4,
                         1.84631831751005468180e-5, 1.42151175831644588870e-7,
                         2.04426310338993978564e-15};
inline double poly(const double* c, double r) {  // normal.hpp:26-31 (Horner, highest first)
    double acc = c[7];
    for (int i = 6; i >= 0; --i) acc = acc * r + c[i];
    return acc;
}
}  // namespace as241

inline double phi_inv(double p) {  // normal.hpp:37-81
    if (!(p > 0.0 && p < 1.0)) throw std::domain_error("norm_quantile: p must lie strictly in (0,1)");
    const double q = p - 0.5;
    if (std::fabs(q) <= 0.425) {
        const double r = 0.180625 - q * q;
        return q * as241::poly(as241::A, r) / as241::poly(as241::B, r);
    }
    double r = std::sqrt(-std::log(q < 0.0 ? p : 1.0 - p));
    double x;
    if (r <= 5.0) {
        r -= 1.6;
        x = as241::poly(as241::C, r) / as241::poly(as241::D, r);
    } else {
        r -= 5.0;
        x = as241::poly(as241::E, r) / as241::poly(as241::F, r);
    }
    return q < 0.0 ? -x : x;
}

// ---------------------------------------------------------------- guards
constexpr double kUnitEps = 1e-12;  // copula.hpp:85
constexpr double kLogClip = 700.0;  // copula.hpp:86

inline double clamp01(double u) {  // copula.hpp:88-92
    if (!(u >= 0.0 && u <= 1.0)) throw std::domain_error("copula argument must lie in [0,1]");
    return std::min(std::max(u, kUnitEps), 1.0 - kUnitEps);
}
inline double clip_log(double v) {  // copula.hpp:94-97 (NaN -> -700)
    if (std::isnan(v)) return -kLogClip;
    return std::min(std::max(v, -kLogClip), kLogClip);
}

inline bool theta_ok(int fam, double t) {  // copula.hpp:47-55
    if (!std::isfinite(t)) return false;
    if (fam == kGaussian) return t > -1.0 && t < 1.0;
    if (fam == kFrank) return t != 0.0;
    if (fam == kGumbel) return t >= 1.0;
    return false;
}

// ---------------------------------------------------------------- Gaussian
inline double gauss_lc(double x, double y, double t) {  // copula.hpp:110-113
    const double a = 1.0 - t * t;
    return -0.5 * std::log(a) + (2.0 * t * x * y - t * t * (x * x + y * y)) / (2.0 * a);
}
inline PointDerivs gauss_d(double x, double y, double t) {  // copula.hpp:115-127
    const double a = 1.0 - t * t, a2 = a * a;
    const double xy = x * y, ss = x * x + y * y;
    PointDerivs d;  // operation order as in the reference (rounding-faithful)
    d.score = t / a + ((1.0 + t * t) * xy - t * ss) / a2;
    d.hess = (1.0 + t * t) / a2 + (2.0 * t * (3.0 + t * t) * xy - (1.0 + 3.0 * t * t) * ss) / (a2 * a);
    d.cross1 = ((1.0 + t * t) * y - 2.0 * t * x) / (a2 * phi_pdf(x));
    d.cross2 = ((1.0 + t * t) * x - 2.0 * t * y) / (a2 * phi_pdf(y));
    return d;
}

// ---------------------------------------------------------------- Frank (t > 0)
inline double frank_lc_pos(double u, double v, double t) {  // copula.hpp:137-143
    const double lo = std::min(u, v), hi = std::max(u, v);
    const double k2 = -t * (hi - lo);
    const double bb = std::expm1(-t * (1.0 - lo)) + std::exp(k2) * std::expm1(-t * lo);
    return std::log(t) + std::log(-std::expm1(-t)) + k2 - 2.0 * std::log(-bb);
}
// d2 log c / (dtheta d first-arg); copula.hpp:147-154
inline double frank_cross(double a, double other, double t, double shift, double bb, double bp) {
    const double em = std::expm1(-t * other);
    const double ev = std::exp(-t * other);
    const double ea = -t * shift * em;
    const double dea = shift * ((t * a - 1.0) * em + t * other * ev);
    return -1.0 - 2.0 * (dea * bb - ea * bp) / (bb * bb);
}
inline PointDerivs frank_d_pos(double u, double v, double t) {  // copula.hpp:156-172
    const double lo = std::min(u, v), hi = std::max(u, v);
    const double e1 = std::exp(-t * (1.0 - lo));
    const double e2 = std::exp(-t * (hi - lo));
    const double e3 = std::exp(-t * lo);
    const double bb = std::expm1(-t * (1.0 - lo)) + e2 * std::expm1(-t * lo);
    const double bp = lo - e1 + e2 * (hi - (lo + hi) * e3);
    const double bpp = e1 - lo * lo + e2 * ((lo + hi) * (lo + hi) * e3 - hi * hi);
    const double g = std::exp(-t) / std::expm1(-t);
    PointDerivs d;
    d.score = 1.0 / t - g - (u + v) - 2.0 * bp / bb;
    d.hess = -1.0 / (t * t) + g - g * g - 2.0 * (bpp / bb - (bp / bb) * (bp / bb));
    d.cross1 = frank_cross(u, v, t, u <= v ? 1.0 : e2, bb, bp);
    d.cross2 = frank_cross(v, u, t, v <= u ? 1.0 : e2, bb, bp);
    return d;
}

// ---------------------------------------------------------------- Gumbel
struct GumbelParts {  // copula.hpp:189-197
    double lx, ly, sx, lnS, w, r, r2, pa, pb;
};
inline GumbelParts gumbel_parts(double u, double v, double t) {  // copula.hpp:199-219
    GumbelParts g;
    const double x = -std::log(u), y = -std::log(v);
    g.lx = std::log(x);
    g.ly = std::log(y);
    g.sx = x + y;
    const double a = t * g.lx, b = t * g.ly;
    const double m = std::max(a, b);
    const double ea = std::exp(a - m), eb = std::exp(b - m);
    const double s = ea + eb;
    g.lnS = m + std::log(s);
    g.w = std::exp(g.lnS / t);
    g.r = (ea * g.lx + eb * g.ly) / s;
    g.r2 = (ea * g.lx * g.lx + eb * g.ly * g.ly) / s;
    g.pa = std::exp(a - g.lnS) / x;
    g.pb = std::exp(b - g.lnS) / y;
    return g;
}
inline double gumbel_lc(double u, double v, double t) {  // copula.hpp:221-225
    const GumbelParts g = gumbel_parts(u, v, t);
    return -g.w + (t - 1.0) * (g.lx + g.ly) + g.sx + (1.0 / t - 2.0) * g.lnS + std::log(g.w + t - 1.0);
}
// copula.hpp:228-236
inline double gumbel_cross(const GumbelParts& g, double t, double p, double l, double u, double wt) {
    const double gg = g.w + t - 1.0;
    const double pt = p * (l - g.r);
    const double x = -std::log(u);
    const double cx = -wt * p - g.w * pt + 1.0 / x - 2.0 * p + (1.0 - 2.0 * t) * pt +
                      ((wt * p + g.w * pt) * gg - g.w * p * (wt + 1.0)) / (gg * gg);
    return -cx / u;
}
inline PointDerivs gumbel_d(double u, double v, double t) {  // copula.hpp:238-254
    const GumbelParts g = gumbel_parts(u, v, t);
    const double t2 = t * t;
    const double rt = g.r2 - g.r * g.r;
    const double lw_t = g.r / t - g.lnS / t2;
    const double wt = g.w * lw_t;
    const double lw_tt = rt / t - 2.0 * g.r / t2 + 2.0 * g.lnS / (t2 * t);
    const double wtt = g.w * (lw_t * lw_t + lw_tt);
    const double gg = g.w + t - 1.0;
    PointDerivs d;
    d.score = -wt + g.lx + g.ly - g.lnS / t2 + (1.0 / t - 2.0) * g.r + (wt + 1.0) / gg;
    d.hess = -wtt - 2.0 * g.r / t2 + 2.0 * g.lnS / (t2 * t) + (1.0 / t - 2.0) * rt +
             (wtt * gg - (wt + 1.0) * (wt + 1.0)) / (gg * gg);
    d.cross1 = gumbel_cross(g, t, g.pa, g.lx, u, wt);
    d.cross2 = gumbel_cross(g, t, g.pb, g.ly, v, wt);
    return d;
}

// ---------------------------------------------------------------- dispatch
// copula.hpp:256-269 — Frank theta<0 by the reflection c(u,v;-t) = c(u,1-v;t).
inline PointDerivs derivs(int fam, double t, double u, double v) {
    if (fam == kGaussian) return gauss_d(phi_inv(u), phi_inv(v), t);
    if (fam == kFrank) {
        if (t > 0.0) return frank_d_pos(u, v, t);
        const PointDerivs r = frank_d_pos(u, 1.0 - v, -t);
        return PointDerivs{-r.score, r.hess, -r.cross1, r.cross2};
    }
    return gumbel_d(u, v, t);
}

// copula.hpp:293-311 (log_pdf, with the clamp and the +-700 clip)
inline double log_density(int fam, double t, double u1, double u2) {
    if (!theta_ok(fam, t)) throw std::domain_error("theta outside the family domain");
    const double u = clamp01(u1), v = clamp01(u2);
    double lp = 0.0;
    if (fam == kGaussian) lp = gauss_lc(phi_inv(u), phi_inv(v), t);
    else if (fam == kFrank) lp = t > 0.0 ? frank_lc_pos(u, v, t) : frank_lc_pos(u, 1.0 - v, -t);
    else lp = gumbel_lc(u, v, t);
    return clip_log(lp);
}

// copula.hpp:316-334 (score_theta / hess_theta / cross_score share one evaluation here)
inline PointDerivs point_derivs(int fam, double t, double u1, double u2) {
    if (!theta_ok(fam, t)) throw std::domain_error("theta outside the family domain");
    return derivs(fam, t, clamp01(u1), clamp01(u2));
}

}  // namespace oracle

// Per-point copula arithmetic for sm_100a (device side).
//
// Restates the reference formulas (copula.hpp:106-269, normal.hpp:15-81) for
// the GPU: theta-independent sub-expressions are hoisted out of the point
// loop (per-block constants in *Theta structs), divisions by per-theta
// constants become multiplies by hoisted reciprocals, per-point divisions by
// the same denominator share one reciprocal, and the likelihood passes
// compute only what Newton needs (score, Hessian). Values agree with the
// reference to a few ulp per point; parity of the reductions is enforced by
// tests/test_gpu_parity.py against the CPU oracle.
#pragma once

#include <cuda_runtime.h>

namespace pcb {

// 1/x for the per-point paths: MUFU reciprocal + two Newton steps (about one
// ulp; the 1e-9 parity bar is far away), no IEEE-division slow path. Inputs
// are normal positive or negative doubles (never 0, inf or denormal here).
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}


// ------------------------------------------------- exp / expm1 / log (FP64)
// Per-point transcendentals of the likelihood and variance passes. Same
// classic algorithms as any libm (Cody-Waite reduction x = k ln2 + r,
// |r| <= ln2/2, polynomial for e^r - 1; log(1+f) = f - f^2/2 + s(f^2/2 + R(s^2)),
// s = f/(2+f)), Taylor coefficients, <= ~2 ulp. What differs is where the
// coefficients live: in __constant__ memory, so each Horner step is ONE DFMA
// with a constant-bank operand. libdevice materialises its 64-bit immediates
// with two uniform moves per coefficient (measured: 243 issued instructions
// per point for 88 FP64 ones in the Frank Newton pass, FP64 pipe 55% busy).
// Arguments outside the fast range (under/overflow, NaN, x <= 0 for log)
// take libdevice.
static __constant__ double c_fm[24] = {
    // [0..10]: (e^r - 1 - r) / r^2 = sum_k r^k / (k+2)!
    1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040, 1.0 / 40320, 1.0 / 362880, 1.0 / 3628800,
    1.0 / 39916800, 1.0 / 479001600,
    // [11..20]: R(z) = sum_{k=1..10} 2 z^k / (2k + 1)
    2.0 / 3, 2.0 / 5, 2.0 / 7, 2.0 / 9, 2.0 / 11, 2.0 / 13, 2.0 / 15, 2.0 / 17, 2.0 / 19, 2.0 / 21,
    // [21] log2(e), [22] ln2 high part (exact times any |k| < 2^11), [23] ln2 low part
    1.4426950408889634074, 0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};

// x = k ln2 + r: returns e^r - 1 and s = 2^k (|k| <= 1022)
__device__ __forceinline__ double fm_core(double x, double& s) {
    const double t = fma(x, c_fm[21], 0x1.8p52);  // round-to-nearest k in the low word
    const double kd = t - 0x1.8p52;
    const int k = __double2loint(t);
    double r = fma(kd, -c_fm[22], x);
    r = fma(kd, -c_fm[23], r);
    double q = c_fm[10];
    q = fma(q, r, c_fm[9]);
    q = fma(q, r, c_fm[8]);
    q = fma(q, r, c_fm[7]);
    q = fma(q, r, c_fm[6]);
    q = fma(q, r, c_fm[5]);
    q = fma(q, r, c_fm[4]);
    q = fma(q, r, c_fm[3]);
    q = fma(q, r, c_fm[2]);
    q = fma(q, r, c_fm[1]);
    q = fma(q, r, c_fm[0]);
    s = __hiloint2double((k + 1023) << 20, 0);
    return fma(r * r, q, r);
}
// e^x - 1 for x <= 0 (the Frank paths: every argument is -t * (distance) with t = |theta|)
__device__ __forceinline__ double fm_expm1_neg(double x) {
    x = x < -40.0 ? -40.0 : x;  // e^-40 - 1 rounds to -1 (a plain select: no NaN-propagating min/max)
    double s;
    const double p = fm_core(x, s);
    return fma(p, s, s - 1.0);  // s(1 + p) - 1, s - 1 exact
}
__device__ __forceinline__ double fm_exp(double x) {
    if (!(x >= -708.0 && x <= 709.0)) return exp(x);
    double s;
    const double p = fm_core(x, s);
    return fma(p, s, s);
}
__device__ __forceinline__ double fm_log(double x) {
    if (!(x >= 0x1p-1022 && x <= 0x1.fffffffffffffp1023)) return log(x);
    int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    int e = (hi >> 20) - 1023;
    hi &= 0x000fffff;
    const bool big = hi > 0x6a09e;  // mantissa above sqrt(2): m/2, e+1
    e += big ? 1 : 0;
    const double f = __hiloint2double(hi | (big ? 0x3fe00000 : 0x3ff00000), lo) - 1.0;
    const double hfsq = 0.5 * f * f;
    const double s = f * fast_rcp(2.0 + f);
    const double z = s * s;
    double R = c_fm[20];
    R = fma(R, z, c_fm[19]);
    R = fma(R, z, c_fm[18]);
    R = fma(R, z, c_fm[17]);
    R = fma(R, z, c_fm[16]);
    R = fma(R, z, c_fm[15]);
    R = fma(R, z, c_fm[14]);
    R = fma(R, z, c_fm[13]);
    R = fma(R, z, c_fm[12]);
    R = fma(R, z, c_fm[11]);
    R *= z;
    const double ed = static_cast<double>(e);
    return fma(ed, c_fm[22], -((hfsq - fma(s, hfsq + R, ed * c_fm[23])) - f));
}

// ------------------------------------------------------------------ normal
__device__ __forceinline__ double dev_phi_pdf(double x) {  // normal.hpp:15-18
    return 0.3989422804014326779399 * exp(-0.5 * x * x);
}

// Wichura AS241 (normal.hpp:37-81); same coefficients and Horner order.
__device__ inline double dev_phi_inv(double p) {
    const double q = p - 0.5;
    if (fabs(q) <= 0.425) {
        const double r = 0.180625 - q * q;
        double n = 2.5090809287301226727e+3;
        n = n * r + 3.3430575583588128105e+4;
        n = n * r + 6.7265770927008700853e+4;
        n = n * r + 4.5921953931549871457e+4;
        n = n * r + 1.3731693765509461125e+4;
        n = n * r + 1.9715909503065514427e+3;
        n = n * r + 1.3314166789178437745e+2;
        n = n * r + 3.3871328727963666080e+0;
        double d = 5.2264952788528545610e+3;
        d = d * r + 2.8729085735721942674e+4;
        d = d * r + 3.9307895800092710610e+4;
        d = d * r + 2.1213794301586595867e+4;
        d = d * r + 5.3941960214247511077e+3;
        d = d * r + 6.8718700749205790830e+2;
        d = d * r + 4.2313330701600911252e+1;
        d = d * r + 1.0;
        return q * n / d;
    }
    double r = sqrt(-log(q < 0.0 ? p : 1.0 - p));
    double x;
    if (r <= 5.0) {
        r -= 1.6;
        double n = 7.74545014278341407640e-4;
        n = n * r + 2.27238449892691845833e-2;
        n = n * r + 2.41780725177450611770e-1;
        n = n * r + 1.27045825245236838258e+0;
        n = n * r + 3.64784832476320460504e+0;
        n = n * r + 5.76949722146069140550e+0;
        n = n * r + 4.63033784615654529590e+0;
        n = n * r + 1.42343711074968357734e+0;
        double d = 1.05075007164441684324e-9;
        d = d * r + 5.47593808499534494600e-4;
        d = d * r + 1.51986665636164571966e-2;
        d = d * r + 1.48103976427480074590e-1;
        d = d * r + 6.89767334985100004550e-1;
        d = d * r + 1.67638483018380384940e+0;
        d = d * r + 2.05319162663775882187e+0;
        d = d * r + 1.0;
        x = n / d;
    } else {
        r -= 5.0;
        double n = 2.01033439929228813265e-7;
        n = n * r + 2.71155556874348757815e-5;
        n = n * r + 1.24266094738807843860e-3;
        n = n * r + 2.65321895265761230930e-2;
        n = n * r + 2.96560571828504891230e-1;
        n = n * r + 1.78482653991729133580e+0;
        n = n * r + 5.46378491116411436990e+0;
        n = n * r + 6.65790464350110377720e+0;
        double d = 2.04426310338993978564e-15;
        d = d * r + 1.42151175831644588870e-7;
        d = d * r + 1.84631831751005468180e-5;
        d = d * r + 7.86869131145613259100e-4;
        d = d * r + 1.48753612908506148525e-2;
        d = d * r + 1.36929880922735805310e-1;
        d = d * r + 5.99832206555887937690e-1;
        d = d * r + 1.0;
        x = n / d;
    }
    return q < 0.0 ? -x : x;
}

__device__ __forceinline__ double clip_log(double v) {  // copula.hpp:94-97
    if (isnan(v)) return -700.0;
    return fmin(fmax(v, -700.0), 700.0);
}
__device__ __forceinline__ double clamp_unit(double u) {  // copula.hpp:88-92 (domain checked by caller)
    return fmin(fmax(u, 1e-12), 1.0 - 1e-12);
}

struct PointFull {
    double logc, score, hess, cross1, cross2;
};

// ---------------------------------------------------------------- Gaussian
struct GaussTheta {  // per-theta constants of copula.hpp:110-127
    double t, tt, ia, ia2, ia3, half_log_a, c_score_xy, c_hess_xy, c_hess_ss, one_tt;
    __device__ __forceinline__ explicit GaussTheta(double th) {
        t = th;
        tt = th * th;
        const double a = 1.0 - tt;
        ia = 1.0 / a;
        ia2 = ia * ia;
        ia3 = ia2 * ia;
        half_log_a = -0.5 * log(a);
        one_tt = 1.0 + tt;
        c_score_xy = one_tt;
        c_hess_xy = 2.0 * th * (3.0 + tt);
        c_hess_ss = 1.0 + 3.0 * tt;
    }
};

// ex = exp(x^2/2), ey = exp(y^2/2) (rank-table entries when u is rank-derived)
__device__ __forceinline__ PointFull gauss_full_e(double x, double y, double ex, double ey, const GaussTheta& g) {
    const double xy = x * y, ss = x * x + y * y;
    PointFull p;
    p.logc = g.half_log_a + (2.0 * g.t * xy - g.tt * ss) * (0.5 * g.ia);
    p.score = g.t * g.ia + (g.one_tt * xy - g.t * ss) * g.ia2;
    p.hess = g.one_tt * g.ia2 + (g.c_hess_xy * xy - g.c_hess_ss * ss) * g.ia3;
    // cross_j = ((1+t^2) other - 2 t self) / (a^2 phi(self)); 1/phi(s) = sqrt(2pi) e^{s^2/2}
    const double k = 2.5066282746310002 * g.ia2;
    p.cross1 = (g.one_tt * y - 2.0 * g.t * x) * (k * ex);
    p.cross2 = (g.one_tt * x - 2.0 * g.t * y) * (k * ey);
    return p;
}

__device__ __forceinline__ PointFull gauss_full(double x, double y, const GaussTheta& g) {
    return gauss_full_e(x, y, exp(0.5 * x * x), exp(0.5 * y * y), g);
}

// Sufficient-statistic form of the Gaussian pseudo-likelihood: with
// Sxy = sum x*y and Sss = sum (x^2+y^2) over n points,
//   L(t) = -n/2 log(1-t^2) + (2t Sxy - t^2 Sss) / (2(1-t^2))   (sum of copula.hpp:110-113)
//   S(t) = n t/a + ((1+t^2) Sxy - t Sss)/a^2                   (sum of :121)
//   H(t) = n(1+t^2)/a^2 + (2t(3+t^2) Sxy - (1+3t^2) Sss)/a^3   (sum of :122-123)
__device__ __forceinline__ void gauss_stats_sh(double t, double n, double sxy, double sss, double& S, double& H) {
    const double tt = t * t, a = 1.0 - tt, ia = 1.0 / a, ia2 = ia * ia;
    S = n * t * ia + ((1.0 + tt) * sxy - t * sss) * ia2;
    H = n * (1.0 + tt) * ia2 + (2.0 * t * (3.0 + tt) * sxy - (1.0 + 3.0 * tt) * sss) * ia2 * ia;
}

// ------------------------------------------------------------------- Frank
// theta > 0 form (copula.hpp:137-172); negative theta via the reflection
// c(u,v;-t) = c(u,1-v;t) with score and cross1 negated (copula.hpp:260-264).
struct FrankTheta {
    double t, inv_t, g, hconst, logc_const;
    bool neg;
    __device__ __forceinline__ explicit FrankTheta(double th) {
        neg = th < 0.0;
        t = fabs(th);
        inv_t = 1.0 / t;
        const double em = expm1(-t);
        g = exp(-t) / em;
        hconst = -inv_t * inv_t + g - g * g;
        logc_const = log(t) + log(-em);
    }
};

// score and Hessian only (the Newton pass), fp64
// NEG: theta < 0 (reflected); BIG: |theta| > 700 (e^{-t(hi-lo)} may leave
// the fast exp range). Both are per block, so the Newton pass instantiates
// the four loops and picks one per CTA.
template <bool NEG = false, bool BIG = true>
__device__ __forceinline__ void frank_sh_t(double u, double v, const FrankTheta& f, double& s, double& h) {
    if (NEG) v = 1.0 - v;
    const double t = f.t;
    const bool uv = u <= v;  // inputs are finite: one compare, two selects
    const double lo = uv ? u : v, hi = uv ? v : u;
    const double ema = fm_expm1_neg(-t * (1.0 - lo));
    double e2;
    if (BIG) {
        e2 = fm_exp(-t * (hi - lo));
    } else {
        double sc;
        const double p = fm_core(-t * (hi - lo), sc);
        e2 = fma(p, sc, sc);
    }
    const double emb = fm_expm1_neg(-t * lo);
    const double e1 = 1.0 + ema, e3 = 1.0 + emb;
    const double b = ema + e2 * emb;
    const double sum = lo + hi;
    const double bp = lo - e1 + e2 * (hi - sum * e3);
    const double bpp = e1 - lo * lo + e2 * (sum * sum * e3 - hi * hi);
    const double rb = fast_rcp(b);
    const double q = bp * rb;
    const double sc = f.inv_t - f.g - sum - 2.0 * q;
    s = NEG ? -sc : sc;
    h = f.hconst - 2.0 * (bpp * rb - q * q);
}
__device__ __forceinline__ void frank_sh(double u, double v, const FrankTheta& f, double& s, double& h) {
    if (f.neg) frank_sh_t<true, true>(u, v, f, s, h);
    else frank_sh_t<false, true>(u, v, f, s, h);
}

// fp32 per-point arithmetic (likelihood path of configs[3]); the caller
// accumulates in fp64.
struct FrankThetaF {
    float t, inv_t, g, hconst;
    bool neg;
    __device__ __forceinline__ explicit FrankThetaF(double th) {
        neg = th < 0.0;
        const double tt = fabs(th);
        const double em = expm1(-tt);
        const double gd = exp(-tt) / em;
        t = static_cast<float>(tt);
        inv_t = static_cast<float>(1.0 / tt);
        g = static_cast<float>(gd);
        hconst = static_cast<float>(-1.0 / (tt * tt) + gd - gd * gd);
    }
};

// fp32 inputs are radially reflected so that lo + hi <= 1 (Frank is
// radially symmetric: c(u,v) = c(1-u,1-v)), hence 1-lo >= 1/2 carries no
// cancellation (SURVEY.md §7 hard part 6).
__device__ __forceinline__ void frank_sh_f(float u, float v, const FrankThetaF& f, float& s, float& h) {
    const float t = f.t;
    const float lo = fminf(u, v), hi = fmaxf(u, v);
    // warm-up accuracy suffices (the fp64 passes decide convergence): fast
    // exponentials except where expm1 of a small argument needs the full one
    const float ema = __expf(-t * (1.0f - lo)) - 1.0f;  // 1 - lo >= 1/2 after the radial reflection
    const float e2 = __expf(-t * (hi - lo));
    const float emb = expm1f(-t * lo);
    const float e1 = 1.0f + ema, e3 = 1.0f + emb;
    const float b = ema + e2 * emb;
    const float sum = lo + hi;
    const float bp = lo - e1 + e2 * (hi - sum * e3);
    const float bpp = e1 - lo * lo + e2 * (sum * sum * e3 - hi * hi);
    const float rb = __frcp_rn(b);
    const float q = bp * rb;
    s = f.inv_t - f.g - sum - 2.0f * q;
    h = f.hconst - 2.0f * (bpp * rb - q * q);
}

// copula.hpp:147-154
__device__ __forceinline__ double frank_cross_dev(double a, double other, double t, double shift, double rb,
                                                  double bp, double rb2) {
    const double em = expm1(-t * other);
    const double ev = 1.0 + em;
    const double ea = -t * shift * em;
    const double dea = shift * ((t * a - 1.0) * em + t * other * ev);
    return -1.0 - 2.0 * (dea * rb - ea * bp * rb2);
}

// log c, score, Hessian, cross terms at (u, v) — the variance pass.
// expm1(-t*u) and expm1(-t*v) are the bracket's own exponentials (u and v are
// lo and hi in some order): expm1(-t*hi) = em2 + emb + em2*emb exactly, so the
// two cross derivatives (copula.hpp:147-154) need no further exponentials.
__device__ __forceinline__ PointFull frank_full(double u, double v, const FrankTheta& f) {
    if (f.neg) v = 1.0 - v;
    const double t = f.t;
    const bool ulo = u <= v;
    const double lo = ulo ? u : v, hi = ulo ? v : u;
    const double ema = fm_expm1_neg(-t * (1.0 - lo));
    const double k2 = -t * (hi - lo);
    const double em2 = fm_expm1_neg(k2);
    const double emb = fm_expm1_neg(-t * lo);
    const double e2 = 1.0 + em2;
    const double e1 = 1.0 + ema, e3 = 1.0 + emb;
    const double b = ema + e2 * emb;
    const double sum = lo + hi;
    const double bp = lo - e1 + e2 * (hi - sum * e3);
    const double bpp = e1 - lo * lo + e2 * (sum * sum * e3 - hi * hi);
    const double rb = fast_rcp(b);
    const double q = bp * rb;
    PointFull p;
    p.logc = f.logc_const + k2 - 2.0 * fm_log(-b);
    const double sc = f.inv_t - f.g - (u + v) - 2.0 * q;
    p.hess = f.hconst - 2.0 * (bpp * rb - q * q);
    const double rb2 = rb * rb;
    const double emhi = em2 + emb + em2 * emb;  // expm1(-t*hi)
    const double em_u = ulo ? emb : emhi, em_v = ulo ? emhi : emb;
    // cross for first argument a with the other argument o: shift = 1 if a <= o else e2
    auto cross = [&](double a, double o, double em_o, double shift) {
        const double ev = 1.0 + em_o;
        const double ea = -t * shift * em_o;
        const double dea = shift * ((t * a - 1.0) * em_o + t * o * ev);
        return -1.0 - 2.0 * (dea * rb - ea * bp * rb2);
    };
    const double c1 = cross(u, v, em_v, ulo ? 1.0 : e2);
    const double c2 = cross(v, u, em_u, ulo ? (u == v ? 1.0 : e2) : 1.0);
    p.score = f.neg ? -sc : sc;
    p.cross1 = f.neg ? -c1 : c1;
    p.cross2 = c2;
    return p;
}

// ------------------------------------------------------------------ Gumbel
struct GumbelTheta {  // per-theta constants of copula.hpp:238-254
    double t, inv_t, inv_t2, inv_t3, c1t;
    __device__ __forceinline__ explicit GumbelTheta(double th) {
        t = th;
        inv_t = 1.0 / th;
        inv_t2 = inv_t * inv_t;
        inv_t3 = inv_t2 * inv_t;
        c1t = inv_t - 2.0;
    }
};

// Newton pass from the hoisted theta-independent pair (ln(-ln u), ln(-ln v))
// (copula.hpp:201-204 computed once per point in the prepare pass).
__device__ __forceinline__ void gumbel_sh(double lx, double ly, const GumbelTheta& g, double& s, double& h) {
    const double a = g.t * lx, b = g.t * ly;
    const bool amax = a >= b;
    const double m = amax ? a : b;
    const double lmax = amax ? lx : ly, lmin = amax ? ly : lx;
    const double e = fm_exp((amax ? b : a) - m);  // the other exponential is exactly 1 (copula.hpp:209-210)
    const double sden = 1.0 + e;
    const double rs = fast_rcp(sden);
    const double lnS = m + fm_log(sden);
    const double w = fm_exp(lnS * g.inv_t);
    const double r = (lmax + e * lmin) * rs;
    const double r2 = (lmax * lmax + e * lmin * lmin) * rs;
    const double rt = r2 - r * r;
    const double lw_t = r * g.inv_t - lnS * g.inv_t2;
    const double wt = w * lw_t;
    const double lw_tt = rt * g.inv_t - 2.0 * r * g.inv_t2 + 2.0 * lnS * g.inv_t3;
    const double wtt = w * (lw_t * lw_t + lw_tt);
    const double gg = w + g.t - 1.0;
    const double rg = fast_rcp(gg);
    const double wt1 = wt + 1.0;
    s = -wt + lx + ly - lnS * g.inv_t2 + g.c1t * r + wt1 * rg;
    h = -wtt - 2.0 * r * g.inv_t2 + 2.0 * lnS * g.inv_t3 + g.c1t * rt + (wtt * gg - wt1 * wt1) * rg * rg;
}

struct GumbelThetaF {
    float t, inv_t, inv_t2, inv_t3, c1t;
    __device__ __forceinline__ explicit GumbelThetaF(double th) {
        t = static_cast<float>(th);
        inv_t = static_cast<float>(1.0 / th);
        inv_t2 = static_cast<float>(1.0 / (th * th));
        inv_t3 = static_cast<float>(1.0 / (th * th * th));
        c1t = static_cast<float>(1.0 / th - 2.0);
    }
};

__device__ __forceinline__ void gumbel_sh_f(float lx, float ly, const GumbelThetaF& g, float& s, float& h) {
    const float a = g.t * lx, b = g.t * ly;
    const bool amax = a >= b;
    const float m = amax ? a : b;
    const float lmax = amax ? lx : ly, lmin = amax ? ly : lx;
    const float e = __expf((amax ? b : a) - m);
    const float sden = 1.0f + e;
    const float rs = __frcp_rn(sden);
    const float lnS = m + __logf(sden);  // warm-up accuracy (absolute error ~1e-7)
    const float w = __expf(lnS * g.inv_t);
    const float r = (lmax + e * lmin) * rs;
    const float r2 = (lmax * lmax + e * lmin * lmin) * rs;
    const float d = lmax - lmin;  // r2 - r^2 = e d^2 / (1+e)^2, free of cancellation
    const float rt = e * d * d * rs * rs;
    (void)r2;
    const float lw_t = r * g.inv_t - lnS * g.inv_t2;
    const float wt = w * lw_t;
    const float lw_tt = rt * g.inv_t - 2.0f * r * g.inv_t2 + 2.0f * lnS * g.inv_t3;
    const float wtt = w * (lw_t * lw_t + lw_tt);
    const float gg = w + g.t - 1.0f;
    const float rg = __frcp_rn(gg);
    const float wt1 = wt + 1.0f;
    s = -wt + lx + ly - lnS * g.inv_t2 + g.c1t * r + wt1 * rg;
    h = -wtt - 2.0f * r * g.inv_t2 + 2.0f * lnS * g.inv_t3 + g.c1t * rt + (wtt * gg - wt1 * wt1) * rg * rg;
}

// Full evaluation for the variance pass (copula.hpp:199-254), from
// lx = ln(-ln u), x = -ln u, ix = 1/x, iu = 1/u (and the same for v): the
// rank-table entries when u is rank-derived. exp(a - m) of the larger
// exponent is exactly 1, and exp(a - ln S) = exp(a - m) / S, so a point costs
// four transcendentals.
__device__ __forceinline__ PointFull gumbel_full_t(double lx, double ly, double x, double y, double ix, double iy,
                                                   double iu, double iv, const GumbelTheta& g) {
    const double a = g.t * lx, b = g.t * ly;
    const bool amax = a >= b;
    const double m = amax ? a : b;
    // libdevice here: the fm_* forms measured slower in this register-heavy
    // pass (23.96 -> 25.9 ms per 1e9 points at C5), unlike the Newton pass
    const double e = exp((amax ? b : a) - m);
    const double ea = amax ? 1.0 : e, eb = amax ? e : 1.0;
    const double sden = 1.0 + e;
    const double rs = fast_rcp(sden);
    const double lnS = m + log(sden);
    const double w = exp(lnS * g.inv_t);
    const double r = (ea * lx + eb * ly) * rs;
    const double r2 = (ea * lx * lx + eb * ly * ly) * rs;
    const double pa = ea * rs * ix, pb = eb * rs * iy;
    const double rt = r2 - r * r;
    const double lw_t = r * g.inv_t - lnS * g.inv_t2;
    const double wt = w * lw_t;
    const double lw_tt = rt * g.inv_t - 2.0 * r * g.inv_t2 + 2.0 * lnS * g.inv_t3;
    const double wtt = w * (lw_t * lw_t + lw_tt);
    const double gg = w + g.t - 1.0;
    const double rg = fast_rcp(gg);
    const double wt1 = wt + 1.0;
    PointFull p;
    p.logc = -w + (g.t - 1.0) * (lx + ly) + (x + y) + g.c1t * lnS + log(gg);
    p.score = -wt + lx + ly - lnS * g.inv_t2 + g.c1t * r + wt1 * rg;
    p.hess = -wtt - 2.0 * r * g.inv_t2 + 2.0 * lnS * g.inv_t3 + g.c1t * rt + (wtt * gg - wt1 * wt1) * rg * rg;
    // copula.hpp:228-236
    const double rg2 = rg * rg;
    {
        const double pt = pa * (lx - r);
        const double cx = -wt * pa - w * pt + ix - 2.0 * pa + (1.0 - 2.0 * g.t) * pt +
                          ((wt * pa + w * pt) * gg - w * pa * wt1) * rg2;
        p.cross1 = -cx * iu;
    }
    {
        const double pt = pb * (ly - r);
        const double cy = -wt * pb - w * pt + iy - 2.0 * pb + (1.0 - 2.0 * g.t) * pt +
                          ((wt * pb + w * pt) * gg - w * pb * wt1) * rg2;
        p.cross2 = -cy * iv;
    }
    return p;
}

__device__ __forceinline__ PointFull gumbel_full(double u, double v, const GumbelTheta& g) {
    const double x = -log(u), y = -log(v);
    return gumbel_full_t(log(x), log(y), x, y, fast_rcp(x), fast_rcp(y), fast_rcp(u), fast_rcp(v), g);
}

// from the hoisted (ln x, ln y) pair of the prepare pass
__device__ __forceinline__ PointFull gumbel_full_l(double u, double v, double lx, double ly, const GumbelTheta& g) {
    const double x = exp(lx), y = exp(ly);
    return gumbel_full_t(lx, ly, x, y, fast_rcp(x), fast_rcp(y), fast_rcp(u), fast_rcp(v), g);
}

// log c only (pseudo_loglik API), any family; u, v already clamped.
__device__ __forceinline__ double logc_any(int fam, double t, double u, double v) {
    if (fam == 0) {
        const double x = dev_phi_inv(u), y = dev_phi_inv(v);
        const double a = 1.0 - t * t;
        return -0.5 * log(a) + (2.0 * t * x * y - t * t * (x * x + y * y)) / (2.0 * a);
    }
    if (fam == 1) {
        double tt = t;
        if (t < 0.0) { tt = -t; v = 1.0 - v; }
        const double lo = fmin(u, v), hi = fmax(u, v);
        const double k2 = -tt * (hi - lo);
        const double b = expm1(-tt * (1.0 - lo)) + exp(k2) * expm1(-tt * lo);
        return log(tt) + log(-expm1(-tt)) + k2 - 2.0 * log(-b);
    }
    const double x = -log(u), y = -log(v);
    const double lx = log(x), ly = log(y);
    const double a = t * lx, b = t * ly;
    const double m = fmax(a, b);
    const double lnS = m + log(exp(a - m) + exp(b - m));
    const double w = exp(lnS / t);
    return -w + (t - 1.0) * (lx + ly) + (x + y) + (1.0 / t - 2.0) * lnS + log(w + t - 1.0);
}

}  // namespace pcb

// K2 lik_reduce + batched safeguarded Newton on sm_100a.
//
// Replaces the reference's absent mpl_estimator `fit` (SPEC.md:216-224,
// 242-244): every block's theta-hat is the root of its pseudo-score
// equation, all blocks in lockstep, one fused score+Hessian reduction launch
// per Newton pass (the asymptotic variance is variance.cu).
// Data layout (HBM): the rank stage leaves packed (r2|pos) u64 per point and
// column ([2][n_rows]); the prepare pass writes the theta-independent
// per-point pair T (double2, or float2 on the fp32 likelihood path) that the
// Newton passes stream:
//   Gaussian : (x, y) = (Phi^-1(u), Phi^-1(v)); the fit itself reduces to the
//              sufficient statistics Sxy, Sss (no Newton data pass); T feeds
//              the variance pass
//   Frank    : (u, v)   (fp32: edge-encoded, see frank_edge)
//   Gumbel   : (ln(-ln u), ln(-ln v))   (copula.hpp:201-204, hoisted)
// Reductions are deterministic (common.cuh tile_reduce): no floating-point
// atomics, so results do not depend on scheduling, the GPU count or the run.
#include <algorithm>
#include <cmath>
#include <string>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "devmath.cuh"
#include "internal.hpp"

namespace pcb {
namespace {

bool getenv_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && v[0] && v[0] != '0';
}

constexpr int kMaxPasses = 64;
// Newton step tolerances (relative to max(1,|theta|)). A converged step of
// size d leaves an error ~C*d^2 (quadratic convergence): 1e-6 -> ~1e-12.
constexpr double kTol64 = 1e-6;
constexpr double kTol32 = 1e-6;
constexpr int kWarmPasses = 2;
#ifndef PCB_GAUSS_T_DEFAULT
#define PCB_GAUSS_T_DEFAULT 0
#endif
constexpr bool kGaussT = PCB_GAUSS_T_DEFAULT != 0;
// fp32 likelihood mode: Frank blocks whose iterate has |theta| below this run
// the pass in fp64 per-point arithmetic (on the same fp32 edge-encoded
// inputs). The Frank score (copula.hpp:156-172) cancels terms of size ~2/theta,
// so fp32 per-point sums lose ~eps32 * 2/theta^2 relative there
// (tools/fp32_edges.py: 1e-4 at theta = 0.3, 0.86 at theta = 0.05).
#ifndef PCB_FRANK32_EXACT
#define PCB_FRANK32_EXACT 2.0
#endif
constexpr double kFrank32Exact = PCB_FRANK32_EXACT;
// Likewise Gumbel blocks with theta < 1.1: near the boundary theta = 1 the
// variance amplifies any error of theta-hat ~100x (a 1e-7 fp32 root error
// became 1.1e-5 in sigma2 at theta-hat = 1.002).
#ifndef PCB_GUMBEL32_EXACT
#define PCB_GUMBEL32_EXACT 1.1
#endif
constexpr double kGumbel32Exact = PCB_GUMBEL32_EXACT;
#ifndef PCB_LIK_UNROLL
#define PCB_LIK_UNROLL 2
#endif
constexpr int kLikUnroll = PCB_LIK_UNROLL;  // fp64 Newton pass: points per thread in flight  // fp32 warm-up passes before the fp64 passes (fp64 mode)

// Spearman-rho -> theta inversion tables for the Archimedean init.
constexpr int NTAB = 256;
__constant__ double c_frank_rho[NTAB], c_frank_theta[NTAB];
__constant__ double c_gumbel_rho[NTAB], c_gumbel_theta[NTAB];

__device__ double invert_table(const double* rho, const double* th, double r) {
    if (r <= rho[0]) return th[0];
    if (r >= rho[NTAB - 1]) return th[NTAB - 1];
    int lo = 0, hi = NTAB - 1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (rho[mid] <= r) lo = mid;
        else hi = mid;
    }
    const double w = (r - rho[lo]) / (rho[hi] - rho[lo]);
    return th[lo] + w * (th[hi] - th[lo]);
}

// Safeguarded Newton step on the pseudo-score (mirrors oracle/mpl_driver.hpp
// Driver::fit's bracket / boundary rules; SPEC.md:242 keeps iterates inside
// the domain). Runs in one thread per block.
// f64: the sums come from fp64 per-point arithmetic. Then a step inside the
// tolerance ends the fit only if the quadratic-convergence residual it
// leaves, |S''| d^2 / (2|H|) with S'' = dH/dtheta from the previous pass,
// is below 1e-13 max(1, |theta|); otherwise the step is taken and one more
// pass runs (score curvature is large near the Gumbel boundary theta = 1,
// where sigma2 also amplifies any error of theta-hat).
__device__ void newton_update(BlockState& s, int fam, double S, double H, double tol, unsigned* running,
                              bool f64 = false) {
    s.iters += 1;
    const double th_prev = s.th_prev, h_prev = s.h_prev;
    // The curvature estimate below differences this pass's Hessian sum with
    // the previous pass's, which on the first fp64 pass is an fp32 warm-up
    // sum. Its rounding can only move the estimated residual by
    // ~eps32 |H| d^2 / dtheta, i.e. turn a borderline stop into one more fp64
    // pass (C5: 139 of 8000 Frank and 4 Gumbel blocks, +0.1 / +0.3 ms) -- it
    // never replaces a curvature estimate by none, which recording fp64
    // passes only would do for the first fp64 pass.
    if (isfinite(H)) {
        s.th_prev = s.theta;
        s.h_prev = H;
    }
    if (tol < 0.0) {  // warm-up pass (fp32 per-point arithmetic): move theta, decide nothing
        if (isfinite(S) && isfinite(H) && H < 0.0) {
            double cand = s.theta - S / H;
            if (fam == kGumbel) cand = fmax(cand, 1.0);
            if (isfinite(cand) && !(fam == kFrank && fabs(cand) < 1e-6)) s.theta = cand;
        }
        return;
    }
    double t = s.theta;
    if (!isfinite(S) || !isfinite(H)) {
        s.status = kNotConverged;
        atomicSub(running, 1u);
        return;
    }
    if (S > 0.0) s.lo = t;
    else s.hi = t;
    if (fam == kGumbel && t == 1.0) {  // boundary theta = 1
        s.tried_one = 1;
        if (S <= 0.0) {
            s.step = 0.0;
            s.status = kConverged;
            atomicSub(running, 1u);
            return;
        }
    }
    double cand = NAN;
    if (H < 0.0) {
        cand = t - S / H;
        bool small = fabs(cand - t) <= tol * fmax(1.0, fabs(t));
        if (small && f64 && isfinite(h_prev) && th_prev != t) {
            const double d = cand - t, s2 = (H - h_prev) / (t - th_prev);
            small = !(fabs(s2) * d * d > 2e-13 * fabs(H) * fmax(1.0, fabs(t)));
        }
        if (small) {
            if (!(fam == kGumbel && cand < 1.0)) t = cand;
            s.step = cand - s.theta;
            s.theta = t;
            s.status = kConverged;
            atomicSub(running, 1u);
            return;
        }
    }
    bool inside = isfinite(cand) && cand > s.lo && cand < s.hi;
    if (!inside && fam == kGumbel && !s.tried_one && isfinite(cand) && cand <= 1.0) {
        cand = 1.0;
        inside = true;
    }
    if (!inside) {
        if (isfinite(s.lo) && isfinite(s.hi)) cand = 0.5 * (s.lo + s.hi);
        else if (isfinite(s.lo)) cand = s.lo + fmax(1.0, fabs(s.lo));
        else cand = s.hi - fmax(1.0, fabs(s.hi));
        if (fam == kGumbel && !(cand > 1.0)) cand = 1.0;
    }
    if (fam == kFrank && fabs(cand) < 1e-6) cand = cand < 0.0 ? -1e-6 : 1e-6;
    s.step = cand - t;
    s.theta = cand;
    if (fabs(s.step) <= 1e-14 * fmax(1.0, fabs(cand))) {
        s.status = kConverged;
        atomicSub(running, 1u);
        return;
    }
    if (s.iters >= kMaxPasses) {
        s.status = kNotConverged;
        atomicSub(running, 1u);
    }
}

// Edge encoding for fp32 Frank inputs: p = u (u <= 1/2) or -(1-u) (u > 1/2),
// computed in fp64, so both u and 1-u keep full fp32 relative precision.
__device__ __forceinline__ float frank_edge(double u) { return static_cast<float>(u <= 0.5 ? u : -(1.0 - u)); }
// fp64 value of an edge-encoded input (fp64 T holds u itself)
__device__ __forceinline__ double frank_decode(float p) { return p >= 0.0f ? static_cast<double>(p) : 1.0 + p; }
__device__ __forceinline__ double frank_decode(double u) { return u; }
__device__ __forceinline__ void frank_unedge(float p, float& val, float& comp) {
    if (p >= 0.0f) {
        val = p;
        comp = 1.0f - p;
    } else {
        val = 1.0f + p;
        comp = -p;
    }
}

__global__ void k_init_state(BlockState* st, const Seg* segs, int nseg, const int32_t* bad, unsigned* running,
                             const double* theta_in) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= nseg) return;
    BlockState s;
    memset(&s, 0, sizeof s);
    s.begin = segs[m].begin;
    s.n = segs[m].n;
    s.theta = theta_in ? theta_in[m] : NAN;
    s.lo = -INFINITY;
    s.hi = INFINITY;
    s.th_prev = NAN;
    s.h_prev = NAN;
    s.loglik = NAN;
    s.sigma2 = NAN;
    if (bad && bad[m]) s.status = kBadData;
    else if (s.n < static_cast<uint64_t>(kMinRows)) s.status = kTooSmall;
    else {
        s.status = theta_in ? kConverged : kRunning;
        if (!theta_in) atomicAdd(running, 1u);
    }
    st[m] = s;
}

// Prepare pass: theta-independent per-point pair + init statistics; the
// segment's last tile computes the starting theta (Gaussian: solves the fit).
// with_fit == 0 (variance-only API): only T is written. `gtab` (rank-derived
// u only) holds the per-rank transform of the block's size: Phi^-1(u)
// (Gaussian) or ln(-ln u) (Gumbel), bit-identical to computing it per point.
template <int FAM, class TO>
#ifndef PCB_PREP_OCC
#define PCB_PREP_OCC 0
#endif
__global__ void __launch_bounds__(FT, PCB_PREP_OCC) k_prepare(BlockState* st, const Seg* segs, int nseg, RankRef R,
                                               const double* __restrict__ u1, const double* __restrict__ u2,
                                               uint64_t n_rows, TO* __restrict__ T, float2* __restrict__ T32,
                                               const double* __restrict__ gtab, const uint64_t* goff,
                                               double* partials, unsigned* tickets, unsigned* running, int with_fit) {
    const uint32_t tile = blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    const int32_t status = st[m].status;
    if (with_fit ? status != kRunning : status != kConverged) return;
    const double scale = 1.0 / (static_cast<double>(S.n) + 1.0);
    const uint32_t base = (tile - S.tile0) * FTILE;
    const double* gt = gtab ? gtab + 4 * goff[m] : nullptr;  // 4 doubles per rank entry
    const bool rt = R.routed && R.routed[m];
    double v[2] = {0.0, 0.0};
#ifndef PCB_U_PREP
#define PCB_U_PREP 4
#endif
#ifndef PCB_U_PREP_U
#define PCB_U_PREP_U 2
#endif
    constexpr int U = FAM == kGumbel ? PCB_U_PREP_U : PCB_U_PREP;  // points per thread in flight (measured at C5)
    for (int k0 = 0; k0 < PPT; k0 += U) {
        double uu[U], ww[U], gx[U], gy[U];
        uint32_t ra[U], rb[U];
        if (!u1) {
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const uint32_t i = base + tile_row(k0 + j);
                if (i < S.n) {
                    const uint64_t row = S.begin + i;
                    if (rt) {
                        ra[j] = R.route[row];
                        rb[j] = R.route[n_rows + row];
                    } else {
                        ra[j] = rank_r2(R.rp[row]);
                        rb[j] = rank_r2(R.rp[n_rows + row]);
                    }
                }
            }
            if (rt) {
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const uint32_t i = base + tile_row(k0 + j);
                    if (i < S.n) {
                        ra[j] = R.r2s[slot_index(R, nseg, 0, m, ra[j])];
                        rb[j] = R.r2s[slot_index(R, nseg, 1, m, rb[j])];
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + tile_row(k0 + j);
            if (i < S.n) {
                const uint64_t row = S.begin + i;
                if (u1) {
                    uu[j] = u1[row];
                    ww[j] = u2[row];
                } else {
                    const uint32_t r1 = ra[j], r2 = rb[j];
                    uu[j] = __dmul_rn(0.5 * static_cast<double>(r1), scale);
                    ww[j] = __dmul_rn(0.5 * static_cast<double>(r2), scale);
                    if (gt) {
                        gx[j] = gt[4 * r1];
                        gy[j] = gt[4 * r2];
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + tile_row(k0 + j);
            if (i >= S.n) continue;
            const uint64_t row = S.begin + i;
            const double u = clamp_unit(uu[j]), w = clamp_unit(ww[j]);
            if (FAM == kGaussian) {
                double x, y;
                if (gt) {
                    x = gx[j];
                    y = gy[j];
                    if (T) T[row] = TO{static_cast<decltype(TO::x)>(x), static_cast<decltype(TO::x)>(y)};
                } else {
                    x = dev_phi_inv(u);
                    y = dev_phi_inv(w);
                    T[row] = TO{static_cast<decltype(TO::x)>(x), static_cast<decltype(TO::x)>(y)};
                }
                v[0] += x * y;
                v[1] += x * x + y * y;
            } else {
                v[0] += u * w;
                if (FAM == kFrank) {
                    if (sizeof(TO) == 8)
                        T[row] = TO{static_cast<decltype(TO::x)>(frank_edge(u)),
                                    static_cast<decltype(TO::x)>(frank_edge(w))};
                    else
                        T[row] = TO{static_cast<decltype(TO::x)>(u), static_cast<decltype(TO::x)>(w)};
                    if (T32) T32[row] = float2{frank_edge(u), frank_edge(w)};
                } else {
                    const double lx = gt ? gx[j] : log(-log(u)), ly = gt ? gy[j] : log(-log(w));
                    T[row] = TO{static_cast<decltype(TO::x)>(lx), static_cast<decltype(TO::x)>(ly)};
                    if (T32) T32[row] = float2{static_cast<float>(lx), static_cast<float>(ly)};
                }
            }
        }
    }
    if (!with_fit) return;
    __shared__ double sh[(FT / 32) * 2];
    if (!tile_reduce<2>(v, sh, partials, tickets, S, m, tile)) return;
    if (threadIdx.x != 0) return;
    BlockState s = st[m];
    const double n = static_cast<double>(S.n);
    s.stat0 = v[0];
    s.stat1 = v[1];
    if (FAM == kGaussian) {
        // Newton on the closed-form S(t), H(t) of the sufficient statistics
        double t = fmin(fmax(v[0] / (0.5 * v[1]), -0.99), 0.99);
        double lo = -1.0, hi = 1.0;
        bool conv = false;
        for (int it = 0; it < 200; ++it) {
            double Sg, Hg;
            gauss_stats_sh(t, n, v[0], v[1], Sg, Hg);
            if (!isfinite(Sg) || !isfinite(Hg)) break;
            if (Sg > 0.0) lo = t;
            else hi = t;
            double cand = NAN;
            if (Hg < 0.0) {
                cand = t - Sg / Hg;
                if (fabs(cand - t) <= 1e-15 * fmax(1.0, fabs(t))) {
                    t = cand;
                    conv = true;
                    break;
                }
            }
            if (!(isfinite(cand) && cand > lo && cand < hi)) cand = 0.5 * (lo + hi);
            if (fabs(cand - t) <= 1e-15 * fmax(1.0, fabs(t))) {
                t = cand;
                conv = true;
                break;
            }
            t = cand;
        }
        s.theta = t;
        s.iters = 1;
        s.status = conv ? kConverged : kNotConverged;
        atomicSub(running, 1u);
    } else {
        // Spearman's rho from the pseudo-observations (no-ties form), inverted
        // through the family's rho(theta) table: a consistent start whose
        // error is O(n^-1/2), so Newton needs ~3 passes.
        const double rho = 12.0 * (n + 1.0) / (n - 1.0) * (v[0] / n - 0.25);
        double t;
        if (FAM == kFrank) {
            t = invert_table(c_frank_rho, c_frank_theta, fabs(rho));
            t = fmax(t, 0.05);
            if (rho < 0.0) t = -t;
        } else {
            t = rho <= 0.0 ? 1.0 : invert_table(c_gumbel_rho, c_gumbel_theta, rho);
            t = fmax(t, 1.0);
        }
        s.theta = t;
        s.lo = FAM == kGumbel ? 1.0 : -INFINITY;
        s.hi = INFINITY;
    }
    st[m] = s;
}

// One Newton pass: fused per-point score + Hessian at each running block's
// current theta, deterministic block reduction, in-kernel Newton update.
// F32: fp32 per-point arithmetic (the warm-up passes, or the fp32 precision
// mode); TI: the stored pair — float2 (T32 / fp32 T) or double2 (fp64 T,
// converted at load: Frank to the edge encoding, Gumbel by rounding).
// Four CTAs per SM: 64 registers (the allocation measured fastest; left to
// itself the fp64 Gumbel pass takes 80 and loses 1.3 ms per family at C5).
#ifndef PCB_LIK_OCC
#define PCB_LIK_OCC 4
#endif
template <int FAM, class TI, bool F32 = (sizeof(TI) == 8)>
__global__ void __launch_bounds__(FT, PCB_LIK_OCC) k_lik(BlockState* st, const Seg* segs, int nseg, const TI* __restrict__ T,
                                           double* partials, unsigned* tickets, unsigned* running, double tol,
                                           const uint32_t* tile_list) {
    const uint32_t tile = tile_list ? tile_list[blockIdx.x] : blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (st[m].status != kRunning) return;
    const double theta = st[m].theta;
    const uint32_t base = (tile - S.tile0) * FTILE;
    const TI* Tb = T + S.begin + base;
    const uint32_t cnt = min(FTILE, S.n - base);
    double v[2] = {0.0, 0.0};
    bool f64pass = !F32;
    auto warm_pair = [](const TI& p) -> float2 {
        if constexpr (sizeof(TI) == 8) {
            return p;
        } else if constexpr (FAM == kFrank) {
            return float2{frank_edge(p.x), frank_edge(p.y)};
        } else {
            return float2{static_cast<float>(p.x), static_cast<float>(p.y)};
        }
    };
    if constexpr (!F32) {  // fp64
        if (FAM == kFrank) {
            const FrankTheta f(theta);
            auto pass = [&](auto neg, auto big) {
#pragma unroll(kLikUnroll)
                for (int k = 0; k < PPT; ++k) {
                    const uint32_t i = k * FT + threadIdx.x;
                    if (i < cnt) {
                        const TI p = Tb[i];
                        double s, h;
                        frank_sh_t<decltype(neg)::value, decltype(big)::value>(p.x, p.y, f, s, h);
                        v[0] += s;
                        v[1] += h;
                    }
                }
            };
            // sign and size of theta are per block: one branch per CTA
            const bool big = f.t > 700.0;
            if (f.neg) {
                if (big) pass(std::true_type{}, std::true_type{});
                else pass(std::true_type{}, std::false_type{});
            } else {
                if (big) pass(std::false_type{}, std::true_type{});
                else pass(std::false_type{}, std::false_type{});
            }
        } else {
            const GumbelTheta g(theta);
#pragma unroll(kLikUnroll)
            for (int k = 0; k < PPT; ++k) {
                const uint32_t i = k * FT + threadIdx.x;
                if (i < cnt) {
                    const TI p = Tb[i];
                    double s, h;
                    gumbel_sh(p.x, p.y, g, s, h);
                    v[0] += s;
                    v[1] += h;
                }
            }
        }
    } else if (tol >= 0.0 && (FAM == kFrank ? fabs(theta) < kFrank32Exact : theta < kGumbel32Exact)) {
        // fp32 mode, ill-conditioned theta: fp64 arithmetic on the decoded
        // fp32 inputs (this pass decides convergence in fp64, like the fp64 mode)
        f64pass = true;
        if (FAM == kFrank) {
            const FrankTheta f(theta);
            for (int k = 0; k < PPT; ++k) {
                const uint32_t i = k * FT + threadIdx.x;
                if (i < cnt) {
                    const TI p = Tb[i];
                    double s, h;
                    frank_sh(frank_decode(p.x), frank_decode(p.y), f, s, h);
                    v[0] += s;
                    v[1] += h;
                }
            }
        } else {
            const GumbelTheta g(theta);
            for (int k = 0; k < PPT; ++k) {
                const uint32_t i = k * FT + threadIdx.x;
                if (i < cnt) {
                    const TI p = Tb[i];
                    double s, h;
                    gumbel_sh(static_cast<double>(p.x), static_cast<double>(p.y), g, s, h);
                    v[0] += s;
                    v[1] += h;
                }
            }
        }
    } else {  // fp32 per-point arithmetic: per-thread fp32 partial sums (PPT points), fp64 beyond
        float fs = 0.0f, fh = 0.0f;
#ifndef PCB_WB
#define PCB_WB 8
#endif
        constexpr int WB = PCB_WB;  // T32 loads in flight per thread
        if (FAM == kFrank) {
            const FrankThetaF f(theta);
            for (int k0 = 0; k0 < PPT; k0 += WB) {
              TI pb[WB];
#pragma unroll
              for (int u = 0; u < WB; ++u) {
                const uint32_t i = (k0 + u) * FT + threadIdx.x;
                if (i < cnt) pb[u] = Tb[i];
              }
#pragma unroll
              for (int u = 0; u < WB; ++u) {
                const uint32_t i = (k0 + u) * FT + threadIdx.x;
                if (i < cnt) {
                    const float2 p = warm_pair(pb[u]);
                    float uv, uc, vv, vc;
                    frank_unedge(p.x, uv, uc);
                    frank_unedge(p.y, vv, vc);
                    if (f.neg) {  // c(u,v;-t) = c(u,1-v;t)
                        const float tmp = vv;
                        vv = vc;
                        vc = tmp;
                    }
                    // radial symmetry c(u,v) = c(1-u,1-v): evaluate on the side with lo + hi <= 1
                    if (uv + vv > 1.0f) {
                        float tmp = uv;
                        uv = uc;
                        uc = tmp;
                        tmp = vv;
                        vv = vc;
                        vc = tmp;
                    }
                    float s, h;
                    frank_sh_f(uv, vv, f, s, h);
                    fs += f.neg ? -s : s;
                    fh += h;
                }
              }
            }
        } else {
            const GumbelThetaF g(theta);
            for (int k0 = 0; k0 < PPT; k0 += WB) {
              TI pb[WB];
#pragma unroll
              for (int u = 0; u < WB; ++u) {
                const uint32_t i = (k0 + u) * FT + threadIdx.x;
                if (i < cnt) pb[u] = Tb[i];
              }
#pragma unroll
              for (int u = 0; u < WB; ++u) {
                const uint32_t i = (k0 + u) * FT + threadIdx.x;
                if (i < cnt) {
                    float s, h;
                    const float2 p = warm_pair(pb[u]);
                    gumbel_sh_f(p.x, p.y, g, s, h);
                    fs += s;
                    fh += h;
                }
              }
            }
        }
        v[0] = fs;
        v[1] = fh;
    }
    __shared__ double sh[(FT / 32) * 2];
    if (!tile_reduce<2>(v, sh, partials, tickets, S, m, tile)) return;
    if (threadIdx.x == 0) {
        BlockState s = st[m];
        newton_update(s, FAM, v[0], v[1], tol, running, f64pass);
        st[m] = s;
    }
}

// The theta-independent per-point transforms of u = (0.5*r2)/(n+1) for every
// r2 in [2, 2n] of a block of n ranked rows, one 32-byte entry (one L2
// sector) per r2, with the same arithmetic as the per-point path:
//   Gaussian {x = Phi^-1(u), exp(x^2/2), 0, 0}
//   Gumbel   {ln(-ln u), -ln u (as exp of the former), 1/(-ln u), 1/u}
__global__ void k_rank_table(double* tab, uint32_t n, int fam) {
    const double scale = 1.0 / (static_cast<double>(n) + 1.0);
    for (uint32_t r2 = blockIdx.x * blockDim.x + threadIdx.x; r2 <= 2 * n; r2 += gridDim.x * blockDim.x) {
        const double u = clamp_unit(__dmul_rn(0.5 * static_cast<double>(r2), scale));
        double4 t = make_double4(0.0, 0.0, 0.0, 0.0);
        if (r2 >= 2) {
            if (fam == kGaussian) {
                const double x = dev_phi_inv(u);
                t = make_double4(x, exp(0.5 * x * x), 0.0, 0.0);
            } else {
                const double lx = log(-log(u)), x = exp(lx);
                t = make_double4(lx, x, 1.0 / x, 1.0 / u);
            }
        }
        reinterpret_cast<double2*>(tab)[2 * r2] = make_double2(t.x, t.y);
        reinterpret_cast<double2*>(tab)[2 * r2 + 1] = make_double2(t.z, t.w);
    }
}

struct RecordOut {  // == pcb_fit_result
    double theta_hat, sigma2, loglik;
    uint64_t n;
    int32_t iterations, converged, status, reserved;
};

__global__ void k_finalize(const BlockState* st, int nseg, RecordOut* out, int with_variance) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= nseg) return;
    const BlockState s = st[m];
    RecordOut r;
    r.theta_hat = (s.status == kBadData || s.status == kTooSmall) ? NAN : s.theta;
    r.sigma2 = with_variance ? s.sigma2 : NAN;
    r.loglik = s.loglik;
    r.n = s.n;
    r.iterations = s.iters;
    r.converged = s.status == kConverged ? 1 : 0;
    r.status = s.status == kRunning ? kNotConverged : s.status;
    r.reserved = 0;
    out[m] = r;
}

__global__ void __launch_bounds__(FT) k_loglik(const Seg* segs, int nseg, const double* theta, const double* u1,
                                              const double* u2, int fam, double* partials, unsigned* tickets,
                                              double* out) {
    const uint32_t tile = blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    const double t = theta[m];
    const uint32_t base = (tile - S.tile0) * FTILE;
    double v[1] = {0.0};
    for (int k = 0; k < PPT; ++k) {
        const uint32_t i = base + k * FT + threadIdx.x;
        if (i >= S.n) break;
        const uint64_t row = S.begin + i;
        v[0] += clip_log(logc_any(fam, t, clamp_unit(u1[row]), clamp_unit(u2[row])));
    }
    __shared__ double sh[FT / 32];
    if (!tile_reduce<1>(v, sh, partials, tickets, S, m, tile)) return;
    if (threadIdx.x == 0) out[m] = v[0];
}

// ------------------------------------------------------------ host tables
double debye(int k, double x) {  // D_k(x) = k/x^k int_0^x t^k/(e^t-1) dt, composite Simpson
    if (x == 0.0) return 1.0;
    const int N = 2000;
    const double h = x / N;
    auto f = [k](double t) { return t == 0.0 ? (k == 1 ? 1.0 : 0.0) : std::pow(t, k) / std::expm1(t); };
    double s = f(0.0) + f(x);
    for (int i = 1; i < N; ++i) s += (i & 1 ? 4.0 : 2.0) * f(i * h);
    return k / std::pow(x, k) * s * h / 3.0;
}

bool g_tables_ready = false;
double h_frank_rho[NTAB], h_frank_theta[NTAB], h_gumbel_rho[NTAB], h_gumbel_theta[NTAB];

void build_tables() {
    if (g_tables_ready) return;
    // Frank: rho_S(theta) = 1 - 12/theta (D1(theta) - D2(theta)), theta > 0
    for (int k = 0; k < NTAB; ++k) {
        const double th = 0.02 + 80.0 * std::pow(static_cast<double>(k) / (NTAB - 1), 2.0);
        h_frank_theta[k] = th;
        h_frank_rho[k] = 1.0 - 12.0 / th * (debye(1, th) - debye(2, th));
    }
    // Gumbel: rho_S(theta) = 12 int int C(u,v) du dv - 3 by tensor Gauss-Legendre
    const int Q = 64;
    std::vector<double> xn(Q), wn(Q);
    for (int i = 0; i < Q; ++i) {  // Legendre nodes by Newton on P_Q
        double x = std::cos(M_PI * (i + 0.75) / (Q + 0.5)), dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = x;
            for (int j = 2; j <= Q; ++j) {
                const double p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            dp = Q * (x * p1 - p0) / (x * x - 1.0);
            const double dx = p1 / dp;
            x -= dx;
            if (std::fabs(dx) < 1e-15) break;
        }
        xn[i] = 0.5 * (x + 1.0);
        wn[i] = 1.0 / ((1.0 - x * x) * dp * dp);  // = 0.5 * 2/((1-x^2)P'^2)
    }
    for (int k = 0; k < NTAB; ++k) {
        const double tau = 0.97 * static_cast<double>(k) / (NTAB - 1);
        const double th = 1.0 / (1.0 - tau);
        double s = 0.0;
        for (int i = 0; i < Q; ++i)
            for (int j = 0; j < Q; ++j) {
                const double x = -std::log(xn[i]), y = -std::log(xn[j]);
                s += wn[i] * wn[j] * std::exp(-std::pow(std::pow(x, th) + std::pow(y, th), 1.0 / th));
            }
        h_gumbel_theta[k] = th;
        h_gumbel_rho[k] = 12.0 * s - 3.0;
    }
    g_tables_ready = true;
}

uint32_t ftiles(uint64_t n) { return static_cast<uint32_t>((n + FTILE - 1) / FTILE); }

template <int FAM>
void launch_prepare(Ctx& c, uint32_t tiles, BlockState* st, const Seg* segs, int K, const FitIO& io, void* T,
                    bool fp32T, float2* T32, const double* gtab, const uint64_t* goff, double* part, unsigned* tick,
                    unsigned* running, int with_fit) {
    if (fp32T)
        k_prepare<FAM, float2><<<tiles, FT, 0, c.stream>>>(st, segs, K, io.rank->ref(), io.u1, io.u2, io.n_rows,
                                                          static_cast<float2*>(T), nullptr, gtab, goff, part, tick,
                                                          running, with_fit);
    else
        k_prepare<FAM, double2><<<tiles, FT, 0, c.stream>>>(st, segs, K, io.rank->ref(), io.u1, io.u2, io.n_rows,
                                                           static_cast<double2*>(T), T32, gtab, goff, part, tick,
                                                           running, with_fit);
    c.count_launch();
}

template <int FAM>
void launch_lik(Ctx& c, uint32_t tiles, BlockState* st, const Seg* segs, int K, bool f32, const void* T,
                double* part, unsigned* tick, unsigned* running, double tol, bool t64 = false,
                const uint32_t* tile_list = nullptr) {
    if (f32 && t64)  // fp32 warm-up arithmetic straight from the fp64 T
        k_lik<FAM, double2, true><<<tiles, FT, 0, c.stream>>>(st, segs, K, static_cast<const double2*>(T), part,
                                                              tick, running, tol, tile_list);
    else if (f32)
        k_lik<FAM, float2><<<tiles, FT, 0, c.stream>>>(st, segs, K, static_cast<const float2*>(T), part, tick,
                                                       running, tol, tile_list);
    else
        k_lik<FAM, double2><<<tiles, FT, 0, c.stream>>>(st, segs, K, static_cast<const double2*>(T), part, tick,
                                                        running, tol, tile_list);
    c.count_launch();
}

// Tiles of the blocks still running (any order: tile_reduce sums a block's
// partials in tile order), so a pass that only a few blocks need does not
// launch, and early-exit, every tile of the family.
__global__ void k_running_tiles(const BlockState* st, const Seg* segs, int nseg, uint32_t* list, unsigned* count) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= nseg || st[m].status != kRunning) return;
    const Seg S = segs[m];
    const uint32_t nt = (S.n + FTILE - 1) / FTILE;
    const uint32_t at = atomicAdd(count, nt);
    for (uint32_t q = 0; q < nt; ++q) list[at + q] = S.tile0 + q;
}

__global__ void k_set_start(BlockState* st, int nseg, const double* theta0) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < nseg && st[m].status == kRunning) st[m].theta = theta0[m];
}

double inv_tau_host(int fam, double tau);  // below

void tau_start(Ctx& c, int fam, const FitIO& io, BlockState* st, int K) {
    auto* d_tau = c.ws.get_t<double>("init.tau", K);
    run_kendall(c, io.x1, io.x2, io.off, 5000u, d_tau);
    std::vector<double> h(K);
    PCB_CUDA(cudaMemcpyAsync(h.data(), d_tau, K * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    PCB_CUDA(cudaStreamSynchronize(c.stream));
    for (int m = 0; m < K; ++m) h[m] = inv_tau_host(fam, h[m]);
    PCB_CUDA(cudaMemcpyAsync(d_tau, h.data(), K * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    k_set_start<<<(K + 127) / 128, 128, 0, c.stream>>>(st, K, d_tau);
    c.count_launch();
}

// inverse_tau clipped into the family's start region the way the oracle's
// driver does (oracle/mpl_driver.hpp fit init)
double inv_tau_host(int fam, double tau) {
    tau = std::min(std::max(tau, -0.999), 0.999);
    if (fam == kGumbel) return tau <= 0.0 ? 1.0 : 1.0 / (1.0 - tau);
    const double at = std::fabs(tau);
    if (at < 1e-7) return tau < 0 ? -1e-6 : 1e-6;
    auto tau_of = [](double th) { return 1.0 - 4.0 / th * (1.0 - debye(1, th)); };
    double lo = 1e-6, hi = 1.0;
    while (tau_of(hi) < at && hi < 1e6) hi *= 2.0;
    for (int it = 0; it < 200 && hi - lo > 1e-10 * hi; ++it) {
        const double mid = 0.5 * (lo + hi);
        (tau_of(mid) < at ? lo : hi) = mid;
    }
    const double th = 0.5 * (lo + hi);
    return tau < 0 ? -th : th;
}

std::vector<Seg> make_segs(const std::vector<uint64_t>& off, uint32_t& tiles) {
    const size_t K = off.size() - 1;
    std::vector<Seg> segs(K);
    tiles = 0;
    for (size_t m = 0; m < K; ++m) {
        segs[m] = Seg{off[m], static_cast<uint32_t>(off[m + 1] - off[m]), tiles};
        tiles += ftiles(off[m + 1] - off[m]);
    }
    return segs;
}

}  // namespace

void init_tables() {
    build_tables();
    PCB_CUDA(cudaMemcpyToSymbol(c_frank_rho, h_frank_rho, sizeof h_frank_rho));
    PCB_CUDA(cudaMemcpyToSymbol(c_frank_theta, h_frank_theta, sizeof h_frank_theta));
    PCB_CUDA(cudaMemcpyToSymbol(c_gumbel_rho, h_gumbel_rho, sizeof h_gumbel_rho));
    PCB_CUDA(cudaMemcpyToSymbol(c_gumbel_theta, h_gumbel_theta, sizeof h_gumbel_theta));
}

void run_fit(Ctx& c, const FitIO& io, void* d_out) {
    const int K = static_cast<int>(io.off.size() - 1);
    if (K <= 0) return;
    cudaStream_t s = c.stream;
    uint32_t tiles = 0;
    std::vector<Seg> segs = make_segs(io.off, tiles);
    auto* d_segs = c.ws.get_t<Seg>("fit.segs", K);
    auto* st = c.ws.get_t<BlockState>("fit.state", K);
    auto* part = c.ws.get_t<double>("fit.partials", static_cast<size_t>(tiles) * 4 + 4);
    auto* tick = c.ws.get_t<unsigned>("fit.tickets", K);
    auto* running = c.ws.get_t<unsigned>("fit.running", 1);
    auto* h_running = static_cast<unsigned*>(c.host_staging(2 * sizeof(unsigned)));  // [1]: tile count
    PCB_CUDA(cudaMemcpyAsync(d_segs, segs.data(), K * sizeof(Seg), cudaMemcpyHostToDevice, s));
    PCB_CUDA(cudaMemsetAsync(tick, 0, K * sizeof(unsigned), s));
    PCB_CUDA(cudaMemsetAsync(running, 0, sizeof(unsigned), s));
    cudaEvent_t* ev = c.ev;
    PCB_CUDA(cudaEventRecord(ev[1], s));
    k_init_state<<<(K + 127) / 128, 128, 0, s>>>(st, d_segs, K, io.bad, running, io.theta_in);
    c.count_launch();
    const int fam = io.family;
    // T: fp32 only for the Archimedean fp32 likelihood path; the Gaussian
    // (x, y) pair is always fp64 (it only feeds the variance pass).
    const bool fp32T = io.precision == 1 && fam != kGaussian;
    // fp64 mode: fp32 warm-up passes from a float copy of T, then fp64 passes
    // decide convergence (the answer is the fp64 score root either way)
    const bool warm = io.precision == 0 && fam != kGaussian && io.do_fit && !getenv_flag("PCB_NO_WARM32");
    // Gaussian scores by rank table (rank-derived u only; few distinct block sizes)
    const double* gtab = nullptr;
    const uint64_t* goff = nullptr;
    if ((fam == kGaussian || fam == kGumbel) && !io.u1 && !getenv_flag("PCB_NO_GTAB")) {
        std::vector<uint32_t> sizes;
        for (int m = 0; m < K; ++m)
            if (std::find(sizes.begin(), sizes.end(), segs[m].n) == sizes.end()) sizes.push_back(segs[m].n);
        if (sizes.size() <= 16) {
            std::vector<uint64_t> base(sizes.size());
            uint64_t tot = 0;
            for (size_t q = 0; q < sizes.size(); ++q) {
                base[q] = tot;
                tot += 2ull * sizes[q] + 1;
            }
            auto* tab = c.ws.get_t<double>("fit.gtab", 4 * tot);  // 4 doubles per entry
            std::vector<uint64_t> hoff(K);
            for (int m = 0; m < K; ++m)
                hoff[m] = base[std::find(sizes.begin(), sizes.end(), segs[m].n) - sizes.begin()];
            auto* d_off = c.ws.get_t<uint64_t>("fit.goff", K);
            PCB_CUDA(cudaMemcpyAsync(d_off, hoff.data(), K * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
            for (size_t q = 0; q < sizes.size(); ++q) {
                const uint32_t nn = sizes[q];
                k_rank_table<<<std::min<uint32_t>(148u * 8u, (2 * nn + 256) / 256), 256, 0, s>>>(tab + 4 * base[q], nn,
                                                                                                   fam);
                c.count_launch();
            }
            gtab = tab;
            goff = d_off;
        }
    }
    // Gaussian with rank tables: the variance pass either gathers the tables
    // again (two random 32-byte entries per point) or streams the (x, y)
    // pairs the prepare pass writes and recomputes exp(x^2/2) -- the same
    // arithmetic as the table entry, so bitwise the same result
    // (PCB_GAUSS_T=0/1 forces either way).
    const char* gtv = std::getenv("PCB_GAUSS_T");
    const bool gauss_t = fam == kGaussian && gtab && (gtv && gtv[0] ? gtv[0] != '0' : kGaussT);
    void* T = (gtab && fam == kGaussian && !gauss_t)
                  ? nullptr
                  : c.ws.get("fit.T", io.n_rows * (fp32T ? sizeof(float2) : sizeof(double2)));
    // T32 (warm-up passes only) and the variance score zb share one 8-byte-per-row buffer.
    // Gumbel's warm-up passes read the fp64 T directly (no T32: measured faster
    // overall); PCB_WARM_FROM_T=0/1 forces either way for both families
    const char* wft = std::getenv("PCB_WARM_FROM_T");
    const bool warm_t64 = warm && !fp32T && (wft && wft[0] ? wft[0] != '0' : fam == kGumbel);
    float2* T32 = (warm && !warm_t64) ? c.ws.get_t<float2>("scratch.row8", io.n_rows) : nullptr;
    if (tiles > 0) {
        const int with_fit = io.do_fit ? 1 : 0;
        if (fam == kGaussian)
            launch_prepare<kGaussian>(c, tiles, st, d_segs, K, io, T, fp32T, T32, gtab, goff, part, tick, running, with_fit);
        else if (fam == kFrank)
            launch_prepare<kFrank>(c, tiles, st, d_segs, K, io, T, fp32T, T32, gtab, goff, part, tick, running, with_fit);
        else
            launch_prepare<kGumbel>(c, tiles, st, d_segs, K, io, T, fp32T, T32, gtab, goff, part, tick, running, with_fit);
    }
    // PCB_INIT=tau: the SPEC's own start, inverse_tau of the empirical Kendall
    // tau of each block's first min(n_m, 5000) rows, in place of
    // the Spearman-rho start; theta-hat is the same root either way
    const char* init = std::getenv("PCB_INIT");
    if (init && std::string(init) == "tau" && io.do_fit && fam != kGaussian && io.x1 && tiles > 0)
        tau_start(c, fam, io, st, K);
    PCB_CUDA(cudaEventRecord(ev[2], s));
    float lik_ms = 0.0f, warm_ms = 0.0f;
    int lik_launches = 0, warm_launches = 0;
    if (io.do_fit && fam != kGaussian && tiles > 0) {
        for (int pass = 0; pass < kMaxPasses; ++pass) {
            const bool wp = warm && pass < kWarmPasses;
            const bool f32 = wp || fp32T;
            const void* Tp = (wp && !warm_t64) ? static_cast<const void*>(T32) : T;
            const double tol = wp ? -1.0 : (fp32T ? kTol32 : kTol64);
            const bool t64 = wp && warm_t64;
            uint32_t grid = tiles;
            const uint32_t* tl = nullptr;
            if (pass > 0 && *h_running * 8u <= static_cast<unsigned>(K)) {  // few blocks left: their tiles only
                auto* list = c.ws.get_t<uint32_t>("fit.tile_list", tiles);
                auto* cnt = c.ws.get_t<unsigned>("fit.tile_count", 1);
                PCB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned), s));
                k_running_tiles<<<(K + 127) / 128, 128, 0, s>>>(st, d_segs, K, list, cnt);
                c.count_launch();
                unsigned* h_cnt = h_running + 1;
                PCB_CUDA(cudaMemcpyAsync(h_cnt, cnt, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
                PCB_CUDA(cudaStreamSynchronize(s));
                grid = *h_cnt;
                tl = list;
                if (grid == 0) break;
            }
            PCB_CUDA(cudaEventRecord(ev[6], s));
            if (fam == kFrank) launch_lik<kFrank>(c, grid, st, d_segs, K, f32, Tp, part, tick, running, tol, t64, tl);
            else launch_lik<kGumbel>(c, grid, st, d_segs, K, f32, Tp, part, tick, running, tol, t64, tl);
            PCB_CUDA(cudaEventRecord(ev[7], s));
            PCB_CUDA(cudaMemcpyAsync(h_running, running, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
            PCB_CUDA(cudaStreamSynchronize(s));
            float ms = 0.0f;
            PCB_CUDA(cudaEventElapsedTime(&ms, ev[6], ev[7]));
            if (wp) {
                warm_ms += ms;
                ++warm_launches;
            } else {
                lik_ms += ms;
                ++lik_launches;
            }
            if (*h_running == 0) break;
        }
    }
    PCB_CUDA(cudaEventRecord(ev[3], s));
    c.stage_ms[5] = lik_ms;
    c.stage_ms[6] = lik_launches;
    c.stage_ms[7] = warm_ms;
    c.stage_ms[8] = warm_launches;
    if (io.do_variance && tiles > 0) {
        VarIO v;
        v.family = fam;
        v.n_rows = io.n_rows;
        v.off = &io.off;
        v.segs = d_segs;
        v.h_segs = &segs;
        v.tiles = tiles;
        v.st = st;
        v.rp = io.rp;
        v.rank = io.rank;
        v.u1 = io.u1;
        v.u2 = io.u2;
        // Gaussian: the rank table (x, exp(x^2/2)) replaces T; Gumbel re-reads
        // T (coalesced) rather than gathering 32-byte table entries at random
        v.gtab = (fam == kGaussian && !gauss_t) ? gtab : nullptr;
        // Frank's fp64 T is (u, v) itself; Gumbel's is (ln(-ln u), ln(-ln v))
        v.T64 = (!v.gtab && (fam == kGaussian || !fp32T)) ? static_cast<const double2*>(T) : nullptr;
        v.goff = goff;
        v.partials = part;
        v.tickets = tick;
        run_variance(c, v);
    }
    PCB_CUDA(cudaEventRecord(ev[4], s));
    k_finalize<<<(K + 127) / 128, 128, 0, s>>>(st, K, static_cast<RecordOut*>(d_out), io.do_variance ? 1 : 0);
    c.count_launch();
    PCB_CUDA(cudaEventRecord(ev[5], s));
}

void run_loglik(Ctx& c, int family, const double* d_theta, const double* u1, const double* u2,
                const std::vector<uint64_t>& off, double* d_out) {
    const int K = static_cast<int>(off.size() - 1);
    uint32_t tiles = 0;
    std::vector<Seg> segs = make_segs(off, tiles);
    auto* d_segs = c.ws.get_t<Seg>("fit.segs", K);
    auto* part = c.ws.get_t<double>("fit.partials", static_cast<size_t>(tiles) * 4 + 4);
    auto* tick = c.ws.get_t<unsigned>("fit.tickets", K);
    PCB_CUDA(cudaMemcpyAsync(d_segs, segs.data(), K * sizeof(Seg), cudaMemcpyHostToDevice, c.stream));
    PCB_CUDA(cudaMemsetAsync(tick, 0, K * sizeof(unsigned), c.stream));
    PCB_CUDA(cudaMemsetAsync(d_out, 0, K * sizeof(double), c.stream));
    if (tiles == 0) return;
    k_loglik<<<tiles, FT, 0, c.stream>>>(d_segs, K, d_theta, u1, u2, family, part, tick, d_out);
    c.count_launch();
}

}  // namespace pcb

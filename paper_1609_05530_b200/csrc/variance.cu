// K3-K5 asymptotic variance on sm_100a.
//
//   sigma2 = M/I^2/n,  I = -(1/n) sum hess_i,
//   M = (1/n) sum (score_i + W1_i + W2_i)^2,
//   W_ji = (1/n) sum_h [1(u_ij <= u_hj) - u_hj] cross_j(u_h)
//        = (1/n) (T_j(first position of i's tie run) - C_j),
//   C_j = sum_h u_hj cross_j(u_h),  T_j(p) = sum of cross_j over sorted positions >= p.
// Pseudo-observations are ranks, so the sort is already done: the rank
// stage's stable position scatters cross_j into sorted order, its run-start
// bit marks where each tie run begins, and one suffix scan gives every W.
//
// Pass 1 (k_var_point, grid of tiles, FP64-bound): per-point log c, score,
//   Hessian, cross_1, cross_2 at theta-hat in point order (coalesced), and the
//   block sums I, C_1, C_2, loglik. cross_j leaves along the route the rank
//   stage's all-to-all took (owner CTA, receive slot): a warp's 32 consecutive
//   rows land in a few short runs of slots, so the scatter is semi-coalesced.
// Pass 2 (k_var_scan, one CTA per (column, block, owner) of the rank stage,
//   independent of each other): load the owner's slots (coalesced), place
//   them at their owner-local sorted positions in shared memory, suffix-scan
//   locally, write the local suffix sum at each slot's tie-run start back per
//   slot (coalesced) and the owner's total. Tie runs never straddle owners.
//   k_var_carry turns the totals into each owner's carry (mass above it).
// Pass 3 (k_var_final, grid of tiles): W_j = (local + carry - C_j)/n and
//   z = score + W_1 + W_2 per row through the route, sum z^2 -> M-hat -> sigma2.
// Blocks the rank stage did not route (global-path ranks, constant columns)
// take the same steps through sorted-order arrays in global memory.
// Deterministic: positions are unique, scans and sums run in fixed order.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "devmath.cuh"
#include "internal.hpp"

namespace pcb {
namespace {

namespace cg = cooperative_groups;


// Per-theta constants, built once per CTA (they cost more than a point).
template <int FAM>
struct ThetaOf;
template <>
struct ThetaOf<kGaussian> {
    using type = GaussTheta;
};
template <>
struct ThetaOf<kFrank> {
    using type = FrankTheta;
};
template <>
struct ThetaOf<kGumbel> {
    using type = GumbelTheta;
};

// Where a point's theta-independent transforms come from
//   kFromTU: T carries u too (Frank: T = (u, v) exactly; Gumbel: T = (ln x,
//   ln y) and u = exp(-x), within an ulp or two), so no rank gathers
enum { kFromU = 0, kFromT64 = 1, kFromTable = 2, kFromTU = 3 };

template <int FAM, int MODE>
__device__ __forceinline__ PointFull eval_point(const typename ThetaOf<FAM>::type& th, double u, double w,
                                                const double2& t64, const double2 (&ta)[2], const double2 (&tb)[2]) {
    if constexpr (FAM == kGaussian) {
        if constexpr (MODE == kFromTable) return gauss_full_e(ta[0].x, tb[0].x, ta[0].y, tb[0].y, th);
        else if constexpr (MODE == kFromT64) return gauss_full(t64.x, t64.y, th);
        else return gauss_full(dev_phi_inv(u), dev_phi_inv(w), th);
    } else if constexpr (FAM == kFrank) {
        return frank_full(u, w, th);
    } else {
        if constexpr (MODE == kFromTable)
            return gumbel_full_t(ta[0].x, tb[0].x, ta[0].y, tb[0].y, ta[1].x, tb[1].x, ta[1].y, tb[1].y, th);
        else if constexpr (MODE == kFromT64 || MODE == kFromTU) return gumbel_full_l(u, w, t64.x, t64.y, th);
        else return gumbel_full(u, w, th);
    }
}

// The run-start flag of a sorted position rides in the least significant
// mantissa bit of its cross value (a <= 1-ulp change, far below the 1e-9
// parity bar and deterministic), so pass 1 scatters one 8-byte word per
// point and column.
__device__ __forceinline__ double with_flag(double x, bool f) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return __longlong_as_double(static_cast<long long>((b & ~1ull) | (f ? 1ull : 0ull)));
}
__device__ __forceinline__ bool flag_of(double x) { return (__double_as_longlong(x) & 1ll) != 0; }

// ------------------------------------------------------------ pass 1
// MODE: where the theta-independent transforms come from (only that path is
// compiled in). With the rank table a Gaussian point needs no transcendental
// and a Gumbel point four.
// resident CTAs per SM the register budget is sized for (0 = compiler's
// choice). Measured at C5: Gumbel 3 (80 regs, -3 ms); forcing Gaussian or
// Frank below the compiler's allocation spills and loses.
#ifndef PCB_VOCC_G
#define PCB_VOCC_G 0
#endif
#ifndef PCB_VOCC_F
#define PCB_VOCC_F 0
#endif
#ifndef PCB_VOCC_U
#define PCB_VOCC_U 3
#endif
template <int FAM>
struct VarOcc {
    static constexpr int value = FAM == kGaussian ? PCB_VOCC_G : (FAM == kFrank ? PCB_VOCC_F : PCB_VOCC_U);
};

template <int FAM, int MODE>
__global__ void __launch_bounds__(FT, VarOcc<FAM>::value) k_var_point(BlockState* st, const Seg* segs, int nseg, RankRef R,
                                                 const double* __restrict__ u1, const double* __restrict__ u2,
                                                 const double2* __restrict__ T64, const double* __restrict__ gtab,
                                                 const uint64_t* goff, uint64_t n_rows, double* __restrict__ zb,
                                                 double* __restrict__ Ag, double* __restrict__ xr, double* partials,
                                                 unsigned* tickets) {
    const uint32_t tile = blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (st[m].status != kConverged) return;
    const typename ThetaOf<FAM>::type th(st[m].theta);
    const double scale = 1.0 / (static_cast<double>(S.n) + 1.0);
    const uint32_t base = (tile - S.tile0) * FTILE;
    const double2* gt = MODE == kFromTable ? reinterpret_cast<const double2*>(gtab + 4 * goff[m]) : nullptr;
    const bool rt = R.routed && R.routed[m];
    const uint64_t c1 = rt ? slot_index(R, nseg, 0, m, 0u) : 0, c2 = rt ? slot_index(R, nseg, 1, m, 0u) : 0;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
#ifndef PCB_U_VPG
#define PCB_U_VPG 4
#endif
#ifndef PCB_U_VP
#define PCB_U_VP 2
#endif
#ifndef PCB_U_VPU
#define PCB_U_VPU 1
#endif
    // points in flight per thread (measured at C5: Gaussian 4, Frank 2, Gumbel 1)
    constexpr int U = (FAM == kGaussian && MODE == kFromTable) ? PCB_U_VPG : (FAM == kGumbel ? PCB_U_VPU : PCB_U_VP);
    for (int k0 = 0; k0 < PPT; k0 += U) {
        unsigned long long p1[U], p2[U];  // packed ranks (by-row blocks)
        uint32_t w1[U], w2[U];            // route words (routed blocks)
        uint32_t q1[U], q2[U];            // r2
        double2 tt[U];
        double2 ta[U][2], tb[U][2];  // rank-table entries of the two columns
        double uu[U], ww[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + tile_row(k0 + j);
            if (i < S.n) {
                const uint64_t row = S.begin + i;
                if (rt) {
                    w1[j] = R.route[row];
                    w2[j] = R.route[n_rows + row];
                } else {
                    p1[j] = R.rp[row];
                    p2[j] = R.rp[n_rows + row];
                }
                if (u1) {
                    uu[j] = u1[row];
                    ww[j] = u2[row];
                }
                if (MODE == kFromT64 || MODE == kFromTU) tt[j] = T64[row];
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + tile_row(k0 + j);
            if (i >= S.n) continue;
            if (!rt) {
                q1[j] = rank_r2(p1[j]);
                q2[j] = rank_r2(p2[j]);
            } else if (!u1 && MODE != kFromTU) {
                q1[j] = R.r2s[c1 + (w1[j] >> 16) * R.rcap + (w1[j] & 0xffffu)];
                q2[j] = R.r2s[c2 + (w2[j] >> 16) * R.rcap + (w2[j] & 0xffffu)];
            }
        }
        if constexpr (MODE == kFromTable) {
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const uint32_t i = base + tile_row(k0 + j);
                if (i >= S.n) continue;
                ta[j][0] = gt[2 * q1[j]];
                tb[j][0] = gt[2 * q2[j]];
                if (FAM == kGumbel) {
                    ta[j][1] = gt[2 * q1[j] + 1];
                    tb[j][1] = gt[2 * q2[j] + 1];
                }
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + tile_row(k0 + j);
            if (i >= S.n) continue;
            const uint64_t row = S.begin + i;
            double u, w;
            if constexpr (MODE == kFromTU) {
                if constexpr (FAM == kFrank) {
                    u = tt[j].x;
                    w = tt[j].y;
                } else {
                    u = exp(-exp(tt[j].x));
                    w = exp(-exp(tt[j].y));
                }
            } else {
                u = u1 ? uu[j] : __dmul_rn(0.5 * static_cast<double>(q1[j]), scale);
                w = u1 ? ww[j] : __dmul_rn(0.5 * static_cast<double>(q2[j]), scale);
                u = clamp_unit(u);
                w = clamp_unit(w);
            }
            const PointFull p = eval_point<FAM, MODE>(th, u, w, tt[j], ta[j], tb[j]);
            zb[row] = p.score;
            if (rt) {  // cross_j to (owner, slot) of the rank stage's route
                xr[c1 + (w1[j] >> 16) * R.rcap + (w1[j] & 0xffffu)] = p.cross1;
                xr[c2 + (w2[j] >> 16) * R.rcap + (w2[j] & 0xffffu)] = p.cross2;
            } else {  // cross_j to its sorted position, run-start flag beside it
                const uint64_t q1 = S.begin + rank_pos(p1[j]), q2 = n_rows + S.begin + rank_pos(p2[j]);
                Ag[q1] = with_flag(p.cross1, rank_first(p1[j]));
                Ag[q2] = with_flag(p.cross2, rank_first(p2[j]));
            }
            v[0] += p.hess;
            v[1] += u * p.cross1;
            v[2] += w * p.cross2;
            v[3] += clip_log(p.logc);
        }
    }
    __shared__ double sh[(FT / 32) * 4];
    if (!tile_reduce<4>(v, sh, partials, tickets, S, m, tile)) return;
    if (threadIdx.x == 0) {
        st[m].info_sum = v[0];
        st[m].c1 = v[1];
        st[m].c2 = v[2];
        st[m].loglik = v[3];
    }
}

__device__ __forceinline__ double finish_sigma2(BlockState& s, double zz, double nd) {
    const double info = -s.info_sum / nd;
    if (!(info > 0.0)) {
        s.status = kInfoNonPos;
        return NAN;
    }
    return (zz / nd) / (info * info) / nd;
}

// ------------------------------------------------------------ pass 2 (routed)
// One CTA per (column, block, owner) region, independent of the others: the
// owner's slots are placed at their owner-local sorted positions in shared
// memory, suffix-scanned locally, and L = local suffix sum at the slot's
// tie-run start is written back per slot; the owner's total goes to `tot`.
// The higher owners' mass (carry) is added in pass 3, so no CTA waits on
// another.
//   place: thread t loads slots t + k*ST (all its loads in flight; RCAP <=
//          SJ*ST), stores each at its position, sets run-start bits
//   scan:  thread t owns PT (odd: few bank conflicts) consecutive positions:
//          thread sum -> block suffix of thread sums -> thread-serial suffix
//   write: per slot, the suffix sum at its run start (bitmap search, local)
#ifndef PCB_SCAN_T
#define PCB_SCAN_T 1024
#endif
#ifndef PCB_SCAN_B
#define PCB_SCAN_B 8
#endif
constexpr int ST = PCB_SCAN_T;     // threads per scan CTA
constexpr int SJ = 16384 / ST;     // slots per thread (RCAP <= 16384)
constexpr int SB = PCB_SCAN_B < SJ ? PCB_SCAN_B : SJ;  // slot loads in flight per thread
constexpr int SW = ST / 32;

__global__ void __launch_bounds__(ST, 1) k_var_scan(const BlockState* st, const int* seg_list, int nseg,
                                                   const uint16_t* __restrict__ posl,
                                                   const uint32_t* __restrict__ ocnt, double* __restrict__ xr,
                                                   double* __restrict__ tot, int CL, uint32_t RCAP,
                                                   unsigned long long* prof, uint32_t pf) {
    long long t_prev = clock64();
    auto mark = [&](int k) {  // optional phase timing (PCB_VAR_PROFILE)
        if (prof && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(prof + k, static_cast<unsigned long long>(t - t_prev));
            t_prev = t;
        }
    };
    const int njobs = gridDim.x / (2 * CL);
    const int col = blockIdx.x / (njobs * CL);
    const int rem = blockIdx.x - col * njobs * CL;
    const int m = seg_list[rem / CL];
    const int r = rem % CL;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    extern __shared__ __align__(16) unsigned char smem[];
    double* A = reinterpret_cast<double*>(smem);             // owner-local sorted positions
    uint32_t* bits = reinterpret_cast<uint32_t*>(A + RCAP);  // run-start bit per position
    __shared__ double s_ws[SW], s_wo[SW];

    const uint64_t rid = (static_cast<uint64_t>(col) * nseg + m) * CL + r;
    const uint64_t reg = rid * RCAP;
    double* X = xr + reg;
    const uint16_t* P = posl + reg;
    // the first loads go out before the block's status and count arrive (the
    // region is RCAP slots long, so reading past the count is in bounds)
    double x0[SB];
    uint32_t pv0[SB];
#pragma unroll
    for (int k = 0; k < SB; ++k) {
        const uint32_t j = tid + k * ST;
        if (j < RCAP) {
            pv0[k] = P[j];
            x0[k] = X[j];
        }
    }
    // the CTA pf positions ahead runs on the next wave (one CTA per SM): pull
    // its slots into L2 while this CTA's scan keeps HBM otherwise idle
    if (tid == 32 && pf && blockIdx.x + pf < gridDim.x) {
        const uint32_t b2 = blockIdx.x + pf;
        const int col2 = static_cast<int>(b2 / (njobs * CL));
        const int rem2 = static_cast<int>(b2 - col2 * njobs * CL);
        const uint64_t rid2 = (static_cast<uint64_t>(col2) * nseg + seg_list[rem2 / CL]) * CL + rem2 % CL;
        const uint32_t T2 = ocnt[rid2];
        if (T2) {
            const uint64_t xlo = reinterpret_cast<uint64_t>(xr + rid2 * RCAP) & ~15ull;
            const uint64_t xhi = (reinterpret_cast<uint64_t>(xr + rid2 * RCAP + T2) + 15ull) & ~15ull;
            const uint64_t plo = reinterpret_cast<uint64_t>(posl + rid2 * RCAP) & ~15ull;
            const uint64_t phi = (reinterpret_cast<uint64_t>(posl + rid2 * RCAP + T2) + 15ull) & ~15ull;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(xlo), "r"(static_cast<uint32_t>(xhi - xlo))
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(plo), "r"(static_cast<uint32_t>(phi - plo))
                         : "memory");
        }
    }
    if (st[m].status != kConverged) return;
    const uint32_t T = ocnt[rid];
    for (uint32_t q = tid; q <= T / 32; q += ST) bits[q] = 0u;
    __syncthreads();
    mark(0);
    uint32_t pk[SJ / 2];  // this thread's local positions (| run-start bit), two per register
#pragma unroll
    for (int h = 0; h < SJ; h += SB) {
        if (tid + h * ST >= T) {
#pragma unroll
            for (int k = 0; k < SB / 2; ++k) pk[(h >> 1) + k] = 0xffffffffu;
            continue;
        }
        double x[SB];
        uint32_t pv[SB];
#pragma unroll
        for (int k = 0; k < SB; ++k) {
            const uint32_t j = tid + (h + k) * ST;
            if (h == 0) {
                pv[k] = j < T ? pv0[k] : 0xffffu;
                x[k] = x0[k];
            } else {
                pv[k] = j < T ? P[j] : 0xffffu;
                x[k] = j < T ? X[j] : 0.0;
            }
        }
#pragma unroll
        for (int k = 0; k < SB; ++k) {
            if (pv[k] != 0xffffu) {
                const uint32_t p = pv[k] & 0x7fffu;
                A[p] = x[k];
                if (pv[k] & 0x8000u) atomicOr(bits + (p >> 5), 1u << (p & 31));
            }
            if (k & 1) pk[(h + k) >> 1] = pv[k - 1] | (pv[k] << 16);
        }
    }
    __syncthreads();
    mark(1);
    // thread-contiguous suffix scan
    const uint32_t PT = ((T + ST - 1) / ST) | 1u;
    const uint32_t p0 = min(T, tid * PT), p1 = min(T, p0 + PT);
    double ts = 0.0;
    for (uint32_t q = p0; q < p1; ++q) ts += A[q];
    double x = ts;  // inclusive suffix over the warp's threads (lanes above)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_down_sync(0xffffffffu, x, o);
        if (lane + o < 32) x += y;
    }
    if (lane == 0) s_ws[wid] = x;
    __syncthreads();
    if (wid == 0) {  // exclusive suffix of the warp totals; owner total
        double w = lane < SW ? s_ws[lane] : 0.0;
        const double w0 = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_down_sync(0xffffffffu, w, o);
            if (lane + o < 32) w += y;
        }
        if (lane < SW) s_wo[lane] = w - w0;
        if (lane == 0) tot[rid] = w;
    }
    __syncthreads();
    double acc = s_wo[wid] + (x - ts);  // mass above this thread's positions
    for (uint32_t q = p1; q-- > p0;) {
        acc += A[q];
        A[q] = acc;
    }
    __syncthreads();
    mark(2);
    // L per slot: local suffix sum at the start of the slot's tie run
#pragma unroll
    for (int k = 0; k < SJ; ++k) {
        const uint32_t j = tid + k * ST;
        if (j >= T) break;
        const uint32_t pv = (pk[k >> 1] >> ((k & 1) * 16)) & 0xffffu;
        uint32_t q = pv & 0x7fffu;
        if (!(pv & 0x8000u)) {
            uint32_t t = q - 1;  // position 0 of an owner always starts a run
            for (;;) {
                const uint32_t w = bits[t >> 5] & (0xffffffffu >> (31 - (t & 31)));
                if (w) {
                    q = (t & ~31u) + (31 - __clz(w));
                    break;
                }
                t = (t & ~31u) - 1;
            }
        }
        X[j] = A[q];
    }
    mark(3);
}

// carry[col][m][d] = mass of the owners above d (fixed order)
__global__ void k_var_carry(const int* seg_list, int njobs, int nseg, int CL, const double* tot, double* carry) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= 2 * njobs) return;
    const int col = q / njobs, m = seg_list[q % njobs];
    const uint64_t b = (static_cast<uint64_t>(col) * nseg + m) * CL;
    double c = 0.0;
    for (int d = CL - 1; d >= 0; --d) {
        carry[b + d] = c;
        c += tot[b + d];
    }
}

// z = score + W_1 + W_2 per row (through the route), sum z^2 -> sigma2
#ifndef PCB_FINAL_OCC
#define PCB_FINAL_OCC 0
#endif
__global__ void __launch_bounds__(FT, PCB_FINAL_OCC) k_var_final(BlockState* st, const Seg* segs, int nseg, RankRef R,
                                                 uint64_t n_rows, const double* __restrict__ zb,
                                                 const double* __restrict__ xr, const double* __restrict__ carry,
                                                 double* partials, unsigned* tickets) {
    const uint32_t tile = blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (!R.routed[m] || st[m].status != kConverged) return;
    const uint32_t RCAP = R.rcap;
    const uint32_t* route = R.route;
    const double* x1 = xr + slot_index(R, nseg, 0, m, 0u);
    const double* x2 = xr + slot_index(R, nseg, 1, m, 0u);
    const double* k1 = carry + static_cast<uint64_t>(m) * R.cl;
    const double* k2 = carry + (static_cast<uint64_t>(nseg) + m) * R.cl;
    const double cj1 = st[m].c1, cj2 = st[m].c2;
    const double inv_n = 1.0 / static_cast<double>(S.n);
    const uint32_t base = (tile - S.tile0) * FTILE;
    double v[1] = {0.0};
#ifndef PCB_U_FINAL
#define PCB_U_FINAL 2
#endif
    constexpr int U = PCB_U_FINAL;
    for (int k0 = 0; k0 < PPT; k0 += U) {
        uint32_t r1[U], r2[U];
        double zz[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + tile_row(k0 + j);
            if (i < S.n) {
                const uint64_t row = S.begin + i;
                r1[j] = route[row];
                r2[j] = route[n_rows + row];
                zz[j] = zb[row];
            }
        }
        double w1[U], w2[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + tile_row(k0 + j);
            if (i < S.n) {
                w1[j] = x1[(r1[j] >> 16) * RCAP + (r1[j] & 0xffffu)] + k1[r1[j] >> 16];
                w2[j] = x2[(r2[j] >> 16) * RCAP + (r2[j] & 0xffffu)] + k2[r2[j] >> 16];
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + tile_row(k0 + j);
            if (i < S.n) {
                double z = zz[j];
                z += (w1[j] - cj1) * inv_n;
                z += (w2[j] - cj2) * inv_n;
                v[0] += z * z;
            }
        }
    }
    __shared__ double sh[FT / 32];
    if (!tile_reduce<1>(v, sh, partials, tickets, S, m, tile)) return;
    if (threadIdx.x == 0) {
        BlockState s = st[m];
        s.sigma2 = finish_sigma2(s, v[0], static_cast<double>(S.n));
        st[m] = s;
    }
}

// ------------------------------------------------------------ pass 2 (global)
// Same steps through HBM for blocks larger than a cluster holds: pass 1 has
// already placed cross_j in sorted order; suffix-scan it, then gather.
// Tile-parallel segmented suffix scan (deterministic): tile sums, a
// per-(block, column) suffix over its tiles, then each tile's own scan.
__global__ void __launch_bounds__(FT) k_tsum_g(const BlockState* st, const Seg* segs, int nseg, const uint8_t* use,
                                              uint64_t n_rows, const double* A, double* tsum, uint32_t ntiles) {
    const uint32_t tile = blockIdx.x, col = blockIdx.y;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (!use[m] || st[m].status != kConverged) return;
    const uint32_t base = (tile - S.tile0) * FTILE, cnt = min(FTILE, S.n - base);
    const double* a = A + static_cast<uint64_t>(col) * n_rows + S.begin + base;
    double v[1] = {0.0};
    for (uint32_t q = threadIdx.x; q < cnt; q += FT) v[0] += a[q];
    __shared__ double sh[FT / 32];
    block_sum<1>(v, sh);
    if (threadIdx.x == 0) tsum[col * ntiles + tile] = v[0];
}

__global__ void k_tscan_g(const BlockState* st, const Seg* segs, int nseg, const uint8_t* use, const double* tsum,
                          double* toff, uint32_t ntiles) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= 2 * nseg) return;
    const int seg = m % nseg, col = m / nseg;
    if (!use[seg] || st[seg].status != kConverged) return;
    const Seg S = segs[seg];
    const uint32_t nt = (S.n + FTILE - 1) / FTILE;
    double run = 0.0;  // mass of the tiles above
    for (uint32_t q = nt; q-- > 0;) {
        toff[col * ntiles + S.tile0 + q] = run;
        run += tsum[col * ntiles + S.tile0 + q];
    }
}

__global__ void __launch_bounds__(FT) k_tapply_g(const BlockState* st, const Seg* segs, int nseg, const uint8_t* use,
                                                uint64_t n_rows, double* A, const double* toff, uint32_t ntiles) {
    const uint32_t tile = blockIdx.x, col = blockIdx.y;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (!use[m] || st[m].status != kConverged) return;
    const uint32_t base = (tile - S.tile0) * FTILE, cnt = min(FTILE, S.n - base);
    double* a = A + static_cast<uint64_t>(col) * n_rows + S.begin + base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr uint32_t WL = FTILE / (FT / 32);  // contiguous elements per warp
    const uint32_t w0 = min(cnt, wid * WL), w1 = min(cnt, w0 + WL);
    double wsum = 0.0;
    for (uint32_t q = w0 + lane; q < w1; q += 32) wsum += a[q];
    wsum = warp_sum(wsum);
    __shared__ double s_wt[FT / 32];
    if (lane == 0) s_wt[wid] = wsum;
    __syncthreads();
    double carry = toff[col * ntiles + tile];
    for (int w = wid + 1; w < FT / 32; ++w) carry += s_wt[w];
    for (uint32_t t = (w1 - w0 + 31) / 32; t-- > 0;) {
        const uint32_t q = w0 + t * 32 + lane;
        const double x0 = q < w1 ? a[q] : 0.0;
        double x = x0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_down_sync(0xffffffffu, x, o);
            if (lane + o < 32) x += y;
        }
        if (q < w1) a[q] = with_flag(carry + x, flag_of(x0));  // the run-start flag stays with its position
        carry += __shfl_sync(0xffffffffu, x, 0);
    }
}

__global__ void __launch_bounds__(FT) k_var_gather_g(BlockState* st, const Seg* segs, int nseg, const uint8_t* use,
                                                    const unsigned long long* rp, uint64_t n_rows, const double* zb,
                                                    const double* A, double* partials, unsigned* tickets) {
    const uint32_t tile = blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (!use[m] || st[m].status != kConverged) return;
    const double nd = static_cast<double>(S.n);
    const double cjs[2] = {st[m].c1, st[m].c2};
    const uint32_t base = (tile - S.tile0) * FTILE;
    double v[1] = {0.0};
    for (int k = 0; k < PPT; ++k) {
        const uint32_t i = base + k * FT + threadIdx.x;
        if (i >= S.n) break;
        const uint64_t row = S.begin + i;
        double z = zb[row];
        for (int col = 0; col < 2; ++col) {
            const unsigned long long p = rp[static_cast<uint64_t>(col) * n_rows + row];
            const uint64_t b0 = static_cast<uint64_t>(col) * n_rows + S.begin;
            uint32_t q = rank_pos(p);
            if (!rank_first(p))
                do {
                    --q;  // position 0 always starts a run
                } while (!flag_of(A[b0 + q]));
            z += (A[b0 + q] - cjs[col]) / nd;
        }
        v[0] += z * z;
    }
    __shared__ double sh[FT / 32];
    if (!tile_reduce<1>(v, sh, partials, tickets, S, m, tile)) return;
    if (threadIdx.x == 0) {
        BlockState s = st[m];
        s.sigma2 = finish_sigma2(s, v[0], nd);
        st[m] = s;
    }
}

template <int FAM>
void launch_var_point(Ctx& c, const VarIO& v, double* zb, double* Ag, double* xr) {
    const int K = static_cast<int>(v.off->size() - 1);
#define PCB_VAR_POINT(MODE)                                                                                   \
    k_var_point<FAM, MODE><<<v.tiles, FT, 0, c.stream>>>(v.st, v.segs, K, v.rank->ref(), v.u1, v.u2, v.T64, v.gtab, \
                                                         v.goff, v.n_rows, zb, Ag, xr, v.partials, v.tickets)
    if (FAM != kFrank && v.gtab) PCB_VAR_POINT(kFromTable);
    else if (FAM != kGaussian && v.T64 && !v.u1 && !std::getenv("PCB_VAR_NO_TU")) PCB_VAR_POINT(kFromTU);
    else if (FAM != kFrank && v.T64) PCB_VAR_POINT(kFromT64);
    else PCB_VAR_POINT(kFromU);
#undef PCB_VAR_POINT
    c.count_launch();
}

void launch_var_scan(Ctx& c, const VarIO& v, const int* seg_list, int njobs, double* xr, double* tot) {
    const RankOut& R = *v.rank;
    const int K = static_cast<int>(v.off->size() - 1);
    const size_t smem = static_cast<size_t>(R.rcap) * 8 + (R.rcap / 32 + 1) * 4;
    PCB_CUDA(cudaFuncSetAttribute(k_var_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    unsigned long long* prof = nullptr;
    const char* pe = std::getenv("PCB_VAR_PROFILE");
    if (pe && pe[0] == '1') {
        prof = c.ws.get_t<unsigned long long>("var.prof", 8);
        PCB_CUDA(cudaMemsetAsync(prof, 0, 8 * sizeof(unsigned long long), c.stream));
    }
    const unsigned grid = 2u * static_cast<unsigned>(njobs) * static_cast<unsigned>(R.cl);
    uint32_t pf = 0;  // L2 prefetch distance in CTAs: one wave of resident CTAs
    if (const char* e = std::getenv("PCB_SCAN_PF")) {
        pf = static_cast<uint32_t>(std::atoi(e));
    } else {
        int per_sm = 0, nsm = 0;
        PCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_var_scan, ST, smem));
        PCB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c.device));
        pf = static_cast<uint32_t>(per_sm * nsm);
    }
    k_var_scan<<<grid, ST, smem, c.stream>>>(v.st, seg_list, K, R.posl, R.ocnt, xr, tot, R.cl, R.rcap, prof, pf);
    c.count_launch();
    if (prof) {
        unsigned long long h[8];
        PCB_CUDA(cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, c.stream));
        PCB_CUDA(cudaStreamSynchronize(c.stream));
        std::fprintf(stderr, "[var profile] CL=%d rcap=%u cycles/CTA (one column): start %.0f  place %.0f  scan %.0f  write %.0f\n",
                     R.cl, R.rcap, h[0] / double(grid), h[1] / double(grid), h[2] / double(grid), h[3] / double(grid));
    }
}

void launch_var_global(Ctx& c, const VarIO& v, const uint8_t* use, double* zb, double* Ag) {
    const int K = static_cast<int>(v.off->size() - 1);
    auto* tsum = c.ws.get_t<double>("var.tsum", 2 * static_cast<size_t>(v.tiles));
    auto* toff = c.ws.get_t<double>("var.toff", 2 * static_cast<size_t>(v.tiles));
    k_tsum_g<<<dim3(v.tiles, 2), FT, 0, c.stream>>>(v.st, v.segs, K, use, v.n_rows, Ag, tsum, v.tiles);
    k_tscan_g<<<(2 * K + 127) / 128, 128, 0, c.stream>>>(v.st, v.segs, K, use, tsum, toff, v.tiles);
    k_tapply_g<<<dim3(v.tiles, 2), FT, 0, c.stream>>>(v.st, v.segs, K, use, v.n_rows, Ag, toff, v.tiles);
    k_var_gather_g<<<v.tiles, FT, 0, c.stream>>>(v.st, v.segs, K, use, v.rp, v.n_rows, zb, Ag, v.partials,
                                                 v.tickets);
    c.count_launch(4);
}

}  // namespace

void run_variance(Ctx& c, const VarIO& v) {
    const std::vector<uint64_t>& off = *v.off;
    const int K = static_cast<int>(off.size() - 1);
    const RankOut& R = *v.rank;
    auto* zb = c.ws.get_t<double>("scratch.row8", v.n_rows);  // T32 is dead by now (fit.cu)
    // routed blocks (both columns ranked by the cluster path) reuse its route;
    // the others go through sorted-order arrays in global memory
    int nrouted = 0;
    for (int m = 0; m < K; ++m) nrouted += R.routed.size() == static_cast<size_t>(K) && R.routed[m];
    double* Ag = nrouted < K ? c.ws.get_t<double>("var.A", 2 * v.n_rows) : nullptr;
    double* xr = nrouted ? c.ws.get_t<double>("var.xr", 2 * static_cast<size_t>(K) * R.cl * R.rcap) : nullptr;
    PCB_CUDA(cudaEventRecord(c.ev[6], c.stream));
    if (v.family == kGaussian) launch_var_point<kGaussian>(c, v, zb, Ag, xr);
    else if (v.family == kFrank) launch_var_point<kFrank>(c, v, zb, Ag, xr);
    else launch_var_point<kGumbel>(c, v, zb, Ag, xr);
    PCB_CUDA(cudaEventRecord(c.ev[7], c.stream));
    if (nrouted) {
        std::vector<int> jobs;
        for (int m = 0; m < K; ++m)
            if (R.routed[m]) jobs.push_back(m);
        int* d_jobs = c.ws.get_t<int>("var.jobs", K);
        PCB_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), jobs.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
        const int nj = static_cast<int>(jobs.size());
        auto* tot = c.ws.get_t<double>("var.tot", 2 * static_cast<size_t>(K) * R.cl);
        auto* carry = c.ws.get_t<double>("var.carry", 2 * static_cast<size_t>(K) * R.cl);
        launch_var_scan(c, v, d_jobs, nj, xr, tot);
        k_var_carry<<<(2 * nj + 127) / 128, 128, 0, c.stream>>>(d_jobs, nj, K, R.cl, tot, carry);
        k_var_final<<<v.tiles, FT, 0, c.stream>>>(v.st, v.segs, K, R.ref(), v.n_rows, zb, xr, carry, v.partials,
                                                  v.tickets);
        c.count_launch(2);
    }
    if (nrouted < K) {
        std::vector<uint8_t> use(K);
        for (int m = 0; m < K; ++m) use[m] = !(R.routed.size() == static_cast<size_t>(K) && R.routed[m]);
        uint8_t* d_use = c.ws.get_t<uint8_t>("var.use", K);
        PCB_CUDA(cudaMemcpyAsync(d_use, use.data(), K, cudaMemcpyHostToDevice, c.stream));
        launch_var_global(c, v, d_use, zb, Ag);
    }
    PCB_CUDA(cudaEventSynchronize(c.ev[7]));
    float ms = 0.0f;
    PCB_CUDA(cudaEventElapsedTime(&ms, c.ev[6], c.ev[7]));
    c.stage_ms[9] = ms;  // variance pass 1 (per-point terms); the rest of [3] is passes 2-3
}

}  // namespace pcb

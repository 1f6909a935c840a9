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
//   block sums I, C_1, C_2, loglik.
// Pass 2 (k_var_w, one thread-block cluster per block): column by column,
//   cross_j is scattered to its sorted position in the cluster's distributed
//   shared memory together with a run-start bitmap, suffix-scanned in place,
//   and gathered back at each point's run start; M-hat and sigma2 follow.
//   HBM sees only the per-point arrays; the permutation traffic is DSMEM.
// Blocks too large for one cluster take the same steps through global memory.
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

constexpr int VT = 1024;  // threads per cluster CTA
constexpr int VNW = VT / 32;
constexpr int kMaxCl = 16;
constexpr size_t kVarSmem = 227 * 1024 - 4096;  // static shared memory lives beside it

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

template <int FAM>
__device__ __forceinline__ PointFull eval_point(const typename ThetaOf<FAM>::type& th, double u, double w,
                                                const double2& t64, bool has_t) {
    if constexpr (FAM == kGaussian) {
        return gauss_full(has_t ? t64.x : dev_phi_inv(u), has_t ? t64.y : dev_phi_inv(w), th);
    } else if constexpr (FAM == kFrank) {
        return frank_full(u, w, th);
    } else {
        return has_t ? gumbel_full_l(u, w, t64.x, t64.y, th) : gumbel_full(u, w, th);
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
template <int FAM>
__global__ void __launch_bounds__(FT) k_var_point(BlockState* st, const Seg* segs, int nseg,
                                                 const unsigned long long* __restrict__ rp,
                                                 const double* __restrict__ u1, const double* __restrict__ u2,
                                                 const double2* __restrict__ T64, const double* __restrict__ gtab,
                                                 const uint64_t* goff, uint64_t n_rows, double* __restrict__ zb,
                                                 double* __restrict__ Ag, double* partials,
                                                 unsigned* tickets) {
    const uint32_t tile = blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (st[m].status != kConverged) return;
    const typename ThetaOf<FAM>::type th(st[m].theta);
    const double scale = 1.0 / (static_cast<double>(S.n) + 1.0);
    const uint32_t base = (tile - S.tile0) * FTILE;
    const double* gt = gtab ? gtab + goff[m] : nullptr;
    const bool has_t = gt || T64;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    constexpr int U = 2;  // points per thread in flight
    for (int k0 = 0; k0 < PPT; k0 += U) {
        unsigned long long p1[U], p2[U];
        double2 tt[U];
        double uu[U], ww[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + (k0 + j) * FT + threadIdx.x;
            if (i < S.n) {
                const uint64_t row = S.begin + i;
                p1[j] = rp[row];
                p2[j] = rp[n_rows + row];
                if (u1) {
                    uu[j] = u1[row];
                    ww[j] = u2[row];
                }
                if (T64) tt[j] = T64[row];
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = base + (k0 + j) * FT + threadIdx.x;
            if (i >= S.n) continue;
            const uint64_t row = S.begin + i;
            double u = u1 ? uu[j] : __dmul_rn(0.5 * static_cast<double>(rank_r2(p1[j])), scale);
            double w = u1 ? ww[j] : __dmul_rn(0.5 * static_cast<double>(rank_r2(p2[j])), scale);
            u = clamp_unit(u);
            w = clamp_unit(w);
            if (gt) tt[j] = make_double2(gt[rank_r2(p1[j])], gt[rank_r2(p2[j])]);
            const PointFull p = eval_point<FAM>(th, u, w, tt[j], has_t);
            zb[row] = p.score;
            // cross_j to its sorted position (random within the block: L2-resident
            // while the block's tiles are in flight), run-start flag beside it
            const uint64_t q1 = S.begin + rank_pos(p1[j]), q2 = n_rows + S.begin + rank_pos(p2[j]);
            Ag[q1] = with_flag(p.cross1, rank_first(p1[j]));
            Ag[q2] = with_flag(p.cross2, rank_first(p2[j]));
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

// ------------------------------------------------------------ pass 2 (cluster)
// W_j(row) += value on the row's home CTA (DSMEM reduction; each row gets
// one store for column 1 and one add for column 2, so the result is exact
// and order-independent).
__device__ __forceinline__ void dsmem_add_f64(double* local_slot, uint32_t rank, double v) {
    const uint32_t la = static_cast<uint32_t>(__cvta_generic_to_shared(local_slot));
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
    asm volatile("red.relaxed.cluster.shared::cluster.add.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

template <int DUMMY>
__global__ void __launch_bounds__(VT, 1) k_var_w(BlockState* st, const Seg* segs, const int* seg_list,
                                                const uint32_t* __restrict__ ord, uint64_t n_rows,
                                                const double* __restrict__ zb, const double* __restrict__ Ag, int CL,
                                                uint32_t SMAX, unsigned long long* prof) {
    long long t_prev = clock64();
    auto mark = [&](int k) {  // optional phase timing (PCB_VAR_PROFILE)
        if (prof && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(prof + k, static_cast<unsigned long long>(t - t_prev));
            t_prev = t;
        }
    };
    cg::cluster_group cluster = cg::this_cluster();
    const int r = static_cast<int>(cluster.block_rank());
    const int m = seg_list[blockIdx.x / CL];
    const Seg S = segs[m];
    if (st[m].status != kConverged) return;  // uniform across the cluster, before any DSMEM access
    const uint32_t n = S.n;
    const uint32_t SL = (n + CL - 1) / CL;
    const uint32_t a = min(n, r * SL), e = min(n, a + SL);
    const uint32_t len = e - a;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const double nd = static_cast<double>(n);

    // CTA r owns sorted positions [a, e) AND home rows [a, e) of the block
    extern __shared__ __align__(16) unsigned char smem[];
    double* A = reinterpret_cast<double*>(smem);               // suffix sums of its positions
    double* wacc = A + SMAX;                                   // W_1 + W_2 of its home rows
    uint32_t* bits = reinterpret_cast<uint32_t*>(wacc + SMAX);  // run-start bit per position
    __shared__ double s_tot, s_z;
    __shared__ double s_red[VNW];
    __shared__ double s_wt[VNW], s_wo[VNW];

    // warp w owns the contiguous positions [w*WL, (w+1)*WL) of the slice (WL % 32 == 0)
    const uint32_t WL = ((len + VNW - 1) / VNW + 31) & ~31u;
    const uint32_t w0 = min(len, wid * WL), w1 = min(len, w0 + WL);

    for (int col = 0; col < 2; ++col) {
        const double cj = col ? st[m].c2 : st[m].c1;
        const double* Aj = Ag + static_cast<uint64_t>(col) * n_rows + S.begin + a;
        const uint32_t* Oj = ord + static_cast<uint64_t>(col) * n_rows + S.begin + a;
        cluster.sync();  // the previous column's walks over A / bits are done everywhere
        mark(0);
        // load this warp's positions (coalesced), peel the run-start bits, warp total
        double wsum = 0.0;
        for (uint32_t q0 = w0; q0 < w1; q0 += 32 * 4) {
            double c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t q = q0 + u * 32 + lane;
                c[u] = q < w1 ? Aj[q] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t q = q0 + u * 32 + lane;
                const unsigned fb = __ballot_sync(0xffffffffu, q < w1 && flag_of(c[u]));
                if (q0 + u * 32 < w1) {
                    if (lane == 0) bits[(q0 + u * 32) >> 5] = fb;
                    if (q < w1) A[q] = c[u];
                    wsum += c[u];
                }
            }
        }
        wsum = warp_sum(wsum);
        if (lane == 0) s_wt[wid] = wsum;
        __syncthreads();
        if (wid == 0) {  // exclusive suffix of the warp totals; slice total
            double x = s_wt[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_down_sync(0xffffffffu, x, o);
                if (lane + o < 32) x += y;
            }
            s_wo[lane] = x - s_wt[lane];
            if (lane == 0) s_tot = x;
        }
        mark(1);
        cluster.sync();  // slice totals published
        double carry = s_wo[wid];
        for (int q = r + 1; q < CL; ++q) carry += *cluster.map_shared_rank(&s_tot, q);  // slices above
        // suffix scan of the warp's positions, top tile first
        for (uint32_t t = (w1 - w0 + 31) / 32; t-- > 0;) {
            const uint32_t q = w0 + t * 32 + lane;
            double x = q < w1 ? A[q] : 0.0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_down_sync(0xffffffffu, x, o);
                if (lane + o < 32) x += y;
            }
            if (q < w1) A[q] = carry + x;
            carry += __shfl_sync(0xffffffffu, x, 0);
        }
        cluster.sync();  // suffix sums complete everywhere
        mark(2);
        // W_j of the row at each of this CTA's positions -> pushed to the row's home CTA
        constexpr int PU = 4;  // order loads in flight per thread
        for (uint32_t p0 = tid; p0 < len; p0 += VT * PU) {
          uint32_t rows[PU];
#pragma unroll
          for (int u = 0; u < PU; ++u) {
            const uint32_t p = p0 + u * VT;
            rows[u] = p < len ? Oj[p] : 0u;
          }
#pragma unroll
          for (int u = 0; u < PU; ++u) {
            const uint32_t p = p0 + u * VT;
            if (p >= len) continue;
            const uint32_t row = rows[u];
            double T;
            if ((bits[p >> 5] >> (p & 31)) & 1u) {
                T = A[p];
            } else {  // tied, not first: highest run-start bit below this position
                uint32_t t = a + p - 1;
                uint32_t q;
                for (;;) {
                    const uint32_t o = t / SL, lt = t - o * SL;
                    uint32_t w = *cluster.map_shared_rank(bits + (lt >> 5), o);
                    w &= 0xffffffffu >> (31 - (lt & 31));
                    if (w) {
                        q = o * SL + (lt & ~31u) + (31 - __clz(w));
                        break;
                    }
                    t = o * SL + (lt & ~31u) - 1;  // position 0 always starts a run
                }
                const uint32_t o = q / SL;
                T = *cluster.map_shared_rank(A + (q - o * SL), o);
            }
            const double wj = (T - cj) / nd;
            const uint32_t h = row / SL, slot = row - h * SL;
            if (col == 0) *cluster.map_shared_rank(wacc + slot, h) = wj;
            else dsmem_add_f64(wacc + slot, h, wj);
          }
        }
        mark(3);
    }
    cluster.sync();  // every W has reached its home row
    double zz = 0.0;
    for (uint32_t i = tid; i < len; i += VT) {
        const double z = zb[S.begin + a + i] + wacc[i];
        zz += z * z;
    }
    // fixed-order reduction of sum z^2: block, then cluster
    double v[1] = {zz};
    block_sum<1>(v, s_red);
    if (tid == 0) s_z = v[0];
    cluster.sync();
    if (r == 0 && tid == 0) {
        double tot = 0.0;
        for (int q = 0; q < CL; ++q) tot += *cluster.map_shared_rank(&s_z, q);
        BlockState s = st[m];
        s.sigma2 = finish_sigma2(s, tot, nd);
        st[m] = s;
    }
    cluster.sync();  // peers' shared memory is read above
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

struct VarPlan {
    int cl = 0;
    uint32_t smax = 0;
    size_t smem = 0;
};

VarPlan plan_var(uint64_t nmax) {
    int forced = 0;
    if (const char* v = std::getenv("PCB_VAR_CL")) forced = std::atoi(v);
    if (const char* v = std::getenv("PCB_VAR_GLOBAL"))
        if (v[0] && v[0] != '0') return VarPlan{};
    for (int cl = 1; cl <= kMaxCl; ++cl) {
        if (forced && cl != forced) continue;
        VarPlan p;
        p.cl = cl;
        p.smax = static_cast<uint32_t>((nmax + cl - 1) / cl);
        p.smax = (p.smax + 31u) & ~31u;
        p.smem = static_cast<size_t>(p.smax) * 16 + (p.smax / 32 + 1) * 4;
        if (p.smem <= kVarSmem) return p;
    }
    return VarPlan{};
}

template <int FAM>
void launch_var_point(Ctx& c, const VarIO& v, double* zb, double* Ag) {
    const int K = static_cast<int>(v.off->size() - 1);
    k_var_point<FAM><<<v.tiles, FT, 0, c.stream>>>(v.st, v.segs, K, v.rp, v.u1, v.u2, v.T64, v.gtab, v.goff,
                                                   v.n_rows, zb, Ag, v.partials, v.tickets);
    c.count_launch();
}

void launch_var_w(Ctx& c, const VarPlan& p, const VarIO& v, const int* seg_list, int njobs, double* zb,
                  const double* Ag) {
    auto k = k_var_w<0>;
    PCB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem)));
    if (p.cl > 8) PCB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(njobs) * static_cast<unsigned>(p.cl));
    cfg.blockDim = dim3(VT);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(p.cl);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    unsigned long long* prof = nullptr;
    const char* pe = std::getenv("PCB_VAR_PROFILE");
    if (pe && pe[0] == '1') {
        prof = c.ws.get_t<unsigned long long>("var.prof", 8);
        PCB_CUDA(cudaMemsetAsync(prof, 0, 8 * sizeof(unsigned long long), c.stream));
    }
    PCB_CUDA(cudaLaunchKernelEx(&cfg, k, v.st, v.segs, seg_list, v.ord, v.n_rows, zb, Ag, p.cl, p.smax, prof));
    c.count_launch();
    if (prof) {
        unsigned long long h[8];
        PCB_CUDA(cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, c.stream));
        PCB_CUDA(cudaStreamSynchronize(c.stream));
        const double ctas = static_cast<double>(njobs) * p.cl;
        std::fprintf(stderr, "[var profile] CL=%d smax=%u cycles/CTA (both columns): sync %.0f  load %.0f  scan %.0f  gather %.0f\n",
                     p.cl, p.smax, h[0] / ctas, h[1] / ctas, h[2] / ctas, h[3] / ctas);
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
    auto* zb = c.ws.get_t<double>("var.z", v.n_rows);
    auto* Ag = c.ws.get_t<double>("var.A", 2 * v.n_rows);
    PCB_CUDA(cudaEventRecord(c.ev[6], c.stream));
    if (v.family == kGaussian) launch_var_point<kGaussian>(c, v, zb, Ag);
    else if (v.family == kFrank) launch_var_point<kFrank>(c, v, zb, Ag);
    else launch_var_point<kGumbel>(c, v, zb, Ag);
    PCB_CUDA(cudaEventRecord(c.ev[7], c.stream));
    uint64_t nmax = 0;
    for (int m = 0; m < K; ++m) nmax = std::max<uint64_t>(nmax, off[m + 1] - off[m]);
    const VarPlan p = plan_var(nmax);
    if (p.cl > 0) {
        std::vector<int> jobs(K);
        for (int m = 0; m < K; ++m) jobs[m] = m;
        int* d_jobs = c.ws.get_t<int>("var.jobs", K);
        PCB_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), K * sizeof(int), cudaMemcpyHostToDevice, c.stream));
        launch_var_w(c, p, v, d_jobs, K, zb, Ag);
    } else {
        std::vector<uint8_t> use(K, 1);
        uint8_t* d_use = c.ws.get_t<uint8_t>("var.use", K);
        PCB_CUDA(cudaMemcpyAsync(d_use, use.data(), K, cudaMemcpyHostToDevice, c.stream));
        launch_var_global(c, v, d_use, zb, Ag);
    }
    PCB_CUDA(cudaEventSynchronize(c.ev[7]));
    float ms = 0.0f;
    PCB_CUDA(cudaEventElapsedTime(&ms, c.ev[6], c.ev[7]));
    c.stage_ms[9] = ms;  // variance pass 1 (per-point terms); the rest of [3] is pass 2
}

}  // namespace pcb

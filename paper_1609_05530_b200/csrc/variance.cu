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

template <int FAM>
__device__ __forceinline__ PointFull eval_point(double theta, double u, double w, const double2* T64, uint64_t row,
                                                const double* gtab, unsigned long long p1, unsigned long long p2) {
    if (FAM == kGaussian) {
        double x, y;
        if (gtab) {
            x = gtab[rank_r2(p1)];
            y = gtab[rank_r2(p2)];
        } else if (T64) {
            const double2 t = T64[row];
            x = t.x;
            y = t.y;
        } else {
            x = dev_phi_inv(u);
            y = dev_phi_inv(w);
        }
        return gauss_full(x, y, GaussTheta(theta));
    }
    if (FAM == kFrank) return frank_full(u, w, FrankTheta(theta));
    if (T64) {
        const double2 t = T64[row];
        return gumbel_full_l(u, w, t.x, t.y, GumbelTheta(theta));
    }
    return gumbel_full(u, w, GumbelTheta(theta));
}

// ------------------------------------------------------------ pass 1
template <int FAM>
__global__ void __launch_bounds__(FT) k_var_point(BlockState* st, const Seg* segs, int nseg,
                                                 const unsigned long long* rp, const double* u1, const double* u2,
                                                 const double2* T64, const double* gtab, const uint64_t* goff,
                                                 uint64_t n_rows, double* zb, double* Ag, uint8_t* Fg,
                                                 double* partials, unsigned* tickets) {
    const uint32_t tile = blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (st[m].status != kConverged) return;
    const double theta = st[m].theta;
    const double scale = 1.0 / (static_cast<double>(S.n) + 1.0);
    const uint32_t base = (tile - S.tile0) * FTILE;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < PPT; ++k) {
        const uint32_t i = base + k * FT + threadIdx.x;
        if (i >= S.n) break;
        const uint64_t row = S.begin + i;
        double u, w;
        point_u(rp, u1, u2, n_rows, row, scale, u, w);
        u = clamp_unit(u);
        w = clamp_unit(w);
        const unsigned long long p1 = rp[row], p2 = rp[n_rows + row];
        const PointFull p = eval_point<FAM>(theta, u, w, T64, row, gtab ? gtab + goff[m] : nullptr, p1, p2);
        zb[row] = p.score;
        // cross_j to its sorted position (random within the block: L2-resident
        // while the block's tiles are in flight), run-start flag beside it
        const uint64_t q1 = S.begin + rank_pos(p1), q2 = n_rows + S.begin + rank_pos(p2);
        Ag[q1] = p.cross1;
        Ag[q2] = p.cross2;
        Fg[q1] = rank_first(p1) ? 1 : 0;
        Fg[q2] = rank_first(p2) ? 1 : 0;
        v[0] += p.hess;
        v[1] += u * p.cross1;
        v[2] += w * p.cross2;
        v[3] += clip_log(p.logc);
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
template <int DUMMY>
__global__ void __launch_bounds__(VT, 1) k_var_w(BlockState* st, const Seg* segs, const int* seg_list,
                                                const unsigned long long* rp, uint64_t n_rows, double* zb,
                                                const double* Ag, const uint8_t* Fg, int CL, uint32_t SMAX) {
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

    extern __shared__ __align__(16) unsigned char smem[];
    double* A = reinterpret_cast<double*>(smem);             // this CTA's slice of sorted positions
    uint8_t* flags = reinterpret_cast<uint8_t*>(A + SMAX);  // run-start byte per position
    __shared__ double s_tot, s_off, s_z;
    __shared__ double s_red[VNW];
    __shared__ double s_ch[VNW], s_ch2[VNW];

    double zz = 0.0;
    constexpr int VU = 4;  // points per thread in flight
    for (int col = 0; col < 2; ++col) {
        const double cj = col ? st[m].c2 : st[m].c1;
        const unsigned long long* rpc = rp + static_cast<uint64_t>(col) * n_rows + S.begin;
        const double* Aj = Ag + static_cast<uint64_t>(col) * n_rows + S.begin + a;
        const uint8_t* Fj = Fg + static_cast<uint64_t>(col) * n_rows + S.begin + a;
        cluster.sync();  // the previous column's gathers from A / flags are done everywhere
        // this slice of the sorted cross values and run-start flags (contiguous, coalesced)
        for (uint32_t q0 = tid; q0 < len; q0 += VT * VU) {
            double c[VU];
            uint8_t f[VU];
#pragma unroll
            for (int u = 0; u < VU; ++u) {
                const uint32_t q = q0 + u * VT;
                if (q < len) {
                    c[u] = Aj[q];
                    f[u] = Fj[q];
                }
            }
#pragma unroll
            for (int u = 0; u < VU; ++u) {
                const uint32_t q = q0 + u * VT;
                if (q < len) {
                    A[q] = c[u];
                    flags[q] = f[u];
                }
            }
        }
        __syncthreads();
        // suffix sums of this slice: slice total first, then a reverse tiled scan
        double tv[1] = {0.0};
        for (uint32_t q = tid; q < len; q += VT) tv[0] += A[q];
        block_sum<1>(tv, s_red);
        if (tid == 0) s_tot = tv[0];
        cluster.sync();  // slice totals published
        if (tid == 0) {
            double off = 0.0;
            for (int q = r + 1; q < CL; ++q) off += *cluster.map_shared_rank(&s_tot, q);
            s_off = off;
        }
        __syncthreads();
        double carry = s_off;
        const uint32_t ntile = (len + VT - 1) / VT;
        for (uint32_t t = ntile; t-- > 0;) {
            const uint32_t q = t * VT + tid;
            const double v = q < len ? A[q] : 0.0;
            double x = v;  // inclusive suffix within the warp
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_down_sync(0xffffffffu, x, o);
                if (lane + o < 32) x += y;
            }
            if (lane == 0) s_ch[wid] = x;
            __syncthreads();
            if (wid == 0) {  // inclusive suffix over the warp totals (fixed order)
                double y = s_ch[lane];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double z2 = __shfl_down_sync(0xffffffffu, y, o);
                    if (lane + o < 32) y += z2;
                }
                s_ch2[lane] = y;
            }
            __syncthreads();
            const double later = wid + 1 < VNW ? s_ch2[wid + 1] : 0.0;  // warps above this one
            if (q < len) A[q] = carry + later + x;
            carry += s_ch2[0];
            __syncthreads();
        }
        cluster.sync();  // suffix sums complete everywhere
        // gather T_j at each point's run start
        for (uint32_t i0 = a + tid; i0 < e; i0 += VT * VU) {
            unsigned long long p[VU];
            double zv[VU];
#pragma unroll
            for (int u = 0; u < VU; ++u) {
                const uint32_t i = i0 + u * VT;
                if (i < e) {
                    p[u] = rpc[i];
                    zv[u] = zb[S.begin + i];
                }
            }
            double tj[VU];
#pragma unroll
            for (int u = 0; u < VU; ++u) {
                if (i0 + u * VT < e) {
                    uint32_t q = rank_pos(p[u]);
                    if (!rank_first(p[u])) {  // tied, not first: nearest run start below q
                        do {
                            --q;  // position 0 always starts a run
                        } while (!*cluster.map_shared_rank(flags + (q - (q / SL) * SL), q / SL));
                    }
                    const uint32_t o = q / SL;
                    tj[u] = *cluster.map_shared_rank(A + (q - o * SL), o);
                }
            }
#pragma unroll
            for (int u = 0; u < VU; ++u) {
                const uint32_t i = i0 + u * VT;
                if (i < e) {
                    const double wj = (tj[u] - cj) / nd;
                    if (col == 0) {
                        zb[S.begin + i] = zv[u] + wj;  // score + W_1
                    } else {
                        const double z = zv[u] + wj;
                        zz += z * z;
                    }
                }
            }
        }
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
    (void)lane;
    (void)wid;
    cluster.sync();  // peers' shared memory is read above
}

// ------------------------------------------------------------ pass 2 (global)
// Same steps through HBM for blocks larger than a cluster holds: pass 1 has
// already placed cross_j in sorted order; suffix-scan it, then gather.
__global__ void __launch_bounds__(1024) k_suffix_g(const BlockState* st, const Seg* segs, int nseg,
                                                  const uint8_t* use, uint64_t n_rows, double* A) {
    const int m = blockIdx.x % nseg;
    const int col = blockIdx.x / nseg;
    if (!use[m] || st[m].status != kConverged) return;
    const Seg S = segs[m];
    double* a = A + static_cast<uint64_t>(col) * n_rows + S.begin;
    const uint32_t n = S.n;
    const uint32_t chunk = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = min(n, threadIdx.x * chunk), b1 = min(n, b0 + chunk);
    double local = 0.0;
    for (uint32_t q = b1; q-- > b0;) local += a[q];
    __shared__ double s_tot[1024];
    s_tot[threadIdx.x] = local;
    __syncthreads();
    for (int o = 1; o < static_cast<int>(blockDim.x); o <<= 1) {
        double add = 0.0;
        if (threadIdx.x + o < blockDim.x) add = s_tot[threadIdx.x + o];
        __syncthreads();
        s_tot[threadIdx.x] += add;
        __syncthreads();
    }
    double run = threadIdx.x + 1 < blockDim.x ? s_tot[threadIdx.x + 1] : 0.0;
    for (uint32_t q = b1; q-- > b0;) {
        run += a[q];
        a[q] = run;
    }
}

__global__ void __launch_bounds__(FT) k_var_gather_g(BlockState* st, const Seg* segs, int nseg, const uint8_t* use,
                                                    const unsigned long long* rp, uint64_t n_rows, const double* zb,
                                                    const double* A, const uint8_t* F, double* partials,
                                                    unsigned* tickets) {
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
                } while (!F[b0 + q]);
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
        p.smem = static_cast<size_t>(p.smax) * 9;
        if (p.smem <= kVarSmem) return p;
    }
    return VarPlan{};
}

template <int FAM>
void launch_var_point(Ctx& c, const VarIO& v, double* zb, double* Ag, uint8_t* Fg) {
    const int K = static_cast<int>(v.off->size() - 1);
    k_var_point<FAM><<<v.tiles, FT, 0, c.stream>>>(v.st, v.segs, K, v.rp, v.u1, v.u2, v.T64, v.gtab, v.goff,
                                                   v.n_rows, zb, Ag, Fg, v.partials, v.tickets);
    c.count_launch();
}

void launch_var_w(Ctx& c, const VarPlan& p, const VarIO& v, const int* seg_list, int njobs, double* zb,
                  const double* Ag, const uint8_t* Fg) {
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
    PCB_CUDA(cudaLaunchKernelEx(&cfg, k, v.st, v.segs, seg_list, v.rp, v.n_rows, zb, Ag, Fg, p.cl, p.smax));
    c.count_launch();
}

void launch_var_global(Ctx& c, const VarIO& v, const uint8_t* use, double* zb, double* Ag, const uint8_t* Fg) {
    const int K = static_cast<int>(v.off->size() - 1);
    k_suffix_g<<<2 * K, 1024, 0, c.stream>>>(v.st, v.segs, K, use, v.n_rows, Ag);
    k_var_gather_g<<<v.tiles, FT, 0, c.stream>>>(v.st, v.segs, K, use, v.rp, v.n_rows, zb, Ag, Fg, v.partials,
                                                 v.tickets);
    c.count_launch(2);
}

}  // namespace

void run_variance(Ctx& c, const VarIO& v) {
    const std::vector<uint64_t>& off = *v.off;
    const int K = static_cast<int>(off.size() - 1);
    auto* zb = c.ws.get_t<double>("var.z", v.n_rows);
    auto* Ag = c.ws.get_t<double>("var.A", 2 * v.n_rows);
    auto* Fg = c.ws.get_t<uint8_t>("var.F", 2 * v.n_rows);
    if (v.family == kGaussian) launch_var_point<kGaussian>(c, v, zb, Ag, Fg);
    else if (v.family == kFrank) launch_var_point<kFrank>(c, v, zb, Ag, Fg);
    else launch_var_point<kGumbel>(c, v, zb, Ag, Fg);
    uint64_t nmax = 0;
    for (int m = 0; m < K; ++m) nmax = std::max<uint64_t>(nmax, off[m + 1] - off[m]);
    const VarPlan p = plan_var(nmax);
    if (p.cl > 0) {
        std::vector<int> jobs(K);
        for (int m = 0; m < K; ++m) jobs[m] = m;
        int* d_jobs = c.ws.get_t<int>("var.jobs", K);
        PCB_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), K * sizeof(int), cudaMemcpyHostToDevice, c.stream));
        launch_var_w(c, p, v, d_jobs, K, zb, Ag, Fg);
    } else {
        std::vector<uint8_t> use(K, 1);
        uint8_t* d_use = c.ws.get_t<uint8_t>("var.use", K);
        PCB_CUDA(cudaMemcpyAsync(d_use, use.data(), K, cudaMemcpyHostToDevice, c.stream));
        launch_var_global(c, v, d_use, zb, Ag, Fg);
    }
}

}  // namespace pcb

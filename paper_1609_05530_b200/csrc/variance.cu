// K3-K5 asymptotic variance on sm_100a.
//
//   sigma2 = M/I^2/n,  I = -(1/n) sum hess_i,
//   M = (1/n) sum (score_i + W1_i + W2_i)^2,
//   W_ji = (1/n) sum_h [1(u_ij <= u_hj) - u_hj] cross_j(u_h)
//        = (1/n) (T_j(run of i) - C_j),  C_j = sum_h u_hj cross_j(u_h),
// where T_j(p) is the suffix sum of cross_j over sorted positions >= the
// first position of i's tie run. Pseudo-observations are ranks, so sorting is
// already done: the rank stage's stable position `pos` scatters cross_j into
// sorted order, r2 (shared by a tie run, non-decreasing along sorted order)
// finds a run's first position, and one suffix scan gives every W.
//
// Cluster path (segments up to CL * SMAX points): one thread-block cluster per
// segment keeps both columns' sorted cross arrays (A_j, 8 B) and run keys
// (R_j, 4 B) in distributed shared memory; the scatter, the scan, and the
// gather are DSMEM traffic, so HBM sees only the per-point inputs. Larger
// segments use the same three steps through global memory.
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

constexpr int VT = 512;  // threads per cluster CTA
constexpr int kMaxCl = 16;
constexpr size_t kVarSmem = 227 * 1024 - 6144;

template <int FAM>
__device__ __forceinline__ PointFull eval_point(double theta, double u, double w, const double2* T64, uint64_t row) {
    if (FAM == kGaussian) {
        double x, y;
        if (T64) {
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

// --------------------------------------------------------------- cluster
template <int FAM>
__global__ void __launch_bounds__(VT, 1) k_var_cluster(BlockState* st, const Seg* segs, const int* seg_list,
                                                      const unsigned long long* rp, const double* u1, const double* u2,
                                                      const double2* T64, uint64_t n_rows, double* score, int CL,
                                                      uint32_t SMAX) {
    cg::cluster_group cluster = cg::this_cluster();
    const int r = static_cast<int>(cluster.block_rank());
    const int m = seg_list[blockIdx.x / CL];
    const Seg S = segs[m];
    if (st[m].status != kConverged) return;  // uniform across the cluster, before any DSMEM access
    const double theta = st[m].theta;
    const uint32_t n = S.n;
    const uint32_t SL = (n + CL - 1) / CL;
    const uint32_t a = min(n, r * SL), e = min(n, a + SL);
    const int tid = threadIdx.x;
    const double scale = 1.0 / (static_cast<double>(n) + 1.0);

    extern __shared__ __align__(16) unsigned char smem[];
    double* A1 = reinterpret_cast<double*>(smem);
    double* A2 = A1 + SMAX;
    uint32_t* R1 = reinterpret_cast<uint32_t*>(A2 + SMAX);
    uint32_t* R2 = R1 + SMAX;
    __shared__ double s_part[4];   // hess, u*cross1, v*cross2, logc of this CTA's points
    __shared__ double s_tot[2];    // this CTA's slice totals of A1, A2
    __shared__ double s_z;         // this CTA's sum of z^2
    __shared__ double s_red[(VT / 32) * 4];
    __shared__ double s_g[4], s_off[2];

    // ---- 1. per-point terms; cross_j -> A_j[pos_j] and r2_j -> R_j[pos_j] (DSMEM)
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint32_t i = a + tid; i < e; i += VT) {
        const uint64_t row = S.begin + i;
        const unsigned long long p1 = rp[row], p2 = rp[n_rows + row];
        double u, w;
        point_u(rp, u1, u2, n_rows, row, scale, u, w);
        u = clamp_unit(u);
        w = clamp_unit(w);
        const PointFull p = eval_point<FAM>(theta, u, w, T64, row);
        score[row] = p.score;
        const uint32_t q1 = rank_pos(p1), q2 = rank_pos(p2);
        const uint32_t o1 = q1 / SL, o2 = q2 / SL;
        *cluster.map_shared_rank(A1 + (q1 - o1 * SL), o1) = p.cross1;
        *cluster.map_shared_rank(R1 + (q1 - o1 * SL), o1) = rank_r2(p1);
        *cluster.map_shared_rank(A2 + (q2 - o2 * SL), o2) = p.cross2;
        *cluster.map_shared_rank(R2 + (q2 - o2 * SL), o2) = rank_r2(p2);
        acc[0] += p.hess;
        acc[1] += u * p.cross1;
        acc[2] += w * p.cross2;
        acc[3] += clip_log(p.logc);
    }
    block_sum<4>(acc, s_red);
    if (tid == 0)
        for (int k = 0; k < 4; ++k) s_part[k] = acc[k];
    cluster.sync();

    // ---- 2. suffix sums of this CTA's slice of A1 / A2 (positions a..e-1)
    if (tid < 4) {  // segment totals, fixed order over CTAs
        double g = 0.0;
        for (int q = 0; q < CL; ++q) g += *cluster.map_shared_rank(&s_part[tid], q);
        s_g[tid] = g;
    }
    const uint32_t len = e - a;
    const uint32_t chunk = (len + VT - 1) / VT;
    const uint32_t c0 = min(len, tid * chunk), c1 = min(len, c0 + chunk);
    __shared__ double s_ch[2][VT];
    for (int col = 0; col < 2; ++col) {
        double* Aj = col ? A2 : A1;
        double loc = 0.0;
        for (uint32_t q = c1; q-- > c0;) loc += Aj[q];
        s_ch[col][tid] = loc;
    }
    __syncthreads();
    // exclusive suffix scan of the chunk totals (Hillis-Steele, fixed order)
    for (int o = 1; o < VT; o <<= 1) {
        double add0 = 0.0, add1 = 0.0;
        if (tid + o < VT) {
            add0 = s_ch[0][tid + o];
            add1 = s_ch[1][tid + o];
        }
        __syncthreads();
        s_ch[0][tid] += add0;
        s_ch[1][tid] += add1;
        __syncthreads();
    }
    for (int col = 0; col < 2; ++col) {
        double* Aj = col ? A2 : A1;
        double run = tid + 1 < VT ? s_ch[col][tid + 1] : 0.0;
        for (uint32_t q = c1; q-- > c0;) {
            run += Aj[q];
            Aj[q] = run;
        }
    }
    if (tid < 2) s_tot[tid] = s_ch[tid][0];
    cluster.sync();
    if (tid < 2) {  // mass of the slices above this one
        double off = 0.0;
        for (int q = r + 1; q < CL; ++q) off += *cluster.map_shared_rank(&s_tot[tid], q);
        s_off[tid] = off;
    }
    __syncthreads();
    for (uint32_t q = tid; q < len; q += VT) {
        A1[q] += s_off[0];
        A2[q] += s_off[1];
    }
    cluster.sync();

    // ---- 3. W_j from the suffix at the tie run's first position; M-hat
    const double c1s = s_g[1], c2s = s_g[2], nd = static_cast<double>(n);
    auto run_start = [&](const uint32_t* Rj, uint32_t pos, uint32_t key) -> uint32_t {
        if (pos == 0) return 0;
        const uint32_t pm = pos - 1, om = pm / SL;
        if (*cluster.map_shared_rank(Rj + (pm - om * SL), om) != key) return pos;
        uint32_t lo = 0, hi = pm;  // first position whose R == key (R non-decreasing)
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1, o = mid / SL;
            if (*cluster.map_shared_rank(Rj + (mid - o * SL), o) < key) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    double z2[1] = {0.0};
    for (uint32_t i = a + tid; i < e; i += VT) {
        const uint64_t row = S.begin + i;
        const unsigned long long p1 = rp[row], p2 = rp[n_rows + row];
        const uint32_t s1 = run_start(R1, rank_pos(p1), rank_r2(p1));
        const uint32_t s2 = run_start(R2, rank_pos(p2), rank_r2(p2));
        const uint32_t o1 = s1 / SL, o2 = s2 / SL;
        const double w1 = (*cluster.map_shared_rank(A1 + (s1 - o1 * SL), o1) - c1s) / nd;
        const double w2 = (*cluster.map_shared_rank(A2 + (s2 - o2 * SL), o2) - c2s) / nd;
        const double z = score[row] + w1 + w2;
        z2[0] += z * z;
    }
    block_sum<1>(z2, s_red);
    if (tid == 0) s_z = z2[0];
    cluster.sync();
    if (r == 0 && tid == 0) {
        double zz = 0.0;
        for (int q = 0; q < CL; ++q) zz += *cluster.map_shared_rank(&s_z, q);
        BlockState s = st[m];
        s.info_sum = s_g[0];
        s.c1 = c1s;
        s.c2 = c2s;
        s.loglik = s_g[3];
        const double info = -s_g[0] / nd;
        if (!(info > 0.0)) {
            s.status = kInfoNonPos;
            s.sigma2 = NAN;
        } else {
            s.sigma2 = (zz / nd) / (info * info) / nd;
        }
        st[m] = s;
    }
    cluster.sync();  // peers' shared memory is read above
}

// ---------------------------------------------------------- global path
// Same three steps through HBM for segments larger than a cluster holds.
template <int FAM>
__global__ void __launch_bounds__(FT) k_var_terms_g(BlockState* st, const Seg* segs, int nseg, const uint8_t* use,
                                                   const unsigned long long* rp, const double* u1, const double* u2,
                                                   const double2* T64, uint64_t n_rows, double* score, double* A,
                                                   uint32_t* R, double* partials, unsigned* tickets) {
    const uint32_t tile = blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (!use[m] || st[m].status != kConverged) return;
    const double theta = st[m].theta;
    const double scale = 1.0 / (static_cast<double>(S.n) + 1.0);
    const uint32_t base = (tile - S.tile0) * FTILE;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < PPT; ++k) {
        const uint32_t i = base + k * FT + threadIdx.x;
        if (i >= S.n) break;
        const uint64_t row = S.begin + i;
        const unsigned long long p1 = rp[row], p2 = rp[n_rows + row];
        double u, w;
        point_u(rp, u1, u2, n_rows, row, scale, u, w);
        u = clamp_unit(u);
        w = clamp_unit(w);
        const PointFull p = eval_point<FAM>(theta, u, w, T64, row);
        score[row] = p.score;
        A[S.begin + rank_pos(p1)] = p.cross1;
        R[S.begin + rank_pos(p1)] = rank_r2(p1);
        A[n_rows + S.begin + rank_pos(p2)] = p.cross2;
        R[n_rows + S.begin + rank_pos(p2)] = rank_r2(p2);
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

__global__ void __launch_bounds__(FT) k_var_final_g(BlockState* st, const Seg* segs, int nseg, const uint8_t* use,
                                                   const unsigned long long* rp, uint64_t n_rows, const double* score,
                                                   const double* A, const uint32_t* R, double* partials,
                                                   unsigned* tickets) {
    const uint32_t tile = blockIdx.x;
    const int m = seg_of_tile(segs, nseg, tile);
    const Seg S = segs[m];
    if (!use[m] || st[m].status != kConverged) return;
    const double nd = static_cast<double>(S.n);
    const double c1 = st[m].c1, c2 = st[m].c2;
    const uint32_t base = (tile - S.tile0) * FTILE;
    auto run_start = [&](const uint32_t* Rj, uint32_t pos, uint32_t key) -> uint32_t {
        if (pos == 0 || Rj[pos - 1] != key) return pos;
        uint32_t lo = 0, hi = pos - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (Rj[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    double v[1] = {0.0};
    for (int k = 0; k < PPT; ++k) {
        const uint32_t i = base + k * FT + threadIdx.x;
        if (i >= S.n) break;
        const uint64_t row = S.begin + i;
        const unsigned long long p1 = rp[row], p2 = rp[n_rows + row];
        const uint32_t* R1 = R + S.begin;
        const uint32_t* R2 = R + n_rows + S.begin;
        const uint32_t s1 = run_start(R1, rank_pos(p1), rank_r2(p1));
        const uint32_t s2 = run_start(R2, rank_pos(p2), rank_r2(p2));
        const double w1 = (A[S.begin + s1] - c1) / nd;
        const double w2 = (A[n_rows + S.begin + s2] - c2) / nd;
        const double z = score[row] + w1 + w2;
        v[0] += z * z;
    }
    __shared__ double sh[FT / 32];
    if (!tile_reduce<1>(v, sh, partials, tickets, S, m, tile)) return;
    if (threadIdx.x == 0) {
        BlockState s = st[m];
        const double info = -s.info_sum / nd;
        if (!(info > 0.0)) {
            s.status = kInfoNonPos;
            s.sigma2 = NAN;
        } else {
            s.sigma2 = (v[0] / nd) / (info * info) / nd;
        }
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
        p.smax = (p.smax + 1u) & ~1u;
        p.smem = static_cast<size_t>(p.smax) * 24;
        if (p.smem <= kVarSmem) return p;
    }
    return VarPlan{};
}

template <int FAM>
void launch_var_cluster(Ctx& c, const VarPlan& p, const VarIO& v, const int* seg_list, int njobs, double* score) {
    auto k = k_var_cluster<FAM>;
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
    PCB_CUDA(cudaLaunchKernelEx(&cfg, k, v.st, v.segs, seg_list, v.rp, v.u1, v.u2, v.T64, v.n_rows, score, p.cl,
                                p.smax));
    c.count_launch();
}

template <int FAM>
void launch_var_global(Ctx& c, const VarIO& v, const uint8_t* use, double* score) {
    const int K = static_cast<int>(v.off->size() - 1);
    auto* A = c.ws.get_t<double>("var.A", 2 * v.n_rows);
    auto* R = c.ws.get_t<uint32_t>("var.R", 2 * v.n_rows);
    k_var_terms_g<FAM><<<v.tiles, FT, 0, c.stream>>>(v.st, v.segs, K, use, v.rp, v.u1, v.u2, v.T64, v.n_rows, score,
                                                     A, R, v.partials, v.tickets);
    k_suffix_g<<<2 * K, 1024, 0, c.stream>>>(v.st, v.segs, K, use, v.n_rows, A);
    k_var_final_g<<<v.tiles, FT, 0, c.stream>>>(v.st, v.segs, K, use, v.rp, v.n_rows, score, A, R, v.partials,
                                                v.tickets);
    c.count_launch(3);
}

}  // namespace

void run_variance(Ctx& c, const VarIO& v) {
    const std::vector<uint64_t>& off = *v.off;
    const int K = static_cast<int>(off.size() - 1);
    auto* score = c.ws.get_t<double>("var.score", v.n_rows);
    uint64_t nmax = 0;
    for (int m = 0; m < K; ++m) nmax = std::max<uint64_t>(nmax, off[m + 1] - off[m]);
    const VarPlan p = plan_var(nmax);
    std::vector<int> jobs;
    std::vector<uint8_t> use(K, 0);
    for (int m = 0; m < K; ++m) {
        if (p.cl > 0) jobs.push_back(m);
        else use[m] = 1;
    }
    if (!jobs.empty()) {
        int* d_jobs = c.ws.get_t<int>("var.jobs", jobs.size());
        PCB_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), jobs.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
        if (v.family == kGaussian) launch_var_cluster<kGaussian>(c, p, v, d_jobs, static_cast<int>(jobs.size()), score);
        else if (v.family == kFrank) launch_var_cluster<kFrank>(c, p, v, d_jobs, static_cast<int>(jobs.size()), score);
        else launch_var_cluster<kGumbel>(c, p, v, d_jobs, static_cast<int>(jobs.size()), score);
    } else {
        uint8_t* d_use = c.ws.get_t<uint8_t>("var.use", K);
        PCB_CUDA(cudaMemcpyAsync(d_use, use.data(), K, cudaMemcpyHostToDevice, c.stream));
        if (v.family == kGaussian) launch_var_global<kGaussian>(c, v, d_use, score);
        else if (v.family == kFrank) launch_var_global<kFrank>(c, v, d_use, score);
        else launch_var_global<kGumbel>(c, v, d_use, score);
    }
}

}  // namespace pcb

// K1 seg_rank — bit-exact segment-local average ranks for sm_100a.
//
// Replaces detail::normalized_rank_column (pseudo_obs.hpp:44-65): for each
// (segment, column) the reference index-sorts by (value, index) and gives a
// tie run i..j the average rank 0.5*((i+1)+(j+1)). The GPU never sorts:
// ranking only needs, per element, lt = #{values < x} and eq = #{values == x}
// in its segment (plus the number of equal values ordered before it, which
// yields a unique position for the variance's suffix sums).
//
// Two paths. Blocks a thread-block cluster can hold (C5: 125,000 rows) take
// the cluster path (k_rank_cluster_t, below): an all-to-all over distributed
// shared memory by value range, counting inside fine local buckets; ranks
// stay per receive slot ("routed"). Larger blocks, skewed data and
// non-finite ranges take the global path described here, which writes packed
// ranks by row.
//
// Global path (one "level" = 8 launches over every range at once):
//   minmax  per-range key / index extremes (64-bit order-preserving keys,
//           -0.0 == +0.0), fused non-finite check (validate_data,
//           pseudo_obs.hpp:30-37)
//   resolve per-range bucket map: value-linear (level 0), key-linear, or
//           row-index-linear for a range whose keys are all equal (a tie run)
//   hist    bucket counts (monotone bucket map => buckets are ordered
//           intervals of the sorted order; ties never straddle buckets)
//   scan    per-range exclusive scan (chunk sums, per-range chunk offsets,
//           chunk scans) -> bucket starts; buckets above CAP are queued for
//           the next level
//   scatter (key, row) into the bucket's slots of a scratch array
//   rank    per element: count smaller / equal / equal-with-smaller-row
//           inside its (small) bucket; lt = range base + bucket start + #less
// Oversize buckets become the next level's ranges (in place, ping-pong
// scratch). Each level shrinks an oversize range's key span by >= nb, so
// the refinement terminates in a few levels even for adversarial inputs;
// uniform-marginal data (every BASELINE config) finishes in level 0.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "internal.hpp"

namespace pcb {
namespace {

constexpr int RT = 256;
constexpr uint32_t RTILE = 4096;
constexpr uint32_t AVG = 8;    // target elements per bucket
constexpr uint32_t CAP = 256;  // buckets larger than this are refined

struct RankRange {
    uint64_t src_base;  // level 0: row offset in the input column; else scratch position
    uint64_t dst_base;  // scratch position of slot 0 of this range's buckets
    uint64_t out_base;  // row offset of the segment (outputs at col*n_rows + out_base + row)
    uint64_t bbase;     // first bucket slot
    unsigned long long kmin, kmax;
    uint64_t width;     // key-linear / index-linear bucket width
    double scale, vmin_half;
    uint32_t imin, imax;
    uint32_t n, nb;
    uint32_t lt_base, run_start, run_len;
    uint32_t tile0;
    int32_t mode;  // 0 value-linear, 1 key-linear, 2 tie run (index-linear)
    int32_t col, seg, pad;
};

struct Oversize {
    uint32_t range, start, count, pad;
};

__device__ __forceinline__ int range_of_tile(const RankRange* rr, int nr, uint32_t tile) {
    int lo = 0, hi = nr - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (rr[mid].tile0 <= tile) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

template <bool L0>
__device__ __forceinline__ void load_elem(const RankRange& R, uint32_t i, const double* c0, const double* c1,
                                          const ulonglong2* srec,
                                          unsigned long long& key, uint32_t& idx, bool& finite) {
    if (L0) {
        const double x = __ldg((R.col ? c1 : c0) + R.src_base + i);
        finite = isfinite(x);
        key = order_key(x);
        idx = i;
    } else {
        const ulonglong2 rec = srec[R.src_base + i];
        key = rec.x;
        idx = static_cast<uint32_t>(rec.y);
        finite = true;
    }
}

__device__ __forceinline__ uint32_t bucket_of(const RankRange& R, unsigned long long key, uint32_t idx) {
    if (R.mode == 0) {
        const double v = key_value(key);
        const double t = (0.5 * v - R.vmin_half) * R.scale;
        return t < static_cast<double>(R.nb) ? static_cast<uint32_t>(t) : R.nb - 1;
    }
    if (R.mode == 1) return static_cast<uint32_t>((key - R.kmin) / R.width);
    return static_cast<uint32_t>((idx - R.imin) / R.width);
}

template <bool L0>
__global__ void __launch_bounds__(RT) k_minmax(RankRange* rr, int nr, const double* c0, const double* c1,
                                              const ulonglong2* srec, int32_t* bad) {
    const int r = range_of_tile(rr, nr, blockIdx.x);
    const RankRange R = rr[r];
    const uint32_t begin = (blockIdx.x - R.tile0) * RTILE;
    const uint32_t end = min(begin + RTILE, R.n);
    unsigned long long kmn = ~0ull, kmx = 0ull;
    uint32_t imn = ~0u, imx = 0u;
    bool allfin = true;
    for (uint32_t i = begin + threadIdx.x; i < end; i += RT) {
        unsigned long long k;
        uint32_t id;
        bool fin;
        load_elem<L0>(R, i, c0, c1, srec, k, id, fin);
        allfin &= fin;
        kmn = min(kmn, k);
        kmx = max(kmx, k);
        imn = min(imn, id);
        imx = max(imx, id);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
        kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
        imn = min(imn, __shfl_xor_sync(0xffffffffu, imn, o));
        imx = max(imx, __shfl_xor_sync(0xffffffffu, imx, o));
    }
    allfin = __all_sync(0xffffffffu, allfin);
    __shared__ unsigned long long s_kmn[RT / 32], s_kmx[RT / 32];
    __shared__ uint32_t s_imn[RT / 32], s_imx[RT / 32];
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_kmn[w] = kmn;
        s_kmx[w] = kmx;
        s_imn[w] = imn;
        s_imx[w] = imx;
        if (!allfin) s_bad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < RT / 32; ++k) {
            kmn = min(kmn, s_kmn[k]);
            kmx = max(kmx, s_kmx[k]);
            imn = min(imn, s_imn[k]);
            imx = max(imx, s_imx[k]);
        }
        atomicMin(&rr[r].kmin, kmn);
        atomicMax(&rr[r].kmax, kmx);
        if (!L0) {
            atomicMin(&rr[r].imin, imn);
            atomicMax(&rr[r].imax, imx);
        }
        if (L0 && s_bad) bad[R.seg] = 1;
    }
}

__global__ void k_resolve(RankRange* rr, int nr, int level0) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nr) return;
    RankRange R = rr[r];
    if (level0) {
        R.imin = 0;
        R.imax = R.n ? R.n - 1 : 0;
    }
    if (R.mode == 0) {
        if (R.kmin == R.kmax) {
            R.mode = 2;
            R.run_start = R.lt_base;
            R.run_len = R.n;
        } else {
            const double vmin = key_value(R.kmin), vmax = key_value(R.kmax);
            const double hm = 0.5 * vmin;
            const double d = 0.5 * vmax - hm;
            const double sc = static_cast<double>(R.nb) / d;
            if (isfinite(sc) && sc > 0.0 && isfinite(hm)) {
                R.scale = sc;
                R.vmin_half = hm;
            } else {
                R.mode = 1;
            }
        }
    }
    if (R.mode == 1) {
        if (R.kmin == R.kmax) {
            R.mode = 2;
            R.run_start = R.lt_base;
            R.run_len = R.n;
        } else {
            R.width = (R.kmax - R.kmin) / R.nb + 1;
        }
    }
    if (R.mode == 2) R.width = static_cast<uint64_t>(R.imax - R.imin) / R.nb + 1;
    rr[r] = R;
}

template <bool L0>
__global__ void __launch_bounds__(RT) k_hist(const RankRange* rr, int nr, const double* c0, const double* c1,
                                            const ulonglong2* srec, uint32_t* hist) {
    const int r = range_of_tile(rr, nr, blockIdx.x);
    const RankRange R = rr[r];
    const uint32_t begin = (blockIdx.x - R.tile0) * RTILE;
    const uint32_t end = min(begin + RTILE, R.n);
    for (uint32_t i = begin + threadIdx.x; i < end; i += RT) {
        unsigned long long k;
        uint32_t id;
        bool fin;
        load_elem<L0>(R, i, c0, c1, srec, k, id, fin);
        atomicAdd(hist + R.bbase + bucket_of(R, k, id), 1u);
    }
}

// Exclusive scan of every range's bucket counts in three phases over chunks
// of SCH buckets (a range's bucket array may hold tens of millions of
// buckets): chunk sums, per-range scan of the chunk sums, chunk scans.
constexpr uint32_t SCH = 8192;
struct ScanChunk {
    uint32_t range, first;  // range index, first (range-local) bucket of the chunk
};

__global__ void __launch_bounds__(256) k_scan_sum(const RankRange* rr, const ScanChunk* ch, const uint32_t* hist,
                                                 uint32_t* csum) {
    const ScanChunk C = ch[blockIdx.x];
    const RankRange R = rr[C.range];
    const uint32_t end = min(C.first + SCH, R.nb);
    uint32_t v = 0;
    for (uint32_t b = C.first + threadIdx.x; b < end; b += blockDim.x) v += hist[R.bbase + b];
    v = __reduce_add_sync(0xffffffffu, v);
    __shared__ uint32_t s_w[8];
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; ++w) t += s_w[w];
        csum[blockIdx.x] = t;
    }
}

// one thread per range: exclusive scan over its (consecutive) chunks
__global__ void k_scan_off(int nr, const uint32_t* chunk0, const uint32_t* csum, uint32_t* coff) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nr) return;
    uint32_t run = 0;
    for (uint32_t c = chunk0[r]; c < chunk0[r + 1]; ++c) {
        coff[c] = run;
        run += csum[c];
    }
}

__global__ void __launch_bounds__(1024) k_scan_apply(const RankRange* rr, const ScanChunk* ch, const uint32_t* hist,
                                                    const uint32_t* coff, uint32_t* bstart, uint32_t* cursor,
                                                    Oversize* ov, uint32_t* ov_count, uint32_t ov_cap) {
    constexpr uint32_t PER = SCH / 1024;  // buckets per thread, consecutive
    const ScanChunk C = ch[blockIdx.x];
    const RankRange R = rr[C.range];
    const uint32_t b0 = C.first + threadIdx.x * PER;
    uint32_t c[PER], loc = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        c[k] = b0 + k < R.nb ? hist[R.bbase + b0 + k] : 0u;
        loc += c[k];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __shared__ uint32_t s_w[32];
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t z = s_w[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        s_w[lane] = z;
    }
    __syncthreads();
    uint32_t run = coff[blockIdx.x] + (w ? s_w[w - 1] : 0u) + x - loc;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const uint32_t b = b0 + k;
        if (b < R.nb) {
            bstart[R.bbase + b] = run;
            cursor[R.bbase + b] = run;
            if (c[k] > CAP) {
                const uint32_t slot = atomicAdd(ov_count, 1u);
                if (slot < ov_cap) ov[slot] = Oversize{C.range, run, c[k], 0u};
            }
        }
        run += c[k];
    }
}

template <bool L0>
__global__ void __launch_bounds__(RT) k_scatter(const RankRange* rr, int nr, const double* c0, const double* c1,
                                               const ulonglong2* srec, uint32_t* cursor, ulonglong2* drec) {
    // (key, index) records of 16 bytes: one scattered store per element (a
    // partial-sector write to a random address is the cost of this pass);
    // SU elements per thread in flight
    constexpr int SU = 4;
    const int r = range_of_tile(rr, nr, blockIdx.x);
    const RankRange R = rr[r];
    const uint32_t begin = (blockIdx.x - R.tile0) * RTILE;
    const uint32_t end = min(begin + RTILE, R.n);
    for (uint32_t i0 = begin + threadIdx.x; i0 < end; i0 += SU * RT) {
        unsigned long long k[SU];
        uint32_t id[SU], slot[SU];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
            const uint32_t i = i0 + u * RT;
            if (i < end) {
                bool fin;
                load_elem<L0>(R, i, c0, c1, srec, k[u], id[u], fin);
            }
        }
#pragma unroll
        for (int u = 0; u < SU; ++u)
            if (i0 + u * RT < end) slot[u] = atomicAdd(cursor + R.bbase + bucket_of(R, k[u], id[u]), 1u);
#pragma unroll
        for (int u = 0; u < SU; ++u)
            if (i0 + u * RT < end) drec[R.dst_base + slot[u]] = make_ulonglong2(k[u], id[u]);
    }
}

// One thread per element of the scattered range; buckets <= CAP are ranked
// by counting inside the bucket (L1-resident neighbours).
__global__ void __launch_bounds__(RT) k_rank(const RankRange* rr, int nr, const ulonglong2* drec,
                                            const uint32_t* hist, const uint32_t* bstart,
                                            uint64_t n_rows, unsigned long long* o_rp) {
    const int r = range_of_tile(rr, nr, blockIdx.x);
    const RankRange R = rr[r];
    const uint32_t begin = (blockIdx.x - R.tile0) * RTILE;
    const uint32_t end = min(begin + RTILE, R.n);
    for (uint32_t p = begin + threadIdx.x; p < end; p += RT) {
        const ulonglong2 me = drec[R.dst_base + p];
        const unsigned long long k = me.x;
        const uint32_t id = static_cast<uint32_t>(me.y);
        const uint32_t b = bucket_of(R, k, id);
        const uint32_t cnt = hist[R.bbase + b];
        if (cnt > CAP) continue;  // refined at the next level
        const uint32_t s = bstart[R.bbase + b];
        const ulonglong2* br = drec + R.dst_base + s;
        uint32_t lt, eq, pos;
        if (R.mode == 2) {
            uint32_t before = 0;
            for (uint32_t q = 0; q < cnt; ++q) before += static_cast<uint32_t>(br[q].y) < id;
            lt = R.run_start;
            eq = R.run_len;
            pos = R.lt_base + s + before;
        } else {
            uint32_t less = 0, same = 0, before = 0;
            for (uint32_t q = 0; q < cnt; ++q) {
                const ulonglong2 rq = br[q];
                const unsigned long long kq = rq.x;
                less += kq < k;
                const bool e = kq == k;
                same += e;
                before += e && (static_cast<uint32_t>(rq.y) < id);
            }
            lt = R.lt_base + s + less;
            eq = same;
            pos = lt + before;
        }
        const uint64_t o = static_cast<uint64_t>(R.col) * n_rows + R.out_base + id;
        o_rp[o] = pack_rank(2u * lt + eq + 1u, pos, R.mode == 2 ? pos == R.run_start : pos == lt);
    }
}

__global__ void k_ranks_to_u(const Seg* segs, int nseg, RankRef R, uint64_t n_rows, double* u1, double* u2) {
    const int m = seg_of_tile(segs, nseg, blockIdx.x);
    const Seg S = segs[m];
    const uint32_t begin = (blockIdx.x - S.tile0) * RTILE;
    const uint32_t end = min(begin + RTILE, S.n);
    const double scale = 1.0 / (static_cast<double>(S.n) + 1.0);  // pseudo_obs.hpp:53
    const bool rt = R.routed && R.routed[m];
    for (uint32_t i = begin + threadIdx.x; i < end; i += RT) {
        const uint64_t row = S.begin + i;
        uint32_t r1, r2;
        rank_pair(R, rt, nseg, m, n_rows, row, r1, r2);
        // pseudo_obs.hpp:59-60: avg = 0.5*((i+1)+(j+1)); u = avg*scale
        u1[row] = __dmul_rn(0.5 * static_cast<double>(r1), scale);
        u2[row] = __dmul_rn(0.5 * static_cast<double>(r2), scale);
    }
}

uint32_t tiles_of(uint64_t n) { return static_cast<uint32_t>((n + RTILE - 1) / RTILE); }

// ====================================================================
// Cluster path: one thread-block cluster ranks one (column, segment) with
// the whole segment held in the cluster's distributed shared memory.
//   1. each CTA loads its slice of the column (HBM, once), cluster-wide
//      min/max through DSMEM
//   2. value-linear split of [min, max] into CL contiguous value ranges
//      (one per CTA) x NBL local buckets; every CTA counts what it sends
//      to each peer; the CL x CL count matrix is read through DSMEM
//   3. every element's key is stored into its value-range owner's receive
//      buffer (one 8-byte DSMEM store); route[row] = (owner, receive slot)
//   4. each owner counting-sorts its elements into NBL local buckets and
//      ranks every element by counting inside its bucket; lt = elements in
//      lower value ranges + bucket start + #less; equal keys are ordered by
//      receive slot
//   5. results per receive slot (coalesced): r2 (u32) and the owner-local
//      sorted position with the run-start bit (u16); consumers read them
//      through route[row]
// HBM traffic per element: 8 B read; 4 B route + 4 B r2 + 2 B position
// written. A slice whose received count would overflow its buffer (heavily
// skewed data) or
// a non-finite range falls back to the global path.
constexpr int CT = 1024;  // threads per cluster CTA
#ifndef PCB_RANK_DBL
#define PCB_RANK_DBL 1
#endif
constexpr int EMAX = 16;         // slice elements per thread (slice <= 16K)
constexpr int QMAX = 16;         // received elements per thread (RCAP <= QMAX * CT)
constexpr int kMaxCluster = 16;
constexpr size_t kSmemLimit = 227 * 1024 - 8192;  // leave room for static shared memory

struct ClusterJob {
    uint64_t begin;
    uint32_t n, col, seg, pad;
};

struct ClusterPlan {
    int cl = 0;            // CTAs per cluster (0: no cluster path)
    uint32_t s = 0;        // max slice
    uint32_t rcap = 0;     // receive capacity per CTA
    uint32_t lg_nbl = 0;   // log2 local buckets per CTA
    size_t smem = 0;
    bool lean = false;     // 512-thread CTAs, two per SM (k_rank_cluster_t<512, true>)
};

inline bool getenv_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && v[0] && v[0] != '0';
}

__host__ __device__ inline uint32_t slice_of(uint64_t n, int cl) {
    return static_cast<uint32_t>(((n + cl - 1) / cl + 31) & ~31ull);
}

inline ClusterPlan plan_for(uint64_t nmax, int cl, bool lean = false) {
    ClusterPlan p;
    p.cl = cl;
    p.lean = lean;
    p.s = slice_of(nmax, cl);
    const uint32_t slack = std::max<uint32_t>(256u, static_cast<uint32_t>(5.5 * std::sqrt(static_cast<double>(p.s))));
    p.rcap = (p.s + slack + 31u) & ~31u;
    uint32_t lg = 1;
    while ((2u << lg) <= std::max<uint32_t>(2u, p.s)) ++lg;  // NBL = largest power of two <= S (>= 2)
    p.lg_nbl = lg;
    // per slot: key 8 + result 4 (aliased by the NBL u16 counters and the
    // slot's u16 local bucket during the local sort; NBL <= S < RCAP) + perm 2;
    // NBL+2 u16 bucket starts
    p.smem = static_cast<size_t>(p.rcap) * (lean ? 10 : 14) + (static_cast<size_t>(1u << lg) + 2) * 2 + 64;
    return p;
}

constexpr int kLeanT = 512;   // threads of a lean CTA
#ifndef PCB_RANK_ROWMAP_DEFAULT
#define PCB_RANK_ROWMAP_DEFAULT 0
#endif
constexpr int kRowMapDefault = PCB_RANK_ROWMAP_DEFAULT;
constexpr int kLeanQ = 18;    // received elements per lean thread
constexpr size_t kLeanSmem = 112 * 1024 - 4096;  // two per SM beside their static shared memory

inline ClusterPlan plan_cluster(uint64_t nmax) {
    int forced = 0;
    if (const char* v = std::getenv("PCB_RANK_CL")) forced = std::atoi(v);
    // lean (two CTAs per SM, opt-in with PCB_RANK_LEAN=1): measured slower at
    // C5 (16-CTA clusters, 42.7 vs 38.2 ms per family) — kept as a variant
    if (getenv_flag("PCB_RANK_LEAN"))
        for (int cl = 2; cl <= kMaxCluster; ++cl) {
            if (forced && cl != forced) continue;
            ClusterPlan p = plan_for(nmax, cl, true);
            if (p.rcap <= static_cast<uint32_t>(kLeanQ * kLeanT) && p.smem <= kLeanSmem &&
                p.s <= static_cast<uint32_t>(EMAX * kLeanT))
                return p;
        }
    for (int cl = 1; cl <= kMaxCluster; ++cl) {
        if (forced && cl != forced) continue;
        ClusterPlan p = plan_for(nmax, cl);
        if (p.rcap <= static_cast<uint32_t>(QMAX * CT) && p.rcap < 32768 && p.smem <= kSmemLimit && p.s <= static_cast<uint32_t>(EMAX * CT) &&
            (static_cast<uint64_t>(cl) << p.lg_nbl) <= (1u << 20))
            return p;
    }
    return ClusterPlan{};
}

// 8-byte store into CTA `rank`'s shared memory at this CTA's shared address
// `saddr` (mapa + st.shared::cluster: 32-bit addressing, no generic window)
__device__ __forceinline__ void dsmem_st64(uint32_t saddr, uint32_t rank, unsigned long long v) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(saddr), "r"(rank));
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(v) : "memory");
}

__device__ __forceinline__ void dsmem_st32(uint32_t saddr, uint32_t rank, uint32_t v) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(saddr), "r"(rank));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}

// Quantile-knot map for skewed blocks (the cluster kernel's second pass):
// kn[0..nk) sorted knot keys with kn[0] <= k, cm[j] = elements before
// interval j (exact, cluster-wide). Interval i = [kn[i], kn[i+1]); the last
// one holds the keys equal to the maximum. Explicit roundings: every CTA
// computes the same position for the same key.
// Knot tables are stored with one pad slot per 16 keys (kpad), so the
// search's power-of-two strides do not all land in one shared-memory bank.
__device__ __forceinline__ uint32_t kpad(uint32_t i) { return i + (i >> 4); }
// Intervals of N keys at once (kn padded with ~0ull, above every finite key,
// to 2^LG entries): a fixed-step search, step-major so the N chains of
// dependent shared loads overlap. Interval = (knots <= k) - 1, >= 0 when kn[0] <= k.
template <int LG, int N>
__device__ __forceinline__ void qsearch(const unsigned long long* kn, const unsigned long long (&k)[N],
                                        uint32_t (&iv)[N]) {
    uint32_t p[N];
#pragma unroll
    for (int u = 0; u < N; ++u) p[u] = 0;
#pragma unroll
    for (uint32_t h = 1u << (LG - 1); h > 0; h >>= 1)
#pragma unroll
        for (int u = 0; u < N; ++u)
            if (kn[kpad(p[u] + h - 1)] <= k[u]) p[u] += h;
#pragma unroll
    for (int u = 0; u < N; ++u) iv[u] = p[u] ? p[u] - 1 : 0;
}
// Interpolated position g in [0, N] of key k in interval i: cm[i] plus
// min(c_i, (k - kn[i]) * sl[i]), sl[i] = c_i / (kn[i+1] - kn[i]) in halved
// values (0 for the last, maximum-equal interval). Monotone in k across
// intervals (g <= cm[i+1] inside interval i).
__device__ __forceinline__ double qpos(unsigned long long k, uint32_t i, const unsigned long long* kn,
                                       const uint32_t* cm, const double* sl) {
    const double v = __dmul_rn(0.5, key_value(k)), q0 = __dmul_rn(0.5, key_value(kn[kpad(i)]));
    const double c = static_cast<double>(cm[i + 1] - cm[i]);
    const double t = fmin(c, fmax(0.0, __dmul_rn(__dsub_rn(v, q0), sl[i])));  // NaN (0 * inf) -> 0
    return __dadd_rn(static_cast<double>(cm[i]), t);
}
__device__ __forceinline__ uint32_t qbucket(double g, double qs, uint32_t nbtot) {
    return min(nbtot - 1u, static_cast<uint32_t>(__dmul_rn(g, qs)));
}

// value-linear global bucket, clamped at both ends (the conversion saturates
// below 0 and maps NaN to 0); monotone in the value. Senders bucket the value
// itself, owners the received key: key_value(order_key(v)) is v (+0 for -0,
// the same t), so both agree bit for bit.
// t = (v/2 - hm) * scale with explicit roundings (v/2 is exact), so the
// owner decision (cbucket_v) and the fine key of the FK kernel agree bit for bit
__device__ __forceinline__ double cmap_t(double v, double hm, double scale) {
    return __dmul_rn(__dsub_rn(__dmul_rn(0.5, v), hm), scale);
}
__device__ __forceinline__ uint32_t cbucket_v(double v, double hm, double scale, uint32_t nbtot) {
    return min(__double2uint_rz(cmap_t(v, hm, scale)), nbtot - 1u);
}
__device__ __forceinline__ uint32_t cbucket(unsigned long long k, double hm, double scale, uint32_t nbtot) {
    return cbucket_v(key_value(k), hm, scale, nbtot);
}

// Same scan over NBL u16 counters packed two per word (`cw`); writes the u16
// starts (start[n] = total) and turns cw into cursors (packed starts).
template <int CTT>
__device__ void block_scan_excl_u16(uint32_t* cw, uint16_t* start, uint32_t n, uint32_t* s_w) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t nw = n / 2;
    const uint32_t per = (nw + CTT - 1) / CTT;
    const uint32_t b0 = min(nw, tid * per), b1 = min(nw, b0 + per);
    uint32_t loc = 0;
    for (uint32_t q = b0; q < b1; ++q) loc += (cw[q] & 0xffffu) + (cw[q] >> 16);
    uint32_t x = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t z = lane < (CTT / 32) ? s_w[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        if (lane < (CTT / 32)) s_w[lane] = z;
    }
    __syncthreads();
    uint32_t run = (wid ? s_w[wid - 1] : 0u) + x - loc;
    for (uint32_t q = b0; q < b1; ++q) {
        const uint32_t w = cw[q];
        const uint32_t s0 = run, s1 = run + (w & 0xffffu);
        start[2 * q] = static_cast<uint16_t>(s0);
        start[2 * q + 1] = static_cast<uint16_t>(s1);
        cw[q] = s0 | (s1 << 16);
        run = s1 + (w >> 16);
    }
    if (tid == CTT - 1) start[n] = static_cast<uint16_t>(run);
    __syncthreads();
}

// CTT threads per CTA. LEAN (512 threads, 2 CTAs per SM): no per-slot result
// array — the local sort keeps (bucket, index) in registers and the ranking
// recomputes the bucket from the key; results are staged in the receive
// buffer once the ranking is done — so a CTA needs 10 B per slot.
//
// FK (opt-in variant, PCB_RANK_FK=1): owners receive 32-bit FINE keys instead of the
// 64-bit order keys. The sender knows the global value-linear map t (the
// owner is floor(t) >> lg_nbl), and the fine key is the position inside the
// owner's range at 2^(32 - lg_nbl) steps per local bucket:
// fk = sat_u32((t - owner_base) * 2^(32-lg)), exact (t has 2^-36 resolution)
// and monotone, so the local bucket is fk's top bits and ranking compares
// 32-bit words. Distinct values that share a fine key, and true ties, are
// resolved from the full order keys, which the sender also writes per
// receive slot to global memory (`kside`, L2-resident; read only for
// equal-fine-key pairs). Halves the DSMEM bytes of the all-to-all and frees
// shared memory for up to 4x the local buckets (NBL up to 32768). Measured
// no faster at C5 (launch_rank_cluster), kept for the record.
template <int CTT, bool LEAN, bool QUANT = false, bool FK = false>
__global__ void __launch_bounds__(CTT, LEAN ? 2 : 1) k_rank_cluster_t(const ClusterJob* jobs, const double* c0, const double* c1,
                                                       uint64_t n_rows, unsigned long long* rp, uint32_t* route,
                                                       uint32_t* r2s_g, uint16_t* posl_g, uint32_t* ocnt, uint32_t K,
                                                       int32_t* fb,
                                                       int32_t* bad, int CL, uint32_t RCAP, uint32_t lg_nbl,
                                                       int tail, unsigned long long* prof, uint32_t njobs,
                                                       uint32_t pf, unsigned long long* kside, int rowmap) {
    namespace cg = cooperative_groups;
    constexpr int QM = LEAN ? 18 : QMAX;  // received elements per thread (RCAP <= QM * CTT)
    // DBL: the receive buffer holds the values themselves (-0 canonicalised to
    // +0 by adding +0.0) instead of their order keys. Every value reaching it
    // is finite (validate_data runs before the send), so double comparisons
    // order them exactly as the keys do (one DSETP instead of two 32-bit
    // compares each for < and ==), and the owner's bucket needs no key_value.
    constexpr bool DBL = PCB_RANK_DBL && !QUANT && !FK && !LEAN;
    long long t_prev = clock64();
    auto mark = [&](int k) {  // optional phase timing (PCB_RANK_PROFILE): thread 0's clock deltas
        if (prof && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(prof + k, static_cast<unsigned long long>(t - t_prev));
            t_prev = t;
        }
    };
    cg::cluster_group cluster = cg::this_cluster();
    const int r = static_cast<int>(cluster.block_rank());
    const uint32_t jid = blockIdx.x / CL;
    const ClusterJob J = jobs[jid];
    const double* x = (J.col ? c1 : c0) + J.begin;
    const uint32_t S = slice_of(J.n, CL);  // 32-aligned slices: a warp's 32 rows share one send pass
    const uint32_t a = min(J.n, r * S), e = min(J.n, a + S);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t NBL = 1u << lg_nbl;

    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* recv_key = reinterpret_cast<unsigned long long*>(smem);
    const double* const recv_dbl = reinterpret_cast<const double*>(smem);  // DBL: the same slots as values
    // FK: [fine keys, 4 B per slot | region B: the staged slice, after the send outw / lhs / perm]
    uint32_t* const recv_fk = reinterpret_cast<uint32_t*>(smem);
    unsigned char* const regB = smem + ((static_cast<size_t>(RCAP) * 4 + 15) & ~static_cast<size_t>(15));
    // LEAN: results staged in the receive buffer after the ranking
    uint32_t* outw = FK ? reinterpret_cast<uint32_t*>(regB)
                        : (LEAN ? reinterpret_cast<uint32_t*>(recv_key) : reinterpret_cast<uint32_t*>(recv_key + RCAP));
    uint16_t* lhs = (LEAN && !FK) ? reinterpret_cast<uint16_t*>(recv_key + RCAP)
                                  : reinterpret_cast<uint16_t*>(outw + RCAP);  // NBL u16 counts -> NBL+1 starts (+1 pad)
    uint32_t* lhw = reinterpret_cast<uint32_t*>(lhs);             // the counts, two per word
    uint16_t* perm = lhs + NBL + 2;

    // the slice is staged into the (not yet used) receive buffer by one bulk
    // async copy; the sample and the cluster-wide extremes overlap it
    __shared__ __align__(8) unsigned long long s_mbar;
    const uint64_t g_lo = reinterpret_cast<uint64_t>(x + a) & ~15ull;
    const uint32_t x_off = static_cast<uint32_t>((reinterpret_cast<uint64_t>(x + a) - g_lo) >> 3);
    const uint64_t g_hi = (reinterpret_cast<uint64_t>(x + e) + 15ull) & ~15ull;
    const bool staged = e > a;
    // tail mode: the slice sits after the receive buffer (where the sort's
    // arrays go later), so it stays readable while peers fill the buffer
    unsigned char* stage_at = FK ? regB : (tail ? smem + static_cast<size_t>(RCAP) * 8 : smem);
    const double* xs = reinterpret_cast<const double*>(stage_at) + x_off - a;  // xs[i] == x[i] for i in [a, e)
    if (tid == 0 && staged) {
        const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar));
        const uint32_t bytes = static_cast<uint32_t>(g_hi - g_lo);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(stage_at))),
            "l"(g_lo), "r"(bytes), "r"(mb)
            : "memory");
    }
    // the job pf positions ahead runs on the next wave of clusters: pull this
    // CTA's slice of it into L2 now, so its staging copy and sample read L2
    if (tid == 32 && pf && jid + pf < njobs) {
        const ClusterJob J2 = jobs[jid + pf];
        const uint32_t S2 = slice_of(J2.n, CL);
        const uint32_t a2 = min(J2.n, r * S2), e2 = min(J2.n, a2 + S2);
        if (e2 > a2) {
            const double* x2 = (J2.col ? c1 : c0) + J2.begin;
            const uint64_t p_lo = reinterpret_cast<uint64_t>(x2 + a2) & ~15ull;
            const uint64_t p_hi = (reinterpret_cast<uint64_t>(x2 + e2) + 15ull) & ~15ull;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p_lo), "r"(static_cast<uint32_t>(p_hi - p_lo))
                         : "memory");
        }
    }
    auto wait_slice = [&]() {
        if (!staged) return;
        const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar));
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra WAIT_%=;\n}" ::"r"(mb)
            : "memory");
    };

    __shared__ unsigned long long s_k[2][(CTT / 32)];
    __shared__ unsigned long long s_rmin, s_rmax, s_gmin, s_gmax;  // s_rmin/s_rmax are read by peers
    __shared__ int s_bad, s_gbad, s_over;
    __shared__ uint32_t s_wc[(CTT / 32)][kMaxCluster];  // per-warp counts -> per-warp send cursors
    __shared__ uint32_t s_cnt[kMaxCluster];         // this CTA's sends per owner (read by peers)
    __shared__ uint32_t s_mat[kMaxCluster * kMaxCluster];
    __shared__ uint32_t s_off[kMaxCluster], s_total, s_base;
    __shared__ uint32_t s_w[(CTT / 32)];

    // ---- 1. bucket-map range from a strided sample (one element per thread).
    // Any monotone map gives exact ranks (values outside the sampled range
    // clamp into the end buckets); the range only sets the load balance. A
    // constant-looking sample triggers an exact pass (constant columns).
    unsigned long long kmn = ~0ull, kmx = 0ull;
    const uint32_t len = e - a;
    if (len > 0) {
        const unsigned long long kk = order_key(x[a + static_cast<uint32_t>((static_cast<uint64_t>(tid) * len) / CTT)]);
        kmn = kk;
        kmx = kk;
    }
    auto cta_extremes = [&]() {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
            kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
        }
        if (lane == 0) {
            s_k[0][wid] = kmn;
            s_k[1][wid] = kmx;
        }
        __syncthreads();
        if (wid == 0) {
            kmn = s_k[0][lane];
            kmx = s_k[1][lane];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
                kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
            }
            if (lane == 0) {
                s_rmin = kmn;
                s_rmax = kmx;
            }
        }
    };
    auto cluster_extremes = [&]() {  // lane q reads CTA q's extremes (parallel DSMEM loads)
        if (wid == 0) {
            unsigned long long gmn = ~0ull, gmx = 0ull;
            if (lane < CL) {
                gmn = *cluster.map_shared_rank(&s_rmin, lane);
                gmx = *cluster.map_shared_rank(&s_rmax, lane);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                gmn = min(gmn, __shfl_xor_sync(0xffffffffu, gmn, o));
                gmx = max(gmx, __shfl_xor_sync(0xffffffffu, gmx, o));
            }
            if (lane == 0) {
                s_gmin = gmn;
                s_gmax = gmx;
            }
        }
        __syncthreads();
    };
    if (tid == 0) s_bad = 0;
    for (int q = tid; q < (CTT / 32) * kMaxCluster; q += CTT) (&s_wc[0][0])[q] = 0u;
    cta_extremes();
    mark(11);
    cluster.sync();
    mark(0);
    cluster_extremes();
    if (s_gmin == s_gmax) {  // exact extremes over every element (all CTAs agree on taking this branch)
        kmn = ~0ull;
        kmx = 0ull;
        for (uint32_t i = a + tid; i < e; i += CTT) {
            const unsigned long long kk = order_key(x[i]);
            kmn = min(kmn, kk);
            kmx = max(kmx, kk);
        }
        __syncthreads();
        cluster.sync();  // everyone has read the sample extremes
        cta_extremes();
        cluster.sync();
        cluster_extremes();
    }
    const double vmin = key_value(s_gmin), vmax = key_value(s_gmax);
    const double hm = 0.5 * vmin;
    const uint32_t nbtot = static_cast<uint32_t>(CL) << lg_nbl;
    const double scale = static_cast<double>(nbtot) / (0.5 * vmax - hm);
    const bool constant = s_gmin == s_gmax;
    if (constant || !(isfinite(scale) && scale > 0.0 && isfinite(hm))) {
        wait_slice();  // no CTA exits with its bulk copy in flight
        if (constant && !isfinite(vmin)) {
            if (r == 0 && tid == 0) {
                bad[J.seg] = 1;
                fb[jid] = 2;  // handled, no route
            }
        } else if (constant) {  // one tie run: avg rank (n+1)/2 for all; written by the host's pass (fb 3)
            if (r == 0 && tid == 0) fb[jid] = 3;
        } else if (r == 0 && tid == 0) {
            fb[jid] = 1;
        }
        cluster.sync();  // peers may still be reading this CTA's shared memory
        return;
    }

    // ---- 2. per-warp counts of what this CTA sends to each value-range owner.
    // The split is value-linear over [min, max] (balanced for uniform-like
    // data, e.g. pseudo-observations). If an owner would overflow its receive
    // buffer (skewed raw marginals: normal, exponential, heavy tails), the
    // block is relaunched (fb 4) through the QUANT variant, which splits by
    // exact quantile knots; only if that still overflows does the block take
    // the global path.
    auto kclamp = [&](unsigned long long k) { return k < s_gmin ? s_gmin : (k > s_gmax ? s_gmax : k); };
    constexpr uint32_t NKMAX = 512;  // quantile knots (sample + exact extremes), < NKMAX used
    constexpr uint32_t SUBK = 128;   // an owner's share of the knot table (< SUBK - 1 intervals)
    // quantile mode tables in the receive buffer (idle until the send phase),
    // in u64 slots: [0,512) own sample (read by peers) | [512,1536) gathered
    // sample / sort exchange | [1536,2080) knots (kpad) | [2080,2336) own
    // interval counts (u32, read by peers) | [2336,2593) cums (u32) |
    // [2600,3112) slopes (f64) | [QTAB, +S/4) interval id per element (u16).
    // The owner's share (knots, cums, slopes) sits in the last SUBSLOTS
    // slots, which the send never reaches in this mode (totals <= RCAP - SUBSLOTS).
    constexpr uint32_t SUBSLOTS = (SUBK + SUBK / 16) + (SUBK / 2 + 1) + SUBK;
    constexpr uint32_t QTAB = 3200;
    __shared__ uint32_t s_ilo[kMaxCluster], s_ihi[kMaxCluster], s_qbad;
    __shared__ double s_qs;  // nbtot / N
    constexpr bool qmode = QUANT;
    unsigned long long* const knot = recv_key + 1536;
    uint32_t* const cum = reinterpret_cast<uint32_t*>(recv_key + 2336);
    double* const slope = reinterpret_cast<double*>(recv_key + 2600);
    unsigned long long* const sk = recv_key + (RCAP - SUBSLOTS);  // owner share
    uint32_t* const sc = reinterpret_cast<uint32_t*>(sk + SUBK + SUBK / 16);
    double* const ssl = reinterpret_cast<double*>(sk + SUBK + SUBK / 16 + SUBK / 2 + 1);
    uint16_t* const ivs = reinterpret_cast<uint16_t*>(recv_key + QTAB);  // interval id per slice element
    uint32_t bk[EMAX / 8];  // owner (4 bits) per element
    wait_slice();  // the mbarrier was initialised before the first __syncthreads
    if constexpr (QUANT) {  // relaunch of the blocks the value-linear split could not balance
        if (!tail || RCAP < QTAB + (S + 3) / 4 + SUBSLOTS) {  // no room for the tables: global path
            if (r == 0 && tid == 0) fb[jid] = 1;
            cluster.sync();
            return;
        }
        // ---- skewed block: equal-count owners from quantile knots. Knots =
        // exact extremes + a strided sample of every slice, sorted identically
        // in every CTA; exact cluster-wide counts per knot interval; positions
        // interpolate linearly inside an interval (~N/NK elements each), so
        // owners balance to within a few elements and local buckets stay
        // ~N/nbtot deep whatever the marginal.
        const uint32_t m = (NKMAX - 3) / CL;  // sample per CTA (knots < NKMAX for the fixed-step search)
        const uint32_t len = e - a;
        kmn = ~0ull;
        kmx = 0ull;
        for (uint32_t i = a + tid; i < e; i += CTT) {
            const unsigned long long kk = order_key(xs[i]);
            kmn = min(kmn, kk);
            kmx = max(kmx, kk);
        }
        if (tid < m) recv_key[tid] = len ? order_key(xs[a + static_cast<uint32_t>((static_cast<uint64_t>(tid) * len) / m)])
                                         : 0ull;  // empty slice: clamped to the minimum below
        uint32_t* const hc = reinterpret_cast<uint32_t*>(recv_key + 2080);
        for (uint32_t q = tid; q < NKMAX; q += CTT) hc[q] = 0u;
        if (tid < CL) {
            s_ilo[tid] = ~0u;
            s_ihi[tid] = 0u;
        }
        if (tid == 0) s_qbad = 0;
        cta_extremes();  // exact slice extremes -> s_rmin/s_rmax
        cluster.sync();  // samples and exact extremes visible
        cluster_extremes();
        const uint32_t ns = m * CL, nk = ns + 2;
        unsigned long long* const raw = recv_key + 512;
        for (uint32_t j = tid; j < ns; j += CTT)
            raw[j] = kclamp(*cluster.map_shared_rank(recv_key + j % m, j / m));
        __syncthreads();
        {  // bitonic sort of the ns < NKMAX samples, one per thread (pads sort last)
            unsigned long long v = static_cast<uint32_t>(tid) < ns ? raw[tid] : ~0ull;
            unsigned long long* const xb = raw;  // exchange buffer (each thread read only its own slot)
            for (uint32_t kb = 2; kb <= NKMAX; kb <<= 1)  // threads >= NKMAX sort pads alongside
                for (uint32_t j = kb >> 1; j > 0; j >>= 1) {
                    unsigned long long pv;
                    if (j >= 32) {
                        xb[tid] = v;
                        __syncthreads();
                        pv = xb[tid ^ j];
                        __syncthreads();
                    } else {
                        pv = __shfl_xor_sync(0xffffffffu, v, j);
                    }
                    const bool up = (tid & kb) == 0, low = (tid & j) == 0;
                    v = (low == up) ? min(v, pv) : max(v, pv);
                }
            if (tid + 1 < static_cast<int>(NKMAX)) knot[kpad(1 + tid)] = v;  // knot[1 + ns ..]: pads (~0ull)
        }
        __syncthreads();
        if (tid == 0) {
            knot[0] = s_gmin;
            knot[kpad(nk - 1)] = s_gmax;
        }
        __syncthreads();
        mark(6);
        for (uint32_t i0 = a + tid; i0 < e; i0 += 8 * CTT) {  // this slice's count per interval
            unsigned long long kk[8];
            uint32_t iv[8];
    #pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = i0 + u * CTT;
                kk[u] = i < e ? order_key(xs[i]) : 0ull;
            }
            qsearch<9>(knot, kk, iv);
    #pragma unroll
            for (int u = 0; u < 8; ++u)
                if (i0 + u * CTT < e) {
                    ivs[i0 + u * CTT - a] = static_cast<uint16_t>(iv[u]);
                    atomicAdd(hc + iv[u], 1u);
                }
        }
        mark(8);
        cluster.sync();  // every CTA's interval counts are final
        mark(9);
        {
            uint32_t c = 0;  // thread t: interval t, summed over the cluster (loads in flight together)
            if (static_cast<uint32_t>(tid) < nk)
                for (int q = 0; q < CL; ++q) c += *cluster.map_shared_rank(hc + tid, q);
            uint32_t x2 = c;
    #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x2, o);
                if (lane >= o) x2 += y;
            }
            if (lane == 31) s_w[wid] = x2;
            __syncthreads();
            if (wid == 0) {
                uint32_t z = lane < (CTT / 32) ? s_w[lane] : 0u;
    #pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
                    if (lane >= o) z += y;
                }
                if (lane < (CTT / 32)) s_w[lane] = z;
            }
            __syncthreads();
            const uint32_t incl = (wid ? s_w[wid - 1] : 0u) + x2;
            if (static_cast<uint32_t>(tid) < nk) cum[tid + 1] = incl;
            if (tid == 0) cum[0] = 0u;
        }
        __syncthreads();
        const double qs = static_cast<double>(nbtot) / static_cast<double>(cum[nk]);
        if (tid == 0) s_qs = qs;
        if (static_cast<uint32_t>(tid) < nk) {  // interval slopes (halved values; 0 for the last)
            const uint32_t cc = cum[tid + 1] - cum[tid];
            double sv = 0.0;
            if (static_cast<uint32_t>(tid) + 1 < nk && cc) {
                const double q0 = __dmul_rn(0.5, key_value(knot[kpad(tid)]));
                const double q1 = __dmul_rn(0.5, key_value(knot[kpad(tid + 1)]));
                sv = __ddiv_rn(static_cast<double>(cc), __dsub_rn(q1, q0));  // +inf for an underflowed width
            }
            slope[tid] = sv;
        }
        if (static_cast<uint32_t>(tid) < nk) {  // owners that interval tid can reach
            const uint32_t o0 = qbucket(static_cast<double>(cum[tid]), qs, nbtot) >> lg_nbl;
            const uint32_t o1 = qbucket(static_cast<double>(cum[tid + 1]), qs, nbtot) >> lg_nbl;
            for (uint32_t o = o0; o <= o1; ++o) {
                atomicMin(&s_ilo[o], static_cast<uint32_t>(tid));
                atomicMax(&s_ihi[o], static_cast<uint32_t>(tid));
            }
        }
        __syncthreads();
        if (tid < CL && s_ilo[tid] != ~0u && s_ihi[tid] - s_ilo[tid] + 1 > SUBK - 2) s_qbad = 1;
        __syncthreads();
        mark(10);
        if (s_qbad) {  // same decision in every CTA (same tables)
            if (r == 0 && tid == 0) fb[jid] = 1;
            cluster.sync();
            mark(2);
            return;
        }
        if (s_ilo[r] != ~0u) {  // this owner's share: knots ilo.., cums ilo..ihi+1
            const uint32_t ilo = s_ilo[r], nint = s_ihi[r] - ilo + 1;
            for (uint32_t q = tid; q < SUBK; q += CTT) {
                sk[kpad(q)] = q <= nint && ilo + q < nk ? knot[kpad(ilo + q)] : ~0ull;
                if (q <= nint) sc[q] = cum[ilo + q];
                ssl[q] = q < nint ? slope[ilo + q] : 0.0;
            }
        }
        for (int q = tid; q < (CTT / 32) * kMaxCluster; q += CTT) (&s_wc[0][0])[q] = 0u;
        __syncthreads();
        mark(7);
    }
    // Element k of this thread. rowmap: warp w owns the contiguous rows
    // [a + w*CW, a + (w+1)*CW) of the slice, 32 per step, so the per-warp
    // send cursors hand each owner its slots in ROW order across the whole
    // slice: the consumers' route gathers and scatters (prepare, variance
    // passes 1 and 3) then see long runs of consecutive slots for
    // consecutive rows (full L2 sectors), and tie runs are ordered by row like
    // the reference's stable sort. Otherwise rows a + k*CTT + tid.
    const uint32_t CW = 32u * ((S + CTT - 1) / CTT);
    auto ei = [&](int k) -> uint32_t {
        if (!rowmap) return a + k * CTT + tid;
        const uint32_t o = static_cast<uint32_t>(k) * 32u + lane;
        return o < CW ? a + wid * CW + o : e;
    };
#pragma unroll
    for (int k = 0; k < EMAX / 8; ++k) bk[k] = 0u;
    bool fin = true;
#pragma unroll
    for (int k = 0; k < EMAX; ++k) {
        const uint32_t i = ei(k);
        if (i < e) {
            const double v = xs[i];
            fin &= isfinite(v);
            const uint32_t d = (qmode ? qbucket(qpos(order_key(v), ivs[i - a], knot, cum, slope), s_qs, nbtot)
                                      : cbucket_v(v, hm, scale, nbtot)) >> lg_nbl;
            bk[k >> 3] |= d << ((k & 7) * 4);
        }
    }
#pragma unroll
    for (int k = 0; k < EMAX; ++k)  // the counts after all the (independent) owner lookups
        if (ei(k) < e) atomicAdd(&s_wc[wid][(bk[k >> 3] >> ((k & 7) * 4)) & 0xfu], 1u);
    if (!__syncthreads_and(fin) && tid == 0) s_bad = 1;  // validate_data (pseudo_obs.hpp:34-36)
    if (tid < CL) {  // totals per owner, and per-warp exclusive bases
        uint32_t run = 0;
        for (int w = 0; w < (CTT / 32); ++w) {
            const uint32_t c = s_wc[w][tid];
            s_wc[w][tid] = run;
            run += c;
        }
        s_cnt[tid] = run;
    }
    cluster.sync();
    mark(1);
    if (tid < CL * CL) s_mat[tid] = *cluster.map_shared_rank(&s_cnt[tid % CL], tid / CL);  // [src][dst]
    if (wid == 1) {
        const int gb = __any_sync(0xffffffffu, lane < CL && *cluster.map_shared_rank(&s_bad, lane) != 0);
        if (lane == 0) s_gbad = gb;
    }
    __syncthreads();
    if (s_gbad) {
        if (r == 0 && tid == 0) {
            bad[J.seg] = 1;
            fb[jid] = 2;
        }
        cluster.sync();
        return;
    }
    const uint32_t cap = qmode ? RCAP - SUBSLOTS : RCAP;
    if (wid == 0) {  // lane d: owner d's receive total and this CTA's offset in it
        uint32_t col = 0, mine = 0;
        if (lane < CL)
            for (int q = 0; q < CL; ++q) {
                const uint32_t v = s_mat[q * CL + lane];
                col += v;
                if (q < r) mine += v;
            }
        if (lane < CL) s_off[lane] = mine;
        const bool over = __any_sync(0xffffffffu, lane < CL && col > cap);
        uint32_t below = lane < r ? col : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
        const uint32_t total = __shfl_sync(0xffffffffu, col, r);
        if (lane == 0) {
            s_total = total;
            s_base = below;
            s_over = over;
        }
    }
    __syncthreads();
    if (s_over) {  // QUANT kernel: the global path takes the block; otherwise the quantile relaunch if it fits
        if (r == 0 && tid == 0)
            fb[jid] = (!QUANT && !LEAN && tail && RCAP >= QTAB + (S + 3) / 4 + SUBSLOTS) ? 4 : 1;
        cluster.sync();
        mark(2);
        return;
    }
    for (int q = tid; q < (CTT / 32) * CL; q += CTT) s_wc[q / CL][q % CL] += s_off[q % CL];
    __syncthreads();

    // ---- 3. scatter keys to the owners (one 8-byte DSMEM store per element).
    // The owner never needs the row: its outputs are written per receive slot
    // and the row finds them through route[row] = (owner, slot).
    constexpr int SB = 8;  // slice reloads in flight per thread (L2 hits)
    const uint32_t recv_sa = static_cast<uint32_t>(__cvta_generic_to_shared(recv_key));
    uint32_t* const route_j = route + static_cast<uint64_t>(J.col) * n_rows + J.begin;
    if constexpr (FK) {
        const double P = static_cast<double>(1ull << (32 - lg_nbl));
        unsigned long long* const kb = kside + (static_cast<uint64_t>(J.col) * K + J.seg) * CL * RCAP;
#pragma unroll
        for (int k = 0; k < EMAX; ++k) {
            const uint32_t i = ei(k);
            if (i < e) {
                const double v = xs[i];
                const uint32_t d = (bk[k >> 3] >> ((k & 7) * 4)) & 0xfu;
                const double t = cmap_t(v, hm, scale);
                const uint32_t fk = __double2uint_rz(fma(t, P, -static_cast<double>(d << lg_nbl) * P));
                const uint32_t slot = atomicAdd(&s_wc[wid][d], 1u);
                route_j[i] = (d << 16) | slot;
                kb[d * RCAP + slot] = order_key(v);
                dsmem_st32(recv_sa + slot * 4u, d, fk);
            }
        }
    } else if (tail) {
#pragma unroll
      for (int k = 0; k < EMAX; ++k) {
        const uint32_t i = ei(k);
        if (i < e) {
            const unsigned long long kk = DBL ? static_cast<unsigned long long>(__double_as_longlong(__dadd_rn(xs[i], 0.0)))
                                              : order_key(xs[i]);
            const uint32_t d = (bk[k >> 3] >> ((k & 7) * 4)) & 0xfu;
            const uint32_t slot = atomicAdd(&s_wc[wid][d], 1u);
            route_j[i] = (d << 16) | slot;
            dsmem_st64(recv_sa + slot * 8u, d, kk);
        }
      }
    } else
#pragma unroll
    for (int h = 0; h < EMAX; h += SB) {
      if (rowmap ? (a + wid * CW + h * 32u >= e || static_cast<uint32_t>(h) * 32u >= CW) : (a + h * CTT >= e)) break;
      double xv[SB];
#pragma unroll
      for (int k = 0; k < SB; ++k) {
        const uint32_t i = ei(h + k);
        xv[k] = i < e ? x[i] : 0.0;
      }
#pragma unroll
      for (int kk2 = 0; kk2 < SB; ++kk2) {
        const int k = h + kk2;
        const uint32_t i = ei(k);
        if (i < e) {
            const unsigned long long kk = DBL ? static_cast<unsigned long long>(__double_as_longlong(__dadd_rn(xv[kk2], 0.0)))
                                              : order_key(xv[kk2]);
            const uint32_t d = (bk[k >> 3] >> ((k & 7) * 4)) & 0xfu;
            const uint32_t slot = atomicAdd(&s_wc[wid][d], 1u);
            route_j[i] = (d << 16) | slot;
            dsmem_st64(recv_sa + slot * 8u, d, kk);
        }
      }
    }
    cluster.sync();  // every receive buffer is complete; no DSMEM access after this point
    mark(3);

    // ---- 4. local counting sort into NBL buckets (the sender's bucket map,
    // recomputed from the key)
    const uint32_t T = s_total, base = s_base;
    const uint32_t lmask = NBL - 1u;
    for (uint32_t q = tid; q <= NBL / 2; q += CTT) lhw[q] = 0u;
    __syncthreads();
    // the counting atomic's old value is the element's index inside its bucket:
    // outw[j] = bucket | index << 14 (NBL <= 16384), so the placement needs no second atomic
    uint32_t keep[QM];  // LEAN: (bucket | index) of slot tid + k*CTT, then the ranking's results
    const uint32_t fk_sh = 32 - lg_nbl;  // FK: local bucket = the fine key's top lg_nbl bits
    if constexpr (FK) {
        for (uint32_t j = tid; j < T; j += CTT) {
            const uint32_t lb = recv_fk[j] >> fk_sh;
            const uint32_t sh = (lb & 1) * 16;
            const uint32_t idx = (atomicAdd(lhw + (lb >> 1), 1u << sh) >> sh) & 0xffffu;
            outw[j] = lb | (idx << 15);
        }
        __syncthreads();
        block_scan_excl_u16<CTT>(lhw, lhs, NBL, s_w);
        for (uint32_t j = tid; j < T; j += CTT) {
            const uint32_t w = outw[j];
            perm[lhs[w & 0x7fffu] + (w >> 15)] = static_cast<uint16_t>(j);
        }
    } else if constexpr (LEAN) {
#pragma unroll
        for (int k2 = 0; k2 < QM; ++k2) {
            const uint32_t j = tid + k2 * CTT;
            if (j >= T) break;
            const uint32_t lb = cbucket(recv_key[j], hm, scale, nbtot) & lmask, sh = (lb & 1) * 16;
            keep[k2] = lb | (((atomicAdd(lhw + (lb >> 1), 1u << sh) >> sh) & 0xffffu) << 14);
        }
        __syncthreads();
        block_scan_excl_u16<CTT>(lhw, lhs, NBL, s_w);
#pragma unroll
        for (int k2 = 0; k2 < QM; ++k2) {
            const uint32_t j = tid + k2 * CTT;
            if (j >= T) break;
            perm[lhs[keep[k2] & 0x3fffu] + (keep[k2] >> 14)] = static_cast<uint16_t>(j);
        }
    } else {
        // quantile mode: positions from the owner's share of the knot table (the senders' values)
        const uint32_t b0 = static_cast<uint32_t>(r) << lg_nbl;
        if (qmode)  // local buckets first (independent searches), kept in outw until the counting below
            for (uint32_t j0 = tid; j0 < T; j0 += 4 * CTT) {
                unsigned long long kq[4];
                uint32_t iv[4], lv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) kq[u] = j0 + u * CTT < T ? recv_key[j0 + u * CTT] : 0ull;
                qsearch<7>(sk, kq, iv);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    lv[u] = min(lmask, qbucket(qpos(kq[u], iv[u], sk, sc, ssl), s_qs, nbtot) - b0);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (j0 + u * CTT < T) outw[j0 + u * CTT] = lv[u];
            }
        for (uint32_t j = tid; j < T; j += CTT) {
            const uint32_t lb = qmode ? outw[j]
                                      : ((DBL ? cbucket_v(recv_dbl[j], hm, scale, nbtot) : cbucket(recv_key[j], hm, scale, nbtot)) &
                                         lmask);
            const uint32_t sh = (lb & 1) * 16;
            const uint32_t idx = (atomicAdd(lhw + (lb >> 1), 1u << sh) >> sh) & 0xffffu;
            outw[j] = lb | (idx << 14);
        }
        __syncthreads();
        block_scan_excl_u16<CTT>(lhw, lhs, NBL, s_w);  // in place: counts -> starts (bucket sizes < 2^16)
        for (uint32_t j = tid; j < T; j += CTT) {
            const uint32_t w = outw[j];
            perm[lhs[w & 0x3fffu] + (w >> 14)] = static_cast<uint16_t>(j);
        }
    }
    __syncthreads();

    mark(4);
    // ---- 5. rank inside each bucket. Equal keys are ordered by receive slot
    // (any fixed order of a tie run gives the same average rank and the same
    // run start, which is all any output depends on). Per slot:
    //   outw = (local r2 << 16) | local sorted position | run-start bit
    // walk the elements in bucket order: a warp's lanes mostly share buckets, so
    // the bucket-mate loads are shared-memory broadcasts
    const uint64_t reg = ((static_cast<uint64_t>(J.col) * K + J.seg) * CL + r) * RCAP;
    if constexpr (FK) {
#pragma unroll
        for (int k = 0; k < QM; ++k) {
            const uint32_t qq = tid + k * CTT;
            if (qq >= T) break;
            const uint32_t j = perm[qq];
            const uint32_t fv = recv_fk[j];
            const uint32_t lb = fv >> fk_sh;
            const uint32_t s0 = lhs[lb], s1 = lhs[lb + 1];
            uint32_t less = 0, eqn = 0;
#pragma unroll 2
            for (uint32_t q = s0; q < s1; ++q) {
                const uint32_t f = recv_fk[perm[q]];
                less += f < fv;
                eqn += f == fv;
            }
            uint32_t same = 1, before = 0;
            if (eqn > 1) {  // a shared fine key: the full order keys decide (ties and collisions)
                const unsigned long long* kr = kside + reg;
                const unsigned long long kv = __ldcg(kr + j);
                same = 0;
                for (uint32_t q = s0; q < s1; ++q) {
                    const uint32_t o = perm[q];
                    if (recv_fk[o] == fv) {
                        const unsigned long long kq = __ldcg(kr + o);
                        less += kq < kv;
                        const uint32_t eq = kq == kv;
                        same += eq;
                        before += eq & static_cast<uint32_t>(o < j);
                    }
                }
            }
            const uint32_t llt = s0 + less;
            outw[j] = ((2u * llt + same + 1u) << 16) | (llt + before) | (before == 0 ? 0x8000u : 0u);
        }
    } else if constexpr (DBL) {
#pragma unroll
        for (int k = 0; k < QM; ++k) {
            const uint32_t qq = tid + k * CTT;
            if (qq >= T) break;
            const uint32_t j = perm[qq];
            const double kv = recv_dbl[j];
            const uint32_t lb = outw[j] & 0x3fffu;
            const uint32_t s0 = lhs[lb], s1 = lhs[lb + 1];
            uint32_t less = 0, sb = 0;  // sb = same | before << 16
#pragma unroll 2
            for (uint32_t q = s0; q < s1; ++q) {
                const uint32_t o = perm[q];
                const double kq = recv_dbl[o];
                less += kq < kv;
                if (kq == kv) sb += 1u + (static_cast<uint32_t>(o < j) << 16);
            }
            const uint32_t same = sb & 0xffffu, before = sb >> 16;
            const uint32_t llt = s0 + less;
            outw[j] = ((2u * llt + same + 1u) << 16) | (llt + before) | (before == 0 ? 0x8000u : 0u);
        }
    } else
#pragma unroll
    for (int k = 0; k < QM; ++k) {
        const uint32_t qq = tid + k * CTT;
        if (qq >= T) break;
        const uint32_t j = perm[qq];
        const unsigned long long kv = recv_key[j];
        const uint32_t lb = LEAN ? (cbucket(kv, hm, scale, nbtot) & lmask) : (outw[j] & 0x3fffu);
        const uint32_t s0 = lhs[lb], s1 = lhs[lb + 1];
        uint32_t less = 0, sb = 0;  // sb = same | before << 16 (both <= 2^14): one accumulator, no moves
#pragma unroll 2
        for (uint32_t q = s0; q < s1; ++q) {
            const uint32_t o = perm[q];
            const unsigned long long kq = recv_key[o];
            less += kq < kv;
            const uint32_t eq = kq == kv;
            sb += eq + ((eq & static_cast<uint32_t>(o < j)) << 16);
        }
        const uint32_t same = sb & 0xffffu, before = sb >> 16;
        const uint32_t llt = s0 + less;  // < T <= 16384, so local r2 = 2*llt + same + 1 <= 2T < 2^16
        const uint32_t res = ((2u * llt + same + 1u) << 16) | (llt + before) | (before == 0 ? 0x8000u : 0u);
        // full CTAs: outw[j] (this element's bucket) is read only by this thread,
        // so the result replaces it at once; LEAN keeps it until the keys are dead
        if constexpr (LEAN) keep[k] = res;
        else outw[j] = res;
    }
    __syncthreads();
    if constexpr (LEAN) {
#pragma unroll
        for (int k = 0; k < QM; ++k) {
            const uint32_t qq = tid + k * CTT;
            if (qq >= T) break;
            outw[perm[qq]] = keep[k];
        }
        __syncthreads();
    }
    if (tid == 0) ocnt[(static_cast<uint64_t>(J.col) * K + J.seg) * CL + r] = T;
    for (uint32_t j = tid; j < T; j += CTT) {  // coalesced, in slot order
        const uint32_t w = outw[j];
        r2s_g[reg + j] = 2u * base + (w >> 16);
        posl_g[reg + j] = static_cast<uint16_t>(w & 0xffffu);
    }
    mark(5);
}

// ====================================================================
// Two CTAs per SM (k_rank_fk2, PCB_RANK_FK2): the FK scheme (32-bit fine keys
// over DSMEM, full order keys in the global side array `kside` for
// equal-fine-key pairs) in a layout small enough for two co-resident CTAs of
// 512 threads, so one CTA's barrier waits overlap the other's work. Per
// receive slot only 6 bytes of shared memory: the fine key (4 B) and the
// bucket-order index (2 B); the slice is not staged (the count and send
// passes read it from global memory, the second time from L2), the counting
// sort places with a second atomic on the same packed u16 counters (so no
// per-slot (bucket, index) word), and the results go straight to their
// per-slot outputs in global memory (write-combined in L2). Value-linear
// split only: a block whose owners would overflow takes the quantile
// relaunch of k_rank_cluster_t, exactly as from the one-per-SM kernel.
constexpr int CT2 = 512;
constexpr int EMAX2 = 32;  // slice elements per thread (S <= EMAX2 * CT2)
constexpr int QM2 = 32;    // received elements per thread (RCAP <= QM2 * CT2)

__global__ void __launch_bounds__(CT2, 2) k_rank_fk2(const ClusterJob* jobs, const double* c0, const double* c1,
                                                    uint64_t n_rows, uint32_t* route, uint32_t* r2s_g,
                                                    uint16_t* posl_g, uint32_t* ocnt, uint32_t K, int32_t* fb,
                                                    int32_t* bad, int CL, uint32_t RCAP, uint32_t lg_nbl,
                                                    int quant_ok, unsigned long long* prof, uint32_t njobs,
                                                    uint32_t pf, unsigned long long* kside) {
    namespace cg = cooperative_groups;
    long long t_prev = clock64();
    auto mark = [&](int k) {
        if (prof && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(prof + k, static_cast<unsigned long long>(t - t_prev));
            t_prev = t;
        }
    };
    cg::cluster_group cluster = cg::this_cluster();
    const int r = static_cast<int>(cluster.block_rank());
    const uint32_t jid = blockIdx.x / CL;
    const ClusterJob J = jobs[jid];
    const double* x = (J.col ? c1 : c0) + J.begin;
    const uint32_t S = slice_of(J.n, CL);
    const uint32_t a = min(J.n, r * S), e = min(J.n, a + S);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t NBL = 1u << lg_nbl;

    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* const recv_fk = reinterpret_cast<uint32_t*>(smem);
    uint16_t* const lhs = reinterpret_cast<uint16_t*>(smem + ((static_cast<size_t>(RCAP) * 4 + 15) & ~static_cast<size_t>(15)));
    uint32_t* const lhw = reinterpret_cast<uint32_t*>(lhs);
    uint16_t* const perm = lhs + NBL + 2;

    if (tid == 32 && pf && jid + pf < njobs) {  // this CTA's slice of the job one wave ahead into L2
        const ClusterJob J2 = jobs[jid + pf];
        const uint32_t S2 = slice_of(J2.n, CL);
        const uint32_t a2 = min(J2.n, r * S2), e2 = min(J2.n, a2 + S2);
        if (e2 > a2) {
            const double* x2 = (J2.col ? c1 : c0) + J2.begin;
            const uint64_t p_lo = reinterpret_cast<uint64_t>(x2 + a2) & ~15ull;
            const uint64_t p_hi = (reinterpret_cast<uint64_t>(x2 + e2) + 15ull) & ~15ull;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p_lo), "r"(static_cast<uint32_t>(p_hi - p_lo))
                         : "memory");
        }
    }

    __shared__ unsigned long long s_k[2][CT2 / 32];
    __shared__ unsigned long long s_rmin, s_rmax, s_gmin, s_gmax;
    __shared__ int s_bad, s_gbad, s_over;
    __shared__ uint32_t s_wc[CT2 / 32][kMaxCluster];
    __shared__ uint32_t s_cnt[kMaxCluster];
    __shared__ uint32_t s_mat[kMaxCluster * kMaxCluster];
    __shared__ uint32_t s_off[kMaxCluster], s_total, s_base;
    __shared__ uint32_t s_w[CT2 / 32];

    // ---- 1. bucket-map range from a strided sample (two elements per thread)
    unsigned long long kmn = ~0ull, kmx = 0ull;
    const uint32_t len = e - a;
    if (len > 0) {
        for (int h = 0; h < 2; ++h) {
            const unsigned long long kk =
                order_key(x[a + static_cast<uint32_t>((static_cast<uint64_t>(tid + h * CT2) * len) / (2 * CT2))]);
            kmn = min(kmn, kk);
            kmx = max(kmx, kk);
        }
    }
    auto cta_extremes = [&]() {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
            kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
        }
        if (lane == 0) {
            s_k[0][wid] = kmn;
            s_k[1][wid] = kmx;
        }
        __syncthreads();
        if (wid == 0) {
            kmn = lane < CT2 / 32 ? s_k[0][lane] : ~0ull;
            kmx = lane < CT2 / 32 ? s_k[1][lane] : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
                kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
            }
            if (lane == 0) {
                s_rmin = kmn;
                s_rmax = kmx;
            }
        }
    };
    auto cluster_extremes = [&]() {
        if (wid == 0) {
            unsigned long long gmn = ~0ull, gmx = 0ull;
            if (lane < CL) {
                gmn = *cluster.map_shared_rank(&s_rmin, lane);
                gmx = *cluster.map_shared_rank(&s_rmax, lane);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                gmn = min(gmn, __shfl_xor_sync(0xffffffffu, gmn, o));
                gmx = max(gmx, __shfl_xor_sync(0xffffffffu, gmx, o));
            }
            if (lane == 0) {
                s_gmin = gmn;
                s_gmax = gmx;
            }
        }
        __syncthreads();
    };
    if (tid == 0) s_bad = 0;
    for (int q = tid; q < (CT2 / 32) * kMaxCluster; q += CT2) (&s_wc[0][0])[q] = 0u;
    cta_extremes();
    mark(11);
    cluster.sync();
    mark(0);
    cluster_extremes();
    if (s_gmin == s_gmax) {  // exact extremes over every element (constant-looking sample)
        kmn = ~0ull;
        kmx = 0ull;
        for (uint32_t i = a + tid; i < e; i += CT2) {
            const unsigned long long kk = order_key(x[i]);
            kmn = min(kmn, kk);
            kmx = max(kmx, kk);
        }
        __syncthreads();
        cluster.sync();
        cta_extremes();
        cluster.sync();
        cluster_extremes();
    }
    const double vmin = key_value(s_gmin), vmax = key_value(s_gmax);
    const double hm = 0.5 * vmin;
    const uint32_t nbtot = static_cast<uint32_t>(CL) << lg_nbl;
    const double scale = static_cast<double>(nbtot) / (0.5 * vmax - hm);
    const bool constant = s_gmin == s_gmax;
    if (constant || !(isfinite(scale) && scale > 0.0 && isfinite(hm))) {
        if (constant && !isfinite(vmin)) {
            if (r == 0 && tid == 0) {
                bad[J.seg] = 1;
                fb[jid] = 2;
            }
        } else if (constant) {
            if (r == 0 && tid == 0) fb[jid] = 3;
        } else if (r == 0 && tid == 0) {
            fb[jid] = 1;
        }
        cluster.sync();
        return;
    }

    // ---- 2. owners and per-warp counts (the slice from global memory)
    uint32_t bk[EMAX2 / 8];
#pragma unroll
    for (int k = 0; k < EMAX2 / 8; ++k) bk[k] = 0u;
    bool fin = true;
#pragma unroll
    for (int h = 0; h < EMAX2 / 8; ++h) {  // 8 loads in flight per thread
        if (a + h * 8 * CT2 >= e) break;
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = a + (h * 8 + u) * CT2 + tid;
            xv[u] = i < e ? __ldg(x + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = a + (h * 8 + u) * CT2 + tid;
            if (i < e) {
                fin &= isfinite(xv[u]);
                bk[h] |= (cbucket_v(xv[u], hm, scale, nbtot) >> lg_nbl) << (u * 4);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < EMAX2; ++k)
        if (a + k * CT2 + tid < e) atomicAdd(&s_wc[wid][(bk[k >> 3] >> ((k & 7) * 4)) & 0xfu], 1u);
    if (!__syncthreads_and(fin) && tid == 0) s_bad = 1;
    if (tid < CL) {
        uint32_t run = 0;
        for (int w = 0; w < CT2 / 32; ++w) {
            const uint32_t c = s_wc[w][tid];
            s_wc[w][tid] = run;
            run += c;
        }
        s_cnt[tid] = run;
    }
    cluster.sync();
    mark(1);
    if (tid < CL * CL) s_mat[tid] = *cluster.map_shared_rank(&s_cnt[tid % CL], tid / CL);
    if (wid == 1) {
        const int gb = __any_sync(0xffffffffu, lane < CL && *cluster.map_shared_rank(&s_bad, lane) != 0);
        if (lane == 0) s_gbad = gb;
    }
    __syncthreads();
    if (s_gbad) {
        if (r == 0 && tid == 0) {
            bad[J.seg] = 1;
            fb[jid] = 2;
        }
        cluster.sync();
        return;
    }
    if (wid == 0) {
        uint32_t col = 0, mine = 0;
        if (lane < CL)
            for (int q = 0; q < CL; ++q) {
                const uint32_t v = s_mat[q * CL + lane];
                col += v;
                if (q < r) mine += v;
            }
        if (lane < CL) s_off[lane] = mine;
        const bool over = __any_sync(0xffffffffu, lane < CL && col > RCAP);
        uint32_t below = lane < r ? col : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
        const uint32_t total = __shfl_sync(0xffffffffu, col, r);
        if (lane == 0) {
            s_total = total;
            s_base = below;
            s_over = over;
        }
    }
    __syncthreads();
    if (s_over) {
        if (r == 0 && tid == 0) fb[jid] = quant_ok ? 4 : 1;
        cluster.sync();
        return;
    }
    for (int q = tid; q < (CT2 / 32) * CL; q += CT2) s_wc[q / CL][q % CL] += s_off[q % CL];
    __syncthreads();

    // ---- 3. send: fine key over DSMEM, full key to the side array, route per row
    const uint32_t recv_sa = static_cast<uint32_t>(__cvta_generic_to_shared(recv_fk));
    uint32_t* const route_j = route + static_cast<uint64_t>(J.col) * n_rows + J.begin;
    const uint64_t reg0 = (static_cast<uint64_t>(J.col) * K + J.seg) * CL;
    {
        const double P = static_cast<double>(1ull << (32 - lg_nbl));
        unsigned long long* const kb = kside + reg0 * RCAP;
#pragma unroll
        for (int h = 0; h < EMAX2 / 8; ++h) {
            if (a + h * 8 * CT2 >= e) break;
            double xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = a + (h * 8 + u) * CT2 + tid;
                xv[u] = i < e ? __ldcg(x + i) : 0.0;  // second read of the slice: L2
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = a + (h * 8 + u) * CT2 + tid;
                if (i < e) {
                    const double v = xv[u];
                    const uint32_t d = (bk[h] >> (u * 4)) & 0xfu;
                    const double t = cmap_t(v, hm, scale);
                    const uint32_t fk = __double2uint_rz(fma(t, P, -static_cast<double>(d << lg_nbl) * P));
                    const uint32_t slot = atomicAdd(&s_wc[wid][d], 1u);
                    route_j[i] = (d << 16) | slot;
                    kb[d * RCAP + slot] = order_key(v);
                    dsmem_st32(recv_sa + slot * 4u, d, fk);
                }
            }
        }
    }
    cluster.sync();  // every receive buffer is complete; no DSMEM access after this point
    mark(3);

    // ---- 4. counting sort into NBL local buckets (the fine key's top bits):
    // count, scan to starts, then place with a second atomic on the same
    // packed counters (afterwards lhs[b] = end of bucket b)
    const uint32_t T = s_total, base = s_base;
    const uint32_t fk_sh = 32 - lg_nbl;
    for (uint32_t q = tid; q <= NBL / 2; q += CT2) lhw[q] = 0u;
    __syncthreads();
    for (uint32_t j = tid; j < T; j += CT2) {
        const uint32_t lb = recv_fk[j] >> fk_sh;
        atomicAdd(lhw + (lb >> 1), 1u << ((lb & 1) * 16));
    }
    __syncthreads();
    block_scan_excl_u16<CT2>(lhw, lhs, NBL, s_w);
    for (uint32_t j = tid; j < T; j += CT2) {
        const uint32_t lb = recv_fk[j] >> fk_sh, sh = (lb & 1) * 16;
        perm[(atomicAdd(lhw + (lb >> 1), 1u << sh) >> sh) & 0xffffu] = static_cast<uint16_t>(j);
    }
    __syncthreads();
    mark(4);

    // ---- 5. rank inside each bucket; results straight to the per-slot outputs
    const uint64_t reg = (reg0 + r) * RCAP;
    const unsigned long long* const kr = kside + reg;
#pragma unroll 1
    for (int k = 0; k < QM2; ++k) {
        const uint32_t qq = tid + k * CT2;
        if (qq >= T) break;
        const uint32_t j = perm[qq];
        const uint32_t fv = recv_fk[j];
        const uint32_t lb = fv >> fk_sh;
        const uint32_t s0 = lb ? lhs[lb - 1] : 0u, s1 = lhs[lb];
        uint32_t less = 0, eqn = 0;
#pragma unroll 2
        for (uint32_t q = s0; q < s1; ++q) {
            const uint32_t f = recv_fk[perm[q]];
            less += f < fv;
            eqn += f == fv;
        }
        uint32_t same = 1, before = 0;
        if (eqn > 1) {  // a shared fine key: the full order keys decide (ties and collisions)
            const unsigned long long kv = __ldcg(kr + j);
            same = 0;
            for (uint32_t q = s0; q < s1; ++q) {
                const uint32_t o = perm[q];
                if (recv_fk[o] == fv) {
                    const unsigned long long kq = __ldcg(kr + o);
                    less += kq < kv;
                    const uint32_t eq = kq == kv;
                    same += eq;
                    before += eq & static_cast<uint32_t>(o < j);
                }
            }
        }
        const uint32_t llt = s0 + less;
        r2s_g[reg + j] = 2u * base + 2u * llt + same + 1u;
        posl_g[reg + j] = static_cast<uint16_t>((llt + before) | (before == 0 ? 0x8000u : 0u));
    }
    if (tid == 0) ocnt[reg0 + r] = T;
    mark(5);
}

// quant: the quantile-knot variant, for the jobs the value-linear split could
// not balance (fb 4 from the first launch); K = blocks (output indexing)
// Shared memory of the FK kernel with 2^lg local buckets: fine keys (4 B per
// slot, 16-aligned), then max(staged slice, outw + lhs + perm).
size_t fk_smem(const ClusterPlan& p, uint32_t lg) {
    const size_t a = (static_cast<size_t>(p.rcap) * 4 + 15) & ~static_cast<size_t>(15);
    const size_t slice = (static_cast<size_t>(p.s) + 2) * 8 + 16;
    const size_t sort = static_cast<size_t>(p.rcap) * 4 + ((static_cast<size_t>(1) << lg) + 2) * 2 +
                        static_cast<size_t>(p.rcap) * 2 + 64;
    return a + std::max(slice, sort);
}

void launch_rank_cluster(Ctx& c, const ClusterPlan& p, const ClusterJob* jobs, uint32_t njobs, uint32_t K,
                         const double* c0, const double* c1, uint64_t n_rows, RankOut& out, int32_t* fb,
                         int32_t* bad, bool quant = false) {
    int optin = 0;
    PCB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
    // FK kernel (32-bit fine keys; opt-in with PCB_RANK_FK=1, PCB_RANK_FK_LG
    // local-bucket bits): measured at C5 no faster than the 64-bit-key kernel
    // (cycles per CTA 67.6k at 2^13 buckets vs 68.0k; the send phase gains
    // from half the DSMEM bytes less than the full-key side store costs, and
    // 2^15 buckets make the bucket scan dominate) -- DESIGN.md, rejected variants
    const char* fke = std::getenv("PCB_RANK_FK");
    bool fk = !p.lean && !quant && (fke && fke[0] == '1') && out.kside != nullptr;
    uint32_t lg_fk = 0;
    if (fk) {
        cudaFuncAttributes fa;
        PCB_CUDA(cudaFuncGetAttributes(&fa, k_rank_cluster_t<CT, false, false, true>));
        uint32_t want = std::min<uint32_t>(p.lg_nbl, 15);
        if (const char* v = std::getenv("PCB_RANK_FK_LG")) want = static_cast<uint32_t>(std::atoi(v));
        for (lg_fk = want; lg_fk > p.lg_nbl; --lg_fk)
            if ((static_cast<uint64_t>(p.cl) << lg_fk) <= (1ull << 20) &&
                fk_smem(p, lg_fk) + fa.sharedSizeBytes <= static_cast<size_t>(optin))
                break;
        if (lg_fk < 1 || lg_fk > 15 || fk_smem(p, lg_fk) + fa.sharedSizeBytes > static_cast<size_t>(optin)) fk = false;
    }
    // two-CTAs-per-SM fine-key kernel (opt-in PCB_RANK_FK2=1; measured 41% slower at C5)
    const char* fk2e = std::getenv("PCB_RANK_FK2");
    if (!p.lean && !quant && out.kside != nullptr && fk2e && fk2e[0] == '1' &&
        p.rcap <= static_cast<uint32_t>(QM2 * CT2) && p.s <= static_cast<uint32_t>(EMAX2 * CT2) && p.lg_nbl <= 15) {
        const size_t smem2 = ((static_cast<size_t>(p.rcap) * 4 + 15) & ~static_cast<size_t>(15)) +
                             ((static_cast<size_t>(1) << p.lg_nbl) + 2) * 2 + static_cast<size_t>(p.rcap) * 2 + 64;
        PCB_CUDA(cudaFuncSetAttribute(k_rank_fk2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2)));
        if (p.cl > 8) PCB_CUDA(cudaFuncSetAttribute(k_rank_fk2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        int per_sm = 0;
        PCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rank_fk2, CT2, smem2));
        if (per_sm >= 2) {
            // would the quantile relaunch (one-per-SM kernel, tail mode) have room for its tables?
            cudaFuncAttributes fq;
            PCB_CUDA(cudaFuncGetAttributes(&fq, k_rank_cluster_t<CT, false, true>));
            const size_t tb = static_cast<size_t>(p.rcap) * 8 + (static_cast<size_t>(p.s) + 2) * 8 + 16;
            const uint32_t subslots = (128 + 128 / 16) + (128 / 2 + 1) + 128;
            const int quant_ok = (tb + fq.sharedSizeBytes <= static_cast<size_t>(optin) &&
                                  p.rcap >= 3200 + (p.s + 3) / 4 + subslots) ? 1 : 0;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(njobs * static_cast<uint32_t>(p.cl));
            cfg.blockDim = dim3(CT2);
            cfg.dynamicSmemBytes = smem2;
            cfg.stream = c.stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = static_cast<unsigned>(p.cl);
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            uint32_t pf = 0;
            if (const char* e = std::getenv("PCB_RANK_PF")) {
                pf = static_cast<uint32_t>(std::atoi(e));
            } else {
                int ncl = 0;
                if (cudaOccupancyMaxActiveClusters(&ncl, reinterpret_cast<const void*>(k_rank_fk2), &cfg) == cudaSuccess &&
                    ncl > 0)
                    pf = static_cast<uint32_t>(ncl);
                cudaGetLastError();
            }
            unsigned long long* prof = nullptr;
            if (getenv_flag("PCB_RANK_PROFILE")) {
                prof = c.ws.get_t<unsigned long long>("rank.prof", 12);
                PCB_CUDA(cudaMemsetAsync(prof, 0, 12 * sizeof(unsigned long long), c.stream));
            }
            PCB_CUDA(cudaLaunchKernelEx(&cfg, k_rank_fk2, jobs, c0, c1, n_rows, out.route, out.r2s, out.posl, out.ocnt,
                                        K, fb, bad, p.cl, p.rcap, p.lg_nbl, quant_ok, prof, njobs, pf, out.kside));
            if (prof) {
                unsigned long long h[12];
                PCB_CUDA(cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, c.stream));
                PCB_CUDA(cudaStreamSynchronize(c.stream));
                const double ctas = static_cast<double>(njobs) * p.cl;
                std::fprintf(stderr, "[rank profile fk2] CL=%d S=%u (2 CTAs/SM): cycles/CTA  minmax %.0f  count %.0f  "
                             "send %.0f  localsort %.0f  rank %.0f\n", p.cl, p.s, h[0] / ctas, h[1] / ctas, h[3] / ctas,
                             h[4] / ctas, h[5] / ctas);
            }
            c.count_launch();
            return;
        }
    }
    auto kern = fk ? k_rank_cluster_t<CT, false, false, true>
                   : (p.lean ? k_rank_cluster_t<kLeanT, true>
                             : (quant ? k_rank_cluster_t<CT, false, true> : k_rank_cluster_t<CT, false>));
    // tail mode when the slice fits after the receive buffer (full CTAs only)
    cudaFuncAttributes fa;
    PCB_CUDA(cudaFuncGetAttributes(&fa, kern));
    const size_t tail_bytes = static_cast<size_t>(p.rcap) * 8 + (static_cast<size_t>(p.s) + 2) * 8 + 16;
    const int tail = fk ? 1
                        : ((!p.lean && tail_bytes + fa.sharedSizeBytes <= static_cast<size_t>(optin) &&
                            !getenv_flag("PCB_RANK_NO_TAIL")) ? 1 : 0);
    const size_t smem = fk ? fk_smem(p, lg_fk) : (tail ? std::max(p.smem, tail_bytes) : p.smem);
    const uint32_t lg_launch = fk ? lg_fk : p.lg_nbl;
    // row-ordered receive slots: the caller's per-family choice (pipeline_blocks:
    // Frank), PCB_RANK_ROWMAP=0/1 forces either map
    const char* rme = std::getenv("PCB_RANK_ROWMAP");
    const int rowmap = (rme && rme[0]) ? (rme[0] == '1' ? 1 : 0) : (out.rowmap >= 0 ? out.rowmap : kRowMapDefault);
    PCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (p.cl > 8) PCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(njobs * static_cast<uint32_t>(p.cl));
    cfg.blockDim = dim3(p.lean ? kLeanT : CT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(p.cl);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // L2 prefetch distance (jobs): one wave of co-resident clusters ahead
    uint32_t pf = 0;
    if (const char* e = std::getenv("PCB_RANK_PF")) {
        pf = static_cast<uint32_t>(std::atoi(e));
    } else {
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, reinterpret_cast<const void*>(kern), &cfg) == cudaSuccess && ncl > 0)
            pf = static_cast<uint32_t>(ncl);
        cudaGetLastError();
    }
    unsigned long long* prof = nullptr;
    if (getenv_flag("PCB_RANK_PROFILE")) {
        prof = c.ws.get_t<unsigned long long>("rank.prof", 12);
        PCB_CUDA(cudaMemsetAsync(prof, 0, 12 * sizeof(unsigned long long), c.stream));
    }
    PCB_CUDA(cudaLaunchKernelEx(&cfg, kern, jobs, c0, c1, n_rows, out.rp, out.route, out.r2s, out.posl,
                                out.ocnt,
                                K, fb, bad, p.cl, p.rcap, lg_launch, tail, prof, njobs, pf, out.kside, rowmap));
    if (prof) {
        unsigned long long h[12];
        PCB_CUDA(cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, c.stream));
        PCB_CUDA(cudaStreamSynchronize(c.stream));
        const double ctas = static_cast<double>(njobs) * p.cl;
        std::fprintf(stderr, "[rank profile%s%s] CL=%d S=%u lean=%d: cycles/CTA  minmax %.0f  count %.0f  matrix %.0f  "
                     "send %.0f  localsort %.0f  rank %.0f  qsample+sort %.0f  qhist-loop %.0f  qhist-sync %.0f  qcum %.0f  "
                     "qshare %.0f  [pre-barrier %.0f]\n", quant ? " quantile" : "", fk ? " fk" : "", p.cl, p.s, int(p.lean), h[0] / ctas, h[1] / ctas, h[2] / ctas, h[3] / ctas,
                     h[4] / ctas, h[5] / ctas, h[6] / ctas, h[8] / ctas, h[9] / ctas, h[10] / ctas, h[7] / ctas, h[11] / ctas);
    }
    c.count_launch();
}

}  // namespace

namespace {

// Global-memory multi-level path for the (column, segment) jobs in `jobs`
// (encoded col * K + m): segments too large for one cluster, or whose values
// are too skewed for the cluster's value-linear split.
void run_ranks_global(Ctx& c, const double* d_col1, const double* d_col2, uint64_t n_rows,
                      const std::vector<uint64_t>& off, const std::vector<uint32_t>& jobs, RankOut out,
                      int32_t* d_bad) {
    const size_t K = off.size() - 1;
    cudaStream_t st = c.stream;
    // ---- level 0: one range per (column, segment) job
    std::vector<RankRange> ranges;
    ranges.reserve(jobs.size());
    uint64_t bsum = 0;
    uint32_t tiles = 0;
    for (uint32_t job : jobs) {
            const int col = static_cast<int>(job / K);
            const size_t m = job % K;
            RankRange R;
            std::memset(&R, 0, sizeof R);
            const uint64_t n = off[m + 1] - off[m];
            R.src_base = off[m];
            R.dst_base = static_cast<uint64_t>(col) * n_rows + off[m];
            R.out_base = off[m];
            R.n = static_cast<uint32_t>(n);
            R.nb = std::max<uint32_t>(1u, static_cast<uint32_t>(n / AVG));
            R.bbase = bsum;
            R.kmin = ~0ull;
            R.kmax = 0ull;
            R.imin = ~0u;
            R.imax = 0u;
            R.mode = 0;
            R.col = col;
            R.seg = static_cast<int32_t>(m);
            R.tile0 = tiles;
            bsum += R.nb;
            tiles += tiles_of(n);
            ranges.push_back(R);
    }
    if (ranges.empty()) return;
    const uint64_t total = 2 * n_rows;
    auto* recA = c.ws.get_t<ulonglong2>("rank.recA", total);
    const uint32_t ov_cap = static_cast<uint32_t>(total / CAP + 16);
    auto* ov = c.ws.get_t<Oversize>("rank.ov", ov_cap);
    auto* ovn = c.ws.get_t<uint32_t>("rank.ovn", 1);
    int nr = static_cast<int>(ranges.size());
    auto* d_rr = c.ws.get_t<RankRange>("rank.ranges", ranges.size());
    auto* hist = c.ws.get_t<uint32_t>("rank.hist", bsum);
    auto* bstart = c.ws.get_t<uint32_t>("rank.bstart", bsum);
    auto* cursor = c.ws.get_t<uint32_t>("rank.cursor", bsum);
    auto* h_ovn = static_cast<uint32_t*>(c.host_staging(sizeof(uint32_t)));

    auto run_level = [&](bool l0, const ulonglong2* srec, ulonglong2* drec, uint64_t nbuckets, uint32_t ntiles) {
        PCB_CUDA(cudaMemcpyAsync(d_rr, ranges.data(), ranges.size() * sizeof(RankRange), cudaMemcpyHostToDevice, st));
        PCB_CUDA(cudaMemsetAsync(hist, 0, nbuckets * sizeof(uint32_t), st));
        PCB_CUDA(cudaMemsetAsync(ovn, 0, sizeof(uint32_t), st));
        if (l0) k_minmax<true><<<ntiles, RT, 0, st>>>(d_rr, nr, d_col1, d_col2, srec, d_bad);
        else k_minmax<false><<<ntiles, RT, 0, st>>>(d_rr, nr, d_col1, d_col2, srec, d_bad);
        k_resolve<<<(nr + 127) / 128, 128, 0, st>>>(d_rr, nr, l0 ? 1 : 0);
        if (l0) k_hist<true><<<ntiles, RT, 0, st>>>(d_rr, nr, d_col1, d_col2, srec, hist);
        else k_hist<false><<<ntiles, RT, 0, st>>>(d_rr, nr, d_col1, d_col2, srec, hist);
        {  // chunked bucket scan
            std::vector<ScanChunk> hc;
            std::vector<uint32_t> c0(ranges.size() + 1);
            for (size_t r = 0; r < ranges.size(); ++r) {
                c0[r] = static_cast<uint32_t>(hc.size());
                for (uint32_t f = 0; f < ranges[r].nb; f += SCH) hc.push_back(ScanChunk{static_cast<uint32_t>(r), f});
            }
            c0[ranges.size()] = static_cast<uint32_t>(hc.size());
            const uint32_t nch = static_cast<uint32_t>(hc.size());
            auto* d_ch = c.ws.get_t<ScanChunk>("rank.chunks", nch);
            auto* d_c0 = c.ws.get_t<uint32_t>("rank.chunk0", c0.size());
            auto* csum = c.ws.get_t<uint32_t>("rank.csum", nch);
            auto* coff = c.ws.get_t<uint32_t>("rank.coff", nch);
            PCB_CUDA(cudaMemcpyAsync(d_ch, hc.data(), nch * sizeof(ScanChunk), cudaMemcpyHostToDevice, st));
            PCB_CUDA(cudaMemcpyAsync(d_c0, c0.data(), c0.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            k_scan_sum<<<nch, 256, 0, st>>>(d_rr, d_ch, hist, csum);
            k_scan_off<<<(nr + 127) / 128, 128, 0, st>>>(nr, d_c0, csum, coff);
            k_scan_apply<<<nch, 1024, 0, st>>>(d_rr, d_ch, hist, coff, bstart, cursor, ov, ovn, ov_cap);
            c.count_launch(2);
        }
        if (l0) k_scatter<true><<<ntiles, RT, 0, st>>>(d_rr, nr, d_col1, d_col2, srec, cursor, drec);
        else k_scatter<false><<<ntiles, RT, 0, st>>>(d_rr, nr, d_col1, d_col2, srec, cursor, drec);
        k_rank<<<ntiles, RT, 0, st>>>(d_rr, nr, drec, hist, bstart, n_rows, out.rp);
        c.count_launch(6);
        PCB_CUDA(cudaMemcpyAsync(h_ovn, ovn, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        PCB_CUDA(cudaStreamSynchronize(st));
        return *h_ovn;
    };

    uint32_t n_ov = run_level(true, nullptr, recA, bsum, tiles);
    // ---- refinement levels (adversarial / heavily skewed inputs only)
    ulonglong2 *cur_rec = recA, *nxt_rec = nullptr;
    int level = 0;
    while (n_ov > 0) {
        if (++level > 80) throw Error(5, "rank refinement did not terminate");
        if (n_ov > ov_cap) throw Error(5, "rank oversize list overflow");
        std::vector<Oversize> hov(n_ov);
        std::vector<RankRange> parents(ranges.size());
        PCB_CUDA(cudaMemcpyAsync(hov.data(), ov, n_ov * sizeof(Oversize), cudaMemcpyDeviceToHost, st));
        PCB_CUDA(cudaMemcpyAsync(parents.data(), d_rr, parents.size() * sizeof(RankRange), cudaMemcpyDeviceToHost, st));
        PCB_CUDA(cudaStreamSynchronize(st));
        if (!nxt_rec) nxt_rec = c.ws.get_t<ulonglong2>("rank.recB", total);
        ranges.clear();
        bsum = 0;
        tiles = 0;
        for (const Oversize& o : hov) {
            const RankRange& P = parents[o.range];
            RankRange R;
            std::memset(&R, 0, sizeof R);
            R.src_base = P.dst_base + o.start;
            R.dst_base = R.src_base;
            R.out_base = P.out_base;
            R.n = o.count;
            R.nb = std::max<uint32_t>(2u, o.count / AVG);
            R.bbase = bsum;
            R.kmin = ~0ull;
            R.kmax = 0ull;
            R.imin = ~0u;
            R.imax = 0u;
            R.lt_base = P.lt_base + o.start;
            R.mode = P.mode == 2 ? 2 : 1;
            R.run_start = P.run_start;
            R.run_len = P.run_len;
            R.col = P.col;
            R.seg = P.seg;
            R.tile0 = tiles;
            bsum += R.nb;
            tiles += tiles_of(o.count);
            ranges.push_back(R);
        }
        nr = static_cast<int>(ranges.size());
        d_rr = c.ws.get_t<RankRange>("rank.ranges", ranges.size());
        hist = c.ws.get_t<uint32_t>("rank.hist", bsum);
        bstart = c.ws.get_t<uint32_t>("rank.bstart", bsum);
        cursor = c.ws.get_t<uint32_t>("rank.cursor", bsum);
        n_ov = run_level(false, cur_rec, nxt_rec, bsum, tiles);
        std::swap(cur_rec, nxt_rec);
    }
}

// By-row packed ranks of a cluster-ranked column (blocks the routed variance
// does not take): rp[row] = (r2, owner base + local position, run start).
__global__ void k_route_to_rows(const ClusterJob* jobs, const uint32_t* list, uint64_t n_rows, uint32_t K, int CL,
                                uint32_t RCAP, const uint32_t* route, const uint32_t* r2s, const uint16_t* posl,
                                const uint32_t* ocnt, unsigned long long* rp) {
    const ClusterJob J = jobs[list[blockIdx.y]];
    __shared__ uint32_t s_base[kMaxCluster];
    const uint64_t cm = static_cast<uint64_t>(J.col) * K + J.seg;
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int d = 0; d < CL; ++d) {
            s_base[d] = run;
            run += ocnt[cm * CL + d];
        }
    }
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < J.n; i += gridDim.x * blockDim.x) {
        const uint64_t row = static_cast<uint64_t>(J.col) * n_rows + J.begin + i;
        const uint32_t w = route[row], d = w >> 16;
        const uint64_t idx = (cm * CL + d) * RCAP + (w & 0xffffu);
        const uint32_t pv = posl[idx];
        rp[row] = pack_rank(r2s[idx], s_base[d] + (pv & 0x7fffu), (pv & 0x8000u) != 0);
    }
}

void route_to_rows(Ctx& c, const ClusterPlan& p, const ClusterJob* jobs, const std::vector<uint32_t>& list,
                   const std::vector<uint64_t>& off, uint64_t n_rows, RankOut& out) {
    auto* d_list = c.ws.get_t<uint32_t>("rank.convert", list.size());
    PCB_CUDA(cudaMemcpyAsync(d_list, list.data(), list.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, c.stream));
    uint64_t nmax = 0;
    for (size_t m = 0; m + 1 < off.size(); ++m) nmax = std::max<uint64_t>(nmax, off[m + 1] - off[m]);
    const dim3 grid(static_cast<unsigned>(std::min<uint64_t>(64, (nmax + 255) / 256)), static_cast<unsigned>(list.size()));
    k_route_to_rows<<<grid, 256, 0, c.stream>>>(jobs, d_list, n_rows, static_cast<uint32_t>(off.size() - 1), p.cl,
                                                p.rcap, out.route, out.r2s, out.posl, out.ocnt, out.rp);
    c.count_launch();
}

}  // namespace

// a constant column: one tie run, avg rank (n+1)/2, positions in row order
__global__ void k_constant_rows(const ClusterJob* jobs, const uint32_t* list, uint64_t n_rows,
                                unsigned long long* rp) {
    const ClusterJob J = jobs[list[blockIdx.y]];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < J.n; i += gridDim.x * blockDim.x)
        rp[static_cast<uint64_t>(J.col) * n_rows + J.begin + i] = pack_rank(J.n + 1u, i, i == 0);
}

// By-row packed ranks are only allocated when some block needs them (global
// path, constant columns, PCB_VAR_GLOBAL): routed blocks never touch them.
unsigned long long* rows_buffer(Ctx& c, uint64_t n_rows) {
    return c.ws.get_t<unsigned long long>("pipe.rp", 2 * n_rows);
}

void run_ranks(Ctx& c, const double* d_col1, const double* d_col2, uint64_t n_rows, const std::vector<uint64_t>& off,
               RankOut& out, int32_t* d_bad) {
    const size_t K = off.size() - 1;
    if (K == 0 || n_rows == 0) return;
    uint64_t nmax = 0;
    for (size_t m = 0; m < K; ++m) {
        const uint64_t n = off[m + 1] - off[m];
        if (n >= (1ull << 30)) throw Error(2, "segment too large for 32-bit ranks");
        nmax = std::max(nmax, n);
    }
    std::vector<uint32_t> fallback;
    for (auto& v : c.rank_paths) v = 0;
    ClusterPlan plan = plan_cluster(nmax);
    if (plan.cl > 0 && !getenv_flag("PCB_RANK_GLOBAL")) {
        const uint32_t njobs = static_cast<uint32_t>(2 * K);
        auto* jobs = c.ws.get_t<ClusterJob>("rank.cjobs", njobs);
        auto* fb = c.ws.get_t<int32_t>("rank.cfb", njobs);
        std::vector<ClusterJob> hj(njobs);
        for (uint32_t j = 0; j < njobs; ++j) {
            const size_t m = j % K;
            hj[j] = ClusterJob{off[m], static_cast<uint32_t>(off[m + 1] - off[m]), static_cast<uint32_t>(j / K),
                               static_cast<uint32_t>(m), 0u};
        }
        PCB_CUDA(cudaMemcpyAsync(jobs, hj.data(), njobs * sizeof(ClusterJob), cudaMemcpyHostToDevice, c.stream));
        PCB_CUDA(cudaMemsetAsync(fb, 0, njobs * sizeof(int32_t), c.stream));
        out.cl = plan.cl;
        out.rcap = plan.rcap;
        const size_t nslot = static_cast<size_t>(njobs) * plan.cl * plan.rcap;
        out.route = c.ws.get_t<uint32_t>("rank.route", 2 * n_rows);
        out.r2s = c.ws.get_t<uint32_t>("rank.r2s", nslot);
        out.posl = c.ws.get_t<uint16_t>("rank.posl", nslot);
        out.ocnt = c.ws.get_t<uint32_t>("rank.ocnt", static_cast<size_t>(njobs) * plan.cl);
        // full order keys per receive slot for the FK kernel's equal-fine-key
        // resolution: shares the variance's routed cross-term buffer (same
        // slot layout), which is written only after the ranks are consumed
        out.kside = c.ws.get_t<unsigned long long>("var.xr", nslot);
        launch_rank_cluster(c, plan, jobs, njobs, static_cast<uint32_t>(K), d_col1, d_col2, n_rows, out, fb, d_bad);
        std::vector<int32_t> hfb(njobs);
        PCB_CUDA(cudaMemcpyAsync(hfb.data(), fb, njobs * sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
        PCB_CUDA(cudaStreamSynchronize(c.stream));
        // skewed blocks (fb 4): relaunch them through the quantile-knot variant
        std::vector<uint32_t> skew;
        for (uint32_t j = 0; j < njobs; ++j)
            if (hfb[j] == 4) skew.push_back(j);
        if (!skew.empty()) {
            const uint32_t nq = static_cast<uint32_t>(skew.size());
            auto* qjobs = c.ws.get_t<ClusterJob>("rank.qjobs", nq);
            auto* qfb = c.ws.get_t<int32_t>("rank.qfb", nq);
            std::vector<ClusterJob> hq(nq);
            for (uint32_t i = 0; i < nq; ++i) hq[i] = hj[skew[i]];
            PCB_CUDA(cudaMemcpyAsync(qjobs, hq.data(), nq * sizeof(ClusterJob), cudaMemcpyHostToDevice, c.stream));
            PCB_CUDA(cudaMemsetAsync(qfb, 0, nq * sizeof(int32_t), c.stream));
            launch_rank_cluster(c, plan, qjobs, nq, static_cast<uint32_t>(K), d_col1, d_col2, n_rows, out, qfb, d_bad,
                                true);
            std::vector<int32_t> hqfb(nq);
            PCB_CUDA(cudaMemcpyAsync(hqfb.data(), qfb, nq * sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
            PCB_CUDA(cudaStreamSynchronize(c.stream));
            for (uint32_t i = 0; i < nq; ++i) hfb[skew[i]] = hqfb[i];
        }
        // a block is routed when both columns went through the cluster path;
        // cluster-ranked columns of other blocks get their by-row ranks rebuilt
        const bool force_rows = getenv_flag("PCB_VAR_GLOBAL");
        out.routed.assign(K, force_rows ? 0 : 1);
        for (uint32_t j = 0; j < njobs; ++j) {
            if (hfb[j]) out.routed[j % K] = 0;
            if (hfb[j] == 1) fallback.push_back(j);
            ++c.rank_paths[hfb[j] == 0 ? 0 : hfb[j] == 1 ? 1 : hfb[j] == 3 ? 2 : 3];
        }
        std::vector<uint32_t> convert, constant;
        for (uint32_t j = 0; j < njobs; ++j) {
            if (hfb[j] == 0 && !out.routed[j % K]) convert.push_back(j);
            if (hfb[j] == 3) constant.push_back(j);
        }
        if (!convert.empty() || !constant.empty() || !fallback.empty()) out.rp = rows_buffer(c, n_rows);
        if (!convert.empty()) route_to_rows(c, plan, jobs, convert, off, n_rows, out);
        if (!constant.empty()) {
            uint64_t nm = 0;
            for (uint32_t j : constant) nm = std::max<uint64_t>(nm, hj[j].n);
            auto* d_list = c.ws.get_t<uint32_t>("rank.constant", constant.size());
            PCB_CUDA(cudaMemcpyAsync(d_list, constant.data(), constant.size() * sizeof(uint32_t),
                                     cudaMemcpyHostToDevice, c.stream));
            const dim3 grid(static_cast<unsigned>(std::min<uint64_t>(64, (nm + 255) / 256)),
                            static_cast<unsigned>(constant.size()));
            k_constant_rows<<<grid, 256, 0, c.stream>>>(jobs, d_list, n_rows, out.rp);
            c.count_launch();
        }
    } else {
        out.cl = 0;
        out.routed.assign(K, 0);
        out.rp = rows_buffer(c, n_rows);
        for (uint32_t j = 0; j < 2 * K; ++j) fallback.push_back(j);
    }
    if (out.cl == 0) c.rank_paths[1] = 2 * K;
    out.d_routed = c.ws.get_t<uint8_t>("rank.routed", K);
    PCB_CUDA(cudaMemcpyAsync(out.d_routed, out.routed.data(), K, cudaMemcpyHostToDevice, c.stream));
    run_ranks_global(c, d_col1, d_col2, n_rows, off, fallback, out, d_bad);
}

void ranks_to_u(Ctx& c, const RankOut& R, uint64_t n_rows, const std::vector<uint64_t>& off, double* u1,
                double* u2) {
    const size_t K = off.size() - 1;
    std::vector<Seg> segs(K);
    uint32_t tiles = 0;
    for (size_t m = 0; m < K; ++m) {
        segs[m] = Seg{off[m], static_cast<uint32_t>(off[m + 1] - off[m]), tiles};
        tiles += tiles_of(off[m + 1] - off[m]);
    }
    if (tiles == 0) return;
    auto* d_segs = c.ws.get_t<Seg>("u.segs", K);
    PCB_CUDA(cudaMemcpyAsync(d_segs, segs.data(), K * sizeof(Seg), cudaMemcpyHostToDevice, c.stream));
    k_ranks_to_u<<<tiles, RT, 0, c.stream>>>(d_segs, static_cast<int>(K), R.ref(), n_rows, u1, u2);
    c.count_launch();
}

}  // namespace pcb

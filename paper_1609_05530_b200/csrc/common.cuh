// Shared device/host definitions of the parcop B200 library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace pcb {

constexpr int kGaussian = 0, kFrank = 1, kGumbel = 2;

// block status (include/parcop_b200.h pcb_block_status) + the running state
constexpr int32_t kConverged = 0, kNotConverged = 1, kInfoNonPos = 2, kBadData = 3, kTooSmall = 4;
constexpr int32_t kRunning = 16;

constexpr int kMinRows = 30;  // SPEC.md:218 row floor

// Per-block solver state, one per segment (device resident).
struct BlockState {
    double theta;  // current iterate (theta-hat once converged)
    double lo, hi; // root bracket
    double step;   // last accepted step
    double th_prev, h_prev;  // theta and Hessian sum of the previous Newton pass (curvature of the score)
    double loglik, sigma2;
    double info_sum;   // sum hess at theta-hat
    double c1, c2;     // sum u*cross1, sum v*cross2 at theta-hat
    double stat0, stat1, stat2;  // init statistics (Gaussian: Sxy, Sss; Archimedean: sum u*v)
    uint64_t begin, n;
    int32_t iters, status;
    int32_t tried_one, pad;
};

struct Seg {  // segment table entry used by tile-mapped kernels
    uint64_t begin;
    uint32_t n;
    uint32_t tile0;  // first tile index of this segment
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum of NV doubles per thread (fixed tree order).
// `sh` must hold (blockDim.x/32)*NV doubles. Result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) sh[wid * NV + k] = v[k];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double x = lane < nw ? sh[lane * NV + k] : 0.0;
            v[k] = warp_sum(x);
        }
    }
    __syncthreads();
}

// Map a tile index to its segment by binary search over Seg::tile0.
__device__ __forceinline__ int seg_of_tile(const Seg* segs, int nseg, uint32_t tile) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (segs[mid].tile0 <= tile) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Order-preserving 64-bit key of a double; -0.0 canonicalised to +0.0 so
// that it ties with +0.0 exactly as operator== does (pseudo_obs.hpp:49,57).
__device__ __forceinline__ uint64_t order_key(double x) {
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    if ((b << 1) == 0) b = 0;
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}

// ------------------------------------------------------ tile reductions
// Fit / variance kernels map one CTA to one tile of FTILE points that never
// straddles a segment (Seg::tile0 = first tile of the segment).
constexpr int FT = 256;  // threads per tile CTA
constexpr int PPT = 32;  // points per thread per tile
constexpr uint32_t FTILE = FT * PPT;

// Row of a tile handled by this thread at step k of the route-gathering /
// scattering passes (prepare, variance passes 1 and 3). PCB_WARP_CHUNK: each
// warp walks its own contiguous FTILE/8 rows, so the 8 warps of a tile touch
// 8 distant slot runs of the rank stage's route instead of the same ones;
// otherwise the tile's threads cover FT consecutive rows per step.
#ifndef PCB_WARP_CHUNK
#define PCB_WARP_CHUNK 0
#endif
__device__ __forceinline__ uint32_t tile_row(uint32_t k) {
#if PCB_WARP_CHUNK
    return (threadIdx.x >> 5) * (FTILE / (FT / 32)) + k * 32u + (threadIdx.x & 31u);
#else
    return k * FT + threadIdx.x;
#endif
}

// Stores this tile's NV partial sums; the segment's last-arriving tile sums
// all the segment's tile partials in tile order (deterministic: fixed
// per-tile trees, fixed final order, no floating-point atomics). Returns
// true in the last tile, with the segment totals in thread 0's v[].
template <int NV>
__device__ bool tile_reduce(double (&v)[NV], double* sh, double* partials, unsigned* tickets, const Seg& S, int m,
                            uint32_t tile) {
    block_sum<NV>(v, sh);
    __shared__ bool s_last;
    const uint32_t nt = (S.n + FTILE - 1) / FTILE;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) partials[static_cast<size_t>(tile) * NV + k] = v[k];
        __threadfence();
        const unsigned ticket = atomicAdd(tickets + m, 1u);
        s_last = ticket == nt - 1;
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    double acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = 0.0;
    for (uint32_t q = threadIdx.x; q < nt; q += blockDim.x) {
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] += __ldcg(partials + static_cast<size_t>(S.tile0 + q) * NV + k);
    }
    block_sum<NV>(acc, sh);
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = acc[k];
    if (threadIdx.x == 0) tickets[m] = 0u;
    return true;
}

// Packed rank of one element of one column (see internal.hpp RankOut):
// bits 0-31 r2, bits 32-62 stable sorted position, bit 63 = first position of
// its tie run (pos == run start; every element of an untied value has it).
__host__ __device__ __forceinline__ unsigned long long pack_rank(uint32_t r2, uint32_t pos, bool first) {
    return static_cast<unsigned long long>(r2) | (static_cast<unsigned long long>(pos & 0x7fffffffu) << 32) |
           (first ? 0x8000000000000000ull : 0ull);
}
__host__ __device__ __forceinline__ uint32_t rank_r2(unsigned long long rp) { return static_cast<uint32_t>(rp); }
__host__ __device__ __forceinline__ uint32_t rank_pos(unsigned long long rp) {
    return static_cast<uint32_t>(rp >> 32) & 0x7fffffffu;
}
__host__ __device__ __forceinline__ bool rank_first(unsigned long long rp) { return (rp >> 63) != 0; }

// How a kernel reads the two ranks (r2 = twice the average rank) of a row:
// blocks the cluster rank path handled ("routed") keep their ranks per
// receive slot of the rank all-to-all, found through route[row]; all other
// blocks keep packed ranks by row.
struct RankRef {
    const unsigned long long* rp;  // [2][n_rows] by row (blocks not routed)
    const uint32_t* route;         // [2][n_rows] (owner << 16) | receive slot
    const uint32_t* r2s;           // [2][nseg][cl][rcap] r2 per slot
    const uint8_t* routed;         // [nseg] or null
    uint32_t cl, rcap;
};

__device__ __forceinline__ uint64_t slot_index(const RankRef& R, int nseg, int col, int m, uint32_t rw) {
    return ((static_cast<uint64_t>(col) * nseg + m) * R.cl + (rw >> 16)) * R.rcap + (rw & 0xffffu);
}

__device__ __forceinline__ void rank_pair(const RankRef& R, bool routed, int nseg, int m, uint64_t n_rows,
                                          uint64_t row, uint32_t& r1, uint32_t& r2) {
    if (routed) {
        const uint32_t w1 = R.route[row], w2 = R.route[n_rows + row];
        r1 = R.r2s[slot_index(R, nseg, 0, m, w1)];
        r2 = R.r2s[slot_index(R, nseg, 1, m, w2)];
    } else {
        r1 = rank_r2(R.rp[row]);
        r2 = rank_r2(R.rp[n_rows + row]);
    }
}

// (u, v) of a point: the caller's pseudo-observations, or exactly
// normalized_rank_column's value from the packed rank (pseudo_obs.hpp:59-60).
__device__ __forceinline__ void point_u(const unsigned long long* rp, const double* u1, const double* u2,
                                        uint64_t n_rows, uint64_t row, double scale, double& u, double& v) {
    if (u1) {
        u = u1[row];
        v = u2[row];
    } else {
        u = __dmul_rn(0.5 * static_cast<double>(rank_r2(rp[row])), scale);
        v = __dmul_rn(0.5 * static_cast<double>(rank_r2(rp[n_rows + row])), scale);
    }
}

}  // namespace pcb

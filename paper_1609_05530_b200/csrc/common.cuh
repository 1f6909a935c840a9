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
    double S, H;   // last score / Hessian sums
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

}  // namespace pcb

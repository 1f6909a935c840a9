// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/copula_math.hpp header).
//
// CPU restatement of the counter-based synthetic-input generator the CUDA
// sampler implements: per-subset seed
// mix_seed(base, {family, n, K, m}) (rng.hpp:24-29), draw d of subset m is
// splitmix64(seed_m + d * 0x9e3779b97f4a7c15) (rng.hpp:15-20; = output d+1 of
// the SplitMix64 stream seeded with seed_m), mapped to (0,1) exactly like
// RngStream::uniform01 (rng.hpp:40-42). Point i of a subset consumes draws
// 4i..4i+3; the family transforms follow copula.hpp:338-407.
//
// Integer draws are bit-identical to the device; the transcendental
// transforms agree to libm/libdevice ulp level (parity tests always feed the
// oracle the device's own bytes, so this is used for shape/statistics checks
// and for the CPU baseline's input generation).
#pragma once

#include <cmath>
#include <cstdint>

#include "copula_math.hpp"

namespace oracle {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

inline uint64_t splitmix64(uint64_t z) {  // rng.hpp:15-20
    z += kGamma;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

inline uint64_t mix_seed4(uint64_t base, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {  // rng.hpp:24-29
    uint64_t h = splitmix64(base);
    h = splitmix64(h ^ a);
    h = splitmix64(h ^ b);
    h = splitmix64(h ^ c);
    h = splitmix64(h ^ d);
    return h;
}

inline double unit_draw(uint64_t seed, uint64_t d) {  // rng.hpp:40-42
    return (static_cast<double>(splitmix64(seed + d * kGamma) >> 11) + 0.5) * 0x1p-53;
}

inline double clamp_sample(double u) { return std::min(std::max(u, 1e-15), 1.0 - 1e-15); }  // copula.hpp:338-340

// One point (index i within its subset) of the family's sampler.
inline void sample_point(int fam, double t, uint64_t seed, uint64_t i, double* a, double* b) {
    const double U0 = unit_draw(seed, 4 * i), U1 = unit_draw(seed, 4 * i + 1);
    if (fam == kGaussian) {  // copula.hpp:365-375 with RngStream::normal's cached twin (rng.hpp:44-55)
        const double r = std::sqrt(-2.0 * std::log(U0));
        const double th = 2.0 * 3.14159265358979323846 * U1;
        const double z1 = r * std::cos(th), z2 = r * std::sin(th);
        const double s = std::sqrt(1.0 - t * t);
        *a = clamp_sample(phi_cdf(z1));
        *b = clamp_sample(phi_cdf(t * z1 + s * z2));
        return;
    }
    if (fam == kFrank) {  // copula.hpp:376-389
        const double tt = std::fabs(t);
        const double dd = std::expm1(-tt);
        const double v = -std::log1p(U1 * dd / (U1 + (1.0 - U1) * std::exp(-tt * U0))) / tt;
        *a = clamp_sample(U0);
        *b = clamp_sample(t < 0.0 ? 1.0 - v : v);
        return;
    }
    // Gumbel, copula.hpp:390-407 and positive_stable 344-351
    if (t == 1.0) {
        *a = U0;
        *b = U1;
        return;
    }
    const double al = 1.0 / t;
    const double th = 3.14159265358979323846 * U0;
    const double w = -std::log(U1);
    const double s1 = std::sin(al * th), s2 = std::sin((1.0 - al) * th), s = std::sin(th);
    const double frail = std::pow(s2 / w, (1.0 - al) / al) * s1 / std::pow(s, 1.0 / al);
    const double e1 = -std::log(unit_draw(seed, 4 * i + 2));
    const double e2 = -std::log(unit_draw(seed, 4 * i + 3));
    *a = clamp_sample(std::exp(-std::pow(e1 / frail, al)));
    *b = clamp_sample(std::exp(-std::pow(e2 / frail, al)));
}

}  // namespace oracle

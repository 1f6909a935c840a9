/*
 * parcop_b200.h — the C-ABI drop-in boundary of the B200-native
 * divide-and-combine copula MPL fit (arXiv:1609.05530 hot path).
 *
 * The reference's "plugin/operator API" for this path is the header-only C++
 * `parcop::` library (/root/reference/proj/include/parcop) plus the SPEC
 * contracts of its absent estimator and partition/combine modules
 * (/root/reference/SPEC.md:195-323). Each entry point below replaces one of
 * those interfaces (cited per function); include/parcop_b200.hpp restores the
 * exact `parcop::` C++ signatures and exception types on top of it, and
 * INTEGRATION.md shows the bindings a maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or CUDA types in signatures.
 *  - Data pointers (columns, pseudo-observations, per-block outputs) may be
 *    HOST or DEVICE pointers of the context's device; the library detects
 *    which (cudaPointerGetAttributes) and stages host buffers itself. All
 *    calls are synchronous on return. Offsets arrays are host arrays.
 *  - Segments: `seg_offsets` holds n_seg+1 ascending row offsets; segment m
 *    is rows [seg_offsets[m], seg_offsets[m+1]) — one subset / block
 *    (SPEC.md:263-267). Ranks are segment-local.
 *  - Errors: an int status (pcb_status) plus pcb_last_error(ctx) text;
 *    codes reuse the SPEC CLI space. Per-block
 *    non-convergence is NOT an error: it is a status in the
 *    block's pcb_fit_result.
 *  - Determinism: every output is bitwise identical across runs and across
 *    any split of the blocks over calls / GPUs.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    call returns PCB_E_CUDA.
 */
#ifndef PARCOP_B200_H
#define PARCOP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCB_ABI_VERSION 2

typedef struct pcb_context pcb_context;

/* copula.hpp:25 — enum class CopulaFamily { Gaussian, Frank, Gumbel } */
enum pcb_family { PCB_GAUSSIAN = 0, PCB_FRANK = 1, PCB_GUMBEL = 2 };

/* likelihood-pass arithmetic: fp64, or fp32 per-point terms with fp64
 * accumulation / Newton / variance (BASELINE.json configs[3]). PCB_FP32
 * applies to the Frank and Gumbel Newton passes; Frank blocks whose iterate
 * has |theta| < 2 run their decision passes in fp64 arithmetic (the score
 * cancels terms of size 2/theta, copula.hpp:156-172), and so do Gumbel blocks
 * with theta < 1.1 (sigma2 amplifies root errors ~100x near theta = 1). The
 * Gaussian fit has no
 * per-point likelihood pass (closed-form sufficient statistics from the rank
 * tables), so PCB_FP32 computes it in fp64. */
enum pcb_precision { PCB_FP64 = 0, PCB_FP32 = 1 };

/* Partition scheme { Contiguous, Strided } */
enum pcb_scheme { PCB_CONTIGUOUS = 0, PCB_STRIDED = 1 };

/* return codes (SPEC.md:469 exit-code space) */
enum pcb_status {
    PCB_OK = 0,
    PCB_E_INVALID = 2,     /* std::invalid_argument: shapes, sizes, enum values */
    PCB_E_DOMAIN = 3,      /* std::domain_error: non-finite data, theta outside domain */
    PCB_E_CONVERGENCE = 4, /* combine: no converged block */
    PCB_E_CUDA = 5         /* device / runtime failure, or no sm_100 device */
};

/* pcb_fit_result.status */
enum pcb_block_status {
    PCB_BLOCK_CONVERGED = 0,
    PCB_BLOCK_NOT_CONVERGED = 1, /* SPEC.md:220 converged=false */
    PCB_BLOCK_INFO_NONPOS = 2,   /* SPEC.md:229 I-hat <= 0 at theta-hat */
    PCB_BLOCK_BAD_DATA = 3,      /* non-finite values in the block (pseudo_obs.hpp:34-36) */
    PCB_BLOCK_TOO_SMALL = 4      /* fewer than 30 rows */
};

/* FitResult { theta_hat, sigma2, n, loglik, iterations, converged } */
typedef struct pcb_fit_result {
    double theta_hat;
    double sigma2; /* v^2/n */
    double loglik; /* pseudo_loglik at theta_hat */
    uint64_t n;
    int32_t iterations; /* likelihood passes over the block's data */
    int32_t converged;  /* 1 / 0 */
    int32_t status;     /* pcb_block_status */
    int32_t reserved;
} pcb_fit_result;

/* CombinedResult scalars (per_block / weights are arrays
 * supplied by the caller) */
typedef struct pcb_combined {
    double theta_combined;
    double total_weight;
    uint64_t blocks_used;
    /* seconds per block, monotonic clock around ranks +
     * fit + variance (pcb_fit_parallel: the pipeline's wall time / M, since
     * the blocks run concurrently on the GPUs; 0 from pcb_combine) */
    double wall_clock_per_block;
} pcb_combined;

/* ---------------------------------------------------------------- context */
pcb_context* pcb_create(int device);  /* NULL on failure (no device, ...) */
/* A context over several devices: the
 * first device runs every single-device call; pcb_fit_blocks and
 * pcb_fit_parallel shard their blocks contiguously over all devices (one
 * host thread per device inside the call, no communication), gather the
 * 48-byte records to the first device by peer copies (NVLink) and combine
 * there in block order -- results are bitwise identical for any device list
 * (SPEC.md:296, 304). A device may be listed more than once (independent
 * streams on one GPU). */
pcb_context* pcb_create_multi(const int* devices, int n_devices);
int pcb_device_count(const pcb_context* ctx);
void pcb_destroy(pcb_context* ctx);
const char* pcb_last_error(const pcb_context* ctx);
int pcb_abi_version(void);
/* Launch on the caller's cudaStream_t (e.g. torch's current stream); NULL
 * restores the context's own stream. */
int pcb_set_stream(pcb_context* ctx, void* cuda_stream);
/* kernels this context launched so far, all devices (the bench's gpu_launches evidence) */
uint64_t pcb_launch_count(const pcb_context* ctx);
/* per-stage device milliseconds of the last pipeline call:
 * [0] rank [1] prepare+init [2] likelihood passes [3] variance [4] finalize
 * [5] fp64 likelihood-kernel ms and [6] its launches (inside [2])
 * [7] fp32 warm-up likelihood-kernel ms and [8] its launches (inside [2])
 * [9] variance pass 1 (per-point terms) ms (inside [3]);
 * returns the count written */
int pcb_stage_times(const pcb_context* ctx, double* ms, int n);
/* block columns (2 per block) of the last rank stage by path: [0] cluster
 * kernel (one thread-block cluster per column), [1] global multi-level
 * bucket path, [2] constant column, [3] non-finite (rejected) */
int pcb_rank_paths(const pcb_context* ctx, uint64_t counts[4]);
/* free cached device workspace */
int pcb_trim(pcb_context* ctx);

/* -------------------------------------------------------------- pseudo_obs */
/* normalized_ranks (pseudo_obs.hpp:71-77 / detail::normalized_rank_column
 * :44-65), segment-local, bit-exact: u = 0.5*((i+1)+(j+1)) * (1/(n_m+1))
 * for the tie run i..j. Validates finiteness (pseudo_obs.hpp:30-37). */
int pcb_normalized_ranks(pcb_context* ctx, const double* col1, const double* col2, uint64_t n_rows,
                         const uint64_t* seg_offsets, uint64_t n_seg, double* u1, double* u2);

/* ----------------------------------------------------------- mpl_estimator */
/* pseudo_loglik per segment at theta[m] (copula.hpp:293-311
 * log_pdf with its clamp and +-700 clip). */
int pcb_pseudo_loglik(pcb_context* ctx, int family, const double* theta, const double* u1, const double* u2,
                      uint64_t n_rows, const uint64_t* seg_offsets, uint64_t n_seg, double* loglik);

/* fit per segment of pseudo-observations; fills sigma2
 * with asymptotic_variance. */
int pcb_fit(pcb_context* ctx, int family, int precision, const double* u1, const double* u2, uint64_t n_rows,
            const uint64_t* seg_offsets, uint64_t n_seg, pcb_fit_result* out);

/* asymptotic_variance per segment at theta_hat[m];
 * sigma2[m] = NaN with PCB_BLOCK_INFO_NONPOS semantics when I-hat <= 0. */
int pcb_asymptotic_variance(pcb_context* ctx, int family, const double* theta_hat, const double* u1,
                            const double* u2, uint64_t n_rows, const uint64_t* seg_offsets, uint64_t n_seg,
                            double* sigma2);

/* -------------------------------------------------------- parallel_combine */
/* partition. CONTIGUOUS: offsets (n_blocks+1) of blocks
 * [m*floor(N/M), (m+1)*floor(N/M)), remainder to the last. STRIDED: offsets
 * of the strided blocks in the row order produced by pcb_fit_parallel's
 * gather (block m = rows i with i mod M == m, in increasing i). Error if a
 * block falls below 30 rows. */
int pcb_partition(uint64_t n_rows, uint64_t n_blocks, int scheme, uint64_t* offsets);

/* combine: theta_c = sum w theta / sum w, w = 1/sigma2,
 * over converged blocks in block order (on device). weights may be NULL. */
int pcb_combine(pcb_context* ctx, const pcb_fit_result* results, uint64_t n_blocks, double* weights,
                pcb_combined* out);

/* One shard of fit_parallel: raw columns -> per-block ranks -> fit ->
 * variance, no combine. With a pcb_create_multi context the blocks are
 * sharded over its devices and the records gathered here; a one-process-
 * per-GPU caller instead gives each process a contiguous range of blocks,
 * all-gathers the records, and calls pcb_combine. Host columns may be pinned
 * or pageable (streamed in block groups while earlier groups compute). */
int pcb_fit_blocks(pcb_context* ctx, int family, int precision, const double* col1, const double* col2,
                   uint64_t n_rows, const uint64_t* seg_offsets, uint64_t n_seg, pcb_fit_result* out);

/* fit_parallel: partition -> per block ranks, fit,
 * variance -> combine. per_block (n_blocks) and weights (n_blocks) may be
 * NULL. Returns PCB_E_CONVERGENCE if no block converged. */
int pcb_fit_parallel(pcb_context* ctx, int family, int precision, const double* col1, const double* col2,
                     uint64_t n_rows, uint64_t n_blocks, int scheme, pcb_fit_result* per_block,
                     double* weights, pcb_combined* out);

/* ------------------------------------------------------------------ inputs */
/* sample (copula.hpp:359-410) on device with counter-based streams: block m
 * of a contiguous partition of n_total rows into n_blocks_total blocks uses
 * seed mix_seed(base_seed, {family, n_total, n_blocks_total, m})
 * (rng.hpp:24-29); rows of blocks [first_block, last_block) are written to
 * col1/col2 starting at index 0. */
int pcb_sample(pcb_context* ctx, int family, double theta, uint64_t n_total, uint64_t n_blocks_total,
               uint64_t first_block, uint64_t last_block, uint64_t base_seed, double* col1, double* col2);

/* -------------------------------------------------------------- sim_study */
/* rel_l1 / rel_l2 (Eq. 19-20): relative L1 and L2 distance
 * of c(.; theta_b) from c(.; theta_a) over the unit square by a tensor
 * Gauss-Legendre rule with quad_nodes^2 interior nodes (quadrature.hpp:22-78),
 * c = exp(log_pdf) with the reference's clamp and clip (copula.hpp:293-313).
 * Equal thetas give exactly 0. */
int pcb_rel_error(pcb_context* ctx, int family, double theta_a, double theta_b, int quad_nodes, double* rel_l1,
                  double* rel_l2);

/* ----------------------------------------------------- CDF and dependence */
/* cdf (copula.hpp:273-290; Gaussian through bvn_cdf, normal.hpp:84-166) at n
 * points (u, v clamped like the reference). */
int pcb_cdf(pcb_context* ctx, int family, double theta, const double* u, const double* v, uint64_t n, double* out);
/* spearman_rho of the model: 12 * int C - 3 by the tensor
 * Gauss-Legendre rule with quad_nodes^2 nodes. */
int pcb_spearman_rho(pcb_context* ctx, int family, double theta, int quad_nodes, double* rho);
/* empirical Kendall tau of each segment's first min(n_m, m_max) rows (the
 * fit's SPEC init; m_max <= 8192): 1 - 2 * discordant / pairs. */
int pcb_kendall_tau(pcb_context* ctx, const double* u1, const double* u2, uint64_t n_rows,
                    const uint64_t* seg_offsets, uint64_t n_seg, uint64_t m_max, double* tau);
/* kendall_tau of the model and inverse_tau, host scalars */
int pcb_model_kendall_tau(int family, double theta, double* tau);
int pcb_inverse_tau(int family, double tau, double* theta);

/* ------------------------------------------------------------- measurement */
/* DFMA-loop microbenchmark: sustained FP64 instructions/s of this device
 * (the FP64 roofline denominator). */
int pcb_measure_fp64_peak(pcb_context* ctx, double* fp64_instr_per_s);

#ifdef __cplusplus
}
#endif

#endif /* PARCOP_B200_H */

// Host-side internals shared by the library's translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"

namespace pcb {

// Errors carry a pcb_status code; the C-ABI layer converts them.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PCB_CUDA(call)                                                                                  \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            throw ::pcb::Error(5, std::string(#call) + " failed: " + cudaGetErrorString(e_) + " at " + \
                                      __FILE__ + ":" + std::to_string(__LINE__));                       \
    } while (0)

// Growable cached device buffers, keyed by name.
struct Workspace {
    struct Buf {
        void* p = nullptr;
        size_t bytes = 0;
    };
    std::map<std::string, Buf> bufs;
    void* get(const std::string& name, size_t bytes) {
        Buf& b = bufs[name];
        if (b.bytes < bytes) {
            if (b.p) cudaFree(b.p);
            b.p = nullptr;
            b.bytes = 0;
            const size_t want = bytes < 256 ? 256 : bytes;
            PCB_CUDA(cudaMalloc(&b.p, want));
            b.bytes = want;
        }
        return b.p;
    }
    template <class T>
    T* get_t(const std::string& name, size_t count) {
        return static_cast<T*>(get(name, count * sizeof(T)));
    }
    void release() {
        for (auto& kv : bufs)
            if (kv.second.p) cudaFree(kv.second.p);
        bufs.clear();
    }
    ~Workspace() { release(); }
};

struct Ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::string err;
    Workspace ws;
    uint64_t launches = 0;
    double stage_ms[12] = {0};
    int n_stage = 0;
    // block columns of the last rank stage by path: [0] cluster, [1] global,
    // [2] constant, [3] invalid (non-finite)
    uint64_t rank_paths[4] = {0, 0, 0, 0};
    cudaEvent_t ev[8] = {};
    cudaStream_t copy_stream = nullptr;  // host->device streaming of inputs (overlaps compute)
    cudaEvent_t cev[4] = {};
    // pinned host staging for small results
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    void* host_staging(size_t bytes) {
        if (pinned_bytes < bytes) {
            if (pinned) cudaFreeHost(pinned);
            pinned = nullptr;
            PCB_CUDA(cudaMallocHost(&pinned, bytes));
            pinned_bytes = bytes;
        }
        return pinned;
    }
    // pageable host inputs: a ring of pinned slots the stager fills in
    // parallel and DMAs from (pipeline_blocks_host)
    void* ring = nullptr;
    size_t ring_slot_bytes = 0;
    int ring_slots = 0;
    cudaEvent_t ring_ev[8] = {};
    void count_launch(int n = 1) {
        launches += static_cast<uint64_t>(n);
        PCB_CUDA(cudaGetLastError());
    }
};

// ---------------------------------------------------------------- ranks
// Segment-local bit-exact rank outputs, [2][n_rows] packed u64
// (pack_rank in common.cuh):
//   bits 0-31  r2  = (i+1)+(j+1), twice the 1-based average rank of the tie run i..j
//   bits 32-62 pos = unique stable sorted position (ties ordered by row index)
//   bit  63    pos is the first position of its tie run
// The run-start bits of a segment, set at the positions, mark where every
// tie run begins; the variance finds a run's first position from them.
// Ranks of both columns of every block. Blocks ranked by the cluster path
// ("routed") keep them in the route space of the rank all-to-all:
//   route [2][n_rows] u32 : (owner CTA << 16) | receive slot of each row
//   r2s   [2][K][cl][rcap] u32 : twice the average rank, per receive slot
//   posl  [2][K][cl][rcap] u16 : owner-local sorted position (15 bits) |
//                                run-start bit, per receive slot
//   ocnt  [2][K][cl] u32 : elements each owner received
// and every other block keeps packed ranks by row in rp.
struct RankOut {
    unsigned long long* rp = nullptr;
    uint32_t* route = nullptr;
    uint32_t* r2s = nullptr;
    uint16_t* posl = nullptr;
    uint32_t* ocnt = nullptr;
    unsigned long long* kside = nullptr;  // FK rank kernel: full order key per receive slot
    // row-ordered receive slots (k_rank_cluster_t rowmap): set by the caller
    // per family (-1: the default, strided)
    int rowmap = -1;
    int cl = 0;
    uint32_t rcap = 0;
    std::vector<uint8_t> routed;  // host copy
    uint8_t* d_routed = nullptr;  // device copy
    RankRef ref() const {
        return RankRef{rp, route, r2s, d_routed, static_cast<uint32_t>(cl), rcap};
    }
};

// Ranks both columns of every segment. `bad` (n_seg int32, device) is set
// non-zero for segments with non-finite values (validate_data).
void run_ranks(Ctx& c, const double* d_col1, const double* d_col2, uint64_t n_rows, const std::vector<uint64_t>& off,
               RankOut& out, int32_t* d_bad);

// u = (0.5*r2) * (1/(n_m+1)), bit-exact to normalized_rank_column
void ranks_to_u(Ctx& c, const RankOut& R, uint64_t n_rows, const std::vector<uint64_t>& off, double* u1,
                double* u2);

// ---------------------------------------------------------------- fit
struct FitIO {
    int family = 0;
    int precision = 0;
    uint64_t n_rows = 0;
    std::vector<uint64_t> off;  // host offsets (n_seg + 1)
    // packed ranks [2][n_rows] (always: the variance needs the stable
    // positions); (u, v) come from u1/u2 when given, else from the ranks
    const unsigned long long* rp = nullptr;
    const RankOut* rank = nullptr;  // route space of cluster-ranked blocks (may be null)
    const double* u1 = nullptr;
    const double* u2 = nullptr;
    const int32_t* bad = nullptr;  // per segment, may be null
    const double* x1 = nullptr;  // device columns the ranks came from (raw or pseudo-observations):
    const double* x2 = nullptr;  // the PCB_INIT=tau start, rank-invariant
    const double* theta_in = nullptr;  // device: skip the fit, evaluate at these (variance API)
    bool do_fit = true;
    bool do_variance = true;
};

// Runs prepare -> init -> Newton passes -> variance; writes n_seg
// pcb_fit_result-compatible records (device) into d_out.
void run_fit(Ctx& c, const FitIO& io, void* d_out_records);

// Asymptotic variance at each converged block's theta.
struct VarIO {
    int family = 0;
    uint64_t n_rows = 0;
    const std::vector<uint64_t>* off = nullptr;
    const Seg* segs = nullptr;                  // device
    const std::vector<Seg>* h_segs = nullptr;   // host copy
    uint32_t tiles = 0;
    BlockState* st = nullptr;
    const unsigned long long* rp = nullptr;
    const RankOut* rank = nullptr;
    const double* u1 = nullptr;
    const double* u2 = nullptr;
    const double2* T64 = nullptr;  // hoisted (x,y) (Gaussian) / (ln(-ln u), ln(-ln v)) (Gumbel fp64), or null
    const double* gtab = nullptr;  // Gaussian scores by rank (fit.cu k_gauss_table), or null
    const uint64_t* goff = nullptr;
    double* partials = nullptr;
    unsigned* tickets = nullptr;
};
void run_variance(Ctx& c, const VarIO& v);

void run_loglik(Ctx& c, int family, const double* d_theta, const double* u1, const double* u2,
                const std::vector<uint64_t>& off, double* d_out);

void run_combine(Ctx& c, const void* d_records, uint64_t n, double* d_weights, double* d_out3);

void run_sample(Ctx& c, int family, double theta, uint64_t n_total, uint64_t k_total, uint64_t first,
                uint64_t last, uint64_t base_seed, double* d_col1, double* d_col2);

// Eq. 19-20 sums over the tensor Gauss-Legendre grid: out4 = {sum |fa-fb|,
// sum (fa-fb)^2, sum fa, sum fa^2} (weighted)
void run_rel_error(Ctx& c, int family, double ta, double tb, int nodes, double out4[4]);
void gauss_legendre01(int n, std::vector<double>& x, std::vector<double>& w);
// copula CDF (copula.hpp:273-290) per point; Spearman rho of the model by the
// tensor rule; empirical Kendall tau of each segment's
// first m_max rows (SPEC.md:243 init)
void run_cdf(Ctx& c, int family, double theta, const double* u, const double* v, uint64_t n, double* out);
double run_spearman(Ctx& c, int family, double theta, int nodes);
void run_kendall(Ctx& c, const double* u1, const double* u2, const std::vector<uint64_t>& off, uint32_t m_max,
                 double* tau);
void run_strided_gather(Ctx& c, const double* src, uint64_t n_rows, uint64_t m, double* dst);

double run_fp64_peak(Ctx& c);

void init_tables();

}  // namespace pcb

// The C-ABI (include/parcop_b200.h): context, pointer staging, argument
// validation with the reference's error semantics, and the pipelines that
// chain the kernels. No CPU fallback exists: every compute path runs on the
// device or fails with PCB_E_CUDA.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <chrono>
#include <condition_variable>
#include <exception>
#include <memory>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/parcop_b200.h"
#include "internal.hpp"

// A context spans one or more devices (pcb_create_multi). `c` is the first
// device: every single-device entry point runs there. fit_blocks and
// fit_parallel shard their blocks over all devices.
struct pcb_context {
    pcb::Ctx c;
    std::vector<std::unique_ptr<pcb::Ctx>> peers;  // devices 2..G of a multi-device context
    int ndev() const { return 1 + static_cast<int>(peers.size()); }
    pcb::Ctx& dev(int g) { return g == 0 ? c : *peers[g - 1]; }
};

namespace {

std::string g_create_error;

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// A read-only input that may live on the host: staged into a named buffer.
template <class T>
const T* dev_in(pcb::Ctx& c, const T* p, size_t count, const char* name) {
    if (count == 0) return p;
    if (is_device_ptr(p)) return p;
    T* d = c.ws.get_t<T>(std::string("in.") + name, count);
    PCB_CUDA(cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, c.stream));
    return d;
}

// An output that may live on the host: written to a device buffer, then
// copied back by finish().
template <class T>
struct DevOut {
    T* user;
    T* dev;
    size_t count;
    bool staged;
    DevOut(pcb::Ctx& c, T* p, size_t n, const char* name) : user(p), dev(p), count(n), staged(false) {
        if (p && n && !is_device_ptr(p)) {
            dev = c.ws.get_t<T>(std::string("out.") + name, n);
            staged = true;
        }
    }
    void finish(pcb::Ctx& c) {
        if (staged && count) PCB_CUDA(cudaMemcpyAsync(user, dev, count * sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    }
};

template <class F>
int guarded(pcb_context* ctx, F&& f) {
    if (!ctx) return PCB_E_INVALID;
    try {
        PCB_CUDA(cudaSetDevice(ctx->c.device));
        f();
        ctx->c.err.clear();
        return PCB_OK;
    } catch (const pcb::Error& e) {
        ctx->c.err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        ctx->c.err = e.what();
        return PCB_E_CUDA;
    }
}

std::vector<uint64_t> check_offsets(const uint64_t* off, uint64_t n_seg, uint64_t n_rows, uint64_t min_rows) {
    if (!off) throw pcb::Error(PCB_E_INVALID, "seg_offsets is NULL");
    if (n_seg < 1) throw pcb::Error(PCB_E_INVALID, "need at least one segment");
    if (off[0] != 0 || off[n_seg] != n_rows)
        throw pcb::Error(PCB_E_INVALID, "seg_offsets must start at 0 and end at n_rows");
    std::vector<uint64_t> v(off, off + n_seg + 1);
    for (uint64_t m = 0; m < n_seg; ++m) {
        if (v[m + 1] < v[m]) throw pcb::Error(PCB_E_INVALID, "seg_offsets must be ascending");
        if (v[m + 1] - v[m] < min_rows)
            throw pcb::Error(PCB_E_INVALID, "data matrix: need at least 2 rows");  // pseudo_obs.hpp:33
    }
    return v;
}

void check_family(int fam) {
    if (fam < 0 || fam > 2) throw pcb::Error(PCB_E_INVALID, "family must be 0 (Gaussian), 1 (Frank) or 2 (Gumbel)");
}
void check_precision(int p) {
    if (p != PCB_FP64 && p != PCB_FP32) throw pcb::Error(PCB_E_INVALID, "precision must be PCB_FP64 or PCB_FP32");
}

bool theta_in_domain(int fam, double t) {  // copula.hpp:47-55
    if (!std::isfinite(t)) return false;
    if (fam == 0) return t > -1.0 && t < 1.0;
    if (fam == 1) return t != 0.0;
    return t >= 1.0;
}

__global__ void k_check_unit(const double* u1, const double* u2, uint64_t n, int strict, int* flag) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double a = u1[i], b = u2[i];
        const bool ok = strict ? (a > 0.0 && a < 1.0 && b > 0.0 && b < 1.0)
                               : (a >= 0.0 && a <= 1.0 && b >= 0.0 && b <= 1.0);
        if (!ok) *flag = 1;
    }
}

// validate_pseudo_sample (pseudo_obs.hpp:79-88) / clamp_unit (copula.hpp:88-92)
void check_unit(pcb::Ctx& c, const double* u1, const double* u2, uint64_t n, bool strict) {
    int* flag = c.ws.get_t<int>("chk.flag", 1);
    PCB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c.stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256 + 1, 148ull * 16));
    k_check_unit<<<grid, 256, 0, c.stream>>>(u1, u2, n, strict ? 1 : 0, flag);
    c.count_launch();
    int* h = static_cast<int*>(c.host_staging(sizeof(int)));
    PCB_CUDA(cudaMemcpyAsync(h, flag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    PCB_CUDA(cudaStreamSynchronize(c.stream));
    if (*h) {
        if (strict) throw pcb::Error(PCB_E_DOMAIN, "pseudo sample: values must lie strictly in (0,1)");
        throw pcb::Error(PCB_E_DOMAIN, "copula argument must lie in [0,1]");
    }
}

struct RankBufs {
    pcb::RankOut r;
    int32_t* bad;
};

RankBufs rank_buffers(pcb::Ctx& c, uint64_t n_rows, uint64_t n_seg) {
    RankBufs b;
    b.r.rp = nullptr;  // allocated by run_ranks only if some block needs by-row ranks
    b.bad = c.ws.get_t<int32_t>("pipe.bad", n_seg);
    PCB_CUDA(cudaMemsetAsync(b.bad, 0, n_seg * sizeof(int32_t), c.stream));
    return b;
}

void finish_stage_times(pcb::Ctx& c) {
    PCB_CUDA(cudaEventSynchronize(c.ev[5]));
    for (int k = 0; k < 5; ++k) {
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, c.ev[k], c.ev[k + 1]) != cudaSuccess) {
            cudaGetLastError();
            ms = -1.0f;
        }
        c.stage_ms[k] = ms;
    }
    c.n_stage = 10;
}

// raw columns (device) -> ranks -> fit -> variance; records to d_out (device)
void pipeline_blocks(pcb::Ctx& c, int fam, int prec, const double* d1, const double* d2, uint64_t n_rows,
                     const std::vector<uint64_t>& off, void* d_out) {
    const uint64_t K = off.size() - 1;
    RankBufs rb = rank_buffers(c, n_rows, K);
    PCB_CUDA(cudaEventRecord(c.ev[0], c.stream));
    // Row-ordered receive slots for Frank: its variance pass 1 is bound by the
    // scatter of the cross terms through the route, which row order turns
    // into full L2 sectors (C5: 18.8 -> 13.7 ms); the Gaussian's route
    // gathers measured slower with it (+4.6 ms), the Gumbel's neutral.
    rb.r.rowmap = fam == PCB_FRANK ? 1 : 0;
    pcb::run_ranks(c, d1, d2, n_rows, off, rb.r, rb.bad);
    pcb::FitIO io;
    io.family = fam;
    io.precision = prec;
    io.n_rows = n_rows;
    io.off = off;
    io.rp = rb.r.rp;
    io.rank = &rb.r;
    io.bad = rb.bad;
    io.x1 = d1;
    io.x2 = d2;
    pcb::run_fit(c, io, d_out);
    finish_stage_times(c);
}

// Parallel host memcpy (pageable -> pinned): a small fixed pool of worker
// threads, each copying one contiguous share of a chunk. One process-wide
// pool; calls are serialised by its mutex (the copies are memory-bandwidth
// bound, so concurrent callers gain nothing from separate pools).
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool p;
        return p;
    }
    void copy(void* dst, const void* src, size_t bytes) {
        std::lock_guard<std::mutex> call(call_mu_);
        const size_t W = threads_.size() + 1;
        const size_t share = ((bytes + W - 1) / W + 63) & ~size_t(63);
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            share_ = share;
            pending_ = threads_.size();
            ++gen_;
        }
        cv_.notify_all();
        part(0);  // the caller copies share 0
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }

  private:
    CopyPool() {
        // the copies are host-memory-bandwidth bound: measured on a 16-core
        // box, C5 through std::vector columns 1.56 / 2.34 / 2.68 / 2.87e9
        // points/s with 4 / 8 / 12 / 16 threads
        unsigned hw = std::thread::hardware_concurrency();
        unsigned n = std::max(1u, std::min(16u, hw));
        if (const char* v = std::getenv("PCB_COPY_THREADS")) n = std::max(1, std::atoi(v));
        for (unsigned k = 1; k < n; ++k) threads_.emplace_back([this, k] { loop(k); });
    }
    void part(size_t k) {
        const size_t b0 = std::min(bytes_, k * share_), b1 = std::min(bytes_, b0 + share_);
        if (b1 > b0) std::memcpy(dst_ + b0, src_ + b0, b1 - b0);
    }
    void loop(size_t k) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            part(k);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> threads_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0, share_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

bool is_pinned_host(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// H2D of `bytes` from pageable `src`: chunks are copied in parallel into the
// context's pinned ring and DMA'd from there on the copy stream; a slot is
// refilled only after its previous DMA completed.
void h2d_pageable(pcb::Ctx& c, void* dst, const void* src, size_t bytes, uint64_t& ring_pos) {
    if (!c.ring) {
        c.ring_slots = 4;
        c.ring_slot_bytes = size_t(32) << 20;
        PCB_CUDA(cudaMallocHost(&c.ring, c.ring_slot_bytes * c.ring_slots));
        for (int k = 0; k < c.ring_slots; ++k) PCB_CUDA(cudaEventCreateWithFlags(&c.ring_ev[k], cudaEventDisableTiming));
    }
    for (size_t off = 0; off < bytes; off += c.ring_slot_bytes) {
        const size_t len = std::min(c.ring_slot_bytes, bytes - off);
        const int k = static_cast<int>(ring_pos++ % c.ring_slots);
        char* slot = static_cast<char*>(c.ring) + k * c.ring_slot_bytes;
        PCB_CUDA(cudaEventSynchronize(c.ring_ev[k]));
        CopyPool::get().copy(slot, static_cast<const char*>(src) + off, len);
        PCB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, slot, len, cudaMemcpyHostToDevice, c.copy_stream));
        PCB_CUDA(cudaEventRecord(c.ring_ev[k], c.copy_stream));
    }
}

// Host-resident inputs: stream the columns block-group by block-group on a
// copy stream into two device buffers, so the H2D of group g+1 overlaps the
// rank/fit/variance of group g. Groups are whole blocks, so every block's
// result is the same as in one call (bitwise).
//
// The copies are issued by a stager thread: with pinned columns
// cudaMemcpyAsync returns at once; pageable columns (a caller's std::vector)
// are copied in parallel into a ring of pinned slots and DMA'd from there
// (h2d_pageable) -- on the stager thread, so that work overlaps the device
// pipeline of the previous group, which this thread drives (its Newton loop
// synchronises on the stream per pass).
// Buffer reuse is stream-ordered: the copy into buffer b waits (on the copy
// stream) for the compute of the group that last used b.
void pipeline_blocks_host(pcb::Ctx& c, int fam, int prec, const double* h1, const double* h2, uint64_t n_rows,
                          const std::vector<uint64_t>& off, pcb_fit_result* d_out) {
    const uint64_t K = off.size() - 1;
    uint64_t target = 1ull << 26;  // rows per group (512 MB per column)
    if (const char* v = std::getenv("PCB_STREAM_ROWS")) target = std::max<uint64_t>(1024, std::strtoull(v, nullptr, 10));
    std::vector<std::pair<uint64_t, uint64_t>> groups;
    for (uint64_t b0 = 0; b0 < K;) {
        uint64_t b1 = b0 + 1;
        while (b1 < K && off[b1 + 1] - off[b0] <= target) ++b1;
        groups.push_back({b0, b1});
        b0 = b1;
    }
    // the last group's compute is the only part no copy hides: split it into
    // halving pieces (1/2, 1/4, ... down to ~target/8) so the exposed tail is small
    if (groups.size() > 1) {
        const auto last = groups.back();
        groups.pop_back();
        uint64_t b0 = last.first;
        while (b0 < last.second) {
            const uint64_t rest = off[last.second] - off[b0];
            uint64_t b1 = last.second;
            if (rest > target / 8) {  // take about half of what is left, in whole blocks
                b1 = b0 + 1;
                while (b1 < last.second && off[b1 + 1] - off[b0] <= rest / 2) ++b1;
            }
            groups.push_back({b0, b1});
            b0 = b1;
        }
    }
    if (groups.size() == 1) {
        const double* d1 = dev_in(c, h1, n_rows, "c1");
        const double* d2 = dev_in(c, h2, n_rows, "c2");
        pipeline_blocks(c, fam, prec, d1, d2, n_rows, off, d_out);
        return;
    }
    uint64_t maxrows = 0;
    for (auto& g : groups) maxrows = std::max(maxrows, off[g.second] - off[g.first]);
    double* buf[2][2];
    for (int b = 0; b < 2; ++b)
        for (int j = 0; j < 2; ++j)
            buf[b][j] = c.ws.get_t<double>(std::string("strm.") + char('0' + b) + char('0' + j), maxrows);
    const size_t G = groups.size();
    std::mutex mu;
    std::condition_variable cv;
    size_t copied = 0;     // groups whose copies are enqueued (copy-done event recorded)
    size_t computed = 0;   // groups whose compute is enqueued (buffer-free event recorded)
    bool abort = false;
    std::string stage_err;
    const int dev = c.device;
    const bool pinned = is_pinned_host(h1) && is_pinned_host(h2);
    uint64_t ring_pos = 0;
    std::thread stager([&] {
        try {
            PCB_CUDA(cudaSetDevice(dev));
            for (size_t g = 0; g < G; ++g) {
                const int b = static_cast<int>(g & 1);
                if (g >= 2) {  // buffer b's previous user is group g-2
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return computed >= g - 1 || abort; });
                    if (abort) return;
                    PCB_CUDA(cudaStreamWaitEvent(c.copy_stream, c.cev[2 + b], 0));
                }
                const uint64_t r0 = off[groups[g].first], rows = off[groups[g].second] - r0;
                if (pinned) {
                    PCB_CUDA(cudaMemcpyAsync(buf[b][0], h1 + r0, rows * sizeof(double), cudaMemcpyHostToDevice,
                                             c.copy_stream));
                    PCB_CUDA(cudaMemcpyAsync(buf[b][1], h2 + r0, rows * sizeof(double), cudaMemcpyHostToDevice,
                                             c.copy_stream));
                } else {
                    h2d_pageable(c, buf[b][0], h1 + r0, rows * sizeof(double), ring_pos);
                    h2d_pageable(c, buf[b][1], h2 + r0, rows * sizeof(double), ring_pos);
                }
                PCB_CUDA(cudaEventRecord(c.cev[b], c.copy_stream));
                {
                    std::lock_guard<std::mutex> lk(mu);
                    copied = g + 1;
                }
                cv.notify_all();
            }
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> lk(mu);
            stage_err = e.what();
            abort = true;
            cv.notify_all();
        }
    });
    try {
        for (size_t g = 0; g < G; ++g) {
            const int b = static_cast<int>(g & 1);
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return copied > g || abort; });
                if (abort) throw pcb::Error(PCB_E_CUDA, "host input staging failed: " + stage_err);
            }
            PCB_CUDA(cudaStreamWaitEvent(c.stream, c.cev[b], 0));
            const uint64_t b0 = groups[g].first, b1 = groups[g].second, r0 = off[b0];
            std::vector<uint64_t> og(b1 - b0 + 1);
            for (uint64_t bb = b0; bb <= b1; ++bb) og[bb - b0] = off[bb] - r0;
            pipeline_blocks(c, fam, prec, buf[b][0], buf[b][1], off[b1] - r0, og, d_out + b0);
            PCB_CUDA(cudaEventRecord(c.cev[2 + b], c.stream));
            {
                std::lock_guard<std::mutex> lk(mu);
                computed = g + 1;
            }
            cv.notify_all();
        }
    } catch (...) {
        {
            std::lock_guard<std::mutex> lk(mu);
            abort = true;
        }
        cv.notify_all();
        stager.join();
        cudaStreamSynchronize(c.copy_stream);
        throw;
    }
    stager.join();
}

int device_of(const void* p) {
    cudaPointerAttributes a;
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? a.device : -1;
}

// Opens device `device` into `c` (streams, events, constant tables); throws
// pcb::Error(PCB_E_CUDA) when it is absent or not an sm_100 part.
void init_ctx(pcb::Ctx& c, int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw pcb::Error(PCB_E_CUDA, "no CUDA device available (the library has no CPU fallback)");
    }
    if (device < 0 || device >= count) throw pcb::Error(PCB_E_CUDA, "device index out of range");
    cudaDeviceProp prop;
    PCB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        throw pcb::Error(PCB_E_CUDA,
                         std::string("device ") + prop.name + " is not sm_100 (this build targets sm_100a only)");
    PCB_CUDA(cudaSetDevice(device));
    c.device = device;
    PCB_CUDA(cudaStreamCreateWithFlags(&c.own_stream, cudaStreamNonBlocking));
    c.stream = c.own_stream;
    for (auto& ev : c.ev) PCB_CUDA(cudaEventCreate(&ev));
    for (auto& ev : c.cev) PCB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    PCB_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    pcb::init_tables();
}

void close_ctx(pcb::Ctx& c) {
    if (!c.own_stream) return;
    cudaSetDevice(c.device);
    cudaStreamSynchronize(c.stream);
    c.ws.release();
    for (auto& ev : c.ev)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : c.cev)
        if (ev) cudaEventDestroy(ev);
    if (c.copy_stream) {
        cudaStreamSynchronize(c.copy_stream);
        cudaStreamDestroy(c.copy_stream);
    }
    if (c.pinned) cudaFreeHost(c.pinned);
    if (c.ring) {
        cudaFreeHost(c.ring);
        for (int k = 0; k < c.ring_slots; ++k) cudaEventDestroy(c.ring_ev[k]);
    }
    cudaStreamDestroy(c.own_stream);
    c.own_stream = nullptr;
}

// Contiguous block range of shard g of G (sizes differ by <= 1; the same
// rule as distributed.shard_blocks)
std::pair<uint64_t, uint64_t> shard_range(uint64_t K, int G, int g) {
    const uint64_t q = K / G, r = K % G;
    const uint64_t first = g * q + std::min<uint64_t>(g, r);
    return {first, first + q + (static_cast<uint64_t>(g) < r ? 1 : 0)};
}

// fit_parallel's shard step over every device of the context (SURVEY.md
// §8(e)): device g takes the contiguous block range shard_range(K, G, g), reads
// its rows from the host (streamed, pipeline_blocks_host) or from the device
// that holds the columns (peer copy over NVLink when it is another device),
// and runs rank -> fit -> variance with no communication. Its records are
// then gathered by peer copies into d_out (device 0, block order), so the
// combine that follows is bitwise the same for every device count. One host
// thread per device drives its pipeline (each pipeline synchronises on its
// own stream per Newton pass).
void fit_blocks_sharded(pcb_context* ctx, int fam, int prec, const double* col1, const double* col2,
                        uint64_t n_rows, const std::vector<uint64_t>& off, pcb_fit_result* d_out) {
    pcb::Ctx& c0 = ctx->c;
    const uint64_t K = off.size() - 1;
    const int G = ctx->ndev();
    const int src1 = device_of(col1), src2 = device_of(col2);
    const bool host_in = src1 < 0 && src2 < 0;
    if (G == 1) {
        if (host_in) {
            pipeline_blocks_host(c0, fam, prec, col1, col2, n_rows, off, d_out);
        } else {
            const double* d1 = dev_in(c0, col1, n_rows, "c1");
            const double* d2 = dev_in(c0, col2, n_rows, "c2");
            pipeline_blocks(c0, fam, prec, d1, d2, n_rows, off, d_out);
        }
        return;
    }
    if (!host_in && (src1 < 0 || src2 < 0 || src1 != src2))
        throw pcb::Error(PCB_E_INVALID, "columns must both be host or both on one device");
    std::vector<std::exception_ptr> errs(G);
    std::vector<pcb_fit_result*> recs(G, nullptr);
    auto shard = [&](int g) {
        try {
            pcb::Ctx& cg = ctx->dev(g);
            PCB_CUDA(cudaSetDevice(cg.device));
            const auto [b0, b1] = shard_range(K, G, g);
            if (b1 == b0) return;
            const uint64_t r0 = off[b0], rows = off[b1] - r0;
            std::vector<uint64_t> og(b1 - b0 + 1);
            for (uint64_t b = b0; b <= b1; ++b) og[b - b0] = off[b] - r0;
            pcb_fit_result* rec = g == 0 ? d_out + b0 : cg.ws.get_t<pcb_fit_result>("multi.rec", b1 - b0);
            recs[g] = rec;
            if (host_in) {
                pipeline_blocks_host(cg, fam, prec, col1 + r0, col2 + r0, rows, og, rec);
            } else if (src1 == cg.device) {
                pipeline_blocks(cg, fam, prec, col1 + r0, col2 + r0, rows, og, rec);
            } else {
                double* d1 = cg.ws.get_t<double>("multi.c1", rows);
                double* d2 = cg.ws.get_t<double>("multi.c2", rows);
                PCB_CUDA(cudaMemcpyPeerAsync(d1, cg.device, col1 + r0, src1, rows * sizeof(double), cg.stream));
                PCB_CUDA(cudaMemcpyPeerAsync(d2, cg.device, col2 + r0, src1, rows * sizeof(double), cg.stream));
                pipeline_blocks(cg, fam, prec, d1, d2, rows, og, rec);
            }
            PCB_CUDA(cudaStreamSynchronize(cg.stream));
        } catch (...) {
            errs[g] = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (int g = 1; g < G; ++g) th.emplace_back(shard, g);
    shard(0);
    for (auto& t : th) t.join();
    PCB_CUDA(cudaSetDevice(c0.device));
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    // K-record gather into device 0, block order (48 B per block)
    for (int g = 1; g < G; ++g) {
        const auto [b0, b1] = shard_range(K, G, g);
        if (b1 == b0) continue;
        PCB_CUDA(cudaMemcpyPeerAsync(d_out + b0, c0.device, recs[g], ctx->dev(g).device,
                                     (b1 - b0) * sizeof(pcb_fit_result), c0.stream));
    }
}

}  // namespace

extern "C" {

int pcb_abi_version(void) { return PCB_ABI_VERSION; }

pcb_context* pcb_create(int device) { return pcb_create_multi(&device, 1); }

pcb_context* pcb_create_multi(const int* devices, int n_devices) {
    pcb_context* ctx = nullptr;
    try {
        if (!devices || n_devices < 1) throw pcb::Error(PCB_E_INVALID, "need at least one device");
        ctx = new pcb_context();
        init_ctx(ctx->c, devices[0]);
        for (int g = 1; g < n_devices; ++g) {
            ctx->peers.emplace_back(new pcb::Ctx());
            init_ctx(*ctx->peers.back(), devices[g]);
            // the record gather (and device-resident inputs) go peer to peer over NVLink
            const int a = devices[0], b = devices[g];
            int ab = 0, ba = 0;
            if (a != b && cudaDeviceCanAccessPeer(&ab, a, b) == cudaSuccess && ab &&
                cudaDeviceCanAccessPeer(&ba, b, a) == cudaSuccess && ba) {
                cudaSetDevice(a);
                cudaDeviceEnablePeerAccess(b, 0);
                cudaSetDevice(b);
                cudaDeviceEnablePeerAccess(a, 0);
                cudaGetLastError();  // cudaErrorPeerAccessAlreadyEnabled is fine
            }
        }
        cudaSetDevice(devices[0]);
        return ctx;
    } catch (const std::exception& ex) {
        g_create_error = ex.what();
        if (ctx) pcb_destroy(ctx);
        return nullptr;
    }
}

int pcb_device_count(const pcb_context* ctx) { return ctx ? ctx->ndev() : 0; }

void pcb_destroy(pcb_context* ctx) {
    if (!ctx) return;
    for (auto& p : ctx->peers) close_ctx(*p);
    close_ctx(ctx->c);
    delete ctx;
}

const char* pcb_last_error(const pcb_context* ctx) { return ctx ? ctx->c.err.c_str() : g_create_error.c_str(); }

int pcb_set_stream(pcb_context* ctx, void* s) {
    if (!ctx) return PCB_E_INVALID;
    ctx->c.stream = s ? static_cast<cudaStream_t>(s) : ctx->c.own_stream;
    return PCB_OK;
}

uint64_t pcb_launch_count(const pcb_context* ctx) {
    if (!ctx) return 0;
    uint64_t n = ctx->c.launches;
    for (const auto& p : ctx->peers) n += p->launches;
    return n;
}

int pcb_stage_times(const pcb_context* ctx, double* ms, int n) {
    if (!ctx || !ms) return 0;
    const int k = std::min(n, ctx->c.n_stage);
    for (int i = 0; i < k; ++i) ms[i] = ctx->c.stage_ms[i];
    return k;
}

int pcb_rank_paths(const pcb_context* ctx, uint64_t* counts) {
    if (!ctx || !counts) return PCB_E_INVALID;
    for (int i = 0; i < 4; ++i) counts[i] = ctx->c.rank_paths[i];
    return PCB_OK;
}

int pcb_trim(pcb_context* ctx) {
    return guarded(ctx, [&] {
        for (int g = 0; g < ctx->ndev(); ++g) {
            pcb::Ctx& cg = ctx->dev(g);
            PCB_CUDA(cudaSetDevice(cg.device));
            PCB_CUDA(cudaStreamSynchronize(cg.stream));
            cg.ws.release();
        }
        PCB_CUDA(cudaSetDevice(ctx->c.device));
    });
}

int pcb_normalized_ranks(pcb_context* ctx, const double* col1, const double* col2, uint64_t n_rows,
                         const uint64_t* seg_offsets, uint64_t n_seg, double* u1, double* u2) {
    return guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        if (!col1 || !col2 || !u1 || !u2) throw pcb::Error(PCB_E_INVALID, "NULL column pointer");
        const auto off = check_offsets(seg_offsets, n_seg, n_rows, 2);
        const double* d1 = dev_in(c, col1, n_rows, "c1");
        const double* d2 = dev_in(c, col2, n_rows, "c2");
        RankBufs rb = rank_buffers(c, n_rows, n_seg);
        pcb::run_ranks(c, d1, d2, n_rows, off, rb.r, rb.bad);
        std::vector<int32_t> bad(n_seg);
        PCB_CUDA(cudaMemcpyAsync(bad.data(), rb.bad, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
        PCB_CUDA(cudaStreamSynchronize(c.stream));
        for (int32_t b : bad)
            if (b) throw pcb::Error(PCB_E_DOMAIN, "data matrix: non-finite value");  // pseudo_obs.hpp:36
        DevOut<double> o1(c, u1, n_rows, "u1"), o2(c, u2, n_rows, "u2");
        pcb::ranks_to_u(c, rb.r, n_rows, off, o1.dev, o2.dev);
        o1.finish(c);
        o2.finish(c);
        PCB_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int pcb_pseudo_loglik(pcb_context* ctx, int family, const double* theta, const double* u1, const double* u2,
                      uint64_t n_rows, const uint64_t* seg_offsets, uint64_t n_seg, double* loglik) {
    return guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        check_family(family);
        if (!theta || !u1 || !u2 || !loglik) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        const auto off = check_offsets(seg_offsets, n_seg, n_rows, 0);
        std::vector<double> th(n_seg);
        if (is_device_ptr(theta))
            PCB_CUDA(cudaMemcpy(th.data(), theta, n_seg * sizeof(double), cudaMemcpyDeviceToHost));
        else
            std::memcpy(th.data(), theta, n_seg * sizeof(double));
        for (double t : th)
            if (!theta_in_domain(family, t)) throw pcb::Error(PCB_E_DOMAIN, "theta outside the family domain");
        const double* d1 = dev_in(c, u1, n_rows, "u1");
        const double* d2 = dev_in(c, u2, n_rows, "u2");
        check_unit(c, d1, d2, n_rows, false);
        const double* dth = dev_in(c, theta, n_seg, "theta");
        DevOut<double> o(c, loglik, n_seg, "loglik");
        pcb::run_loglik(c, family, dth, d1, d2, off, o.dev);
        o.finish(c);
        PCB_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int pcb_fit(pcb_context* ctx, int family, int precision, const double* u1, const double* u2, uint64_t n_rows,
            const uint64_t* seg_offsets, uint64_t n_seg, pcb_fit_result* out) {
    return guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        check_family(family);
        check_precision(precision);
        if (!u1 || !u2 || !out) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        const auto off = check_offsets(seg_offsets, n_seg, n_rows, 0);
        const double* d1 = dev_in(c, u1, n_rows, "u1");
        const double* d2 = dev_in(c, u2, n_rows, "u2");
        check_unit(c, d1, d2, n_rows, true);
        RankBufs rb = rank_buffers(c, n_rows, n_seg);
        PCB_CUDA(cudaEventRecord(c.ev[0], c.stream));
        pcb::run_ranks(c, d1, d2, n_rows, off, rb.r, rb.bad);  // order statistics for the W-term
        pcb::FitIO io;
        io.family = family;
        io.precision = precision;
        io.n_rows = n_rows;
        io.off = off;
        io.u1 = d1;
        io.u2 = d2;
        io.x1 = d1;
        io.x2 = d2;
        io.rp = rb.r.rp;
        io.rank = &rb.r;
        DevOut<pcb_fit_result> o(c, out, n_seg, "fit");
        pcb::run_fit(c, io, o.dev);
        finish_stage_times(c);
        o.finish(c);
        PCB_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int pcb_asymptotic_variance(pcb_context* ctx, int family, const double* theta_hat, const double* u1,
                            const double* u2, uint64_t n_rows, const uint64_t* seg_offsets, uint64_t n_seg,
                            double* sigma2) {
    bool info_bad = false;
    int rc = guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        check_family(family);
        if (!theta_hat || !u1 || !u2 || !sigma2) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        const auto off = check_offsets(seg_offsets, n_seg, n_rows, 0);
        std::vector<double> th(n_seg);
        if (is_device_ptr(theta_hat))
            PCB_CUDA(cudaMemcpy(th.data(), theta_hat, n_seg * sizeof(double), cudaMemcpyDeviceToHost));
        else
            std::memcpy(th.data(), theta_hat, n_seg * sizeof(double));
        for (double t : th)
            if (!theta_in_domain(family, t)) throw pcb::Error(PCB_E_DOMAIN, "theta outside the family domain");
        const double* d1 = dev_in(c, u1, n_rows, "u1");
        const double* d2 = dev_in(c, u2, n_rows, "u2");
        check_unit(c, d1, d2, n_rows, true);
        const double* dth = dev_in(c, theta_hat, n_seg, "theta");
        RankBufs rb = rank_buffers(c, n_rows, n_seg);
        PCB_CUDA(cudaEventRecord(c.ev[0], c.stream));
        pcb::run_ranks(c, d1, d2, n_rows, off, rb.r, rb.bad);
        pcb::FitIO io;
        io.family = family;
        io.n_rows = n_rows;
        io.off = off;
        io.u1 = d1;
        io.u2 = d2;
        io.x1 = d1;
        io.x2 = d2;
        io.rp = rb.r.rp;
        io.rank = &rb.r;
        io.theta_in = dth;
        io.do_fit = false;
        auto* rec = c.ws.get_t<pcb_fit_result>("var.rec", n_seg);
        pcb::run_fit(c, io, rec);
        std::vector<pcb_fit_result> h(n_seg);
        PCB_CUDA(cudaMemcpyAsync(h.data(), rec, n_seg * sizeof(pcb_fit_result), cudaMemcpyDeviceToHost, c.stream));
        PCB_CUDA(cudaStreamSynchronize(c.stream));
        std::vector<double> s2(n_seg);
        for (uint64_t m = 0; m < n_seg; ++m) {
            s2[m] = h[m].sigma2;
            if (h[m].status == PCB_BLOCK_INFO_NONPOS) info_bad = true;
        }
        if (is_device_ptr(sigma2))
            PCB_CUDA(cudaMemcpy(sigma2, s2.data(), n_seg * sizeof(double), cudaMemcpyHostToDevice));
        else
            std::memcpy(sigma2, s2.data(), n_seg * sizeof(double));
    });
    if (rc == PCB_OK && info_bad) {
        ctx->c.err = "asymptotic_variance: information <= 0";
        return PCB_E_DOMAIN;
    }
    return rc;
}

int pcb_partition(uint64_t n_rows, uint64_t n_blocks, int scheme, uint64_t* offsets) {
    if (!offsets || n_blocks < 1) return PCB_E_INVALID;
    if (scheme != PCB_CONTIGUOUS && scheme != PCB_STRIDED) return PCB_E_INVALID;
    const uint64_t q = n_rows / n_blocks;
    if (q < 30) return PCB_E_INVALID;
    if (scheme == PCB_CONTIGUOUS) {
        for (uint64_t m = 0; m < n_blocks; ++m) offsets[m] = m * q;
        offsets[n_blocks] = n_rows;
    } else {
        const uint64_t rem = n_rows % n_blocks;
        uint64_t acc = 0;
        for (uint64_t m = 0; m < n_blocks; ++m) {
            offsets[m] = acc;
            acc += q + (m < rem ? 1 : 0);
        }
        offsets[n_blocks] = acc;
    }
    return PCB_OK;
}

int pcb_combine(pcb_context* ctx, const pcb_fit_result* results, uint64_t n_blocks, double* weights,
                pcb_combined* out) {
    bool none = false;
    int rc = guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        if (!results || !out || n_blocks < 1) throw pcb::Error(PCB_E_INVALID, "combine: empty input");
        const pcb_fit_result* dr = dev_in(c, results, n_blocks, "comb");
        DevOut<double> w(c, weights, weights ? n_blocks : 0, "w");
        double* d3 = c.ws.get_t<double>("comb.out", 3);
        pcb::run_combine(c, dr, n_blocks, weights ? w.dev : nullptr, d3);
        double h3[3];
        PCB_CUDA(cudaMemcpyAsync(h3, d3, sizeof h3, cudaMemcpyDeviceToHost, c.stream));
        w.finish(c);
        PCB_CUDA(cudaStreamSynchronize(c.stream));
        pcb_combined r;
        r.theta_combined = h3[0];
        r.total_weight = h3[1];
        r.blocks_used = static_cast<uint64_t>(h3[2]);
        r.wall_clock_per_block = 0.0;
        if (is_device_ptr(out)) PCB_CUDA(cudaMemcpy(out, &r, sizeof r, cudaMemcpyHostToDevice));
        else *out = r;
        none = r.blocks_used == 0;
    });
    if (rc == PCB_OK && none) {
        ctx->c.err = "combine: no converged blocks";
        return PCB_E_CONVERGENCE;
    }
    return rc;
}

int pcb_fit_blocks(pcb_context* ctx, int family, int precision, const double* col1, const double* col2,
                   uint64_t n_rows, const uint64_t* seg_offsets, uint64_t n_seg, pcb_fit_result* out) {
    return guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        check_family(family);
        check_precision(precision);
        if (!col1 || !col2 || !out) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        const auto off = check_offsets(seg_offsets, n_seg, n_rows, 2);
        DevOut<pcb_fit_result> o(c, out, n_seg, "fit");
        fit_blocks_sharded(ctx, family, precision, col1, col2, n_rows, off, o.dev);
        o.finish(c);
        PCB_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int pcb_fit_parallel(pcb_context* ctx, int family, int precision, const double* col1, const double* col2,
                     uint64_t n_rows, uint64_t n_blocks, int scheme, pcb_fit_result* per_block, double* weights,
                     pcb_combined* out) {
    bool none = false;
    int rc = guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        check_family(family);
        check_precision(precision);
        if (!col1 || !col2 || !out) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        std::vector<uint64_t> off(n_blocks + 1);
        if (n_blocks < 1) throw pcb::Error(PCB_E_INVALID, "partition: need M >= 1");
        if (pcb_partition(n_rows, n_blocks, scheme, off.data()) != PCB_OK)
            throw pcb::Error(PCB_E_INVALID, "partition: block below the 30-row floor");
        auto* rec = c.ws.get_t<pcb_fit_result>("par.rec", n_blocks);
        // per-block wall clock measured with a monotonic clock
        // around ranks + fit + variance (all blocks run at once on the GPUs:
        // the pipeline's wall time divided by the block count)
        const auto t0 = std::chrono::steady_clock::now();
        if (scheme == PCB_STRIDED) {  // row i -> block i mod M: gathered on the first device
            const double* d1 = dev_in(c, col1, n_rows, "c1");
            const double* d2 = dev_in(c, col2, n_rows, "c2");
            double* g1 = c.ws.get_t<double>("strided.c1", n_rows);
            double* g2 = c.ws.get_t<double>("strided.c2", n_rows);
            pcb::run_strided_gather(c, d1, n_rows, n_blocks, g1);
            pcb::run_strided_gather(c, d2, n_rows, n_blocks, g2);
            fit_blocks_sharded(ctx, family, precision, g1, g2, n_rows, off, rec);
        } else {
            fit_blocks_sharded(ctx, family, precision, col1, col2, n_rows, off, rec);
        }
        PCB_CUDA(cudaStreamSynchronize(c.stream));
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        DevOut<double> w(c, weights, weights ? n_blocks : 0, "w");
        double* d3 = c.ws.get_t<double>("comb.out", 3);
        pcb::run_combine(c, rec, n_blocks, weights ? w.dev : nullptr, d3);
        double h3[3];
        PCB_CUDA(cudaMemcpyAsync(h3, d3, sizeof h3, cudaMemcpyDeviceToHost, c.stream));
        w.finish(c);
        if (per_block) {
            if (is_device_ptr(per_block))
                PCB_CUDA(cudaMemcpyAsync(per_block, rec, n_blocks * sizeof(pcb_fit_result), cudaMemcpyDeviceToDevice,
                                         c.stream));
            else
                PCB_CUDA(cudaMemcpyAsync(per_block, rec, n_blocks * sizeof(pcb_fit_result), cudaMemcpyDeviceToHost,
                                         c.stream));
        }
        PCB_CUDA(cudaStreamSynchronize(c.stream));
        out->theta_combined = h3[0];
        out->total_weight = h3[1];
        out->blocks_used = static_cast<uint64_t>(h3[2]);
        out->wall_clock_per_block = wall / static_cast<double>(n_blocks);
        none = out->blocks_used == 0;
    });
    if (rc == PCB_OK && none) {
        ctx->c.err = "fit_parallel: all blocks failed";
        return PCB_E_CONVERGENCE;
    }
    return rc;
}

int pcb_sample(pcb_context* ctx, int family, double theta, uint64_t n_total, uint64_t n_blocks_total,
               uint64_t first_block, uint64_t last_block, uint64_t base_seed, double* col1, double* col2) {
    return guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        check_family(family);
        if (!theta_in_domain(family, theta)) throw pcb::Error(PCB_E_DOMAIN, "theta outside the family domain");
        if (n_blocks_total < 1 || n_total < n_blocks_total || first_block > last_block || last_block > n_blocks_total)
            throw pcb::Error(PCB_E_INVALID, "sample: bad block range");
        if (!col1 || !col2) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        const uint64_t q = n_total / n_blocks_total;
        const uint64_t rows = (last_block == n_blocks_total ? n_total : last_block * q) - first_block * q;
        DevOut<double> o1(c, col1, rows, "s1"), o2(c, col2, rows, "s2");
        pcb::run_sample(c, family, theta, n_total, n_blocks_total, first_block, last_block, base_seed, o1.dev, o2.dev);
        o1.finish(c);
        o2.finish(c);
        PCB_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int pcb_rel_error(pcb_context* ctx, int family, double theta_a, double theta_b, int quad_nodes, double* rel_l1,
                  double* rel_l2) {
    return guarded(ctx, [&] {
        check_family(family);
        if (!theta_in_domain(family, theta_a) || !theta_in_domain(family, theta_b))
            throw pcb::Error(PCB_E_DOMAIN, "theta outside the family domain");
        if (quad_nodes < 1 || quad_nodes > 65536) throw pcb::Error(PCB_E_INVALID, "rel_error: quad_nodes out of range");
        if (!rel_l1 || !rel_l2) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        double s[4];
        pcb::run_rel_error(ctx->c, family, theta_a, theta_b, quad_nodes, s);
        *rel_l1 = s[0] / s[2];                        // Eq. 19
        *rel_l2 = std::sqrt(s[1]) / std::sqrt(s[3]);  // Eq. 20
    });
}

int pcb_cdf(pcb_context* ctx, int family, double theta, const double* u, const double* v, uint64_t n, double* out) {
    return guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        check_family(family);
        if (!theta_in_domain(family, theta)) throw pcb::Error(PCB_E_DOMAIN, "theta outside the family domain");
        if (n && (!u || !v || !out)) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        const double* du = dev_in(c, u, n, "cu");
        const double* dv = dev_in(c, v, n, "cv");
        DevOut<double> o(c, out, n, "cdf");
        pcb::run_cdf(c, family, theta, du, dv, n, o.dev);
        o.finish(c);
        PCB_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int pcb_spearman_rho(pcb_context* ctx, int family, double theta, int quad_nodes, double* rho) {
    return guarded(ctx, [&] {
        check_family(family);
        if (!theta_in_domain(family, theta)) throw pcb::Error(PCB_E_DOMAIN, "theta outside the family domain");
        if (quad_nodes < 1 || quad_nodes > 65536) throw pcb::Error(PCB_E_INVALID, "spearman_rho: bad quad_nodes");
        if (!rho) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        *rho = pcb::run_spearman(ctx->c, family, theta, quad_nodes);
    });
}

int pcb_kendall_tau(pcb_context* ctx, const double* u1, const double* u2, uint64_t n_rows,
                    const uint64_t* seg_offsets, uint64_t n_seg, uint64_t m_max, double* tau) {
    return guarded(ctx, [&] {
        pcb::Ctx& c = ctx->c;
        const std::vector<uint64_t> off = check_offsets(seg_offsets, n_seg, n_rows, 0);
        if (m_max < 2 || m_max > 8192) throw pcb::Error(PCB_E_INVALID, "kendall_tau: m_max must lie in [2, 8192]");
        if (!u1 || !u2 || !tau) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        const double* d1 = dev_in(c, u1, n_rows, "k1");
        const double* d2 = dev_in(c, u2, n_rows, "k2");
        DevOut<double> o(c, tau, n_seg, "tau");
        pcb::run_kendall(c, d1, d2, off, static_cast<uint32_t>(m_max), o.dev);
        o.finish(c);
        PCB_CUDA(cudaStreamSynchronize(c.stream));
    });
}

}  // extern "C"

namespace {
// quadrature.hpp:82-120: adaptive Simpson and the first Debye function
template <class F>
double simpson_step(F& f, double a, double b, double fa, double fm, double fb, double whole, double tol, int depth) {
    const double m = 0.5 * (a + b), lm = 0.5 * (a + m), rm = 0.5 * (m + b);
    const double flm = f(lm), frm = f(rm);
    const double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm), right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
    const double delta = left + right - whole;
    if (depth <= 0 || std::fabs(delta) <= 15.0 * tol) return left + right + delta / 15.0;
    return simpson_step(f, a, m, fa, flm, fm, left, 0.5 * tol, depth - 1) +
           simpson_step(f, m, b, fm, frm, fb, right, 0.5 * tol, depth - 1);
}
double debye1_host(double x) {
    if (x == 0.0) return 1.0;
    if (x < 0.0) return debye1_host(-x) - x / 2.0;
    auto f = [](double t) { return t == 0.0 ? 1.0 : t / std::expm1(t); };
    const double fa = f(0.0), fm = f(0.5 * x), fb = f(x);
    return simpson_step(f, 0.0, x, fa, fm, fb, x / 6.0 * (fa + 4.0 * fm + fb), 1e-13 * std::max(1.0, x), 48) / x;
}
double model_tau(int fam, double t) {
    if (fam == 0) return 2.0 / 3.14159265358979323846 * std::asin(t);
    if (fam == 2) return 1.0 - 1.0 / t;
    return 1.0 - 4.0 / t * (1.0 - debye1_host(t));
}
}  // namespace

extern "C" {

int pcb_model_kendall_tau(int family, double theta, double* tau) {
    if (family < 0 || family > 2 || !tau) return PCB_E_INVALID;
    if (!theta_in_domain(family, theta)) return PCB_E_DOMAIN;
    *tau = model_tau(family, theta);
    return PCB_OK;
}

int pcb_inverse_tau(int family, double tau, double* theta) {
    if (family < 0 || family > 2 || !theta || !std::isfinite(tau)) return PCB_E_INVALID;
    if (tau <= -1.0 || tau >= 1.0 || (family == 2 && tau < 0.0)) return PCB_E_DOMAIN;  // unattainable
    if (family == 0) {
        *theta = std::sin(0.5 * 3.14159265358979323846 * tau);
    } else if (family == 2) {
        *theta = 1.0 / (1.0 - tau);
    } else {
        if (tau == 0.0) return PCB_E_DOMAIN;  // the Frank family excludes theta = 0
        const double at = std::fabs(tau);
        double lo = 1e-9, hi = 1.0;
        while (model_tau(1, hi) < at && hi < 1e6) hi *= 2.0;
        for (int it = 0; it < 300 && hi - lo > 1e-12 * hi; ++it) {
            const double mid = 0.5 * (lo + hi);
            (model_tau(1, mid) < at ? lo : hi) = mid;
        }
        *theta = tau < 0.0 ? -0.5 * (lo + hi) : 0.5 * (lo + hi);
    }
    return PCB_OK;
}

int pcb_measure_fp64_peak(pcb_context* ctx, double* v) {
    return guarded(ctx, [&] {
        if (!v) throw pcb::Error(PCB_E_INVALID, "NULL pointer");
        *v = pcb::run_fp64_peak(ctx->c);
    });
}

}  // extern "C"

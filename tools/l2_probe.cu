// L2 read-throughput probe: every SM streams an L2-resident buffer (32 MB,
// read repeatedly, 16-byte coalesced loads); reports bytes per second and
// 32-byte sectors per second. Used as the L2 roofline of the gather-bound
// kernels.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/l2_probe.cu -o /tmp/l2_probe && /tmp/l2_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const uint4* __restrict__ p, size_t n16, int reps, unsigned long long* sink) {
    uint32_t acc = 0;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
            const uint4 v = __ldcg(p + i);  // L2, bypass L1
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// random 4-byte gathers (one 32-byte sector each) from the same L2-resident buffer
__global__ void gather(const uint32_t* __restrict__ p, uint32_t mask, int reps, unsigned long long* sink) {
    uint32_t acc = 0, h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    for (int r = 0; r < reps; ++r) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            h = h * 1664525u + 1013904223u;
            v[k] = __ldcg(p + ((h >> 3) & mask));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k];
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
    const size_t bytes = 32ull << 20;
    uint4* p;
    unsigned long long* sink;
    cudaMalloc(&p, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(p, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int reps = 200;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    for (int t = 0; t < 5; ++t) {
        cudaEventRecord(a);
        rd<<<sms * 4, 512>>>(p, bytes / 16, reps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double tbs = static_cast<double>(bytes) * reps / (ms * 1e-3) / 1e12;
        if (tbs > best) best = tbs;
    }
    double gbest = 0;  // random sector gathers per second
    const int greps = 256;
    for (int t = 0; t < 5; ++t) {
        cudaEventRecord(a);
        gather<<<sms * 4, 512>>>(reinterpret_cast<const uint32_t*>(p), static_cast<uint32_t>(bytes / 4 - 1), greps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double g = static_cast<double>(sms) * 4 * 512 * greps * 8 / (ms * 1e-3);
        if (g > gbest) gbest = g;
    }
    printf("{\"l2_read_tbs\": %.2f, \"l2_stream_sectors_per_s\": %.3e, \"l2_random_sectors_per_s\": %.3e, "
           "\"buffer_mb\": 32, \"sms\": %d}\n", best, best * 1e12 / 32, gbest, sms);
    return 0;
}

// smem_bench.cu -- shared-memory peaks of one B200 SM for the tile sieve's
// two access kinds:
//   1. red.shared.and.b32 to random words of an 8 KB tile (the medium-prime
//      scatter: one clear per lane, bank conflicts as random addresses give)
//   2. red.shared.and.b32 with lane-distinct banks (conflict-free bound)
//   3. LDS.128 of consecutive 16-byte chunks across the warp (the scan loads)
// Each kernel runs 4 CTAs x 256 threads per SM (the tile kernel's shape),
// timed per CTA with clock64; the rate is per SM per SM-clock cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o experiments/smem_bench tools/smem_bench.cu
//   ./experiments/smem_bench
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int kThreads = 256, kCtasPerSm = 4, kWords = 2048, kIters = 4096;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) smem_kernel(unsigned long long *cycles, uint32_t *sink) {
    __shared__ __align__(16) uint32_t tile[kWords];
    for (int i = threadIdx.x; i < kWords; i += kThreads) tile[i] = ~0u;
    __syncthreads();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(tile);
    uint32_t x = hash32(threadIdx.x * 7919u + blockIdx.x * 104729u);
    uint32_t acc = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
        if (MODE == 0) {  // random word, random bit
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x = x * 1664525u + 1013904223u;
                const uint32_t o = x >> 16;  // 0..65535 slot
                const uint32_t addr = base + ((o >> 5) << 2);
                asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(addr), "r"(~(1u << (o & 31))) : "memory");
            }
        } else if (MODE == 1) {  // lane-distinct banks
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                x = x * 1664525u + 1013904223u;
                const uint32_t w = ((x >> 21) & ~31u) | (threadIdx.x & 31);
                asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(base + 4 * (w & (kWords - 1))),
                             "r"(~(1u << (x & 31))) : "memory");
            }
        } else {  // LDS.128, consecutive chunks across the warp
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t w = (4 * (threadIdx.x + 64 * u + 8 * it)) & (kWords - 4);  // 8 distinct chunks
                const uint4 v = *reinterpret_cast<const uint4 *>(&tile[w]);
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
}

template <int MODE>
double run(int sms, const char *name, double per_op_units, const char *unit) {
    const int grid = sms * kCtasPerSm;
    unsigned long long *cyc;
    uint32_t *sink;
    cudaMalloc(&cyc, grid * 8);
    cudaMalloc(&sink, 4);
    smem_kernel<MODE><<<grid, kThreads>>>(cyc, sink);  // warm-up
    smem_kernel<MODE><<<grid, kThreads>>>(cyc, sink);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(grid);
    cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    const double cycles = (double)h[grid / 2];  // median CTA (the 4 CTAs of an SM overlap)
    const double ops_per_sm = (double)kCtasPerSm * kThreads * kIters * 8;  // lane operations
    const double rate = ops_per_sm / cycles * per_op_units;
    printf("%-40s %8.2f %s per SM per cycle (median CTA %.0f cycles)\n", name, rate, unit, cycles);
    cudaFree(cyc);
    cudaFree(sink);
    return rate;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, dev);
    printf("%s, %d SMs, max SM clock %.0f MHz; 4 CTAs x 256 threads per SM\n", p.name, sms, clk / 1e3);
    run<0>(sms, "red.shared.and.b32 random words (8 KB)", 1.0, "lanes");
    run<1>(sms, "red.shared.and.b32 lane-distinct banks", 1.0, "lanes");
    run<2>(sms, "LDS.128 consecutive (conflict-free)", 16.0, "bytes");
    return 0;
}

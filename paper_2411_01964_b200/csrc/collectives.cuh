// collectives.cuh -- the small device-wide collectives of the hot path,
// hand-written (no CUB device kernels on the per-call path):
//   * scan_counts_kernel: exclusive prefix sum of n uint32 counts into n + 1
//     offsets (offsets[n] = total) by ONE CTA -- the inputs are per-segment or
//     per-bucket-tile counts (<= 2^15 in the prime generator, <= 2^25 in the
//     rare exact-bucket fallback), a single pass over them costs less than the
//     two launches of a decoupled look-back scan;
//   * bitonic sorts of the (normally empty) failure list: one CTA in shared
//     memory up to kSortSmem keys, global merge steps beyond.
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace sqf2k {

constexpr int kScanThreads = 1024;

// Exclusive scan of one value per thread across a CTA of NT threads (a
// multiple of 32, <= 1024); returns the prefix, *total gets the CTA sum.
// warp_sums: NT / 32 shared entries.
template <class T, int NT = kScanThreads>
__device__ __forceinline__ T block_exclusive_scan(T v, T *warp_sums, T *total) {
    static_assert(NT % 32 == 0 && NT <= 1024, "whole warps");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T s = lane < NT / 32 ? warp_sums[lane] : T(0);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= d) s += y;
        }
        if (lane < NT / 32) warp_sums[lane] = s;  // inclusive warp prefix
    }
    __syncthreads();
    const T before = warp ? warp_sums[warp - 1] : T(0);
    *total = warp_sums[NT / 32 - 1];
    __syncthreads();  // warp_sums may be reused by the caller's next round
    return before + x - v;
}

// (kernels: internal linkage, one copy per translation unit that uses them)
namespace {

// offsets[i] = sum of counts[0 .. i), i = 0 .. n (one CTA, kScanThreads).
// Thread t owns the contiguous run [t * per, (t + 1) * per): one read pass for
// the run sums, one block scan, one write pass.
template <class Out>
__global__ void __launch_bounds__(kScanThreads) scan_counts_kernel(const uint32_t *__restrict__ counts,
                                                                   uint64_t n, Out *__restrict__ offsets) {
    __shared__ unsigned long long warp_sums[32];
    const uint64_t per = (n + kScanThreads - 1) / kScanThreads;
    const uint64_t lo = min((uint64_t)threadIdx.x * per, n), hi = min(lo + per, n);
    unsigned long long s = 0;
    for (uint64_t i = lo; i < hi; ++i) s += counts[i];
    unsigned long long total;
    unsigned long long run = block_exclusive_scan<unsigned long long>(s, warp_sums, &total);
    for (uint64_t i = lo; i < hi; ++i) {
        offsets[i] = (Out)run;
        run += counts[i];
    }
    if (threadIdx.x == 0) offsets[n] = (Out)total;
}

// ---- failure sort -------------------------------------------------------------

constexpr int kSortSmem = 4096;  // keys sorted by one CTA in shared memory

// Sort n <= kSortSmem keys in place (one CTA of kScanThreads threads).
__global__ void __launch_bounds__(kScanThreads) sort_small_kernel(unsigned long long *keys, uint32_t n) {
    __shared__ unsigned long long s[kSortSmem];
    uint32_t m = 1;
    while (m < n) m <<= 1;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) s[i] = i < n ? keys[i] : ~0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= m; k <<= 1) {
        for (uint32_t j = k >> 1; j; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    if ((s[i] > s[l]) == up) {
                        const unsigned long long t = s[i];
                        s[i] = s[l];
                        s[l] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) keys[i] = s[i];
}

// One compare-exchange step (k, j) of a bitonic sort over m = 2^e keys in HBM.
__global__ void bitonic_step_kernel(unsigned long long *keys, uint64_t m, uint64_t k, uint64_t j) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t l = i ^ j;
        if (l > i) {
            unsigned long long a = keys[i], b = keys[l];
            const bool up = (i & k) == 0;
            if ((a > b) == up) {
                keys[i] = b;
                keys[l] = a;
            }
        }
    }
}

__global__ void pad_keys_kernel(unsigned long long *keys, uint64_t n, uint64_t m) {
    for (uint64_t i = n + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = ~0ull;
}

}  // namespace

}  // namespace sqf2k

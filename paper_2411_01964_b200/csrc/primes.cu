// primes.cu -- L0 prime table on the GPU (replaces primes.py:26-40).
//
// All primes <= limit (limit <= 2^32) as ascending uint32:
//   1. base primes <= isqrt(limit) by one CTA (Eratosthenes in shared memory);
//   2. segmented odd-only sieve, one CTA per 2^16 odd numbers, bits in shared
//      memory, per-segment popcount;
//   3. exclusive scan of the segment counts (CUB) and an in-order compaction.
// Output index 0 is the prime 2.  Runs once per verify call.
#include <algorithm>
#include <cmath>

#include <cub/cub.cuh>

#include "common.cuh"
#include "tile.cuh"

namespace sqf2k {

namespace {

constexpr int kSegOdds = 1 << 16;          // odd numbers per segment
constexpr int kSegWords = kSegOdds / 32;   // 2048 u32 words
constexpr int kSieveThreads = 512;
constexpr int kMaxBase = 6600;             // pi(65536) = 6542 >= pi(isqrt(2^32))

// Split of a table holding every prime <= limit: positional (kPiPow2).
__device__ void fill_info(PrimeInfo *info, unsigned long long n) {
    info->count = n;
    info->i_lo = (uint32_t)min(n, (unsigned long long)kPiBelowPMed);
    info->i_hi = (uint32_t)n;
    for (int j = 0; j <= kClasses; ++j) info->cls[j] = (uint32_t)min(n, (unsigned long long)pi_pow2(j));
}

// Whole table for limit < 2^17 (one segment) in one CTA: base primes, a byte
// per odd candidate in shared memory (plain byte stores, no atomics), ordered
// compaction and the split.
__global__ void __launch_bounds__(kSieveThreads) prime_small_kernel(uint64_t limit,
                                                                     uint32_t *__restrict__ out,
                                                                     PrimeInfo *__restrict__ info) {
    extern __shared__ uint8_t flag[];  // flag[i] for the odd number 2i+1
    __shared__ uint32_t base[128];
    __shared__ uint32_t nbase;
    const uint32_t r = (uint32_t)isqrt_u64(limit);  // <= 362
    const uint32_t n_idx = (uint32_t)((limit + 1) / 2);  // odd numbers <= limit
    if (threadIdx.x < 32) {
        // odd base primes <= r by trial division, ordered by a warp ballot
        uint32_t nb = 0;
        for (uint32_t c0 = 3; c0 <= r; c0 += 64) {
            const uint32_t cand = c0 + 2 * threadIdx.x;
            bool prime = cand <= r;
            for (uint32_t d = 3; prime && d * d <= cand; d += 2) prime = cand % d != 0;
            const uint32_t bal = __ballot_sync(0xffffffffu, prime);
            if (prime) base[nb + __popc(bal & ((1u << threadIdx.x) - 1u))] = cand;
            nb += __popc(bal);
        }
        if (threadIdx.x == 0) nbase = nb;
    }
    for (uint32_t i = threadIdx.x; i < n_idx; i += blockDim.x) flag[i] = i != 0;  // 1 is not prime
    __syncthreads();
    for (uint32_t k = 0; k < nbase; ++k) {
        const uint32_t p = base[k];
        for (uint32_t i = (p * p - 1) / 2 + threadIdx.x * p; i < n_idx; i += blockDim.x * p)
            flag[i] = 0;
    }
    __syncthreads();
    const uint32_t chunk = (n_idx + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(threadIdx.x * chunk, n_idx), hi = min(lo + chunk, n_idx);
    uint32_t cnt = 0;
    for (uint32_t i = lo; i < hi; ++i) cnt += flag[i];
    using Scan = cub::BlockScan<uint32_t, kSieveThreads>;
    __shared__ typename Scan::TempStorage tmp;
    uint32_t off, total;
    Scan(tmp).ExclusiveSum(cnt, off, total);
    uint32_t pos = off + (limit >= 2 ? 1 : 0);
    for (uint32_t i = lo; i < hi; ++i)
        if (flag[i]) out[pos++] = 2 * i + 1;
    if (threadIdx.x == 0) {
        if (limit >= 2) out[0] = 2;
        fill_info(info, total + (limit >= 2 ? 1 : 0));
    }
}

// Odd base primes 3..r (r <= 65536) into base[], count into *nbase.
__global__ void __launch_bounds__(1024) base_primes_kernel(uint32_t r, uint32_t *base,
                                                           uint32_t *nbase) {
    extern __shared__ uint8_t comp[];  // comp[i] for odd 2i+1, i < (r+1)/2
    const uint32_t n = (r + 1) / 2 + 1;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) comp[i] = (i == 0);
    __syncthreads();
    for (uint32_t p = 3; p * p <= r; p += 2) {
        if (!comp[(p - 1) / 2]) {
            for (uint32_t m = p * p + 2 * p * threadIdx.x; m <= r; m += 2 * p * blockDim.x)
                comp[(m - 1) / 2] = 1;
        }
        __syncthreads();
    }
    // ordered compaction with a block scan over per-thread chunks
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    const uint32_t last = (r - 1) / 2;  // largest index with 2i+1 <= r
    const uint32_t chunk = (last + blockDim.x) / blockDim.x;
    uint32_t lo = 1 + threadIdx.x * chunk, hi = min(lo + chunk, last + 1);
    uint32_t cnt = 0;
    for (uint32_t i = lo; i < hi; ++i) cnt += !comp[i];
    uint32_t off;
    Scan(tmp).ExclusiveSum(cnt, off);
    for (uint32_t i = lo; i < hi; ++i)
        if (!comp[i]) base[off++] = 2 * i + 1;
    if (threadIdx.x == blockDim.x - 1) *nbase = off;
}

// One segment of odd numbers m = 2i+1, i in [seg*kSegOdds, +kSegOdds).
__global__ void __launch_bounds__(kSieveThreads) prime_segment_kernel(
    uint64_t limit, const uint32_t *__restrict__ base, const uint32_t *__restrict__ nbase_p,
    uint32_t *__restrict__ bits, uint32_t *__restrict__ counts) {
    __shared__ uint32_t w[kSegWords];
    __shared__ uint32_t first[kMaxBase];
    const uint32_t nbase = *nbase_p;
    const uint64_t i_lo = (uint64_t)blockIdx.x * kSegOdds;
    const uint64_t m_lo = 2 * i_lo + 1, m_hi = m_lo + 2 * (uint64_t)kSegOdds;  // [m_lo, m_hi)
    for (int j = threadIdx.x; j < kSegWords; j += blockDim.x) {
        // valid odd m in [3, limit]
        uint64_t m0 = m_lo + 64ull * j;
        uint32_t word = 0xffffffffu;
        if (m0 + 62 > limit) {
            word = 0;
            for (int b = 0; b < 32; ++b)
                if (m0 + 2ull * b <= limit) word |= 1u << b;
        }
        if (m0 == 1) word &= ~1u;
        w[j] = word;
    }
    // first index (relative to the segment) of an odd multiple of p >= max(p^2, m_lo)
    for (uint32_t k = threadIdx.x; k < nbase; k += blockDim.x) {
        uint64_t p = base[k];
        uint64_t m = p * p;
        if (m < m_lo) {
            m = (m_lo + p - 1) / p * p;
            if (!(m & 1)) m += p;
        }
        first[k] = m >= m_hi ? 0xffffffffu : (uint32_t)((m - m_lo) / 2);
    }
    __syncthreads();
    // small primes: every thread strides over the hits of one prime
    uint32_t k = 0;
    for (; k < nbase && base[k] < 2048; ++k) {
        uint32_t p = base[k], i0 = first[k];
        if (i0 == 0xffffffffu) continue;
        for (uint32_t i = i0 + threadIdx.x * p; i < (uint32_t)kSegOdds; i += blockDim.x * p)
            atomicAnd(&w[i >> 5], ~(1u << (i & 31)));
    }
    // larger primes: one prime per thread (< 32 hits each)
    for (uint32_t kk = k + threadIdx.x; kk < nbase; kk += blockDim.x) {
        uint32_t p = base[kk];
        for (uint32_t i = first[kk]; i < (uint32_t)kSegOdds; i += p)
            atomicAnd(&w[i >> 5], ~(1u << (i & 31)));
    }
    __syncthreads();
    uint32_t cnt = 0;
    for (int j = threadIdx.x; j < kSegWords; j += blockDim.x) {
        uint32_t word = w[j];
        bits[(uint64_t)blockIdx.x * kSegWords + j] = word;
        cnt += __popc(word);
    }
    using Red = cub::BlockReduce<uint32_t, kSieveThreads>;
    __shared__ typename Red::TempStorage rt;
    uint32_t tot = Red(rt).Sum(cnt);
    if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

// Write the primes of one segment in ascending order at offsets[seg] (+1 for 2).
__global__ void __launch_bounds__(kSieveThreads) prime_compact_kernel(
    const uint32_t *__restrict__ bits, const uint64_t *__restrict__ offsets,
    uint32_t *__restrict__ out, int with_two, const uint64_t *__restrict__ total,
    PrimeInfo *__restrict__ info) {
    constexpr int kPer = kSegWords / kSieveThreads;  // 4 words per thread
    const uint32_t *w = bits + (uint64_t)blockIdx.x * kSegWords + threadIdx.x * kPer;
    uint32_t v[kPer], cnt = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        v[j] = w[j];
        cnt += __popc(v[j]);
    }
    using Scan = cub::BlockScan<uint32_t, kSieveThreads>;
    __shared__ typename Scan::TempStorage tmp;
    uint32_t off;
    Scan(tmp).ExclusiveSum(cnt, off);
    uint64_t pos = offsets[blockIdx.x] + off + (with_two ? 1 : 0);
    const uint64_t i_base = (uint64_t)blockIdx.x * kSegOdds + (uint64_t)threadIdx.x * kPer * 32;
#pragma unroll
    for (int j = 0; j < kPer; ++j)
        for (uint32_t x = v[j]; x; x &= x - 1) {
            uint64_t i = i_base + 32 * j + __ffs(x) - 1;
            out[pos++] = (uint32_t)(2 * i + 1);
        }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (with_two) out[0] = 2;
        // the table is every prime <= limit: the split is positional
        const unsigned long long n = *total + (with_two ? 1 : 0);
        fill_info(info, n);
    }
}

__global__ void widen_kernel(const uint32_t *__restrict__ in, int64_t *__restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

}  // namespace

uint64_t pi_upper(uint64_t x) {
    // pi(x) < 1.25506 x / ln x for x > 1 (Rosser & Schoenfeld)
    if (x < 17) return 8;
    return (uint64_t)(1.25506 * (double)x / std::log((double)x)) + 16;
}

// Launch the generator for every prime <= limit; count and split land in
// ctx.prime_info (device), the table in ctx.primes_u32.  No host sync.
void generate_primes_async(uint64_t limit) {
    Context &c = ctx();
    if (limit > 0xffffffffull) throw Error{SQF2K_EINVAL, "prime limit above 2^32"};
    c.primes_limit = limit;
    c.primes_u32.reserve(256);
    c.prime_info.reserve(sizeof(PrimeInfo));
    PrimeInfo *info = c.prime_info.as<PrimeInfo>();
    if (limit < 2) {
        SQF2K_CUDA(cudaMemsetAsync(info, 0, sizeof(PrimeInfo), c.stream));
        return;
    }
    uint32_t r = (uint32_t)isqrt_u64(limit);
    if (r < 3) r = 3;
    const uint64_t n_odd = (limit + 1) / 2;  // odd numbers 1..limit (index i <-> 2i+1)
    const uint64_t nseg = ceil_div(n_odd, kSegOdds);
    if (nseg == 1) {  // small tables: one CTA does everything
        c.primes_u32.reserve(pi_upper(limit) * 4);
        static bool attr = false;
        if (!attr) {
            SQF2K_CUDA(cudaFuncSetAttribute(prime_small_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, kSegOdds));
            attr = true;
        }
        launch("primes_small", prime_small_kernel, dim3(1), dim3(kSieveThreads),
               (size_t)std::max<uint64_t>(n_odd, 16), limit, c.primes_u32.as<uint32_t>(), info);
        return;
    }

    c.prime_bits.reserve(nseg * kSegWords * 4 + (kMaxBase + 1) * 4);
    c.prime_counts.reserve((nseg + 2) * 4);  // counts[0..nseg] + base-prime count
    c.prime_offsets.reserve((nseg + 1) * 8);
    c.primes_u32.reserve(pi_upper(limit) * 4);
    uint32_t *bits = c.prime_bits.as<uint32_t>();
    uint32_t *base = bits + nseg * kSegWords;  // tail of the same allocation
    uint32_t *counts = c.prime_counts.as<uint32_t>();
    uint32_t *nbase = counts + nseg + 1;

    launch("primes_base", base_primes_kernel, dim3(1), dim3(1024), (size_t)(r + 1) / 2 + 2, r,
           base, nbase);
    launch("primes_sieve", prime_segment_kernel, dim3((unsigned)nseg), dim3(kSieveThreads), 0,
           limit, (const uint32_t *)base, (const uint32_t *)nbase, bits, counts);
    // exclusive scan of counts (uint32 in, uint64 out); counts[nseg] = 0 puts
    // the total in offsets[nseg]
    uint64_t *offsets = c.prime_offsets.as<uint64_t>();
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, offsets, (int)nseg + 1, c.stream);
    c.scan_tmp.reserve(std::max<size_t>(tmp_bytes, 64));
    SQF2K_CUDA(cudaMemsetAsync(counts + nseg, 0, 4, c.stream));
    SQF2K_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.ptr, tmp_bytes, counts, offsets,
                                             (int)nseg + 1, c.stream));
    launch("primes_compact", prime_compact_kernel, dim3((unsigned)nseg), dim3(kSieveThreads), 0,
           (const uint32_t *)bits, (const uint64_t *)offsets, c.primes_u32.as<uint32_t>(), 1,
           offsets + nseg, info);
}

// Generate every prime <= limit into ctx.primes_u32; returns the count.
uint64_t generate_primes_device(uint64_t limit) {
    Context &c = ctx();
    generate_primes_async(limit);
    PrimeInfo h;
    copy_d2h(&h, c.prime_info.ptr, sizeof h);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    c.primes_count = h.count;
    return h.count;
}

void widen_primes(const uint32_t *in, int64_t *out, uint64_t n) {
    if (!n) return;
    unsigned blocks = (unsigned)std::min<uint64_t>(ceil_div(n, 256), 4096);
    launch("primes_widen", widen_kernel, dim3(blocks), dim3(256), 0, in, out, n);
}

}  // namespace sqf2k

using namespace sqf2k;

extern "C" int sqf2k_prime_count(uint64_t limit, uint64_t *count) {
    if (limit < 1) return fail(SQF2K_EINVAL, "limit must be positive, got %llu",
                               (unsigned long long)limit);
    return guarded([=](Context &) -> int {
        *count = generate_primes_device(limit);
        return SQF2K_OK;
    });
}

extern "C" int sqf2k_primes(uint64_t limit, int64_t *out, uint64_t cap, uint64_t *count) {
    if (limit < 1) return fail(SQF2K_EINVAL, "limit must be positive, got %llu",
                               (unsigned long long)limit);
    return guarded([=](Context &c) -> int {
        uint64_t n = generate_primes_device(limit);
        *count = n;
        if (n > cap) return fail(SQF2K_ECAPACITY, "prime buffer holds %llu, need %llu",
                                 (unsigned long long)cap, (unsigned long long)n);
        if (n) {
            c.host_primes.reserve(n * 8);
            widen_primes(c.primes_u32.as<uint32_t>(), c.host_primes.as<int64_t>(), n);
            copy_d2h(out, c.host_primes.ptr, n * 8);
            SQF2K_CUDA(cudaStreamSynchronize(c.stream));
        }
        return SQF2K_OK;
    });
}

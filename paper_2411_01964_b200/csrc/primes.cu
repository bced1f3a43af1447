// primes.cu -- L0 prime table on the GPU (replaces primes.py:26-40).
//
// All primes <= limit (limit <= 2^32) as ascending uint32:
//   1. base primes <= isqrt(limit) by one CTA (Eratosthenes in shared memory);
//   2. segmented odd-only sieve, one CTA per 2^16 odd numbers, bits in shared
//      memory, per-segment popcount;
//   3. exclusive scan of the segment counts (one CTA, collectives.cuh) and an
//      in-order compaction.
// Output index 0 is the prime 2.  Runs once per verify call.
#include <algorithm>
#include <cmath>

#include "collectives.cuh"
#include "common.cuh"
#include "tile.cuh"

namespace sqf2k {

namespace {

constexpr int kSegOdds = 1 << 16;          // odd numbers per segment
constexpr int kSegWords = kSegOdds / 32;   // 2048 u32 words
constexpr int kSieveThreads = 512;
constexpr int kMaxBase = 6600;             // pi(65536) = 6542 >= pi(isqrt(2^32))

__constant__ uint32_t c_pi_pow2[kClasses + 1] = SQF2K_PI_POW2;

// Split of a table holding every prime <= limit: positional (pi(2^m)).
__device__ void fill_info(PrimeInfo *info, unsigned long long n) {
    info->count = n;
    info->i_lo = (uint32_t)min(n, (unsigned long long)kPiBelowPMed);
    info->i_hi = (uint32_t)n;
#pragma unroll
    for (int j = 0; j <= kClasses; ++j) info->cls[j] = (uint32_t)min(n, (unsigned long long)c_pi_pow2[j]);
}

// Whole table for limit < 2^17 (at most 2048 words of odd candidates) in one
// CTA of 1024 threads, a bit per odd candidate in shared memory: the ten odd
// primes below 32 are applied per word as shifted periodic patterns (i0 mod
// p by a multiply-high with a magic constant, exact for i0 < 2^16), the
// larger base primes clear their multiples from p^2 with shared-memory
// atomics spread over all threads (~7 per thread at limit 2^15).  Ordered
// compaction: block scan, primes staged in shared memory, one coalesced
// copy out.
constexpr int kSmallThreads = 1024;
constexpr int kSmallStage = 12288;  // > pi(2^17) = 12251
constexpr int kNumOddBase = 71;     // odd primes <= 361 = isqrt(2^17 - 1)
__constant__ uint16_t c_odd_base[kNumOddBase] = {
    3,   5,   7,   11,  13,  17,  19,  23,  29,  31,  37,  41,  43,  47,  53,  59,  61,  67,
    71,  73,  79,  83,  89,  97,  101, 103, 107, 109, 113, 127, 131, 137, 139, 149, 151, 157,
    163, 167, 173, 179, 181, 191, 193, 197, 199, 211, 223, 227, 229, 233, 239, 241, 251, 257,
    263, 269, 271, 277, 281, 283, 293, 307, 311, 313, 317, 331, 337, 347, 349, 353, 359};
// floor(2^32 / p) + 1: floor(i0 / p) = umulhi(i0, magic) for i0 < 2^16
__constant__ uint32_t c_odd_magic[kNumOddBase] = {
    1431655766u, 858993460u, 613566757u, 390451573u, 330382100u, 252645136u,
    226050911u, 186737709u, 148102321u, 138547333u, 116080198u, 104755300u,
    99882961u, 91382283u, 81037119u, 72796056u, 70409300u, 64103990u,
    60492498u, 58835169u, 54366675u, 51746594u, 48258060u, 44278014u,
    42524429u, 41698712u, 40139882u, 39403370u, 38008561u, 33818641u,
    32786010u, 31350127u, 30899046u, 28825284u, 28443493u, 27356480u,
    26349493u, 25718368u, 24826401u, 23994231u, 23729102u, 22486740u,
    22253717u, 21801865u, 21582751u, 20355296u, 19259944u, 18920561u,
    18755316u, 18433337u, 17970575u, 17821442u, 17111424u, 16711936u,
    16330675u, 15966422u, 15848588u, 15505298u, 15284582u, 15176563u,
    14658592u, 13990122u, 13810185u, 13721941u, 13548793u, 12975733u,
    12744711u, 12377428u, 12306497u, 12167047u, 11963698u,
};
// bits 0, p, 2p, ... < 32 for the ten odd primes below 32
__constant__ uint32_t c_odd_rep[10] = {0x49249249u, 0x42108421u, 0x10204081u, 0x400801u,
                                       0x4002001u,  0x20001u,    0x80001u,    0x800001u,
                                       0x20000001u, 0x80000001u};

struct SmallTables {
    uint32_t p[kNumOddBase], magic[kNumOddBase], rep[10];
};

// word w with the multiples of the odd primes below 32 (other than
// themselves) cleared; nb10 = how many of them have p^2 <= limit
__device__ __forceinline__ uint32_t small_word(const SmallTables &T, uint32_t w, uint32_t n_idx,
                                               uint32_t nb10) {
    const uint32_t i0 = 32 * w;
    uint32_t v = i0 + 32 <= n_idx ? ~0u : (i0 >= n_idx ? 0u : (1u << (n_idx - i0)) - 1u);
    if (w == 0) v &= ~1u;  // 1 is not prime
    uint32_t mask = 0;
#pragma unroll
    for (uint32_t k = 0; k < 10; ++k) {
        if (k >= nb10) break;
        const uint32_t p = T.p[k];
        const uint32_t r = i0 - p * __umulhi(i0, T.magic[k]);  // i0 mod p
        const uint32_t hp = (p - 1) / 2;  // p | 2i + 1  <=>  i = hp mod p
        const uint32_t y = hp >= r ? hp - r : hp + p - r;  // first such i >= i0, minus i0
        mask |= T.rep[k] << y;
    }
    if (w == 0) mask &= ~0xcb6eu;  // bits (p-1)/2 of the primes 3..31 themselves
    return v & ~mask;
}

__global__ void __launch_bounds__(kSmallThreads) prime_small_kernel(uint64_t limit,
                                                                     uint32_t *__restrict__ out,
                                                                     PrimeInfo *__restrict__ info) {
    grid_dependents_launch();  // the bucket fill may launch now (it waits for this grid)
    extern __shared__ uint32_t stage[];  // kSmallStage primes
    // the constant tables go to shared memory in one parallel round trip (a
    // cold constant cache would serialise one miss per line inside the loop)
    __shared__ SmallTables T;
    __shared__ uint32_t s_nb;
    if (threadIdx.x < kNumOddBase) {
        const uint32_t p = c_odd_base[threadIdx.x];
        T.p[threadIdx.x] = p;
        T.magic[threadIdx.x] = c_odd_magic[threadIdx.x];
        if (threadIdx.x < 10) T.rep[threadIdx.x] = c_odd_rep[threadIdx.x];
        // odd base primes with p^2 <= limit: the last one records the count
        const bool in = (uint64_t)p * p <= limit;
        const bool next_in = threadIdx.x + 1 < kNumOddBase &&
                             (uint64_t)c_odd_base[threadIdx.x + 1] * c_odd_base[threadIdx.x + 1] <= limit;
        if (threadIdx.x == 0 && !in) s_nb = 0;
        if (in && !next_in) s_nb = threadIdx.x + 1;
    }
    __syncthreads();
    const uint32_t nb = s_nb;
    const uint32_t n_idx = (uint32_t)((limit + 1) / 2);  // odd numbers <= limit (index i: 2i+1)
    const uint32_t n_words = (n_idx + 31) / 32;
    const uint32_t wpt = n_words <= kSmallThreads ? 1 : 2;
    const uint32_t w0 = wpt * threadIdx.x;
    __shared__ __align__(8) uint32_t bits[2 * kSmallThreads];
    bits[w0] = small_word(T, w0, n_idx, min(nb, 10u));
    if (wpt == 2) bits[w0 + 1] = small_word(T, w0 + 1, n_idx, min(nb, 10u));
    __syncthreads();
    if (nb > 10) {  // p >= 37: clear p^2, p^2 + 2p, ... ; nl threads per prime
        const uint32_t np = nb - 10, nl = kSmallThreads / np;
        const uint32_t g = threadIdx.x % np, l = threadIdx.x / np;
        if (l < nl) {
            const uint32_t p = T.p[10 + g];
            for (uint32_t i = (p * p - 1) / 2 + l * p; i < n_idx; i += nl * p)
                atomicAnd(&bits[i >> 5], ~(1u << (i & 31)));
        }
        __syncthreads();
    }
    const uint32_t v0 = bits[w0];
    const uint32_t v1 = wpt == 2 ? bits[w0 + 1] : 0u;
    __shared__ uint32_t sums[kSmallThreads / 32];
    uint32_t total;
    uint32_t off = block_exclusive_scan<uint32_t, kSmallThreads>((uint32_t)(__popc(v0) + __popc(v1)),
                                                                 sums, &total);
    for (uint32_t x = v0; x; x &= x - 1) stage[off++] = 2 * (32 * w0 + __ffs(x) - 1) + 1;
    for (uint32_t x = v1; x; x &= x - 1) stage[off++] = 2 * (32 * w0 + 32 + __ffs(x) - 1) + 1;
    __syncthreads();
    const uint32_t two = limit >= 2 ? 1 : 0;
    for (uint32_t i = threadIdx.x; i < total; i += kSmallThreads) out[two + i] = stage[i];
    if (threadIdx.x == 0) {
        if (two) out[0] = 2;
        fill_info(info, total + two);
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
    __shared__ uint32_t sums[32];
    const uint32_t last = (r - 1) / 2;  // largest index with 2i+1 <= r
    const uint32_t chunk = (last + blockDim.x) / blockDim.x;
    uint32_t lo = 1 + threadIdx.x * chunk, hi = min(lo + chunk, last + 1);
    uint32_t cnt = 0;
    for (uint32_t i = lo; i < hi; ++i) cnt += !comp[i];
    uint32_t tot;
    uint32_t off = block_exclusive_scan<uint32_t, 1024>(cnt, sums, &tot);
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
    __shared__ uint32_t sums[kSieveThreads / 32];
    uint32_t tot;
    block_exclusive_scan<uint32_t, kSieveThreads>(cnt, sums, &tot);
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
    __shared__ uint32_t sums[kSieveThreads / 32];
    uint32_t tot;
    const uint32_t off = block_exclusive_scan<uint32_t, kSieveThreads>(cnt, sums, &tot);
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
        static_assert(kSegWords <= 2 * kSmallThreads, "prime_small_kernel: <= 2 words per thread");
        static bool attr = false;
        if (!attr) {
            SQF2K_CUDA(cudaFuncSetAttribute(prime_small_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            kSmallStage * 4));
            attr = true;
        }
        launch("primes_small", prime_small_kernel, dim3(1), dim3(kSmallThreads),
               (size_t)kSmallStage * 4, limit, c.primes_u32.as<uint32_t>(), info);
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
    // exclusive scan of the nseg segment counts (uint32 in, uint64 out);
    // offsets[nseg] = the total
    uint64_t *offsets = c.prime_offsets.as<uint64_t>();
    launch("primes_scan", scan_counts_kernel<uint64_t>, dim3(1), dim3(kScanThreads), 0,
           (const uint32_t *)counts, nseg, offsets);
    launch("primes_compact", prime_compact_kernel, dim3((unsigned)nseg), dim3(kSieveThreads), 0,
           (const uint32_t *)bits, (const uint64_t *)offsets, c.primes_u32.as<uint32_t>(), 1,
           offsets + nseg, info);
}

// The table only if the cached one does not already hold every prime <=
// limit (a larger table is fine for trial division: warp_squarefree stops at
// p^2 > m).  The verify path always regenerates (a run builds its table,
// runner.py:192); recheck and is_squarefree reuse it.
void ensure_primes(uint64_t limit) {
    Context &c = ctx();
    if (c.primes_limit >= std::max<uint64_t>(limit, 2)) return;
    generate_primes_async(limit);
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

// tile.cu -- one batch of the tile pipeline: the p = 3, 5, 7 pattern table,
// the bucketed large-prime hit lists and the tile kernel (fused sieve +
// min-k scan, or sieve export).  No host synchronisation inside a batch.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <tuple>
#include <vector>

#include "collectives.cuh"
#include "common.cuh"
#include "finish.cuh"
#include "tile.cuh"

namespace sqf2k {

namespace {

#ifndef SQF2K_WAIT_SLEEP_NS
#define SQF2K_WAIT_SLEEP_NS 0
#endif
#ifndef SQF2K_WAIT_HINT_NS
#define SQF2K_WAIT_HINT_NS 1000000
#endif
#ifndef SQF2K_TMA_START
#define SQF2K_TMA_START 1
#endif
#ifndef SQF2K_START_BARS
#define SQF2K_START_BARS 1
#endif
// the thread that issues the tile starts' bulk copies and waits for them
#ifndef SQF2K_START_WARP
#define SQF2K_START_WARP 0
#endif
constexpr uint32_t kStarter = 32 * SQF2K_START_WARP;
// tile starts by one bulk copy from the pattern table need 16-byte aligned
// sources: four copies of the table, shifted by one word each
constexpr uint32_t kPatCopies = SQF2K_TMA_START ? 4 : 1;
constexpr uint32_t kPatStride = (kPatWordsMax + kTileWords + 3) / 4 * 4;

// -------------------------------------------------------------------------
// p = 3, 5, 7 (11): word g of the domain (slots 32g..32g+31) with every slot
// u such that 9, 25, 49 (or 121) divides n(u) cleared.  Period pattern_words
// words; the first kTileWords words are repeated after the period so that a
// tile's words [pbase, pbase + kTileWords) never wrap.
// First hit at or after 32g: y = (r - 32g) mod q; the word's hits are the
// bits y, y+q, ... < 32, i.e. (bits 0, q, 2q, ...) << y.
struct PatResidues {
    uint32_t r[5];  // slot_residue(base_n, q) for q = 9, 25, 49, 121, 169 (host-computed)
};

__global__ void pattern_kernel(PatResidues res, uint32_t present, uint32_t *__restrict__ table,
                               uint32_t words, uint32_t copies, uint32_t stride) {
    constexpr uint32_t q[5] = {9, 25, 49, 121, 169};
    const uint32_t pat[5] = {0x08040201u, 0x02000001u, 0x1u, 0x1u, 0x1u};
    // Copy r (at table + r * stride, copies <= 4) holds word g at index g - r,
    // so a tile start at any pattern index has a 16-byte aligned source
    // (kinds 0 and 1; kind 2 has one copy of four periods).  Thread i builds
    // the aligned 4-word chunks c = i, i + T, ... of every copy: words 4c ..
    // 4c + 6 once, then one 16-byte store per copy (chunk c of copy r is
    // words 4c + r .. 4c + r + 3).  First-hit offsets step by -32 slots per
    // word and by -128T per chunk, mod q; the residues of base_n come from
    // the host, the per-thread offsets are 32-bit constant-divisor
    // remainders (the 64-bit remainders and the scalar stores of the first
    // version took 14 us for the kind-1 table, now ~5).
    const uint32_t T = gridDim.x * blockDim.x, c0 = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n_chunks = (words + 3) / 4;
    uint32_t y[5], dec[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const uint32_t off = (128u * (c0 % q[i])) % q[i];  // 32 * 4 c0 mod q
        y[i] = (res.r[i] + q[i] - off) % q[i];
        dec[i] = (128u * (T % q[i])) % q[i];
    }
    for (uint32_t c = c0; c < n_chunks; c += T) {
        uint32_t w[7], yy[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) yy[i] = y[i];
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            uint32_t clr = 0;
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const uint32_t d1 = 32u % q[i];
                if (((present >> i) & 1u) && yy[i] < 32) clr |= pat[i] << yy[i];
                yy[i] = yy[i] >= d1 ? yy[i] - d1 : yy[i] + q[i] - d1;
            }
            w[k] = ~clr;
        }
#pragma unroll
        for (uint32_t r = 0; r < 4; ++r)
            if (r < copies)
                *reinterpret_cast<uint4 *>(table + (size_t)r * stride + 4ull * c) =
                    make_uint4(w[r], w[r + 1], w[r + 2], w[r + 3]);
#pragma unroll
        for (int i = 0; i < 5; ++i) y[i] = y[i] >= dec[i] ? y[i] - dec[i] : y[i] + q[i] - dec[i];
    }
}

PatResidues pat_residues(int64_t base_n) {
    PatResidues p;
    const uint64_t q[5] = {9, 25, 49, 121, 169};
    for (int i = 0; i < 5; ++i) p.r[i] = (uint32_t)slot_residue(base_n, q[i]);
    return p;
}

// Kind-2 table (tile.cuh) as the AND of the p <= 11 table (period P11 words,
// one copy) and the p = 13 words (period 169 words, in shared memory): one
// L2 load and one store per word, where pattern_kernel spends ~25
// instructions per word on the five residues (2.5 ms -> HBM-write-bound for
// the 3.6 GB table).
__global__ void pattern13_kernel(int64_t base_n, const uint32_t *__restrict__ t11, uint32_t *__restrict__ out,
                                 uint32_t words) {
    constexpr uint32_t P11 = kPatWords3 * 121, Q = 169;
    __shared__ uint32_t s13[Q];
    const uint32_t r = (uint32_t)slot_residue(base_n, Q);
    for (uint32_t j = threadIdx.x; j < Q; j += blockDim.x) {
        const uint32_t y = (r + Q - (32u * j) % Q) % Q;  // first hit at or after slot 32j
        s13[j] = y < 32 ? ~(1u << y) : ~0u;
    }
    __syncthreads();
    const uint32_t T = gridDim.x * blockDim.x, g0 = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t d11 = T % P11, d13 = T % Q;
    uint32_t i11 = g0 % P11, i13 = g0 % Q;
    for (uint32_t g = g0; g < words; g += T) {
        out[g] = __ldg(t11 + i11) & s13[i13];
        i11 += d11;
        if (i11 >= P11) i11 -= P11;
        i13 += d13;
        if (i13 >= Q) i13 -= Q;
    }
}

// -------------------------------------------------------------------------
// Bucket pass: every hit u of a bucket prime (p >= kPMed, p^2 <= n_max) in the
// batch domain [0, U), as a 16-bit offset in the list of bucket tile u >> kBucketShift.
// Work units are (prime, sub-range) pairs of <= 5 hits (see kClasses), one
// flat index space over all classes so each thread runs one short chain.
//   MODE 0 (fixed): hit i of tile t goes to hits[t * kBucketCap + i]; counts
//          beyond the capacity raise *overflow (the batch is then redone in
//          exact mode).
//   MODE 1 (count) / MODE 2 (fill): exact lists after an exclusive scan of
//          the counts; the fill places hits at offsets[t] + (--counts[t]).
// a mod q for q < 2^62 through a double-precision quotient estimate (one
// DMUL with the precomputed 1/q, one 64-bit multiply-subtract): the estimate
// is within 2 of floor(a / q) for a < 2^62, and the fix-ups make it exact --
// ~15 instructions instead of the ~70 of the 64-bit integer remainder routine.
__device__ __forceinline__ uint64_t mod_q(uint64_t a, uint64_t q, double inv_q) {
    const uint64_t f = __double2ull_rz(__ull2double_rn(a) * inv_q);
    int64_t r = (int64_t)(a - f * q);
#pragma unroll
    for (int i = 0; i < 3; ++i) r += r < 0 ? (int64_t)q : 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) r -= r >= (int64_t)q ? (int64_t)q : 0;
    return (uint64_t)r;
}

// slot_residue (tile.cuh) through mod_q: the first slot u >= 0 with q | base_n + 2u
__device__ __forceinline__ uint64_t slot_residue_q(int64_t base_n, uint64_t q, double inv_q) {
    const uint64_t a = base_n >= 0 ? mod_q((uint64_t)base_n, q, inv_q) : 0u;
    const uint64_t an = base_n >= 0 ? (a ? q - a : 0) : mod_q((uint64_t)(-base_n), q, inv_q);
    return (an & 1) ? (an + q) / 2 : an / 2;
}

template <int MODE>
__global__ void __launch_bounds__(256) bucket_kernel(
    const uint32_t *__restrict__ primes, const PrimeInfo *__restrict__ info, int64_t base_n,
    uint64_t U, uint32_t *__restrict__ counts, const uint32_t *__restrict__ offsets,
    uint16_t *__restrict__ hits, unsigned int *__restrict__ overflow, int j_min) {
    grid_dependents_launch();  // the tile kernel may start its prime-free prologue
    grid_dependency_wait();    // launched early (PDL) behind the prime table: wait for it
    static_assert(kClasses <= 32, "one lane per class");
    __shared__ unsigned long long s_end[kClasses];  // cumulative work per class
    __shared__ uint32_t s_lo[kClasses];
    __shared__ unsigned long long s_nsub[kClasses];
    if (threadIdx.x < 32) {  // class table: a lane per class, warp prefix sum
        const int j = threadIdx.x;
        unsigned long long work = 0;
        if (j < kClasses && j >= j_min) {  // (classes below j_min: bucket_dense_kernel)
            const uint32_t p_lo = max(info->cls[j], info->i_lo);
            const uint32_t p_hi = min(info->cls[j + 1], info->i_hi);
            const int sh = min(22 + 2 * j, 62);
            const unsigned long long n_sub = (U + (1ull << sh) - 1) >> sh;
            s_lo[j] = p_lo;
            s_nsub[j] = n_sub;
            work = p_lo < p_hi ? (unsigned long long)(p_hi - p_lo) * n_sub : 0ull;
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long x = __shfl_up_sync(0xffffffffu, work, d);
            if (j >= d) work += x;
        }
        if (j < kClasses) s_end[j] = work;
    }
    __syncthreads();
    const unsigned long long n_work = s_end[kClasses - 1];
    for (unsigned long long w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < n_work;
         w += (uint64_t)gridDim.x * blockDim.x) {
        int j = 0;
        while (w >= s_end[j]) ++j;
        const unsigned long long local = w - (j ? s_end[j - 1] : 0ull);
        const unsigned long long n_sub = s_nsub[j];
        const int sh = min(22 + 2 * j, 62);
        // (prime, sub-range) of the unit: 32-bit division when the class fits
        uint64_t pi, k;
        if (local < (1ull << 32) && n_sub < (1ull << 32)) {
            pi = (uint32_t)local / (uint32_t)n_sub;
            k = (uint32_t)local - (uint32_t)pi * (uint32_t)n_sub;
        } else {
            pi = local / n_sub;
            k = local - pi * n_sub;
        }
        const uint64_t p = primes[s_lo[j] + pi];
        const uint64_t lo = k << sh;
        const uint64_t hi = lo + (1ull << sh) < U ? lo + (1ull << sh) : U;
        const uint64_t q = p * p;
        const double inv_q = 1.0 / (double)q;
        // first slot u >= 0 with q | base_n + 2u (slot_residue), by mod_q
        const uint64_t r = slot_residue_q(base_n, q, inv_q);
        const uint64_t lm = mod_q(lo, q, inv_q);
        // <= 5 hits (q >= 2^(20+2j), range 2^(22+2j)): all atomics in flight
        // together, then the stores -- one round trip, not one per hit
        const uint64_t u0 = lo + (r >= lm ? r - lm : r + q - lm);
        // hits u0 + i q < hi, compared as i q < hi - u0: u0 + i q itself can
        // pass 2^64 near the domain top (q < 2^62, so 4 q does not)
        const uint64_t span = u0 < hi ? hi - u0 : 0;
        int nh = 0;
#pragma unroll
        for (int i = 0; i < 5; ++i) nh += ((uint64_t)i * q < span) ? 1 : 0;
        uint32_t hu[5], pos[5];
        uint32_t bt[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if (i >= nh) break;
            const uint64_t u = u0 + (uint64_t)i * q;
            bt[i] = (uint32_t)(u >> kBucketShift);
            hu[i] = (uint32_t)(u & (kBucketTile - 1));
            if (MODE == 0) pos[i] = atomicAdd(&counts[bt[i]], 1u);
            else if (MODE == 1) atomicAdd(&counts[bt[i]], 1u);
            else pos[i] = atomicSub(&counts[bt[i]], 1u);
        }
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if (i >= nh) break;
            if (MODE == 0) {
                if (pos[i] < (uint32_t)kBucketCap)
                    hits[(uint64_t)bt[i] * kBucketCap + pos[i]] = (uint16_t)hu[i];
                else
                    atomicOr(overflow, 1u);
            } else if (MODE == 2) {
                hits[offsets[bt[i]] + pos[i] - 1u] = (uint16_t)hu[i];
            }
        }
    }
}

// Dense bucket primes (kPMed <= p < 2^(10 + kDenseClasses)) tile-major, for
// the fixed-capacity lists: CTA b owns the kDenseTiles bucket tiles from
// b * kDenseTiles, gathers every dense prime's hits there into shared-memory
// lists (shared atomics) and writes lists and counts out whole -- coalesced
// 128-byte lines, where the prime-major pass pays a global atomic and a
// partial-sector store per hit.  bucket_kernel<0> then appends the sparse
// classes (j >= kDenseClasses).  The dense classes (p < 8192) hold ~90 % of
// the bucket hits.  Measured: C5 449.4 -> 421.8 ms per call, C4 28.7 -> 26.8 ms.
#ifndef SQF2K_DENSE_CLASSES
#define SQF2K_DENSE_CLASSES 3
#endif
#ifndef SQF2K_DENSE_TILES
#define SQF2K_DENSE_TILES 256
#endif
constexpr int kDenseClasses = SQF2K_DENSE_CLASSES;  // 0: prime-major pass only
constexpr int kDenseTiles = SQF2K_DENSE_TILES;
// small domains keep the single prime-major pass (an extra launch on the
// critical path costs more there than the atomics: C2 0.085 vs 0.094 ms)
constexpr uint32_t kDenseMinTiles = 1u << 15;
__host__ __device__ inline int dense_classes(uint32_t n_bt) {
    return n_bt >= kDenseMinTiles ? kDenseClasses : 0;
}
static_assert(kBucketCap % 8 == 0, "lists copied as 16-byte vectors");
__global__ void __launch_bounds__(256) bucket_dense_kernel(
    const uint32_t *__restrict__ primes, const PrimeInfo *__restrict__ info, int64_t base_n,
    uint64_t U, uint32_t *__restrict__ counts, uint16_t *__restrict__ hits,
    unsigned int *__restrict__ overflow) {
    __shared__ uint32_t s_cnt[kDenseTiles];
    __shared__ __align__(16) uint16_t s_hits[kDenseTiles * kBucketCap];
    grid_dependency_wait();  // launched early (PDL) behind the prime table
    for (int i = threadIdx.x; i < kDenseTiles; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    const uint64_t bt0 = (uint64_t)blockIdx.x * kDenseTiles;
    const uint64_t lo = bt0 << kBucketShift;
    const uint64_t hi = min(lo + ((uint64_t)kDenseTiles << kBucketShift), U);
    const uint32_t p_lo = info->i_lo, p_hi = min(info->cls[kDenseClasses], info->i_hi);
    for (uint32_t i = p_lo + threadIdx.x; i < p_hi; i += blockDim.x) {
        const uint64_t p = primes[i], q = p * p;
        const double inv_q = 1.0 / (double)q;
        const uint64_t r = slot_residue_q(base_n, q, inv_q);
        const uint64_t lm = mod_q(lo, q, inv_q);
        for (uint64_t u = lo + (r >= lm ? r - lm : r + q - lm); u < hi; u += q) {
            const uint32_t lt = (uint32_t)((u - lo) >> kBucketShift);
            const uint32_t pos = atomicAdd(&s_cnt[lt], 1u);
            if (pos < (uint32_t)kBucketCap) s_hits[lt * kBucketCap + pos] = (uint16_t)(u & (kBucketTile - 1));
        }
    }
    __syncthreads();
    const uint32_t nt = (uint32_t)((hi - lo + kBucketTile - 1) >> kBucketShift);
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) {
        const uint32_t c = s_cnt[i];
        counts[bt0 + i] = c;
        if (c > (uint32_t)kBucketCap) atomicOr(overflow, 1u);
    }
    uint4 *dst = reinterpret_cast<uint4 *>(hits + bt0 * kBucketCap);
    const uint4 *src = reinterpret_cast<const uint4 *>(s_hits);
    for (uint32_t i = threadIdx.x; i < nt * (kBucketCap / 8); i += blockDim.x) dst[i] = src[i];
}

// -------------------------------------------------------------------------
// Shared memory of a tile CTA.  The tile is sieved directly in packed form:
// 32-bit words, one bit per odd slot, in a ring of kRingTiles tile buffers --
// tile t occupies buffer t mod kRingTiles and its halo (the previous tile's
// last 2^(k_eff-1) slots) is the tail of buffer t - 1.  A word starts as the
// p = 3, 5, 7 pattern; the medium and bucket primes clear their hits with
// shared-memory atomics (random scatter: bank-conflict bound at ~9
// lanes/cycle/SM on B200, the same rate as byte stores, so no byte array and
// no pack pass).
#ifndef SQF2K_SPLIT_PHASE
#define SQF2K_SPLIT_PHASE 1
#endif
// live tiles per phase: t-2 .. t+2 (5), or t-3 .. t+2 with the split phase
// (tiles started 3 ahead, warps up to one phase apart) -- see tile_kernel
constexpr int kRingTiles = SQF2K_SPLIT_PHASE ? 6 : 5;
constexpr int kRingWords = kRingTiles * kTileWords;
__device__ __forceinline__ uint32_t ring_base(uint32_t t) { return (t % kRingTiles) * kTileWords; }
// ring word i - d (d <= kTileWords), wrapping below 0
__device__ __forceinline__ uint32_t ring_back(uint32_t i, uint32_t d) {
    return i >= d ? i - d : i + kRingWords - d;
}
// SQF2K_RING_ALIGN: the ring starts on an 8 KB boundary of the shared
// window (the bookkeeping fields go in front, padded), so every tile buffer
// -- and every halo, whose offset inside its buffer is a multiple of the
// halo's byte length -- is aligned past its largest word offset and a hit's
// word address is one LOP3 ((o >> 3) & 0x1ffc | base) instead of AND + ADD.
#ifndef SQF2K_RING_ALIGN
#define SQF2K_RING_ALIGN 1
#endif
struct TileSmemHead {
    unsigned long long first[kDepthMax + 1];
    uint32_t first_t[2][6];       // k <= 5: least tile-local slot of tile t (buffer t & 1)
    uint32_t need;                // bit k: least n with exponent k still unknown
    uint32_t cnt[kDepthMax + 1];  // counts of k > kMainMax (rare); [0]: slots left after the main passes
    // words left after the main passes of tile t (queue t & 1), finished
    // while tile t + 1 is scanned
    uint32_t res_w[2][kResCap], res_p[2][kResCap];
    uint32_t n_res[2];
    unsigned long long mbar;  // split phase: one arrival per thread per phase
    unsigned long long mbar_start;  // TMA tile starts: one bulk copy per use
    unsigned long long start_bar[kRingTiles];  // SQF2K_START_BARS: buffer b's start landed
    uint32_t last;      // this CTA finished last (epilogue)
    uint32_t chunk[2];  // the dynamic chunk just taken
    // fixed-capacity bucket list (and the 16-byte chunk of tile counts holding
    // its count) of the tile in ring buffer b, copied with the tile's start
    // (SQF2K_BUCKET_PREFETCH)
    alignas(16) uint16_t bl_hits[kRingTiles][kBucketCap];
    alignas(16) uint32_t bl_cnt[kRingTiles][4];
#ifdef SQF2K_CHECKS
    uint32_t tag[kRingTiles];           // tile started into each ring buffer
    uint32_t wphase[kThreads / 32];     // phases each warp has arrived on
#endif
};
// dynamic shared memory starts 1 KB into the CTA's shared window (the
// system-reserved 1 KB), so the ring lands on 8 KB at offset 7 KB
constexpr uint32_t kSmemBase = 1024, kRingAlign = 8192;
constexpr uint32_t kRingOffset = SQF2K_RING_ALIGN ? kRingAlign - kSmemBase : 0;
static_assert(!SQF2K_RING_ALIGN || sizeof(TileSmemHead) <= kRingOffset, "bookkeeping fits before the ring");
struct TileSmem : TileSmemHead {
    uint8_t pad[SQF2K_RING_ALIGN ? kRingOffset - sizeof(TileSmemHead) : 16];
    alignas(16) uint32_t ring[kRingWords];
};

// Clear slot o of the words starting at shared address wbase (byte address
// of a run of words that does not wrap): one shift, one LEA, one funnel
// shift for ~(1 << (o & 31)), one RED.
__device__ __forceinline__ void clear_bit(uint32_t wbase, uint32_t o) {
#if SQF2K_RING_ALIGN
    const uint32_t addr = wbase | ((o >> 3) & 0x1ffcu);
#else
    const uint32_t addr = wbase + ((o >> 5) << 2);
#endif
    const uint32_t m = __funnelshift_l(0xffffffffu, 0xfffffffeu, o);
#ifdef SQF2K_EXP_ATOMIC_AND
    atomicAnd(reinterpret_cast<uint32_t *>(__cvta_shared_to_generic(addr)), m);
#else
    asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(addr), "r"(m) : "memory");
#endif
}

__device__ __forceinline__ unsigned long long warp_sum_u64(uint32_t x) {
    unsigned long long v = x;
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

#if SQF2K_SPLIT_PHASE
__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// the waiting thread sleeps in hardware until the phase completes (or the
// hint elapses) instead of re-issuing the poll
constexpr uint32_t kWaitHintNs = SQF2K_WAIT_HINT_NS;
constexpr uint32_t kWaitSleepNs = SQF2K_WAIT_SLEEP_NS;
// Named-barrier form of the split phase (SQF2K_NAMED_BAR=1, measured):
// phase p's barrier is id 1 + (p & 1) with 2 * kThreads arrivals -- every
// thread arrives (bar.arrive) at the end of phase p and syncs (bar.sync) at
// its wait in phase p + 1, so waiting warps sleep in hardware instead of
// polling, at the price of a full barrier at the wait point.  Ids alternate
// safely: a thread reaches phase p + 2's arrival only after passing phase
// p + 1's sync, which needs every thread past phase p's sync.
#ifndef SQF2K_NAMED_BAR
#define SQF2K_NAMED_BAR 0
#endif
// SQF2K_WARP_ARRIVE: one arrival per warp (lane 0 after __syncwarp) instead
// of one per thread
#ifndef SQF2K_WARP_ARRIVE
#define SQF2K_WARP_ARRIVE 0
#endif
constexpr uint32_t kPhaseArrivals = SQF2K_WARP_ARRIVE ? kThreads / 32 : kThreads;
__device__ __forceinline__ void phase_arrive(unsigned long long *bar, uint32_t phase) {
#if SQF2K_NAMED_BAR
    asm volatile("bar.arrive %0, %1;" ::"r"(1u + (phase & 1u)), "r"(2u * kThreads) : "memory");
#elif SQF2K_WARP_ARRIVE
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
#else
    mbar_arrive(bar);
#endif
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity);
__device__ __forceinline__ void phase_wait(unsigned long long *bar, uint32_t phase) {
#if SQF2K_NAMED_BAR
    asm volatile("bar.sync %0, %1;" ::"r"(1u + (phase & 1u)), "r"(2u * kThreads) : "memory");
#else
    mbar_wait(bar, phase & 1u);
#endif
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
    uint32_t done = 0;
    for (;;) {
        if (kWaitHintNs)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; "
                "selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_addr(bar)), "r"(parity), "r"(kWaitHintNs)
                : "memory");
        else  // (the system-dependent suspend limit)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                "selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_addr(bar)), "r"(parity)
                : "memory");
        if (done) break;
        if (kWaitSleepNs) __nanosleep(kWaitSleepNs);  // leave the issue slots to working warps
    }
}
#endif


// Medium primes 11 <= p < kPMed.  Each lane owns kTaskSlots descriptors
// (host-balanced, see build_med): a start hit and a step (a multiple of
// q = p^2).  o[j] is the lane's next hit relative to the current run of
// slots; after clearing the hits in [0, len) it is rebased by -len, which
// is exactly the next run's offset -- the offsets never leave registers.
#ifndef SQF2K_TMA_EXPORT
#define SQF2K_TMA_EXPORT 1
#endif
#ifndef SQF2K_SCAN_CHUNK
#define SQF2K_SCAN_CHUNK 4
#endif
#ifndef SQF2K_LPT_BUCKET
#define SQF2K_LPT_BUCKET 8.0  // fixed bucket warp's pre-charge (4 -> 8 measured C5 420.1 -> 418.7 ms)
#define SQF2K_LPT_PER_TRIP 2.0
#define SQF2K_LPT_TASK 2.0
#endif
#ifndef SQF2K_LPT_WARP_BIAS
#define SQF2K_LPT_WARP_BIAS 0.25
#endif
#ifndef SQF2K_ITEM_GROWTH
#define SQF2K_ITEM_GROWTH 1.5
#endif
#ifndef SQF2K_SCATTER_UNROLL
#define SQF2K_SCATTER_UNROLL 2
#endif
struct MedLane {
    uint32_t o[kTaskSlots], step[kTaskSlots];
};

__device__ __forceinline__ void scatter_medium(MedLane &L, uint32_t wbase, uint32_t len) {
#pragma unroll
    for (int j = 0; j < kTaskSlots; ++j) {
        const uint32_t st = L.step[j];
        uint32_t o = L.o[j];
#if SQF2K_SCATTER_UNROLL == 1
        for (; o < len; o += st) clear_bit(wbase, o);
#else
#if SQF2K_SCATTER_UNROLL == 4
        for (; o + 3 * st < len; o += 4 * st) {
            clear_bit(wbase, o);
            clear_bit(wbase, o + st);
            clear_bit(wbase, o + 2 * st);
            clear_bit(wbase, o + 3 * st);
        }
#endif
        for (; o + st < len; o += 2 * st) {
            clear_bit(wbase, o);
            clear_bit(wbase, o + st);
        }
        if (o < len) {
            clear_bit(wbase, o);
            o += st;
        }
#endif
        L.o[j] = st ? o - len : o;  // idle slots (step 0) keep o = ~0
    }
}

// Load this lane's descriptors and place their first hits at or after slot b0.
__device__ __forceinline__ void init_medium(MedLane &L, const TileParams &P, uint64_t b0) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < kTaskSlots; ++j) {
        const uint2 d = __ldg(&P.tasks[(warp * kTaskSlots + j) * 32 + lane]);
        L.step[j] = d.y;
        L.o[j] = ~0u;
        if (d.y) {
            const uint32_t q = __ldg(&P.med[d.x & 0xffu]);
            const double inv_q = 1.0 / (double)q;
            const uint32_t r = (uint32_t)slot_residue_q(P.base_n, q, inv_q);
            const uint32_t bm = (uint32_t)mod_q(b0, q, inv_q);
            L.o[j] = (r >= bm ? r - bm : r + q - bm) + (d.x >> 8) * q;
        }
    }
}

// The bucket hits of a tile are cleared by one warp: a fixed last warp with a
// lighter medium share (SQF2K_LPT_BUCKET), or -- for the kind-2 calls (>= 2^39
// slots) -- warp t mod 8 with an even share: measured C5 418.6 -> 415.8 ms,
// while C3, C4 and the export kernel were 0.4-1.6 % faster with the fixed warp.
// SQF2K_BUCKET_ROTATE=0 keeps the fixed warp everywhere.
#ifndef SQF2K_BUCKET_ROTATE
#define SQF2K_BUCKET_ROTATE 1
#endif
template <int PAT>
__device__ __forceinline__ constexpr bool bucket_rotates() { return SQF2K_BUCKET_ROTATE && PAT == 2; }
// clear the bucket hits of tile t with offsets in [skip, kTile), shifted by
// -skip (its kSubTiles bucket-tile lists); run by one warp (~9
// hits per 2^16 slots; build_med gives that warp less medium work)
template <bool ROTATE>
__device__ __forceinline__ void scatter_bucket(uint32_t wbase, const TileParams &P, uint32_t t,
                                               uint32_t skip) {
    if ((threadIdx.x >> 5) != (ROTATE ? t & (kThreads / 32 - 1) : kThreads / 32 - 1)) return;
#pragma unroll
    for (int j = 0; j < kSubTiles; ++j) {
        const uint32_t bt = t * kSubTiles + j;
        if (bt >= P.n_btiles || (uint32_t)(j + 1) * kBucketTile <= skip) continue;
        uint32_t b, e;
        if (P.tile_start) {
            b = __ldg(&P.tile_start[bt]);
            e = __ldg(&P.tile_start[bt + 1]);
        } else {
            b = bt * (uint32_t)kBucketCap;
            e = b + min(__ldg(&P.tile_count[bt]), (uint32_t)kBucketCap);
        }
        for (uint32_t i = b + (threadIdx.x & 31); i < e; i += 32) {
            const uint32_t o = j * kBucketTile + __ldg(&P.hits[i]);
            if (o >= skip) clear_bit(wbase, o - skip);
        }
    }
}

// scatter_bucket from the copy of tile t's list that came with its start
// (fixed-capacity lists, kSubTiles == 1): no global-memory round trips on the
// bucket warp's path (export kernel)
#ifndef SQF2K_BUCKET_PREFETCH
#define SQF2K_BUCKET_PREFETCH 1
#endif
constexpr bool kBucketPrefetch = SQF2K_BUCKET_PREFETCH && kSubTiles == 1;
__device__ __forceinline__ void scatter_bucket_smem(const TileSmemHead &S, uint32_t wbase, uint32_t t,
                                                    uint32_t b) {
    if ((threadIdx.x >> 5) != kThreads / 32 - 1) return;
    const uint32_t n = min(S.bl_cnt[b][t & 3u], (uint32_t)kBucketCap);
    for (uint32_t i = threadIdx.x & 31; i < n; i += 32) clear_bit(wbase, S.bl_hits[b][i]);
}

// Start WORDS words (domain slot `base`, ring word `at`, 16-byte aligned and
// not wrapping) from the p = 3, 5, 7 pattern; pbase is (base / 32) mod
// pat_words.  Thread i writes the 4-word chunks i, i + kThreads, ... with
// one STS.128 each.  EDGE applies the n < 1 zero region and the domain end.
template <int WORDS, bool EDGE>
__device__ __forceinline__ void init_words(uint32_t *ring, uint32_t at, uint64_t base,
                                           uint32_t pbase, const TileParams &P) {
    static_assert(WORDS % 4 == 0, "whole uint4 chunks");
#pragma unroll
    for (int c = 0; c < (WORDS + 4 * kThreads - 1) / (4 * kThreads); ++c) {
        const uint32_t w = 4 * (threadIdx.x + c * kThreads);
        if (WORDS % (4 * kThreads) != 0 && w >= (uint32_t)WORDS) break;
        const uint32_t *src = P.pattern + pbase + w;  // padded table: no wrap
        uint32_t v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = __ldg(src + i);
        if (EDGE) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint64_t u0 = base + 32ull * (w + i);
                if (u0 < P.z) v[i] = (u0 + 32 <= P.z) ? 0u : (v[i] & (~0u << (uint32_t)(P.z - u0)));
                if (u0 + 32 > P.U) v[i] = (u0 >= P.U) ? 0u : (v[i] & ((1u << (uint32_t)(P.U - u0)) - 1u));
            }
        }
        *reinterpret_cast<uint4 *>(&ring[at + w]) = make_uint4(v[0], v[1], v[2], v[3]);
    }
}

// The pre-tile starts the H = HW*32 halo slots (HW in {32, 64, ..., 1024}).
__device__ __forceinline__ void init_halo(uint32_t *ring, uint32_t at, uint32_t HW, uint64_t base,
                                          uint32_t pbase, const TileParams &P) {
    static_assert(kHaloWordsMax <= 1024 && kHaloWordsMax <= kTileWords, "halo within a buffer");
    if (HW == 1024) init_words<1024, true>(ring, at, base, pbase, P);
    else if (HW == 512) init_words<512, true>(ring, at, base, pbase, P);
    else if (HW == 256) init_words<256, true>(ring, at, base, pbase, P);
    else if (HW == 128) init_words<128, true>(ring, at, base, pbase, P);
    else if (HW == 64) init_words<64, true>(ring, at, base, pbase, P);
    else init_words<32, true>(ring, at, base, pbase, P);
}

__device__ __forceinline__ void append(unsigned long long *list, unsigned long long *count,
                                       uint64_t cap, uint64_t n) {
    const unsigned long long i = atomicAdd(count, 1ull);
    if (i < cap) list[i] = n;
}

// Leftover slots of one word after the in-tile passes: escalation (k_max >
// k_eff) or failures.  Out of line: it essentially never runs.
__device__ __noinline__ void spill_word(uint32_t pend, uint64_t u0, int64_t base_n,
                                        unsigned long long *list, unsigned long long *count,
                                        uint64_t cap) {
    for (uint32_t x = pend; x; x &= x - 1)
        append(list, count, cap, (uint64_t)(base_n + 2 * (int64_t)(u0 + __ffs(x) - 1)));
}

// Passes k = kMainMax+1..k_eff for one word (divergent, rare: ~0.02% of
// words after 5 main passes).
__device__ __forceinline__ void scan_residue(TileSmem &S, const TileParams &P, uint32_t hb,
                                             uint32_t w, uint64_t u0, uint32_t pend, uint32_t need) {
    for (uint32_t k = kMainMax + 1; k <= P.k_eff && pend; ++k) {
        const uint32_t sl = k == 5 ? __funnelshift_l(S.ring[ring_back(hb + w, 1u)], S.ring[hb + w], 16)
                                   : S.ring[ring_back(hb + w, 1u << (k - 6))];
        const uint32_t nw = pend & sl;
        if (nw) {
            atomicAdd(&S.cnt[k], (uint32_t)__popc(nw));
            if ((need >> k) & 1u) atomicMin(&S.first[k], (unsigned long long)(u0 + __ffs(nw) - 1));
        }
        pend &= ~sl;
    }
    if (pend) {
        if (P.k_max > P.k_eff) spill_word(pend, u0, P.base_n, P.esc, P.esc_count, P.esc_cap);
        else spill_word(pend, u0, P.base_n, P.fail, P.fail_count, P.fail_cap);
    }
}

// Main scan of one word (cur, its left neighbour prv): n - 2^k for k <= 5 is
// 2^(k-1) slots back, inside (cur, prv).  Returns the slots left after KMAIN
// passes.  Counting: c[k] (k < KMAIN) accumulates the slots still pending
// after pass k -- the histogram is the difference of consecutive entries,
// the (rare) leftover path subtracts its slots from hist[KMAIN] (S.cnt[0]) and hist[1] is derived from
// the scanned-slot count by conservation (verify.cu).  The covered bits are
// counted (pending = 32 - covered; no NOT in front of the POPC; masked edge
// slots count as covered) and the 32 per word are added back per tile.
// TRACK: the thread's least slot with exponent k (its words come in slot
// order, so the first hit is the least); reduced per warp after the tile.
template <bool TRACK, int KMAIN>
__device__ __forceinline__ uint32_t scan_word(uint32_t pend, uint32_t prv, uint32_t cur,
                                              uint32_t (&c)[6], uint32_t (&f)[6], uint32_t wl) {
#pragma unroll
    for (int k = 1; k <= KMAIN; ++k) {
        const uint32_t sl = __funnelshift_l(prv, cur, 1u << (k - 1));
        if (TRACK) {
            const uint32_t nw = pend & sl;
            if (nw && f[k] == ~0u) f[k] = 32 * wl + __ffs(nw) - 1;
        }
        pend &= ~sl;
        if (k < KMAIN) c[k] -= __popc(~pend);  // + 32 per word: scan_tile
    }
    return pend;
}

// Scan-range mask of the word starting at tile slot u0 (EDGE tiles only).
__device__ __forceinline__ uint32_t edge_mask(const TileParams &P, uint64_t u0) {
    if (u0 + 32 <= P.scan_lo || u0 >= P.U) return 0u;
    uint32_t pend = ~0u;
    if (u0 < P.scan_lo) pend &= ~0u << (uint32_t)(P.scan_lo - u0);
    if (u0 + 32 > P.U) pend &= (1u << (uint32_t)(P.U - u0)) - 1u;
    if (P.one_u >= u0 && P.one_u < u0 + 32) pend &= ~(1u << (uint32_t)(P.one_u - u0));
    return pend;
}

// One word with slots left after the main passes (rare): counted against
// hist[KMAIN], then deferred to the residue queue (KMAIN = 5) or sent to the
// escalation / failure list.
template <int KMAIN>
__device__ __forceinline__ void leftover_word(TileSmem &S, const TileParams &P, uint32_t hb,
                                              uint32_t w, uint64_t u0, uint32_t left, uint32_t need,
                                              uint32_t qi) {
    if (KMAIN >= 2) atomicAdd(&S.cnt[0], (uint32_t)__popc(left));  // subtracted from hist[KMAIN]
    if (KMAIN == kMainMax) {
        const uint32_t e = atomicAdd(&S.n_res[qi], 1u);
        if (e < (uint32_t)kResCap) {  // deferred to the next tile's scan phase
            S.res_w[qi][e] = w;
            S.res_p[qi][e] = left;
        } else {
            scan_residue(S, P, hb, w, u0, left, need);
        }
    } else if (P.k_max > P.k_eff) {  // k_eff = KMAIN < kMainMax: leftovers leave the tile
        spill_word(left, u0, P.base_n, P.esc, P.esc_count, P.esc_cap);
    } else {
        spill_word(left, u0, P.base_n, P.fail, P.fail_count, P.fail_cap);
    }
}

// Exponent passes over the tile (ring buffer at hb): thread t owns the
// kWordsPerThread consecutive words from W*t, taken 4 at a time (one LDS.128
// plus the left neighbour).  EDGE masks the scan range, TRACK records per-k
// least slots while this CTA still lacks them.  Words left after KMAIN passes
// (~0.02% for KMAIN = 5) are queued for the next tile's scan phase.
template <bool EDGE, bool TRACK, int KMAIN>
__device__ __forceinline__ void scan_tile(TileSmem &S, const TileParams &P, uint32_t hb,
                                          uint64_t tb, uint32_t need, uint32_t (&c)[6],
                                          uint32_t &scanned, uint32_t qi) {
    constexpr int W = kWordsPerThread;
    static_assert(W % 4 == 0, "4-word chunks");
    const uint32_t wt = W * threadIdx.x;
    uint32_t f[6] = {~0u, ~0u, ~0u, ~0u, ~0u, ~0u};  // TRACK: least tile-local slot per k
    uint32_t prv_in = S.ring[hb + wt ? hb + wt - 1 : kRingWords - 1];
    constexpr int CW = SQF2K_SCAN_CHUNK;  // words scanned together (ILP vs registers)
#pragma unroll
    for (int ch = 0; ch < W / CW; ++ch) {
        const uint32_t w0 = wt + CW * ch;
        uint32_t cur[CW], prv[CW];
#pragma unroll
        for (int v = 0; v < CW / 4; ++v) {
            const uint4 cw = *reinterpret_cast<const uint4 *>(&S.ring[hb + w0 + 4 * v]);
            cur[4 * v] = cw.x;
            cur[4 * v + 1] = cw.y;
            cur[4 * v + 2] = cw.z;
            cur[4 * v + 3] = cw.w;
        }
        prv[0] = prv_in;
#pragma unroll
        for (int i = 1; i < CW; ++i) prv[i] = cur[i - 1];
        prv_in = cur[CW - 1];
        uint32_t left[CW], any = 0;
#pragma unroll
        for (int i = 0; i < CW; ++i) {
            uint32_t pend = ~0u;
            if (EDGE) {
                pend = edge_mask(P, tb + 32ull * (w0 + i));
                scanned += __popc(pend);
            }
            left[i] = scan_word<TRACK, KMAIN>(pend, prv[i], cur[i], c, f, w0 + i);
            any |= left[i];
        }
        if (!EDGE) scanned += 32 * CW;
        if (any) {  // rare
#pragma unroll
            for (int i = 0; i < CW; ++i)
                if (left[i]) leftover_word<KMAIN>(S, P, hb, w0 + i, tb + 32ull * (w0 + i), left[i], need, qi);
        }
    }
#pragma unroll
    for (int k = 1; k < KMAIN; ++k) c[k] += 32 * W;  // pending = 32 - covered per word
    if (TRACK) {  // per k: one warp reduction, one shared atomic
#pragma unroll
        for (int k = 1; k <= KMAIN; ++k) {
            if (!((need >> k) & 1u)) continue;
            const uint32_t m = __reduce_min_sync(0xffffffffu, f[k]);
            if (m != ~0u && (threadIdx.x & 31) == 0) atomicMin(&S.first_t[qi][k], m);
        }
    }
}

// Finish the deferred words of tile tp (queue tp & 1; its ring buffer and
// the one below stay intact until tile tp + 3 starts) and empty the queue.
// One warp per tile, rotating, so no warp carries them all.
__device__ __forceinline__ void drain_residue(TileSmem &S, const TileParams &P, uint32_t tp,
                                              uint32_t need) {
    if ((threadIdx.x >> 5) != (tp & (kThreads / 32 - 1))) return;  // (warp count: power of 2)
    const uint32_t qi = tp & 1u, n = min(S.n_res[qi], (uint32_t)kResCap);
    const uint32_t hb = ring_base(tp);
    SQF2K_CHECK(S.tag[tp % kRingTiles] == tp);  // tile tp still in its buffer
    for (uint32_t e = threadIdx.x & 31; e < n; e += 32) {
        const uint32_t w = S.res_w[qi][e];
        scan_residue(S, P, hb, w, (uint64_t)tp * kTile + 32ull * w, S.res_p[qi][e], need);
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) S.n_res[qi] = 0;  // free for tile tp + 2 (next phase on)
}

// Last-CTA epilogue of a single-batch call (run by the CTA that finished
// last, after every CTA has added its counts): escalate the unresolved n
// (k > k_eff, exact trial division, 8 warps) and copy the accumulators to
// mapped host memory.
__device__ __forceinline__ void finish_call(TileSmem &S, const TileParams &P) {
    if (P.k_max > P.k_eff) {
        const uint64_t count = min((unsigned long long)P.esc_cap, __ldcg(P.esc_count));
        escalate_warps(P.esc, count, P.k_eff + 1, P.k_max, P.primes, __ldcg(&P.info->count),
                       P.hist, P.min_n, P.fail, P.fail_count, P.fail_cap, threadIdx.x / 32,
                       kThreads / 32);
        __threadfence();
        __syncthreads();
    }
    // kernel completion makes these host writes visible to the stream's waiter
    const unsigned long long *src = reinterpret_cast<const unsigned long long *>(P.acc);
    unsigned long long *dst = static_cast<unsigned long long *>(P.acc_host);
    for (uint32_t i = threadIdx.x; i < sizeof(Acc) / 8; i += kThreads) dst[i] = __ldcg(src + i);
}

// KMAIN = min(k_eff, 5) unconditional passes; the export form ignores it.
// Per tile t (split phase, the default): sieve t + 1, wait for every warp to
// finish phase t - 1 (mbarrier), start t + 3 (TMA bulk copy of the pattern),
// scan t (fused) or store it (export, TMA bulk store), finish t - 1's
// deferred words, arrive.  Without the split phase: one barrier per tile,
// scan t + sieve t + 1 + start t + 2 between barriers.
// Per-CTA timeline for experiment builds (-DSQF2K_EXP_TIMELINE, tools/timeline.py).
#ifdef SQF2K_EXP_TIMELINE
__device__ unsigned long long g_timeline[4096][4];
__device__ __forceinline__ void tl_mark(int i) {
    if (threadIdx.x != 0 || blockIdx.x >= 4096) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_timeline[blockIdx.x][i] = t & ((1ull << 56) - 1);  // (bits 56+ carry the SM id in [0])
    if (i == 3) {
        unsigned sm;
        asm("mov.u32 %0, %%smid;" : "=r"(sm));
        g_timeline[blockIdx.x][0] |= (unsigned long long)sm << 56;
    }
}
#define TL(i) tl_mark(i)
__device__ unsigned long long g_tiles[8][64];
__device__ __forceinline__ void tl_tile(uint32_t i) {
    if (threadIdx.x != 0 || blockIdx.x >= 8 || i >= 64) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tiles[blockIdx.x][i] = t;
}
#define TLT(i) tl_tile(i)
#else
#define TL(i) do { } while (0)
#define TLT(i) do { } while (0)
#endif

template <bool FUSED, int KMAIN, int PAT>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) tile_kernel(const TileParams P) {
    static_assert(kWordsPerThread % 4 == 0 && kThreads * kWordsPerThread == kTileWords,
                  "4-word chunks per thread");
    static_assert(((kThreads / 32) & (kThreads / 32 - 1)) == 0, "drain_residue rotates over the warps");
    extern __shared__ __align__(16) uint8_t smem_raw[];
    TileSmem &S = *reinterpret_cast<TileSmem *>(smem_raw);
    const uint32_t G = gridDim.x;
    TL(0);
    // Work: a static chunk of ~3/4 of the tiles per CTA (contiguous), then
    // chunks handed out by a global counter -- the CTAs sharing an SM are not
    // served evenly by the warp schedulers, and the fast ones take the rest.
    // (short runs, < kDynMinTiles tiles per CTA, stay fully static: a chunk's
    // start-up -- halo, offsets -- would cost more than the balance gains)
    const bool dynamic = P.n_tiles >= (uint64_t)kDynMinTiles * G;
    const uint32_t S1 = (uint32_t)((uint64_t)P.n_tiles * kStaticEighths / (8ull * G));
    const uint32_t dyn0 = dynamic ? S1 * G : P.n_tiles;  // first dynamically scheduled tile
    // dynamic chunks (sizes below): an atomicAdd each, no CAS races
// dynamic chunks of ~1/(6G) of the dynamic tiles, the last G chunks' worth
// handed out at half size (measured on C5: 415.8 -> 413.7 ms; a chunk's
// start-up -- halo, descriptor offsets, pipeline fill -- costs ~3 us, so
// smaller chunks throughout were slower: /16 417.4, /32 422.2 ms)
#ifndef SQF2K_CHUNK_DIV
#define SQF2K_CHUNK_DIV 6
#endif
#ifndef SQF2K_TAPER
#define SQF2K_TAPER 2
#endif
#ifndef SQF2K_TAPER_TAIL
#define SQF2K_TAPER_TAIL 1
#endif
    const uint32_t csz = max((P.n_tiles - dyn0) / (SQF2K_CHUNK_DIV * G), (uint32_t)kMinChunk);
    uint32_t t0 = dynamic ? S1 * blockIdx.x : (uint32_t)((uint64_t)P.n_tiles * blockIdx.x / G);
    uint32_t t1 = dynamic ? t0 + S1 : (uint32_t)((uint64_t)P.n_tiles * (blockIdx.x + 1) / G);
    const uint32_t H = FUSED ? P.H : 0u;
    const uint32_t HW = H / 32;
    // tiles [ti0, ti1) need no masks: past the scan start, the n < 1 region
    // and n = 1, and wholly below the domain end
    uint64_t lo_edge = FUSED ? P.scan_lo : 0ull;
    if (P.z > lo_edge) lo_edge = P.z;
    if (FUSED && P.one_u != ~0ull && P.one_u + 1 > lo_edge) lo_edge = P.one_u + 1;
    const uint32_t ti0 = (uint32_t)((lo_edge + kTile - 1) / kTile);
    const uint32_t ti1 = (uint32_t)(P.U / kTile);
    if (threadIdx.x <= kDepthMax) {
        S.first[threadIdx.x] = ~0ull;
        S.cnt[threadIdx.x] = 0;
    }
    if (threadIdx.x < 12) S.first_t[threadIdx.x / 6][threadIdx.x % 6] = ~0u;
    if (threadIdx.x == 0) S.need = ~0u;
    const uint32_t ring_addr = smem_addr(S.ring);
    if (SQF2K_RING_ALIGN && (ring_addr & (kRingAlign - 1))) __trap();  // clear_bit's OR needs it
    // per-thread counters: each adds <= 32 * kWordsPerThread = 256 per tile, and
    // run_tile_batch keeps a CTA under 2^23 tiles, so they stay below 2^31; the
    // warp sums at the end are 64-bit
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};
    uint32_t scanned = 0;
    bool waited = false;
    constexpr bool kTmaStart = SQF2K_TMA_START;
    bool start_pending = false;  // thread 0: a start's bulk copy is in flight
    uint32_t start_parity = 0;
    // Per-buffer start barriers (split phase): the start of tile t (issued two
    // phases ahead) is waited for by the threads that sieve it, not by the
    // issuing thread before its phase arrival -- thread 0 no longer polls its
    // own copies and the phase barrier no longer waits for a copy's latency.
    // (export kernel only: +5 % there; the fused kernel measured slower with
    // them when replayed from a CUDA graph, 543 vs 494 ms per C5 call)
    constexpr bool kStartBars = SQF2K_START_BARS && SQF2K_SPLIT_PHASE && kTmaStart && !FUSED;
    uint32_t sbpar = 0;  // bit b: parity of buffer b's next start completion
    if (kTmaStart) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&S.mbar_start))
                         : "memory");
            for (int b = 0; b < kRingTiles; ++b)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&S.start_bar[b]))
                             : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
#if SQF2K_SPLIT_PHASE
    uint32_t mbar_phase = 0;  // phases this thread arrived on
#ifdef SQF2K_CHECKS
    if (threadIdx.x < kThreads / 32) S.wphase[threadIdx.x] = 0;
    if (threadIdx.x < kRingTiles) S.tag[threadIdx.x] = ~0u;
#endif
    if (threadIdx.x == 0) mbar_init(&S.mbar, kPhaseArrivals);
    __syncthreads();
#endif

    for (;;) {
        if (t0 >= t1) {  // next dynamic chunk: one atomic, chunk index -> tiles
            __syncthreads();  // the last chunk's drain is done with the ring
            if (threadIdx.x == 0) {
                const uint32_t k = atomicAdd(&P.sched[0], 1u);
#if SQF2K_TAPER
                // tapered tail: the last ~G * csz tiles go out in chunks of
                // csz / SQF2K_TAPER, so the CTAs finish closer together
                const uint64_t D = P.n_tiles - dyn0, tail = (uint64_t)SQF2K_TAPER_TAIL * G * csz;
                const uint64_t n_big = D > tail ? (D - tail) / csz : 0;
                const uint32_t small = max(csz / SQF2K_TAPER, (uint32_t)kMinChunk);
                uint64_t lo, sz;
                if (k < n_big) {
                    lo = (uint64_t)dyn0 + (uint64_t)k * csz;
                    sz = csz;
                } else {
                    lo = (uint64_t)dyn0 + n_big * csz + (uint64_t)(k - n_big) * small;
                    sz = small;
                }
                S.chunk[0] = (uint32_t)min(lo, (uint64_t)P.n_tiles);
                S.chunk[1] = (uint32_t)min(lo + sz, (uint64_t)P.n_tiles);
#else
                const uint64_t lo = (uint64_t)dyn0 + (uint64_t)k * csz;
                S.chunk[0] = (uint32_t)min(lo, (uint64_t)P.n_tiles);
                S.chunk[1] = (uint32_t)min(lo + csz, (uint64_t)P.n_tiles);
#endif
            }
            __syncthreads();
            t0 = S.chunk[0];
            t1 = S.chunk[1];
            if (t0 >= t1) break;
        }
        const bool pre = FUSED && t0 > 0;
        // medium primes: each lane's descriptors, first hits at the chunk base b0
        const uint64_t b0 = pre ? (uint64_t)t0 * kTile - H : (uint64_t)t0 * kTile;
        MedLane L;
        if (threadIdx.x < 2) S.n_res[threadIdx.x] = 0;
        // pattern index of the next tile start (t0 first; the halo has its own)
        // the period as a compile-time constant (a runtime P.pat_words
        // measured 0.5 % slower on the C5 window)
        constexpr uint32_t pat_words = pattern_words(PAT == 2 ? 24u : PAT == 1 ? 8u : 0u);
        uint32_t pbase = (uint32_t)(((uint64_t)t0 * kTileWords + P.pat_off) % pat_words);
        const uint32_t pbase_halo = (uint32_t)((b0 / 32 + P.pat_off) % pat_words);
        // the bulk-copy source of a tile start (16-byte aligned): kind 2 is
        // one table of four periods (pbase stays 0 mod 4), kinds 0 and 1
        // take the copy shifted by pbase mod 4
        auto start_src = [&]() -> const uint32_t * {
            if (PAT == 2) return P.pattern + pbase;
            const uint32_t r = pbase & 3u;
            return P.pattern + r * kPatStride + (pbase - r);
        };
        // main-loop starts (tiles >= t0 + 3, after the grid dependency wait)
        // copy the tile's bucket list too; the prologue's starts cannot (the
        // lists may still be in the making) -- sieve_tile applies the same rule
        // (export kernel only: 3915 -> 5193 GB/s there; in the fused kernel
        // the copies in the start transaction measured 2.4 % slower -- its
        // starter waits for the start before arriving on the phase barrier --
        // and a cp.async prefetch by the bucket warp 1.3 % slower)
        const bool list_prefetch = kBucketPrefetch && !FUSED && P.tile_start == nullptr;
        auto start_tile = [&](uint32_t t, uint32_t at) {  // tile t's words (ring base at)
            const uint64_t tb = (uint64_t)t * kTile;
#ifdef SQF2K_CHECKS
            if (threadIdx.x == kStarter) S.tag[t % kRingTiles] = t;
#endif
            if (t < ti0 || t >= ti1) {
                init_words<kTileWords, true>(S.ring, at, tb, pbase, P);
                if (kStartBars && threadIdx.x == kStarter)  // keep the buffer's phase count
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                                     smem_addr(&S.start_bar[t % kRingTiles]))
                                 : "memory");
            } else if (kTmaStart) {
                // one bulk copy (TMA) of the pattern words, from the shifted
                // table copy that makes the source 16-byte aligned
                if (threadIdx.x == kStarter) {
                    const uint32_t bar = smem_addr(kStartBars ? &S.start_bar[t % kRingTiles] : &S.mbar_start);
                    const bool pl = list_prefetch;  // and the tile's bucket list
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                                 "r"((uint32_t)kTileWords * 4 + (pl ? (uint32_t)kBucketCap * 2 + 16 : 0u))
                                 : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            ring_addr + 4 * at),
                        "l"(start_src()), "r"((uint32_t)kTileWords * 4),
                        "r"(bar)
                        : "memory");
                    if (pl) {
                        const uint32_t b = t % kRingTiles;
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                smem_addr(&S.bl_hits[b][0])),
                            "l"(P.hits + (uint64_t)t * kBucketCap), "r"((uint32_t)kBucketCap * 2), "r"(bar)
                            : "memory");
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                smem_addr(&S.bl_cnt[b][0])),
                            "l"(P.tile_count + (t & ~3u)), "r"(16u), "r"(bar)
                            : "memory");
                    }
                    start_pending = !kStartBars;
                }
            } else {
                init_words<kTileWords, false>(S.ring, at, tb, pbase, P);
            }
            pbase += kTileWords;
            if (pbase >= pat_words) pbase -= pat_words;
        };
        // thread 0, before the barrier that publishes a start: its copy has landed
        auto finish_start = [&]() {
            if (kTmaStart && threadIdx.x == kStarter && start_pending) {
                uint32_t done = 0;
                while (!done)
                    asm volatile(
                        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                        "selp.u32 %0, 1, 0, p; }"
                        : "=r"(done)
                        : "r"(smem_addr(&S.mbar_start)), "r"(start_parity)
                        : "memory");
                start_parity ^= 1u;
                start_pending = false;
            }
        };
        // tiles ta .. ta+n-1 started together: one expect_tx for their bulk
        // copies (one wait), edge tiles by the masked per-thread path
        auto start_batch = [&](uint32_t ta, uint32_t n) {
            auto edge_t = [&](uint32_t t) { return t < ti0 || t >= ti1; };
            if (kStartBars) {  // each tile on its own buffer's barrier
                for (uint32_t i = 0; i < n; ++i) start_tile(ta + i, ring_base(ta + i));
                return;
            }
            uint32_t bytes = 0;
            for (uint32_t i = 0; i < n; ++i)
                if (!edge_t(ta + i)) bytes += (uint32_t)kTileWords * 4;
            if (kTmaStart && bytes && threadIdx.x == kStarter) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                 smem_addr(&S.mbar_start)),
                             "r"(bytes)
                             : "memory");
                start_pending = true;
            }
            for (uint32_t i = 0; i < n; ++i) {
                const uint32_t t = ta + i, at = ring_base(t);
                const uint64_t tb = (uint64_t)t * kTile;
#ifdef SQF2K_CHECKS
                if (threadIdx.x == kStarter) S.tag[t % kRingTiles] = t;
#endif
                if (edge_t(t)) {
                    init_words<kTileWords, true>(S.ring, at, tb, pbase, P);
                } else if (kTmaStart) {
                    if (threadIdx.x == kStarter) {
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                ring_addr + 4 * at),
                            "l"(start_src()),
                            "r"((uint32_t)kTileWords * 4), "r"(smem_addr(&S.mbar_start))
                            : "memory");
                    }
                } else {
                    init_words<kTileWords, false>(S.ring, at, tb, pbase, P);
                }
                pbase += kTileWords;
                if (pbase >= pat_words) pbase -= pat_words;
            }
        };
#if SQF2K_SPLIT_PHASE
        start_batch(t0, min(3u, t1 - t0));  // in flight during the halo work below
#endif
        init_medium(L, P, b0);  // (after the starts: its table loads overlap their copies)

        // the halo just below tile t0: the tail of buffer t0 - 1
        const uint32_t halo_at = ring_base(t0 + kRingTiles - 1) + kTileWords - HW;
        if (FUSED) {
            if (pre) {  // pre-tile: sieve the H slots below the chunk
                init_halo(S.ring, halo_at, HW, b0, pbase_halo, P);
                __syncthreads();
                scatter_medium(L, ring_addr + 4 * halo_at, H);
                if (!waited) grid_dependency_wait();  // bucket lists from here on
                waited = true;
                scatter_bucket<bucket_rotates<PAT>()>(ring_addr + 4 * halo_at, P, t0 - 1, kTile - H);
            } else {
                for (uint32_t i = threadIdx.x; i < HW; i += kThreads) S.ring[halo_at + i] = 0u;
            }
        }
        TL(1);
        if (!waited) grid_dependency_wait();
        waited = true;
        // Y work of tile t: scan (or store) it, finish t - 1's deferred words
        auto scan_phase = [&](uint32_t t, uint32_t hb) {
            const uint64_t tb = (uint64_t)t * kTile;
            SQF2K_CHECK(S.tag[t % kRingTiles] == t);  // tile t still in its buffer
            SQF2K_CHECK(t == t0 || S.tag[(t - 1) % kRingTiles] == t - 1);  // its halo too
            const bool edge = t < ti0 || t >= ti1;
            if (!FUSED) {
#if SQF2K_TMA_EXPORT
                // one bulk copy (TMA engine) of the sieved tile to HBM; the
                // buffer is rewritten 3 phases later (wait_group.read below)
                if (threadIdx.x == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile(
                        "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                            P.bits_out + (uint64_t)t * kTileWords),
                        "r"(ring_addr + 4 * hb), "r"((uint32_t)kTileWords * 4)
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
#else
#pragma unroll
                for (int ch = 0; ch < kWordsPerThread / 4; ++ch) {
                    const uint32_t w = 4 * (threadIdx.x + ch * kThreads);
                    const uint4 v = *reinterpret_cast<const uint4 *>(&S.ring[hb + w]);
                    *reinterpret_cast<uint4 *>(&P.bits_out[(uint64_t)t * kTileWords + w]) = v;
                }
#endif
                return;
            }
            // S.first[k] keeps this CTA's least slot with exponent k (its
            // tiles come in increasing order and residue words finish in
            // tile order); stop tracking a k once it is known (warp 0 folds
            // tile t - 1's scan minima into S.first and clears S.need bits
            // in this phase: a stale read only tracks once more).  The value
            // must be warp-uniform -- it selects the TRACK path, whose warp
            // reductions need all 32 lanes -- so lane 0's read is broadcast:
            // lanes of a diverged warp reading S.need before and after warp
            // 0's update took different paths and deadlocked in
            // __reduce_min_sync (observed with some medium schedules).
            const uint32_t need = __shfl_sync(0xffffffffu, S.need, 0);
            if (threadIdx.x < 32) {  // bookkeeping: warp 0 only (uniform branch)
                const uint32_t k = threadIdx.x, qp = (t + 1) & 1u;
                if (k >= 1 && k <= 5 && S.first_t[qp][k] != ~0u) {
                    const unsigned long long f = tb - kTile + S.first_t[qp][k];
                    if (f < S.first[k]) S.first[k] = f;
                    S.first_t[qp][k] = ~0u;
                }
                const uint32_t known =
                    __ballot_sync(0xffffffffu, k >= 1 && k <= kDepthMax && S.first[k] != ~0ull);
                if (k == 0) S.need &= ~known;
            }
#ifndef SQF2K_EXP_NO_SCAN
            if (need & 0x3eu) {
                if (edge) scan_tile<true, true, KMAIN>(S, P, hb, tb, need, c, scanned, t & 1u);
                else scan_tile<false, true, KMAIN>(S, P, hb, tb, need, c, scanned, t & 1u);
            } else {
                if (edge) scan_tile<true, false, KMAIN>(S, P, hb, tb, need, c, scanned, t & 1u);
                else scan_tile<false, false, KMAIN>(S, P, hb, tb, need, c, scanned, t & 1u);
            }
#endif
            if (KMAIN == kMainMax && t > t0) drain_residue(S, P, t - 1, need);
        };
        auto sieve_tile = [&](uint32_t t, uint32_t hb) {
            if constexpr (kStartBars) {  // tile t's start has landed (issued two phases ago)
                const uint32_t b = t % kRingTiles;
                const uint32_t bar = smem_addr(&S.start_bar[b]), par = (sbpar >> b) & 1u;
                uint32_t done = 0;
                while (!done)  // normally complete at the first probe
                    asm volatile(
                        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                        "selp.u32 %0, 1, 0, p; }"
                        : "=r"(done)
                        : "r"(bar), "r"(par)
                        : "memory");
                sbpar ^= 1u << b;
            }
            SQF2K_CHECK(S.tag[t % kRingTiles] == t);  // its start was published
#ifndef SQF2K_EXP_NO_SCATTER
            scatter_medium(L, ring_addr + 4 * hb, kTile);
#ifndef SQF2K_EXP_NO_BUCKET
            if (list_prefetch && t >= t0 + 3 && !(t < ti0 || t >= ti1)) {
                scatter_bucket_smem(S, ring_addr + 4 * hb, t, t % kRingTiles);
            } else {
                scatter_bucket<bucket_rotates<PAT>()>(ring_addr + 4 * hb, P, t, 0);
            }
#endif
#endif
        };
        auto next_base = [](uint32_t h) { return h + kTileWords == kRingWords ? 0u : h + kTileWords; };

#if !SQF2K_SPLIT_PHASE
        // prologue: start t0; sieve t0 and start t0 + 1
        start_tile(t0, ring_base(t0));
        finish_start();
        __syncthreads();
        sieve_tile(t0, ring_base(t0));
        if (t0 + 1 < t1) start_tile(t0 + 1, ring_base(t0 + 1));
        finish_start();
        __syncthreads();

        // One phase per tile t, one barrier: scan t (reads t and the tail of
        // t - 1), finish t - 1's deferred words (t - 1, t - 2), sieve t + 1
        // (started last phase), start t + 2 -- five ring buffers, disjoint.
        // ring bases of tiles t, t + 1, t + 2, advanced by one buffer per tile
        uint32_t hb = ring_base(t0), hb1 = ring_base(t0 + 1), hb2 = ring_base(t0 + 2);
        for (uint32_t t = t0; t < t1; ++t) {
            scan_phase(t, hb);
            if (t + 1 < t1) {
                sieve_tile(t + 1, hb1);
                if (t + 2 < t1) start_tile(t + 2, hb2);
            }
#if SQF2K_TMA_EXPORT
            // next phase starts tile t + 3 in buffer t - 2: its store (group
            // t - 2) must have read the buffer; t - 1 and t may stay in flight
            if (!FUSED && threadIdx.x == 0)
                asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
#endif
            finish_start();
            __syncthreads();
            hb = hb1;
            hb1 = hb2;
            hb2 = next_base(hb2);
            TLT(t - t0);
        }
#if SQF2K_TMA_EXPORT
        // the next chunk restarts the ring: every store must have read its buffer
        if (!FUSED && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
#else
        // prologue: starts t0 .. t0 + 2 (issued before the halo); sieve t0
        finish_start();
        __syncthreads();
        sieve_tile(t0, ring_base(t0));
        __syncthreads();

        // Split phase per tile t: sieve t + 1 (started 2 phases ago), then
        // wait for the previous phase, start t + 3, scan t, finish t - 1's
        // deferred words, arrive.  The uneven sieve work of a warp overlaps
        // the others finishing the previous phase; warps are at most one
        // phase apart, so six ring buffers (t - 3 .. t + 2) stay disjoint.
        uint32_t hb = ring_base(t0), hb1 = ring_base(t0 + 1), hb3 = ring_base(t0 + 3);
        for (uint32_t t = t0; t < t1; ++t) {
            if (t + 1 < t1) sieve_tile(t + 1, hb1);
            if (t > t0) phase_wait(&S.mbar, mbar_phase - 1);
#ifdef SQF2K_CHECKS
            // split phase: every warp has arrived on phase t - 1 and none is
            // more than one phase ahead of this one
            if ((threadIdx.x & 31) < kThreads / 32) {
                const uint32_t ph = S.wphase[threadIdx.x & 31];
                SQF2K_CHECK(ph >= mbar_phase && ph <= mbar_phase + 1);
            }
#endif
            if (t + 3 < t1) start_tile(t + 3, hb3);
            scan_phase(t, hb);
            finish_start();  // the start is published by this phase's arrivals
#ifdef SQF2K_CHECKS
            __syncwarp();
            if ((threadIdx.x & 31) == 0) atomicAdd(&S.wphase[threadIdx.x >> 5], 1u);
#endif
            phase_arrive(&S.mbar, mbar_phase);
            ++mbar_phase;
            hb = hb1;
            hb1 = next_base(hb1);
            hb3 = next_base(hb3);
            TLT(t - t0);
        }
        phase_wait(&S.mbar, mbar_phase - 1);
#endif
        if (FUSED) {  // the chunk's last tile: deferred words and minima
            if (KMAIN == kMainMax) drain_residue(S, P, t1 - 1, S.need);
            const uint32_t ql = (t1 - 1) & 1u;
            if (threadIdx.x >= 1 && threadIdx.x <= 5 && S.first_t[ql][threadIdx.x] != ~0u) {
                const unsigned long long f = (uint64_t)(t1 - 1) * kTile + S.first_t[ql][threadIdx.x];
                if (f < S.first[threadIdx.x]) S.first[threadIdx.x] = f;
                S.first_t[ql][threadIdx.x] = ~0u;
            }
        }
        t0 = t1;  // take the next chunk
    }

    TL(2);
#if SQF2K_TMA_EXPORT
    if (!FUSED && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
    if (FUSED) {  // this CTA's minima and counts
        __syncthreads();
        if (threadIdx.x >= 1 && threadIdx.x <= kDepthMax) {
            const unsigned long long f = S.first[threadIdx.x];
            if (f != ~0ull)
                atomicMin(&P.min_n[threadIdx.x], (unsigned long long)(P.base_n + 2 * (int64_t)f));
        }
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int k = 2; k <= KMAIN; ++k) {  // met at k: pending after k - 1, not after k
            const unsigned long long s = warp_sum_u64(c[k - 1] - c[k]);
            if (lane == 0 && s) atomicAdd(&P.hist[k], s);
        }
        if (KMAIN >= 2 && threadIdx.x == 0 && S.cnt[0])  // (mod 2^64: the sum comes out right)
            atomicAdd(&P.hist[KMAIN], 0ull - (unsigned long long)S.cnt[0]);
        const unsigned long long sc = warp_sum_u64(scanned);
        if (lane == 0 && sc) atomicAdd(P.scanned, sc);
        if (threadIdx.x > kMainMax && threadIdx.x <= kDepthMax && S.cnt[threadIdx.x])
            atomicAdd(&P.hist[threadIdx.x], (unsigned long long)S.cnt[threadIdx.x]);
    }
    // the last CTA resets the scheduler for the next launch and (single-batch
    // fused calls) finishes the call
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) S.last = atomicAdd(&P.sched[1], 1u) == G - 1;
    __syncthreads();
    if (S.last) {
        __threadfence();
        if (FUSED && P.acc) finish_call(S, P);
        if (threadIdx.x == 0) {
            P.sched[0] = 0;
            P.sched[1] = 0;
        }
    }
    TL(3);
}

// -------------------------------------------------------------------------
// Medium-prime scatter schedule, built on the host from the table's primes in
// [11, kPMed) and cached on the device per set.  A prime with h = kTile/q
// hits per tile (q = p^2) and h >= 16*item is swept by whole warps (S sweeps of
// ~item hits per lane: lane l starts at hit l + 32s, step 32*S*q); a rarer
// prime is split into ~item-hit descriptors (start j, step parts*q).
// Descriptors sorted by trip count fill 32-lane tasks, and the tasks go to
// the kThreads/32 warps longest-first, at most kTaskSlots per warp (the
// item size grows until they fit).
struct MedTables {
    std::vector<uint32_t> q;      // p^2 per medium prime
    std::vector<uint32_t> tasks;  // (x, y) pairs: [warp][kTaskSlots][lane]
    uint32_t n_tasks = 0;
};

// schedule constant `name`, overridable by the environment (tuning sweeps:
// tools/med_sweep.sh)
double med_knob(const char *name, double dflt) {
    const char *v = std::getenv(name);
    return v ? atof(v) : dflt;
}

MedTables build_med(const std::vector<uint32_t> &med_primes, bool rotate) {
    constexpr int kWarps = kThreads / 32;
    struct Desc {
        double trips;
        uint32_t x, y;
    };
    // kind-2 calls (rotating bucket warp): constants from a random search over
    // item / bias / per-trip / per-task on C5 (experiments: 41 schedules,
    // 407.8 ms best against 410.4 for the best item-only choice, 7.5 hits)
    const double item0 = med_knob("SQF2K_MED_ITEM", rotate ? kItemHitsRotate : kItemHits);
    const double growth = med_knob("SQF2K_MED_GROWTH", SQF2K_ITEM_GROWTH);
    const double c_bucket = rotate ? 0.0 : med_knob("SQF2K_MED_BUCKET", SQF2K_LPT_BUCKET);
    const double c_bias = med_knob("SQF2K_MED_BIAS", rotate ? 0.75 : SQF2K_LPT_WARP_BIAS);
    const double c_trip = med_knob("SQF2K_MED_PER_TRIP", SQF2K_LPT_PER_TRIP);
    const double c_task = med_knob("SQF2K_MED_TASK", rotate ? 0.0 : SQF2K_LPT_TASK);
    for (double item = item0; item <= kTile; item *= growth) {
        MedTables t;
        std::vector<Desc> descs;
        for (uint32_t p : med_primes) {
            if (t.q.size() >= (size_t)kMaxMed) break;
            const uint32_t q = p * p, m = (uint32_t)t.q.size();
            t.q.push_back(q);
            const double h = (double)kTile / q;
            if (h >= 16.0 * item) {  // >= item/2 hits per lane
                const uint32_t S = std::max<uint32_t>(1, (uint32_t)(h / (32.0 * item) + 0.5));
                for (uint32_t sw = 0; sw < S; ++sw)
                    for (uint32_t l = 0; l < 32; ++l)
                        descs.push_back({h / (32.0 * S) + 1.0, m | ((l + 32 * sw) << 8), 32 * S * q});
            } else {
                const uint32_t parts = std::max<uint32_t>(1, (uint32_t)(h / item + 0.5));
                for (uint32_t j = 0; j < parts; ++j)
                    descs.push_back({h / parts + 1.0, m | (j << 8), parts * q});
            }
        }
        std::stable_sort(descs.begin(), descs.end(),
                         [](const Desc &a, const Desc &b) { return a.trips > b.trips; });
        const uint32_t n_tasks = (uint32_t)((descs.size() + 31) / 32);
        if (n_tasks > (uint32_t)(kWarps * kTaskSlots)) continue;
        std::vector<double> load(kWarps, 0.0);
        load[kWarps - 1] = c_bucket;  // the bucket warp (scatter_bucket)
        // the warp schedulers favour high warp ids: pre-charge the low ones
        for (int w = 0; w < kWarps; ++w) load[w] += c_bias * (kWarps - 1 - w);
        std::vector<int> used(kWarps, 0);
        t.tasks.assign((size_t)kWarps * kTaskSlots * 64, 0u);  // step 0: idle lane
        for (uint32_t k = 0; k < n_tasks; ++k) {  // longest first, least-loaded warp with room
            int w = -1;
            for (int i = 0; i < kWarps; ++i)
                if (used[i] < kTaskSlots && (w < 0 || load[i] < load[w])) w = i;
            // cost of a task: its longest lane (loop of 4 clears per trip) + overhead
            load[w] += descs[32 * k].trips / c_trip + c_task;
            const size_t at = ((size_t)w * kTaskSlots + used[w]++) * 64;
            for (uint32_t l = 0; l < 32; ++l) {
                const uint32_t i = 32 * k + l;
                if (i >= descs.size()) break;
                t.tasks[at + 2 * l] = descs[i].x;
                t.tasks[at + 2 * l + 1] = descs[i].y;
            }
        }
        t.n_tasks = n_tasks;
        return t;
    }
    throw Error{SQF2K_ECUDA, "medium-prime schedule does not fit the task slots"};
}

struct MedCache {
    std::vector<uint32_t> key;
    DevBuf buf;  // kMaxMed q values, then the task table
};

// one schedule per pattern kind (11 in the table or in the scatter), so
// calls alternating between small and large domains rebuild nothing; the
// library serialises calls
MedCache g_med[3];
MedCache &med_cache(const BatchArgs &a) { return g_med[pattern_kind(a.pattern_present)]; }

}  // namespace

// small primes by a host sieve (configuration data for the item schedule)
std::vector<uint32_t> small_primes(uint32_t below) {
    std::vector<uint8_t> comp(below + 1, 0);
    std::vector<uint32_t> out;
    for (uint32_t i = 2; i < below; ++i) {
        if (comp[i]) continue;
        out.push_back(i);
        for (uint64_t j = (uint64_t)i * i; j < below; j += i) comp[j] = 1;
    }
    return out;
}

size_t tile_smem_bytes() { return sizeof(TileSmem); }

// Upper bound of the bucket hits of a domain of U slots: sum over odd p >= 1031
// of (U/p^2 + 1) <= U / (2 * 1029) + n_bucket_primes.
uint64_t bucket_hits_bound(uint64_t U, uint64_t n_bucket) { return U / 2058 + 1 + n_bucket; }

template <bool FUSED, int KMAIN, int PAT>
void launch_tile_as(const char *name, unsigned grid, size_t smem, const TileParams &P, bool pdl) {
    static bool attr = false;
    if (!attr) {
        SQF2K_CUDA(cudaFuncSetAttribute(tile_kernel<FUSED, KMAIN, PAT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // carve only the shared memory kCtasPerSm CTAs need: the rest stays L1,
        // which holds the pattern table every tile reads
        const int pct = (int)((kCtasPerSm * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
        SQF2K_CUDA(cudaFuncSetAttribute(tile_kernel<FUSED, KMAIN, PAT>,
                                        cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        attr = true;
    }
    launch_ex(ctx().stream, pdl, name, tile_kernel<FUSED, KMAIN, PAT>, dim3(grid), dim3(kThreads),
              smem, P);
}

// pdl: programmatic dependent launch (the prologue overlaps the bucket fill
// before it on the stream).  Not for the batches of an overlapped multi-batch
// call, whose stream predecessor is the previous batch's tile kernel: early
// launched CTAs there measured 12-25 % slower calls in graph replays (C4:
// 29.5 -> 33.0-36.6 ms, timing-dependent) and the bucket fill is on the side
// stream anyway.
template <bool FUSED, int KMAIN>
void launch_tile(const char *name, unsigned grid, size_t smem, const TileParams &P, bool pdl) {
    if (kPattern13 && P.pat_words == pattern_words(24u)) {
        // (verify.cu selects kind 2 for fused default-depth calls only)
        if (!FUSED || KMAIN != kMainMax) throw Error{SQF2K_ECUDA, "pattern kind 2 needs the fused main-depth kernel"};
        launch_tile_as<FUSED, KMAIN, kPattern13 ? 2 : 0>(name, grid, smem, P, pdl);
    } else if (kPattern11 && P.pat_words == pattern_words(8u)) {
        launch_tile_as<FUSED, KMAIN, kPattern11 ? 1 : 0>(name, grid, smem, P, pdl);
    } else {
        launch_tile_as<FUSED, KMAIN, 0>(name, grid, smem, P, pdl);
    }
}

// Wheel tables.  The pattern words of a domain whose slot 0 is the odd n =
// base depend on base only through its residues mod q = 9, 25, 49 (121,
// 169), and a shift by one word (32 slots = 64 in n) steps every residue by
// 64, a unit mod their product Q: the table of base is the table of base 1
// read d words in, d = (base - 1) / 64 mod Q.  So each kind has one table,
// built for base 1 the first time a call needs it (kind 2: 3.6 GB, ~1 ms)
// and read by every later batch at its own offset.
uint64_t inv_mod(uint64_t a, uint64_t m) {  // a^-1 mod m (gcd(a, m) = 1)
    int64_t t = 0, nt = 1, r = (int64_t)m, nr = (int64_t)(a % m);
    while (nr) {
        const int64_t q = r / nr;
        std::tie(t, nt) = std::make_pair(nt, t - q * nt);
        std::tie(r, nr) = std::make_pair(nr, r - q * nr);
    }
    return (uint64_t)(t < 0 ? t + (int64_t)m : t);
}

uint32_t wheel_offset(int64_t base_n, uint32_t present) {
    const int kind = pattern_kind(present);
    const uint64_t Q = kind == 2 ? kPatPeriod13 : pattern_words(present);
    static const uint64_t inv[3] = {inv_mod(64, kPatWords3), inv_mod(64, kPatWords3 * 121ull),
                                    inv_mod(64, kPatPeriod13)};
    const int64_t diff = (base_n - 1) % (int64_t)Q;
    const uint64_t d = (uint64_t)(diff < 0 ? diff + (int64_t)Q : diff) * inv[kind] % Q;
    if (kind != 2) return (uint32_t)d;
    // kind 2 (four periods, no shifted copies): the d' = d mod Q that is 0
    // mod 4 keeps every tile start 16-byte aligned
    uint64_t e = d;
    while (e & 3u) e += Q;
    return (uint32_t)e;
}

void ensure_wheel(int kind, uint32_t present, cudaStream_t st) {
    Context &c = ctx();
    if (c.wheel_present[kind] == present) return;
    const PatResidues base1 = pat_residues(1);
    if (kind == 2) {
        // the p <= 11 table (kind 1) first, then its AND with the p = 13 words
        ensure_wheel(1, present & 15u, st);
        const uint32_t words = pattern_words(present) + kTileWords;
        c.pattern13.reserve((size_t)words * 4);
        c.wheel_present[2] = ~0u;
        launch_on(st, "pattern13", pattern13_kernel, dim3((unsigned)c.sm_count * 8), dim3(256), 0, (int64_t)1,
                  (const uint32_t *)c.pattern_b.as<uint32_t>(), c.pattern13.as<uint32_t>(), words);
    } else {
        // kPatCopies shifted copies (a tile start at any index has a 16-byte
        // aligned source), each a period plus a tile so that no start wraps
        DevBuf &t = kind == 1 ? c.pattern_b : c.pattern;
        const uint32_t pw = pattern_words(present);
        t.reserve((size_t)kPatCopies * kPatStride * 4);
        c.wheel_present[kind] = ~0u;
        launch_on(st, "pattern", pattern_kernel,
                  dim3((unsigned)std::min<uint64_t>(ceil_div(pw + kTileWords, 1024), c.sm_count * 8)), dim3(256),
                  0, base1, present, t.as<uint32_t>(), std::min(pw + kTileWords, kPatStride),
                  (uint32_t)kPatCopies, kPatStride);
    }
    c.wheel_present[kind] = present;
    dev_alloc_bump();  // captured graphs read the tables: a rebuilt one retires them
}

// Work of a batch that does not need the prime table: the medium schedule
// (host-built, cached), the p = 3, 5, 7 pattern and the bucket counters --
// on stream `st` (the side stream for the first batch of a call).
void prep_tile_batch(const BatchArgs &a, cudaStream_t st) {
    Context &c = ctx();

    // medium tables: cached per distinct prime set
    constexpr size_t kTaskWords = (size_t)(kThreads / 32) * kTaskSlots * 64;
    MedCache &med = med_cache(a);
    if (med.key != *a.med_primes || !med.buf.ptr) {
        MedTables t = build_med(*a.med_primes, SQF2K_BUCKET_ROTATE && pattern_kind(a.pattern_present) == 2);
        med.key = *a.med_primes;
        med.buf.reserve((kMaxMed + kTaskWords) * 4);
        std::vector<uint32_t> host(kMaxMed + kTaskWords, 0);
        std::copy(t.q.begin(), t.q.end(), host.begin());
        std::copy(t.tasks.begin(), t.tasks.end(), host.begin() + kMaxMed);
        SQF2K_CUDA(cudaMemcpy(med.buf.ptr, host.data(), host.size() * 4, cudaMemcpyHostToDevice));
        dev_alloc_bump();  // captured graphs read this table
    }

    // the wheel table of this kind (built once per context: its words depend
    // only on the primes in it; a batch reads it at wheel_offset)
    DevBuf &counts = a.buf ? c.tile_counts_b : c.tile_counts;
    ensure_wheel(pattern_kind(a.pattern_present), a.pattern_present, st);
    const uint32_t n_bt = (uint32_t)ceil_div(a.U, kBucketTile);
    counts.reserve((n_bt + 4) * 4);  // (+3: the tile starts copy 16-byte chunks)
    SQF2K_CUDA(cudaMemsetAsync(counts.ptr, 0, (n_bt + 1) * 4, st));
}

// prime-major bucket pass grid cap per SM (latency-bound chains of one unit
// per thread: 32 measured 418.5 vs 419.9 ms per C5 call for 8)
#ifndef SQF2K_BUCKET_GRID_PER_SM
#define SQF2K_BUCKET_GRID_PER_SM 32
#endif
// bucket work units (upper bound from pi(2^m) and the table size)
static unsigned bucket_grid(const BatchArgs &a, int j_min = 0) {
    uint64_t n_work = 0;
    static const uint32_t pi2[kClasses + 1] = SQF2K_PI_POW2;
    for (int j = j_min; j < kClasses; ++j) {
        const uint64_t hi = std::min<uint64_t>(pi2[j + 1], a.n_primes_bound);
        if (hi <= pi2[j]) break;
        const int sh = std::min(22 + 2 * j, 62);
        n_work += (hi - pi2[j]) * ((a.U + (1ull << sh) - 1) >> sh);
    }
    return (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>(ceil_div(n_work, 256), (uint64_t)ctx().sm_count * SQF2K_BUCKET_GRID_PER_SM));
}

// Fixed-capacity bucket lists of a batch on stream st (after its prep and
// the prime table): lets a multi-batch call build batch b's lists while
// batch b - 1's tile kernel runs.
void bucket_batch(const BatchArgs &a, cudaStream_t st) {
    Context &c = ctx();
    const uint32_t n_bt = (uint32_t)ceil_div(a.U, kBucketTile);
    DevBuf &hits = a.buf ? c.hits_b : c.hits;
    DevBuf &counts = a.buf ? c.tile_counts_b : c.tile_counts;
    hits.reserve((size_t)n_bt * kBucketCap * 2 + 64);
    if (dense_classes(n_bt))
        launch_on(st, "bucket_dense", bucket_dense_kernel, dim3((unsigned)ceil_div(n_bt, kDenseTiles)), dim3(256),
                  0, a.primes, a.info, a.base_n, a.U, counts.as<uint32_t>(), hits.as<uint16_t>(), a.overflow);
    launch_on(st, "bucket_fill", bucket_kernel<0>, dim3(bucket_grid(a, dense_classes(n_bt))), dim3(256), 0, a.primes,
              a.info, a.base_n, a.U, counts.as<uint32_t>(), (const uint32_t *)nullptr,
              hits.as<uint16_t>(), a.overflow, dense_classes(n_bt));
}

// Bucket lists and the tile kernel of a batch (after prep_tile_batch and the
// prime table), on the library stream.
void run_tile_batch(const BatchArgs &a) {
    Context &c = ctx();
    if (a.U > (1ull << 41)) throw Error{SQF2K_EINVAL, "batch domain above 2^41 slots"};
    const uint32_t n_tiles = (uint32_t)ceil_div(a.U, kTile);
    const uint32_t n_bt = (uint32_t)ceil_div(a.U, kBucketTile);

    // bucket lists (sizes bounded on the host: no sync)
    DevBuf &hits = a.buf ? c.hits_b : c.hits;
    uint32_t *counts = (a.buf ? c.tile_counts_b : c.tile_counts).as<uint32_t>();
    const unsigned bgrid = bucket_grid(a);
    const uint32_t *tile_start = nullptr;
    if (a.bucket_stream) {
        // lists already built by bucket_batch
    } else if (!a.exact_buckets) {
        hits.reserve((size_t)n_bt * kBucketCap * 2 + 64);
        if (dense_classes(n_bt))
            launch_pdl("bucket_dense", bucket_dense_kernel, dim3((unsigned)ceil_div(n_bt, kDenseTiles)), dim3(256), 0,
                       a.primes, a.info, a.base_n, a.U, counts, hits.as<uint16_t>(), a.overflow);
        launch_pdl("bucket_fill", bucket_kernel<0>, dim3(bucket_grid(a, dense_classes(n_bt))), dim3(256), 0,
                   a.primes, a.info,
                   a.base_n, a.U, counts, (const uint32_t *)nullptr, hits.as<uint16_t>(),
                   a.overflow, dense_classes(n_bt));
    } else {
        c.tile_offsets.reserve((n_bt + 1) * 4);
        uint32_t *offsets = c.tile_offsets.as<uint32_t>();
        hits.reserve(bucket_hits_bound(a.U, a.n_primes_bound) * 2 + 64);
        launch("bucket_count", bucket_kernel<1>, dim3(bgrid), dim3(256), 0, a.primes, a.info,
               a.base_n, a.U, counts, (const uint32_t *)offsets, (uint16_t *)nullptr, a.overflow, 0);
        launch("bucket_scan", scan_counts_kernel<uint32_t>, dim3(1), dim3(kScanThreads), 0,
               (const uint32_t *)counts, (uint64_t)n_bt, offsets);
        launch("bucket_fill", bucket_kernel<2>, dim3(bgrid), dim3(256), 0, a.primes, a.info,
               a.base_n, a.U, counts, (const uint32_t *)offsets, hits.as<uint16_t>(),
               a.overflow, 0);
        tile_start = offsets;
    }

    TileParams P;
    std::memset(&P, 0, sizeof P);
    P.base_n = a.base_n;
    P.U = a.U;
    P.scan_lo = a.scan_lo;
    P.z = a.z;
    P.one_u = a.one_u;
    P.H = a.H;
    P.n_tiles = n_tiles;
    P.n_btiles = n_bt;
    P.k_eff = a.k_eff;
    P.k_max = a.k_max;

    P.pat_words = pattern_words(a.pattern_present);
    P.pat_off = wheel_offset(a.base_n, a.pattern_present);
    const int kind = pattern_kind(a.pattern_present);
    if (ctx().wheel_present[kind] != a.pattern_present) throw Error{SQF2K_ECUDA, "wheel table not built"};
    P.pattern = (kind == 2 ? c.pattern13 : kind == 1 ? c.pattern_b : c.pattern).as<uint32_t>();
    P.med = med_cache(a).buf.as<uint32_t>();
    P.tasks = reinterpret_cast<const uint2 *>(med_cache(a).buf.as<uint32_t>() + kMaxMed);
    P.tile_start = tile_start;
    P.tile_count = counts;
    P.hits = hits.as<uint16_t>();
    P.hist = a.hist;
    P.min_n = a.min_n;
    P.esc = a.esc;
    P.esc_count = a.esc_count;
    P.esc_cap = a.esc_cap;
    P.fail = a.fail;
    P.fail_count = a.fail_count;
    P.fail_cap = a.fail_cap;
    P.scanned = a.scanned;
    P.bits_out = a.bits_out;
    P.acc = a.fused ? a.finish_acc : nullptr;
    if (!c.sched.ptr) {  // self-resetting scheduler words, zeroed once
        c.sched.reserve(64);
        SQF2K_CUDA(cudaMemset(c.sched.ptr, 0, 64));
    }
    P.sched = c.sched.as<unsigned int>();
    P.acc_host = a.finish_host;
    P.primes = a.primes;
    P.info = a.info;

    const size_t smem = tile_smem_bytes();
    uint64_t grid_cap = (uint64_t)c.sm_count * kCtasPerSm;
    if (const char *g = std::getenv("SQF2K_DEBUG_GRID")) grid_cap = std::max(1, atoi(g));
    // at least ceil(n_tiles / 2^23) CTAs: the per-thread 32-bit counters
    grid_cap = std::max<uint64_t>(grid_cap, ceil_div(n_tiles, 1ull << 23));
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(n_tiles, grid_cap));
    const bool pdl = !a.bucket_stream;
    if (a.fused) {
        const uint32_t kmain = std::min<uint32_t>(a.k_eff, kMainMax);
        if (kmain == 1) launch_tile<true, 1>("tile_fused", grid, smem, P, pdl);
        else if (kmain == 2) launch_tile<true, 2>("tile_fused", grid, smem, P, pdl);
        else if (kmain == 3) launch_tile<true, 3>("tile_fused", grid, smem, P, pdl);
        else if (kmain == 4) launch_tile<true, 4>("tile_fused", grid, smem, P, pdl);
        else launch_tile<true, 5>("tile_fused", grid, smem, P, pdl);
    } else {
        launch_tile<false, 1>("tile_export", grid, smem, P, pdl);
    }
}

#ifdef SQF2K_EXP_TIMELINE
extern "C" int sqf2k_exp_timeline(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_timeline, sizeof(g_timeline)) == cudaSuccess ? 0 : -1;
}
extern "C" int sqf2k_exp_tiles(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_tiles, sizeof(g_tiles)) == cudaSuccess ? 0 : -1;
}
#endif

}  // namespace sqf2k

// tile.cuh -- the shared-memory tile sieve and the in-tile min-k scan.
//
// Domain of one launch ("batch"): slots u in [0, U) standing for the odd
// integers n(u) = base_n + 2u (base_n odd, possibly <= 0; n < 1 reads as
// "not squarefree", search.py:101-105).  Tiles are kTile consecutive slots.
//
// Per tile a CTA sieves the tile directly in packed form (one bit per odd
// slot, 32-bit LSB-first words in shared memory):
//   1. each word starts as the periodic mask of p = 3, 5, 7 (one table word
//      per u-word mod 9*25*49; a whole tile by one TMA bulk copy);
//   2. the odd multiples of p^2 are cleared with shared-memory atomic ANDs --
//      medium primes 11 <= p < kPMed from per-lane "descriptors" whose next
//      hit offset lives in a register across tiles (no division, no table
//      walk), bucket primes p >= kPMed from per-tile hit lists in HBM;
//   3. fused mode: runs the exponent passes k = 1..k_eff of search.py:187-200
//      over the words -- passes 1..5 unconditionally for every word (funnel
//      shifts of the word and its left neighbour), the rare remainder
//      divergently -- reading n - 2^k from the tile or the previous tile's
//      tail (2^(k_eff-1) slots of halo); export mode: stores the words (one
//      TMA bulk copy per tile).
#pragma once

#include <stdint.h>

#include <cuda_runtime.h>

#include <vector>

namespace sqf2k {

#ifndef SQF2K_TILE_SHIFT
#define SQF2K_TILE_SHIFT 16
#endif
constexpr int kTileShift = SQF2K_TILE_SHIFT;
constexpr int kTile = 1 << kTileShift;  // slots per tile (65536)
constexpr int kTileWords = kTile / 32;  // 2048 packed words
// bucket lists are kept per "bucket tile" of 2^kBucketShift slots (16-bit
// offsets); a tile holds kSubTiles of them
#ifndef SQF2K_BUCKET_SHIFT
#define SQF2K_BUCKET_SHIFT 16
#endif
constexpr int kBucketShift = SQF2K_BUCKET_SHIFT;
constexpr int kBucketTile = 1 << kBucketShift;
constexpr int kSubTiles = kTile / kBucketTile;
static_assert(kTile >= kBucketTile, "tiles are whole bucket tiles");
#ifndef SQF2K_WORDS_PER_THREAD
#define SQF2K_WORDS_PER_THREAD 8
#endif
constexpr int kWordsPerThread = SQF2K_WORDS_PER_THREAD;  // words per thread in pack and scan
constexpr int kThreads = kTileWords / kWordsPerThread;  // CTA size
#ifndef SQF2K_CTAS_PER_SM
#define SQF2K_CTAS_PER_SM 4
#endif
constexpr int kCtasPerSm = SQF2K_CTAS_PER_SM;
constexpr int kDepthMax = 16;           // max exponent resolved in-tile
#ifndef SQF2K_KMAIN_MAX
#define SQF2K_KMAIN_MAX 5
#endif
constexpr int kMainMax = SQF2K_KMAIN_MAX;  // unconditional scan passes (4 or 5)
static_assert(kMainMax == 4 || kMainMax == 5, "main passes");
#ifndef SQF2K_DEPTH_DEFAULT
#define SQF2K_DEPTH_DEFAULT 16
#endif
// default in-tile depth (k <= 13 for every odd n < 2^50, PAPER.md:258-261;
// 13 measured no faster, so the default keeps the widest in-tile range)
constexpr int kDepthDefault = SQF2K_DEPTH_DEFAULT;
constexpr int kHaloMax = 1 << (kDepthMax - 1);
constexpr int kHaloWordsMax = kHaloMax / 32;
constexpr uint32_t kPMed = 1024;        // medium primes: 11 <= p < kPMed
constexpr int kMaxMed = 176;            // pi(1023) - 4 = 168
#ifndef SQF2K_TASK_SLOTS
#define SQF2K_TASK_SLOTS 2
#endif
constexpr int kTaskSlots = SQF2K_TASK_SLOTS;  // 32-lane scatter tasks per warp (registers)
#ifndef SQF2K_ITEM_HITS
#define SQF2K_ITEM_HITS 9.0
#endif
// target hits per lane per tile of the medium schedule (build_med); swept on
// the C4/C5 windows with tools/med_sweep.sh: 9 (with SQF2K_LPT_WARP_BIAS
// 0.25) 28.6 ms per C4 call against 29.5-30.0 for 3..8 and 10..16
constexpr double kItemHits = SQF2K_ITEM_HITS;
constexpr double kItemHitsRotate = 6.24;  // the same for the kind-2 schedule (tile.cu)
#ifndef SQF2K_PATTERN_11
#define SQF2K_PATTERN_11 1
#endif
// p = 3, 5, 7 (and 11) are applied as one periodic word pattern: period
// 9*25*49 words, or 9*25*49*121 with 11 (1.33 M words, 5.3 MB per copy,
// L2-resident).  Taking 11 (541 hits per 2^16-slot tile, 27 % of the medium
// scatter) out of the scatter measured 484.6 -> 467.7 ms per C5 call.  The
// tables are wheel constants (tile.cu: ensure_wheel, built once per context
// for the odd n = 1 and read at a per-batch word offset), so every domain
// takes them: C2 0.088 -> 0.084 ms per call once the per-call build (9.5 us
// for the 11 table) left the critical path.  SQF2K_PATTERN_11=0 never uses 11.
constexpr bool kPattern11 = SQF2K_PATTERN_11 != 0;
constexpr uint32_t kPatWords3 = 9 * 25 * 49;
constexpr uint32_t kPatWordsMax = kPatWords3 * (kPattern11 ? 121 : 1);
#ifndef SQF2K_PATTERN_11_MIN_SLOTS
#define SQF2K_PATTERN_11_MIN_SLOTS 0
#endif
constexpr uint64_t kPattern11MinSlots = SQF2K_PATTERN_11_MIN_SLOTS;
// ... and 13 as well for fused calls from 2^28 slots (SQF2K_PATTERN_13):
// period 9*25*49*121*169 = 225.45 M words (3.6 GB, stored as four periods so
// that every tile start is 16-byte aligned without shifted copies, read from
// HBM by the tile starts: 8 KB per 2^16-slot tile); it takes the 388 hits per
// tile of p = 13 out of the scatter (A/B against the per-call tables of
// before: C2 0.084 -> 0.083, C3 1.734 -> 1.705, C4 26.48 -> 25.59, C5
// 407.7 -> 406.7 ms per call; smaller calls do not allocate it).
#ifndef SQF2K_PATTERN_13
#define SQF2K_PATTERN_13 1
#endif
constexpr bool kPattern13 = SQF2K_PATTERN_13 != 0 && kPattern11;
constexpr uint32_t kPatPeriod13 = kPatWords3 * 121 * 169;
#ifndef SQF2K_PATTERN_13_MIN_SLOTS
#define SQF2K_PATTERN_13_MIN_SLOTS (1ull << 28)
#endif
constexpr uint64_t kPattern13MinSlots = SQF2K_PATTERN_13_MIN_SLOTS;
// index period of the table whose present mask is `present` (bit 3: prime
// 11, bit 4: prime 13 -- four periods, see above)
__host__ __device__ constexpr uint32_t pattern_words(uint32_t present) {
    return (present & 16u) ? 4 * kPatPeriod13 : (present & 8u) ? kPatWords3 * 121 : kPatWords3;
}
// table kind: 0 (3, 5, 7), 1 (+ 11), 2 (+ 11, 13)
__host__ __device__ constexpr int pattern_kind(uint32_t present) {
    return (present & 16u) ? 2 : (present & 8u) ? 1 : 0;
}
#ifndef SQF2K_MIN_CHUNK
#define SQF2K_MIN_CHUNK 4
#endif
#ifndef SQF2K_STATIC_EIGHTHS
#define SQF2K_STATIC_EIGHTHS 6
#endif
constexpr int kMinChunk = SQF2K_MIN_CHUNK;  // smallest dynamic chunk (tiles; each adds a halo)
constexpr int kStaticEighths = SQF2K_STATIC_EIGHTHS;  // static share of the tiles, in eighths
#ifndef SQF2K_DYN_MIN_TILES
#define SQF2K_DYN_MIN_TILES 64
#endif
constexpr int kDynMinTiles = SQF2K_DYN_MIN_TILES;  // dynamic balancing from this many tiles per CTA
constexpr int kResCap = 256;           // deferred residue words per tile
// fixed-capacity bucket list per bucket tile (mean <= 9.2 hits per 2^16
// slots: sum over p >= 1031 of 2^16 / p^2; an overflow reruns the batch with
// exact lists)
constexpr int kBucketCap = kBucketShift >= 16 ? 64 : 24;
constexpr uint32_t kPiBelowPMed = 172;  // pi(1023): table index of the first bucket prime
constexpr uint32_t kPiSubRoot = 1028;   // pi(8191): last "dense" bucket prime (p^2 < 2^26)

// Bucket primes come in classes j = 0..kClasses-1 of p in [2^(10+j), 2^(11+j)).
// A class-j work unit is one prime over a sub-range of 2^(22+2j) slots, so it
// has at most 2^(22+2j) / 2^(20+2j) + 1 = 5 hits: short atomic chains.
constexpr int kClasses = 22;  // up to p < 2^32
// pi(2^m) for m = 10..32 (OEIS A007053): class boundaries of a table that
// holds every prime <= limit.
#define SQF2K_PI_POW2                                                                       \
    {172u,      309u,      564u,      1028u,     1900u,      3512u,      6542u,     12251u,  \
     23000u,    43390u,    82025u,    155611u,   295947u,    564163u,    1077871u,  2063689u, \
     3957809u,  7603553u,  14630843u, 28192750u, 54400028u, 105097565u, 203280221u}

// Prime-table split, kept in device memory so no host sync is needed.
struct PrimeInfo {
    unsigned long long count;  // primes in the table
    uint32_t i_lo;             // first bucket prime (p >= kPMed)
    uint32_t i_hi;             // end of the bucket primes (p^2 <= n_max)
    uint32_t cls[kClasses + 1];  // index of the first prime >= 2^(10+j), clipped to count
};

struct TileParams {
    int64_t base_n;      // n(u) = base_n + 2u
    uint64_t U;          // slots in the domain
    uint64_t scan_lo;    // first slot scanned (fused mode)
    uint64_t z;          // slots u < z have n < 1: all zero
    uint64_t one_u;      // slot of n = 1 if scanned (excluded), else ~0
    uint32_t H;          // halo slots (multiple of 1024; 0 in export mode)
    uint32_t n_tiles;
    uint32_t n_btiles;   // bucket tiles (2^16 slots) in the domain
    uint32_t k_eff;      // passes inside the tile
    uint32_t k_max;      // run limit: escalate when k_max > k_eff
    uint32_t pat_words;          // period of the pattern table (pattern_words)
    uint32_t pat_off;            // word offset of this batch's domain in the wheel table (wheel_offset)
    const uint32_t *pattern;     // p = 3, 5, 7 (11) mask by u-word mod pat_words (+ kTileWords
                                 // repeated words, so a tile never wraps)
    const uint32_t *med;         // q = p^2 of the medium primes
    const uint2 *tasks;          // [warp][kTaskSlots][lane]: (m | mult << 8, step), step 0 idle
    const uint32_t *tile_start;  // exact bucket lists: bounds, n_btiles + 1 (or null)
    const uint32_t *tile_count;  // fixed-capacity lists: hits of bucket tile b at b*kBucketCap
    const uint16_t *hits;        // bucket hits, offsets within the bucket tile
    unsigned long long *hist;    // [65]
    unsigned long long *min_n;   // [65]
    unsigned long long *esc;     // escalation list (n values)
    unsigned long long *esc_count;
    uint64_t esc_cap;
    unsigned long long *fail;
    unsigned long long *fail_count;
    uint64_t fail_cap;
    unsigned long long *scanned; // fused mode: odd n entering the scan (hist[1] by conservation)
    uint32_t *bits_out;          // export mode: packed words of the domain
    // last-CTA epilogue (single-batch fused calls): escalate, then copy the
    // accumulators to mapped host memory -- no escalate launch, no memcpy
    struct Acc *acc;             // null: no epilogue
    void *acc_host;
    const uint32_t *primes;
    const PrimeInfo *info;
    unsigned int *sched;         // [0] dynamic chunks taken, [1] CTAs done (reset by the last)
};

// Protocol checks (build with -DSQF2K_CHECKS; tools/checks.sh): ring-buffer
// ownership tags, barrier phases and index bounds asserted on the device --
// the in-house substitute for compute-sanitizer's racecheck/synccheck/memcheck,
// which this pool does not allow.  A failed check prints and traps.
#ifdef SQF2K_CHECKS
#define SQF2K_CHECK(cond, ...)                                                   \
    do {                                                                         \
        if (!(cond)) {                                                           \
            printf("SQF2K_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x, #cond);          \
            __trap();                                                            \
        }                                                                        \
    } while (0)
#else
#define SQF2K_CHECK(cond, ...) do { } while (0)
#endif

// residue of the first slot u >= 0 with q | base_n + 2u, i.e. u = -base_n/2 mod q
__device__ __host__ __forceinline__ uint64_t slot_residue(int64_t base_n, uint64_t q) {
    uint64_t a;
    if (base_n >= 0) {
        uint64_t t = (uint64_t)base_n % q;
        a = t ? q - t : 0;
    } else {
        a = ((uint64_t)(-base_n)) % q;
    }
    return (a & 1) ? (a + q) / 2 : a / 2;
}

// Host description of one batch domain for run_tile_batch (tile.cu).
struct BatchArgs {
    bool fused;
    int64_t base_n;
    uint64_t U, scan_lo, z, one_u;
    uint32_t H, k_eff, k_max;
    const uint32_t *primes;       // device table
    const PrimeInfo *info;        // device split
    uint64_t n_primes_bound;      // host upper bound of the table size
    uint32_t pattern_present;     // bit i: prime 3/5/7/11/13 in the table
    const std::vector<uint32_t> *med_primes;
    unsigned long long *hist, *min_n, *esc, *esc_count, *fail, *fail_count;
    uint64_t esc_cap, fail_cap;
    unsigned long long *scanned;
    uint32_t *bits_out;
    bool exact_buckets;           // count + scan + fill instead of fixed capacity
    unsigned int *overflow;       // set when a fixed-capacity list overflowed
    int buf;                      // buffer set (pattern, bucket lists): 0 or 1
    cudaStream_t bucket_stream;   // non-null: run_tile_batch skips the (fixed) bucket fill,
                                  //   done earlier by bucket_batch on that stream
    struct Acc *finish_acc;       // non-null: the tile kernel's last CTA finishes the call
    void *finish_host;            //   (escalation + accumulators to this mapped host buffer)
};
void prep_tile_batch(const BatchArgs &a, cudaStream_t st);
void bucket_batch(const BatchArgs &a, cudaStream_t st);
void run_tile_batch(const BatchArgs &a);

}  // namespace sqf2k

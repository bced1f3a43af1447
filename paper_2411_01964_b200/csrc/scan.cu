// scan.cu -- L2 min-k scan over a packed bitmap window in HBM
// (replaces search.py:219-252 scan_segment and search.py:255-279
// scan_exponents; window rules of search.py:97-135).
//
// The window is one device bitmap: zeros | predecessor bits | current bits |
// zero pad, with current slot 0 at a 128-bit boundary.  One thread owns 128
// consecutive slots (one uint4): passes k <= 8 (shift < 128 slots) are funnel
// shifts of the thread's own uint4 and its left neighbour, passes k >= 9 are
// aligned 128-bit loads 2^(k-8) vectors back.  Per-k counts stay in registers,
// per-k least n goes through a block-level atomicMin, failures (or, in the
// two-pass verify pipeline, escalations) are appended to a device list.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace sqf2k {

uint64_t generate_primes_device(uint64_t limit);
void finish_summary(sqf2k_summary_t *out, const uint64_t *fail_sorted_head, uint64_t n_fail);
int deliver_failures(unsigned long long *fail_dev, uint64_t n_fail, uint64_t *failures,
                     uint64_t fail_cap, uint64_t *smallest);

namespace {

constexpr int kScanThreads = 256;

struct ScanParams {
    const uint4 *w4;     // window as 128-bit vectors
    uint64_t c0;         // vector index of current slot 0
    uint64_t n_slots;
    uint64_t first_n;    // n of current slot 0
    uint64_t one_slot;   // slot of n = 1 (excluded), ~0 if none
    uint32_t k_scan;     // passes
    uint32_t k_max;      // escalate leftovers when k_max > k_scan
    unsigned long long *hist, *min_n;
    unsigned long long *esc, *esc_count;
    uint64_t esc_cap;
    unsigned long long *fail, *fail_count;
    uint64_t fail_cap;
    uint8_t *kvals;      // exponent-dump mode
    unsigned long long *scanned;  // fast kernel: odd n entering the scan
};

// ---------------------------------------------------------------------------
// Fast summary scan (HBM-bound by design): each thread-iteration covers a
// group of 4 uint4 = 16 words = 512 slots, read with 4 LDG.128 (+ the word
// before the group).  Passes k = 1..4 run unconditionally on every word
// (funnel shifts of the word and its left neighbour); words still pending
// (~0.4%) continue through k = 5..k_scan with scalar loads.  Blocks own
// contiguous runs of groups, so each thread sees its slots in increasing
// order and records the least slot of each k = 1..4 the first time it meets
// it (register mask, rare-path atomics).  hist[1] is not counted: the host
// derives it from `scanned` by conservation, as for the fused kernel.
constexpr int kFastThreads = 256;
constexpr int kGroupWords = 8;

// Pending mask of the word starting at slot a (end of range, n = 1).
__device__ __forceinline__ uint32_t wscan_mask(const ScanParams &P, uint64_t a) {
    uint32_t pend = a >= P.n_slots ? 0u
                    : (a + 32 <= P.n_slots ? ~0u : ((1u << (uint32_t)(P.n_slots - a)) - 1u));
    if (P.one_slot >= a && P.one_slot < a + 32) pend &= ~(1u << (uint32_t)(P.one_slot - a));
    return pend;
}

// A word still pending after the main passes (rare): redo passes 1..KMAIN
// uncounted from the bits in memory, continue up to k_scan, then escalate or
// fail what is left.
__device__ void wscan_residue(const ScanParams &P, const uint32_t *__restrict__ w, uint64_t word,
                              uint64_t slot0, uint32_t kmain, uint32_t *s_cnt,
                              unsigned long long *s_first) {
    const uint32_t cur = w[word], prv = w[word - 1];
    uint32_t pend = wscan_mask(P, slot0);
    for (uint32_t k = 1; k <= P.k_scan && pend; ++k) {
        uint32_t sl;
        if (k <= 5) sl = __funnelshift_l(prv, cur, 1u << (k - 1));
        else if (k == 6) sl = prv;
        else sl = w[word - (1ull << (k - 6))];
        const uint32_t nw = pend & sl;
        if (nw && k > kmain) {
            atomicAdd(&s_cnt[k], (uint32_t)__popc(nw));
            atomicMin(&s_first[k], (unsigned long long)(slot0 + __ffs(nw) - 1));
        }
        pend &= ~sl;
    }
    if (pend) {
        const bool esc = P.k_max > P.k_scan;
        for (uint32_t x = pend; x; x &= x - 1) {
            const uint64_t n = P.first_n + 2 * (slot0 + __ffs(x) - 1);
            unsigned long long *list = esc ? P.esc : P.fail;
            unsigned long long *count = esc ? P.esc_count : P.fail_count;
            const uint64_t cap = esc ? P.esc_cap : P.fail_cap;
            const unsigned long long j = atomicAdd(count, 1ull);
            if (j < cap) list[j] = n;
        }
    }
}

// One group of kGroupWords words: passes 1..KMAIN on every word, leftovers
// (~2e-4 of the words after 5 passes) to the residue path.  TRACK records
// least slots of k = 1..5 the thread has not met yet; EDGE masks the end of
// the range and n = 1.  The common path (neither) is ~18 ops per 32 slots.
template <int KMAIN, bool TRACK, bool EDGE>
__device__ __forceinline__ void wscan_group(const ScanParams &P, const uint32_t *__restrict__ w,
                                            uint64_t g, uint64_t word0, const uint32_t (&cur)[kGroupWords],
                                            uint32_t prv, uint32_t (&c)[6],
                                            unsigned long long &scanned, uint32_t &tneed,
                                            uint32_t *s_cnt, unsigned long long *s_first) {
    const uint64_t wg = word0 + g * kGroupWords;
    const uint64_t s0 = g * 32 * kGroupWords;  // first slot of the group
    uint32_t which = 0;  // words still pending after the main passes
#pragma unroll
    for (int i = 0; i < kGroupWords; ++i) {
        uint32_t pend = ~0u;
        if (EDGE) {
            pend = wscan_mask(P, s0 + 32 * i);
            scanned += __popc(pend);
        }
        const uint32_t cu = cur[i];
#pragma unroll
        for (int k = 1; k <= KMAIN; ++k) {
            const uint32_t sl = __funnelshift_l(prv, cu, 1u << (k - 1));
            const uint32_t nw = pend & sl;
            if (k >= 2) c[k] += __popc(nw);
            if (TRACK && nw && ((tneed >> k) & 1u)) {
                tneed &= ~(1u << k);
                atomicMin(&s_first[k], (unsigned long long)(s0 + 32 * i + __ffs(nw) - 1));
            }
            pend &= ~sl;
        }
        which |= (pend != 0u) << i;
        prv = cu;
    }
    if (!EDGE) scanned += 32 * kGroupWords;
    while (which) {
        const int i = __ffs(which) - 1;
        which &= which - 1;
        wscan_residue(P, w, wg + i, s0 + 32 * i, KMAIN, s_cnt, s_first);
    }
}

// the group's words (2 x LDG.128); lanes hold consecutive groups
[[maybe_unused]] __device__ __forceinline__ void wscan_load(const ScanParams &P, uint64_t wg,
                                           uint32_t (&cur)[kGroupWords]) {
#pragma unroll
    for (int v = 0; v < kGroupWords / 4; ++v) {
        const uint4 x = __ldcs(&P.w4[wg / 4 + v]);  // streamed once
        cur[4 * v] = x.x;
        cur[4 * v + 1] = x.y;
        cur[4 * v + 2] = x.z;
        cur[4 * v + 3] = x.w;
    }
}

template <int KMAIN>
__global__ void __launch_bounds__(kFastThreads) wscan_kernel(const ScanParams P) {
    __shared__ unsigned long long s_first[65];
    __shared__ uint32_t s_cnt[65];
    for (int k = threadIdx.x; k < 65; k += blockDim.x) {
        s_first[k] = ~0ull;
        s_cnt[k] = 0;
    }
    __syncthreads();
    const uint32_t *w = reinterpret_cast<const uint32_t *>(P.w4);
    const uint64_t word0 = P.c0 * 4;  // word index of slot 0
    const uint64_t n_groups = (P.n_slots + 32 * kGroupWords - 1) / (32 * kGroupWords);
    const uint64_t g_lo = n_groups * blockIdx.x / gridDim.x;
    const uint64_t g_hi = n_groups * (blockIdx.x + 1) / gridDim.x;
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};
    unsigned long long scanned = 0;
    uint32_t tneed = (2u << KMAIN) - 2u;  // k = 1..KMAIN not met yet by this thread
    const uint64_t g_edge = P.n_slots / (32 * kGroupWords);  // groups >= this touch the end
    const uint64_t g_one = P.one_slot == ~0ull ? ~0ull : P.one_slot / (32 * kGroupWords);
    const uint32_t lane = threadIdx.x & 31;
    // software pipeline: the next iteration's words are in flight while this
    // one is scanned; the left neighbour word comes from the lane before
    // (consecutive groups), lane 0 loads it
    uint32_t nxt[kGroupWords];
    uint64_t g = g_lo + threadIdx.x;
    const uint64_t g_first = g_lo + (threadIdx.x & ~31u);  // this warp's first group
    if (g_first < g_hi) {
        if (g < g_hi) wscan_load(P, word0 + g * kGroupWords, nxt);
    }
    for (uint64_t gw = g_first; gw < g_hi; gw += blockDim.x, g += blockDim.x) {
        uint32_t cur[kGroupWords];
#pragma unroll
        for (int i = 0; i < kGroupWords; ++i) cur[i] = nxt[i];
        const bool live = g < g_hi;
        uint32_t prv = __shfl_up_sync(0xffffffffu, cur[kGroupWords - 1], 1);
        if (lane == 0 && live) prv = w[word0 + g * kGroupWords - 1];
        if (g + blockDim.x < g_hi) wscan_load(P, word0 + (g + blockDim.x) * kGroupWords, nxt);
        if (live) {
            if (g >= g_edge || g == g_one)
                wscan_group<KMAIN, true, true>(P, w, g, word0, cur, prv, c, scanned, tneed, s_cnt, s_first);
            else if (tneed)
                wscan_group<KMAIN, true, false>(P, w, g, word0, cur, prv, c, scanned, tneed, s_cnt, s_first);
            else
                wscan_group<KMAIN, false, false>(P, w, g, word0, cur, prv, c, scanned, tneed, s_cnt, s_first);
        }
    }
#pragma unroll
    for (int k = 2; k <= 5; ++k) {
        const uint32_t s = __reduce_add_sync(0xffffffffu, c[k]);
        if ((threadIdx.x & 31) == 0 && s) atomicAdd(&s_cnt[k], s);
    }
    for (int d = 16; d >= 1; d >>= 1) scanned += __shfl_xor_sync(0xffffffffu, scanned, d);
    if ((threadIdx.x & 31) == 0 && scanned) atomicAdd(P.scanned, scanned);
    __syncthreads();
    for (int k = threadIdx.x; k < 65; k += blockDim.x) {
        if (s_cnt[k]) atomicAdd(&P.hist[k], (unsigned long long)s_cnt[k]);
        if (s_first[k] != ~0ull)
            atomicMin(&P.min_n[k], (unsigned long long)(P.first_n + 2 * s_first[k]));
    }
}

// TMA-fed pending-count scan (the default): the CTA's contiguous run of
// groups streams through a kStages-deep ring of 8 KB shared-memory blocks,
// each filled by one bulk copy (cp.async.bulk global -> shared, completion on
// an mbarrier) issued by thread 0 kStages - 1 blocks ahead -- no per-thread
// global loads and no prefetch registers on the path.  A thread reads its
// 8-word group (2 x LDS.128) and the word before it from shared memory and
// runs passes 1..5 as funnel shifts, counting the slots still *pending*
// after passes 1..4 (covered-bit popcounts, as tile_kernel does: ~16
// instructions per 32-slot word instead of ~25).  Groups at the range ends
// and the groups of the first block that still track per-k least slots take
// the direct-count path (wscan_group); the leftovers after pass 5 (~2e-4 of
// the words) go to wscan_residue for k >= 6.
// stages of the TMA ring: 2 x 8 KB with 8 CTAs per SM measured 3457 vs 3379
// GB/s for 4 stages at 6 CTAs per SM (the kernel is XU/ALU-bound: occupancy
// hides more than a deeper ring)
#ifndef SQF2K_SCAN_STAGES
#define SQF2K_SCAN_STAGES 2
#endif
constexpr int kStages = SQF2K_SCAN_STAGES;
constexpr int kBlockGroups = kFastThreads;                  // groups per block
constexpr int kBlockWords = kBlockGroups * kGroupWords;     // 2048 words = 8 KB
constexpr int kStageWords = kBlockWords + 4;                // + 16 B: the word before

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// Passes 1..5 of one group by pending counts: p[k] -= covered(k) per word
// (+ 32 per word added by the caller); returns the words with slots left.
__device__ __forceinline__ uint32_t wscan_pc_group(const uint32_t (&cur)[kGroupWords], uint32_t prv,
                                                   uint32_t (&p)[5]) {
    uint32_t all = ~0u;
#pragma unroll
    for (int i = 0; i < kGroupWords; ++i) {
        const uint32_t cu = cur[i];
        const uint32_t v1 = __funnelshift_l(prv, cu, 1);
        const uint32_t v2 = v1 | __funnelshift_l(prv, cu, 2);
        const uint32_t v3 = v2 | __funnelshift_l(prv, cu, 4);
        const uint32_t v4 = v3 | __funnelshift_l(prv, cu, 8);
        const uint32_t v5 = v4 | __funnelshift_l(prv, cu, 16);
        p[1] -= __popc(v1);
        p[2] -= __popc(v2);
        p[3] -= __popc(v3);
        p[4] -= __popc(v4);
        all &= v5;
        prv = cu;
    }
    return all;
}

#ifndef SQF2K_SCAN_GRID_PER_SM
#define SQF2K_SCAN_GRID_PER_SM 64
#endif
#ifndef SQF2K_SCAN_MIN_CTAS
#define SQF2K_SCAN_MIN_CTAS 8
#endif
template <int KMAIN>
__global__ void __launch_bounds__(kFastThreads, SQF2K_SCAN_MIN_CTAS) wscan_tma_kernel(const ScanParams P) {
    extern __shared__ __align__(128) uint32_t stage[];  // kStages x kStageWords
    __shared__ __align__(8) unsigned long long full[kStages];
    __shared__ unsigned long long s_first[65];
    __shared__ uint32_t s_cnt[65];
    for (int k = threadIdx.x; k < 65; k += blockDim.x) {
        s_first[k] = ~0ull;
        s_cnt[k] = 0;
    }
    if (threadIdx.x == 0)
        for (int i = 0; i < kStages; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const uint32_t *w = reinterpret_cast<const uint32_t *>(P.w4);
    const uint64_t word0 = P.c0 * 4;  // word index of slot 0 (a multiple of 4)
    const uint64_t n_groups = (P.n_slots + 32 * kGroupWords - 1) / (32 * kGroupWords);
    const uint64_t g_lo = n_groups * blockIdx.x / gridDim.x;
    const uint64_t g_hi = n_groups * (blockIdx.x + 1) / gridDim.x;
    const uint64_t n_blocks = (g_hi - g_lo + kBlockGroups - 1) / kBlockGroups;
    auto issue = [&](uint64_t j) {  // block j of this CTA into stage j % kStages
        const uint64_t g0 = g_lo + j * kBlockGroups;
        const uint64_t left_g = g_hi - g0;
        const uint32_t ng = left_g < (uint64_t)kBlockGroups ? (uint32_t)left_g : (uint32_t)kBlockGroups;
        const uint32_t bytes = (ng * kGroupWords + 4) * 4;
        const uint32_t st = (uint32_t)(j % kStages);
        const uint32_t bar = smem_u32(&full[st]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(stage + st * kStageWords)),
            "l"(w + word0 + g0 * kGroupWords - 4), "r"(bytes), "r"(bar)
            : "memory");
    };
    if (threadIdx.x == 0)
        for (uint64_t j = 0; j < kStages - 1 && j < n_blocks; ++j) issue(j);
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};  // direct counts (edge / tracking groups)
    uint32_t p[5] = {0, 0, 0, 0, 0};     // pending after pass k (pending-count groups)
    uint32_t left5 = 0;                  // their slots left after pass 5
    unsigned long long scanned = 0;
    const uint32_t all_k = (2u << KMAIN) - 2u;
    uint32_t need = all_k;  // k = 1..KMAIN whose least slot this CTA has not met
    const uint64_t g_edge = P.n_slots / (32 * kGroupWords);  // groups >= this touch the end
    const uint64_t g_one = P.one_slot == ~0ull ? ~0ull : P.one_slot / (32 * kGroupWords);
    for (uint64_t j = 0; j < n_blocks; ++j) {
        const uint32_t st = (uint32_t)(j % kStages);
        if (threadIdx.x == 0 && j + kStages - 1 < n_blocks) issue(j + kStages - 1);
        // wait for block j (phase parity of its stage)
        const uint32_t parity = (uint32_t)((j / kStages) & 1);
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                "selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_u32(&full[st])), "r"(parity)
                : "memory");
        const uint64_t g = g_lo + j * kBlockGroups + threadIdx.x;
        if (g < g_hi) {
            const uint32_t *b = stage + st * kStageWords + 4 + threadIdx.x * kGroupWords;
            uint32_t cur[kGroupWords];
#pragma unroll
            for (int v = 0; v < kGroupWords / 4; ++v) {
                const uint4 x = *reinterpret_cast<const uint4 *>(b + 4 * v);
                cur[4 * v] = x.x;
                cur[4 * v + 1] = x.y;
                cur[4 * v + 2] = x.z;
                cur[4 * v + 3] = x.w;
            }
            const uint32_t prv = b[-1];
            uint32_t tneed = need;
            if (g >= g_edge || g == g_one) {
                wscan_group<KMAIN, true, true>(P, w, g, word0, cur, prv, c, scanned, tneed, s_cnt, s_first);
            } else if (KMAIN < 5 || need) {
                if (need) wscan_group<KMAIN, true, false>(P, w, g, word0, cur, prv, c, scanned, tneed, s_cnt, s_first);
                else wscan_group<KMAIN, false, false>(P, w, g, word0, cur, prv, c, scanned, tneed, s_cnt, s_first);
            } else {
                const uint32_t all = wscan_pc_group(cur, prv, p);
#pragma unroll
                for (int k = 1; k <= 4; ++k) p[k] += 32 * kGroupWords;
                scanned += 32 * kGroupWords;
                if (all != ~0u) {  // rare: some slots left after pass 5
                    uint32_t pv = prv;
                    const uint64_t wg = word0 + g * kGroupWords, s0 = g * 32 * kGroupWords;
#pragma unroll
                    for (int i = 0; i < kGroupWords; ++i) {
                        const uint32_t cu = cur[i];
                        const uint32_t v5 = __funnelshift_l(pv, cu, 1) | __funnelshift_l(pv, cu, 2) |
                                            __funnelshift_l(pv, cu, 4) | __funnelshift_l(pv, cu, 8) |
                                            __funnelshift_l(pv, cu, 16);
                        pv = cu;
                        if (v5 == ~0u) continue;
                        left5 += __popc(~v5);
                        wscan_residue(P, w, wg + i, s0 + 32 * i, 5, s_cnt, s_first);
                    }
                }
            }
        }
        __syncthreads();  // stage st may be refilled (block j + kStages) from here on
        if (need) {       // least slots met in this block end the tracking (later blocks are larger)
            uint32_t nn = 0;
#pragma unroll
            for (int k = 1; k <= KMAIN; ++k)
                if (s_first[k] == ~0ull) nn |= 1u << k;
            need = nn & all_k;
        }
    }
#pragma unroll
    for (int k = 2; k <= 5; ++k) {  // direct counts, then the pending differences
        unsigned long long v = c[k];
        if (KMAIN == 5) v += (k < 5 ? (unsigned long long)(p[k - 1] - p[k]) : (unsigned long long)(p[4] - left5));
        const unsigned long long s = warp_sum64(v);
        if ((threadIdx.x & 31) == 0 && s) atomicAdd(&P.hist[k], s);
    }
    scanned = warp_sum64(scanned);
    if ((threadIdx.x & 31) == 0 && scanned) atomicAdd(P.scanned, scanned);
    __syncthreads();
    for (int k = threadIdx.x; k < 65; k += blockDim.x) {
        if (s_cnt[k]) atomicAdd(&P.hist[k], (unsigned long long)s_cnt[k]);
        if (s_first[k] != ~0ull)
            atomicMin(&P.min_n[k], (unsigned long long)(P.first_n + 2 * s_first[k]));
    }
}


template <bool EXPO>
__global__ void __launch_bounds__(kScanThreads) window_scan_kernel(const ScanParams P) {
    __shared__ unsigned long long s_first[65];
    __shared__ unsigned int s_hist[65];
    for (int k = threadIdx.x; k < 65; k += blockDim.x) {
        s_first[k] = ~0ull;
        s_hist[k] = 0;
    }
    __syncthreads();
    uint32_t cnt[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) cnt[k] = 0;
    const uint64_t n_vec = (P.n_slots + 127) / 128;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n_vec;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 cur = P.w4[P.c0 + v];
        const uint4 prv = P.w4[P.c0 + v - 1];
        const uint64_t s0 = 128 * v;
        uint32_t pend[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint64_t a = s0 + 32 * i;
            uint32_t m = 0;
            if (a < P.n_slots) m = (a + 32 <= P.n_slots) ? ~0u : ((1u << (uint32_t)(P.n_slots - a)) - 1u);
            if (P.one_slot >= a && P.one_slot < a + 32) m &= ~(1u << (uint32_t)(P.one_slot - a));
            pend[i] = m;
        }
        const uint32_t wv[6] = {prv.z, prv.w, cur.x, cur.y, cur.z, cur.w};  // words -2..3
        for (uint32_t k = 1; k <= P.k_scan; ++k) {
            if (!(pend[0] | pend[1] | pend[2] | pend[3])) break;
            uint32_t sl[4];
            if (k <= 5) {
                const uint32_t s = 1u << (k - 1);
#pragma unroll
                for (int i = 0; i < 4; ++i) sl[i] = __funnelshift_l(wv[i + 1], wv[i + 2], s);
            } else if (k == 6) {
#pragma unroll
                for (int i = 0; i < 4; ++i) sl[i] = wv[i + 1];
            } else if (k == 7) {
#pragma unroll
                for (int i = 0; i < 4; ++i) sl[i] = wv[i];
            } else if (k == 8) {
                sl[0] = prv.x; sl[1] = prv.y; sl[2] = prv.z; sl[3] = prv.w;
            } else {
                const uint4 b = P.w4[P.c0 + v - (1ull << (k - 8))];
                sl[0] = b.x; sl[1] = b.y; sl[2] = b.z; sl[3] = b.w;
            }
            uint32_t c = 0;
            uint64_t first = ~0ull;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t nw = pend[i] & sl[i];
                if (nw) {
                    c += __popc(nw);
                    if (first == ~0ull) first = s0 + 32 * i + __ffs(nw) - 1;
                    if (EXPO)
                        for (uint32_t x = nw; x; x &= x - 1)
                            P.kvals[s0 + 32 * i + __ffs(x) - 1] = (uint8_t)k;
                }
                pend[i] &= ~sl[i];
            }
            if (c) {
#pragma unroll
                for (int kk = 1; kk <= 8; ++kk)
                    if (kk == (int)k) cnt[kk] += c;
                if (k > 8) atomicAdd(&s_hist[k], c);
                atomicMin(&s_first[k], first);
            }
        }
        if (!EXPO && (pend[0] | pend[1] | pend[2] | pend[3])) {
            const bool esc = P.k_max > P.k_scan;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                for (uint32_t x = pend[i]; x; x &= x - 1) {
                    const uint64_t n = P.first_n + 2 * (s0 + 32 * i + __ffs(x) - 1);
                    unsigned long long *list = esc ? P.esc : P.fail;
                    unsigned long long *count = esc ? P.esc_count : P.fail_count;
                    const uint64_t cap = esc ? P.esc_cap : P.fail_cap;
                    unsigned long long j = atomicAdd(count, 1ull);
                    if (j < cap) list[j] = n;
                }
        }
    }
    if (!EXPO) {
#pragma unroll
        for (int k = 1; k <= 8; ++k) {
            uint32_t s = __reduce_add_sync(0xffffffffu, cnt[k]);
            if ((threadIdx.x & 31) == 0 && s) atomicAdd(&s_hist[k], s);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < 65; k += blockDim.x) {
            if (s_hist[k]) atomicAdd(&P.hist[k], (unsigned long long)s_hist[k]);
            if (s_first[k] != ~0ull)
                atomicMin(&P.min_n[k], (unsigned long long)(P.first_n + 2 * s_first[k]));
        }
    }
}

// Copy predecessor bits (LSB-first bytes, prev_n bits) so that bit i lands at
// window bit D + i; words [D/32, end_word) are written, bits below D are 0.
__global__ void place_bits_kernel(const uint32_t *__restrict__ src, uint64_t src_bits,
                                  uint64_t D, uint64_t end_word, uint32_t *__restrict__ dst) {
    const uint64_t w_lo = D / 32;
    for (uint64_t j = w_lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < end_word;
         j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t out = 0;
        for (int b = 0; b < 32; ++b) {
            uint64_t pos = 32 * j + b;
            if (pos < D) continue;
            uint64_t i = pos - D;
            if (i >= src_bits) break;
            out |= ((src[i >> 5] >> (i & 31)) & 1u) << b;
        }
        dst[j] = out;
    }
}

struct ScanAcc {
    unsigned long long hist[SQF2K_HIST_LEN];
    unsigned long long min_n[SQF2K_HIST_LEN];
    unsigned long long esc_count, fail_count;
    unsigned long long scanned;
};

unsigned grid_for(uint64_t n_vec) {
    Context &c = ctx();
    return (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>(ceil_div(n_vec, kScanThreads), (uint64_t)c.sm_count * 8));
}

// Build the device window of search.py:97-135 (validation already done).
// Returns the vector index of current slot 0.
uint64_t build_window(const uint8_t *prev, uint64_t prev_n, const uint8_t *cur, uint64_t cur_n,
                      uint64_t prev_eff) {
    Context &c = ctx();
    const uint64_t P0 = ceil_div(std::max<uint64_t>(prev_eff, 128), 128) * 128;  // bits
    const uint64_t cur_bytes = ceil_div(cur_n, 64) * 8;
    const uint64_t total_bits = P0 + ceil_div(cur_n, 512) * 512 + 1024;  // whole scan groups + pad
    const uint64_t total_bytes = total_bits / 8;
    const uint64_t prev_bytes = prev ? ceil_div(prev_n, 64) * 8 : 0;
    c.window.reserve(total_bytes + prev_bytes + 64);
    uint8_t *w = c.window.as<uint8_t>();
    SQF2K_CUDA(cudaMemsetAsync(w, 0, total_bytes, c.stream));
    if (prev && prev_n) {
        uint8_t *staging = w + total_bytes + (8 - total_bytes % 8) % 8;
        copy_h2d(staging, prev, prev_bytes);
        const uint64_t D = P0 - prev_n;
        const uint64_t nw = P0 / 32 - D / 32;
        launch("window_place", place_bits_kernel,
               dim3((unsigned)std::min<uint64_t>(ceil_div(nw, 256), 4096)), dim3(256), 0,
               (const uint32_t *)staging, prev_n, D, P0 / 32, (uint32_t *)w);
    }
    copy_h2d(w + P0 / 8, cur, cur_bytes);
    return P0 / 128;
}

// Validation of search.py:38-43 and search.py:107-130; returns the
// effective predecessor depth (slots) or -1 with the error set.
int64_t window_depth(const uint8_t *prev, uint64_t prev_start, uint64_t prev_end,
                     uint64_t cur_start, uint64_t cur_end, uint32_t k_max) {
    if (cur_start < 1 || cur_start % 2 == 0 || cur_end <= cur_start || (cur_end - cur_start) % 2) {
        fail(SQF2K_EINVAL, "bad segment bounds [%llu, %llu)", (unsigned long long)cur_start,
             (unsigned long long)cur_end);
        return -1;
    }
    if (k_max < 1 || k_max > 63) {
        fail(SQF2K_EINVAL, "k_max must be positive, got %u", k_max);
        return -1;
    }
    const uint64_t need = ceil_div(1ull << (k_max - 1), 64) * 64;
    if (!prev) {
        if (cur_start != 1) {
            fail(SQF2K_EINVAL, "window starting at %llu needs a predecessor segment",
                 (unsigned long long)cur_start);
            return -1;
        }
        return (int64_t)need;
    }
    if (prev_end != cur_start) {
        fail(SQF2K_EINVAL, "segments not adjacent: previous ends at %llu, current starts at %llu",
             (unsigned long long)prev_end, (unsigned long long)cur_start);
        return -1;
    }
    const uint64_t pn = (prev_end - prev_start) / 2;
    if (pn >= need && pn % 64 == 0) return (int64_t)pn;
    if (prev_start == 1) return (int64_t)std::max(need, ceil_div(pn, 64) * 64);
    fail(SQF2K_EINVAL, "predecessor [%llu, %llu) is too shallow or unaligned for k_max %u",
         (unsigned long long)prev_start, (unsigned long long)prev_end, k_max);
    return -1;
}

}  // namespace

void scan_bitmap_device(const uint32_t *words, uint64_t cur_word0, uint64_t n_slots,
                        uint64_t first_n, uint32_t k_scan, uint32_t k_max, uint64_t one_slot,
                        unsigned long long *hist, unsigned long long *min_n,
                        unsigned long long *esc, unsigned long long *esc_count, uint64_t esc_cap,
                        unsigned long long *fail, unsigned long long *fail_count,
                        uint64_t fail_cap, unsigned long long *scanned) {
    ScanParams P;
    std::memset(&P, 0, sizeof P);
    P.w4 = reinterpret_cast<const uint4 *>(words);
    P.c0 = cur_word0 / 4;
    P.n_slots = n_slots;
    P.first_n = first_n;
    P.one_slot = one_slot;
    P.k_scan = k_scan;
    P.k_max = k_max;
    P.hist = hist;
    P.min_n = min_n;
    P.esc = esc;
    P.esc_count = esc_count;
    P.esc_cap = esc_cap;
    P.fail = fail;
    P.fail_count = fail_count;
    P.fail_cap = fail_cap;
    P.scanned = scanned;
    const uint64_t groups = ceil_div(n_slots, 32 * kGroupWords);
    // several waves of CTAs with contiguous runs: CTAs that finish early are
    // replaced by the next wave's (measured faster than one wave of long runs)
    // (TMA kernel: 32 CTAs per SM, 3.39 vs 3.08 TB/s at 8; the register-pipelined
    // kernel prefers 8)
    static const char *grid_env = std::getenv("SQF2K_SCAN_GRID_PER_SM");  // A/B measurements
    auto waves = [&](auto, size_t, uint64_t dflt) {
        const uint64_t per_sm = grid_env ? (uint64_t)std::max(1, atoi(grid_env)) : dflt;
        return (unsigned)std::max<uint64_t>(
            1, std::min<uint64_t>(ceil_div(groups, kFastThreads), (uint64_t)ctx().sm_count * per_sm));
    };
    static const bool ldg = [] {  // SQF2K_SCAN_KERNEL=ldg: the register-pipelined kernel (A/B)
        const char *e = std::getenv("SQF2K_SCAN_KERNEL");
        return e && std::strcmp(e, "ldg") == 0;
    }();
    if (!ldg) {
        const size_t smem = (size_t)kStages * kStageWords * 4;
        static bool attr = false;
        if (!attr) {
            for (auto *k : {wscan_tma_kernel<1>, wscan_tma_kernel<2>, wscan_tma_kernel<3>,
                            wscan_tma_kernel<4>, wscan_tma_kernel<5>})
                SQF2K_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = true;
        }
        const unsigned grid = waves(wscan_tma_kernel<5>, smem, SQF2K_SCAN_GRID_PER_SM);
        switch (std::min<uint32_t>(k_scan, 5)) {
            case 1: launch("window_scan", wscan_tma_kernel<1>, dim3(grid), dim3(kFastThreads), smem, P); break;
            case 2: launch("window_scan", wscan_tma_kernel<2>, dim3(grid), dim3(kFastThreads), smem, P); break;
            case 3: launch("window_scan", wscan_tma_kernel<3>, dim3(grid), dim3(kFastThreads), smem, P); break;
            case 4: launch("window_scan", wscan_tma_kernel<4>, dim3(grid), dim3(kFastThreads), smem, P); break;
            default: launch("window_scan", wscan_tma_kernel<5>, dim3(grid), dim3(kFastThreads), smem, P); break;
        }
        return;
    }
    const unsigned grid = waves(wscan_kernel<5>, 0, 8);
    switch (std::min<uint32_t>(k_scan, 5)) {
        case 1: launch("window_scan", wscan_kernel<1>, dim3(grid), dim3(kFastThreads), 0, P); break;
        case 2: launch("window_scan", wscan_kernel<2>, dim3(grid), dim3(kFastThreads), 0, P); break;
        case 3: launch("window_scan", wscan_kernel<3>, dim3(grid), dim3(kFastThreads), 0, P); break;
        case 4: launch("window_scan", wscan_kernel<4>, dim3(grid), dim3(kFastThreads), 0, P); break;
        default: launch("window_scan", wscan_kernel<5>, dim3(grid), dim3(kFastThreads), 0, P); break;
    }
}

}  // namespace sqf2k

using namespace sqf2k;

extern "C" int sqf2k_scan_window(const uint8_t *prev_bits, uint64_t prev_start, uint64_t prev_end,
                                 const uint8_t *cur_bits, uint64_t cur_start, uint64_t cur_end,
                                 uint32_t k_max, sqf2k_summary_t *out, uint64_t *failures,
                                 uint64_t fail_cap) {
    int64_t depth = window_depth(prev_bits, prev_start, prev_end, cur_start, cur_end, k_max);
    if (depth < 0) return SQF2K_EINVAL;
    return guarded([&](Context &c) -> int {
        const uint64_t cur_n = (cur_end - cur_start) / 2;
        const uint64_t prev_n = prev_bits ? (prev_end - prev_start) / 2 : 0;
        uint64_t dev_cap = std::max<uint64_t>(fail_cap, 1 << 12);
        for (int attempt = 0; attempt < 3; ++attempt) {
            const uint64_t c0 = build_window(prev_bits, prev_n, cur_bits, cur_n, (uint64_t)depth);
            c.acc.reserve(sizeof(ScanAcc));
            c.fail.reserve(dev_cap * 8);
            ScanAcc init;
            std::memset(&init, 0, sizeof init);
            for (int k = 0; k < SQF2K_HIST_LEN; ++k) init.min_n[k] = ~0ull;
            ScanAcc *acc = c.acc.as<ScanAcc>();
            copy_h2d(acc, &init, sizeof init);
            scan_bitmap_device(c.window.as<uint32_t>(), c0 * 4, cur_n, cur_start, k_max, k_max,
                               cur_start == 1 ? 0 : ~0ull, acc->hist, acc->min_n, nullptr,
                               &acc->esc_count, 0, c.fail.as<unsigned long long>(),
                               &acc->fail_count, dev_cap, &acc->scanned);
            ScanAcc h;
            copy_d2h(&h, acc, sizeof h);
            SQF2K_CUDA(cudaStreamSynchronize(c.stream));
            if (h.fail_count > dev_cap && h.fail_count <= fail_cap) {
                dev_cap = h.fail_count;
                continue;
            }
            std::memset(out, 0, sizeof *out);
            out->start = cur_start;
            out->end = cur_end;
            out->k_max = k_max;
            for (int k = 0; k < SQF2K_HIST_LEN; ++k) {
                out->hist[k] = h.hist[k];
                out->min_n[k] = h.min_n[k];
            }
            {  // k = 1 is not counted by the kernel: conservation, coverage checked
                const uint64_t expect = cur_n - (cur_start == 1 ? 1 : 0);
                if (h.scanned != expect)
                    return fail(SQF2K_ECUDA, "scan coverage %llu != %llu odd n",
                                (unsigned long long)h.scanned, (unsigned long long)expect);
                uint64_t rest = h.fail_count;
                for (int k = 2; k < SQF2K_HIST_LEN; ++k) rest += h.hist[k];
                out->hist[1] = h.scanned - rest;
            }
            if (h.fail_count > fail_cap) {
                out->n_failures = h.fail_count;
                return fail(SQF2K_ECAPACITY, "%llu failures exceed the buffer of %llu",
                            (unsigned long long)h.fail_count, (unsigned long long)fail_cap);
            }
            uint64_t smallest = SQF2K_NONE;
            deliver_failures(c.fail.as<unsigned long long>(), h.fail_count, failures, fail_cap,
                             &smallest);
            finish_summary(out, &smallest, h.fail_count);
            return SQF2K_OK;
        }
        return fail(SQF2K_ECUDA, "scan did not converge on buffer sizes");
    });
}

extern "C" int sqf2k_scan_exponents(const uint8_t *prev_bits, uint64_t prev_start,
                                    uint64_t prev_end, const uint8_t *cur_bits,
                                    uint64_t cur_start, uint64_t cur_end, uint32_t k_max,
                                    uint8_t *kvals, uint64_t n_slots) {
    int64_t depth = window_depth(prev_bits, prev_start, prev_end, cur_start, cur_end, k_max);
    if (depth < 0) return SQF2K_EINVAL;
    if (n_slots != (cur_end - cur_start) / 2)
        return fail(SQF2K_EINVAL, "kvals holds %llu slots, segment has %llu",
                    (unsigned long long)n_slots, (unsigned long long)((cur_end - cur_start) / 2));
    return guarded([&](Context &c) -> int {
        const uint64_t prev_n = prev_bits ? (prev_end - prev_start) / 2 : 0;
        const uint64_t c0 = build_window(prev_bits, prev_n, cur_bits, n_slots, (uint64_t)depth);
        c.kvals.reserve(n_slots + 16);
        SQF2K_CUDA(cudaMemsetAsync(c.kvals.ptr, 0, n_slots, c.stream));
        ScanParams P;
        std::memset(&P, 0, sizeof P);
        P.w4 = reinterpret_cast<const uint4 *>(c.window.ptr);
        P.c0 = c0;
        P.n_slots = n_slots;
        P.first_n = cur_start;
        P.one_slot = cur_start == 1 ? 0 : ~0ull;
        P.k_scan = k_max;
        P.k_max = k_max;
        P.kvals = c.kvals.as<uint8_t>();
        launch("window_exponents", window_scan_kernel<true>,
               dim3(grid_for(ceil_div(n_slots, 128))), dim3(kScanThreads), 0, P);
        copy_d2h(kvals, c.kvals.ptr, n_slots);
        SQF2K_CUDA(cudaStreamSynchronize(c.stream));
        return SQF2K_OK;
    });
}

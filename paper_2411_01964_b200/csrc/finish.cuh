// finish.cuh -- the end of a verify call on the device: the accumulators,
// exact escalation of the n left unresolved by the in-tile passes, and the
// trial-division squarefree test they use.
#pragma once

#include <stdint.h>

#include "../../include/sqf2k_b200.h"
#include "tile.cuh"

namespace sqf2k {

// Device accumulators of one verify call (zeroed / min_n set to ~0 per call).
struct Acc {
    unsigned long long hist[SQF2K_HIST_LEN];
    unsigned long long min_n[SQF2K_HIST_LEN];
    unsigned long long esc_count, fail_count;
    unsigned long long scanned;  // fused pipeline: odd n that entered the scan
    unsigned int overflow;
    unsigned int done;           // tile CTAs finished (last-CTA epilogue)
};

// Exact squarefree test by trial division, one warp per m (odd m >= 1):
// lanes take the odd primes p (index >= 1) with p^2 <= m.
__device__ inline bool warp_squarefree(uint64_t m, const uint32_t *__restrict__ primes,
                                       uint64_t n_primes) {
    const int lane = threadIdx.x & 31;
    for (uint64_t base = 1; base < n_primes; base += 32) {
        const uint64_t i = base + lane;
        bool live = false, hit = false;
        if (i < n_primes) {
            const uint64_t p = primes[i];
            const uint64_t q = p * p;
            live = q <= m;
            hit = live && (m % q == 0);
        }
        if (__any_sync(0xffffffffu, hit)) return false;
        if (!__any_sync(0xffffffffu, live)) break;
    }
    return true;
}

__device__ inline void append_n(unsigned long long *list, unsigned long long *count, uint64_t cap,
                                uint64_t n) {
    const unsigned long long i = atomicAdd(count, 1ull);
    if (i < cap) list[i] = n;
}

// Escalation (search.py:168-216 for k > the tile depth): every listed n
// tries k = k_from..k_max exactly; warp `warp` of `n_warps` takes every
// n_warps-th entry.
__device__ inline void escalate_warps(const unsigned long long *esc, uint64_t count,
                                      uint32_t k_from, uint32_t k_max, const uint32_t *primes,
                                      uint64_t n_primes, unsigned long long *hist,
                                      unsigned long long *min_n, unsigned long long *fail,
                                      unsigned long long *fail_count, uint64_t fail_cap,
                                      uint64_t warp, uint64_t n_warps) {
    for (uint64_t i = warp; i < count; i += n_warps) {
        const uint64_t n = esc[i];
        uint32_t found = 0;
        for (uint32_t k = k_from; k <= k_max && !found; ++k) {
            if (n <= (1ull << k)) break;  // n - 2^k < 1
            if (warp_squarefree(n - (1ull << k), primes, n_primes)) found = k;
        }
        if ((threadIdx.x & 31) == 0) {
            if (found) {
                atomicAdd(&hist[found], 1ull);
                atomicMin(&min_n[found], (unsigned long long)n);
            } else {
                append_n(fail, fail_count, fail_cap, n);
            }
        }
    }
}

}  // namespace sqf2k

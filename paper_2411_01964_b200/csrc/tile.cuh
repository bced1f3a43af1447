// tile.cuh -- the shared-memory tile sieve and the in-tile min-k scan.
//
// Domain of one launch ("batch"): slots u in [0, U) standing for the odd
// integers n(u) = base_n + 2u (base_n odd, possibly <= 0; n < 1 reads as
// "not squarefree", search.py:282-286).  Tiles are kTile consecutive slots.
//
// Per tile a CTA
//   1. sets one byte per slot to 1 and stores 0 at every odd multiple of p^2
//      for the medium primes 11 <= p < kPMed (balanced "items" of <= ~9 hits,
//      per-CTA incremental offsets, no divisions) and for the bucket primes
//      p >= kPMed (hit lists precomputed per tile in HBM);
//   2. packs the bytes into 32-bit LSB-first words, ANDing in the periodic
//      patterns of p = 3, 5, 7 (q = 9, 25, 49) computed in registers;
//   3. (fused mode) runs the exponent passes k = 1..k_eff of search.py:368-381
//      on the packed words, reading n - 2^k from the tile or from the rolled
//      halo of the previous tile (2^(k_eff-1) slots);
//      (export mode) stores the packed words to HBM.
//
// Bytes are laid out so that packing 32 slots is two conflict-free LDS.128
// and seven shift-or's: within each 1024-slot block, slot s (local) lives at
//   ((s>>3)&3) | ((s&3)<<2) | (((s>>5)&31)<<4) | (((s>>2)&1)<<9)
// i.e. the 32-bit word x_i (i = s&7) of a 32-slot group holds the slots
// 8j+i in its bytes j, so  word = OR_i x_i << i.
#pragma once

#include <stdint.h>

namespace sqf2k {

constexpr int kTile = 1 << 16;          // slots per tile
constexpr int kTileWords = kTile / 32;  // 2048 packed words
constexpr int kThreads = 512;           // CTA size of the tile kernels
constexpr int kCtasPerSm = 2;
constexpr int kDepthMax = 16;           // max exponent resolved in-tile
constexpr int kHaloMax = 1 << (kDepthMax - 1);
constexpr int kHaloWordsMax = kHaloMax / 32;
constexpr uint32_t kPMed = 1024;        // medium primes: 11 <= p < kPMed
constexpr int kMaxMed = 176;            // pi(1023) - 4 = 168
constexpr int kMaxItems = 1024;
constexpr int kItemHits = 8;            // target hits per item per tile

struct TileParams {
    int64_t base_n;      // n(u) = base_n + 2u
    uint64_t U;          // slots in the domain
    uint64_t scan_lo;    // first slot scanned (fused mode)
    uint64_t z;          // slots u < z have n < 1: all zero
    uint64_t one_u;      // slot of n = 1 if scanned (excluded), else ~0
    uint32_t H;          // halo slots (multiple of 1024; 0 in export mode)
    uint32_t n_tiles;
    uint32_t k_eff;      // passes inside the tile
    uint32_t k_max;      // run limit: escalate when k_max > k_eff
    uint32_t pat_q[3];   // 9, 25, 49 (1 when that prime is absent)
    uint32_t pat_bits[3];
    uint32_t pat_r[3];   // residue of the first hit slot
    uint32_t n_med;
    uint32_t n_items;
    const uint32_t *med;    // per medium prime: q, residue, kTile mod q   (3 x n_med)
    const uint32_t *items;  // per item: (med << 16 | j), stride          (2 x n_items)
    const uint32_t *tile_start;  // bucket hit list bounds, n_tiles + 1
    const uint16_t *hits;        // bucket hits, offsets within the tile
    unsigned long long *hist;    // [65]
    unsigned long long *min_n;   // [65]
    unsigned long long *esc;     // escalation list (n values)
    unsigned long long *esc_count;
    uint64_t esc_cap;
    unsigned long long *fail;
    unsigned long long *fail_count;
    uint64_t fail_cap;
    uint32_t *bits_out;          // export mode: packed words of the domain
};

__device__ __forceinline__ uint32_t byte_pos(uint32_t s) {
    return (s & ~1023u) | ((s >> 3) & 3u) | ((s & 3u) << 2) | (((s >> 5) & 31u) << 4) |
           (((s >> 2) & 1u) << 9);
}

// shift left with PTX clamping: amounts >= 32 give 0
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t s) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
    return r;
}

// x mod q for the CTA-uniform 64-bit position u (q < 2^32)
__device__ __forceinline__ uint32_t mod_u64(uint64_t u, uint32_t q) { return (uint32_t)(u % q); }

}  // namespace sqf2k

// warp_tile.cuh -- the fused sieve + min-k scan with WARP-INDEPENDENT tiles
// (included by tile.cu inside its anonymous namespace; uses its helpers).
//
// Every warp owns a contiguous run of "warp tiles" of kWt = 2^14 odd slots
// (512 words) and a private ring of kWtRing = 3 tile buffers in shared
// memory (6 KB).  Per tile t a warp, on its own:
//   1. waits for tile t's start (the p = 3, 5, 7 pattern, one TMA bulk copy
//      issued two tiles earlier, completion on the buffer's mbarrier);
//   2. sieves it: medium primes 11 <= p < kPMed by red.shared.and from the
//      lane's register-resident descriptors (next-hit offsets that never leave
//      the registers, rebased by -kWt per tile), bucket primes p >= kPMed from
//      the tile's precomputed hit list (bucket tiles are warp tiles);
//   3. scans it (__syncwarp in between): passes k = 1..5 of search.py:187-205
//      unconditionally per word as funnel shifts of the word and its left
//      neighbour, counted by covered-bit popcounts; the rare words with slots
//      left after pass 5 continue in place with k = 6..k_eff, reading n - 2^k
//      up to 2^14 slots back -- inside tile t - 1, which is still in the ring;
//   4. issues the start of tile t + 2 into tile t - 1's buffer.
// There is no CTA barrier anywhere in the loop: a warp never waits for
// another warp, so the 32 warps of an SM stay busy independently (the CTA
// shape only packs warps and their rings into shared memory).
//
// Work split: a static contiguous share of ~3/4 of the tiles per warp, the
// rest in chunks handed out by one global atomic; a chunk starting at t0 > 0
// first re-sieves tile t0 - 1 (the halo below it, as seed_predecessor does,
// runner.py:93-102).  Domain, edge masks, counting and the last-CTA epilogue
// follow tile_kernel exactly.

#ifndef SQF2K_WT_SHIFT
#define SQF2K_WT_SHIFT 14
#endif
#ifndef SQF2K_WT_WARPS
#define SQF2K_WT_WARPS 8
#endif
#ifndef SQF2K_WT_CTAS
#define SQF2K_WT_CTAS 3
#endif
#ifndef SQF2K_WT_SLOTS
#define SQF2K_WT_SLOTS 8
#endif
#ifndef SQF2K_WT_ITEM
#define SQF2K_WT_ITEM 4.0
#endif
#ifndef SQF2K_WT_DYN_MIN
#define SQF2K_WT_DYN_MIN 48
#endif

constexpr int kWtShift = SQF2K_WT_SHIFT;
constexpr int kWt = 1 << kWtShift;              // slots per warp tile
constexpr int kWtWords = kWt / 32;               // 512 words
constexpr int kWtRing = 3;                       // tile buffers per warp
constexpr int kWtRingWords = kWtRing * kWtWords;
constexpr int kWtLaneWords = kWtWords / 32;      // words per lane in the scan (16)
constexpr int kWtWarps = SQF2K_WT_WARPS;         // warps per CTA
constexpr int kWtThreads = 32 * kWtWarps;
constexpr int kWtCtasPerSm = SQF2K_WT_CTAS;
constexpr int kWtSlots = SQF2K_WT_SLOTS;         // medium descriptors per lane
constexpr int kWtDepthMax = kWtShift + 1;        // n - 2^k stays within the previous tile
constexpr int kWtDynMin = SQF2K_WT_DYN_MIN;      // dynamic chunks from this many tiles per warp
static_assert(kWtLaneWords % 4 == 0, "4-word scan chunks");
static_assert(kBucketShift <= kWtShift, "warp tiles are whole bucket tiles");
constexpr int kWtSubTiles = kWt / kBucketTile;   // bucket lists per warp tile

struct alignas(128) WarpRing {
    uint32_t ring[kWtRingWords];
    unsigned long long bar[kWtRing];  // start of buffer b: one phase per start
    unsigned long long first[kMainMax + 1];  // least slot with exponent k (k <= 5) in this chunk
#ifdef SQF2K_CHECKS
    uint32_t tag[kWtRing];  // tile held by buffer b (started), checks only
#endif
};
struct WtSmem {
    WarpRing w[kWtWarps];
    uint32_t step[kWtSlots][32];  // descriptor steps (the same for every warp)
    uint32_t last;
};

__device__ __forceinline__ uint32_t wt_base(uint32_t t) { return (t % kWtRing) * kWtWords; }
__device__ __forceinline__ uint32_t wt_back(uint32_t i, uint32_t d) {  // ring word i - d
    return i >= d ? i - d : i + kWtRingWords - d;
}

// the lane's next-hit offsets (registers); the steps are read from the
// CTA's shared copy of the table each tile (registers are the limit)
struct WtLane {
    uint32_t o[kWtSlots];
};

// Lane's descriptors, first hits at or after slot b0 (relative offsets);
// once per chunk.
__device__ __forceinline__ void wt_init_medium(WtLane &L, const TileParams &P, uint64_t b0) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < kWtSlots; ++j) {
        const uint2 d = __ldg(&P.wtasks[j * 32 + lane]);
        L.o[j] = ~0u;
        if (d.y) {
            const uint32_t q = __ldg(&P.med[d.x & 0xffu]);
            const uint32_t r = (uint32_t)slot_residue(P.base_n, q);
            const uint32_t bm = (uint32_t)(b0 % q);
            L.o[j] = (r >= bm ? r - bm : r + q - bm) + (d.x >> 8) * q;
        }
    }
}

// Clear the lane's medium hits in [0, kWt) of the tile at shared address
// wbase and rebase the offsets to the next tile.  Slot j of all lanes has
// similar trip counts (host-sorted), so the loop diverges little.
__device__ __forceinline__ void wt_scatter_medium(WtLane &L, const uint32_t (*steps)[32],
                                                  uint32_t wbase) {
    constexpr uint32_t len = kWt;
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < kWtSlots; ++j) {
        const uint32_t st = steps[j][lane];
        uint32_t o = L.o[j];
        for (; o + st < len; o += 2 * st) {
            clear_bit(wbase, o);
            clear_bit(wbase, o + st);
        }
        if (o < len) {
            clear_bit(wbase, o);
            o += st;
        }
        SQF2K_CHECK(!st || o >= len);  // every hit below len was cleared
        L.o[j] = st ? o - len : o;  // idle slots (step 0) keep o = ~0
    }
}

// Bucket hits of warp tile t (one list per tile: bucket tiles are warp
// tiles).  The lists live in HBM, written by bucket_kernel just before, so
// each load is a full memory round trip: the loop prefetches -- the list
// bounds two tiles ahead, the lane's hit one tile ahead -- and a tile's
// sieve only consumes registers.
static_assert(kWtSubTiles == 1, "one bucket list per warp tile");
struct WtBucket {
    uint32_t base, count;  // list bounds of a tile
};
__device__ __forceinline__ WtBucket wt_bucket_bounds(const TileParams &P, uint32_t t) {
    WtBucket b{0u, 0u};
    if (t < P.n_btiles) {
        if (P.tile_start) {
            b.base = __ldg(&P.tile_start[t]);
            b.count = __ldg(&P.tile_start[t + 1]) - b.base;
        } else {
            b.base = t * (uint32_t)kBucketCap;
            b.count = min(__ldg(&P.tile_count[t]), (uint32_t)kBucketCap);
        }
    }
    return b;
}
// the lane's first hit of a list (0xffff: none)
__device__ __forceinline__ uint32_t wt_bucket_hit(const TileParams &P, WtBucket b) {
    const uint32_t lane = threadIdx.x & 31;
    return lane < b.count ? (uint32_t)__ldg(&P.hits[b.base + lane]) : 0xffffu;
}
// clear a tile's bucket hits: the prefetched one per lane, the rest (lists
// longer than a warp: exact-mode lists only) loaded here
__device__ __forceinline__ void wt_scatter_bucket(uint32_t wbase, const TileParams &P, WtBucket b,
                                                  uint32_t hit) {
    SQF2K_CHECK(hit == 0xffffu || hit < (uint32_t)kBucketTile);
    SQF2K_CHECK(b.count <= 32 || P.tile_start);
    if (hit != 0xffffu) clear_bit(wbase, hit);
    for (uint32_t i = b.base + 32 + (threadIdx.x & 31); i < b.base + b.count; i += 32)
        clear_bit(wbase, __ldg(&P.hits[i]));
}

// Start an edge tile (n < 1 region or the domain end): masked per-lane
// stores, then one plain arrival on the buffer's mbarrier.
__device__ __forceinline__ void wt_start_edge(WarpRing &M, const TileParams &P, uint32_t t, uint32_t pbase) {
    const uint32_t lane = threadIdx.x & 31, at = wt_base(t);
    const uint64_t tb = (uint64_t)t * kWt;
#pragma unroll
    for (int c = 0; c < kWtWords / 128; ++c) {
        const uint32_t w = 4 * (lane + 32 * c);
        uint32_t v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[i] = __ldg(P.pattern + pbase + w + i);  // padded table: no wrap
            const uint64_t u0 = tb + 32ull * (w + i);
            if (u0 < P.z) v[i] = (u0 + 32 <= P.z) ? 0u : (v[i] & (~0u << (uint32_t)(P.z - u0)));
            if (u0 + 32 > P.U) v[i] = (u0 >= P.U) ? 0u : (v[i] & ((1u << (uint32_t)(P.U - u0)) - 1u));
        }
        *reinterpret_cast<uint4 *>(&M.ring[at + w]) = make_uint4(v[0], v[1], v[2], v[3]);
    }
    __syncwarp();
    if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&M.bar[t % kWtRing]))
                     : "memory");
}

// Start tile t in its buffer: one TMA bulk copy of the pattern words (lane 0)
// or, for an edge tile, masked per-lane stores; either way one phase of the
// buffer's mbarrier.  pbase: (t * kWtWords) mod kPatWords.
__device__ __forceinline__ void wt_start(WarpRing &M, uint32_t ring_addr, const TileParams &P,
                                         uint32_t t, uint32_t pbase, bool edge) {
    const uint32_t lane = threadIdx.x & 31, at = wt_base(t);
    const uint32_t bar = smem_addr(&M.bar[t % kWtRing]);
#ifdef SQF2K_CHECKS
    __syncwarp();  // (the checks read tags of the other buffers)
    if (lane == 0) M.tag[t % kWtRing] = t;
    __syncwarp();
#endif
    if (!edge) {
        if (lane == 0) {
            const uint32_t r = pbase & 3u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                         "r"((uint32_t)kWtWords * 4)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    ring_addr + 4 * at),
                "l"(P.pattern + r * kPatStride + (pbase - r)), "r"((uint32_t)kWtWords * 4), "r"(bar)
                : "memory");
        }
        return;
    }
    wt_start_edge(M, P, t, pbase);
}

__device__ __forceinline__ void wt_wait(WarpRing &M, uint32_t b, uint32_t &par) {
    const uint32_t bar = smem_addr(&M.bar[b]);
    const uint32_t parity = (par >> b) & 1u;
    uint32_t done = 0;
    for (;;) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) break;
    }
    par ^= 1u << b;
}
__device__ __forceinline__ void wt_check_tile(WarpRing &M, uint32_t t, uint32_t tp) {
#ifdef SQF2K_CHECKS
    SQF2K_CHECK(M.tag[t % kWtRing] == t);                      // tile t in its buffer
    if (t > tp) SQF2K_CHECK(M.tag[(t - 1) % kWtRing] == t - 1);  // its halo still intact
#endif
}

// Passes k = 6..k_eff for one word with slots left after the main passes
// (divergent, ~0.02% of words): n - 2^k is 2^(k-6) words back in the ring.
__device__ __forceinline__ void wt_residue(const uint32_t *ring, const TileParams &P, uint32_t i,
                                        uint64_t u0, uint32_t pend) {
    for (uint32_t k = kMainMax + 1; k <= P.k_eff && pend; ++k) {
        const uint32_t sl = ring[wt_back(i, 1u << (k - 6))];
        const uint32_t nw = pend & sl;
        if (nw) {
            atomicAdd(&P.hist[k], (unsigned long long)__popc(nw));
            atomicMin(&P.min_n[k], (unsigned long long)(P.base_n + 2 * (int64_t)(u0 + __ffs(nw) - 1)));
        }
        pend &= ~sl;
    }
    if (pend) {
        if (P.k_max > P.k_eff) spill_word(pend, u0, P.base_n, P.esc, P.esc_count, P.esc_cap);
        else spill_word(pend, u0, P.base_n, P.fail, P.fail_count, P.fail_cap);
    }
}

// The words of a 4-word chunk (ring word i0, domain slot u0) with slots left
// after the main passes: deeper passes (KMAIN = 5) or the escalation /
// failure lists.  Returns the leftover count (subtracted from hist[KMAIN]).
template <int KMAIN>
__device__ __forceinline__ uint32_t wt_leftovers(const uint32_t *ring, const TileParams &P, uint32_t i0,
                                              uint64_t u0, uint32_t l0, uint32_t l1, uint32_t l2,
                                              uint32_t l3) {
    const uint32_t left[4] = {l0, l1, l2, l3};
    uint32_t n = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (!left[i]) continue;
        n += __popc(left[i]);
        const uint64_t u = u0 + 32ull * i;
        if (KMAIN == kMainMax) wt_residue(ring, P, i0 + i, u, left[i]);
        else if (P.k_max > P.k_eff) spill_word(left[i], u, P.base_n, P.esc, P.esc_count, P.esc_cap);
        else spill_word(left[i], u, P.base_n, P.fail, P.fail_count, P.fail_cap);
    }
    return n;
}

// Scan of warp tile t (buffer at ring word hb): lane l takes the 4-word
// chunks 128 c + 4 l, c = 0..3 (one conflict-free LDS.128 per chunk across
// the warp); a chunk's left neighbour word comes from lane l - 1 by a
// shuffle (lane 0: lane 31 of the previous chunk, or the previous tile's
// last word).  A lane's words still come in increasing order, so its first
// hit per k (TRACK) is its least one.
template <bool EDGE, bool TRACK, int KMAIN>
__device__ __forceinline__ void wt_scan(const uint32_t *ring, const TileParams &P, uint32_t hb,
                                        uint64_t tb, uint32_t (&c)[6], uint32_t (&f)[6],
                                        uint32_t &scanned, uint32_t &left5) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t carry = ring[wt_back(hb, 1)];  // word before the chunk row (lane 0's neighbour)
#pragma unroll
    for (int ch = 0; ch < kWtWords / 128; ++ch) {
        const uint32_t w0 = 128 * ch + 4 * lane;
        const uint4 cw = *reinterpret_cast<const uint4 *>(&ring[hb + w0]);
        const uint32_t up = __shfl_up_sync(0xffffffffu, cw.w, 1);
        const uint32_t cur[4] = {cw.x, cw.y, cw.z, cw.w};
        const uint32_t prv[4] = {lane ? up : carry, cw.x, cw.y, cw.z};
        carry = __shfl_sync(0xffffffffu, cw.w, 31);
        uint32_t left[4], any = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t pend = ~0u;
            if (EDGE) {
                pend = edge_mask(P, tb + 32ull * (w0 + i));
                scanned += __popc(pend);
            }
            left[i] = scan_word<TRACK, KMAIN>(pend, prv[i], cur[i], c, f, w0 + i);
            any |= left[i];
        }
        if (!EDGE) scanned += 128;
        if (any)  // rare: finish these words in place (out of line: keeps the loop small)
            left5 += wt_leftovers<KMAIN>(ring, P, hb + w0, tb + 32ull * w0, left[0], left[1], left[2],
                                         left[3]);
    }
#pragma unroll
    for (int k = 1; k < KMAIN; ++k) c[k] += 32 * kWtLaneWords;  // pending = 32 - covered per word
}

template <int KMAIN>
__device__ __forceinline__ void wt_flush_counts(const TileParams &P, const uint32_t (&c)[6],
                                                uint32_t scanned, uint32_t left5) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= KMAIN; ++k) {  // met at k: pending after k - 1, not after k
        const unsigned long long s = warp_sum_u64(c[k - 1] - c[k]);
        if (lane == 0 && s) atomicAdd(&P.hist[k], s);
    }
    if (KMAIN >= 2) {  // slots left after pass KMAIN were counted in hist[KMAIN] (mod 2^64)
        const unsigned long long l = warp_sum_u64(left5);
        if (lane == 0 && l) atomicAdd(&P.hist[KMAIN], 0ull - l);
    }
    const unsigned long long sc = warp_sum_u64(scanned);
    if (lane == 0 && sc) atomicAdd(P.scanned, sc);
}

// The rare scan variant (edge masks and per-k least slot tracking: the first
// tiles of a chunk and the domain edges).  One instantiation, inlined in its
// own branch of the tile loop, so the steady-state path stays compact; its
// counts go straight to the accumulators (the hot counters stay in the
// caller's registers).  Returns the k still untracked.
template <int KMAIN>
__device__ __forceinline__ uint32_t wt_scan_slow(WarpRing &M, const TileParams &P, uint32_t hb,
                                                 uint64_t tb, uint32_t need) {
    uint32_t f[6] = {~0u, ~0u, ~0u, ~0u, ~0u, ~0u};
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};
    uint32_t scanned = 0, left5 = 0;
    wt_scan<true, true, KMAIN>(M.ring, P, hb, tb, c, f, scanned, left5);
    wt_flush_counts<KMAIN>(P, c, scanned, left5);
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 1; k <= KMAIN; ++k) {
        if (!((need >> k) & 1u)) continue;
        const uint32_t m = __reduce_min_sync(0xffffffffu, f[k]);
        if (m != ~0u) {
            need &= ~(1u << k);
            if (lane == 0) M.first[k] = tb + m;
        }
    }
    return need;
}

template <int KMAIN>
__global__ void __launch_bounds__(kWtThreads, kWtCtasPerSm) wtile_kernel(const __grid_constant__ TileParams P) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    WtSmem &S = *reinterpret_cast<WtSmem *>(smem_raw);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpRing &M = S.w[warp];
    const uint32_t ring_addr = smem_addr(M.ring);
    const uint32_t GW = gridDim.x * kWtWarps, gw = blockIdx.x * kWtWarps + warp;
    const uint32_t NT = P.n_tiles;

    // static share (~3/4) then dynamic chunks, per warp
    const bool dynamic = NT >= (uint64_t)kWtDynMin * GW;
    const uint32_t S1 = (uint32_t)((uint64_t)NT * kStaticEighths / (8ull * GW));
    const uint32_t dyn0 = dynamic ? S1 * GW : NT;
    const uint32_t csz = max((NT - dyn0) / (8 * GW), (uint32_t)kMinChunk);
    uint32_t t0 = dynamic ? S1 * gw : (uint32_t)((uint64_t)NT * gw / GW);
    uint32_t t1 = dynamic ? t0 + S1 : (uint32_t)((uint64_t)NT * (gw + 1) / GW);

    // tiles [ti0, ti1) need no masks (as tile_kernel)
    uint64_t lo_edge = P.scan_lo;
    if (P.z > lo_edge) lo_edge = P.z;
    if (P.one_u != ~0ull && P.one_u + 1 > lo_edge) lo_edge = P.one_u + 1;
    const uint32_t ti0 = (uint32_t)((lo_edge + kWt - 1) / kWt);
    const uint32_t ti1 = (uint32_t)(P.U / kWt);

    for (uint32_t i = threadIdx.x; i < kWtSlots * 32; i += kWtThreads)
        S.step[i / 32][i % 32] = __ldg(&P.wtasks[i]).y;
    __syncthreads();
    if (lane < kWtRing) {
#ifdef SQF2K_CHECKS
        M.tag[lane] = ~0u;
#endif
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&M.bar[lane])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t par = 0;  // bit b: parity of buffer b's next start
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};
    uint32_t scanned = 0, left5 = 0;
    bool waited = false;

    for (;;) {
        if (t0 >= t1) {  // next dynamic chunk
            uint32_t k = 0;
            if (lane == 0) k = atomicAdd(&P.sched[0], 1u);
            k = __shfl_sync(0xffffffffu, k, 0);
            const uint64_t lo = (uint64_t)dyn0 + (uint64_t)k * csz;
            t0 = (uint32_t)min(lo, (uint64_t)NT);
            t1 = (uint32_t)min(lo + csz, (uint64_t)NT);
            if (t0 >= t1) break;
        }
        // tiles tp .. t1 - 1 are sieved; tp = t0 - 1 (the halo below the
        // chunk, not scanned) unless the chunk starts the domain
        const uint32_t tp = t0 > 0 ? t0 - 1 : t0;
        WtLane L;
        wt_init_medium(L, P, (uint64_t)tp * kWt);
        uint32_t pnext = (uint32_t)(((uint64_t)tp * kWtWords) % kPatWords);  // pattern index
        auto adv = [](uint32_t x) {
            x += kWtWords;
            return x >= kPatWords ? x - kPatWords : x;
        };
        auto edge_t = [&](uint32_t t) { return t < ti0 || t >= ti1; };
        for (uint32_t i = 0; i < 2 && tp + i < t1; ++i) {  // starts of tp, tp + 1
            wt_start(M, ring_addr, P, tp + i, pnext, edge_t(tp + i));
            pnext = adv(pnext);
        }
        if (!waited) {  // bucket lists come from the grid launched before this one
            grid_dependency_wait();
            waited = true;
        }
        // bucket lists: bounds two tiles ahead, the lane's hit one tile ahead
        WtBucket bk0 = wt_bucket_bounds(P, tp), bk1 = wt_bucket_bounds(P, tp + 1);
        uint32_t hit0 = wt_bucket_hit(P, bk0);
        // least slot per k <= 5 in this chunk: tracked while unknown
        uint32_t need = ((2u << KMAIN) - 2u) & 0x3eu;
        if (lane <= kMainMax) M.first[lane] = ~0ull;
        for (uint32_t t = tp; t < t1; ++t) {
            const uint32_t hb = wt_base(t);
            const uint64_t tb = (uint64_t)t * kWt;
            const WtBucket bk2 = wt_bucket_bounds(P, t + 2);  // in flight during this tile
            const uint32_t hit1 = wt_bucket_hit(P, bk1);
            wt_wait(M, t % kWtRing, par);
            wt_check_tile(M, t, tp);
            wt_scatter_medium(L, S.step, ring_addr + 4 * hb);
            wt_scatter_bucket(ring_addr + 4 * hb, P, bk0, hit0);
            bk0 = bk1;
            bk1 = bk2;
            hit0 = hit1;
            __syncwarp();
            wt_check_tile(M, t, tp);
            if (t < t0) {
                // the halo tile: sieved only
            } else if (need || edge_t(t)) {  // first tiles of a chunk, domain edges: out of line
                need = wt_scan_slow<KMAIN>(M, P, hb, tb, need);
            } else {
                uint32_t f[6];
                wt_scan<false, false, KMAIN>(M.ring, P, hb, tb, c, f, scanned, left5);
            }
            wt_check_tile(M, t, tp);  // nothing overwrote t or t - 1 during the scan
            __syncwarp();  // every lane is done with tile t - 1's buffer
            if (t + 2 < t1) {
                wt_start(M, ring_addr, P, t + 2, pnext, edge_t(t + 2));
                pnext = adv(pnext);
            }
        }
        __syncwarp();
        if (lane >= 1 && lane <= KMAIN && M.first[lane] != ~0ull)
            atomicMin(&P.min_n[lane], (unsigned long long)(P.base_n + 2 * (int64_t)M.first[lane]));
        t0 = t1;
    }

    wt_flush_counts<KMAIN>(P, c, scanned, left5);  // per warp: 64-bit sums, one atomic per k

    // the last CTA resets the scheduler and (single-batch calls) finishes the call
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) S.last = atomicAdd(&P.sched[1], 1u) == gridDim.x - 1;
    __syncthreads();
    if (S.last) {
        __threadfence();
        if (P.acc) {
            if (P.k_max > P.k_eff) {
                const uint64_t count = min((unsigned long long)P.esc_cap, __ldcg(P.esc_count));
                escalate_warps(P.esc, count, P.k_eff + 1, P.k_max, P.primes, __ldcg(&P.info->count),
                               P.hist, P.min_n, P.fail, P.fail_count, P.fail_cap, warp, kWtWarps);
                __threadfence();
                __syncthreads();
            }
            const unsigned long long *src = reinterpret_cast<const unsigned long long *>(P.acc);
            unsigned long long *dst = static_cast<unsigned long long *>(P.acc_host);
            for (uint32_t i = threadIdx.x; i < sizeof(Acc) / 8; i += kWtThreads) dst[i] = __ldcg(src + i);
        }
        if (threadIdx.x == 0) {
            P.sched[0] = 0;
            P.sched[1] = 0;
        }
    }
}

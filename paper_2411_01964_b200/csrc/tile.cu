// tile.cu -- one batch of the tile pipeline: the p = 3, 5, 7 pattern table,
// the bucketed large-prime hit lists and the tile kernel (fused sieve +
// min-k scan, or sieve export).  No host synchronisation inside a batch.
#include <algorithm>
#include <cstring>
#include <map>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "tile.cuh"

namespace sqf2k {

namespace {

// -------------------------------------------------------------------------
// p = 3, 5, 7: word g of the domain (slots 32g..32g+31) with every slot u
// such that 9, 25 or 49 divides n(u) cleared.  Period 11025 words.
// First hit at or after 32g: y = (r - 32g) mod q; the word's hits are the
// bits y, y+q, ... < 32, i.e. (bits 0, q, 2q, ...) << y.
__global__ void pattern_kernel(int64_t base_n, uint32_t present, uint32_t *__restrict__ table) {
    const uint32_t q[3] = {9, 25, 49};
    const uint32_t pat[3] = {0x08040201u, 0x02000001u, 0x1u};
    uint32_t r[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) r[i] = (uint32_t)slot_residue(base_n, q[i]);
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < kPatWords;
         g += gridDim.x * blockDim.x) {
        uint32_t clr = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (!((present >> i) & 1u)) continue;
            const uint32_t y = (r[i] + q[i] - (32u * g) % q[i]) % q[i];
            if (y < 32) clr |= pat[i] << y;
        }
        table[g] = ~clr;
    }
}

// -------------------------------------------------------------------------
// Bucket pass: every hit u of a bucket prime (p >= kPMed, p^2 <= n_max) in the
// batch domain [0, U), as a 16-bit offset in the list of tile u >> 16.
// Work units are (prime, sub-range) pairs of <= 5 hits (see kClasses).
// FILL places hit i of tile t at offsets[t] + (--counts[t]): the count pass
// leaves counts[t] = size, the fill pass brings it back to 0.
template <bool FILL>
__global__ void __launch_bounds__(256) bucket_kernel(
    const uint32_t *__restrict__ primes, const PrimeInfo *__restrict__ info, int64_t base_n,
    uint64_t U, uint32_t *__restrict__ counts, const uint32_t *__restrict__ offsets,
    uint16_t *__restrict__ hits) {
    const uint32_t i_hi = info->i_hi;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (int j = 0; j < kClasses; ++j) {
        const uint32_t p_lo = max(info->cls[j], info->i_lo);
        const uint32_t p_hi = min(info->cls[j + 1], i_hi);
        if (p_lo >= p_hi) continue;
        const int sh = min(22 + 2 * j, 62);
        const uint64_t n_sub = (U + (1ull << sh) - 1) >> sh;
        const uint64_t n_work = (uint64_t)(p_hi - p_lo) * n_sub;
        for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < n_work; w += stride) {
            const uint64_t p = primes[p_lo + w / n_sub];
            const uint64_t lo = (w % n_sub) << sh;
            const uint64_t hi = lo + (1ull << sh) < U ? lo + (1ull << sh) : U;
            const uint64_t q = p * p;
            const uint64_t r = slot_residue(base_n, q);
            const uint64_t lm = lo % q;
            for (uint64_t u = lo + (r >= lm ? r - lm : r + q - lm); u < hi; u += q) {
                const uint32_t t = (uint32_t)(u >> 16);
                if (FILL) {
                    const uint32_t pos = offsets[t] + atomicSub(&counts[t], 1u) - 1u;
                    hits[pos] = (uint16_t)(u & 0xffff);
                } else {
                    atomicAdd(&counts[t], 1u);
                }
            }
        }
    }
}

// -------------------------------------------------------------------------
struct TileSmem {
    uint8_t bytes[kTile];                       // 64 KB, 16-byte aligned
    uint32_t bits[kHaloWordsMax + kTileWords];  // halo + tile (12 KB)
    uint32_t med_q[kMaxMed], med_tq[kMaxMed], off[kMaxMed];
    unsigned long long first[kDepthMax + 1];
    uint32_t cnt[kDepthMax + 1];                // counts of k >= 5 (rare)
    uint32_t need;
};

__device__ __forceinline__ void init_bytes(uint8_t *bytes, uint32_t len) {
    const uint4 one = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    for (uint32_t i = threadIdx.x; i < len / 16; i += kThreads)
        reinterpret_cast<uint4 *>(bytes)[i] = one;
}

// clear the medium-prime hits in [0, len) of the current base
__device__ __forceinline__ void scatter_medium(uint8_t *bytes, const uint32_t *off,
                                               const uint32_t *med_q, const TileParams &P,
                                               uint32_t len) {
    for (uint32_t it = threadIdx.x; it < P.n_items; it += kThreads) {
        const uint32_t mj = __ldg(&P.items[2 * it]), stride = __ldg(&P.items[2 * it + 1]);
        const uint32_t m = mj >> 16;
        uint32_t o = off[m] + (mj & 0xffffu) * med_q[m];
        for (; o + stride < len; o += 2 * stride) {
            bytes[byte_pos(o)] = 0;
            bytes[byte_pos(o + stride)] = 0;
        }
        if (o < len) bytes[byte_pos(o)] = 0;
    }
}

// clear the bucket hits of tile t with offsets in [skip, kTile), shifted by -skip
__device__ __forceinline__ void scatter_bucket(uint8_t *bytes, const TileParams &P, uint32_t t,
                                               uint32_t skip) {
    const uint32_t b = __ldg(&P.tile_start[t]), e = __ldg(&P.tile_start[t + 1]);
    for (uint32_t i = b + threadIdx.x; i < e; i += kThreads) {
        const uint32_t o = __ldg(&P.hits[i]);
        if (o >= skip) bytes[byte_pos(o - skip)] = 0;
    }
}

// move the medium offsets forward by `step[m]` (= len mod q) slots
__device__ __forceinline__ void advance_offsets(uint32_t *off, const uint32_t *med_q,
                                                const uint32_t *step, uint32_t n_med) {
    for (uint32_t m = threadIdx.x; m < n_med; m += kThreads) {
        const uint32_t o = off[m] - step[m];  // wraps when negative
        off[m] = min(o, o + med_q[m]);
    }
}

// Pack WORDS words of bytes (domain slot `base`) into out[].  pbase is
// (base / 32) mod kPatWords.  EDGE applies the n < 1 zero region and the end.
template <int WORDS, bool EDGE>
__device__ __forceinline__ void pack_words(const uint8_t *bytes, uint32_t *out, uint64_t base,
                                           uint32_t pbase, const TileParams &P) {
#pragma unroll
    for (int r = 0; r < (WORDS + kThreads - 1) / kThreads; ++r) {
        const uint32_t w = threadIdx.x + r * kThreads;
        if (WORDS % kThreads != 0 && w >= (uint32_t)WORDS) break;
        const uint8_t *blk = bytes + ((w >> 5) << 10) + ((w & 31) << 4);
        const uint4 a = *reinterpret_cast<const uint4 *>(blk);
        const uint4 b = *reinterpret_cast<const uint4 *>(blk + 512);
        // bytes are 0/1 and the shifted words never overlap: + is |, and
        // compiles to a chain of shift-adds
        uint32_t word = a.x + (a.y << 1) + (a.z << 2) + (a.w << 3) + (b.x << 4) + (b.y << 5) +
                        (b.z << 6) + (b.w << 7);
        uint32_t idx = pbase + w;  // pbase < kPatWords, w < kTileWords < kPatWords
        if (idx >= kPatWords) idx -= kPatWords;
        word &= __ldg(&P.pattern[idx]);
        if (EDGE) {
            const uint64_t u0 = base + 32ull * w;
            if (u0 < P.z) word = (u0 + 32 <= P.z) ? 0u : (word & (~0u << (uint32_t)(P.z - u0)));
            if (u0 + 32 > P.U) word = (u0 >= P.U) ? 0u : (word & ((1u << (uint32_t)(P.U - u0)) - 1u));
        }
        out[w] = word;
    }
}

// The pre-tile packs H = HW*32 slots (HW in {32, 64, ..., 1024}).
__device__ __forceinline__ void pack_halo(const uint8_t *bytes, uint32_t *out, uint32_t HW,
                                          uint64_t base, uint32_t pbase, const TileParams &P) {
    if (HW > 512) pack_words<kHaloWordsMax, true>(bytes, out, base, pbase, P);
    else if (HW > 256) pack_words<512, true>(bytes, out, base, pbase, P);
    else if (HW > 128) pack_words<256, true>(bytes, out, base, pbase, P);
    else if (HW > 64) pack_words<128, true>(bytes, out, base, pbase, P);
    else pack_words<64, true>(bytes, out, base, pbase, P);
}

__device__ __forceinline__ void append(unsigned long long *list, unsigned long long *count,
                                       uint64_t cap, uint64_t n) {
    const unsigned long long i = atomicAdd(count, 1ull);
    if (i < cap) list[i] = n;
}

// passes k >= 5 for one word (divergent, rare), then escalation / failure
__device__ __forceinline__ void scan_residue(TileSmem &S, const TileParams &P, uint32_t HW,
                                          uint32_t w, uint64_t u0, uint32_t pend, uint32_t need) {
    const uint32_t cur = S.bits[HW + w], prv = S.bits[HW + w - 1];
    for (uint32_t k = 5; k <= P.k_eff && pend; ++k) {
        uint32_t sl;
        if (k == 5) sl = __funnelshift_l(prv, cur, 16);
        else if (k == 6) sl = prv;
        else sl = S.bits[HW + w - (1u << (k - 6))];
        const uint32_t nw = pend & sl;
        if (nw) {
            atomicAdd(&S.cnt[k], (uint32_t)__popc(nw));
            if ((need >> k) & 1u) atomicMin(&S.first[k], (unsigned long long)(u0 + __ffs(nw) - 1));
        }
        pend &= ~sl;
    }
    if (pend) {
        const bool esc = P.k_max > P.k_eff;
        for (uint32_t x = pend; x; x &= x - 1) {
            const uint64_t n = (uint64_t)(P.base_n + 2 * (int64_t)(u0 + __ffs(x) - 1));
            if (esc) append(P.esc, P.esc_count, P.esc_cap, n);
            else append(P.fail, P.fail_count, P.fail_cap, n);
        }
    }
}

// One pass of the main scan on one word.
template <bool TRACK>
__device__ __forceinline__ void pass(uint32_t &pend, uint32_t sl, uint32_t &cnt, int k,
                                     uint32_t need, uint64_t u0, TileSmem &S) {
    const uint32_t nw = pend & sl;
    cnt += __popc(nw);
    if (TRACK && nw && ((need >> k) & 1u))
        atomicMin(&S.first[k], (unsigned long long)(u0 + __ffs(nw) - 1));
    pend &= ~sl;
}

// Exponent passes over the tile's words.  EDGE masks the scan range, TRACK
// records per-k least slots while this CTA still lacks them, KMAIN is the
// number of unconditional passes (4, or k_eff when smaller).
template <bool EDGE, bool TRACK, int KMAIN>
__device__ __forceinline__ void scan_tile(TileSmem &S, const TileParams &P, uint32_t HW,
                                          uint64_t tb, uint32_t need, uint32_t (&c)[5]) {
#pragma unroll
    for (int r = 0; r < kWordsPerThread; ++r) {
        const uint32_t w = threadIdx.x + r * kThreads;
        const uint64_t u0 = tb + 32ull * w;
        uint32_t pend = ~0u;
        if (EDGE) {
            if (u0 + 32 <= P.scan_lo || u0 >= P.U) {
                pend = 0u;
            } else {
                if (u0 < P.scan_lo) pend &= ~0u << (uint32_t)(P.scan_lo - u0);
                if (u0 + 32 > P.U) pend &= (1u << (uint32_t)(P.U - u0)) - 1u;
                if (P.one_u >= u0 && P.one_u < u0 + 32) pend &= ~(1u << (uint32_t)(P.one_u - u0));
            }
        }
        const uint32_t cur = S.bits[HW + w], prv = S.bits[HW + w - 1];
        pass<TRACK>(pend, __funnelshift_l(prv, cur, 1), c[1], 1, need, u0, S);
        if (KMAIN >= 2) pass<TRACK>(pend, __funnelshift_l(prv, cur, 2), c[2], 2, need, u0, S);
        if (KMAIN >= 3) pass<TRACK>(pend, __funnelshift_l(prv, cur, 4), c[3], 3, need, u0, S);
        if (KMAIN >= 4) pass<TRACK>(pend, __funnelshift_l(prv, cur, 8), c[4], 4, need, u0, S);
        if (pend) {
            if (KMAIN == 4) {
                scan_residue(S, P, HW, w, u0, pend, need);
            } else {  // k_eff = KMAIN < 4: leftovers are final
                const bool esc = P.k_max > P.k_eff;
                for (uint32_t x = pend; x; x &= x - 1) {
                    const uint64_t n = (uint64_t)(P.base_n + 2 * (int64_t)(u0 + __ffs(x) - 1));
                    if (esc) append(P.esc, P.esc_count, P.esc_cap, n);
                    else append(P.fail, P.fail_count, P.fail_cap, n);
                }
            }
        }
    }
}

template <int KMAIN>
__device__ __forceinline__ void scan_dispatch(TileSmem &S, const TileParams &P, uint32_t HW,
                                              uint64_t tb, bool edge, uint32_t need,
                                              uint32_t (&c)[5]) {
    const bool track = (need & 0x1eu) != 0;
    if (edge) {
        if (track) scan_tile<true, true, KMAIN>(S, P, HW, tb, need, c);
        else scan_tile<true, false, KMAIN>(S, P, HW, tb, need, c);
    } else {
        if (track) scan_tile<false, true, KMAIN>(S, P, HW, tb, need, c);
        else scan_tile<false, false, KMAIN>(S, P, HW, tb, need, c);
    }
}

template <bool FUSED>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) tile_kernel(const TileParams P) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    TileSmem &S = *reinterpret_cast<TileSmem *>(smem_raw);
    const uint32_t G = gridDim.x;
    const uint32_t t0 = (uint32_t)((uint64_t)P.n_tiles * blockIdx.x / G);
    const uint32_t t1 = (uint32_t)((uint64_t)P.n_tiles * (blockIdx.x + 1) / G);
    if (t0 >= t1) return;
    const uint32_t H = FUSED ? P.H : 0u;
    const uint32_t HW = H / 32;
    const bool pre = FUSED && t0 > 0;

    // medium primes: q, kTile mod q and the first hit at the chunk base b0
    const uint64_t b0 = pre ? (uint64_t)t0 * kTile - H : (uint64_t)t0 * kTile;
    for (uint32_t m = threadIdx.x; m < P.n_med; m += kThreads) {
        const uint32_t q = __ldg(&P.med[2 * m]);
        const uint32_t r = (uint32_t)slot_residue(P.base_n, q);
        const uint32_t bm = (uint32_t)(b0 % q);
        S.med_q[m] = q;
        S.med_tq[m] = __ldg(&P.med[2 * m + 1]);
        S.off[m] = r >= bm ? r - bm : r + q - bm;
    }
    if (threadIdx.x <= kDepthMax) {
        S.first[threadIdx.x] = ~0ull;
        S.cnt[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) S.need = ~0u;
    uint32_t pbase = (uint32_t)((b0 / 32) % kPatWords);
    init_bytes(S.bytes, pre ? H : (uint32_t)kTile);
    __syncthreads();

    if (FUSED) {
        if (pre) {
            // pre-tile: sieve the H slots below the chunk into the halo words
            scatter_medium(S.bytes, S.off, S.med_q, P, H);
            scatter_bucket(S.bytes, P, t0 - 1, kTile - H);
            __syncthreads();
            pack_halo(S.bytes, S.bits, HW, b0, pbase, P);
            for (uint32_t m = threadIdx.x; m < P.n_med; m += kThreads) {
                const uint32_t o = S.off[m] - H % S.med_q[m];
                S.off[m] = min(o, o + S.med_q[m]);
            }
            pbase += HW;
            if (pbase >= kPatWords) pbase -= kPatWords;
            __syncthreads();
            init_bytes(S.bytes, kTile);
        } else {
            for (uint32_t i = threadIdx.x; i < HW; i += kThreads) S.bits[i] = 0u;
        }
        __syncthreads();
    }

    uint32_t c[5] = {0, 0, 0, 0, 0};
    const uint32_t kmain = P.k_eff < 4 ? P.k_eff : 4;
    for (uint32_t t = t0; t < t1; ++t) {
        const uint64_t tb = (uint64_t)t * kTile;
        scatter_medium(S.bytes, S.off, S.med_q, P, kTile);
        scatter_bucket(S.bytes, P, t, 0);
        __syncthreads();
        const bool edge_pack = tb < P.z || tb + kTile > P.U;
        if (edge_pack) pack_words<kTileWords, true>(S.bytes, S.bits + HW, tb, pbase, P);
        else pack_words<kTileWords, false>(S.bytes, S.bits + HW, tb, pbase, P);
        advance_offsets(S.off, S.med_q, S.med_tq, P.n_med);
        pbase += kTileWords;
        if (pbase >= kPatWords) pbase -= kPatWords;
        __syncthreads();
        if (!FUSED) {
            for (uint32_t w = threadIdx.x; w < kTileWords; w += kThreads)
                P.bits_out[(uint64_t)t * kTileWords + w] = S.bits[w];
            init_bytes(S.bytes, kTile);
            __syncthreads();
            continue;
        }
        // ---- exponent passes (search.py:368-381) over the packed tile ----
        const uint32_t need = S.need;
        const bool edge = tb < P.scan_lo || tb + kTile > P.U ||
                          (P.one_u >= tb && P.one_u < tb + kTile);
        switch (kmain) {
            case 1: scan_dispatch<1>(S, P, HW, tb, edge, need, c); break;
            case 2: scan_dispatch<2>(S, P, HW, tb, edge, need, c); break;
            case 3: scan_dispatch<3>(S, P, HW, tb, edge, need, c); break;
            default: scan_dispatch<4>(S, P, HW, tb, edge, need, c); break;
        }
        if (t + 1 < t1) init_bytes(S.bytes, kTile);  // the next tile's bytes
        __syncthreads();
        if (threadIdx.x >= 1 && threadIdx.x <= kDepthMax) {
            const unsigned long long f = S.first[threadIdx.x];
            if (f != ~0ull) {
                atomicMin(&P.min_n[threadIdx.x], (unsigned long long)(P.base_n + 2 * (int64_t)f));
                atomicAnd(&S.need, ~(1u << threadIdx.x));
                S.first[threadIdx.x] = ~0ull;
            }
        }
        // roll the halo: the last H slots of this tile precede the next one
        for (uint32_t i = threadIdx.x; i < HW; i += kThreads) S.bits[i] = S.bits[kTileWords + i];
        // (the next tile's scatter touches only bytes; its pack follows a barrier)
    }

    if (FUSED) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int k = 1; k <= 4; ++k) {
            const uint32_t s = __reduce_add_sync(0xffffffffu, c[k]);
            if (lane == 0 && s) atomicAdd(&P.hist[k], (unsigned long long)s);
        }
        __syncthreads();
        if (threadIdx.x >= 5 && threadIdx.x <= kDepthMax && S.cnt[threadIdx.x])
            atomicAdd(&P.hist[threadIdx.x], (unsigned long long)S.cnt[threadIdx.x]);
    }
}

// -------------------------------------------------------------------------
// Medium-prime tables (q, kTile mod q) and balanced items, built on the host
// from the table's primes in [11, kPMed) and cached on the device per set.
struct MedTables {
    std::vector<uint32_t> med, items;
    uint32_t n_med = 0, n_items = 0;
};

MedTables build_med(const std::vector<uint32_t> &med_primes) {
    MedTables t;
    for (uint32_t p : med_primes) {
        if (t.n_med >= (uint32_t)kMaxMed) break;
        const uint32_t q = p * p;
        t.med.push_back(q);
        t.med.push_back((uint32_t)kTile % q);
        uint32_t m = (uint32_t)kTile / (q * (uint32_t)kItemHits);
        m = std::max<uint32_t>(1, std::min<uint32_t>(m, 64));
        for (uint32_t j = 0; j < m && t.n_items < (uint32_t)kMaxItems; ++j, ++t.n_items) {
            t.items.push_back((t.n_med << 16) | j);
            t.items.push_back(m * q);
        }
        ++t.n_med;
    }
    return t;
}

struct MedCache {
    std::vector<uint32_t> key;
    uint32_t n_med = 0, n_items = 0;
    DevBuf buf;
};

MedCache g_med;  // the library serialises calls

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


void run_tile_batch(const BatchArgs &a) {
    Context &c = ctx();
    const uint32_t n_tiles = (uint32_t)ceil_div(a.U, kTile);

    // medium tables: cached per distinct prime set
    if (g_med.key != *a.med_primes || !g_med.buf.ptr) {
        MedTables t = build_med(*a.med_primes);
        g_med.key = *a.med_primes;
        g_med.n_med = t.n_med;
        g_med.n_items = t.n_items;
        g_med.buf.reserve((2 * kMaxMed + 2 * kMaxItems) * 4);
        std::vector<uint32_t> host(2 * kMaxMed + 2 * kMaxItems, 0);
        std::copy(t.med.begin(), t.med.end(), host.begin());
        std::copy(t.items.begin(), t.items.end(), host.begin() + 2 * kMaxMed);
        SQF2K_CUDA(cudaMemcpy(g_med.buf.ptr, host.data(), host.size() * 4, cudaMemcpyHostToDevice));
    }

    // p = 3, 5, 7 pattern of this domain
    c.pattern.reserve(kPatWords * 4);
    launch("pattern", pattern_kernel, dim3(ceil_div(kPatWords, 256)), dim3(256), 0, a.base_n,
           a.pattern_present, c.pattern.as<uint32_t>());

    // bucket lists: count, scan, fill (sizes bounded on the host: no sync)
    c.tile_counts.reserve((n_tiles + 1) * 4);
    c.tile_offsets.reserve((n_tiles + 1) * 4);
    uint32_t *counts = c.tile_counts.as<uint32_t>();
    uint32_t *offsets = c.tile_offsets.as<uint32_t>();
    SQF2K_CUDA(cudaMemsetAsync(counts, 0, (n_tiles + 1) * 4, c.stream));
    const unsigned bgrid = (unsigned)c.sm_count * 8;
    c.hits.reserve(bucket_hits_bound(a.U, a.n_primes_bound) * 2 + 64);
    launch("bucket_count", bucket_kernel<false>, dim3(bgrid), dim3(256), 0, a.primes, a.info,
           a.base_n, a.U, counts, (const uint32_t *)offsets, (uint16_t *)nullptr);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, offsets, (int)n_tiles + 1, c.stream);
    c.scan_tmp.reserve(std::max<size_t>(tmp_bytes, 64));
    SQF2K_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.ptr, tmp_bytes, counts, offsets,
                                             (int)n_tiles + 1, c.stream));
    launch("bucket_fill", bucket_kernel<true>, dim3(bgrid), dim3(256), 0, a.primes, a.info,
           a.base_n, a.U, counts, (const uint32_t *)offsets, c.hits.as<uint16_t>());

    TileParams P;
    std::memset(&P, 0, sizeof P);
    P.base_n = a.base_n;
    P.U = a.U;
    P.scan_lo = a.scan_lo;
    P.z = a.z;
    P.one_u = a.one_u;
    P.H = a.H;
    P.n_tiles = n_tiles;
    P.k_eff = a.k_eff;
    P.k_max = a.k_max;
    P.n_med = g_med.n_med;
    P.n_items = g_med.n_items;
    P.pattern = c.pattern.as<uint32_t>();
    P.med = g_med.buf.as<uint32_t>();
    P.items = g_med.buf.as<uint32_t>() + 2 * kMaxMed;
    P.tile_start = offsets;
    P.hits = c.hits.as<uint16_t>();
    P.hist = a.hist;
    P.min_n = a.min_n;
    P.esc = a.esc;
    P.esc_count = a.esc_count;
    P.esc_cap = a.esc_cap;
    P.fail = a.fail;
    P.fail_count = a.fail_count;
    P.fail_cap = a.fail_cap;
    P.bits_out = a.bits_out;

    const size_t smem = tile_smem_bytes();
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>(n_tiles, (uint64_t)c.sm_count * kCtasPerSm));
    static bool attr[2] = {false, false};
    if (a.fused) {
        if (!attr[1]) {
            SQF2K_CUDA(cudaFuncSetAttribute(tile_kernel<true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr[1] = true;
        }
        launch("tile_fused", tile_kernel<true>, dim3(grid), dim3(kThreads), smem, P);
    } else {
        if (!attr[0]) {
            SQF2K_CUDA(cudaFuncSetAttribute(tile_kernel<false>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr[0] = true;
        }
        launch("tile_export", tile_kernel<false>, dim3(grid), dim3(kThreads), smem, P);
    }
}

}  // namespace sqf2k

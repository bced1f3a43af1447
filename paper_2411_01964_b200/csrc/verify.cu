// verify.cu -- the GPU hot path of run_verify: per-batch setup, bucketed
// large-prime hit lists, the fused tile kernel (sieve + min-k scan in shared
// memory), the exact escalation kernel and the failure recheck; plus the
// segment-export form of the same tile kernel behind sieve_segment.
//
// Reference semantics restated (per odd n, search.py:368-397, runner.py:93-102):
//   k(n) = min{ k in [1, k_max] : n - 2^k >= 1 and n - 2^k squarefree },
//   n = 1 excluded, unresolved n are failures; hist[k] counts, min_n[k] keeps
//   the least n with k(n) = k (record candidates are its suffix minima).
#include <algorithm>
#include <cstring>

#include <cub/cub.cuh>

#include "common.cuh"
#include "tile.cuh"

namespace sqf2k {

uint64_t generate_primes_device(uint64_t limit);

namespace {

constexpr uint64_t kDefaultBatch = 1ull << 36;

// -------------------------------------------------------------------------
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

// -------------------------------------------------------------------------
// Setup of one batch: medium-prime table, balanced items, pattern residues.
// primes: ascending table (u32); [i_med0, i_med1) are the primes 11..kPMed-1.
struct BatchSetup {
    uint32_t n_med, n_items;
    uint32_t pat_q[3], pat_bits[3], pat_r[3];
};

__global__ void setup_kernel(const uint32_t *__restrict__ primes, uint32_t n_primes,
                             int64_t base_n, uint32_t *__restrict__ med,
                             uint32_t *__restrict__ items, BatchSetup *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    BatchSetup s;
    const uint32_t pq[3] = {9, 25, 49}, pb[3] = {0x08040201u, 0x02000001u, 0x1u};
    for (int i = 0; i < 3; ++i) {
        s.pat_q[i] = 1;
        s.pat_bits[i] = 0;
        s.pat_r[i] = 0;
    }
    uint32_t nm = 0, ni = 0;
    for (uint32_t i = 0; i < n_primes; ++i) {
        uint32_t p = primes[i];
        if (p >= kPMed) break;
        if (p == 3 || p == 5 || p == 7) {
            int j = p == 3 ? 0 : (p == 5 ? 1 : 2);
            s.pat_q[j] = pq[j];
            s.pat_bits[j] = pb[j];
            s.pat_r[j] = (uint32_t)slot_residue(base_n, pq[j]);
            continue;
        }
        if (p < 11 || nm >= (uint32_t)kMaxMed) continue;
        uint32_t q = p * p;
        med[3 * nm + 0] = q;
        med[3 * nm + 1] = (uint32_t)slot_residue(base_n, q);
        med[3 * nm + 2] = (uint32_t)kTile % q;
        uint32_t m = (uint32_t)kTile / (q * (uint32_t)kItemHits);
        m = m < 1 ? 1 : (m > 64 ? 64 : m);
        for (uint32_t j = 0; j < m && ni < (uint32_t)kMaxItems; ++j, ++ni) {
            items[2 * ni + 0] = (nm << 16) | j;
            items[2 * ni + 1] = m * q;
        }
        ++nm;
    }
    s.n_med = nm;
    s.n_items = ni;
    *out = s;
}

// -------------------------------------------------------------------------
// Bucket pass: every hit u of a bucket prime (p >= kPMed, p^2 <= n_max) in the
// batch domain [0, U), as a 16-bit offset in the list of tile u >> 16.
// Dense primes (q < kSub) are split into (prime, sub-range) work units.
constexpr uint64_t kSub = 1ull << 26;

template <bool FILL>
__global__ void __launch_bounds__(256) bucket_kernel(
    const uint32_t *__restrict__ primes, uint32_t i_lo, uint32_t i_mid, uint32_t i_hi,
    int64_t base_n, uint64_t U, uint64_t n_sub, uint32_t *__restrict__ counts,
    uint32_t *__restrict__ cursor, uint16_t *__restrict__ hits) {
    const uint64_t n_dense = (uint64_t)(i_mid - i_lo) * n_sub;
    const uint64_t n_work = n_dense + (i_hi - i_mid);
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < n_work;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t p, lo, hi;
        if (w < n_dense) {
            p = primes[i_lo + w / n_sub];
            lo = (w % n_sub) * kSub;
            hi = min(lo + kSub, U);
            if (lo >= U) continue;
        } else {
            p = primes[i_mid + (w - n_dense)];
            lo = 0;
            hi = U;
        }
        const uint64_t q = p * p;
        const uint64_t r = slot_residue(base_n, q);
        uint64_t lm = lo % q;
        uint64_t u = lo + (r >= lm ? r - lm : r + q - lm);
        for (; u < hi; u += q) {
            uint32_t t = (uint32_t)(u >> 16);
            if (FILL) {
                uint32_t pos = atomicAdd(&cursor[t], 1u);
                hits[pos] = (uint16_t)(u & 0xffff);
            } else {
                atomicAdd(&counts[t], 1u);
            }
        }
    }
}

// -------------------------------------------------------------------------
// The tile kernel.
template <bool FUSED>
struct TileSmem {
    uint8_t bytes[kTile];                               // 64 KB, 16-byte aligned
    uint32_t bits[kHaloWordsMax + kTileWords];          // halo + tile (12 KB)
    uint32_t med_q[kMaxMed], med_tq[kMaxMed], off[kMaxMed];
    unsigned long long first[kDepthMax + 1];
    uint32_t need;
};

__device__ __forceinline__ void init_bytes(uint8_t *bytes, uint32_t len) {
    uint4 one = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    for (uint32_t i = threadIdx.x; i < len / 16; i += kThreads)
        reinterpret_cast<uint4 *>(bytes)[i] = one;
}

// clear the medium-prime hits in [0, len) of the current base
__device__ __forceinline__ void scatter_medium(uint8_t *bytes, const uint32_t *off,
                                               const uint32_t *med_q, const TileParams &P,
                                               uint32_t len) {
    for (uint32_t it = threadIdx.x; it < P.n_items; it += kThreads) {
        uint32_t mj = __ldg(&P.items[2 * it]), stride = __ldg(&P.items[2 * it + 1]);
        uint32_t m = mj >> 16, j = mj & 0xffffu;
        for (uint32_t o = off[m] + j * med_q[m]; o < len; o += stride) bytes[byte_pos(o)] = 0;
    }
}

// clear the bucket hits of tile t with offsets in [skip, kTile), shifted by -skip
__device__ __forceinline__ void scatter_bucket(uint8_t *bytes, const TileParams &P, uint32_t t,
                                               uint32_t skip) {
    uint32_t b = __ldg(&P.tile_start[t]), e = __ldg(&P.tile_start[t + 1]);
    for (uint32_t i = b + threadIdx.x; i < e; i += kThreads) {
        uint32_t o = __ldg(&P.hits[i]);
        if (o >= skip) bytes[byte_pos(o - skip)] = 0;
    }
}

// advance the medium offsets from base to base + len (len <= kTile)
__device__ __forceinline__ void advance_medium(uint32_t *off, const uint32_t *med_q,
                                               const uint32_t *step, const TileParams &P) {
    for (uint32_t m = threadIdx.x; m < P.n_med; m += kThreads) {
        int32_t o = (int32_t)off[m] - (int32_t)step[m];
        off[m] = (uint32_t)(o < 0 ? o + (int32_t)med_q[m] : o);
    }
}

// Pack `words` words of bytes (base slot `base`) into out[], applying the
// p = 3, 5, 7 patterns, the n < 1 zero region and the domain end.
// Y[i] = (pat_r - base) mod pat_q  (CTA-uniform).
__device__ __forceinline__ void pack_words(const uint8_t *bytes, uint32_t *out, uint32_t words,
                                           uint64_t base, const TileParams &P, const uint32_t Y[3]) {
    uint32_t y[3], step[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const uint32_t q = P.pat_q[i];
        uint32_t c = (32u * threadIdx.x) % q;
        y[i] = Y[i] >= c ? Y[i] - c : Y[i] + q - c;
        step[i] = (32u * kThreads) % q;
    }
    for (uint32_t w = threadIdx.x; w < words; w += kThreads) {
        const uint8_t *blk = bytes + ((w >> 5) << 10) + ((w & 31) << 4);
        uint4 a = *reinterpret_cast<const uint4 *>(blk);
        uint4 b = *reinterpret_cast<const uint4 *>(blk + 512);
        uint32_t word = a.x | (a.y << 1) | (a.z << 2) | (a.w << 3) | (b.x << 4) | (b.y << 5) |
                        (b.z << 6) | (b.w << 7);
        uint32_t clr = shl_clamp(P.pat_bits[0], y[0]) | shl_clamp(P.pat_bits[1], y[1]) |
                       shl_clamp(P.pat_bits[2], y[2]);
        word &= ~clr;
        const uint64_t u0 = base + 32ull * w;
        if (u0 < P.z) word = (u0 + 32 <= P.z) ? 0u : (word & (~0u << (uint32_t)(P.z - u0)));
        if (u0 + 32 > P.U) word = (u0 >= P.U) ? 0u : (word & ((1u << (uint32_t)(P.U - u0)) - 1u));
        out[w] = word;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            int32_t t = (int32_t)y[i] - (int32_t)step[i];
            y[i] = (uint32_t)(t < 0 ? t + (int32_t)P.pat_q[i] : t);
        }
    }
}

__device__ __forceinline__ void append(unsigned long long *list, unsigned long long *count,
                                       uint64_t cap, uint64_t n) {
    unsigned long long i = atomicAdd(count, 1ull);
    if (i < cap) list[i] = n;
}

template <bool FUSED>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) tile_kernel(const TileParams P) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    TileSmem<FUSED> &S = *reinterpret_cast<TileSmem<FUSED> *>(smem_raw);
    const uint32_t G = gridDim.x;
    const uint32_t t0 = (uint32_t)((uint64_t)P.n_tiles * blockIdx.x / G);
    const uint32_t t1 = (uint32_t)((uint64_t)P.n_tiles * (blockIdx.x + 1) / G);
    if (t0 >= t1) return;
    const uint32_t H = FUSED ? P.H : 0u;
    const uint32_t HW = H / 32;

    // medium primes: q, kTile mod q, offset of the first hit at the chunk base
    const uint64_t b0 = (FUSED && t0 > 0) ? (uint64_t)t0 * kTile - H : (uint64_t)t0 * kTile;
    for (uint32_t m = threadIdx.x; m < P.n_med; m += kThreads) {
        uint32_t q = P.med[3 * m], r = P.med[3 * m + 1];
        S.med_q[m] = q;
        S.med_tq[m] = P.med[3 * m + 2];
        uint32_t bm = mod_u64(b0, q);
        S.off[m] = r >= bm ? r - bm : r + q - bm;
    }
    uint32_t Y[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        uint32_t bm = mod_u64(b0, P.pat_q[i]);
        Y[i] = P.pat_r[i] >= bm ? P.pat_r[i] - bm : P.pat_r[i] + P.pat_q[i] - bm;
    }
    if (FUSED && threadIdx.x <= kDepthMax) S.first[threadIdx.x] = ~0ull;
    if (FUSED && threadIdx.x == 0) S.need = ~0u;
    __syncthreads();

    if (FUSED) {
        if (t0 > 0) {
            // pre-tile: sieve the H slots below the chunk into the halo words
            init_bytes(S.bytes, H);
            __syncthreads();
            scatter_medium(S.bytes, S.off, S.med_q, P, H);
            scatter_bucket(S.bytes, P, t0 - 1, kTile - H);
            __syncthreads();
            pack_words(S.bytes, S.bits, HW, b0, P, Y);
            // offsets and patterns move to the chunk's first tile
            for (uint32_t m = threadIdx.x; m < P.n_med; m += kThreads) {
                uint32_t q = S.med_q[m], d = H % q;
                int32_t o = (int32_t)S.off[m] - (int32_t)d;
                S.off[m] = (uint32_t)(o < 0 ? o + (int32_t)q : o);
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                uint32_t d = H % P.pat_q[i];
                Y[i] = Y[i] >= d ? Y[i] - d : Y[i] + P.pat_q[i] - d;
            }
        } else {
            for (uint32_t i = threadIdx.x; i < HW; i += kThreads) S.bits[i] = 0u;
        }
        __syncthreads();
    }

    uint32_t cnt[kDepthMax + 1];
#pragma unroll
    for (int k = 0; k <= kDepthMax; ++k) cnt[k] = 0;

    for (uint32_t t = t0; t < t1; ++t) {
        const uint64_t tb = (uint64_t)t * kTile;
        init_bytes(S.bytes, kTile);
        __syncthreads();
        scatter_medium(S.bytes, S.off, S.med_q, P, kTile);
        scatter_bucket(S.bytes, P, t, 0);
        __syncthreads();
        pack_words(S.bytes, S.bits + HW, kTileWords, tb, P, Y);
        advance_medium(S.off, S.med_q, S.med_tq, P);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            uint32_t d = (uint32_t)kTile % P.pat_q[i];
            Y[i] = Y[i] >= d ? Y[i] - d : Y[i] + P.pat_q[i] - d;
        }
        __syncthreads();
        if (!FUSED) {
            for (uint32_t w = threadIdx.x; w < kTileWords; w += kThreads)
                P.bits_out[(uint64_t)t * kTileWords + w] = S.bits[w];
            __syncthreads();
            continue;
        }
        // ---- exponent passes (search.py:368-381) over the packed tile ----
        const uint32_t need = S.need;
        const bool interior = tb >= P.scan_lo && tb + kTile <= P.U &&
                              (P.one_u < tb || P.one_u >= tb + kTile);
        for (uint32_t w = threadIdx.x; w < kTileWords; w += kThreads) {
            const uint64_t u0 = tb + 32ull * w;
            uint32_t pend = ~0u;
            if (!interior) {
                if (u0 + 32 <= P.scan_lo || u0 >= P.U) pend = 0u;
                else {
                    if (u0 < P.scan_lo) pend &= ~0u << (uint32_t)(P.scan_lo - u0);
                    if (u0 + 32 > P.U) pend &= (1u << (uint32_t)(P.U - u0)) - 1u;
                    if (P.one_u >= u0 && P.one_u < u0 + 32) pend &= ~(1u << (uint32_t)(P.one_u - u0));
                }
            }
            const uint32_t cur = S.bits[HW + w], prv = S.bits[HW + w - 1];
#pragma unroll
            for (int k = 1; k <= kDepthMax; ++k) {
                if ((uint32_t)k > P.k_eff) break;
                if (!__any_sync(0xffffffffu, pend)) break;
                uint32_t sl;
                if (k <= 5) sl = __funnelshift_l(prv, cur, 1u << (k - 1));
                else if (k == 6) sl = prv;
                else sl = S.bits[HW + w - (1u << (k - 6))];
                const uint32_t nw = pend & sl;
                cnt[k] += __popc(nw);
                if (nw && ((need >> k) & 1u))
                    atomicMin(&S.first[k], (unsigned long long)(u0 + __ffs(nw) - 1));
                pend &= ~sl;
            }
            if (pend) {
                const bool esc = P.k_max > P.k_eff;
                for (uint32_t x = pend; x; x &= x - 1) {
                    uint64_t n = (uint64_t)(P.base_n + 2 * (int64_t)(u0 + __ffs(x) - 1));
                    if (esc) append(P.esc, P.esc_count, P.esc_cap, n);
                    else append(P.fail, P.fail_count, P.fail_cap, n);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x >= 1 && threadIdx.x <= kDepthMax) {
            unsigned long long f = S.first[threadIdx.x];
            if (f != ~0ull) {
                atomicMin(&P.min_n[threadIdx.x],
                          (unsigned long long)(P.base_n + 2 * (int64_t)f));
                atomicAnd(&S.need, ~(1u << threadIdx.x));
                S.first[threadIdx.x] = ~0ull;
            }
        }
        // roll the halo: the last H slots of this tile precede the next one
        for (uint32_t i = threadIdx.x; i < HW; i += kThreads) S.bits[i] = S.bits[kTileWords + i];
        __syncthreads();
    }

    if (FUSED) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int k = 1; k <= kDepthMax; ++k) {
            if ((uint32_t)k > P.k_eff) break;
            uint32_t s = __reduce_add_sync(0xffffffffu, cnt[k]);
            if (lane == 0 && s) atomicAdd(&P.hist[k], (unsigned long long)s);
        }
    }
}

// -------------------------------------------------------------------------
// Exact squarefree test by trial division, one warp per m (odd m >= 1):
// lanes take the odd primes p (index >= 1) with p^2 <= m.
__device__ bool warp_squarefree(uint64_t m, const uint32_t *__restrict__ primes,
                                uint64_t n_primes) {
    const int lane = threadIdx.x & 31;
    for (uint64_t base = 1; base < n_primes; base += 32) {
        uint64_t i = base + lane;
        bool live = false, hit = false;
        if (i < n_primes) {
            uint64_t p = primes[i];
            uint64_t q = p * p;
            live = q <= m;
            hit = live && (m % q == 0);
        }
        if (__any_sync(0xffffffffu, hit)) return false;
        if (!__any_sync(0xffffffffu, live)) break;
    }
    return true;
}

// Escalation: n unresolved at the tile depth, exponents k_from..k_max exactly.
__global__ void escalate_kernel(const unsigned long long *__restrict__ esc,
                                const unsigned long long *__restrict__ esc_count,
                                uint32_t k_from, uint32_t k_max,
                                const uint32_t *__restrict__ primes, uint64_t n_primes,
                                unsigned long long *hist, unsigned long long *min_n,
                                unsigned long long *fail, unsigned long long *fail_count,
                                uint64_t fail_cap) {
    const uint64_t count = *esc_count;
    const uint64_t warps = (uint64_t)gridDim.x * blockDim.x / 32;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32; i < count;
         i += warps) {
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
                append(fail, fail_count, fail_cap, n);
            }
        }
    }
}

// runner.py:105-114: least k in [1, 63] with n - 2^k squarefree, 0 if none.
__global__ void recheck_kernel(const unsigned long long *__restrict__ ns, uint64_t count,
                               const uint32_t *__restrict__ primes, uint64_t n_primes,
                               int32_t *__restrict__ k_out) {
    const uint64_t warps = (uint64_t)gridDim.x * blockDim.x / 32;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32; i < count;
         i += warps) {
        const uint64_t n = ns[i];
        int32_t found = 0;
        for (uint32_t k = 1; k <= 63 && !found; ++k) {
            if (n <= (1ull << k)) break;
            if (warp_squarefree(n - (1ull << k), primes, n_primes)) found = (int32_t)k;
        }
        if ((threadIdx.x & 31) == 0) k_out[i] = found;
    }
}

__global__ void squarefree_kernel(const unsigned long long *__restrict__ ns, uint64_t count,
                                  const uint32_t *__restrict__ primes, uint64_t n_primes,
                                  uint8_t *__restrict__ out) {
    const uint64_t warps = (uint64_t)gridDim.x * blockDim.x / 32;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32; i < count;
         i += warps) {
        const uint64_t n = ns[i];
        // p = 2 counts here: the reference oracle divides by every p <= isqrt(n)
        bool sf = (n % 4) != 0 && warp_squarefree(n, primes, n_primes);
        if ((threadIdx.x & 31) == 0) out[i] = sf ? 1 : 0;
    }
}

__global__ void narrow_primes_kernel(const int64_t *__restrict__ in, uint32_t *__restrict__ out,
                                     uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

// -------------------------------------------------------------------------
// Host side

struct Acc {
    unsigned long long hist[SQF2K_HIST_LEN];
    unsigned long long min_n[SQF2K_HIST_LEN];
    unsigned long long esc_count, fail_count;
};

// index of the first entry >= v in the ascending device table (host copy of
// the few needed values is avoided: binary search on the device)
__global__ void lower_bound_kernel(const uint32_t *__restrict__ a, uint64_t n, uint64_t v,
                                   uint64_t *out) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if ((uint64_t)a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    *out = lo;
}

uint64_t lower_bound(const uint32_t *a, uint64_t n, uint64_t v) {
    Context &c = ctx();
    c.scan_tmp.reserve(64);
    uint64_t *d = c.scan_tmp.as<uint64_t>();
    launch("lower_bound", lower_bound_kernel, dim3(1), dim3(1), 0, a, n, v, d);
    uint64_t h = 0;
    copy_d2h(&h, d, 8);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    return h;
}

struct PrimeSplit {
    uint32_t i_lo, i_mid, i_hi;  // bucket primes [i_lo, i_hi), dense ones [i_lo, i_mid)
};

PrimeSplit split_primes(const uint32_t *primes, uint64_t n_primes, uint64_t n_max) {
    PrimeSplit s;
    s.i_lo = (uint32_t)lower_bound(primes, n_primes, kPMed);
    uint64_t root = isqrt_u64(n_max);
    s.i_hi = (uint32_t)lower_bound(primes, n_primes, root + 1);
    if (s.i_hi < s.i_lo) s.i_hi = s.i_lo;
    uint64_t sub_root = isqrt_u64(kSub - 1);  // q < kSub  <=>  p <= isqrt(kSub - 1)
    s.i_mid = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(lower_bound(primes, n_primes, sub_root + 1), s.i_lo), s.i_hi);
    return s;
}

static size_t tile_smem_bytes() { return sizeof(TileSmem<true>); }

// One batch domain: slots [0, U) for n(u) = base_n + 2u.  Builds the setup
// and bucket lists, then launches the tile kernel.
void run_tile_batch(bool fused, int64_t base_n, uint64_t U, uint64_t scan_lo, uint64_t z,
                    uint64_t one_u, uint32_t H, uint32_t k_eff, uint32_t k_max,
                    const uint32_t *primes, uint64_t n_primes, const PrimeSplit &ps,
                    Acc *acc_dev, uint64_t esc_cap, uint64_t fail_cap, uint32_t *bits_out) {
    Context &c = ctx();
    const uint32_t n_tiles = (uint32_t)ceil_div(U, kTile);

    // setup (medium primes, items, patterns)
    c.items.reserve(3 * kMaxMed * 4 + 2 * kMaxItems * 4 + sizeof(BatchSetup) + 64);
    uint32_t *med = c.items.as<uint32_t>();
    uint32_t *items = med + 3 * kMaxMed;
    BatchSetup *setup = reinterpret_cast<BatchSetup *>(items + 2 * kMaxItems);
    const uint32_t n_small = (uint32_t)std::min<uint64_t>(n_primes, ps.i_lo);
    launch("setup", setup_kernel, dim3(1), dim3(32), 0, primes, n_small, base_n, med, items,
           setup);

    // bucket lists: count, scan, fill
    c.tile_counts.reserve((n_tiles + 1) * 4);
    c.tile_offsets.reserve((n_tiles + 1) * 4);
    c.tile_cursor.reserve((n_tiles + 1) * 4);
    uint32_t *counts = c.tile_counts.as<uint32_t>();
    uint32_t *offsets = c.tile_offsets.as<uint32_t>();
    uint32_t *cursor = c.tile_cursor.as<uint32_t>();
    SQF2K_CUDA(cudaMemsetAsync(counts, 0, (n_tiles + 1) * 4, c.stream));
    const uint64_t n_sub = ceil_div(U, kSub);
    const uint64_t n_work = (uint64_t)(ps.i_mid - ps.i_lo) * n_sub + (ps.i_hi - ps.i_mid);
    const unsigned bgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n_work, 256), (uint64_t)c.sm_count * 8));
    if (n_work)
        launch("bucket_count", bucket_kernel<false>, dim3(bgrid), dim3(256), 0, primes, ps.i_lo,
               ps.i_mid, ps.i_hi, base_n, U, n_sub, counts, cursor, (uint16_t *)nullptr);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, offsets, (int)n_tiles + 1, c.stream);
    c.scan_tmp.reserve(std::max<size_t>(tmp_bytes, 64));
    SQF2K_CUDA(cub::DeviceScan::ExclusiveSum(c.scan_tmp.ptr, tmp_bytes, counts, offsets,
                                             (int)n_tiles + 1, c.stream));
    uint32_t total = 0;
    copy_d2h(&total, offsets + n_tiles, 4);
    SQF2K_CUDA(cudaMemcpyAsync(cursor, offsets, (n_tiles + 1) * 4, cudaMemcpyDeviceToDevice,
                               c.stream));
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    c.hits.reserve((size_t)total * 2 + 16);
    if (n_work && total)
        launch("bucket_fill", bucket_kernel<true>, dim3(bgrid), dim3(256), 0, primes, ps.i_lo,
               ps.i_mid, ps.i_hi, base_n, U, n_sub, counts, cursor, c.hits.as<uint16_t>());

    BatchSetup hs;
    copy_d2h(&hs, setup, sizeof hs);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));

    TileParams P;
    std::memset(&P, 0, sizeof P);
    P.base_n = base_n;
    P.U = U;
    P.scan_lo = scan_lo;
    P.z = z;
    P.one_u = one_u;
    P.H = H;
    P.n_tiles = n_tiles;
    P.k_eff = k_eff;
    P.k_max = k_max;
    for (int i = 0; i < 3; ++i) {
        P.pat_q[i] = hs.pat_q[i];
        P.pat_bits[i] = hs.pat_bits[i];
        P.pat_r[i] = hs.pat_r[i];
    }
    P.n_med = hs.n_med;
    P.n_items = hs.n_items;
    P.med = med;
    P.items = items;
    P.tile_start = offsets;
    P.hits = c.hits.as<uint16_t>();
    if (acc_dev) {
        P.hist = acc_dev->hist;
        P.min_n = acc_dev->min_n;
        P.esc = c.esc.as<unsigned long long>();
        P.esc_count = &acc_dev->esc_count;
        P.esc_cap = esc_cap;
        P.fail = c.fail.as<unsigned long long>();
        P.fail_count = &acc_dev->fail_count;
        P.fail_cap = fail_cap;
    }
    P.bits_out = bits_out;

    const size_t smem = tile_smem_bytes();
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>(n_tiles, (uint64_t)c.sm_count * kCtasPerSm));
    if (fused) {
        static bool attr = false;
        if (!attr) {
            SQF2K_CUDA(cudaFuncSetAttribute(tile_kernel<true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = true;
        }
        launch("tile_fused", tile_kernel<true>, dim3(grid), dim3(kThreads), smem, P);
    } else {
        static bool attr = false;
        if (!attr) {
            SQF2K_CUDA(cudaFuncSetAttribute(tile_kernel<false>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = true;
        }
        launch("tile_export", tile_kernel<false>, dim3(grid), dim3(kThreads), smem, P);
    }
}

}  // namespace

// window scan over an exported bitmap (scan.cu)
void scan_bitmap_device(const uint32_t *words, uint64_t cur_word0, uint64_t n_slots,
                        uint64_t first_n, uint32_t k_scan, uint32_t k_max, uint64_t one_slot,
                        unsigned long long *hist, unsigned long long *min_n,
                        unsigned long long *esc, unsigned long long *esc_count, uint64_t esc_cap,
                        unsigned long long *fail, unsigned long long *fail_count,
                        uint64_t fail_cap);

// Summary derivation shared with scan.cu: k_sum, k_max_observed, candidates.
void finish_summary(sqf2k_summary_t *out, const uint64_t *fail_sorted_head, uint64_t n_fail) {
    out->k_sum = 0;
    out->k_max_observed = 0;
    for (int k = 1; k < SQF2K_HIST_LEN; ++k) {
        out->k_sum += (uint64_t)k * out->hist[k];
        if (out->hist[k]) out->k_max_observed = (uint32_t)k;
    }
    // cand[m] = least n with k(n) > m  (failures count as beyond k_max)
    uint64_t run = n_fail ? fail_sorted_head[0] : SQF2K_NONE;
    for (int m = SQF2K_HIST_LEN - 1; m >= 0; --m) {
        out->cand[m] = (m >= 1 && (uint32_t)m <= out->k_max) ? run : SQF2K_NONE;
        if (m >= 1 && out->min_n[m] < run) run = out->min_n[m];
    }
    out->n_failures = n_fail;
}

// Sort the device failure list (count <= capacity) and copy to the caller.
int deliver_failures(unsigned long long *fail_dev, uint64_t n_fail, uint64_t *failures,
                     uint64_t fail_cap, uint64_t *smallest) {
    Context &c = ctx();
    *smallest = SQF2K_NONE;
    if (!n_fail) return SQF2K_OK;
    c.fail_sorted.reserve(n_fail * 8);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp, fail_dev, c.fail_sorted.as<unsigned long long>(),
                                   (int)n_fail, 0, 64, c.stream);
    c.scan_tmp.reserve(std::max<size_t>(tmp, 64));
    SQF2K_CUDA(cub::DeviceRadixSort::SortKeys(c.scan_tmp.ptr, tmp, fail_dev,
                                              c.fail_sorted.as<unsigned long long>(), (int)n_fail,
                                              0, 64, c.stream));
    uint64_t head = 0;
    copy_d2h(&head, c.fail_sorted.ptr, 8);
    if (failures && fail_cap)
        copy_d2h(failures, c.fail_sorted.ptr, std::min(n_fail, fail_cap) * 8);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    *smallest = head;
    return SQF2K_OK;
}

// The verify driver: batches of independent sub-ranges.
int verify_range(uint64_t start, uint64_t end, uint32_t k_max, const sqf2k_verify_opts_t &o,
                 sqf2k_summary_t *out, uint64_t *failures, uint64_t fail_cap) {
    Context &c = ctx();
    const uint32_t depth = o.tile_depth ? o.tile_depth : kDepthMax;
    if (depth < 1 || depth > (uint32_t)kDepthMax)
        return fail(SQF2K_EINVAL, "tile_depth must be in 1..%d", kDepthMax);
    const uint32_t k_eff = std::min(k_max, depth);
    const uint32_t H = std::max<uint32_t>(1024u, 1u << (k_eff - 1));
    uint64_t batch = o.batch_slots ? o.batch_slots : kDefaultBatch;
    batch = std::max<uint64_t>(batch, (uint64_t)kTile);
    const uint64_t n_slots = (end - start) / 2;

    // prime table up to isqrt(end - 1) (runner.py:192)
    const uint64_t limit = isqrt_u64(end - 1);
    const uint64_t n_primes = generate_primes_device(limit);
    const uint32_t *primes = c.primes_u32.as<uint32_t>();
    const PrimeSplit ps = split_primes(primes, n_primes, end - 1);

    uint64_t esc_cap = 1 << 16, dev_fail_cap = std::max<uint64_t>(fail_cap, 1 << 12);
    for (int attempt = 0; attempt < 4; ++attempt) {
        c.acc.reserve(sizeof(Acc));
        c.esc.reserve(esc_cap * 8);
        c.fail.reserve(dev_fail_cap * 8);
        Acc *acc = c.acc.as<Acc>();
        {
            Acc init;
            std::memset(&init, 0, sizeof init);
            for (int k = 0; k < SQF2K_HIST_LEN; ++k) init.min_n[k] = ~0ull;
            copy_h2d(acc, &init, sizeof init);
        }
        for (uint64_t s0 = 0; s0 < n_slots; s0 += batch) {
            const uint64_t sb = std::min(batch, n_slots - s0);
            const uint64_t A = start + 2 * s0;  // first n of the batch
            if (o.pipeline == 1) {
                // two-pass: export the bitmap of [A - 2H, A + 2 sb) then scan it
                const int64_t base_n = (int64_t)A - 2 * (int64_t)H;
                const uint64_t U = H + sb;
                const uint64_t z = base_n < 1 ? (uint64_t)((1 - base_n) / 2) : 0;
                const uint32_t nt = (uint32_t)ceil_div(U, kTile);
                c.window.reserve((size_t)nt * kTile / 8 + 64);
                run_tile_batch(false, base_n, U, 0, z, ~0ull, 0, k_eff, k_max, primes, n_primes,
                               ps, nullptr, 0, 0, c.window.as<uint32_t>());
                scan_bitmap_device(c.window.as<uint32_t>(), H / 32, sb, A, k_eff, k_max,
                                   A == 1 ? 0 : ~0ull, acc->hist, acc->min_n,
                                   c.esc.as<unsigned long long>(), &acc->esc_count, esc_cap,
                                   c.fail.as<unsigned long long>(), &acc->fail_count,
                                   dev_fail_cap);
            } else {
                const int64_t base_n = (int64_t)A - 2 * (int64_t)H;
                const uint64_t U = H + sb;
                const uint64_t z = base_n < 1 ? (uint64_t)((1 - base_n) / 2) : 0;
                const uint64_t one_u = A == 1 ? (uint64_t)H : ~0ull;
                run_tile_batch(true, base_n, U, H, z, one_u, H, k_eff, k_max, primes, n_primes,
                               ps, acc, esc_cap, dev_fail_cap, nullptr);
            }
        }
        Acc h;
        copy_d2h(&h, acc, sizeof h);
        SQF2K_CUDA(cudaStreamSynchronize(c.stream));
        if (h.esc_count > esc_cap) {  // rerun with room for every escalation
            esc_cap = h.esc_count + 1024;
            continue;
        }
        if (h.esc_count) {
            launch("escalate", escalate_kernel, dim3((unsigned)std::min<uint64_t>(ceil_div(h.esc_count, 8), 4096)),
                   dim3(256), 0, (const unsigned long long *)c.esc.ptr,
                   (const unsigned long long *)&acc->esc_count, k_eff + 1, k_max, primes, n_primes,
                   acc->hist, acc->min_n, c.fail.as<unsigned long long>(), &acc->fail_count,
                   dev_fail_cap);
            copy_d2h(&h, acc, sizeof h);
            SQF2K_CUDA(cudaStreamSynchronize(c.stream));
        }
        if (h.fail_count > dev_fail_cap) {
            if (h.fail_count > fail_cap) {
                out->n_failures = h.fail_count;
                return fail(SQF2K_ECAPACITY, "%llu failures exceed the buffer of %llu",
                            (unsigned long long)h.fail_count, (unsigned long long)fail_cap);
            }
            dev_fail_cap = h.fail_count + 1024;
            continue;
        }
        std::memset(out, 0, sizeof *out);
        out->start = start;
        out->end = end;
        out->k_max = k_max;
        for (int k = 0; k < SQF2K_HIST_LEN; ++k) {
            out->hist[k] = h.hist[k];
            out->min_n[k] = h.min_n[k];
        }
        uint64_t smallest = SQF2K_NONE;
        if (h.fail_count > fail_cap) {
            out->n_failures = h.fail_count;
            finish_summary(out, &smallest, 0);
            out->n_failures = h.fail_count;
            return fail(SQF2K_ECAPACITY, "%llu failures exceed the buffer of %llu",
                        (unsigned long long)h.fail_count, (unsigned long long)fail_cap);
        }
        deliver_failures(c.fail.as<unsigned long long>(), h.fail_count, failures, fail_cap,
                         &smallest);
        finish_summary(out, &smallest, h.fail_count);
        return SQF2K_OK;
    }
    return fail(SQF2K_ECUDA, "verify did not converge on buffer sizes");
}

// sieve_segment: export mode with H = 0 over [start, end), caller's primes.
int sieve_bits(uint64_t start, uint64_t end, const int64_t *primes_h, uint64_t n_primes_h,
               uint8_t *out, uint64_t nbytes) {
    Context &c = ctx();
    const uint64_t n_slots = (end - start) / 2;
    // only primes with p^2 <= end - 1 can clear a slot (sieve.py:137)
    const uint64_t root = isqrt_u64(end - 1);
    uint64_t np = 0;
    {
        uint64_t lo = 0, hi = n_primes_h;
        while (lo < hi) {
            uint64_t mid = (lo + hi) / 2;
            if ((uint64_t)primes_h[mid] <= root) lo = mid + 1;
            else hi = mid;
        }
        np = lo;
    }
    c.host_primes.reserve(std::max<uint64_t>(np, 1) * 8);
    c.primes_u32.reserve(std::max<uint64_t>(np, 1) * 4);
    if (np) {
        copy_h2d(c.host_primes.ptr, primes_h, np * 8);
        launch("primes_narrow", narrow_primes_kernel,
               dim3((unsigned)std::min<uint64_t>(ceil_div(np, 256), 4096)), dim3(256), 0,
               (const int64_t *)c.host_primes.ptr, c.primes_u32.as<uint32_t>(), np);
    }
    c.primes_limit = 0;  // the cached table is now the caller's
    c.primes_count = np;
    const uint32_t *primes = c.primes_u32.as<uint32_t>();
    const PrimeSplit ps = split_primes(primes, np, end - 1);
    const uint32_t nt = (uint32_t)ceil_div(n_slots, kTile);
    c.bits_out.reserve((size_t)nt * kTile / 8 + 64);
    run_tile_batch(false, (int64_t)start, n_slots, 0, 0, ~0ull, 0, 1, 1, primes, np, ps, nullptr,
                   0, 0, c.bits_out.as<uint32_t>());
    copy_d2h(out, c.bits_out.ptr, nbytes);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    return SQF2K_OK;
}

int recheck(const uint64_t *n, uint64_t count, uint64_t prime_limit, int32_t *k_out) {
    Context &c = ctx();
    if (!count) return SQF2K_OK;
    const uint64_t n_primes = generate_primes_device(prime_limit);
    c.esc.reserve(count * 8);
    c.fail.reserve(count * 4);
    copy_h2d(c.esc.ptr, n, count * 8);
    launch("recheck", recheck_kernel, dim3((unsigned)std::min<uint64_t>(ceil_div(count, 8), 4096)),
           dim3(256), 0, (const unsigned long long *)c.esc.ptr, count,
           (const uint32_t *)c.primes_u32.ptr, n_primes, c.fail.as<int32_t>());
    copy_d2h(k_out, c.fail.ptr, count * 4);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    return SQF2K_OK;
}

int is_squarefree(const uint64_t *n, uint64_t count, uint64_t prime_limit, uint8_t *out) {
    Context &c = ctx();
    if (!count) return SQF2K_OK;
    const uint64_t n_primes = generate_primes_device(prime_limit);
    c.esc.reserve(count * 8);
    c.fail.reserve(count + 16);
    copy_h2d(c.esc.ptr, n, count * 8);
    launch("squarefree", squarefree_kernel,
           dim3((unsigned)std::min<uint64_t>(ceil_div(count, 8), 4096)), dim3(256), 0,
           (const unsigned long long *)c.esc.ptr, count, (const uint32_t *)c.primes_u32.ptr,
           n_primes, c.fail.as<uint8_t>());
    copy_d2h(out, c.fail.ptr, count);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    return SQF2K_OK;
}

}  // namespace sqf2k

using namespace sqf2k;

extern "C" int sqf2k_is_squarefree(const uint64_t *n, uint64_t count, uint64_t prime_limit,
                                   uint8_t *out) {
    if (prime_limit > 0xffffffffull) return fail(SQF2K_EINVAL, "prime_limit above 2^32");
    for (uint64_t i = 0; i < count; ++i) {
        if (n[i] < 1) return fail(SQF2K_EINVAL, "n must be positive, got 0");
        if (isqrt_u64(n[i]) > prime_limit)
            return fail(SQF2K_EINVAL, "n = %llu needs primes beyond %llu",
                        (unsigned long long)n[i], (unsigned long long)prime_limit);
    }
    return guarded([&](Context &) -> int { return is_squarefree(n, count, prime_limit, out); });
}

static int check_range(uint64_t start, uint64_t end) {
    if (start < 1 || start % 2 == 0)
        return fail(SQF2K_EINVAL, "start must be a positive odd integer, got %llu",
                    (unsigned long long)start);
    if (end <= start)
        return fail(SQF2K_EINVAL, "end must exceed start, got [%llu, %llu)",
                    (unsigned long long)start, (unsigned long long)end);
    if ((end - start) % 2)
        return fail(SQF2K_EINVAL, "segment must cover whole odd slots, got [%llu, %llu)",
                    (unsigned long long)start, (unsigned long long)end);
    if (end > kMaxEnd)
        return fail(SQF2K_EINVAL, "end %llu beyond the GPU domain 2^62",
                    (unsigned long long)end);
    return SQF2K_OK;
}

extern "C" int sqf2k_verify(uint64_t start, uint64_t end, uint32_t k_max,
                            const sqf2k_verify_opts_t *opts, sqf2k_summary_t *out,
                            uint64_t *failures, uint64_t fail_cap) {
    int rc = check_range(start, end);
    if (rc) return rc;
    if (k_max < 1 || k_max > 63) return fail(SQF2K_EINVAL, "k_max must be in 1..63, got %u", k_max);
    sqf2k_verify_opts_t o;
    std::memset(&o, 0, sizeof o);
    if (opts) o = *opts;
    if (o.pipeline > 1) return fail(SQF2K_EINVAL, "unknown pipeline %u", o.pipeline);
    return guarded([&](Context &) -> int { return verify_range(start, end, k_max, o, out, failures, fail_cap); });
}

extern "C" int sqf2k_sieve_bits(uint64_t start, uint64_t end, const int64_t *primes,
                                uint64_t n_primes, uint8_t *out, uint64_t nbytes) {
    int rc = check_range(start, end);
    if (rc) return rc;
    const uint64_t n_slots = (end - start) / 2;
    if (nbytes != ceil_div(n_slots, 64) * 8)
        return fail(SQF2K_EINVAL, "output holds %llu bytes, segment needs %llu",
                    (unsigned long long)nbytes, (unsigned long long)(ceil_div(n_slots, 64) * 8));
    return guarded([&](Context &) -> int { return sieve_bits(start, end, primes, n_primes, out, nbytes); });
}

extern "C" int sqf2k_recheck(const uint64_t *n, uint64_t count, uint64_t prime_limit,
                             int32_t *k_out) {
    if (prime_limit > 0xffffffffull) return fail(SQF2K_EINVAL, "prime_limit above 2^32");
    for (uint64_t i = 0; i < count; ++i)
        if (n[i] > kMaxEnd || isqrt_u64(n[i]) > prime_limit)
            return fail(SQF2K_EINVAL, "n = %llu needs primes beyond %llu",
                        (unsigned long long)n[i], (unsigned long long)prime_limit);
    return guarded([&](Context &) -> int { return recheck(n, count, prime_limit, k_out); });
}

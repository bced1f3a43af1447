// verify.cu -- the run_verify hot path on the GPU (driver of tile.cu's batch
// pipeline), the exact escalation kernel, the failure recheck, the
// squarefree oracle, and the sieve_segment export entry point.
//
// Reference semantics restated (per odd n, search.py:187-216, runner.py:93-102):
//   k(n) = min{ k in [1, k_max] : n - 2^k >= 1 and n - 2^k squarefree },
//   n = 1 excluded, unresolved n are failures; hist[k] counts, min_n[k] keeps
//   the least n with k(n) = k (record candidates are its suffix minima).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "collectives.cuh"
#include "common.cuh"
#include "finish.cuh"
#include "tile.cuh"

namespace sqf2k {

std::vector<uint32_t> small_primes(uint32_t below);


void scan_bitmap_device(const uint32_t *words, uint64_t cur_word0, uint64_t n_slots,
                        uint64_t first_n, uint32_t k_scan, uint32_t k_max, uint64_t one_slot,
                        unsigned long long *hist, unsigned long long *min_n,
                        unsigned long long *esc, unsigned long long *esc_count, uint64_t esc_cap,
                        unsigned long long *fail, unsigned long long *fail_count,
                        uint64_t fail_cap, unsigned long long *scanned);

namespace {

constexpr uint64_t kDefaultBatch = 1ull << 37;  // measured: 2^36 525, 2^37 487, 2^38 494, 2^39 507 ms per C5 call
constexpr uint64_t kMaxBatch = 1ull << 40;

// Escalation: n unresolved at the tile depth, exponents k_from..k_max exactly.
__global__ void escalate_kernel(const unsigned long long *__restrict__ esc,
                                const unsigned long long *__restrict__ esc_count, uint64_t esc_cap,
                                uint32_t k_from, uint32_t k_max,
                                const uint32_t *__restrict__ primes,
                                const PrimeInfo *__restrict__ info, unsigned long long *hist,
                                unsigned long long *min_n, unsigned long long *fail,
                                unsigned long long *fail_count, uint64_t fail_cap) {
    const uint64_t count = min((unsigned long long)esc_cap, *esc_count);
    escalate_warps(esc, count, k_from, k_max, primes, info->count, hist, min_n, fail, fail_count,
                   fail_cap, (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32,
                   (uint64_t)gridDim.x * blockDim.x / 32);
}

// runner.py:105-114: least k in [1, 63] with n - 2^k squarefree, 0 if none.
__global__ void recheck_kernel(const unsigned long long *__restrict__ ns, uint64_t count,
                               const uint32_t *__restrict__ primes,
                               const PrimeInfo *__restrict__ info, int32_t *__restrict__ k_out) {
    const uint64_t n_primes = info->count;
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

// sieve.py:114-131: trial division by p^2 for every prime p <= isqrt(n)
__global__ void squarefree_kernel(const unsigned long long *__restrict__ ns, uint64_t count,
                                  const uint32_t *__restrict__ primes,
                                  const PrimeInfo *__restrict__ info, uint8_t *__restrict__ out) {
    const uint64_t n_primes = info->count;
    const uint64_t warps = (uint64_t)gridDim.x * blockDim.x / 32;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32; i < count;
         i += warps) {
        const uint64_t n = ns[i];
        // p = 2 counts here: the reference oracle divides by every p <= isqrt(n)
        const bool sf = (n % 4) != 0 && warp_squarefree(n, primes, n_primes);
        if ((threadIdx.x & 31) == 0) out[i] = sf ? 1 : 0;
    }
}

__global__ void narrow_primes_kernel(const int64_t *__restrict__ in, uint32_t *__restrict__ out,
                                     uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}


unsigned warp_grid(uint64_t items) {
    const uint64_t cap = (uint64_t)ctx().sm_count * 2;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(items, 8), cap));
}

// Medium primes and the p = 3, 5, 7 (11) presence of "all primes <= limit".
struct SmallSet {
    std::vector<uint32_t> med;
    uint32_t present = 0;
};

SmallSet small_set_upto_impl(uint64_t limit, int kind) {
    static const std::vector<uint32_t> all = small_primes(kPMed);
    SmallSet s;
    for (uint32_t p : all) {
        if (p > limit) break;
        if (p == 3) s.present |= 1;
        else if (p == 5) s.present |= 2;
        else if (p == 7) s.present |= 4;
        else if (p == 11 && kind >= 1) s.present |= 8;
        else if (p == 13 && kind >= 2) s.present |= 16;
#ifdef SQF2K_EXP_DROP13
        else if (p == 13 && kind >= 1) continue;  // timing experiment only: wrong results
#endif
        else if (p >= 11) s.med.push_back(p);
    }
    return s;
}

// The pattern table kind of a call (tile.cuh): 11 joins the table for domains
// of kPattern11MinSlots slots or more, 13 too (the 3.6 GB wheel table) for
// fused main-depth calls of kPattern13MinSlots or more.
SmallSet small_set_upto(uint64_t limit, uint64_t n_slots, bool allow13) {
    int kind = kPattern11 && n_slots >= kPattern11MinSlots ? 1 : 0;
    // (SQF2K_DEBUG_PAT13_MIN lowers the threshold: tests reach kind 2 on
    // small multi-batch windows)
    static const uint64_t min13 = [] {
        const char *e = std::getenv("SQF2K_DEBUG_PAT13_MIN");
        return e ? std::strtoull(e, nullptr, 0) : kPattern13MinSlots;
    }();
    if (kind && kPattern13 && allow13 && n_slots >= min13) kind = 2;
    if (limit >= kPMed) {  // every range above 2^20: the full sets, built once
        static const SmallSet full[3] = {small_set_upto_impl(kPMed, 0), small_set_upto_impl(kPMed, 1),
                                         small_set_upto_impl(kPMed, 2)};
        return full[kind];
    }
    return small_set_upto_impl(limit, kind);
}

}  // namespace

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

// Sort the device failure list (count <= capacity) and copy to the caller:
// bitonic sort on the GPU (collectives.cuh), one CTA up to kSortSmem keys.
int deliver_failures(unsigned long long *fail_dev, uint64_t n_fail, uint64_t *failures,
                     uint64_t fail_cap, uint64_t *smallest) {
    Context &c = ctx();
    *smallest = SQF2K_NONE;
    if (!n_fail) return SQF2K_OK;
    uint64_t m = 1;
    while (m < n_fail) m <<= 1;
    c.fail_sorted.reserve(m * 8);
    unsigned long long *keys = c.fail_sorted.as<unsigned long long>();
    SQF2K_CUDA(cudaMemcpyAsync(keys, fail_dev, n_fail * 8, cudaMemcpyDeviceToDevice, c.stream));
    if (m <= (uint64_t)kSortSmem) {
        launch("sort_failures", sort_small_kernel, dim3(1), dim3(kScanThreads), 0, keys,
               (uint32_t)n_fail);
    } else {
        const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(m, 256), 4096);
        launch("sort_pad", pad_keys_kernel, dim3(grid), dim3(256), 0, keys, n_fail, m);
        for (uint64_t k = 2; k <= m; k <<= 1)
            for (uint64_t j = k >> 1; j; j >>= 1)
                launch("sort_step", bitonic_step_kernel, dim3(grid), dim3(256), 0, keys, m, k, j);
    }
    uint64_t head = 0;
    copy_d2h(&head, keys, 8);
    if (failures && fail_cap) copy_d2h(failures, keys, std::min(n_fail, fail_cap) * 8);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    *smallest = head;
    return SQF2K_OK;
}

// Everything one verify call puts on the stream, from the prime table to the
// accumulator readback into pinned memory; no host synchronisation inside.
struct VerifyPlan {
    uint64_t start, end, n_slots, batch, limit, esc_cap, dev_fail_cap;
    uint32_t k_max, k_eff, H, pipeline;
    bool exact, default_depth;
    SmallSet small;
};

void enqueue_verify(const VerifyPlan &pl) {
    Context &c = ctx();
    c.acc.reserve(sizeof(Acc));
    c.esc.reserve(pl.esc_cap * 8);
    c.fail.reserve(pl.dev_fail_cap * 8);
    Acc *acc = c.acc.as<Acc>();
    BatchArgs a;
    std::memset(&a, 0, sizeof a);
    a.k_eff = pl.k_eff;
    a.k_max = pl.k_max;
    a.n_primes_bound = pi_upper(pl.limit);
    a.pattern_present = pl.small.present;
    a.med_primes = &pl.small.med;
    a.hist = acc->hist;
    a.min_n = acc->min_n;
    a.esc_count = &acc->esc_count;
    a.esc_cap = pl.esc_cap;
    a.fail_count = &acc->fail_count;
    a.fail_cap = pl.dev_fail_cap;
    a.exact_buckets = pl.exact;
    a.overflow = &acc->overflow;
    a.scanned = &acc->scanned;
    const uint32_t H = pl.H;
    // batch s0 covers the odd n from A = start + 2 s0 on; its domain starts H
    // slots (the halo) below A
    auto set_batch = [&](uint64_t s0) {
        const uint64_t sb = std::min(pl.batch, pl.n_slots - s0);
        const uint64_t A = pl.start + 2 * s0;
        a.base_n = (int64_t)A - 2 * (int64_t)H;
        a.U = H + sb;
        a.z = a.base_n < 1 ? (uint64_t)((1 - a.base_n) / 2) : 0;
        if (pl.pipeline == 1) {  // two-pass: export [A - 2H, A + 2 sb), then scan it
            a.fused = false;
            a.scan_lo = 0;
            a.one_u = ~0ull;
            a.H = 0;
            const uint32_t nt = (uint32_t)ceil_div(a.U, kTile);
            c.window.reserve((size_t)nt * kTile / 8 + 64);
            a.bits_out = c.window.as<uint32_t>();
        } else {
            a.fused = true;
            a.scan_lo = H;
            a.one_u = A == 1 ? (uint64_t)H : ~0ull;
            a.H = H;
            a.bits_out = nullptr;
        }
        return std::make_pair(A, sb);
    };
    a.esc = c.esc.as<unsigned long long>();
    a.fail = c.fail.as<unsigned long long>();
    set_batch(0);  // allocations before the fork

    // side stream: accumulators and the first batch's prime-free preparation,
    // in parallel with the prime table (runner.py:192) on the main stream
    fork_side();
    SQF2K_CUDA(cudaMemsetAsync(acc, 0, sizeof(Acc), c.side));
    SQF2K_CUDA(cudaMemsetAsync(acc->min_n, 0xff, sizeof acc->min_n, c.side));
    // the tile scheduler's words reset themselves (last CTA); also cleared per
    // call so an aborted launch cannot leak a stale state (off the critical path)
    if (!c.sched.ptr) {
        c.sched.reserve(64);
        SQF2K_CUDA(cudaMemset(c.sched.ptr, 0, 64));
    }
    SQF2K_CUDA(cudaMemsetAsync(c.sched.ptr, 0, 64, c.side));
    prep_tile_batch(a, c.profiling ? c.stream : c.side);  // (profile mode: one kernel at a time)
    generate_primes_async(pl.limit);
    a.primes = c.primes_u32.as<uint32_t>();  // (re)allocated by the generator
    a.info = c.prime_info.as<PrimeInfo>();
    join_side();
    // one fused batch at the default depth: the tile kernel's last CTA does
    // the (rare) escalations and writes the accumulators to pinned memory
    const bool finish_in_tile = pl.pipeline == 0 && pl.n_slots <= pl.batch && pl.default_depth;
    // several fused batches with fixed-capacity lists: batch b's pattern and
    // bucket lists are built on the side stream (buffer set b & 1) while batch
    // b - 1's tile kernel runs on the main stream (its tail frees the SMs)
    static const bool no_overlap = std::getenv("SQF2K_NO_OVERLAP") != nullptr;  // A/B experiments
    // (profile mode runs the batches without the side-stream overlap: a side
    // kernel's events would otherwise time its wait for the SMs the tile
    // kernel holds, not the kernel)
    const bool overlap = pl.pipeline == 0 && !pl.exact && pl.n_slots > pl.batch && !no_overlap && !c.profiling;
    if (overlap) SQF2K_CUDA(cudaEventRecord(c.ev_primes, c.stream));
    uint64_t b = 0;
    for (uint64_t s0 = 0; s0 < pl.n_slots; s0 += pl.batch, ++b) {
        const auto [A, sb] = set_batch(s0);
        a.finish_acc = finish_in_tile ? acc : nullptr;
        a.finish_host = c.pinned;
        if (overlap) {
            a.buf = (int)(b & 1);
            a.bucket_stream = c.side;
            if (b) {
                if (b >= 2) SQF2K_CUDA(cudaStreamWaitEvent(c.side, c.ev_tile[b & 1], 0));
                prep_tile_batch(a, c.side);  // buffer set b & 1 is free again
            } else {
                SQF2K_CUDA(cudaStreamWaitEvent(c.side, c.ev_primes, 0));
            }
            bucket_batch(a, c.side);
            SQF2K_CUDA(cudaEventRecord(c.ev_prep, c.side));
            SQF2K_CUDA(cudaStreamWaitEvent(c.stream, c.ev_prep, 0));
            run_tile_batch(a);
            SQF2K_CUDA(cudaEventRecord(c.ev_tile[b & 1], c.stream));
            continue;
        }
        if (s0) prep_tile_batch(a, c.stream);
        run_tile_batch(a);
        if (pl.pipeline == 1)
            scan_bitmap_device(c.window.as<uint32_t>(), H / 32, sb, A, pl.k_eff, pl.k_max,
                               A == 1 ? 0 : ~0ull, acc->hist, acc->min_n, a.esc, a.esc_count,
                               pl.esc_cap, a.fail, a.fail_count, pl.dev_fail_cap, a.scanned);
    }
    if (finish_in_tile) {
        c.d2h_bytes += sizeof(Acc);  // written to mapped host memory by the kernel
        return;
    }
    if (pl.k_max > pl.k_eff)
        launch("escalate", escalate_kernel, dim3(warp_grid(pl.esc_cap)), dim3(256), 0,
               (const unsigned long long *)a.esc, (const unsigned long long *)a.esc_count,
               pl.esc_cap, pl.k_eff + 1, pl.k_max, a.primes, a.info, acc->hist, acc->min_n,
               a.fail, a.fail_count, pl.dev_fail_cap);
    copy_d2h(c.pinned, acc, sizeof(Acc));
}

// Replay cache: the launch sequence of a call is a pure function of its
// arguments, so it is captured once into a CUDA graph and replayed (every
// kernel still runs on every call; only the CPU launch cost goes away).
// Entries die whenever a device buffer is reallocated.
struct GraphEntry {
    uint64_t key[8];
    uint64_t gen;
    uint64_t h2d, d2h;  // copy accounting of one call
    cudaGraphExec_t exec;
};
std::vector<GraphEntry> g_graphs;

bool graphs_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("SQF2K_NO_GRAPHS");
        return !(e && *e && *e != '0');
    }();
    return on && !ctx().profiling;
}

void plan_key(const VerifyPlan &pl, uint64_t key[8]) {
    key[0] = pl.start;
    key[1] = pl.end;
    key[2] = pl.k_max | ((uint64_t)pl.k_eff << 8) | ((uint64_t)pl.pipeline << 16) |
             ((uint64_t)pl.exact << 24) | ((uint64_t)pl.default_depth << 32);
    key[3] = pl.batch;
    key[4] = pl.esc_cap;
    key[5] = pl.dev_fail_cap;
    key[6] = pl.H;
    // the tile grid is read from SQF2K_DEBUG_GRID at enqueue time: a replayed
    // graph must have been captured under the same cap
    const char *g = std::getenv("SQF2K_DEBUG_GRID");
    key[7] = g ? (uint64_t)std::max(1, atoi(g)) : 0;
}

GraphEntry *find_graph(const uint64_t key[8]) {
    for (auto &g : g_graphs)
        if (g.gen == dev_alloc_generation() && std::memcmp(g.key, key, sizeof g.key) == 0) return &g;
    return nullptr;
}

void capture_graph(const VerifyPlan &pl, const uint64_t key[8]) {
    Context &c = ctx();
    const uint64_t gen = dev_alloc_generation(), h2d = c.h2d_bytes, d2h = c.d2h_bytes;
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    bool ok = true;
    try {
        enqueue_verify(pl);
    } catch (const Error &) {
        ok = false;
    }
    if (cudaStreamEndCapture(c.stream, &graph) != cudaSuccess) ok = false;
    cudaGetLastError();
    GraphEntry e;
    std::memcpy(e.key, key, sizeof e.key);
    e.gen = gen;
    e.h2d = c.h2d_bytes - h2d;
    e.d2h = c.d2h_bytes - d2h;
    c.h2d_bytes = h2d;  // capturing copied nothing
    c.d2h_bytes = d2h;
    if (ok && graph && dev_alloc_generation() == gen &&
        cudaGraphInstantiate(&e.exec, graph,
                             SQF2K_PRIORITY ? cudaGraphInstantiateFlagUseNodePriority : 0) ==
            cudaSuccess) {
        for (auto &g : g_graphs)
            if (g.gen != gen) cudaGraphExecDestroy(g.exec);
        g_graphs.erase(std::remove_if(g_graphs.begin(), g_graphs.end(),
                                      [gen](const GraphEntry &g) { return g.gen != gen; }),
                       g_graphs.end());
        if (g_graphs.size() >= 16) {
            cudaGraphExecDestroy(g_graphs.front().exec);
            g_graphs.erase(g_graphs.begin());
        }
        g_graphs.push_back(e);
    }
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
}

// The verify driver: batches of independent sub-ranges, one host sync.
int verify_range(uint64_t start, uint64_t end, uint32_t k_max, const sqf2k_verify_opts_t &o,
                 sqf2k_summary_t *out, uint64_t *failures, uint64_t fail_cap) {
    Context &c = ctx();
    if (o.tile_depth > (uint32_t)kDepthMax)
        return fail(SQF2K_EINVAL, "tile_depth must be in 1..%d", kDepthMax);
    const uint32_t depth = o.tile_depth ? o.tile_depth : (uint32_t)kDepthDefault;
    VerifyPlan pl;
    pl.start = start;
    pl.end = end;
    pl.k_max = k_max;
    pl.k_eff = std::min(k_max, depth);
    pl.default_depth = o.tile_depth == 0;
    pl.H = std::max<uint32_t>(1024u, 1u << (pl.k_eff - 1));
    pl.batch = std::max<uint64_t>(o.batch_slots ? o.batch_slots : kDefaultBatch, (uint64_t)kTile);
    pl.n_slots = (end - start) / 2;
    pl.limit = isqrt_u64(end - 1);
    pl.pipeline = o.pipeline;
    pl.small = small_set_upto(pl.limit, pl.n_slots,
                              pl.pipeline == 0 && pl.k_eff >= (uint32_t)kMainMax && pl.batch % 128 == 0);
    pl.esc_cap = 1 << 16;
    pl.dev_fail_cap = std::max<uint64_t>(fail_cap, 1 << 12);
    pl.exact = (o.flags & SQF2K_EXACT_BUCKETS) != 0;
    const uint64_t n_slots = pl.n_slots;

    for (int attempt = 0; attempt < 5; ++attempt) {
        uint64_t key[8];
        plan_key(pl, key);
        const bool graphs = graphs_enabled();
        GraphEntry *g = graphs ? find_graph(key) : nullptr;
        if (g) {
            SQF2K_CUDA(cudaGraphLaunch(g->exec, c.stream));
            c.primes_limit = pl.limit;  // the replay rebuilt this call's table
            c.h2d_bytes += g->h2d;
            c.d2h_bytes += g->d2h;
        } else {
            enqueue_verify(pl);
        }
        SQF2K_CUDA(cudaStreamSynchronize(c.stream));
        const Acc h = *static_cast<const Acc *>(c.pinned);
        if (h.overflow) {  // a bucket list outgrew its fixed capacity: exact lists
            pl.exact = true;
            continue;
        }
        if (h.esc_count > pl.esc_cap) {  // rerun with room for every escalation
            pl.esc_cap = h.esc_count + 1024;
            continue;
        }
        if (h.fail_count > pl.dev_fail_cap && h.fail_count <= fail_cap) {
            pl.dev_fail_cap = h.fail_count + 1024;
            continue;
        }
        if (graphs && !g) capture_graph(pl, key);  // replay the next identical call
        std::memset(out, 0, sizeof *out);
        out->start = start;
        out->end = end;
        out->k_max = k_max;
        for (int k = 0; k < SQF2K_HIST_LEN; ++k) {
            out->hist[k] = h.hist[k];
            out->min_n[k] = h.min_n[k];
        }
        const uint64_t n_fail = h.fail_count;
        {
            // the kernels do not count k = 1: every scanned n is in exactly
            // one bucket k >= 1 or a failure (coverage checked)
            const uint64_t expect = n_slots - (start == 1 ? 1 : 0);
            if (h.scanned != expect)
                return fail(SQF2K_ECUDA, "scan coverage %llu != %llu odd n",
                            (unsigned long long)h.scanned, (unsigned long long)expect);
            uint64_t rest = n_fail;
            for (int k = 2; k < SQF2K_HIST_LEN; ++k) rest += out->hist[k];
            out->hist[1] = h.scanned - rest;
        }
        if (n_fail > fail_cap) {
            uint64_t none = SQF2K_NONE;
            finish_summary(out, &none, 0);
            out->n_failures = n_fail;
            return fail(SQF2K_ECAPACITY, "%llu failures exceed the buffer of %llu",
                        (unsigned long long)n_fail, (unsigned long long)fail_cap);
        }
        uint64_t smallest = SQF2K_NONE;
        deliver_failures(c.fail.as<unsigned long long>(), n_fail, failures, fail_cap, &smallest);
        finish_summary(out, &smallest, n_fail);
        return SQF2K_OK;
    }
    return fail(SQF2K_ECUDA, "verify did not converge on buffer sizes");
}

// sieve_segment: export mode over [start, end) with the caller's prime table.
int sieve_bits(uint64_t start, uint64_t end, const int64_t *primes_h, uint64_t n_primes_h,
               uint8_t *out, uint64_t nbytes) {
    Context &c = ctx();
    const uint64_t n_slots = (end - start) / 2;
    // only primes with p^2 <= end - 1 can clear a slot (sieve.py:97)
    const uint64_t root = isqrt_u64(end - 1);
    const uint64_t np = std::upper_bound(primes_h, primes_h + n_primes_h, (int64_t)root) - primes_h;
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
    // split of the caller's table (positions by value)
    PrimeInfo pi;
    std::memset(&pi, 0, sizeof pi);
    pi.count = np;
    pi.i_lo = (uint32_t)(std::lower_bound(primes_h, primes_h + np, (int64_t)kPMed) - primes_h);
    pi.i_hi = (uint32_t)np;
    for (int j = 0; j <= kClasses; ++j)
        pi.cls[j] = (uint32_t)(std::lower_bound(primes_h, primes_h + np, (int64_t)1 << (10 + j)) -
                               primes_h);
    c.prime_info.reserve(sizeof pi);
    copy_h2d(c.prime_info.ptr, &pi, sizeof pi);
    SmallSet small;
    for (uint64_t i = 0; i < pi.i_lo; ++i) {
        const uint32_t p = (uint32_t)primes_h[i];
        if (p == 3) small.present |= 1;
        else if (p == 5) small.present |= 2;
        else if (p == 7) small.present |= 4;
        else if (p == 11 && kPattern11 && n_slots >= kPattern11MinSlots) small.present |= 8;
        else if (p >= 11) small.med.push_back(p);
    }
    const uint32_t nt = (uint32_t)ceil_div(n_slots, kTile);
    c.bits_out.reserve((size_t)nt * kTile / 8 + 64);
    BatchArgs a;
    std::memset(&a, 0, sizeof a);
    a.fused = false;
    a.base_n = (int64_t)start;
    a.U = n_slots;
    a.one_u = ~0ull;
    a.k_eff = a.k_max = 1;
    a.primes = c.primes_u32.as<uint32_t>();
    a.info = c.prime_info.as<PrimeInfo>();
    a.n_primes_bound = np;
    a.pattern_present = small.present;
    a.med_primes = &small.med;
    a.bits_out = c.bits_out.as<uint32_t>();
    c.acc.reserve(sizeof(Acc));
    a.overflow = &c.acc.as<Acc>()->overflow;
    for (int attempt = 0; attempt < 2; ++attempt) {
        SQF2K_CUDA(cudaMemsetAsync(a.overflow, 0, sizeof(unsigned int), c.stream));
        a.exact_buckets = attempt > 0;
        prep_tile_batch(a, c.stream);
        run_tile_batch(a);
        unsigned int &ovf = *static_cast<unsigned int *>(c.pinned);
        copy_d2h(&ovf, a.overflow, sizeof ovf);
        SQF2K_CUDA(cudaStreamSynchronize(c.stream));
        if (!ovf) break;
    }
    copy_d2h(out, c.bits_out.ptr, nbytes);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    return SQF2K_OK;
}

int recheck(const uint64_t *n, uint64_t count, uint64_t prime_limit, int32_t *k_out) {
    Context &c = ctx();
    if (!count) return SQF2K_OK;
    ensure_primes(prime_limit);
    c.esc.reserve(count * 8);
    c.fail.reserve(count * 4);
    copy_h2d(c.esc.ptr, n, count * 8);
    launch("recheck", recheck_kernel, dim3(warp_grid(count)), dim3(256), 0,
           (const unsigned long long *)c.esc.ptr, count, (const uint32_t *)c.primes_u32.ptr,
           (const PrimeInfo *)c.prime_info.ptr, c.fail.as<int32_t>());
    copy_d2h(k_out, c.fail.ptr, count * 4);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    return SQF2K_OK;
}

int is_squarefree(const uint64_t *n, uint64_t count, uint64_t prime_limit, uint8_t *out) {
    Context &c = ctx();
    if (!count) return SQF2K_OK;
    ensure_primes(prime_limit);
    c.esc.reserve(count * 8);
    c.fail.reserve(count + 16);
    copy_h2d(c.esc.ptr, n, count * 8);
    launch("squarefree", squarefree_kernel, dim3(warp_grid(count)), dim3(256), 0,
           (const unsigned long long *)c.esc.ptr, count, (const uint32_t *)c.primes_u32.ptr,
           (const PrimeInfo *)c.prime_info.ptr, c.fail.as<uint8_t>());
    copy_d2h(out, c.fail.ptr, count);
    SQF2K_CUDA(cudaStreamSynchronize(c.stream));
    return SQF2K_OK;
}

}  // namespace sqf2k

using namespace sqf2k;

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
    if (o.batch_slots > kMaxBatch)
        return fail(SQF2K_EINVAL, "batch_slots must be at most 2^40, got %llu",
                    (unsigned long long)o.batch_slots);
    if (o.tile_depth > (uint32_t)kDepthMax)
        return fail(SQF2K_EINVAL, "tile_depth must be in 1..%d", kDepthMax);
    return guarded([&](Context &) -> int {
        return verify_range(start, end, k_max, o, out, failures, fail_cap);
    });
}

extern "C" int sqf2k_sieve_bits(uint64_t start, uint64_t end, const int64_t *primes,
                                uint64_t n_primes, uint8_t *out, uint64_t nbytes) {
    int rc = check_range(start, end);
    if (rc) return rc;
    const uint64_t n_slots = (end - start) / 2;
    if (nbytes != ceil_div(n_slots, 64) * 8)
        return fail(SQF2K_EINVAL, "output holds %llu bytes, segment needs %llu",
                    (unsigned long long)nbytes, (unsigned long long)(ceil_div(n_slots, 64) * 8));
    for (uint64_t i = 1; i < n_primes; ++i)
        if (primes[i] <= primes[i - 1])
            return fail(SQF2K_EINVAL, "prime table must be strictly increasing");
    return guarded([&](Context &) -> int {
        return sieve_bits(start, end, primes, n_primes, out, nbytes);
    });
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

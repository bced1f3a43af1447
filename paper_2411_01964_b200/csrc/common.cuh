// common.cuh -- runtime plumbing of libsqf2k_b200: error reporting across the
// C ABI, the per-process device context (one GPU, one stream), grow-only
// device buffers and event-bracketed kernel launches for profiling.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sqf2k_b200.h"

namespace sqf2k {

// ---- errors -----------------------------------------------------------------

struct Error {
    int code;
    std::string msg;
};

void set_error(int code, const char *fmt, ...);
int fail(int code, const char *fmt, ...);

#define SQF2K_CUDA(expr)                                                          \
    do {                                                                          \
        cudaError_t e_ = (expr);                                                  \
        if (e_ != cudaSuccess) {                                                  \
            int c_ = (e_ == cudaErrorMemoryAllocation) ? SQF2K_ENOMEM : SQF2K_ECUDA; \
            throw ::sqf2k::Error{c_, std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
        }                                                                         \
    } while (0)

// ---- device buffers -----------------------------------------------------------

// bumped whenever a device buffer is (re)allocated: captured graphs hold raw
// pointers and are only replayed within one generation
uint64_t dev_alloc_generation();
void dev_alloc_bump();  // contents of a shared table changed in place

struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    void reserve(size_t n);  // grow-only, contents not preserved
    void release();
    template <class T>
    T *as() const { return static_cast<T *>(ptr); }
};

// ---- context --------------------------------------------------------------------

struct KStat {
    std::string name;
    uint64_t launches = 0;
    double total_ms = 0.0;
};

struct Context {
    int device = -1;
    int sm_count = 0;
    size_t smem_optin = 0;
    cudaStream_t stream = nullptr;
    // side stream for work independent of the prime table (fork/join by events,
    // captured into the same graph as parallel branches)
    cudaStream_t side = nullptr;
    // launch priorities (SQF2K_PRIORITY=1): main-stream kernels outrank the
    // side stream's, so a ready tile kernel takes the SMs ahead of the next
    // batch's bucket fill (measured no different on C4: off by default)
    int prio_main = 0, prio_side = 0;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // multi-batch calls: batch b's bucket lists are built on the side stream
    // (buffer set b & 1) while batch b - 1's tile kernel runs
    cudaEvent_t ev_primes = nullptr, ev_prep = nullptr, ev_tile[2] = {nullptr, nullptr};
    std::recursive_mutex mu;

    // profiling: events recorded around launches, resolved lazily
    bool profiling = false;
    struct Pending {
        int stat;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    std::vector<KStat> stats;

    // named scratch buffers reused across calls
    DevBuf primes_u32, prime_bits, prime_counts, prime_offsets, scan_tmp;
    DevBuf residues, items, tile_counts, tile_offsets, hits;
    DevBuf acc, esc, fail, fail_sorted, window, kvals, bits_out, host_primes;
    DevBuf pattern, prime_info, sched;
    DevBuf pattern_b, tile_counts_b, hits_b;  // second buffer set (batch parity 1)
    DevBuf pattern13;                         // wheel table with 11 and 13 (tile.cuh)
    // present mask of the wheel table held by pattern (kind 0), pattern_b
    // (kind 1) and pattern13 (kind 2); ~0u: not built
    uint32_t wheel_present[3] = {~0u, ~0u, ~0u};
    void *pinned = nullptr;  // small pinned host staging (summary readback)
    uint64_t h2d_bytes = 0, d2h_bytes = 0;  // copy accounting (bench e2e)
    uint64_t primes_limit = 0;  // primes_u32 holds all primes <= primes_limit
    uint64_t primes_count = 0;

    int stat_index(const char *name);
    cudaEvent_t get_event();
    void resolve_profile();  // synchronises
};

Context &ctx();            // throws Error{SQF2K_ENODEV} if not initialised
Context *ctx_or_null();

#ifndef SQF2K_PRIORITY
#define SQF2K_PRIORITY 0
#endif

// Launch `kernel` on stream `st` (`pdl`: programmatic dependent launch -- the
// kernel may start while its stream predecessor is still running, once that
// grid triggers, and must execute griddepcontrol.wait before touching the
// predecessor's output), with the stream's priority as a launch attribute
// (kept by graph capture), bracketed by events when profiling.
template <class... KArgs, class... Args>
void launch_ex(cudaStream_t st, bool pdl, const char *name, void (*kernel)(KArgs...), dim3 grid,
               dim3 block, size_t smem, Args... args) {
    Context &c = ctx();
    cudaEvent_t a = nullptr, b = nullptr;
    if (c.profiling) {  // per-launch events would serialise PDL anyway
        a = c.get_event();
        b = c.get_event();
        SQF2K_CUDA(cudaEventRecord(a, st));
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    static const bool no_pdl = std::getenv("SQF2K_NO_PDL") != nullptr;  // A/B experiments
    if (pdl && !no_pdl) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n++].val.programmaticStreamSerializationAllowed = c.profiling ? 0 : 1;
    }
    if (SQF2K_PRIORITY) {
        attr[n].id = cudaLaunchAttributePriority;
        attr[n++].val.priority = st == c.side ? c.prio_side : c.prio_main;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
    if (e != cudaSuccess)  // (with CUDA_LAUNCH_BLOCKING=1: this kernel's own fault)
        throw Error{e == cudaErrorMemoryAllocation ? SQF2K_ENOMEM : SQF2K_ECUDA,
                    std::string("launch of ") + name + ": " + cudaGetErrorString(e)};
    if (c.profiling) {
        SQF2K_CUDA(cudaEventRecord(b, st));
        c.pending.push_back({c.stat_index(name), a, b});
    }
}

template <class... KArgs, class... Args>
void launch_on(cudaStream_t st, const char *name, void (*kernel)(KArgs...), dim3 grid, dim3 block,
               size_t smem, Args... args) {
    launch_ex(st, false, name, kernel, grid, block, smem, args...);
}

template <class... KArgs, class... Args>
void launch_pdl(const char *name, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                Args... args) {
    launch_ex(ctx().stream, true, name, kernel, grid, block, smem, args...);
}

// griddepcontrol (sm_90+): wait for the predecessor grid / let the dependent start
__device__ __forceinline__ void grid_dependency_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void grid_dependents_launch() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

// Launch `kernel` on the library stream.
template <class Kernel, class... Args>
void launch(const char *name, Kernel kernel, dim3 grid, dim3 block, size_t smem,
            Args... args) {
    launch_on(ctx().stream, name, kernel, grid, block, smem, args...);
}

// Fork the side stream off the library stream / join it back.
inline void fork_side() {
    Context &c = ctx();
    SQF2K_CUDA(cudaEventRecord(c.ev_fork, c.stream));
    SQF2K_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
}
inline void join_side() {
    Context &c = ctx();
    SQF2K_CUDA(cudaEventRecord(c.ev_join, c.side));
    SQF2K_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
}

// Counted host<->device copies on the library stream.
inline void copy_h2d(void *dst, const void *src, size_t n) {
    Context &c = ctx();
    SQF2K_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, c.stream));
    c.h2d_bytes += n;
}
inline void copy_d2h(void *dst, const void *src, size_t n) {
    Context &c = ctx();
    SQF2K_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, c.stream));
    c.d2h_bytes += n;
}

// Wrap an ABI body: maps exceptions to codes, holds the context lock.
template <class F>
int guarded(F &&body) {
    try {
        Context &c = ctx();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        return body(c);
    } catch (const Error &e) {
        set_error(e.code, "%s", e.msg.c_str());
        return e.code;
    } catch (const std::bad_alloc &) {
        set_error(SQF2K_ENOMEM, "host allocation failed");
        return SQF2K_ENOMEM;
    } catch (...) {
        set_error(SQF2K_ECUDA, "unexpected internal error");
        return SQF2K_ECUDA;
    }
}

// ---- small host helpers --------------------------------------------------------

__host__ __device__ static inline uint64_t isqrt_u64(uint64_t n) {
    uint64_t r = 0, bit = 1ULL << 62;
    while (bit > n) bit >>= 2;
    while (bit) {
        if (n >= r + bit) {
            n -= r + bit;
            r = (r >> 1) + bit;
        } else {
            r >>= 1;
        }
        bit >>= 2;
    }
    return r;
}

static inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Largest end the GPU path accepts: p <= 2^31 keeps p^2 < 2^62 in uint64.
constexpr uint64_t kMaxEnd = 1ULL << 62;

// GPU prime generator: every prime <= limit into ctx().primes_u32 and the
// PrimeInfo split into ctx().prime_info, without a host sync (async) or
// returning the count (sync).
void generate_primes_async(uint64_t limit);
void ensure_primes(uint64_t limit);
uint64_t generate_primes_device(uint64_t limit);
// Upper bound of pi(x) (Rosser-Schoenfeld), for buffer sizing without a sync.
uint64_t pi_upper(uint64_t x);

}  // namespace sqf2k

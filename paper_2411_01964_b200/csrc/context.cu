// context.cu -- error state, device context and profiling of libsqf2k_b200.
#include <cstring>

#include "common.cuh"

namespace sqf2k {

static thread_local std::string t_last_error = "no error";
static Context *g_ctx = nullptr;
static std::mutex g_init_mu;

void set_error(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    (void)code;
    t_last_error = buf;
}

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_last_error = buf;
    return code;
}

static uint64_t g_alloc_gen = 1;
uint64_t dev_alloc_generation() { return g_alloc_gen; }
void dev_alloc_bump() { ++g_alloc_gen; }

void DevBuf::reserve(size_t n) {
    if (n <= bytes) return;
    ++g_alloc_gen;
    release();
    size_t want = n < 256 ? 256 : n;
    cudaError_t e = cudaMalloc(&ptr, want);
    if (e != cudaSuccess) {
        ptr = nullptr;
        bytes = 0;
        cudaGetLastError();
        throw Error{SQF2K_ENOMEM, std::string("cudaMalloc(") + std::to_string(want) +
                                      " bytes): " + cudaGetErrorString(e)};
    }
    bytes = want;
}

void DevBuf::release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
}

int Context::stat_index(const char *name) {
    for (size_t i = 0; i < stats.size(); ++i)
        if (stats[i].name == name) return (int)i;
    stats.push_back(KStat{name, 0, 0.0});
    return (int)stats.size() - 1;
}

cudaEvent_t Context::get_event() {
    if (!event_pool.empty()) {
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    SQF2K_CUDA(cudaEventCreate(&e));
    return e;
}

void Context::resolve_profile() {
    if (pending.empty()) return;
    SQF2K_CUDA(cudaStreamSynchronize(stream));
    for (auto &p : pending) {
        float ms = 0.f;
        SQF2K_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        stats[p.stat].launches += 1;
        stats[p.stat].total_ms += ms;
        event_pool.push_back(p.a);
        event_pool.push_back(p.b);
    }
    pending.clear();
}

Context *ctx_or_null() { return g_ctx; }

Context &ctx() {
    if (!g_ctx) throw Error{SQF2K_ENODEV, "sqf2k_init() has not bound a CUDA device"};
    SQF2K_CUDA(cudaSetDevice(g_ctx->device));
    return *g_ctx;
}

}  // namespace sqf2k

using namespace sqf2k;

extern "C" {

int sqf2k_abi_version(void) { return SQF2K_ABI_VERSION; }

const char *sqf2k_last_error(void) { return t_last_error.c_str(); }

int sqf2k_device_count(int *count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *count = 0;
        return fail(SQF2K_ENODEV, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    *count = n;
    return SQF2K_OK;
}

int sqf2k_init(int device) {
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (g_ctx && g_ctx->device == device) return SQF2K_OK;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(SQF2K_ENODEV, "no CUDA device visible (%s)",
                    e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
    }
    if (device < 0 || device >= n)
        return fail(SQF2K_EINVAL, "device %d out of range (%d visible)", device, n);
    if (g_ctx) {
        return fail(SQF2K_EINVAL, "library already bound to device %d; call sqf2k_shutdown first",
                    g_ctx->device);
    }
    cudaDeviceProp prop;
    if ((e = cudaSetDevice(device)) != cudaSuccess ||
        (e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) {
        cudaGetLastError();
        return fail(SQF2K_ECUDA, "device %d: %s", device, cudaGetErrorString(e));
    }
    if (prop.major != 10)
        return fail(SQF2K_ENODEV, "device %d is sm_%d%d; this library is built for sm_100a (B200)",
                    device, prop.major, prop.minor);
    Context *c = new Context();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    cudaDeviceGetStreamPriorityRange(&c->prio_side, &c->prio_main);  // (least, greatest)
    if (!SQF2K_PRIORITY) c->prio_side = c->prio_main = 0;
    if ((e = cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, c->prio_main)) !=
        cudaSuccess) {
        delete c;
        return fail(SQF2K_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    if ((e = cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, c->prio_side)) !=
            cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_primes, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_prep, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_tile[0], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_tile[1], cudaEventDisableTiming)) != cudaSuccess) {
        cudaStreamDestroy(c->stream);
        delete c;
        return fail(SQF2K_ECUDA, "side stream: %s", cudaGetErrorString(e));
    }
    if ((e = cudaMallocHost(&c->pinned, 1 << 16)) != cudaSuccess) {
        cudaStreamDestroy(c->stream);
        delete c;
        return fail(SQF2K_ECUDA, "cudaMallocHost: %s", cudaGetErrorString(e));
    }
    g_ctx = c;
    return SQF2K_OK;
}

void sqf2k_shutdown(void) {
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (!g_ctx) return;
    Context *c = g_ctx;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (DevBuf *b : {&c->primes_u32, &c->prime_bits, &c->prime_counts, &c->prime_offsets,
                      &c->scan_tmp, &c->residues, &c->items, &c->tile_counts,
                      &c->tile_offsets, &c->hits, &c->acc, &c->esc,
                      &c->fail, &c->fail_sorted, &c->window, &c->kvals, &c->bits_out,
                      &c->host_primes, &c->pattern, &c->prime_info, &c->sched,
                      &c->pattern_b, &c->tile_counts_b, &c->hits_b})
        b->release();
    if (c->pinned) cudaFreeHost(c->pinned);
    for (auto &p : c->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    cudaStreamSynchronize(c->side);
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
    for (cudaEvent_t ev : {c->ev_primes, c->ev_prep, c->ev_tile[0], c->ev_tile[1]}) cudaEventDestroy(ev);
    cudaStreamDestroy(c->side);
    cudaStreamDestroy(c->stream);
    delete c;
    g_ctx = nullptr;
}

int sqf2k_sync(void) {
    return guarded([](Context &c) -> int {
        SQF2K_CUDA(cudaStreamSynchronize(c.stream));
        return SQF2K_OK;
    });
}

int sqf2k_profile_enable(int on) {
    return guarded([on](Context &c) -> int {
        c.profiling = on != 0;
        return SQF2K_OK;
    });
}

void *sqf2k_stream(void) {
    Context *c = ctx_or_null();
    return c ? (void *)c->stream : nullptr;
}

int sqf2k_copy_stats(uint64_t *h2d_bytes, uint64_t *d2h_bytes) {
    return guarded([=](Context &c) -> int {
        *h2d_bytes = c.h2d_bytes;
        *d2h_bytes = c.d2h_bytes;
        return SQF2K_OK;
    });
}

int sqf2k_profile_reset(void) {
    return guarded([](Context &c) -> int {
        c.resolve_profile();
        c.stats.clear();
        c.h2d_bytes = c.d2h_bytes = 0;
        return SQF2K_OK;
    });
}

int sqf2k_profile_read(sqf2k_kstat_t *out, int cap, int *n) {
    return guarded([=](Context &c) -> int {
        c.resolve_profile();
        int m = 0;
        for (auto &s : c.stats) {
            if (m < cap) {
                std::memset(out[m].name, 0, sizeof out[m].name);
                std::strncpy(out[m].name, s.name.c_str(), sizeof out[m].name - 1);
                out[m].launches = s.launches;
                out[m].total_ms = s.total_ms;
            }
            ++m;
        }
        *n = m;
        return SQF2K_OK;
    });
}

}  // extern "C"

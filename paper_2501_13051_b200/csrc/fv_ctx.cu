// Per-GPU context: stream, stream-ordered memory pool, look-back scratch.
// Replaces the reference's Executor (P/include/colog/parallel.hpp:19-73):
// where the reference hands every operator a TBB arena, every operator here
// receives the context whose stream orders all of its kernels.
#include "fv_common.cuh"

#include <cstdio>
#include <cstdlib>

namespace fv {

namespace {
constexpr u32 kMaxCounters = 4096;
constexpr u32 kMaxEpoch = (1u << 20) - 1;
}  // namespace

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%d) at %s:%d: %s", cudaGetErrorString(e),
                  static_cast<int>(e), file, line, what);
    (void)cudaGetLastError();  // clear sticky-free errors
    throw Error(e == cudaErrorMemoryAllocation ? FV_ERR_OOM : FV_ERR_CUDA, buf);
}

void Ctx::activate() const { FV_CUDA(cudaSetDevice(device)); }

void* Ctx::alloc(size_t bytes) {
    void* p = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, stream);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        // Give cached blocks back and retry once before reporting OOM.
        FV_CUDA(cudaStreamSynchronize(stream));
        FV_CUDA(cudaMemPoolTrimTo(pool, 0));
        ++pool_trims;
        e = cudaMallocFromPoolAsync(&p, bytes, pool, stream);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            char buf[128];
            std::snprintf(buf, sizeof buf, "device allocation of %zu bytes failed", bytes);
            throw Error(FV_ERR_OOM, buf);
        }
    }
    return p;
}

void Ctx::reserve(size_t bytes) {
    u64 have = 0;
    FV_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &have));
    if (have >= bytes) return;
    void* p = alloc(bytes - have);
    release(p);
    sync();
}

void Ctx::release(void* p) {
    if (p) cudaFreeAsync(p, stream);
}

namespace {
// FVLOG_TRACE_SYNCS=1: name the function behind every host round trip.
const bool g_trace_syncs = std::getenv("FVLOG_TRACE_SYNCS") != nullptr;
}  // namespace

void Ctx::sync(const char* who) {
    ++syncs;
    if (g_trace_syncs) std::fprintf(stderr, "[sync] %s\n", who);
    FV_CUDA(cudaStreamSynchronize(stream));
    if (!prof_pending.empty()) prof_flush();
}

cudaEvent_t Ctx::prof_begin() {
    cudaEvent_t e;
    if (prof_events.empty()) {
        FV_CUDA(cudaEventCreate(&e));
    } else {
        e = prof_events.back();
        prof_events.pop_back();
    }
    FV_CUDA(cudaEventRecord(e, stream));
    return e;
}

void Ctx::prof_end(const char* name, cudaEvent_t a, double bytes) {
    cudaEvent_t b;
    if (prof_events.empty()) {
        FV_CUDA(cudaEventCreate(&b));
    } else {
        b = prof_events.back();
        prof_events.pop_back();
    }
    FV_CUDA(cudaEventRecord(b, stream));
    prof_pending.push_back({name, a, b, bytes});
}

void Ctx::prof_flush() {
    for (auto& r : prof_pending) {
        float ms = 0.f;
        FV_CUDA(cudaEventSynchronize(r.b));
        FV_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        ProfAgg* agg = nullptr;
        for (auto& [n, a] : prof_agg)
            if (n == r.name) agg = &a;
        if (!agg) {
            prof_agg.emplace_back(r.name, ProfAgg{});
            agg = &prof_agg.back().second;
        }
        agg->launches += 1;
        agg->ms += ms;
        agg->bytes += r.bytes;
        prof_events.push_back(r.a);
        prof_events.push_back(r.b);
    }
    prof_pending.clear();
}

u32 Ctx::lookback_epoch(u64 words, u32** tile_counter) {
    if (words > lb.capacity) {
        if (lb.status) release(lb.status);
        u64 cap = words < (1u << 16) ? (1u << 16) : words + words / 2;
        lb.status = static_cast<u64*>(alloc(cap * sizeof(u64)));
        FV_CUDA(cudaMemsetAsync(lb.status, 0, cap * sizeof(u64), stream));
        lb.capacity = cap;
        lb.epoch = 0;
    }
    if (lb.epoch >= kMaxEpoch) {
        FV_CUDA(cudaMemsetAsync(lb.status, 0, lb.capacity * sizeof(u64), stream));
        lb.epoch = 0;
    }
    ++lb.epoch;
    if (counter_next == kMaxCounters) {
        FV_CUDA(cudaMemsetAsync(lb.counters, 0, kMaxCounters * sizeof(u32), stream));
        counter_next = 0;
    }
    *tile_counter = lb.counters + counter_next++;
    return lb.epoch;
}

void Ctx::read_scalars(const u64* d, u64* h, int n, const char* who) {
    ++syncs;
    if (g_trace_syncs) std::fprintf(stderr, "[sync] %s\n", who);
    FV_CUDA(cudaMemcpyAsync(pinned, d, sizeof(u64) * n, cudaMemcpyDeviceToHost, stream));
    FV_CUDA(cudaStreamSynchronize(stream));
    std::memcpy(h, pinned, sizeof(u64) * n);
    if (!prof_pending.empty()) prof_flush();
}

Ctx* ctx_new(int device) {
    int count = 0;
    FV_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
        fail(FV_ERR_RANGE, "fv_ctx_create: no CUDA device " + std::to_string(device));
    Ctx* c = new Ctx();
    c->device = device;
    try {
        c->activate();
        cudaDeviceProp prop{};
        FV_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            fail(FV_ERR_CUDA, std::string("fvlog is built for sm_100a (Blackwell); device is ") +
                                  prop.name);
        FV_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        FV_CUDA(cudaDeviceGetDefaultMemPool(&c->pool, device));
        // Keep freed blocks cached in the pool: relations are rebuilt every
        // iteration and must not pay cudaMalloc each time.
        u64 threshold = ~u64(0);
        FV_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &threshold));
        FV_CUDA(cudaMallocHost(&c->pinned, 64 * sizeof(u64)));
        c->lb.counters = static_cast<u32*>(c->alloc(kMaxCounters * sizeof(u32)));
        FV_CUDA(cudaMemsetAsync(c->lb.counters, 0, kMaxCounters * sizeof(u32), c->stream));
        c->d_scalars = static_cast<u64*>(c->alloc(64 * sizeof(u64)));
        FV_CUDA(cudaMemsetAsync(c->d_scalars, 0, 64 * sizeof(u64), c->stream));
        c->sync();
    } catch (...) {
        ctx_delete(c);
        throw;
    }
    return c;
}

void ctx_delete(Ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->lb.status) cudaFreeAsync(c->lb.status, c->stream);
    if (c->lb.counters) cudaFreeAsync(c->lb.counters, c->stream);
    if (c->d_scalars) cudaFreeAsync(c->d_scalars, c->stream);
    if (c->stream) {
        cudaStreamSynchronize(c->stream);
        cudaStreamDestroy(c->stream);
    }
    if (c->pinned) cudaFreeHost(c->pinned);
    for (auto& r : c->prof_pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : c->prof_events) cudaEventDestroy(e);
    delete c;
}

}  // namespace fv

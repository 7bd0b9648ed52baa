// Shared device/host plumbing for the fvlog sm_100a runtime.
//
// The reference's only runtime substrate is the TBB Executor
// (P/include/colog/parallel.hpp:19-73). Here it becomes a per-GPU context
// (one CUDA stream, a stream-ordered memory pool sized for HBM residency)
// plus the single-pass decoupled look-back machinery every scan, compaction
// and radix pass in this library is built on.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fvlog.h"

namespace fv {

using u8 = std::uint8_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;

// ---- errors --------------------------------------------------------------

struct Error : std::runtime_error {
    fv_status status;
    Error(fv_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define FV_CUDA(x)                                                              \
    do {                                                                        \
        cudaError_t fv_e_ = (x);                                                \
        if (fv_e_ != cudaSuccess) ::fv::throw_cuda(fv_e_, #x, __FILE__, __LINE__); \
    } while (0)

[[noreturn]] inline void fail(fv_status s, const std::string& m) { throw Error(s, m); }

// ---- context -------------------------------------------------------------

struct Ctx;

// Scratch for decoupled look-back: one u64 status word per (tile, lane-slot).
// Words carry [epoch:20 | flag:2 | value:42]; a word is only valid when its
// epoch matches the launch's epoch, so the array never needs clearing
// between launches (it is zeroed only when the epoch counter wraps).
struct LookbackPool {
    u64* status = nullptr;
    u64 capacity = 0;  // words
    u32* counters = nullptr; // dynamic tile counters, kMaxCounters
    u32 epoch = 0;
};

// Per-kernel-class timing with CUDA events on the launching stream (enabled
// by fv_ctx_profile; used by bench.py for the live roofline numbers).
struct ProfAgg {
    u64 launches = 0;
    double ms = 0.0;
    double bytes = 0.0;  // algorithmic bytes (implementation-independent)
};

class Transport;

struct Ctx {
    int device = 0;
    // Row exchange with the other ranks of a partitioned evaluation
    // (transport.h); null for a single-GPU evaluation. Not owned.
    Transport* tx = nullptr;
    bool prof = false;
    struct ProfRec {
        const char* name;
        cudaEvent_t a, b;
        double bytes;
    };
    std::vector<ProfRec> prof_pending;
    std::vector<cudaEvent_t> prof_events;
    std::vector<std::pair<std::string, ProfAgg>> prof_agg;
    cudaEvent_t prof_begin();
    void prof_end(const char* name, cudaEvent_t a, double bytes);
    void prof_flush();  // after a stream sync
    void prof_add_bytes(const char* name, double bytes) {
        if (!prof) return;
        prof_flush();
        for (auto& [n, a] : prof_agg)
            if (n == name) a.bytes += bytes;
    }
    cudaStream_t stream = nullptr;
    cudaMemPool_t pool = nullptr;
    std::string last_error;
    u64 launches = 0;
    u64 syncs = 0;  // host synchronisations (sync / read_scalars): the per-iteration host round trips
    LookbackPool lb;
    u64* pinned = nullptr; // small pinned host buffer for scalar readbacks
    u64* d_scalars = nullptr; // device scalar slots
    u32 counter_next = 0;
    u64 pool_trims = 0;       // allocation retries after trimming the pool

    void* alloc(size_t bytes);
    void reserve(size_t bytes);  // pre-map pool memory (fv_ctx_reserve)
    void release(void* p);
    void activate() const;  // cudaSetDevice
    void sync(const char* who = __builtin_FUNCTION());
    // Reserve `words` look-back status words and a fresh epoch; returns the
    // epoch to pass to the kernel. Also hands out a zeroed tile counter.
    u32 lookback_epoch(u64 words, u32** tile_counter);
    // Copy n u64 device scalars to host (one synchronisation).
    void read_scalars(const u64* d, u64* h, int n, const char* who = __builtin_FUNCTION());
    void count_launch(int n = 1) { launches += n; }
};

Ctx* ctx_new(int device);
void ctx_delete(Ctx* c);

// RAII timing of one kernel launch (no-op unless profiling is enabled).
class ProfScope {
public:
    ProfScope(Ctx* c, const char* name, double bytes) : c_(c), name_(name), bytes_(bytes) {
        if (c_->prof) a_ = c_->prof_begin();
    }
    ~ProfScope() {
        if (c_->prof && a_) c_->prof_end(name_, a_, bytes_);
    }
    ProfScope(const ProfScope&) = delete;
    ProfScope& operator=(const ProfScope&) = delete;

private:
    Ctx* c_;
    const char* name_;
    double bytes_;
    cudaEvent_t a_ = nullptr;
};

// ---- device buffers ------------------------------------------------------

template <typename T>
class DBuf {
public:
    DBuf() = default;
    DBuf(Ctx* c, u64 n) : ctx_(c), n_(n) {
        if (n) p_ = static_cast<T*>(c->alloc(sizeof(T) * n));
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept { swap(o); }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            reset();
            swap(o);
        }
        return *this;
    }
    ~DBuf() { reset(); }

    void reset() {
        if (p_ && ctx_) ctx_->release(p_);
        p_ = nullptr;
        n_ = 0;
    }
    void swap(DBuf& o) noexcept {
        std::swap(ctx_, o.ctx_);
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
    }
    // Drop ownership semantics for a size change without reallocation.
    void set_size(u64 n) { n_ = n; }
    // Hand the allocation to another owner (e.g. a differently typed DBuf).
    T* release() {
        T* p = p_;
        p_ = nullptr;
        n_ = 0;
        return p;
    }
    static DBuf adopt(Ctx* c, T* p, u64 n) {
        DBuf b;
        b.ctx_ = c;
        b.p_ = p;
        b.n_ = n;
        return b;
    }

    T* get() const { return p_; }
    u64 size() const { return n_; }
    Ctx* ctx() const { return ctx_; }

    void upload(const T* h, u64 n, u64 offset = 0) {
        if (n) FV_CUDA(cudaMemcpyAsync(p_ + offset, h, sizeof(T) * n, cudaMemcpyHostToDevice, ctx_->stream));
    }
    void download(T* h, u64 n, u64 offset = 0, const char* who = __builtin_FUNCTION()) const {
        if (n) {
            FV_CUDA(cudaMemcpyAsync(h, p_ + offset, sizeof(T) * n, cudaMemcpyDeviceToHost, ctx_->stream));
            ctx_->sync(who);  // counted as a host round trip
        }
    }

private:
    Ctx* ctx_ = nullptr;
    T* p_ = nullptr;
    u64 n_ = 0;
};

template <typename T>
DBuf<T> make_dbuf(Ctx* c, const T* h, u64 n) {
    DBuf<T> b(c, n);
    b.upload(h, n);
    return b;
}

#ifdef __CUDACC__
#define FV_HD __host__ __device__
#else
#define FV_HD
#endif

FV_HD inline u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

// ---- device helpers ------------------------------------------------------

#ifdef __CUDACC__

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ u32 lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ u64 ld_relaxed_u64(const u64* p) {
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(u64* p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Look-back status words.
constexpr u64 kLbFlagAggregate = 1;
constexpr u64 kLbFlagInclusive = 2;
constexpr int kLbValueBits = 42;
constexpr u64 kLbValueMask = (u64(1) << kLbValueBits) - 1;

__device__ __forceinline__ u64 lb_pack(u32 epoch, u64 flag, u64 value) {
    return (u64(epoch) << 44) | (flag << 42) | (value & kLbValueMask);
}
__device__ __forceinline__ bool lb_valid(u64 w, u32 epoch) { return (w >> 44) == epoch; }
__device__ __forceinline__ u64 lb_flag(u64 w) { return (w >> 42) & 3; }
__device__ __forceinline__ u64 lb_value(u64 w) { return w & kLbValueMask; }

// Scalar look-back by one thread: sum of predecessors' values at
// status[(t) * stride + slot] for t < tile, stopping at the first inclusive.
__device__ __forceinline__ u64 lookback_thread(const u64* status, u32 tile, u32 stride, u32 slot,
                                               u32 epoch) {
    u64 excl = 0;
    long long t = static_cast<long long>(tile) - 1;
    while (t >= 0) {
        u64 w;
        do {
            w = ld_relaxed_u64(status + u64(t) * stride + slot);
        } while (!lb_valid(w, epoch));
        excl += lb_value(w);
        if (lb_flag(w) == kLbFlagInclusive) break;
        --t;
    }
    return excl;
}

// lookback_thread with Q predecessors' words loaded per round (independent
// loads; with slot = the thread's lane-contiguous index each round is one
// coalesced row per warp), consumed newest first up to the first inclusive.
template <int Q>
__device__ __forceinline__ u64 lookback_thread_deep(const u64* status, u32 tile, u32 stride, u32 slot,
                                                    u32 epoch) {
    u64 excl = 0;
    long long t = static_cast<long long>(tile) - 1;
    while (t >= 0) {
        u64 w[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q)
            w[q] = t - q >= 0 ? ld_relaxed_u64(status + u64(t - q) * stride + slot) : lb_pack(epoch, kLbFlagInclusive, 0);
        bool done = false;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (done) break;
            while (!lb_valid(w[q], epoch)) {
#ifdef FV_LB_SLEEP
                __nanosleep(FV_LB_SLEEP);
#endif
                w[q] = ld_relaxed_u64(status + u64(t - q) * stride + slot);
            }
            excl += lb_value(w[q]);
            done = lb_flag(w[q]) == kLbFlagInclusive;
        }
        if (done) break;
        t -= Q;
    }
    return excl;
}

// Warp-cooperative look-back (lane-parallel window of 32 predecessors);
// call from all lanes of one warp; returns the exclusive prefix in every lane.
__device__ __forceinline__ u64 lookback_warp(const u64* status, u32 tile, u32 epoch) {
    u64 excl = 0;
    long long window_end = static_cast<long long>(tile) - 1;  // newest predecessor
    const u32 lane = lane_id();
    while (window_end >= 0) {
        long long t = window_end - lane;
        u64 w = 0;
        if (t >= 0) {
            do {
                w = ld_relaxed_u64(status + t);
            } while (!lb_valid(w, epoch));
        }
        const bool incl = t >= 0 && lb_flag(w) == kLbFlagInclusive;
        const u32 incl_mask = __ballot_sync(0xffffffffu, incl);
        // Lanes up to and including the nearest inclusive one contribute.
        u32 limit = incl_mask ? (__ffs(incl_mask) - 1) : 31;
        u64 v = (t >= 0 && lane <= limit) ? lb_value(w) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (incl_mask) break;
        window_end -= 32;
    }
    return excl;
}

// splitmix64 finalizer: the fingerprint/hash mixer shared by host and device.
__host__ __device__ __forceinline__ u64 mix64(u64 z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ u32 hash32(u32 k) {
    k ^= k >> 16;
    k *= 0x85ebca6bu;
    k ^= k >> 13;
    k *= 0xc2b2ae35u;
    k ^= k >> 16;
    return k;
}

#endif  // __CUDACC__

}  // namespace fv

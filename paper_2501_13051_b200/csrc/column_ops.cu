#include <cstdio>
#include <cstdlib>
// Column-store operators on sm_100a: the device implementations behind the
// operator-level C ABI (P/src/column.cpp, P/src/relation.cpp,
// P/src/kernels.cpp). Orders reproduce the reference wherever its tests pin
// them (SURVEY.md §8b "Order contract"):
//   build_index   ties ascending by id        (stable LSD from iota)
//   column_join   probe-major, sorted_idx order within a probe row
//                 (output-partitioned expansion, Algorithm 1)
//   dedup_rows    first-occurrence order      (min id per group, re-sorted)
//   filters / difference / select_eq preserve input order (look-back scans)
#include <atomic>

#include "column.h"
#include "prim.cuh"
#include "radix_sort.h"

namespace fv {

namespace {

std::atomic<u64> g_gather_volume{0};

unsigned grid_for(u64 n, int block = 256) {
    const u64 want = ceil_div(n, block);
    const u64 cap = u64(kNumSMs) * 16;
    return static_cast<unsigned>(want == 0 ? 1 : (want < cap ? want : cap));
}

#define GRID_STRIDE(i, n) \
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); i += u64(gridDim.x) * blockDim.x)

// ---- unique index ----------------------------------------------------------

struct RleOp {
    const u32* keys;  // sorted
    u32* ukeys;
    u32* ustart;
    __device__ u64 value(u64 i) const { return (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0; }
    __device__ void emit(u64 i, u64 p, u64 v) const {
        if (v) {
            ukeys[p] = keys[i];
            ustart[p] = static_cast<u32>(i);
        }
    }
};

__global__ void rle_counts_kernel(const u32* __restrict__ ustart, u32* __restrict__ ucount, u64 nu,
                                  u64 n) {
    GRID_STRIDE(i, nu) {
        const u64 end = i + 1 < nu ? ustart[i + 1] : n;
        ucount[i] = static_cast<u32>(end - ustart[i]);
    }
}

__global__ void hash_insert_kernel(const u32* __restrict__ ukeys, u64 nu,
                                   unsigned long long* __restrict__ slots, u32 mask) {
    GRID_STRIDE(i, nu) {
        const u32 key = ukeys[i];
        const unsigned long long packed = (static_cast<unsigned long long>(key) << 32) | u32(i);
        u32 h = hash32(key) & mask;
        while (atomicCAS(slots + h, ~0ull, packed) != ~0ull) h = (h + 1) & mask;
    }
}

__device__ __forceinline__ bool ht_find(const u64* __restrict__ slots, u32 mask, u32 key,
                                        u32* idx) {
    u32 h = hash32(key) & mask;
    while (true) {
        const u64 s = slots[h];
        if (s == kEmptySlot) return false;
        if (static_cast<u32>(s >> 32) == key) {
            *idx = static_cast<u32>(s);
            return true;
        }
        h = (h + 1) & mask;
    }
}

__global__ void probe_kernel(const u64* __restrict__ slots, u32 mask, const u32* __restrict__ ustart,
                             const u32* __restrict__ ucount, const u32* __restrict__ values, u64 n,
                             u32* __restrict__ starts, u32* __restrict__ counts) {
    GRID_STRIDE(i, n) {
        u32 r;
        if (slots && ht_find(slots, mask, values[i], &r)) {
            starts[i] = ustart[r];
            counts[i] = ucount[r];
        } else {
            starts[i] = 0;
            counts[i] = 0;
        }
    }
}

// ---- joins ------------------------------------------------------------------

struct SelectMatchOp {
    const u32* starts;
    const u32* counts;
    u32* mstarts;
    u32* mcounts;
    u32* matched;
    __device__ u64 value(u64 i) const { return counts[i] ? 1 : 0; }
    __device__ void emit(u64 i, u64 p, u64 v) const {
        if (v) {
            matched[p] = static_cast<u32>(i);
            mstarts[p] = starts[i];
            mcounts[p] = counts[i];
        }
    }
};

__global__ void sum_u32_kernel(const u32* __restrict__ in, u64 n, unsigned long long* out) {
    unsigned long long s = 0;
    GRID_STRIDE(i, n) s += in[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane_id() == 0 && s) atomicAdd(out, s);
}

struct JoinWriteOp {
    const u32* mstarts;
    const u32* matched;
    const u32* sorted_idx;
    u32* a;
    u32* b;
    __device__ void emit(u64 o, u64 j, u64 rank) const {
        a[o] = matched[j];
        b[o] = sorted_idx[mstarts[j] + rank];
    }
};

// ---- filters -----------------------------------------------------------------

struct PairsEqOp {
    const u32* a;
    const u32* b;
    const u32* ra;
    const u32* rb;
    u32* oa;
    u32* ob;
    __device__ u64 value(u64 k) const { return ra[a[k]] == rb[b[k]] ? 1 : 0; }
    __device__ void emit(u64 k, u64 p, u64 v) const {
        if (v) {
            oa[p] = a[k];
            ob[p] = b[k];
        }
    }
};

struct NeqOp {
    const u32* x;
    const u32* y;
    u32* out;
    __device__ u64 value(u64 k) const { return x[k] != y[k] ? 1 : 0; }
    __device__ void emit(u64 k, u64 p, u64 v) const {
        if (v) out[p] = static_cast<u32>(k);
    }
};

// ---- dedup ---------------------------------------------------------------------

struct ColPtrs {
    const u32* p[FV_MAX_ARITY];
};

struct HeadsOp {
    ColPtrs cols;
    u32 arity;
    const u32* perm;
    u32* keep;
    __device__ u64 value(u64 i) const {
        if (i == 0) return 1;
        const u32 a = perm[i - 1], b = perm[i];
        for (u32 j = 0; j < arity; ++j)
            if (cols.p[j][a] != cols.p[j][b]) return 1;
        return 0;
    }
    __device__ void emit(u64 i, u64 p, u64 v) const {
        if (v && keep) keep[p] = perm[i];
    }
};

// Algorithm 2 marking loop (P/src/kernels.cpp:185-206, 232-254): a row of NEW
// is in FULL iff its per-column id runs (ascending sorted_idx slices) share
// an id. Rows with a missing column value are dropped without intersecting.
struct RunsArgs {
    const u32* sorted[FV_MAX_ARITY];
    const u32* starts[FV_MAX_ARITY];
    const u32* counts[FV_MAX_ARITY];
};

__global__ void runs_intersect_kernel(RunsArgs args, u32 arity, u64 n, u8* __restrict__ flags) {
    GRID_STRIDE(i, n) {
        u32 pos[FV_MAX_ARITY];
        u32 len[FV_MAX_ARITY];
        const u32* run[FV_MAX_ARITY];
        bool hit = true;
        for (u32 j = 0; j < arity; ++j) {
            len[j] = args.counts[j][i];
            if (len[j] == 0) hit = false;
            run[j] = args.sorted[j] + args.starts[j][i];
            pos[j] = 0;
        }
        u8 f = 0;
        if (hit) {
            if (arity == 1) {
                f = 1;
            } else {
                while (true) {
                    u32 max_id = run[0][pos[0]];
                    bool all_equal = true;
                    for (u32 j = 1; j < arity; ++j) {
                        const u32 v = run[j][pos[j]];
                        if (v != max_id) {
                            all_equal = false;
                            if (v > max_id) max_id = v;
                        }
                    }
                    if (all_equal) {
                        f = 1;
                        break;
                    }
                    bool exhausted = false;
                    for (u32 j = 0; j < arity && !exhausted; ++j) {
                        while (pos[j] < len[j] && run[j][pos[j]] < max_id) ++pos[j];
                        if (pos[j] >= len[j]) exhausted = true;
                    }
                    if (exhausted) break;
                }
            }
        }
        flags[i] = f;
    }
}

// Rows of arity <= 2 as one u64 key: (c0 << bits) | c1 (bits = value width).
__global__ void pack_rows_kernel(const u32* __restrict__ c0, const u32* __restrict__ c1, u64 n, u32 bits,
                                 u64* __restrict__ keys) {
    GRID_STRIDE(i, n) keys[i] = c1 ? (static_cast<u64>(c0[i]) << bits) | c1[i] : c0[i];
}

// flags[i] = NEW row i occurs in FULL: binary search of its packed key in the
// sorted FULL keys.
__global__ void member_kernel(const u32* __restrict__ c0, const u32* __restrict__ c1, u64 n, u32 bits,
                              const u64* __restrict__ full_keys, u64 n_full, u8* __restrict__ flags) {
    GRID_STRIDE(i, n) {
        const u64 key = c1 ? (static_cast<u64>(c0[i]) << bits) | c1[i] : c0[i];
        u64 lo = 0, hi = n_full;
        while (lo < hi) {
            const u64 mid = (lo + hi) >> 1;
            if (full_keys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        flags[i] = (lo < n_full && full_keys[lo] == key) ? 1 : 0;
    }
}

__device__ __forceinline__ u64 upper_bound_u64(const u64* __restrict__ a, u64 len, u64 x) {
    u64 lo = 0, hi = len;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

}  // namespace

// ---- load-balanced expansion (Algorithm 1, write phase) ------------------------
//
// Output-partitioned: CTA b owns outputs [b*TILE, (b+1)*TILE). Its first and
// last source rows come from two binary searches over the u64 offsets; every
// row starting inside the tile marks its first output slot in shared memory
// (atomicMax resolves zero-count rows that share an offset) and a block-wide
// max-scan propagates owners, so each output finds its row in O(1) instead
// of the reference's per-output upper_bound (P/src/kernels.cpp:110-117), and
// skewed ranges cost the same per output as short ones.
constexpr int kLbsBlock = 256;
constexpr int kLbsItems = 8;
constexpr int kLbsTile = kLbsBlock * kLbsItems;

template <class Op>
__global__ void __launch_bounds__(kLbsBlock) lbs_kernel(const u64* __restrict__ offsets, u64 m,
                                                        u64 total, Op op) {
    __shared__ u32 s_owner[kLbsTile];
    __shared__ u64 s_jlo, s_jhi;
    __shared__ u32 s_warp[kLbsBlock / 32];
    const u32 tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const u64 o0 = u64(blockIdx.x) * kLbsTile;
    const u64 o_end = min(o0 + kLbsTile, total);
    if (tid == 0) {
        s_jlo = upper_bound_u64(offsets, m + 1, o0) - 1;
        s_jhi = upper_bound_u64(offsets, m + 1, o_end - 1) - 1;
    }
    for (u32 i = tid; i < kLbsTile; i += kLbsBlock) s_owner[i] = 0;
    __syncthreads();
    const u64 jlo = s_jlo, jhi = s_jhi;
    for (u64 j = jlo + 1 + tid; j <= jhi; j += kLbsBlock) {
        const u64 p = offsets[j] - o0;
        atomicMax(&s_owner[p], static_cast<u32>(j - jlo));
    }
    __syncthreads();
    // Block inclusive max-scan over s_owner (blocked: thread owns 8 slots).
    u32 v[kLbsItems];
    u32 run = 0;
#pragma unroll
    for (int k = 0; k < kLbsItems; ++k) {
        run = max(run, s_owner[tid * kLbsItems + k]);
        v[k] = run;
    }
    u32 x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<u32>(o)) x = max(x, y);
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    u32 carry = 0;
    for (u32 w = 0; w < warp; ++w) carry = max(carry, s_warp[w]);
    const u32 prev = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane > 0) carry = max(carry, prev);
#pragma unroll
    for (int k = 0; k < kLbsItems; ++k) s_owner[tid * kLbsItems + k] = max(v[k], carry);
    __syncthreads();
    for (u32 i = tid; i < kLbsTile; i += kLbsBlock) {
        const u64 o = o0 + i;
        if (o >= o_end) break;
        const u64 j = jlo + s_owner[i];
        op.emit(o, j, o - offsets[j]);
    }
}

template <class Op>
void lbs_launch(Ctx* c, const u64* offsets, u64 m, u64 total, const Op& op) {
    if (total == 0) return;
    const u64 tiles = ceil_div(total, kLbsTile);
    lbs_kernel<Op><<<static_cast<unsigned>(tiles), kLbsBlock, 0, c->stream>>>(offsets, m, total, op);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

// ---- gather volume -------------------------------------------------------------

void add_gather_volume(u64 n) { g_gather_volume.fetch_add(n, std::memory_order_relaxed); }
u64 gather_volume() { return g_gather_volume.load(std::memory_order_relaxed); }
void reset_gather_volume() { g_gather_volume.store(0, std::memory_order_relaxed); }

// ---- index build -------------------------------------------------------------

void build_index(Ctx* c, const u32* raw, u64 n, DBuf<u32>& sorted_idx, DBuf<u32>& ukeys,
                 DBuf<u32>& ustart, DBuf<u32>& ucount, u64& n_unique) {
    if (n > 0xffffffffull) fail(FV_ERR_LENGTH, "column exceeds 32-bit tuple id space");
    n_unique = 0;
    sorted_idx = DBuf<u32>(c, n);
    if (n == 0) {
        ukeys = DBuf<u32>();
        ustart = DBuf<u32>();
        ucount = DBuf<u32>();
        return;
    }
    u64* dmax = c->d_scalars;
    reduce_max_u32(c, raw, n, dmax);
    u64 vmax = 0;
    c->read_scalars(dmax, &vmax, 1);
    const u32 bits = bit_width_u64(vmax);

    DBuf<u32> keys(c, n), keys_alt(c, n), vals_alt(c, n);
    FV_CUDA(cudaMemcpyAsync(keys.get(), raw, sizeof(u32) * n, cudaMemcpyDeviceToDevice, c->stream));
    iota_u32(c, sorted_idx.get(), n);
    const bool alt =
        radix_sort_pairs_u32(c, keys.get(), keys_alt.get(), sorted_idx.get(), vals_alt.get(), n, 0, bits);
    if (alt) {
        keys.swap(keys_alt);
        sorted_idx.swap(vals_alt);
    }
    keys_alt.reset();
    vals_alt.reset();

    DBuf<u32> uk(c, n), us(c, n);
    u64* dnu = c->d_scalars + 1;
    tile_scan(c, RleOp{keys.get(), uk.get(), us.get()}, n, dnu);
    c->read_scalars(dnu, &n_unique, 1);
    ukeys = DBuf<u32>(c, n_unique);
    ustart = DBuf<u32>(c, n_unique);
    ucount = DBuf<u32>(c, n_unique);
    FV_CUDA(cudaMemcpyAsync(ukeys.get(), uk.get(), sizeof(u32) * n_unique, cudaMemcpyDeviceToDevice, c->stream));
    FV_CUDA(cudaMemcpyAsync(ustart.get(), us.get(), sizeof(u32) * n_unique, cudaMemcpyDeviceToDevice, c->stream));
    rle_counts_kernel<<<grid_for(n_unique), 256, 0, c->stream>>>(ustart.get(), ucount.get(), n_unique, n);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void build_hash(Ctx* c, const u32* ukeys, u64 n_unique, HashIndex& ht) {
    if (n_unique == 0) {
        ht.slots = DBuf<u64>();
        ht.mask = 0;
        return;
    }
    u64 cap = 64;
    while (cap < 2 * n_unique) cap <<= 1;
    ht.slots = DBuf<u64>(c, cap);
    ht.mask = static_cast<u32>(cap - 1);
    FV_CUDA(cudaMemsetAsync(ht.slots.get(), 0xff, sizeof(u64) * cap, c->stream));
    hash_insert_kernel<<<grid_for(n_unique), 256, 0, c->stream>>>(
        ukeys, n_unique, reinterpret_cast<unsigned long long*>(ht.slots.get()), ht.mask);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

std::unique_ptr<Column> column_build(Ctx* c, DBuf<u32>&& raw, u64 n) {
    auto col = std::make_unique<Column>();
    col->ctx = c;
    col->n = n;
    col->raw = std::move(raw);
    build_index(c, col->raw.get(), n, col->sorted_idx, col->ukeys, col->ustart, col->ucount,
                col->n_unique);
    build_hash(c, col->ukeys.get(), col->n_unique, col->ht);
    return col;
}

std::unique_ptr<Version> version_empty(Ctx* c, u32 arity) {
    std::vector<DBuf<u32>> cols(arity);
    return version_from_device(c, std::move(cols), 0);
}

std::unique_ptr<Version> version_from_device(Ctx* c, std::vector<DBuf<u32>>&& cols, u64 n) {
    // Every row operator keeps per-column pointers in FV_MAX_ARITY-sized
    // arrays (ColPtrs, RunsArgs): a wider version is rejected here, at its
    // only constructor, instead of overrunning them later.
    if (cols.size() > FV_MAX_ARITY)
        fail(FV_ERR_ARITY, "version arity " + std::to_string(cols.size()) + " exceeds FV_MAX_ARITY");
    auto v = std::make_unique<Version>();
    v->ctx = c;
    v->arity = static_cast<u32>(cols.size());
    // Version::rows() is 0 for a version without columns (P/include/colog/relation.hpp:31).
    v->rows = cols.empty() ? 0 : n;
    for (auto& col : cols) v->cols.push_back(column_build(c, std::move(col), n));
    return v;
}

// ---- probes / gathers --------------------------------------------------------------

void column_probe_device(Ctx* c, const Column& col, const u32* values, u64 n, u32* starts,
                         u32* counts) {
    if (!n) return;
    ProfScope prof(c, "column_probe", double(n) * 12.0);
    probe_kernel<<<grid_for(n), 256, 0, c->stream>>>(col.ht.slots.get(), col.ht.mask,
                                                      col.ustart.get(), col.ucount.get(), values, n,
                                                      starts, counts);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void check_ids(Ctx* c, const u32* ids, u64 n, u64 bound, const char* msg) {
    if (n == 0) return;
    if (bound == 0) fail(FV_ERR_RANGE, msg);
    u64* dmax = c->d_scalars + 2;
    reduce_max_u32(c, ids, n, dmax);
    u64 m = 0;
    c->read_scalars(dmax, &m, 1);
    if (m >= bound) fail(FV_ERR_RANGE, msg);
}

DBuf<u32> gather_device(Ctx* c, const u32* src, const u32* ids, u64 n) {
    DBuf<u32> out(c, n);
    gather_u32(c, src, ids, out.get(), n);
    add_gather_volume(n);
    return out;
}

std::unique_ptr<Match> join_probe_phase(Ctx* c, const u32* probe, u64 n, const Column& build) {
    auto m = std::make_unique<Match>();
    m->ctx = c;
    if (n == 0) return m;
    DBuf<u32> starts(c, n), counts(c, n);
    column_probe_device(c, build, probe, n, starts.get(), counts.get());
    DBuf<u32> ms(c, n), mc(c, n), mm(c, n);
    u64* dm = c->d_scalars + 3;
    tile_scan(c, SelectMatchOp{starts.get(), counts.get(), ms.get(), mc.get(), mm.get()}, n, dm);
    c->read_scalars(dm, &m->m, 1);
    m->starts = std::move(ms);
    m->counts = std::move(mc);
    m->matched = std::move(mm);
    return m;
}

u64 join_total_size(Ctx* c, const Match& m) {
    u64* d = c->d_scalars + 4;
    FV_CUDA(cudaMemsetAsync(d, 0, sizeof(u64), c->stream));
    if (m.m) {
        sum_u32_kernel<<<grid_for(m.m), 256, 0, c->stream>>>(m.counts.get(), m.m,
                                                              reinterpret_cast<unsigned long long*>(d));
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    }
    u64 t = 0;
    c->read_scalars(d, &t, 1);
    return t;
}

DBuf<u64> join_offsets(Ctx* c, const Match& m) {
    DBuf<u64> off(c, m.m + 1);
    exclusive_scan_counts(c, m.counts.get(), off.get(), m.m);
    return off;
}

void join_write_phase(Ctx* c, const Match& m, const u64* offsets, u64 total, const Column& build,
                      DBuf<u32>& a, DBuf<u32>& b) {
    a = DBuf<u32>(c, total);
    b = DBuf<u32>(c, total);
    // Per output: its sorted_idx entry read and the id pair written.
    ProfScope prof(c, "join_write_phase", double(m.m) * 16.0 + double(total) * 12.0);
    lbs_launch(c, offsets, m.m, total,
               JoinWriteOp{m.starts.get(), m.matched.get(), build.sorted_idx.get(), a.get(), b.get()});
}

void filter_pairs_eq(Ctx* c, const u32* a, const u32* b, u64 n, const Column& ca,
                     const Column& cb, DBuf<u32>& oa, DBuf<u32>& ob, u64& n_out) {
    check_ids(c, a, n, ca.n, "filter_pairs_eq: tuple id past end of column");
    check_ids(c, b, n, cb.n, "filter_pairs_eq: tuple id past end of column");
    DBuf<u32> ta(c, n), tb(c, n);
    u64* d = c->d_scalars + 5;
    tile_scan(c, PairsEqOp{a, b, ca.raw.get(), cb.raw.get(), ta.get(), tb.get()}, n, d);
    c->read_scalars(d, &n_out, 1);
    oa = std::move(ta);
    ob = std::move(tb);
}

DBuf<u32> filter_neq(Ctx* c, const Version& v, u32 i, u32 j, u64& n_out) {
    if (i >= v.arity || j >= v.arity) fail(FV_ERR_RANGE, "filter_neq: column index past arity");
    DBuf<u32> out(c, v.rows);
    u64* d = c->d_scalars + 6;
    tile_scan(c, NeqOp{v.cols[i]->raw.get(), v.cols[j]->raw.get(), out.get()}, v.rows, d);
    c->read_scalars(d, &n_out, 1);
    return out;
}

DBuf<u32> select_eq(Ctx* c, const Column& col, u32 v, u64& n_out) {
    n_out = 0;
    if (col.n == 0) return DBuf<u32>();
    DBuf<u32> dv = make_dbuf(c, &v, 1);
    DBuf<u32> se(c, 2);
    column_probe_device(c, col, dv.get(), 1, se.get(), se.get() + 1);
    u32 h[2];
    se.download(h, 2);
    n_out = h[1];
    DBuf<u32> out(c, n_out);
    if (n_out)
        FV_CUDA(cudaMemcpyAsync(out.get(), col.sorted_idx.get() + h[0], sizeof(u32) * n_out,
                                cudaMemcpyDeviceToDevice, c->stream));
    return out;
}

std::unique_ptr<Version> project(Ctx* c, const Version& v, const u32* ids, u64 n,
                                 const std::vector<u32>& col_map) {
    std::vector<DBuf<u32>> cols;
    for (u32 src : col_map) {
        if (src >= v.arity) fail(FV_ERR_RANGE, "project: column index past arity");
        check_ids(c, ids, n, v.rows, "gather: tuple id past end of column");
        cols.push_back(gather_device(c, v.cols[src]->raw.get(), ids, n));
    }
    return version_from_device(c, std::move(cols), n);
}

DBuf<u32> lexicographic_order(Ctx* c, const u32* const* cols, u32 arity, u64 n, const char* who) {
    static const bool trace_sorts = std::getenv("FVLOG_TRACE_SORTS") != nullptr;
    if (trace_sorts) std::fprintf(stderr, "[sort-call] lexicographic_order from %s n=%llu arity=%u\n", who,
                                  static_cast<unsigned long long>(n), arity);
    DBuf<u32> perm(c, n), perm_alt(c, n), keys(c, n), keys_alt(c, n);
    iota_u32(c, perm.get(), n);
    for (int j = static_cast<int>(arity) - 1; j >= 0; --j) {
        u64* dmax = c->d_scalars + 7;
        reduce_max_u32(c, cols[j], n, dmax);
        u64 vmax = 0;
        c->read_scalars(dmax, &vmax, 1);
        gather_u32(c, cols[j], perm.get(), keys.get(), n);
        const bool alt = radix_sort_pairs_u32(c, keys.get(), keys_alt.get(), perm.get(),
                                              perm_alt.get(), n, 0, bit_width_u64(vmax));
        if (alt) perm.swap(perm_alt);
    }
    return perm;
}

static ColPtrs col_ptrs(const Version& v) {
    ColPtrs p{};
    for (u32 j = 0; j < v.arity; ++j) p.p[j] = v.cols[j]->raw.get();
    return p;
}

std::unique_ptr<Version> dedup_rows(Ctx* c, const Version& v) {
    const u64 n = v.rows;
    if (n == 0) return version_empty(c, v.arity);
    if (v.arity > FV_MAX_ARITY) fail(FV_ERR_ARITY, "dedup_rows: arity exceeds FV_MAX_ARITY");
    std::vector<const u32*> cp(v.arity);
    for (u32 j = 0; j < v.arity; ++j) cp[j] = v.cols[j]->raw.get();
    DBuf<u32> perm = lexicographic_order(c, cp.data(), v.arity, n);
    DBuf<u32> keep(c, n);
    u64* d = c->d_scalars + 8;
    tile_scan(c, HeadsOp{col_ptrs(v), v.arity, perm.get(), keep.get()}, n, d);
    u64 nk = 0;
    c->read_scalars(d, &nk, 1);
    // Group heads carry the smallest id; restoring id order gives
    // first-occurrence order (P/src/relation.cpp:76-80).
    DBuf<u32> keep_alt(c, nk);
    if (radix_sort_keys_u32(c, keep.get(), keep_alt.get(), nk, 0, bit_width_u64(n - 1)))
        keep.swap(keep_alt);
    std::vector<DBuf<u32>> cols;
    for (u32 j = 0; j < v.arity; ++j) cols.push_back(gather_device(c, v.cols[j]->raw.get(), keep.get(), nk));
    return version_from_device(c, std::move(cols), nk);
}

bool has_duplicate_rows(Ctx* c, const Version& v) {
    if (v.rows < 2) return false;
    if (v.arity > FV_MAX_ARITY) fail(FV_ERR_ARITY, "has_duplicate_rows: arity exceeds FV_MAX_ARITY");
    std::vector<const u32*> cp(v.arity);
    for (u32 j = 0; j < v.arity; ++j) cp[j] = v.cols[j]->raw.get();
    DBuf<u32> perm = lexicographic_order(c, cp.data(), v.arity, v.rows);
    u64* d = c->d_scalars + 9;
    tile_scan(c, HeadsOp{col_ptrs(v), v.arity, perm.get(), nullptr}, v.rows, d);
    u64 nk = 0;
    c->read_scalars(d, &nk, 1);
    return nk < v.rows;
}

DBuf<u8> deduplicate(Ctx* c, const Version& nv, const Version& full) {
    if (nv.arity != full.arity) fail(FV_ERR_ARITY, "deduplicate: arity mismatch");
    if (nv.arity > FV_MAX_ARITY) fail(FV_ERR_ARITY, "deduplicate: arity exceeds FV_MAX_ARITY");
    const u64 n = nv.rows;
    DBuf<u8> flags(c, n);
    if (n == 0) return flags;
    if (full.rows == 0) {
        FV_CUDA(cudaMemsetAsync(flags.get(), 0, n, c->stream));
        return flags;
    }
    if (nv.arity <= 2) {
        // Same flags as Algorithm 2 (a NEW row is marked iff it occurs in
        // FULL), computed as membership of packed row keys in FULL's sorted
        // keys instead of intersecting per-column id runs (runs of hot
        // values are thousands of ids long): one radix sort of FULL + one
        // binary search per NEW row.
        u64* dmax = c->d_scalars + 12;
        FV_CUDA(cudaMemsetAsync(dmax, 0, sizeof(u64), c->stream));
        for (u32 j = 0; j < nv.arity; ++j) {
            reduce_max_u32(c, nv.cols[j]->raw.get(), n, dmax, true);
            reduce_max_u32(c, full.cols[j]->raw.get(), full.rows, dmax, true);
        }
        u64 vmax = 0;
        c->read_scalars(dmax, &vmax, 1);
        const u32 bits = std::max<u32>(1, bit_width_u64(vmax));
        const u32* f1 = nv.arity == 2 ? full.cols[1]->raw.get() : nullptr;
        const u32* n1 = nv.arity == 2 ? nv.cols[1]->raw.get() : nullptr;
        DBuf<u64> keys(c, full.rows), alt(c, full.rows);
        ProfScope prof(c, "deduplicate", double(full.rows) * (4.0 * nv.arity + 8.0) + double(n) * (4.0 * nv.arity + 1.0));
        pack_rows_kernel<<<grid_for(full.rows), 256, 0, c->stream>>>(full.cols[0]->raw.get(), f1, full.rows, bits,
                                                                     keys.get());
        FV_CUDA(cudaGetLastError());
        if (radix_sort_keys_u64(c, keys.get(), alt.get(), full.rows, 0, nv.arity == 2 ? 2 * bits : bits))
            keys.swap(alt);
        member_kernel<<<grid_for(n), 256, 0, c->stream>>>(nv.cols[0]->raw.get(), n1, n, bits, keys.get(), full.rows,
                                                          flags.get());
        FV_CUDA(cudaGetLastError());
        c->count_launch(2);
        return flags;
    }
    // One probe loop per column, as in the reference (kernels.cpp:220-233).
    std::vector<DBuf<u32>> starts, counts;
    RunsArgs args{};
    for (u32 j = 0; j < nv.arity; ++j) {
        starts.emplace_back(c, n);
        counts.emplace_back(c, n);
        column_probe_device(c, *full.cols[j], nv.cols[j]->raw.get(), n, starts[j].get(), counts[j].get());
        args.sorted[j] = full.cols[j]->sorted_idx.get();
        args.starts[j] = starts[j].get();
        args.counts[j] = counts[j].get();
    }
    runs_intersect_kernel<<<grid_for(n), 256, 0, c->stream>>>(args, nv.arity, n, flags.get());
    FV_CUDA(cudaGetLastError());
    c->count_launch();
    return flags;
}

std::unique_ptr<Version> difference(Ctx* c, const Version& nv, const u8* flags) {
    DBuf<u32> ids(c, nv.rows);
    u64* d = c->d_scalars + 10;
    tile_scan(c, SelectFlagsOp{flags, 0, ids.get()}, nv.rows, d);
    u64 nk = 0;
    c->read_scalars(d, &nk, 1);
    std::vector<DBuf<u32>> cols;
    for (u32 j = 0; j < nv.arity; ++j) cols.push_back(gather_device(c, nv.cols[j]->raw.get(), ids.get(), nk));
    return version_from_device(c, std::move(cols), nk);
}

std::unique_ptr<Version> version_append(Ctx* c, const Version& v, const Version& extra) {
    if (extra.arity != v.arity) fail(FV_ERR_ARITY, "append: arity mismatch");
    const u64 n = v.rows + extra.rows;
    std::vector<DBuf<u32>> cols;
    for (u32 j = 0; j < v.arity; ++j) {
        DBuf<u32> col(c, n);
        if (v.rows)
            FV_CUDA(cudaMemcpyAsync(col.get(), v.cols[j]->raw.get(), sizeof(u32) * v.rows,
                                    cudaMemcpyDeviceToDevice, c->stream));
        if (extra.rows)
            FV_CUDA(cudaMemcpyAsync(col.get() + v.rows, extra.cols[j]->raw.get(),
                                    sizeof(u32) * extra.rows, cudaMemcpyDeviceToDevice, c->stream));
        cols.push_back(std::move(col));
    }
    return version_from_device(c, std::move(cols), n);
}

void version_reconstruct(const Version& v, u32* rows_out) {
    std::vector<u32> col(v.rows);
    for (u32 j = 0; j < v.arity; ++j) {
        v.cols[j]->raw.download(col.data(), v.rows);
        for (u64 i = 0; i < v.rows; ++i) rows_out[i * v.arity + j] = col[i];
    }
}

}  // namespace fv

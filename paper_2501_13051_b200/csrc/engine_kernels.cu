// sm_100a kernels of the fixpoint engine (see engine.h for the data layout).
//
//   probe_count   join phase 1 (Algorithm 1, P/src/kernels.cpp:59-92): one
//                 hash probe per probe row -> (run start, run length)
//   materialize   join phase 2 (kernels.cpp:104-123) fused with the residual
//                 equalities (kernels.cpp:137-165), the != guards
//                 (engine.cpp:128-145) and the head projection
//                 (engine.cpp:122-125): output-partitioned, each CTA expands
//                 a fixed tile of join outputs and writes head rows directly
//                 (as packed row keys for the dedup sort) — no IdPairSet,
//                 no per-source id arrays, no wide Version.
//   merge         dedup_rows + deduplicate + difference + merge_delta
//                 (relation.cpp:71-108, kernels.cpp:210-268) as ONE
//                 merge-path pass over sorted FULL and sorted candidates.
#include <cmath>
#include <cstdio>
#include <optional>
#include <cstdlib>

#include "engine.h"
#include "prim.cuh"
#include "radix_sort.h"

namespace fv {

namespace {

unsigned grid_for(u64 n, int block = 256) {
    const u64 want = ceil_div(n, block);
    const u64 cap = u64(kNumSMs) * 16;
    return static_cast<unsigned>(want == 0 ? 1 : (want < cap ? want : cap));
}

#define GRID_STRIDE(i, n) \
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); i += u64(gridDim.x) * blockDim.x)

__device__ __forceinline__ u32 slot(const SlotRef& s, u64 i, u64 p) { return s.ptr[s.side ? p : i]; }

__device__ __forceinline__ bool pass_filters(const Filter* f, u32 n, u64 i, u64 p) {
#pragma unroll
    for (int k = 0; k < kMaxFilters; ++k) {
        if (k >= static_cast<int>(n)) break;
        const u32 a = slot(f[k].a, i, p);
        if (f[k].op == kFilterConst) {
            if (a != f[k].value) return false;
        } else if (f[k].op == kFilterOwner) {
            if (static_cast<u32>((static_cast<u64>(hash32(a >> f[k].oshift)) * f[k].world) >> 32) != f[k].value)
                return false;
        } else {
            const u32 b = slot(f[k].b, i, p);
            if ((a == b) != (f[k].op == kFilterEq)) return false;
        }
    }
    return true;
}

__device__ __forceinline__ bool ht_lookup(const u64* __restrict__ slots, u32 mask, u32 key, u32* idx) {
    u32 h = hash32(key) & mask;
    while (true) {
        const u64 s = __ldg(slots + h);
        if (s == kEmptySlot) return false;
        if (static_cast<u32>(s >> 32) == key) {
            *idx = static_cast<u32>(s);
            return true;
        }
        h = (h + 1) & mask;
    }
}

// Run (start, count) of value v in a direct-address index (ends: ucount
// holds the run's end, 0 when there is none).
__device__ __forceinline__ void direct_run(const u32* __restrict__ ustart, const u32* __restrict__ ucount, bool ends,
                                           u32 v, u32* s, u32* c) {
    if (!ucount) {  // interleaved (start, end) pairs: one 8-byte load
        const uint2 p = reinterpret_cast<const uint2*>(ustart)[v];
        if (p.y) {
            *s = p.x;
            *c = p.y - p.x;
        }
        return;
    }
    const u32 e = ucount[v];
    if (ends) {
        if (e) {
            *s = ustart[v];
            *c = e - *s;
        }
    } else {
        *s = ustart[v];
        *c = e;
    }
}

__global__ void probe_count_kernel(const u32* __restrict__ probe, u64 n, const u64* __restrict__ slots,
                                   u32 mask, const u32* __restrict__ ustart, const u32* __restrict__ ucount,
                                   u64 domain, bool ends, RowFilter pred, u32* __restrict__ starts,
                                   u32* __restrict__ counts) {
    GRID_STRIDE(i, n) {
        u32 s = 0, c = 0, r;
        if (pass_filters(pred.f, pred.n, i, 0)) {
            const u32 v = probe[i];
            if (domain) {  // direct-address index: run of value v at ustart[v], ucount[v]
                if (v < domain) direct_run(ustart, ucount, ends, v, &s, &c);
            } else if (ht_lookup(slots, mask, v, &r)) {
                s = ustart[r];
                c = ucount[r];
            }
        }
        starts[i] = s;
        counts[i] = c;
    }
}

__device__ __forceinline__ u64 row_key1(const OutSpec& spec, u64 i, u64 p) {
    const u64 hi = slot(spec.col[0], i, p);
    return spec.n_out >= 2 ? (hi << spec.shift) | slot(spec.col[1], i, p) : hi;
}

// Key-set home slot (KeySet::group_bits = b): the low b bits of the key are
// kept and the rest is scattered, so the 2^b keys that differ only there
// (same first column, adjacent second-column ids) share a sector. A DRAM miss
// costs a 128-byte line on this part (tools/membench.cu), so b = 1 halves the
// misses of a relation whose candidates are mostly new (SG: 76 -> 54 ms);
// when most candidates are repeats, grouped keys concentrate the probes of a
// hub's outputs on a few L2 lines and b = 0 (plain scattering) is faster
// (C2 141 vs 162 ms, C4 248 vs 271 ms). The engine picks b per relation from
// the last iteration's candidates per new row. Growth keeps the property the
// streaming rehash needs (new home = old home + j * old capacity).
__device__ __forceinline__ u64 keyset_line_hash(u64 key, u32 bits) { return mix64(key >> bits); }
__device__ __forceinline__ u64 keyset_home(u64 line_hash, u64 key, u32 bits, u64 mask) {
    return ((line_hash << bits) | (key & ((u64(1) << bits) - 1))) & mask;
}

// Set-insert of one key: true when the key was absent (this thread inserted
// it). Duplicates are detected with a plain load first; only empty slots
// are claimed with a CAS.
__device__ __forceinline__ bool keyset_insert_probe_from(u64* __restrict__ slots, u64 mask, u64 key, u64 h) {
    while (true) {
        const u64 s = __ldcg(slots + h);
        if (s == key) return false;
        if (s == kEmptySlot) {
            const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(slots + h), ~0ull,
                                       static_cast<unsigned long long>(key));
            if (prev == ~0ull) return true;
            if (prev == key) return false;
        }
        h = (h + 1) & mask;
    }
}

// Insert resolution after a speculative first-slot load `s` (issued early so
// a thread has many independent table loads in flight).
__device__ __forceinline__ bool keyset_insert_from(u64* __restrict__ slots, u64 mask, u64 key, u64 h, u64 s) {
    if (s == key) return false;
    if (s == kEmptySlot) {
        const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(slots + h), ~0ull,
                                   static_cast<unsigned long long>(key));
        if (prev == ~0ull) return true;
        if (prev == key) return false;
    }
    return keyset_insert_probe_from(slots, mask, key, (h + 1) & mask);
}

// Warp-aggregated append of the keys flagged new (all lanes must call).
__device__ __forceinline__ void append_new(u64* __restrict__ out, u64* counter, bool is_new, u64 key) {
    const u32 m = __ballot_sync(0xffffffffu, is_new);
    if (!m) return;
    const u32 lane = lane_id();
    const u32 leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(reinterpret_cast<unsigned long long*>(counter), static_cast<unsigned long long>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (is_new) out[base + __popc(m & lanemask_lt())] = key;
}

// Warp-aggregated append of every item flagged in `mask` (bit k: key[k] is
// new) with ONE counter atomic per warp for all items: the counter is a single
// global word that every warp of the grid hits, so its atomic rate, not the
// key set, caps the join when each item takes its own atomic.
template <int N>
__device__ __forceinline__ void append_new_items(u64* __restrict__ out, u64* counter, u32 mask, const u64 (&key)[N]) {
    const u32 lane = lane_id();
    const u32 cnt = __popc(mask);
    u32 incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<u32>(o)) incl += y;
    }
    const u32 total = __shfl_sync(0xffffffffu, incl, 31);
    if (!total) return;
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(reinterpret_cast<unsigned long long*>(counter), static_cast<unsigned long long>(total));
    u64 pos = __shfl_sync(0xffffffffu, base, 31) + (incl - cnt);
#pragma unroll
    for (int k = 0; k < N; ++k)
        if ((mask >> k) & 1u) out[pos++] = key[k];
}

// ---- block set (BlockSet, engine.h) ------------------------------------------------

// A longer probe run sends the key to the overflow list (the host grows the
// directory and inserts it): the loop is bounded whatever the load.
constexpr int kBlockMaxProbes = 64;

// Block id and bit position (word << 5 | bit) of a packed row key.
__device__ __forceinline__ u64 block_of(u64 key, u32 shift, u32 arity, u32* bitpos) {
    if (arity == 2) {
        const u64 a = key >> shift;
        const u64 b = key & ((u64(1) << shift) - 1);
        *bitpos = (static_cast<u32>(a & 31) << 5) | static_cast<u32>(b & 31);
        return ((a >> 5) << 27) | (b >> 5);
    }
    *bitpos = static_cast<u32>(key & 1023);
    return key >> 10;
}
__device__ __forceinline__ u64 block_home(u64 bid, u64 mask) { return mix64(bid) & mask; }

// Directory slot of block `bid` given the first probed slot h (holding v);
// claims an empty slot for a new block. ~0: no slot (overflow).
// (Arguments by value: a reference into the kernel's parameter block would
// force the whole OutSpec into local memory.)
// *inserted counts this thread's new blocks; the caller adds a warp's total
// to the block count with one atomic (a single hot counter otherwise takes
// one atomic per new block). The limit check reads a count that may lag by
// the warps in flight — the load limit is 3/4 of capacity, and a full probe
// window still falls back to the overflow list.
__device__ __forceinline__ u64 blockset_find(u64* dir, u64 mask, u64* count, u64 limit, u64 bid, u64 h, u64 v,
                                             u32* inserted) {
    for (int probe = 0; probe < kBlockMaxProbes; ++probe) {
        if (v == bid) return h;
        if (v == kEmptySlot) {
            if (ld_relaxed_u64(count) >= limit) return ~u64(0);
            const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(dir + h), ~0ull,
                                       static_cast<unsigned long long>(bid));
            if (prev == ~0ull) {
                ++*inserted;
                return h;
            }
            if (prev == bid) return h;
        }
        h = (h + 1) & mask;
        v = __ldcg(dir + h);
    }
    return ~u64(0);
}

// One atomic per warp for its lanes' new blocks (call from all 32 lanes).
__device__ __forceinline__ void add_block_count(u64* count, u32 inserted) {
    const u32 t = __reduce_add_sync(0xffffffffu, inserted);
    if (lane_id() == 0 && t) atomicAdd(reinterpret_cast<unsigned long long*>(count), static_cast<unsigned long long>(t));
}

// Set-insert of N keys (bit k of `live`: key[k] is a candidate). All
// directory loads are issued first, then all bitmap loads, then the atomics of
// the bits found clear (repeats of present rows never issue an atomic).
// Returns the new mask; keys that found no slot are flagged in *ovf_mask.
template <int N>
__device__ __forceinline__ u32 blockset_insert_items(const BlockSetArgs& s, u32 live, const u64 (&key)[N],
                                                     u32* ovf_mask) {
    u64 slot[N];
    u32 bp[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        slot[k] = 0;
        bp[k] = 0;
        if ((live >> k) & 1u) slot[k] = block_of(key[k], s.shift, s.arity, &bp[k]);  // bid for now
    }
    u64 dv[N];
#pragma unroll
    for (int k = 0; k < N; ++k) dv[k] = ((live >> k) & 1u) ? __ldcg(s.dir + block_home(slot[k], s.mask)) : 0;
    u32 om = 0, inserted = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        if (!((live >> k) & 1u)) continue;
        const u64 bid = slot[k], h = block_home(bid, s.mask);
        const u64 f = dv[k] == bid ? h : blockset_find(s.dir, s.mask, s.count, s.limit, bid, h, dv[k], &inserted);
        if (f == ~u64(0)) {
            om |= 1u << k;
            live &= ~(1u << k);
        }
        slot[k] = f;
    }
    add_block_count(s.count, inserted);
    u32 wv[N];
#pragma unroll
    for (int k = 0; k < N; ++k) wv[k] = ((live >> k) & 1u) ? __ldcg(s.bits + slot[k] * 32 + (bp[k] >> 5)) : 0;
    u32 nm = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        if (!((live >> k) & 1u)) continue;
        const u32 m = 1u << (bp[k] & 31);
        if (wv[k] & m) continue;
        if (!(atomicOr(s.bits + slot[k] * 32 + (bp[k] >> 5), m) & m)) nm |= 1u << k;
    }
    *ovf_mask = om;
    return nm;
}

// ---- word form of a binary relation (RelState::word_mode, engine.h) ---------------
//
// A row set is carried as words: a word key (x << shift | z & ~31) plus a
// 32-bit mask of the z's of that word present. One word is the 32 bits of
// one row of a BlockSet block, so inserting it into FULL is ONE bitmap OR and
// a composition join emits one candidate per (probe row, DELTA word) instead
// of one per tuple.

// Word key and bit of a packed binary tuple key.
__device__ __forceinline__ u64 word_key_of(u64 key, u32 shift, u32* bit) {
    const u64 z = key & ((u64(1) << shift) - 1);
    *bit = 1u << static_cast<u32>(z & 31);
    return ((key >> shift) << shift) | (z & ~u64(31));
}

// Set-insert of N words (bit k of `live`: key[k] / bits[k] is a candidate):
// all directory loads first, then all bitmap-word loads, then an atomic OR
// only where some bit is still clear. The bits that were clear in FULL are
// also OR-ed into the block's DELTA bitmap (s.dbits, same slot): the insert
// that finds that DELTA word empty is its first writer this iteration and
// is flagged in *first (its key is appended once; the merged mask is read at
// finalize). *ones = the new bits of this thread. Words whose block found no
// directory slot are flagged in *ovf_mask.
// A plain load of the FULL word before its atomicOr (repeats take no atomic):
// measured without it C2 21.7 -> 23.9 ms, C4 64.9 -> 65.2.
#ifndef FV_WORD_TEST_LOAD
#define FV_WORD_TEST_LOAD 1
#endif
template <int N>
__device__ __forceinline__ void blockset_word_items(const BlockSetArgs& s, u32 live, const u64 (&key)[N],
                                                    const u32 (&bits)[N], u32* first, u32* ones, u32* ovf_mask,
                                                    u32 (&widx)[N]) {
    u64 slot[N];
    u32 wi[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        slot[k] = 0;
        wi[k] = 0;
        if ((live >> k) & 1u) {
            u32 bp;
            slot[k] = block_of(key[k], s.shift, 2, &bp);  // bid for now
            wi[k] = bp >> 5;
        }
    }
    u64 dv[N];
#pragma unroll
    for (int k = 0; k < N; ++k) dv[k] = ((live >> k) & 1u) ? __ldcg(s.dir + block_home(slot[k], s.mask)) : 0;
    u32 om = 0, inserted = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        if (!((live >> k) & 1u)) continue;
        const u64 bid = slot[k], h = block_home(bid, s.mask);
        const u64 f = dv[k] == bid ? h : blockset_find(s.dir, s.mask, s.count, s.limit, bid, h, dv[k], &inserted);
        if (f == ~u64(0)) {
            om |= 1u << k;
            live &= ~(1u << k);
        }
        slot[k] = f * 32 + wi[k];  // bitmap word index from here on
    }
    add_block_count(s.count, inserted);
    u32 nb[N];
#if FV_WORD_TEST_LOAD
    // a plain load first: a word whose bits are all present takes no atomic
    u32 wv[N];
#pragma unroll
    for (int k = 0; k < N; ++k) wv[k] = ((live >> k) & 1u) ? __ldcg(s.bits + slot[k]) : ~0u;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        nb[k] = 0;
        if (!((live >> k) & 1u) || (wv[k] & bits[k]) == bits[k]) continue;
        nb[k] = bits[k] & ~atomicOr(s.bits + slot[k], bits[k]);
    }
#else
#pragma unroll
    for (int k = 0; k < N; ++k) nb[k] = ((live >> k) & 1u) ? bits[k] & ~atomicOr(s.bits + slot[k], bits[k]) : 0u;
#endif
    u32 fm = 0, n1 = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        widx[k] = static_cast<u32>(slot[k]);  // bitmap word index (valid until the directory grows)
        if (!nb[k]) continue;
        n1 += __popc(nb[k]);
        if (atomicOr(s.dbits + slot[k], nb[k]) == 0) fm |= 1u << k;
    }
    *first = fm;
    *ones = n1;
    *ovf_mask = om;
}

// Warp-aggregated append of the keys flagged in `mask` (one counter atomic
// per warp), plus `ones` (per thread) summed into *tuples when non-null.
template <int N>
__device__ __forceinline__ void append_words(u64* __restrict__ out, u32* __restrict__ out_bits, u64* counter,
                                             u64* tuples, u32 ones, u32 mask, const u64 (&key)[N],
                                             const u32 (&bits)[N]) {
    const u32 lane = lane_id();
    const u32 cnt = __popc(mask);
    u32 incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<u32>(o)) incl += y;
    }
    const u32 total = __shfl_sync(0xffffffffu, incl, 31);
    if (tuples) {
        const u32 t = __reduce_add_sync(0xffffffffu, ones);
        if (lane == 0 && t) atomicAdd(reinterpret_cast<unsigned long long*>(tuples), static_cast<unsigned long long>(t));
    }
    if (!total) return;
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(reinterpret_cast<unsigned long long*>(counter), static_cast<unsigned long long>(total));
    u64 pos = __shfl_sync(0xffffffffu, base, 31) + (incl - cnt);
#pragma unroll
    for (int k = 0; k < N; ++k)
        if ((mask >> k) & 1u) {
            out[pos] = key[k];
            if (out_bits) out_bits[pos] = bits[k];
            ++pos;
        }
}

// Write one output row (values computed from slots) at position pos.
__device__ __forceinline__ void write_row(const OutSpec& spec, u64 pos, u64 i, u64 p) {
    if (spec.key_mode) {
        const u32 w = (spec.n_out + 1) / 2;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k >= static_cast<int>(w)) break;
            const u64 hi = slot(spec.col[2 * k], i, p);
            u64 word;
            if (2 * k + 1 < static_cast<int>(spec.n_out))
                word = (hi << spec.shift) | slot(spec.col[2 * k + 1], i, p);
            else
                word = hi;
            spec.keys[k][pos] = word;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kMaxSlots; ++k) {
            if (k >= static_cast<int>(spec.n_out)) break;
            spec.out_cols[k][pos] = slot(spec.col[k], i, p);
        }
    }
}

// 512 threads x 4 outputs per 2048-output tile: the fused key-set probes are
// latency-bound random loads, and more warps with fewer items each keep more
// of them in flight (C2 141.7 -> 123.7 ms, C3 55.3 -> 46.2, C4 250 -> 223
// against 256 x 8; 1024 x 2 is equal on C2/C3 and slower on C4).
#ifndef FV_MAT_BLOCK
#define FV_MAT_BLOCK 512
#endif
constexpr int kMatBlock = FV_MAT_BLOCK;
constexpr int kMatItems = 2048 / kMatBlock;  // one 2048-output tile per CTA
constexpr int kMatTile = kMatBlock * kMatItems;
constexpr int kMatSparseSpan = 8 * kMatTile;
// Tile-local set: one slot per output (load <= 1 when every output is
// distinct; repeats share slots). Measured against 2 slots per output:
// C2 23.8-24.1 -> 23.6 ms, C3 17.06 -> 16.98, C4 69.98 -> 69.85 (less shared
// memory to clear per tile; an unplaced key is simply probed globally).
#ifndef FV_MAT_SET_SLOTS
#define FV_MAT_SET_SLOTS kMatTile
#endif
constexpr int kMatSetSlots = FV_MAT_SET_SLOTS;
#ifndef FV_MAT_APPEND_CTA
#define FV_MAT_APPEND_CTA 0
#endif
#ifndef FV_MAT_BATCH_CAS
#define FV_MAT_BATCH_CAS 2  // 2: batched for the plain join only (the filtered variant spills: C3 32.9 vs 32.5 ms)
#endif
#ifndef FV_MAT_SET_PROBES
#define FV_MAT_SET_PROBES 16  // measured: 4 slower (C2 93.5 vs 92.7 ms), 64 equal
#endif
constexpr int kMatSetProbes = FV_MAT_SET_PROBES;               // bounded: an unplaced key is simply probed globally

__device__ __forceinline__ u64 upper_bound_u64(const u64* __restrict__ a, u64 len, u64 x) {
    u64 lo = 0, hi = len;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Block-wide exclusive sum of u32 (256 threads); returns prefix, *total.
__device__ __forceinline__ u32 block_excl_u32(u32 v, u32* s_warp, u32* total) {
    const u32 lane = lane_id(), warp = threadIdx.x >> 5;
    u32 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<u32>(o)) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 run = 0;
        for (int w = 0; w < kMatBlock / 32; ++w) {
            const u32 t = s_warp[w];
            s_warp[w] = run;
            run += t;
        }
        s_warp[kMatBlock / 32] = run;
    }
    __syncthreads();
    const u32 r = s_warp[warp] + x - v;
    *total = s_warp[kMatBlock / 32];
    __syncthreads();
    return r;
}

// First and last source row of every output tile (parallel binary searches).
// upper_bound by one warp: a 32-ary search (each round one load per lane,
// log32(len) rounds instead of log2(len) dependent loads). All lanes call
// it with the same x and get the same result.
__device__ __forceinline__ u64 upper_bound_warp(const u64* __restrict__ a, u64 len, u64 x) {
    const u32 lane = lane_id();
    u64 lo = 0, hi = len;  // answer in [lo, hi]
    while (hi - lo > 32) {
        const u64 step = (hi - lo + 31) / 32;
        const u64 idx = lo + u64(lane) * step;
        const bool valid = idx < hi;
        // probes with a[idx] <= x form a prefix of the valid ones
        const u32 c = __popc(__ballot_sync(0xffffffffu, valid && a[idx] <= x));
        const u32 nvalid = __popc(__ballot_sync(0xffffffffu, valid));
        const u64 nlo = c ? lo + u64(c - 1) * step + 1 : lo;
        const u64 nhi = c < nvalid ? lo + u64(c) * step : hi;
        lo = nlo;
        hi = nhi;
    }
    const u64 idx = lo + lane;
    const u32 m = __ballot_sync(0xffffffffu, idx < hi && a[idx] > x);
    return m ? lo + __ffs(m) - 1 : hi;
}

// One warp per output tile: the rows holding its first and last output.
__global__ void tile_rows_kernel(const u64* __restrict__ offsets, u64 m, u64 o_begin, u64 total, u64 tiles,
                                 u64* __restrict__ jlo, u64* __restrict__ jhi) {
    const u64 warps = u64(gridDim.x) * (blockDim.x / 32);
    for (u64 b = (u64(blockIdx.x) * blockDim.x + threadIdx.x) / 32; b < tiles; b += warps) {
        const u64 o0 = o_begin + b * kMatTile;
        const u64 o_end = min(o0 + kMatTile, total);
        const u64 lo = upper_bound_warp(offsets, m + 1, o0) - 1;
        const u64 hi = upper_bound_warp(offsets, m + 1, o_end - 1) - 1;
        if (lane_id() == 0) {
            jlo[b] = lo;
            jhi[b] = hi;
        }
    }
}

struct MatShared {
    u32 owner[kMatTile];
    unsigned long long set[kMatSetSlots];  // tile-local key set (dedup modes only)
    u64 base;
    u32 warp[kMatBlock / 32 + 1];
    u32 set_fill;                           // keys inserted into `set` since its last reset
    unsigned long long tuples;              // word form: new tuples of this CTA (one global atomic at the end)
};

// One output tile of the output-partitioned join expansion (see lbs_kernel in
// column_ops.cu). All threads of the block call it for the same tile.
template <bool COMPACT, bool REMOTE, bool BLOCKS, bool WORDS>
__device__ __forceinline__ void materialize_tile(const u64* __restrict__ offsets, u64 o_begin, u64 total,
                                                 const u32* __restrict__ starts, const u64* __restrict__ tile_jlo,
                                                 const u64* __restrict__ tile_jhi, const OutSpec& spec, u64 t,
                                                 MatShared& sh, u32* __restrict__ s_acc) {
    u32* s_owner = sh.owner;
    unsigned long long* s_set = sh.set;
    u32* s_warp = sh.warp;
    u64& s_base = sh.base;
    const u32 tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const u64 o0 = o_begin + t * kMatTile;
    const u64 o_end = min(o0 + kMatTile, total);
    const u64 jlo = tile_jlo[t], jhi = tile_jhi[t];
    // A tile whose source rows span far more than its outputs is mostly
    // zero-count rows (probe misses): marking would walk every one of them,
    // so each output binary-searches its row instead (block-uniform branch).
    const bool sparse = jhi - jlo > u64(kMatSparseSpan);
    if (!sparse) {
        for (u32 i = tid; i < kMatTile; i += kMatBlock) s_owner[i] = 0;
        __syncthreads();
        for (u64 j = jlo + 1 + tid; j <= jhi; j += kMatBlock)
            atomicMax(&s_owner[offsets[j] - o0], static_cast<u32>(j - jlo));
        __syncthreads();
        u32 v[kMatItems];
        u32 run = 0;
#pragma unroll
        for (int k = 0; k < kMatItems; ++k) {
            run = max(run, s_owner[tid * kMatItems + k]);
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
        // carry-in = max over the earlier warps: one shared read per lane
        // and a warp max-reduction instead of a serial loop over them.
        u32 carry = __reduce_max_sync(0xffffffffu, lane < warp ? s_warp[lane] : 0u);
        const u32 prev = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane > 0) carry = max(carry, prev);
#pragma unroll
        for (int k = 0; k < kMatItems; ++k) s_owner[tid * kMatItems + k] = max(v[k], carry);
        __syncthreads();
    }
    // Items are strided by the block size so consecutive lanes take
    // consecutive outputs (coalesced build-side reads and output writes).
    u64 ii[kMatItems];
    u32 pp[kMatItems];
    u32 keep_mask = 0;
#pragma unroll
    for (int k = 0; k < kMatItems; ++k) {
        const u32 local = k * kMatBlock + tid;
        const u64 o = o0 + local;
        ii[k] = 0;
        pp[k] = 0;
        if (o < o_end) {
            const u64 i = sparse ? jlo + upper_bound_u64(offsets + jlo, jhi - jlo + 1, o) - 1 : jlo + s_owner[local];
            const u64 p = starts[i] + (o - offsets[i]);
            ii[k] = i;
            pp[k] = static_cast<u32>(p);
            if (!COMPACT || pass_filters(spec.f, spec.n_filters, i, p)) keep_mask |= 1u << k;
        }
    }
    if ((BLOCKS ? spec.bs.dir != nullptr : spec.ht_slots != nullptr) || spec.tile_dedup) {
        // Fused dedup. First a tile-local key set in shared memory drops the
        // repeats inside the tile: consecutive outputs share the probe row's
        // head columns, so one derivation per tile and key reaches HBM (about
        // half of all TC candidates are same-iteration repeats). Survivors
        // probe/insert FULL's key set; all first-slot loads are issued before
        // any is resolved (8 in flight per thread).
        u64 key[kMatItems], hs[kMatItems], sv[kMatItems];
#pragma unroll
        for (int k = 0; k < kMatItems; ++k) {
            key[k] = ((keep_mask >> k) & 1u) ? row_key1(spec, ii[k], pp[k]) : 0;
            hs[k] = keyset_line_hash(key[k], spec.ht_group_bits);
        }
        if constexpr (WORDS) {
            // Word form: each output is a whole DELTA word; OR it into FULL's
            // bitmap and append the bits that were new.
            u32 wb[kMatItems], first, ones, ovf_mask;
            if (spec.wbits.ptr) {
#pragma unroll
                for (int k = 0; k < kMatItems; ++k) wb[k] = ((keep_mask >> k) & 1u) ? slot(spec.wbits, ii[k], pp[k]) : 0;
                if (spec.word_neq) {
#pragma unroll
                    for (int k = 0; k < kMatItems; ++k) {
                        const u64 x = key[k] >> spec.shift, zb = key[k] & ((u64(1) << spec.shift) - 1);
                        if ((x & ~u64(31)) == zb) wb[k] &= ~(1u << static_cast<u32>(x & 31));
                        if (!wb[k]) keep_mask &= ~(1u << k);
                    }
                }
            } else {
                // tuple candidates into a word sink: one-bit words
#pragma unroll
                for (int k = 0; k < kMatItems; ++k) {
                    wb[k] = 0;
                    if ((keep_mask >> k) & 1u) {
                        key[k] = word_key_of(key[k], spec.shift, &wb[k]);
                        hs[k] = keyset_line_hash(key[k], spec.ht_group_bits);
                    }
                }
            }
            if (spec.cand_count) {
                u32 tc = 0;
#pragma unroll
                for (int k = 0; k < kMatItems; ++k)
                    if ((keep_mask >> k) & 1u) tc += __popc(wb[k]);
                tc = __reduce_add_sync(0xffffffffu, tc);
                if (lane == 0 && tc) atomicAdd(reinterpret_cast<unsigned long long*>(spec.cand_count), static_cast<unsigned long long>(tc));
            }
            if (spec.tile_set) {
                // Tile-local combine: outputs of one tile that hit the same
                // FULL word (one probe row's x with the same z word from
                // several DELTA rows) OR their masks in shared memory; only
                // the first of them goes to the global bitmap.
                __syncthreads();  // s_set / s_acc initialised (the sparse path has no barrier before this)
                u32 own = 0, joined = 0, hslot[kMatItems];
#pragma unroll
                for (int k = 0; k < kMatItems; ++k) {
                    hslot[k] = 0;
                    if (!((keep_mask >> k) & 1u)) continue;
                    u32 h = static_cast<u32>(hs[k] >> 40) & (kMatSetSlots - 1);
                    for (int probe = 0; probe < kMatSetProbes; ++probe) {
                        const unsigned long long prev = atomicCAS(s_set + h, ~0ull, static_cast<unsigned long long>(key[k]));
                        if (prev == ~0ull || prev == key[k]) {
                            (prev == ~0ull ? own : joined) |= 1u << k;
                            hslot[k] = h;
                            atomicOr(s_acc + h, wb[k]);
                            break;
                        }
                        h = (h + 1) & (kMatSetSlots - 1);
                    }
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < kMatItems; ++k)
                    if ((own >> k) & 1u) wb[k] = s_acc[hslot[k]];
                keep_mask &= ~joined;
            }
            if (spec.probe_count) {
                const u32 m = __reduce_add_sync(0xffffffffu, __popc(keep_mask));
                if (lane == 0 && m) atomicAdd(reinterpret_cast<unsigned long long*>(spec.probe_count), static_cast<unsigned long long>(m));
            }
            u32 widx[kMatItems];
            blockset_word_items(spec.bs, keep_mask, key, wb, &first, &ones, &ovf_mask, widx);
            append_words(spec.new_keys, spec.new_widx, spec.new_count, static_cast<u64*>(nullptr), 0u, first, key,
                         widx);
            {
                const u32 t = __reduce_add_sync(0xffffffffu, ones);
                if (lane == 0 && t) atomicAdd(&sh.tuples, static_cast<unsigned long long>(t));
            }
            append_words(spec.ovf_keys, spec.ovf_bits, spec.ovf_count, static_cast<u64*>(nullptr), 0u, ovf_mask, key,
                         wb);
            return;
        }
        __syncthreads();  // s_set initialised (the sparse path has no barrier before this)
#pragma unroll
        for (int k = 0; k < kMatItems; ++k) {
            if (!((keep_mask >> k) & 1u)) continue;
            u32 h = static_cast<u32>(hs[k] >> 40) & (kMatSetSlots - 1);
            for (int probe = 0; probe < (spec.tile_set ? kMatSetProbes : 0); ++probe) {
                const unsigned long long prev = atomicCAS(s_set + h, ~0ull, static_cast<unsigned long long>(key[k]));
                if (prev == ~0ull) break;                 // first in the tile
                if (prev == key[k]) {                     // repeat: drop
                    keep_mask &= ~(1u << k);
                    break;
                }
                h = (h + 1) & (kMatSetSlots - 1);
            }
            hs[k] = keyset_home(hs[k], key[k], spec.ht_group_bits, spec.ht_mask);
        }
        {
            const u32 m = __reduce_add_sync(0xffffffffu, __popc(keep_mask));
            if (lane == 0 && m) atomicAdd(&sh.set_fill, m);
        }
        if (REMOTE) {
            // Rows owned by another rank go to the routing pool (one
            // warp-aggregated append each) instead of the local key set.
            u32 remote_mask = 0;
#pragma unroll
            for (int k = 0; k < kMatItems; ++k) {
                if ((keep_mask >> k) & 1u) {
                    const u32 hv = static_cast<u32>(spec.n_out < 2 ? key[k]
                                                    : spec.remote_col ? key[k] & ((u64(1) << spec.shift) - 1)
                                                                      : key[k] >> spec.shift);
                    if (static_cast<u32>((static_cast<u64>(hash32(hv >> spec.remote_oshift)) * spec.remote_world) >> 32) !=
                        spec.remote_rank)
                        remote_mask |= 1u << k;
                }
            }
            append_new_items(spec.keys[0], spec.d_count, remote_mask, key);
            keep_mask &= ~remote_mask;
        }
        if (spec.probe_count) {
            const u32 m = __reduce_add_sync(0xffffffffu, __popc(keep_mask));
            if (lane == 0 && m) atomicAdd(reinterpret_cast<unsigned long long*>(spec.probe_count), static_cast<unsigned long long>(m));
        }
        if (spec.tile_dedup) {
            // Pooled candidates (partitioned runs route them before dedup):
            // append only the tile's distinct keys, one atomic per CTA.
            u32 tot;
            const u32 excl = block_excl_u32(__popc(keep_mask), s_warp, &tot);
            if (tid == 0)
                s_base = tot ? atomicAdd(reinterpret_cast<unsigned long long*>(spec.d_count),
                                         static_cast<unsigned long long>(tot))
                             : 0;
            __syncthreads();
            u64 pos = s_base + excl;
#pragma unroll
            for (int k = 0; k < kMatItems; ++k)
                if (keep_mask & (1u << k)) spec.keys[0][pos++] = key[k];
            return;
        }
        if constexpr (BLOCKS) {
            // Block-set dedup: survivors test-and-set their bit in FULL's
            // blocked bitmap (L2-resident for clustered relations).
            u32 ovf_mask;
            const u32 new_mask = blockset_insert_items(spec.bs, keep_mask, key, &ovf_mask);
            append_new_items(spec.new_keys, spec.new_count, new_mask, key);
            append_new_items(spec.ovf_keys, spec.ovf_count, ovf_mask, key);
            return;
        } else {
#pragma unroll
        for (int k = 0; k < kMatItems; ++k) sv[k] = ((keep_mask >> k) & 1u) ? __ldcg(spec.ht_slots + hs[k]) : 0;
        constexpr bool kBatchCas = FV_MAT_BATCH_CAS == 1 || (FV_MAT_BATCH_CAS == 2 && !COMPACT);
        if constexpr (kBatchCas) {
        // Every claim of an empty first slot is issued before any result is
        // read (the CASes are as independent as the loads); collisions with
        // another key fall back to the probe loop.
        u32 new_mask = 0, slow_mask = 0;
#pragma unroll
        for (int k = 0; k < kMatItems; ++k) {
            if (!((keep_mask >> k) & 1u) || sv[k] == key[k]) {
                keep_mask &= ~(1u << k);
            } else if (sv[k] == kEmptySlot) {
                sv[k] = atomicCAS(reinterpret_cast<unsigned long long*>(spec.ht_slots + hs[k]), ~0ull,
                                  static_cast<unsigned long long>(key[k]));
            }
        }
#pragma unroll
        for (int k = 0; k < kMatItems; ++k) {
            if (!((keep_mask >> k) & 1u)) continue;
            if (sv[k] == kEmptySlot) new_mask |= 1u << k;          // claimed
            else if (sv[k] != key[k]) slow_mask |= 1u << k;        // another key there
        }
#pragma unroll
        for (int k = 0; k < kMatItems; ++k)
            if (((slow_mask >> k) & 1u) &&
                keyset_insert_probe_from(spec.ht_slots, spec.ht_mask, key[k], (hs[k] + 1) & spec.ht_mask))
                new_mask |= 1u << k;
#if FV_MAT_APPEND_CTA
        {
            u32 tot;
            const u32 excl = block_excl_u32(__popc(new_mask), s_warp, &tot);
            if (tid == 0)
                s_base = tot ? atomicAdd(reinterpret_cast<unsigned long long*>(spec.new_count),
                                         static_cast<unsigned long long>(tot))
                             : 0;
            __syncthreads();
            u64 pos = s_base + excl;
#pragma unroll
            for (int k = 0; k < kMatItems; ++k)
                if ((new_mask >> k) & 1u) spec.new_keys[pos++] = key[k];
        }
#else
        append_new_items(spec.new_keys, spec.new_count, new_mask, key);
#endif
        } else {
#pragma unroll
        for (int k = 0; k < kMatItems; ++k) {
            const bool keep = (keep_mask >> k) & 1u;
            const bool is_new = keep && keyset_insert_from(spec.ht_slots, spec.ht_mask, key[k], hs[k], sv[k]);
            append_new(spec.new_keys, spec.new_count, is_new, key[k]);
        }
        }
        }
        return;
    }
    if (!COMPACT) {
#pragma unroll
        for (int k = 0; k < kMatItems; ++k)
            if (keep_mask & (1u << k)) write_row(spec, o0 + k * kMatBlock + tid, ii[k], pp[k]);
        return;
    }
    u32 tot;
    const u32 excl = block_excl_u32(__popc(keep_mask), s_warp, &tot);
    if (tid == 0) s_base = tot ? atomicAdd(reinterpret_cast<unsigned long long*>(spec.d_count),
                                           static_cast<unsigned long long>(tot))
                               : 0;
    __syncthreads();
    u64 pos = s_base + excl;
#pragma unroll
    for (int k = 0; k < kMatItems; ++k)
        if (keep_mask & (1u << k)) write_row(spec, pos++, ii[k], pp[k]);
}

// Dedup modes can walk `group` consecutive tiles per CTA and keep the
// tile-local key set across them (reset once a quarter full, so a tile's
// 2048 keys never push it past 3/4): a high-degree probe row's outputs span
// many tiles and their repeats only meet when the set outlives one tile.
// That halves TC's key-set probes, but the dropped ones were L2 hits and the
// serialised tiles cost more than they save, so the default is one tile.
constexpr int kMatGroup = 1;  // measured: 1 is best on C1-C4 (FVLOG_MAT_GROUP overrides)
// REMOTE: partitioned fused dedup (spec.remote_world > 0), a separate
// instantiation so the single-GPU kernel keeps its register budget.
// Three 512-thread CTAs per SM (<= 42 registers): C2 125 -> 121 ms, C4 208 ->
// 194 ms against the compiler's unbounded choice (48 registers, 2 CTAs).
#ifndef FV_MAT_MIN_BLOCKS
#define FV_MAT_MIN_BLOCKS 3
#endif
#ifndef FV_MAT_MIN_BLOCKS_BS
#define FV_MAT_MIN_BLOCKS_BS 2
#endif
// Word form: 3 CTAs per SM (40 registers, a 136-byte spill) beat 2 (60
// registers): C2 24.7 -> 23.7 ms, C3 18.4 -> 17.1, C4 73.4 -> 70.4 (4 CTAs:
// 32 registers, 332-byte spill, 24.7 ms).
#ifndef FV_MAT_MIN_BLOCKS_W
#define FV_MAT_MIN_BLOCKS_W 3
#endif
template <bool COMPACT, bool REMOTE, bool BLOCKS, bool WORDS>
__global__ void __launch_bounds__(kMatBlock, WORDS ? FV_MAT_MIN_BLOCKS_W : (BLOCKS ? FV_MAT_MIN_BLOCKS_BS : FV_MAT_MIN_BLOCKS)) materialize_kernel(const u64* __restrict__ offsets, u64 m,
                                                                 u64 o_begin, u64 total,
                                                                 const u32* __restrict__ starts,
                                                                 const u64* __restrict__ tile_jlo,
                                                                 const u64* __restrict__ tile_jhi, u64 tiles,
                                                                 u32 group, OutSpec spec) {
    __shared__ MatShared sh;
    extern __shared__ u32 s_acc[];  // word form only: combined masks of the tile set (kMatSetSlots, dynamic)
    const bool dedup = (BLOCKS ? spec.bs.dir != nullptr : spec.ht_slots != nullptr) || spec.tile_dedup;
    const u64 t0 = u64(blockIdx.x) * group;
    const u64 t1 = min(t0 + group, tiles);
    if (WORDS && threadIdx.x == 0) sh.tuples = 0;  // ordered by the loop's first barrier
    for (u64 t = t0; t < t1; ++t) {
        __syncthreads();  // previous tile's shared reads/updates are done
        const bool reset = dedup && (t == t0 || sh.set_fill > kMatSetSlots / 4);
        __syncthreads();  // every thread has read set_fill before it is cleared
        if (reset) {
            for (u32 i = threadIdx.x; i < kMatSetSlots; i += kMatBlock) {
                sh.set[i] = ~0ull;
                if (WORDS) s_acc[i] = 0;
            }
            if (threadIdx.x == 0) sh.set_fill = 0;
            __syncthreads();
        }
        materialize_tile<COMPACT, REMOTE, BLOCKS, WORDS>(offsets, o_begin, total, starts, tile_jlo, tile_jhi, spec, t, sh,
                                                         s_acc);
    }
    if (WORDS) {
        __syncthreads();
        if (threadIdx.x == 0 && sh.tuples) atomicAdd(reinterpret_cast<unsigned long long*>(spec.new_tuples), sh.tuples);
    }
}

template <bool COMPACT>
__global__ void __launch_bounds__(kMatBlock) project_kernel(u64 n, OutSpec spec) {
    __shared__ u32 s_warp[kMatBlock / 32 + 1];
    __shared__ u64 s_base;
    const u64 r0 = u64(blockIdx.x) * kMatTile;
    u32 keep_mask = 0;
#pragma unroll
    for (int k = 0; k < kMatItems; ++k) {
        const u64 i = r0 + k * kMatBlock + threadIdx.x;
        if (i < n && (!COMPACT || pass_filters(spec.f, spec.n_filters, i, 0))) keep_mask |= 1u << k;
    }
    if (!COMPACT) {
#pragma unroll
        for (int k = 0; k < kMatItems; ++k)
            if (keep_mask & (1u << k)) {
                const u64 i = r0 + k * kMatBlock + threadIdx.x;
                write_row(spec, i, i, 0);
            }
        return;
    }
    u32 tot;
    const u32 excl = block_excl_u32(__popc(keep_mask), s_warp, &tot);
    if (threadIdx.x == 0)
        s_base = tot ? atomicAdd(reinterpret_cast<unsigned long long*>(spec.d_count),
                                 static_cast<unsigned long long>(tot))
                     : 0;
    __syncthreads();
    u64 pos = s_base + excl;
#pragma unroll
    for (int k = 0; k < kMatItems; ++k)
        if (keep_mask & (1u << k)) {
            const u64 i = r0 + k * kMatBlock + threadIdx.x;
            write_row(spec, pos++, i, 0);
        }
}

// ---- runs / hash for join indexes ------------------------------------------------

struct RunsOp {
    const u32* keys;
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

// Direct-address run index of sorted keys: the first row of each run stores
// its position at the run's value, the last row its length.
// (keys >= domain: the 0xffffffff tail of a word build sized by its bound,
// not indexed)
// Run (start, end) of every value into pair[2v], pair[2v + 1] (pair cleared:
// end 0 = no run).
__global__ void direct_runs_kernel(const u32* __restrict__ keys, u64 n, u32* __restrict__ pair, u64 domain) {
    GRID_STRIDE(i, n) {
        const u32 k = keys[i];
        if (k >= domain) continue;
        if (i == 0 || keys[i - 1] != k) pair[2 * u64(k)] = static_cast<u32>(i);
        if (i + 1 == n || keys[i + 1] != k) pair[2 * u64(k) + 1] = static_cast<u32>(i + 1);
    }
}

// d_nu (optional): the run count on the device; nu is then only its bound.
__global__ void runs_count_kernel(const u32* __restrict__ ustart, u32* __restrict__ ucount, u64 nu, u64 n,
                                  const u64* __restrict__ d_nu) {
    if (d_nu) nu = *d_nu;
    GRID_STRIDE(i, nu) {
        const u64 end = i + 1 < nu ? ustart[i + 1] : n;
        ucount[i] = static_cast<u32>(end - ustart[i]);
    }
}

__global__ void hash_build_kernel(const u32* __restrict__ ukeys, u64 nu, unsigned long long* __restrict__ slots,
                                  u32 mask, const u64* __restrict__ d_nu) {
    if (d_nu) nu = *d_nu;
    GRID_STRIDE(i, nu) {
        const u32 key = ukeys[i];
        const unsigned long long packed = (static_cast<unsigned long long>(key) << 32) | u32(i);
        u32 h = hash32(key) & mask;
        while (atomicCAS(slots + h, ~0ull, packed) != ~0ull) h = (h + 1) & mask;
    }
}

// ---- keys ------------------------------------------------------------------------------

struct Cols8 {
    const u32* p[FV_MAX_ARITY];
};
struct OutCols8 {
    u32* p[FV_MAX_ARITY];
};
struct Words4 {
    u64* p[4];
};

__device__ __forceinline__ u64 pack_word(const Cols8& c, u32 arity, u32 w, u64 row, u32 shift) {
    const u64 hi = c.p[2 * w][row];
    if (2 * w + 1 < arity) return (hi << shift) | c.p[2 * w + 1][row];
    return hi;
}

__global__ void pack_kernel(Cols8 c, u32 arity, u64 n, u32 shift, Words4 out) {
    const u32 W = (arity + 1) / 2;
    GRID_STRIDE(i, n) {
        for (u32 w = 0; w < W; ++w) out.p[w][i] = pack_word(c, arity, w, i, shift);
    }
}

__global__ void gather_u64_kernel(const u64* __restrict__ src, const u32* __restrict__ idx,
                                  u64* __restrict__ out, u64 n) {
    GRID_STRIDE(i, n) out[i] = src[idx[i]];
}

// ---- merge-path unique + difference + merge ---------------------------------------------

template <int W>
struct Key {
    u64 w[W];
};

template <int W>
__device__ __forceinline__ bool key_le(const Key<W>& a, const Key<W>& b) {
#pragma unroll
    for (int k = 0; k < W; ++k)
        if (a.w[k] != b.w[k]) return a.w[k] < b.w[k];
    return true;
}
template <int W>
__device__ __forceinline__ bool key_eq(const Key<W>& a, const Key<W>& b) {
#pragma unroll
    for (int k = 0; k < W; ++k)
        if (a.w[k] != b.w[k]) return false;
    return true;
}

template <int W>
__device__ __forceinline__ Key<W> load_a(const Cols8& a, u32 arity, u64 row, u32 shift) {
    Key<W> k;
#pragma unroll
    for (int w = 0; w < W; ++w) k.w[w] = pack_word(a, arity, w, row, shift);
    return k;
}
template <int W>
__device__ __forceinline__ Key<W> load_b(const Words4& b, u64 row) {
    Key<W> k;
#pragma unroll
    for (int w = 0; w < W; ++w) k.w[w] = b.p[w][row];
    return k;
}

template <int W>
__device__ __forceinline__ void store_row(const OutCols8& out, u32 arity, u32 shift, u64 pos, const Key<W>& k) {
    const u64 lo_mask = shift >= 64 ? ~u64(0) : ((u64(1) << shift) - 1);
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const u32 c0 = 2 * w;
        if (c0 + 1 < arity) {
            out.p[c0][pos] = static_cast<u32>(k.w[w] >> shift);
            out.p[c0 + 1][pos] = static_cast<u32>(k.w[w] & lo_mask);
        } else if (c0 < arity) {
            out.p[c0][pos] = static_cast<u32>(k.w[w]);
        }
    }
}

template <int W>
struct MergeTraits {
    static constexpr int kItems = W == 1 ? 8 : (W == 2 ? 4 : 2);
    static constexpr int kBlock = 256;
    static constexpr int kTile = kItems * kBlock;
};

template <int W>
__device__ u64 merge_path_global(const Cols8& a, u32 arity, u32 shift, u64 n_a, const Words4& b, u64 n_b, u64 d) {
    u64 lo = d > n_b ? d - n_b : 0;
    u64 hi = d < n_a ? d : n_a;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (key_le<W>(load_a<W>(a, arity, mid, shift), load_b<W>(b, d - 1 - mid))) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Merge-path split of every tile boundary, one thread per boundary (all
// binary searches in parallel instead of serially inside each merge CTA).
template <int W>
__global__ void merge_partition_kernel(Cols8 a, u64 n_a, Words4 b, u64 n_b, u32 arity, u32 shift, u64 tiles,
                                       u64* __restrict__ splits) {
    constexpr int TILE = MergeTraits<W>::kTile;
    GRID_STRIDE(t, tiles + 1) {
        const u64 d = min(u64(t) * TILE, n_a + n_b);
        splits[t] = merge_path_global<W>(a, arity, shift, n_a, b, n_b, d);
    }
}

template <int W>
__global__ void __launch_bounds__(MergeTraits<W>::kBlock)
    merge_kernel(Cols8 a, u64 n_a, Words4 b, u64 n_b, u32 arity, u32 shift, OutCols8 cout, OutCols8 dout,
                 const u64* __restrict__ splits, u64* __restrict__ status, u32 epoch, u32* __restrict__ tile_counter,
                 u64* __restrict__ d_new) {
    constexpr int ITEMS = MergeTraits<W>::kItems;
    constexpr int BLOCK = MergeTraits<W>::kBlock;
    constexpr int TILE = MergeTraits<W>::kTile;
    // Padded tiles (one slot per 16): each thread walks its own stretch of
    // the merge, so lanes access keys ~ITEMS apart; without padding those
    // strided u64 accesses hit the same banks (16-way conflicts).
    constexpr int PADDED = TILE + TILE / 16;
    __shared__ Key<W> s_keys[PADDED];  // inputs: A part then B part; later C outputs
    __shared__ Key<W> s_dout[PADDED];
    auto pad = [](u32 i) { return i + (i >> 4); };
    __shared__ u32 s_tile;
    __shared__ u64 s_a0, s_a1, s_dups_before;
    __shared__ Key<W> s_prev;
    __shared__ int s_has_prev;
    __shared__ u64 s_warp64[BLOCK / 32 + 1];

    const u32 tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const u32 tile = s_tile;
    const u64 total = n_a + n_b;
    const u64 d0 = u64(tile) * TILE;
    const u64 d1 = min(d0 + TILE, total);
    if (tid == 0) {
        const u64 a0 = splits[tile];
        const u64 a1 = splits[tile + 1];
        s_a0 = a0;
        s_a1 = a1;
        const u64 b0 = d0 - a0;
        int has = 0;
        Key<W> pv;
        if (a0 > 0) {
            pv = load_a<W>(a, arity, a0 - 1, shift);
            has = 1;
        }
        if (b0 > 0) {
            const Key<W> pb = load_b<W>(b, b0 - 1);
            if (!has || key_le<W>(pv, pb)) pv = pb;
            has = 1;
        }
        if (has) s_prev = pv;
        s_has_prev = has;
    }
    __syncthreads();
    const u64 a0 = s_a0, a1 = s_a1;
    const u64 b0 = d0 - a0, b1 = d1 - a1;
    const u32 na = static_cast<u32>(a1 - a0), nb = static_cast<u32>(b1 - b0);
#define SA(i) s_keys[pad(i)]
#define SB(j) s_keys[pad(na + (j))]
    for (u32 j = tid; j < na; j += BLOCK) SA(j) = load_a<W>(a, arity, a0 + j, shift);
    for (u32 j = tid; j < nb; j += BLOCK) SB(j) = load_b<W>(b, b0 + j);
    __syncthreads();

    // Thread-level merge path inside the tile.
    const u32 len = na + nb;
    const u32 t0 = min(tid * ITEMS, len);
    u32 lo = t0 > nb ? t0 - nb : 0, hi = min(t0, na);
    while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (key_le<W>(SA(mid), SB(t0 - 1 - mid))) lo = mid + 1;
        else hi = mid;
    }
    u32 ai = lo, bi = t0 - lo;
    Key<W> prev;
    bool has_prev;
    if (t0 == 0) {
        has_prev = s_has_prev != 0;
        if (has_prev) prev = s_prev;
    } else {
        has_prev = true;
        if (ai > 0 && bi > 0) prev = key_le<W>(SA(ai - 1), SB(bi - 1)) ? SB(bi - 1) : SA(ai - 1);
        else if (ai > 0) prev = SA(ai - 1);
        else prev = SB(bi - 1);
    }
    Key<W> item[ITEMS];
    u32 valid = 0, from_b = 0, dup = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (t0 + k < len) {
            const bool take_a = bi >= nb || (ai < na && key_le<W>(SA(ai), SB(bi)));
            const Key<W> key = take_a ? SA(ai) : SB(bi);
            if (take_a) ++ai;
            else ++bi;
            valid |= 1u << k;
            if (!take_a) {
                from_b |= 1u << k;
                if (has_prev && key_eq<W>(key, prev)) dup |= 1u << k;
            }
            item[k] = key;
            prev = key;
            has_prev = true;
        }
    }
    const u32 nondup = __popc(valid & ~dup);
    const u32 nondup_b = __popc(from_b & ~dup);
    // One block scan over both counts packed in a u64.
    u64 agg;
    const u64 excl = block_exclusive_scan<BLOCK>((u64(nondup_b) << 32) | nondup, s_warp64, &agg);
    const u32 tile_nondup = static_cast<u32>(agg), tile_nondup_b = static_cast<u32>(agg >> 32);
    const u64 tile_dups = u64(len) - tile_nondup;

    if (tid < 32) {
        u64 before = 0;
        if (tile == 0) {
            if (tid == 0) st_relaxed_u64(status, lb_pack(epoch, kLbFlagInclusive, tile_dups));
        } else {
            if (tid == 0) st_relaxed_u64(status + tile, lb_pack(epoch, kLbFlagAggregate, tile_dups));
            before = lookback_warp(status, tile, epoch);
            if (tid == 0) st_relaxed_u64(status + tile, lb_pack(epoch, kLbFlagInclusive, before + tile_dups));
        }
        if (tid == 0) s_dups_before = before;
    }
    __syncthreads();  // also: all reads of sA/sB done before reuse below
    const u64 dups_before = s_dups_before;
    u32 cpos = static_cast<u32>(excl);
    u32 dpos = static_cast<u32>(excl >> 32);
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u32 bit = 1u << k;
        if ((valid & bit) && !(dup & bit)) {
            s_keys[pad(cpos++)] = item[k];
            if (from_b & bit) s_dout[pad(dpos++)] = item[k];
        }
    }
    __syncthreads();
#undef SA
#undef SB
    const u64 c_base = d0 - dups_before;
    const u64 d_base = b0 - dups_before;
    for (u32 j = tid; j < tile_nondup; j += BLOCK) store_row<W>(cout, arity, shift, c_base + j, s_keys[pad(j)]);
    for (u32 j = tid; j < tile_nondup_b; j += BLOCK)
        store_row<W>(dout, arity, shift, d_base + j, s_dout[pad(j)]);
    if (tid == 0 && d1 == total) *d_new = d_base + tile_nondup_b;
}

// ---- fingerprint ------------------------------------------------------------------------

__global__ void fingerprint_kernel(Cols8 c, u32 arity, u64 n, unsigned long long* out) {
    unsigned long long acc = 0;
    GRID_STRIDE(i, n) {
        u64 h = 0x2545F4914F6CDD1Dull;
        for (u32 j = 0; j < arity; ++j) h = mix64(h ^ c.p[j][i]);
        acc += h;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane_id() == 0) atomicAdd(out, acc);
}

// Fingerprint of a block set's rows straight from its bitmaps (the same sum
// over rows as fingerprint_kernel): one thread per bitmap word.
__global__ void blockset_fingerprint_kernel(const u64* __restrict__ dir, const u32* __restrict__ bits, u64 cap,
                                            u32 arity, unsigned long long* out) {
    unsigned long long acc = 0;
    GRID_STRIDE(t, cap * 32) {
        const u64 slot = t >> 5;
        const u32 r = static_cast<u32>(t & 31);
        const u64 bid = dir[slot];
        if (bid == kEmptySlot) continue;
        u32 w = bits[t];
        while (w) {
            const u32 b = __ffs(w) - 1;
            w &= w - 1;
            u64 h = 0x2545F4914F6CDD1Dull;
            if (arity == 2) {
                h = mix64(h ^ static_cast<u32>((bid >> 27) * 32 + r));
                h = mix64(h ^ static_cast<u32>((bid & ((u64(1) << 27) - 1)) * 32 + b));
            } else {
                h = mix64(h ^ static_cast<u32>(bid * 1024 + r * 32 + b));
            }
            acc += h;
        }
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane_id() == 0) atomicAdd(out, acc);
}

}  // namespace

u64 engine_blockset_fingerprint(Ctx* c, const BlockSet& s, u32 arity) {
    const u64 cap = s.capacity();
    if (!cap) return 0;
    u64* d = c->d_scalars + 43;
    FV_CUDA(cudaMemsetAsync(d, 0, 8, c->stream));
    {
        ProfScope prof(c, "fingerprint", 136.0 * double(cap));
        blockset_fingerprint_kernel<<<grid_for(cap * 32), 256, 0, c->stream>>>(
            s.dir.get(), s.bits.get(), cap, arity, reinterpret_cast<unsigned long long*>(d));
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    }
    u64 h = 0;
    c->read_scalars(d, &h, 1);
    return h;
}

namespace {

#ifndef FV_INSERT_ITEMS
#define FV_INSERT_ITEMS 4
#endif
#ifdef FV_INSERT_MINB
#define FV_INSERT_BOUNDS __launch_bounds__(256, FV_INSERT_MINB)
#else
#define FV_INSERT_BOUNDS
#endif
// Four keys per thread. With one counter atomic and one CAS round trip per
// item, one key per thread was best (partitioned C2: 167.6 ms at 8, 97 at 1);
// with the claims batched and one append atomic per warp for all items, more
// items keep more independent loads in flight (8-rank C2 on one GPU, all
// ranks' inserts under ncu: 113 ms at 1 key/thread, 96 at 2, 76 at 4, 74 at 8).
constexpr int kInsertItems = FV_INSERT_ITEMS;
__global__ void FV_INSERT_BOUNDS hash_insert_keys_kernel(const u64* __restrict__ keys, u64 n,
                                                         u64* __restrict__ slots, u64 mask, u32 bits,
                                                         u64* __restrict__ new_keys, u64* new_count) {
    constexpr int ITEMS = kInsertItems;
    const u64 base = u64(blockIdx.x) * blockDim.x * ITEMS + threadIdx.x;
    u64 key[ITEMS], hs[ITEMS], sv[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u64 i = base + u64(k) * blockDim.x;
        key[k] = i < n ? keys[i] : 0;
        hs[k] = keyset_home(keyset_line_hash(key[k], bits), key[k], bits, mask);
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) sv[k] = (base + u64(k) * blockDim.x < n) ? __ldcg(slots + hs[k]) : 0;
    // As in the fused join: claims of empty first slots issued together,
    // collisions through the probe loop, one counter atomic per warp.
    u32 new_mask = 0, slow_mask = 0, cas_mask = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (base + u64(k) * blockDim.x >= n || sv[k] == key[k]) continue;
        if (sv[k] == kEmptySlot) {
            sv[k] = atomicCAS(reinterpret_cast<unsigned long long*>(slots + hs[k]), ~0ull,
                              static_cast<unsigned long long>(key[k]));
            cas_mask |= 1u << k;
        } else {
            slow_mask |= 1u << k;
        }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        if (!((cas_mask >> k) & 1u)) continue;
        if (sv[k] == kEmptySlot) new_mask |= 1u << k;
        else if (sv[k] != key[k]) slow_mask |= 1u << k;
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k)
        if (((slow_mask >> k) & 1u) && keyset_insert_probe_from(slots, mask, key[k], (hs[k] + 1) & mask))
            new_mask |= 1u << k;
    if (new_keys) append_new_items(new_keys, new_count, new_mask, key);
}

// Block-set insert of n keys (pooled candidates, seeds, routed rows): four
// keys per thread, the same batched path as the fused join.
__global__ void blockset_insert_kernel(const u64* __restrict__ keys, u64 n, BlockSetArgs s,
                                       u64* __restrict__ new_keys, u64* new_count, u64* __restrict__ ovf,
                                       u64* ovf_count) {
    constexpr int ITEMS = 4;
    const u64 base = u64(blockIdx.x) * blockDim.x * ITEMS + threadIdx.x;
    u64 key[ITEMS];
    u32 live = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u64 i = base + u64(k) * blockDim.x;
        key[k] = i < n ? keys[i] : 0;
        if (i < n) live |= 1u << k;
    }
    u32 om;
    const u32 nm = blockset_insert_items(s, live, key, &om);
    if (new_keys) append_new_items(new_keys, new_count, nm, key);
    append_new_items(ovf, ovf_count, om, key);
}

// Word-form block-set insert of n entries: word keys with their masks
// (bits_in), or packed binary tuple keys (bits_in null) turned into one-bit
// words. Words first written to DELTA this iteration are appended to
// new_keys (new bits counted in *new_tuples), entries without a directory
// slot go to the overflow list with their full mask.
#ifndef FV_INSERT_WARP_COMBINE
#define FV_INSERT_WARP_COMBINE 1
#endif
__global__ void blockset_word_insert_kernel(const u64* __restrict__ keys, const u32* __restrict__ bits_in, u64 n,
                                            BlockSetArgs s, u64* __restrict__ new_keys, u32* __restrict__ new_widx,
                                            u64* new_count, u64* new_tuples, u64* __restrict__ ovf,
                                            u32* __restrict__ ovf_bits, u64* ovf_count) {
    constexpr int ITEMS = 4;
    const u64 base = u64(blockIdx.x) * blockDim.x * ITEMS + threadIdx.x;
    u64 key[ITEMS];
    u32 b[ITEMS];
    u32 live = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u64 i = base + u64(k) * blockDim.x;
        key[k] = 0;
        b[k] = 0;
        if (i < n) {
            if (bits_in) {
                key[k] = keys[i];
                b[k] = bits_in[i];
            } else {
                key[k] = word_key_of(keys[i], s.shift, &b[k]);
            }
            live |= 1u << k;
        }
    }
#if FV_INSERT_WARP_COMBINE
    // Lanes holding the same word (sorted inputs: a seed or a copy of a
    // sorted version — consecutive keys share words and blocks) OR their
    // masks first; only one of them goes to the set.
    const u32 lane = lane_id();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u64 wk = ((live >> k) & 1u) ? key[k] : ~u64(lane);  // out-of-range lanes: unique
        const u32 peers = __match_any_sync(0xffffffffu, wk);
        const u32 m = __reduce_or_sync(peers, b[k]);
        if ((live >> k) & 1u) {
            if (lane == static_cast<u32>(__ffs(peers) - 1)) b[k] = m;
            else live &= ~(1u << k);
        }
    }
#endif
    u32 om, first, ones, widx[ITEMS];
    blockset_word_items(s, live, key, b, &first, &ones, &om, widx);
    append_words(new_keys, new_widx, new_count, new_tuples, ones, first, key, widx);
    append_words(ovf, ovf_bits, ovf_count, static_cast<u64*>(nullptr), 0u, om, key, b);
}

// DELTA's merged masks: entry i (a word first written this iteration) reads
// its block's DELTA bitmap word and clears it for the next iteration. With
// widx (no directory growth since the entries were appended) the word index
// recorded at append time is used; otherwise the block is looked up.
// Read-and-clear of the DELTA words by atomicExch (one L2 request per
// word) instead of a load and a store: C2 23.46 -> 21.77 ms.
#ifndef FV_COLLECT_EXCH
#define FV_COLLECT_EXCH 1
#endif
#ifndef FV_COLLECT_ITEMS
#define FV_COLLECT_ITEMS 4
#endif
constexpr int kCollectItems = FV_COLLECT_ITEMS;  // independent gathers in flight per thread
__global__ void blockset_collect_kernel(const u64* __restrict__ keys, const u32* __restrict__ widx, u64 n,
                                        BlockSetArgs s, u32* __restrict__ out) {
    const u64 base = u64(blockIdx.x) * blockDim.x * kCollectItems + threadIdx.x;
    u64 w[kCollectItems];
#pragma unroll
    for (int k = 0; k < kCollectItems; ++k) {
        const u64 i = base + u64(k) * blockDim.x;
        w[k] = ~u64(0);
        if (i >= n) continue;
        if (widx) {
            w[k] = widx[i];
        } else {
            u32 bp;
            const u64 bid = block_of(keys[i], s.shift, 2, &bp);
            u64 h = block_home(bid, s.mask);
            while (__ldcg(s.dir + h) != bid) h = (h + 1) & s.mask;  // present: inserted this iteration
            w[k] = h * 32 + (bp >> 5);
        }
    }
    u32 v[kCollectItems];
#if FV_COLLECT_EXCH
    // read-and-clear as one L2 atomic per word (one request instead of a
    // load and a store: the kernel is bound by the random requests)
#pragma unroll
    for (int k = 0; k < kCollectItems; ++k) v[k] = w[k] != ~u64(0) ? atomicExch(s.dbits + w[k], 0u) : 0;
#pragma unroll
    for (int k = 0; k < kCollectItems; ++k)
        if (w[k] != ~u64(0)) out[base + u64(k) * blockDim.x] = v[k];
#else
#pragma unroll
    for (int k = 0; k < kCollectItems; ++k) v[k] = w[k] != ~u64(0) ? __ldcg(s.dbits + w[k]) : 0;
#pragma unroll
    for (int k = 0; k < kCollectItems; ++k) {
        if (w[k] == ~u64(0)) continue;
        out[base + u64(k) * blockDim.x] = v[k];
        s.dbits[w[k]] = 0;
    }
#endif
}


// Exclusive prefix of the masks' popcounts (the tuples' output offsets).
struct PopcOffsetsOp {
    const u32* bits;
    u64* off;  // n + 1 entries: off[n] = the total
    u64 n;
    __device__ u64 value(u64 i) const { return __popc(bits[i]); }
    __device__ void emit(u64 i, u64 p, u64 v) const {
        off[i] = p;
        if (i == n - 1) off[n] = p + v;
    }
};

// Warp-cooperative expansion of word entries into packed tuple keys: a warp
// takes 32 consecutive words and writes their tuples 32 at a time, each
// lane finding its word by a shuffle search over the warp's offsets and its
// bit with __fns, so the writes are coalesced (a thread-per-word loop writes
// up to 32 scattered rows per thread).
// out_x (optional): the tuples as SoA columns (x = key >> shift, z) instead
// of packed keys.
__global__ void expand_word_keys_kernel(const u64* __restrict__ keys, const u32* __restrict__ bits,
                                        const u64* __restrict__ off, u64 n, u64* __restrict__ out,
                                        u32* __restrict__ out_x, u32* __restrict__ out_z, u32 shift) {
    const u32 lane = lane_id();
    const u64 warps = (n + 31) / 32;
    for (u64 w = (u64(blockIdx.x) * blockDim.x + threadIdx.x) / 32; w < warps;
         w += (u64(gridDim.x) * blockDim.x) / 32) {
        const u64 i = w * 32 + lane;
        const bool valid = i < n;
        const u64 k = valid ? keys[i] : 0;
        const u32 m = valid ? bits[i] : 0;
        const u64 o = valid ? off[i] : 0;
        const u64 base = __shfl_sync(0xffffffffu, o, 0);
        const u32 rel = static_cast<u32>(o - base);  // this word's first output within the warp
        const u32 cnt = __popc(m);
        u32 tot = valid ? rel + cnt : 0;  // the warp's output count: the largest end offset
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) tot = max(tot, __shfl_xor_sync(0xffffffffu, tot, d));
        for (u32 j = 0; j < tot; j += 32) {
            const u32 t = j + lane;  // output index within the warp's range
            // last word whose first output <= t (words with no bits are skipped)
            u32 lo = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const u32 cand = lo + step;
                const u32 r = __shfl_sync(0xffffffffu, valid ? rel : 0xffffffffu, cand);
                if (r <= t) lo = cand;
            }
            const u32 wr = __shfl_sync(0xffffffffu, rel, lo);
            const u32 wm = __shfl_sync(0xffffffffu, m, lo);
            const u64 wk = __shfl_sync(0xffffffffu, k, lo);
            if (t < tot) {
                const u32 b = __fns(wm, 0, t - wr + 1);
                if (out_x) {
                    out_x[base + t] = static_cast<u32>(wk >> shift);
                    out_z[base + t] = static_cast<u32>(wk & ((u64(1) << shift) - 1)) + b;
                } else {
                    out[base + t] = wk + b;
                }
            }
        }
    }
}

// Words of a lexicographically sorted binary version: one entry per run of
// rows with the same (x, z >> 5) (runs are at most 32 rows: rows are distinct).
struct TuplesToWordsOp {
    const u32* c0;
    const u32* c1;
    u64 n;
    u32* x;
    u32* zb;
    u32* bits;
    __device__ u64 value(u64 i) const {
        return (i == 0 || c0[i] != c0[i - 1] || (c1[i] >> 5) != (c1[i - 1] >> 5)) ? 1 : 0;
    }
    // Every row ORs its bit into its word (p + v - 1: the word starts
    // before it, this one included); bits[] is zeroed first. (A serial walk
    // from each word start was latency-bound: 188 us for 7 M rows.)
    __device__ void emit(u64 i, u64 p, u64 v) const {
        const u32 z = c1[i];
        if (v) {
            x[p] = c0[i];
            zb[p] = z & ~31u;
        }
        atomicOr(bits + (p + v - 1), 1u << (z & 31));
    }
};

// Tuples of word entries (x, z base, mask), in entry order: entry i's set
// bits become rows (x, base + bit) at its prefix of the popcounts.
struct ExpandWordsOp {
    const u32* x;
    const u32* zb;
    const u32* bits;
    u32* out_x;
    u32* out_z;
    __device__ u64 value(u64 i) const { return __popc(bits[i]); }
    __device__ void emit(u64 i, u64 p, u64 v) const {
        if (!v || !out_x) return;  // counting pass
        const u32 xi = x[i], z0 = zb[i];
        u32 m = bits[i];
        while (m) {
            const u32 b = __ffs(m) - 1;
            m &= m - 1;
            out_x[p] = xi;
            out_z[p] = z0 + b;
            ++p;
        }
    }
};

__global__ void set_u64_kernel(u64* p, u64 v) { *p = v; }

// p[i] = (p[i] & and_mask) | or_bits
__global__ void mask_u64_kernel(u64* __restrict__ p, u64 n, u64 and_mask, u64 or_bits) {
    GRID_STRIDE(i, n) p[i] = (p[i] & and_mask) | or_bits;
}

// Block ids of packed keys (the distinct count sizes a directory).
__global__ void block_ids_kernel(const u64* __restrict__ keys, u64 n, u32 shift, u32 arity, u64* __restrict__ out) {
    GRID_STRIDE(i, n) {
        u32 bp;
        out[i] = block_of(keys[i], shift, arity, &bp);
    }
}

// HyperLogLog sketch of the distinct block ids of n packed keys (2^12
// registers, ~1.6 % standard error): one pass, shared-memory registers per
// CTA merged with one atomicMax each. Sizes block-set directories, where a
// few percent do not matter and the exact count's 54-bit radix sort does.
constexpr int kHllBits = 12;
constexpr int kHllRegs = 1 << kHllBits;
__global__ void block_sketch_kernel(const u64* __restrict__ keys, u64 n, u32 shift, u32 arity, u32* __restrict__ regs) {
    __shared__ u32 s[kHllRegs];
    for (u32 i = threadIdx.x; i < kHllRegs; i += blockDim.x) s[i] = 0;
    __syncthreads();
    GRID_STRIDE(i, n) {
        u32 bp;
        // arity 0: the distinct keys themselves (not their blocks)
        const u64 h = mix64(arity ? block_of(keys[i], shift, arity, &bp) : keys[i]);
        const u32 idx = static_cast<u32>(h >> (64 - kHllBits));
        const u32 rho = static_cast<u32>(__clzll((h << kHllBits) | (u64(1) << (kHllBits - 1)))) + 1;
        atomicMax(s + idx, rho);
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < kHllRegs; i += blockDim.x)
        if (s[i]) atomicMax(regs + i, s[i]);
}

struct DistinctOp {
    const u64* v;
    __device__ u64 value(u64 i) const { return (i == 0 || v[i] != v[i - 1]) ? 1 : 0; }
    __device__ void emit(u64, u64, u64) const {}
};

// ---- sorted rows straight from a block set (dumps of block-set relations) -----------
//
// The bitmaps hold FULL exactly, so the lexicographic dump needs no sort of
// the tuples: the used directory slots are compacted and their block ids
// radix-sorted (10^6 blocks for C2's 6.5·10^8 tuples), then every (block,
// row) bitmap word is placed in row-major output order — for block row A
// with blocks j0..j1 (ascending b), word r of block j is item
// 32·j0 + r·(j1 - j0) + (j - j0) — its popcount prefix-summed and its bits
// written as rows.

struct BlockCompactOp {
    const u64* dir;
    u64* bids;
    u32* slots;
    __device__ u64 value(u64 i) const { return dir[i] != kEmptySlot ? 1 : 0; }
    __device__ void emit(u64 i, u64 p, u64 v) const {
        if (!v) return;
        bids[p] = dir[i];
        slots[p] = static_cast<u32>(i);
    }
};

// First block of every block row (binary: bid >> 27) among the sorted ids.
struct RowStartOp {
    const u64* bids;
    u32* starts;
    __device__ u64 value(u64 j) const { return (j == 0 || (bids[j] >> 27) != (bids[j - 1] >> 27)) ? 1 : 0; }
    __device__ void emit(u64 j, u64 p, u64 v) const {
        if (v) starts[p] = static_cast<u32>(j);
    }
};

__device__ __forceinline__ void block_item(const u32* __restrict__ starts, u64 rows, u64 m, u64 j, u32 r, u32 arity,
                                           u64* g) {
    if (arity != 2) {
        *g = j * 32 + r;
        return;
    }
    // block row of j: last start <= j
    u64 lo = 0, hi = rows;
    while (hi - lo > 1) {
        const u64 mid = (lo + hi) >> 1;
        if (starts[mid] <= j) lo = mid;
        else hi = mid;
    }
    const u64 j0 = starts[lo], j1 = lo + 1 < rows ? starts[lo + 1] : m;
    *g = 32 * j0 + u64(r) * (j1 - j0) + (j - j0);
}

// words = 0: the item's tuple count (popcount); 1: whether it is a non-empty word.
__global__ void block_count_kernel(const u64* __restrict__ bids, const u32* __restrict__ slots,
                                   const u32* __restrict__ bits, const u32* __restrict__ starts, u64 rows, u64 m,
                                   u32 arity, u32 words, u32* __restrict__ cnt) {
    GRID_STRIDE(t, m * 32) {
        const u64 j = t >> 5;
        const u32 r = static_cast<u32>(t & 31);
        u64 g;
        block_item(starts, rows, m, j, r, arity, &g);
        const u32 w = bits[u64(slots[j]) * 32 + r];
        cnt[g] = words ? (w != 0) : __popc(w);
    }
}

// The non-empty bitmap words in row-major order: (x, z base, mask).
__global__ void block_words_kernel(const u64* __restrict__ bids, const u32* __restrict__ slots,
                                   const u32* __restrict__ bits, const u32* __restrict__ starts, u64 rows, u64 m,
                                   const u64* __restrict__ off, u32* __restrict__ x, u32* __restrict__ zb,
                                   u32* __restrict__ wbits) {
    GRID_STRIDE(t, m * 32) {
        const u64 j = t >> 5;
        const u32 r = static_cast<u32>(t & 31);
        const u32 w = bits[u64(slots[j]) * 32 + r];
        if (!w) continue;
        u64 g;
        block_item(starts, rows, m, j, r, 2, &g);
        const u64 pos = off[g];
        const u64 bid = bids[j];
        x[pos] = static_cast<u32>((bid >> 27) * 32 + r);
        zb[pos] = static_cast<u32>((bid & ((u64(1) << 27) - 1)) * 32);
        wbits[pos] = w;
    }
}

__global__ void block_expand_kernel(const u64* __restrict__ bids, const u32* __restrict__ slots,
                                    const u32* __restrict__ bits, const u32* __restrict__ starts, u64 rows, u64 m,
                                    u32 arity, const u64* __restrict__ off, u32* __restrict__ c0,
                                    u32* __restrict__ c1) {
    GRID_STRIDE(t, m * 32) {
        const u64 j = t >> 5;
        const u32 r = static_cast<u32>(t & 31);
        u32 w = bits[u64(slots[j]) * 32 + r];
        if (!w) continue;
        u64 g;
        block_item(starts, rows, m, j, r, arity, &g);
        u64 pos = off[g];
        const u64 bid = bids[j];
        if (arity == 2) {
            const u32 a = static_cast<u32>((bid >> 27) * 32 + r);
            const u32 b0 = static_cast<u32>((bid & ((u64(1) << 27) - 1)) * 32);
            while (w) {
                const u32 b = __ffs(w) - 1;
                w &= w - 1;
                c0[pos] = a;
                c1[pos] = b0 + b;
                ++pos;
            }
        } else {
            const u32 v0 = static_cast<u32>(bid * 1024 + r * 32);
            while (w) {
                const u32 b = __ffs(w) - 1;
                w &= w - 1;
                c0[pos++] = v0 + b;
            }
        }
    }
}

// Directory growth: every used old slot re-homed in the new directory, its
// 128-byte bitmap moved with 16-byte vector loads/stores. Block ids are
// distinct, so a block only has to find an empty slot.
__global__ void blockset_grow_kernel(const u64* __restrict__ from_dir, const u32* __restrict__ from_bits,
                                     const u32* __restrict__ from_dbits, u64 n, BlockSetArgs to) {
    GRID_STRIDE(i, n) {
        const u64 bid = __ldcs(from_dir + i);
        if (bid == kEmptySlot) continue;
        u64 h = block_home(bid, to.mask);
        while (atomicCAS(reinterpret_cast<unsigned long long*>(to.dir + h), ~0ull,
                         static_cast<unsigned long long>(bid)) != ~0ull)
            h = (h + 1) & to.mask;
        const uint4* src = reinterpret_cast<const uint4*>(from_bits + i * 32);
        uint4* dst = reinterpret_cast<uint4*>(to.bits + h * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = __ldcs(src + q);
        if (to.dbits) {  // word form: the block's DELTA bitmap moves along
            const uint4* dsrc = reinterpret_cast<const uint4*>(from_dbits + i * 32);
            uint4* ddst = reinterpret_cast<uint4*>(to.dbits + h * 32);
#pragma unroll
            for (int q = 0; q < 8; ++q) ddst[q] = __ldcs(dsrc + q);
        }
    }
}

// One tile of consecutive old slots per block (not grid-stride): blocks run
// roughly in index order, so the inserts of all resident blocks fall into a
// few narrow windows of the new table that stay in L2.
constexpr int kRehashItems = 8;
__global__ void hash_rehash_kernel(const u64* __restrict__ from, u64 n, u64* __restrict__ to, u64 mask, u32 bits) {
    const u64 base = u64(blockIdx.x) * blockDim.x * kRehashItems + threadIdx.x;
    u64 key[kRehashItems];
#pragma unroll
    for (int k = 0; k < kRehashItems; ++k) {
        const u64 i = base + u64(k) * blockDim.x;
        key[k] = i < n ? __ldcs(from + i) : kEmptySlot;
    }
    // Keys are distinct: a key only has to find an empty slot. All first-slot
    // loads, then all claims, are in flight together; the rest probe on.
    u64 hs[kRehashItems], sv[kRehashItems];
#pragma unroll
    for (int k = 0; k < kRehashItems; ++k) {
        hs[k] = keyset_home(keyset_line_hash(key[k], bits), key[k], bits, mask);
        sv[k] = key[k] != kEmptySlot ? __ldcg(to + hs[k]) : 0;
    }
#pragma unroll
    for (int k = 0; k < kRehashItems; ++k)
        if (key[k] != kEmptySlot && sv[k] == kEmptySlot)
            sv[k] = atomicCAS(reinterpret_cast<unsigned long long*>(to + hs[k]), ~0ull,
                              static_cast<unsigned long long>(key[k]));
#pragma unroll
    for (int k = 0; k < kRehashItems; ++k)
        if (key[k] != kEmptySlot && sv[k] != kEmptySlot)
            keyset_insert_probe_from(to, mask, key[k], (hs[k] + 1) & mask);
}

// Growth without a memset or global atomics. With the new capacity F times
// the old (same layout bits), a key's new home is its old home + j * old
// capacity for some j < F, so the keys of one tile of old slots [a, a + T)
// land in the F windows [a + j * old, a + j * old + T), which partition the
// new table. A block builds each of its windows in shared memory (linear
// probing with shared atomics) and streams it out whole, empty slots
// included. Keys that cannot be placed inside their window — their home lies
// in an earlier tile (displaced across the tile boundary) or their probe run
// reaches the window's end — go to an overflow list that a plain insert
// places afterwards, when every slot has been written.
#ifndef FV_GROW_VEC
#define FV_GROW_VEC 1
#endif
#ifndef FV_GROW_MINB
#define FV_GROW_MINB 5  // 48 registers, 5 blocks per SM: C2 93.1 -> 92.8 ms, C3 31.2 -> 30.9 (1: 58 registers, 4 blocks)
#endif
constexpr int kGrowItems = 8;
constexpr int kGrowBlock = 256;
constexpr u32 kGrowTile = kGrowItems * kGrowBlock;
__global__ void __launch_bounds__(kGrowBlock, FV_GROW_MINB) hash_grow_kernel(const u64* __restrict__ from, u64 old_cap,
                                                               u32 log_old, u32 factor, u64* __restrict__ to,
                                                               u64 new_mask, u32 bits, u64* __restrict__ overflow,
                                                               u64 overflow_cap, u64* overflow_count) {
    __shared__ __align__(16) unsigned long long win[kGrowTile];
    const u64 a = u64(blockIdx.x) * kGrowTile;
    u64 key[kGrowItems];
    u32 local[kGrowItems];
    u32 jj[kGrowItems];
    u32 spill = 0;  // bit k: key k goes to the overflow list
#pragma unroll
    for (int k = 0; k < kGrowItems; ++k) {
        const u64 i = a + u64(k) * kGrowBlock + threadIdx.x;
        key[k] = i < old_cap ? __ldcs(from + i) : kEmptySlot;
        local[k] = 0;
        jj[k] = 0;
        if (key[k] == kEmptySlot) continue;
        const u64 h = keyset_home(keyset_line_hash(key[k], bits), key[k], bits, new_mask);
        const u64 lo = h & (old_cap - 1);
        jj[k] = static_cast<u32>(h >> log_old);
        if (lo < a || lo >= a + kGrowTile) spill |= 1u << k;
        else local[k] = static_cast<u32>(lo - a);
    }
    for (u32 j = 0; j < factor; ++j) {
        for (u32 i = threadIdx.x; i < kGrowTile; i += kGrowBlock) win[i] = ~0ull;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kGrowItems; ++k) {
            if (key[k] == kEmptySlot || jj[k] != j || ((spill >> k) & 1u)) continue;
            u32 q = local[k];
            while (true) {
                if (atomicCAS(win + q, ~0ull, static_cast<unsigned long long>(key[k])) == ~0ull) break;
                if (++q == kGrowTile) {  // run leaves the window
                    spill |= 1u << k;
                    break;
                }
            }
        }
        __syncthreads();
        const u64 w0 = a + (u64(j) << log_old);
#if FV_GROW_VEC
        // 16-byte streaming stores (windows start at multiples of the tile).
        for (u32 i = 2 * threadIdx.x; i < kGrowTile; i += 2 * kGrowBlock)
            __stcs(reinterpret_cast<ulonglong2*>(to + w0 + i), *reinterpret_cast<const ulonglong2*>(win + i));
#else
        for (u32 i = threadIdx.x; i < kGrowTile && a + i < old_cap; i += kGrowBlock) __stcs(to + w0 + i, static_cast<u64>(win[i]));
#endif
        __syncthreads();
    }
    // Overflow keys (rare: about one per tile). The count keeps growing past
    // the list's capacity so the host can see that it must fall back.
    const u32 lane = lane_id();
    const u32 cnt = __popc(spill);
    u32 incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<u32>(o)) incl += y;
    }
    const u32 total = __shfl_sync(0xffffffffu, incl, 31);
    if (!total) return;
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(reinterpret_cast<unsigned long long*>(overflow_count), static_cast<unsigned long long>(total));
    u64 pos = __shfl_sync(0xffffffffu, base, 31) + (incl - cnt);
#pragma unroll
    for (int k = 0; k < kGrowItems; ++k)
        if ((spill >> k) & 1u) {
            if (pos < overflow_cap) overflow[pos] = key[k];
            ++pos;
        }
}

// ---- grouping of one-word keys by their first column (counting sort) ----------------
//
// Levels-mode DELTA only has to be grouped by column 0 for its join index
// (rows of one column-0 value contiguous, any order inside). With a domain of
// at most 2^kGroupMaxBits first-column values that is a counting sort: count
// per value (shared-nothing L2 atomics on a small counter array), scan, and
// scatter each key to base[value] + atomicAdd(cursor[value]) — two reads and
// one write of the keys instead of a histogram plus three onesweep passes.
// DELTA arrives in probe-row order, so a value's keys come in short runs
// (interleaved by the join's per-warp appends): every warp aggregates equal
// values with __match_any_sync and takes one atomic per distinct value, the
// group's lanes writing consecutive slots. Warps whose 32 keys share one
// value skip the match.
#ifndef FV_GROUP_MATCH
#define FV_GROUP_MATCH 1
#endif

__global__ void group_count_kernel(const u64* __restrict__ keys, u64 n, u32 shift, u32* __restrict__ cnt) {
    const u64 n_round = ceil_div(n, 32) * 32;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n_round; i += u64(gridDim.x) * blockDim.x) {
        const bool valid = i < n;
        const u32 g = valid ? static_cast<u32>(keys[i] >> shift) : ~0u;
        const u32 g0 = __shfl_sync(0xffffffffu, g, 0);
        if (__all_sync(0xffffffffu, g == g0)) {
            if (lane_id() == 0 && valid) atomicAdd(cnt + g0, 32u);
        } else {
#if FV_GROUP_MATCH
            const u32 peers = __match_any_sync(0xffffffffu, g);
            if (valid && lane_id() == __ffs(peers) - 1) atomicAdd(cnt + g, static_cast<u32>(__popc(peers)));
#else
            if (valid) atomicAdd(cnt + g, 1u);
#endif
        }
    }
}

__global__ void group_scatter_kernel(const u64* __restrict__ keys, u64 n, u32 shift, const u64* __restrict__ base,
                                     u32* __restrict__ cursor, u64* __restrict__ out, u32* __restrict__ c0,
                                     u32* __restrict__ c1, const u32* __restrict__ pay_in,
                                     u32* __restrict__ pay_out, const u32* __restrict__ gather_idx,
                                     u32* __restrict__ gather_src) {
    const u64 n_round = ceil_div(n, 32) * 32;
    const u32 lane = lane_id();
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n_round; i += u64(gridDim.x) * blockDim.x) {
        const bool valid = i < n;
        const u64 key = valid ? keys[i] : 0;
        const u32 g = valid ? static_cast<u32>(key >> shift) : ~0u;
        const u32 g0 = __shfl_sync(0xffffffffu, g, 0);
        u64 pos;
        if (__all_sync(0xffffffffu, g == g0)) {
            u32 b = 0;
            if (lane == 0 && valid) b = atomicAdd(cursor + g0, 32u);
            pos = valid ? base[g0] + __shfl_sync(0xffffffffu, b, 0) + lane : 0;
        } else {
#if FV_GROUP_MATCH
            const u32 peers = __match_any_sync(0xffffffffu, g);
            const u32 leader = __ffs(peers) - 1;
            u32 b = 0;
            if (valid && lane == leader) b = atomicAdd(cursor + g, static_cast<u32>(__popc(peers)));
            b = __shfl_sync(0xffffffffu, b, leader);
            pos = valid ? base[g] + b + __popc(peers & ((1u << lane) - 1)) : 0;
#else
            pos = valid ? base[g] + atomicAdd(cursor + g, 1u) : 0;
#endif
        }
        if (valid) {
            if (pay_out) {  // word masks travel with their keys
                if (gather_idx) {  // read (and clear) from the DELTA bitmap: no separate collect pass
                    const u32 w = gather_idx[i];
                    pay_out[pos] = gather_src[w];
                    gather_src[w] = 0;
                } else {
                    pay_out[pos] = pay_in[i];
                }
            }
            if (c0) {  // unpacked straight into SoA columns
                c0[pos] = g;
                c1[pos] = static_cast<u32>(key & ((u64(1) << shift) - 1));
            } else {
                out[pos] = key;
            }
        }
    }
}

// Runs of the grouped keys straight from the counters: one row per non-empty
// value (value, base, count) — the column-0 join index of the grouped DELTA
// without a pass over its rows.

struct GroupBaseOp {
    const u32* cnt;
    u64* base;
    u32* base32;  // optional: the run starts as u32 (direct-address join index)
    __device__ u64 value(u64 i) const { return cnt[i]; }
    __device__ void emit(u64 i, u64 p, u64) const {
        base[i] = p;
        if (base32) base32[i] = static_cast<u32>(p);
    }
};

__global__ void unpack_keys_kernel(const u64* __restrict__ keys, u64 n, u32 arity, u32 shift, u32* c0, u32* c1) {
    const u64 lo_mask = (u64(1) << shift) - 1;
    GRID_STRIDE(i, n) {
        const u64 k = keys[i];
        if (arity == 2) {
            c0[i] = static_cast<u32>(k >> shift);
            c1[i] = static_cast<u32>(k & lo_mask);
        } else {
            c0[i] = static_cast<u32>(k);
        }
    }
}

// SoA columns -> row-major rows (the dump layout), one row per thread.
__global__ void interleave_kernel(Cols8 c, u32 arity, u64 n, u32* __restrict__ out) {
    GRID_STRIDE(i, n) {
#pragma unroll
        for (int j = 0; j < FV_MAX_ARITY; ++j) {
            if (j >= static_cast<int>(arity)) break;
            out[i * arity + j] = c.p[j][i];
        }
    }
}

// Distinct rows of sorted packed keys, unpacked into SoA columns (one
// look-back compaction: a row is kept when any word differs from its
// predecessor's).
struct UniqueUnpackOp {
    Words4 w;
    u32 words, arity, shift;
    OutCols8 out;
    __device__ u64 value(u64 i) const {
        if (i == 0) return 1;
        for (u32 k = 0; k < words; ++k)
            if (w.p[k][i] != w.p[k][i - 1]) return 1;
        return 0;
    }
    __device__ void emit(u64 i, u64 pos, u64 v) const {
        if (!v) return;
        const u64 lo_mask = (u64(1) << shift) - 1;
        for (u32 k = 0; k < words; ++k) {
            const u64 x = w.p[k][i];
            if (2 * k + 1 < arity) {
                out.p[2 * k][pos] = static_cast<u32>(x >> shift);
                out.p[2 * k + 1][pos] = static_cast<u32>(x & lo_mask);
            } else {
                out.p[2 * k][pos] = static_cast<u32>(x);
            }
        }
    }
};

constexpr int kMaxRanks = 64;
constexpr u32 kGroupMaxBits = 24;       // engine_group_keys: counter arrays of <= 16 M entries
constexpr u32 kGroupMaxPerValue = 512;  // ... and at most this many keys per value on average
// engine_build_runs: builds of at most this many rows size their run arrays
// and hash table by the rows (no host read of the run count).
constexpr u64 kRunsBoundRows = u64(1) << 20;

__device__ __forceinline__ u32 route_dest(const RouteKey& k, u64 i, u32 world) {
    u32 v;
    if (k.col) v = k.col[i];
    else v = static_cast<u32>(k.hi ? (k.word[i] >> k.shift) : (k.word[i] & k.mask));
    return static_cast<u32>((static_cast<u64>(hash32(v >> k.oshift)) * world) >> 32);
}

__global__ void route_cursor_kernel(const u64* counts, u64* cursors, u32 world) {
    u64 run = 0;
    for (u32 p = 0; p < world; ++p) {
        cursors[p] = run;
        run += counts[p];
    }
}

__global__ void route_count_kernel(RouteKey key, u64 n, u32 world, unsigned long long* counts) {
    __shared__ u32 s_cnt[kMaxRanks];
    for (u32 p = threadIdx.x; p < world; p += blockDim.x) s_cnt[p] = 0;
    __syncthreads();
    GRID_STRIDE(i, n) atomicAdd(&s_cnt[route_dest(key, i, world)], 1u);
    __syncthreads();
    for (u32 p = threadIdx.x; p < world; p += blockDim.x)
        if (s_cnt[p]) atomicAdd(counts + p, static_cast<unsigned long long>(s_cnt[p]));
}

__global__ void route_scatter_kernel(RouteKey key, u64 n, u32 world, unsigned long long* cursor, Cols8 in32,
                                     OutCols8 out32, u32 n32, Words4 in64, Words4 out64, u32 n64) {
    __shared__ u32 s_cnt[kMaxRanks];
    __shared__ u64 s_base[kMaxRanks];
    constexpr int ITEMS = 8;
    const u64 r0 = u64(blockIdx.x) * blockDim.x * ITEMS;
    for (u32 p = threadIdx.x; p < world; p += blockDim.x) s_cnt[p] = 0;
    __syncthreads();
    u32 dest[ITEMS], rank[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u64 i = r0 + u64(k) * blockDim.x + threadIdx.x;
        dest[k] = i < n ? route_dest(key, i, world) : 0;
        rank[k] = i < n ? atomicAdd(&s_cnt[dest[k]], 1u) : 0;
    }
    __syncthreads();
    for (u32 p = threadIdx.x; p < world; p += blockDim.x)
        s_base[p] = s_cnt[p] ? atomicAdd(cursor + p, static_cast<unsigned long long>(s_cnt[p])) : 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u64 i = r0 + u64(k) * blockDim.x + threadIdx.x;
        if (i >= n) continue;
        const u64 pos = s_base[dest[k]] + rank[k];
        for (u32 j = 0; j < n32; ++j) out32.p[j][pos] = in32.p[j][i];
        for (u32 j = 0; j < n64; ++j) out64.p[j][pos] = in64.p[j][i];
    }
}

struct SelectRowsOp {
    RowFilter pred;
    u32* ids;
    __device__ u64 value(u64 i) const { return pass_filters(pred.f, pred.n, i, 0) ? 1 : 0; }
    __device__ void emit(u64 i, u64 p, u64 v) const {
        if (v) ids[p] = static_cast<u32>(i);
    }
};
}  // namespace

// ---- host launchers -------------------------------------------------------------------------

void engine_hash_insert(Ctx* c, const u64* keys, u64 n, KeySet& set, u64* new_keys, u64* d_new) {
    if (!n) return;
    ProfScope prof(c, "hash_insert", double(n) * (8.0 + 16.0));
    hash_insert_keys_kernel<<<static_cast<unsigned>(ceil_div(n, 256 * kInsertItems)), 256, 0, c->stream>>>(
        keys, n, set.slots.get(), set.mask, set.group_bits, new_keys, d_new);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void engine_blockset_alloc(Ctx* c, BlockSet& s, u64 cap, u64 blocks, bool delta_bits) {
    s.dir = DBuf<u64>(c, cap);
    s.bits = DBuf<u32>(c, cap * 32);
    s.dbits = delta_bits ? DBuf<u32>(c, cap * 32) : DBuf<u32>();
    if (delta_bits) FV_CUDA(cudaMemsetAsync(s.dbits.get(), 0, 128 * cap, c->stream));
    s.count = DBuf<u64>(c, 1);
    s.mask = cap - 1;
    s.blocks = blocks;
    FV_CUDA(cudaMemsetAsync(s.dir.get(), 0xff, 8 * cap, c->stream));
    FV_CUDA(cudaMemsetAsync(s.bits.get(), 0, 128 * cap, c->stream));
    set_u64_kernel<<<1, 1, 0, c->stream>>>(s.count.get(), blocks);  // stream-ordered, no host sync
    FV_CUDA(cudaGetLastError());
}

void engine_blockset_grow(Ctx* c, const BlockSet& from, BlockSet& to) {
    const u64 n = from.capacity();
    if (!n) return;
    BlockSetArgs a;
    a.dir = to.dir.get();
    a.bits = to.bits.get();
    a.dbits = from.dbits.get() ? to.dbits.get() : nullptr;
    a.mask = to.mask;
    const double per_block = a.dbits ? 264.0 : 136.0;
    ProfScope prof(c, "blockset_grow", per_block * double(n) + per_block * double(to.blocks));
    blockset_grow_kernel<<<grid_for(n), 256, 0, c->stream>>>(from.dir.get(), from.bits.get(), from.dbits.get(), n,
                                                              a);
    FV_CUDA(cudaGetLastError());
    FV_CUDA(cudaMemcpyAsync(to.count.get(), from.count.get(), 8, cudaMemcpyDeviceToDevice, c->stream));
    c->count_launch();
}

void engine_blockset_insert(Ctx* c, const u64* keys, u64 n, const BlockSetArgs& s, u64* new_keys, u64* d_new,
                            u64* ovf, u64* d_ovf) {
    if (!n) return;
    ProfScope prof(c, "blockset_insert", 16.0 * double(n));
    const unsigned grid = static_cast<unsigned>(ceil_div(n, u64(256) * 4));
    blockset_insert_kernel<<<grid, 256, 0, c->stream>>>(keys, n, s, new_keys, d_new, ovf, d_ovf);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void engine_blockset_word_insert(Ctx* c, const u64* keys, const u32* bits, u64 n, const BlockSetArgs& s,
                                 u64* new_keys, u32* new_widx, u64* d_new, u64* d_tuples, u64* ovf, u32* ovf_bits,
                                 u64* d_ovf) {
    if (!n) return;
    ProfScope prof(c, "blockset_insert", (bits ? 12.0 : 8.0) * double(n));
    const unsigned grid = static_cast<unsigned>(ceil_div(n, u64(256) * 4));
    blockset_word_insert_kernel<<<grid, 256, 0, c->stream>>>(keys, bits, n, s, new_keys, new_widx, d_new, d_tuples,
                                                             ovf, ovf_bits, d_ovf);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void engine_blockset_collect(Ctx* c, const u64* keys, const u32* widx, u64 n, const BlockSetArgs& s, u32* out_bits) {
    if (!n) return;
    ProfScope prof(c, "blockset_collect", (widx ? 16.0 : 20.0) * double(n));
    blockset_collect_kernel<<<static_cast<unsigned>(ceil_div(n, u64(256) * kCollectItems)), 256, 0, c->stream>>>(
        keys, widx, n, s, out_bits);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void engine_expand_word_keys(Ctx* c, const u64* keys, const u32* bits, u64 n, u64* out, u32* out_x, u32* out_z,
                             u32 shift, u64* off_out) {
    if (!n) return;
    DBuf<u64> off_own;
    u64* off = off_out;
    if (!off) {
        off_own = DBuf<u64>(c, n + 1);
        off = off_own.get();
    }
    ProfScope prof(c, "expand_words", 12.0 * double(n));
    tile_scan(c, PopcOffsetsOp{bits, off, n}, n, nullptr);
    expand_word_keys_kernel<<<grid_for(n), 256, 0, c->stream>>>(keys, bits, off, n, out, out_x, out_z, shift);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

u64 engine_tuples_to_words(Ctx* c, const u32* c0, const u32* c1, u64 n, u32* x, u32* zb, u32* bits, bool exact) {
    if (!n) return 0;
    u64* d = c->d_scalars + 45;
    // Not exact: the n rows past the words keep x = 0xffffffff (outside
    // every value domain below 2^32: no index holds them, no probe meets
    // them) and the bound n is returned without a host round trip.
    if (!exact) FV_CUDA(cudaMemsetAsync(x, 0xff, 4 * n, c->stream));
    FV_CUDA(cudaMemsetAsync(bits, 0, 4 * n, c->stream));
    {
        ProfScope prof(c, "tuples_to_words", 8.0 * double(n));
        tile_scan(c, TuplesToWordsOp{c0, c1, n, x, zb, bits}, n, d);
    }
    if (!exact) return n;
    u64 total = 0;
    c->read_scalars(d, &total, 1);
    return total;
}

u64 engine_expand_words(Ctx* c, const u32* x, const u32* zb, const u32* bits, u64 n, u32* out_x, u32* out_z,
                        bool count) {
    if (!n) return 0;
    u64* d = c->d_scalars + 40;
    {
        ProfScope prof(c, "expand_words", 12.0 * double(n));
        tile_scan(c, ExpandWordsOp{x, zb, bits, out_x, out_z}, n, d);
    }
    if (!count) return 0;
    u64 total = 0;
    c->read_scalars(d, &total, 1);
    return total;
}

u64 engine_count_blocks(Ctx* c, const u64* keys, u64 n, u32 shift, u32 arity) {
    if (!n) return 0;
    u64* d = c->d_scalars + 42;
    engine_count_blocks_async(c, keys, n, shift, arity, d);
    u64 m = 0;
    c->read_scalars(d, &m, 1);
    return m;
}

void engine_count_blocks_async(Ctx* c, const u64* keys, u64 n, u32 shift, u32 arity, u64* d_out) {
    if (!n) {
        FV_CUDA(cudaMemsetAsync(d_out, 0, 8, c->stream));
        return;
    }
    DBuf<u64> ids(c, n), alt(c, n);
    {
        ProfScope prof(c, "count_blocks", 16.0 * double(n));
        block_ids_kernel<<<grid_for(n), 256, 0, c->stream>>>(keys, n, shift, arity, ids.get());
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    }
    if (radix_sort_keys_u64(c, ids.get(), alt.get(), n, 0, 54)) ids.swap(alt);
    tile_scan(c, DistinctOp{ids.get()}, n, d_out);
}

namespace {
// Sorted block ids (with their slots) and block-row starts of a block set.
struct SortedBlocks {
    DBuf<u64> bids;
    DBuf<u32> slots, starts;
    u64 m = 0, rows = 0;
};

// x_bits > 0: only group the blocks by their row group (block id bits
// [27, 27 + x_bits): x >> 5) instead of a full (x, z) order — enough for
// consumers that need each x's words together but not z-ordered.
SortedBlocks sorted_blocks(Ctx* c, const BlockSet& s, u32 arity, u32 x_bits = 0) {
    SortedBlocks b;
    const u64 cap = s.capacity();
    u64* d = c->d_scalars + 41;
    b.bids = DBuf<u64>(c, cap);
    b.slots = DBuf<u32>(c, cap);
    DBuf<u64> bids_alt(c, cap);
    DBuf<u32> slots_alt(c, cap);
    {
        ProfScope prof(c, "blockset_dump", 8.0 * double(cap));
        tile_scan(c, BlockCompactOp{s.dir.get(), b.bids.get(), b.slots.get()}, cap, d);
    }
    c->read_scalars(d, &b.m, 1);
    if (!b.m) return b;
    // binary ids are (a >> 5) << 27 | (b >> 5): bits [0, 27) and [27, 54)
    const u32 lo_bit = x_bits ? 27 : 0, hi_bit = x_bits ? std::min(54u, 27 + x_bits) : 54;
    if (radix_sort_pairs_u64(c, b.bids.get(), bids_alt.get(), b.slots.get(), slots_alt.get(), b.m, lo_bit, hi_bit)) {
        b.bids.swap(bids_alt);
        b.slots.swap(slots_alt);
    }
    b.starts = DBuf<u32>(c, arity == 2 ? b.m : 1);
    if (arity == 2) {
        tile_scan(c, RowStartOp{b.bids.get(), b.starts.get()}, b.m, d);
        c->read_scalars(d, &b.rows, 1);
    }
    return b;
}
}  // namespace

u64 engine_blockset_words(Ctx* c, const BlockSet& s, u32* x, u32* zb, u32* bits, u64 cap_out, u32 key_shift) {
    if (!s.capacity()) return 0;
    // words grouped by x (a join index on x needs no z order): the blocks
    // are sorted on their row group only (3 radix passes instead of 7)
    SortedBlocks b = sorted_blocks(c, s, 2, key_shift > 5 ? key_shift - 5 : 1);
    if (!b.m) return 0;
    const u64 items = b.m * 32;
    DBuf<u32> cnt(c, items);
    DBuf<u64> off(c, items + 1);
    ProfScope prof(c, "blockset_words", 136.0 * double(b.m));
    block_count_kernel<<<grid_for(items), 256, 0, c->stream>>>(b.bids.get(), b.slots.get(), s.bits.get(),
                                                                b.starts.get(), b.rows, b.m, 2, 1, cnt.get());
    FV_CUDA(cudaGetLastError());
    exclusive_scan_counts(c, cnt.get(), off.get(), items);
    FV_CUDA(cudaMemcpyAsync(c->pinned, off.get() + items, 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    const u64 total = c->pinned[0];
    if (total > cap_out) fail(FV_ERR_INVALID, "blockset_words: more words than the output holds");
    block_words_kernel<<<grid_for(items), 256, 0, c->stream>>>(b.bids.get(), b.slots.get(), s.bits.get(),
                                                                b.starts.get(), b.rows, b.m, off.get(), x, zb, bits);
    FV_CUDA(cudaGetLastError());
    c->count_launch(2);
    return total;
}

u64 engine_blockset_dump(Ctx* c, const BlockSet& s, u32 arity, u32* c0, u32* c1) {
    const u64 cap = s.capacity();
    if (!cap) return 0;
    SortedBlocks b = sorted_blocks(c, s, arity);
    const u64 m = b.m, rows = b.rows;
    if (!m) return 0;
    DBuf<u64>& bids = b.bids;
    DBuf<u32>& slots = b.slots;
    DBuf<u32>& starts = b.starts;
    DBuf<u32> cnt(c, m * 32);
    DBuf<u64> off(c, m * 32 + 1);
    u64 total = 0;
    {
        ProfScope prof(c, "blockset_dump", 136.0 * double(m));
        block_count_kernel<<<grid_for(m * 32), 256, 0, c->stream>>>(bids.get(), slots.get(), s.bits.get(),
                                                                     starts.get(), rows, m, arity, 0, cnt.get());
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    }
    exclusive_scan_counts(c, cnt.get(), off.get(), m * 32);
    {
        FV_CUDA(cudaMemcpyAsync(c->pinned, off.get() + m * 32, 8, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        total = c->pinned[0];
    }
    if (c0) {
        ProfScope prof(c, "blockset_dump", 4.0 * double(arity) * double(total));
        block_expand_kernel<<<grid_for(m * 32), 256, 0, c->stream>>>(bids.get(), slots.get(), s.bits.get(),
                                                                      starts.get(), rows, m, arity, off.get(),
                                                                      c0, c1);
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    }
    return total;
}

void engine_hash_rehash(Ctx* c, const KeySet& from, KeySet& to) {
    const u64 n = from.capacity();
    if (!n) return;
    // Algorithmic bytes: the old table read once, each key written once.
    ProfScope prof(c, "hash_rehash", double(n) * 8.0 + double(from.count) * 8.0);
    hash_rehash_kernel<<<static_cast<unsigned>(ceil_div(n, 256 * kRehashItems)), 256, 0, c->stream>>>(
        from.slots.get(), n, to.slots.get(), to.mask, to.group_bits);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

bool engine_hash_grow(Ctx* c, const KeySet& from, KeySet& to) {
    const u64 old_cap = from.capacity(), new_cap = to.capacity();
    if (!old_cap || new_cap <= old_cap || from.group_bits != to.group_bits || old_cap % kGrowTile) return false;
    const u64 factor = new_cap / old_cap;
    u32 log_old = 0;
    while ((u64(1) << log_old) < old_cap) ++log_old;
    // Overflow list: a few keys per tile are expected; more (a pathological
    // clustering) falls back to the memset + atomic rehash.
    // FVLOG_GROW_OVERFLOW_CAP (tests): a tiny list forces the fallback.
    const char* forced = std::getenv("FVLOG_GROW_OVERFLOW_CAP");
    const long long forced_cap = forced ? std::atoll(forced) : -1ll;
    const u64 ov_cap = forced_cap > 0 ? static_cast<u64>(forced_cap) : std::max<u64>(u64(1) << 16, old_cap / 64);
    DBuf<u64> ov(c, ov_cap);
    u64* d = c->d_scalars + 36;
    FV_CUDA(cudaMemsetAsync(d, 0, 8, c->stream));
    {
        // Algorithmic bytes: the old table read once, the new one written once.
        ProfScope prof(c, "hash_grow", double(old_cap) * 8.0 + double(new_cap) * 8.0);
        hash_grow_kernel<<<static_cast<unsigned>(old_cap / kGrowTile), kGrowBlock, 0, c->stream>>>(
            from.slots.get(), old_cap, log_old, static_cast<u32>(factor), to.slots.get(), to.mask, to.group_bits,
            ov.get(), ov_cap, d);
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    }
    u64 n_ov = 0;
    c->read_scalars(d, &n_ov, 1);
    if (n_ov > ov_cap) return false;  // nothing of `to` is relied on: the caller redoes it
    if (n_ov) engine_hash_insert(c, ov.get(), n_ov, to, nullptr, nullptr);
    return true;
}

static void build_run_hash(Ctx* c, JoinIndex& idx, const u64* d_nu = nullptr);

bool engine_group_keys(Ctx* c, DBuf<u64>& keys, u64 n, u32 shift, JoinIndex* runs, u32* col0, u32* col1,
                       const u32* pay_in, u32* pay_out, const u32* gather_idx, u32* gather_src) {
    // Small domains with thousands of keys per value serialize on the
    // counters (C1: 2.6 K keys per value, 2.2 -> 5.1 ms); radix there.
    if (shift > kGroupMaxBits || n > (u64(kGroupMaxPerValue) << shift)) return false;
    if (n <= 1) return false;  // already grouped; the caller indexes it the usual way
    const u64 domain = u64(1) << shift;
    DBuf<u32> cnt(c, domain), cursor(c, domain), base32(c, runs ? domain : 0);
    DBuf<u64> base(c, domain), out(c, col0 ? 0 : n);
    FV_CUDA(cudaMemsetAsync(cnt.get(), 0, 4 * domain, c->stream));
    FV_CUDA(cudaMemsetAsync(cursor.get(), 0, 4 * domain, c->stream));
    {
        ProfScope prof(c, "group_keys", double(n) * 8.0 * 3.0);
        group_count_kernel<<<grid_for(n), 256, 0, c->stream>>>(keys.get(), n, shift, cnt.get());
        FV_CUDA(cudaGetLastError());
        tile_scan(c, GroupBaseOp{cnt.get(), base.get(), runs ? base32.get() : nullptr}, domain, nullptr);
        group_scatter_kernel<<<grid_for(n), 256, 0, c->stream>>>(keys.get(), n, shift, base.get(), cursor.get(),
                                                                  out.get(), col0, col1, pay_in, pay_out,
                                                                  gather_idx, gather_src);
        FV_CUDA(cudaGetLastError());
        c->count_launch(2);
    }
    if (!col0) keys.swap(out);
    if (runs) {
        // Direct-address run index over the value domain: the run of value v
        // is (base32[v], cnt[v]) — no compaction, no hash table, no host
        // readback of the run count.
        runs->domain = domain;
        runs->ends = false;  // counts
        runs->n_unique = n;  // not counted; non-zero marks a non-empty index
        runs->ustart = std::move(base32);
        runs->ucount = std::move(cnt);
        runs->ukeys = DBuf<u32>();
        runs->ht = HashIndex();
    }
    return true;
}

void engine_unpack_keys(Ctx* c, const u64* keys, u64 n, u32 arity, u32 shift, const std::vector<u32*>& cols) {
    if (!n) return;
    if (arity > 2) fail(FV_ERR_ARITY, "unpack_keys: arity > 2");
    ProfScope prof(c, "unpack_keys", double(n) * (8.0 + 4.0 * arity));
    unpack_keys_kernel<<<grid_for(n), 256, 0, c->stream>>>(keys, n, arity, shift, cols[0],
                                                            arity == 2 ? cols[1] : nullptr);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void engine_interleave(Ctx* c, const std::vector<const u32*>& cols, u64 n, u32* out) {
    if (!n) return;
    const u32 arity = static_cast<u32>(cols.size());
    if (arity == 0 || arity > FV_MAX_ARITY) fail(FV_ERR_ARITY, "interleave: arity out of range");
    Cols8 cp{};
    for (u32 j = 0; j < arity; ++j) cp.p[j] = cols[j];
    ProfScope prof(c, "dump_interleave", 8.0 * double(n) * arity);
    interleave_kernel<<<grid_for(n), 256, 0, c->stream>>>(cp, arity, n, out);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

u64 engine_unique_unpack(Ctx* c, const std::vector<DBuf<u64>>& words, u64 n, u32 arity, u32 shift,
                         const std::vector<u32*>& cols) {
    if (!n) return 0;
    UniqueUnpackOp op{};
    op.words = static_cast<u32>(words.size());
    op.arity = arity;
    op.shift = shift;
    for (u32 k = 0; k < op.words; ++k) op.w.p[k] = const_cast<u64*>(words[k].get());
    for (u32 j = 0; j < arity; ++j) op.out.p[j] = cols[j];
    u64* d = c->d_scalars + 19;
    {
        ProfScope prof(c, "unique_unpack", double(n) * 8.0 * op.words);
        tile_scan(c, op, n, d);
    }
    u64 k = 0;
    c->read_scalars(d, &k, 1);
    c->prof_add_bytes("unique_unpack", 4.0 * double(k) * arity);
    return k;
}

// Distinct rows of sorted packed keys, kept packed (pool compaction).
struct UniqueWordsOp {
    Words4 w, out;
    u32 words;
    __device__ u64 value(u64 i) const {
        if (i == 0) return 1;
        for (u32 k = 0; k < words; ++k)
            if (w.p[k][i] != w.p[k][i - 1]) return 1;
        return 0;
    }
    __device__ void emit(u64 i, u64 pos, u64 v) const {
        if (!v) return;
        for (u32 k = 0; k < words; ++k) out.p[k][pos] = w.p[k][i];
    }
};

u64 engine_unique_words(Ctx* c, const std::vector<DBuf<u64>>& words, u64 n, std::vector<DBuf<u64>>& out) {
    out.clear();
    UniqueWordsOp op{};
    op.words = static_cast<u32>(words.size());
    for (u32 k = 0; k < op.words; ++k) {
        out.emplace_back(c, n);
        op.w.p[k] = const_cast<u64*>(words[k].get());
        op.out.p[k] = out.back().get();
    }
    if (!n) return 0;
    u64* d = c->d_scalars + 35;
    {
        ProfScope prof(c, "unique_words", double(n) * 8.0 * op.words);
        tile_scan(c, op, n, d);
    }
    u64 k = 0;
    c->read_scalars(d, &k, 1);
    return k;
}

u64 engine_select_rows(Ctx* c, u64 n, const RowFilter& pred, u32* ids) {
    if (!n) return 0;
    u64* d = c->d_scalars + 18;
    tile_scan(c, SelectRowsOp{pred, ids}, n, d);
    u64 k = 0;
    c->read_scalars(d, &k, 1);
    return k;
}

// Probe + exclusive scan in one single-pass kernel: each row's run lookup is
// the scan's item value (its run start stored on the way), so the counts are
// never written and read back (12 bytes per probe row less, one launch less).
struct ProbeScanOp {
    const u32* probe;
    const u64* slots;
    u32 mask;
    const u32* ustart;
    const u32* ucount;
    u64 domain;
    bool ends;
    RowFilter pred;
    u32* starts;
    u64* offsets;
    u64 n;
    __device__ u64 value(u64 i) const {
        u32 s = 0, c = 0, r;
        if (pass_filters(pred.f, pred.n, i, 0)) {
            const u32 v = probe[i];
            if (domain) {
                if (v < domain) direct_run(ustart, ucount, ends, v, &s, &c);
            } else if (ht_lookup(slots, mask, v, &r)) {
                s = ustart[r];
                c = ucount[r];
            }
        }
        starts[i] = s;
        return c;
    }
    __device__ void emit(u64 i, u64 prefix, u64 v) const {
        offsets[i] = prefix;
        if (i == n - 1) offsets[n] = prefix + v;
    }
};

void engine_probe_offsets(Ctx* c, const u32* probe, u64 n, const JoinIndex& idx, const RowFilter& pred,
                          u32* starts, u64* offsets) {
    if (!n || idx.n_unique == 0) {  // empty build side: every probe misses
        FV_CUDA(cudaMemsetAsync(offsets, 0, 8 * (n + 1), c->stream));
        if (n) FV_CUDA(cudaMemsetAsync(starts, 0, 4 * n, c->stream));
        return;
    }
    ProfScope prof(c, "join_probe_count", double(n) * 20.0);
    tile_scan(c,
              ProbeScanOp{probe, idx.ht.slots.get(), idx.ht.mask, idx.ustart.get(), idx.ucount.get(), idx.domain,
                          idx.ends, pred, starts, offsets, n},
              n, nullptr);
}

void engine_probe_count(Ctx* c, const u32* probe, u64 n, const JoinIndex& idx, const RowFilter& pred,
                        u32* starts, u32* counts) {
    if (!n) return;
    if (idx.n_unique == 0) {  // empty build side: every probe misses
        FV_CUDA(cudaMemsetAsync(counts, 0, 4 * n, c->stream));
        FV_CUDA(cudaMemsetAsync(starts, 0, 4 * n, c->stream));
        return;
    }
    ProfScope prof(c, "join_probe_count", double(n) * 20.0);
    probe_count_kernel<<<grid_for(n), 256, 0, c->stream>>>(probe, n, idx.ht.slots.get(), idx.ht.mask,
                                                            idx.ustart.get(), idx.ucount.get(), idx.domain,
                                                            idx.ends, pred,
                                                            starts, counts);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void engine_materialize(Ctx* c, const u64* offsets, u64 m, u64 total, const u32* starts,
                        const OutSpec& spec, u64 o_begin, u64 o_end) {
    if (o_end > total) o_end = total;
    if (o_begin >= o_end) return;
    const u64 outs = o_end - o_begin;
    const u64 tiles = ceil_div(outs, kMatTile);
    // Algorithmic bytes: per probe row its offset and run start; per output
    // its build-side operands and the written row. With the fused dedup
    // (spec.ht_slots) the candidate row is never materialized; it is still
    // charged as written once and read once by dedup (SURVEY.md §8d:
    // 2 * 4h bytes per candidate), so the figure is the same implementation-
    // independent lower bound as the unfused pipeline.
    double side1 = 0, side0 = 0;
    for (u32 k = 0; k < spec.n_out; ++k) (spec.col[k].side ? side1 : side0) += 4;
    for (u32 k = 0; k < spec.n_filters; ++k) {
        (spec.f[k].a.side ? side1 : side0) += 4;
        if (spec.f[k].op != kFilterConst) (spec.f[k].b.side ? side1 : side0) += 4;
    }
    if (spec.wbits.ptr) (spec.wbits.side ? side1 : side0) += 4;
    const double row_bytes = (spec.key_mode ? 8.0 * ((spec.n_out + 1) / 2) : 4.0 * spec.n_out) +
                             (spec.wbits.ptr ? 4.0 : 0.0);
    const double out_bytes = fused_set(spec) ? 2.0 * row_bytes : row_bytes;
    const double frac = double(outs) / double(total);  // a chunk reads its share of the probe rows
    DBuf<u64> rows(c, 2 * tiles);
    tile_rows_kernel<<<grid_for(tiles * 32), 256, 0, c->stream>>>(offsets, m, o_begin, o_end, tiles, rows.get(),
                                                                  rows.get() + tiles);
    FV_CUDA(cudaGetLastError());
    // The fused join + key-set dedup is profiled as "join_dedup". Word
    // outputs are charged per tuple candidate they stand for (SURVEY.md
    // §8(d)'s B_alg is implementation-independent): each costs its build-side
    // value (4 B) and its write + read by dedup (2 * 8 B), counted by the
    // kernel when profiling.
    const bool word_prof = c->prof && spec.word_sink && spec.wbits.ptr;
    OutSpec pspec = spec;
    if (word_prof) {
        pspec.cand_count = c->d_scalars + 46;
        FV_CUDA(cudaMemsetAsync(pspec.cand_count, 0, 8, c->stream));
    }
    std::optional<ProfScope> prof;
    prof.emplace(c, fused_set(spec) ? "join_dedup" : "join_materialize",
                 frac * double(m) * (12.0 + side0) + (word_prof ? 0.0 : double(outs) * (side1 + out_bytes)));
    static const u32 env_group = [] {
        const char* e = std::getenv("FVLOG_MAT_GROUP");
        return e ? static_cast<u32>(std::atoi(e)) : 0u;
    }();
    const u32 group = (fused_set(spec) || spec.tile_dedup) ? (env_group ? env_group : u32(kMatGroup)) : 1u;
    const unsigned grid = static_cast<unsigned>(ceil_div(tiles, group));
    const u64* jlo = rows.get();
    const u64* jhi = rows.get() + tiles;
    // Instantiations: filtered (COMPACT), partitioned routing (REMOTE) and
    // block-set dedup (BLOCKS) each keep their own register budget.
#define FV_MAT_LAUNCH(C_, R_, B_) FV_MAT_LAUNCH_W(C_, R_, B_, false)
#define FV_MAT_LAUNCH_W(C_, R_, B_, W_)                                                                         \
    do {                                                                                                        \
        const size_t dyn = W_ ? sizeof(u32) * kMatSetSlots : 0;                                                 \
        if (W_) {                                                                                               \
            static const bool attr_set = [] {                                                                   \
                return cudaFuncSetAttribute(materialize_kernel<C_, R_, B_, W_>,                                 \
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,                        \
                                            static_cast<int>(sizeof(u32) * kMatSetSlots)) == cudaSuccess;      \
            }();                                                                                                \
            if (!attr_set) fail(FV_ERR_CUDA, "materialize: dynamic shared memory attribute");                   \
        }                                                                                                       \
        materialize_kernel<C_, R_, B_, W_><<<grid, kMatBlock, dyn, c->stream>>>(offsets, m, o_begin, o_end,     \
                                                                                 starts, jlo, jhi, tiles, group, \
                                                                                 pspec);                         \
    } while (0)
    const bool blocks = spec.bs.dir != nullptr;
    const bool cmp = spec.n_filters != 0;
    const bool words = spec.word_sink != 0;
    if (words && (!blocks || spec.remote_world)) fail(FV_ERR_INVALID, "word-form join needs a local block set");
    if (spec.remote_world) {
        if (blocks) {
            if (cmp) FV_MAT_LAUNCH(true, true, true);
            else FV_MAT_LAUNCH(false, true, true);
        } else {
            if (cmp) FV_MAT_LAUNCH(true, true, false);
            else FV_MAT_LAUNCH(false, true, false);
        }
    } else if (words) {
        if (cmp) FV_MAT_LAUNCH_W(true, false, true, true);
        else FV_MAT_LAUNCH_W(false, false, true, true);
    } else if (blocks) {
        if (cmp) FV_MAT_LAUNCH(true, false, true);
        else FV_MAT_LAUNCH(false, false, true);
    } else {
        if (cmp) FV_MAT_LAUNCH(true, false, false);
        else FV_MAT_LAUNCH(false, false, false);
    }
#undef FV_MAT_LAUNCH
#undef FV_MAT_LAUNCH_W
    FV_CUDA(cudaGetLastError());
    c->count_launch(2);
    prof.reset();  // the launch's event closes before the candidate count is read
    if (word_prof) {
        u64 tc = 0;
        c->read_scalars(pspec.cand_count, &tc, 1);
        c->prof_add_bytes("join_dedup", double(tc) * (4.0 + 16.0));
    }
}

void engine_project(Ctx* c, u64 n, const OutSpec& spec) {
    if (!n) return;
    const u64 tiles = ceil_div(n, kMatTile);
    ProfScope prof(c, "project", double(n) * (4.0 * (spec.n_out + 2 * spec.n_filters) +
                                               8.0 * ((spec.n_out + 1) / 2)));
    if (spec.n_filters)
        project_kernel<true><<<static_cast<unsigned>(tiles), kMatBlock, 0, c->stream>>>(n, spec);
    else
        project_kernel<false><<<static_cast<unsigned>(tiles), kMatBlock, 0, c->stream>>>(n, spec);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void engine_build_runs(Ctx* c, const u32* sorted_keys, u64 n, JoinIndex& idx, u32 key_bits, bool force_direct) {
    idx.n_unique = 0;
    idx.domain = 0;
    idx.ends = false;
    if (n == 0) return;
    // (only where the domain is not much larger than the rows: the arrays
    // and their clearing scale with the domain)
    if (key_bits && key_bits <= kGroupMaxBits && (force_direct || (u64(1) << key_bits) <= 16 * n)) {
        // Direct-address index over the value domain: run starts and ends
        // at their values (one light pass, only the ends cleared; no
        // compaction, no hash table, no host readback of the run count).
        const u64 domain = u64(1) << key_bits;
        idx.domain = domain;
        idx.ends = true;
        idx.n_unique = n;  // not counted; non-zero marks a non-empty index
        // (start, end) interleaved: a probe is one 8-byte load (ucount empty)
        idx.ustart = DBuf<u32>(c, 2 * domain);
        idx.ucount = DBuf<u32>();
        idx.ukeys = DBuf<u32>();
        idx.ht = HashIndex();
        FV_CUDA(cudaMemsetAsync(idx.ustart.get(), 0, 8 * domain, c->stream));
        ProfScope prof(c, "direct_index", 4.0 * double(n));
        direct_runs_kernel<<<grid_for(n), 256, 0, c->stream>>>(sorted_keys, n, idx.ustart.get(), domain);
        FV_CUDA(cudaGetLastError());
        c->count_launch();
        return;
    }
    DBuf<u32> uk(c, n), us(c, n);
    u64* d = c->d_scalars + 16;
    tile_scan(c, RunsOp{sorted_keys, uk.get(), us.get()}, n, d);
    if (n <= kRunsBoundRows) {
        // Small builds: sized by the row count (the run count stays on the
        // device, read by the kernels) instead of a host round trip.
        DBuf<u64> d_nu(c, 1);
        FV_CUDA(cudaMemcpyAsync(d_nu.get(), d, 8, cudaMemcpyDeviceToDevice, c->stream));
        idx.n_unique = n;  // a bound; non-zero marks a non-empty index
        idx.ukeys = std::move(uk);
        idx.ustart = std::move(us);
        idx.ucount = DBuf<u32>(c, n);
        runs_count_kernel<<<grid_for(n), 256, 0, c->stream>>>(idx.ustart.get(), idx.ucount.get(), n, n, d_nu.get());
        FV_CUDA(cudaGetLastError());
        c->count_launch();
        build_run_hash(c, idx, d_nu.get());
        return;
    }
    c->read_scalars(d, &idx.n_unique, 1);
    const u64 nu = idx.n_unique;
    idx.ukeys = DBuf<u32>(c, nu);
    idx.ustart = DBuf<u32>(c, nu);
    idx.ucount = DBuf<u32>(c, nu);
    FV_CUDA(cudaMemcpyAsync(idx.ukeys.get(), uk.get(), 4 * nu, cudaMemcpyDeviceToDevice, c->stream));
    FV_CUDA(cudaMemcpyAsync(idx.ustart.get(), us.get(), 4 * nu, cudaMemcpyDeviceToDevice, c->stream));
    runs_count_kernel<<<grid_for(nu), 256, 0, c->stream>>>(idx.ustart.get(), idx.ucount.get(), nu, n, nullptr);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
    build_run_hash(c, idx);
}

// Hash table over the unique keys of idx (key -> run number); d_nu: their
// count on the device, idx.n_unique then a bound.
static void build_run_hash(Ctx* c, JoinIndex& idx, const u64* d_nu) {
    const u64 nu = idx.n_unique;
    u64 cap = 64;
    while (cap < 2 * nu) cap <<= 1;
    idx.ht.slots = DBuf<u64>(c, cap);
    idx.ht.mask = static_cast<u32>(cap - 1);
    FV_CUDA(cudaMemsetAsync(idx.ht.slots.get(), 0xff, 8 * cap, c->stream));
    if (!nu) return;
    hash_build_kernel<<<grid_for(nu), 256, 0, c->stream>>>(
        idx.ukeys.get(), nu, reinterpret_cast<unsigned long long*>(idx.ht.slots.get()), idx.ht.mask, d_nu);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

static Cols8 cols8(const std::vector<const u32*>& cols) {
    Cols8 c{};
    for (size_t j = 0; j < cols.size() && j < FV_MAX_ARITY; ++j) c.p[j] = cols[j];
    return c;
}

void engine_pack_keys(Ctx* c, const std::vector<const u32*>& cols, u64 n, u32 shift, u64* const* words) {
    if (!n) return;
    const u32 arity = static_cast<u32>(cols.size());
    Words4 w{};
    for (u32 k = 0; k < (arity + 1) / 2; ++k) w.p[k] = words[k];
    ProfScope prof(c, "pack_keys", double(n) * (4.0 * arity + 8.0 * ((arity + 1) / 2)));
    pack_kernel<<<grid_for(n), 256, 0, c->stream>>>(cols8(cols), arity, n, shift, w);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

template <int W>
static void merge_launch(Ctx* c, const Cols8& a, u64 n_a, const Words4& b, u64 n_b, u32 arity, u32 shift,
                         const OutCols8& co, const OutCols8& dout, u64* d_new) {
    const u64 tiles = ceil_div(n_a + n_b, MergeTraits<W>::kTile);
    u32* counter = nullptr;
    const u32 epoch = c->lookback_epoch(tiles, &counter);
    // Reads FULL and the candidates once, rewrites FULL; the 2 x |DELTA| row
    // writes are added by the caller once |DELTA| is known (prof_add_bytes).
    DBuf<u64> splits(c, tiles + 1);
    {
        ProfScope prof(c, "merge_partition", double(tiles + 1) * 8.0);
        merge_partition_kernel<W><<<grid_for(tiles + 1), 256, 0, c->stream>>>(a, n_a, b, n_b, arity, shift, tiles,
                                                                              splits.get());
        FV_CUDA(cudaGetLastError());
    }
    ProfScope prof(c, "merge_dedup", 8.0 * double(n_a) * arity + 8.0 * W * double(n_b));
    merge_kernel<W><<<static_cast<unsigned>(tiles), MergeTraits<W>::kBlock, 0, c->stream>>>(
        a, n_a, b, n_b, arity, shift, co, dout, splits.get(), c->lb.status, epoch, counter, d_new);
    FV_CUDA(cudaGetLastError());
    c->count_launch(2);
}

void engine_merge(Ctx* c, const std::vector<const u32*>& a_cols, u64 n_a, u64* const* b_words, u64 n_b,
                  u32 arity, u32 shift, const std::vector<u32*>& c_cols, const std::vector<u32*>& d_cols,
                  u64* d_new) {
    if (n_a + n_b == 0 || n_b == 0) {
        // Nothing new: C = A (caller copies), D empty.
        FV_CUDA(cudaMemsetAsync(d_new, 0, sizeof(u64), c->stream));
        if (n_a) {
            for (u32 j = 0; j < arity; ++j)
                FV_CUDA(cudaMemcpyAsync(c_cols[j], a_cols[j], 4 * n_a, cudaMemcpyDeviceToDevice, c->stream));
        }
        return;
    }
    const Cols8 a = cols8(a_cols);
    Words4 b{};
    const u32 W = (arity + 1) / 2;
    for (u32 k = 0; k < W; ++k) b.p[k] = b_words[k];
    OutCols8 co{}, dout{};
    for (u32 j = 0; j < arity; ++j) {
        co.p[j] = c_cols[j];
        dout.p[j] = d_cols[j];
    }
    switch (W) {
        case 1: merge_launch<1>(c, a, n_a, b, n_b, arity, shift, co, dout, d_new); break;
        case 2: merge_launch<2>(c, a, n_a, b, n_b, arity, shift, co, dout, d_new); break;
        case 3: merge_launch<3>(c, a, n_a, b, n_b, arity, shift, co, dout, d_new); break;
        case 4: merge_launch<4>(c, a, n_a, b, n_b, arity, shift, co, dout, d_new); break;
        default: fail(FV_ERR_ARITY, "arity exceeds FV_MAX_ARITY");
    }
}

void engine_route(Ctx* c, u64 n, const RouteKey& key, u32 world, const std::vector<const u32*>& c32,
                  const std::vector<u32*>& c32_out, const std::vector<const u64*>& c64,
                  const std::vector<u64*>& c64_out, u64* cnt, u64* off, u64* d_counts_out) {
    if (world > static_cast<u32>(kMaxRanks)) fail(FV_ERR_INVALID, "more than 64 ranks");
    if (c32.size() > FV_MAX_ARITY || c64.size() > 4) fail(FV_ERR_INVALID, "route: too many columns");
    DBuf<u64> d(c, 2 * world);
    FV_CUDA(cudaMemsetAsync(d.get(), 0, 16 * world, c->stream));
    if (n) {
        ProfScope prof(c, "route_count", double(n) * 4.0);
        route_count_kernel<<<grid_for(n), 256, 0, c->stream>>>(key, n, world,
                                                                reinterpret_cast<unsigned long long*>(d.get()));
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    }
    if (d_counts_out) {
        // Counts stay on the device (the exchange gathers them there);
        // the bucket cursors are their exclusive prefix, computed in place.
        FV_CUDA(cudaMemcpyAsync(d_counts_out, d.get(), 8 * world, cudaMemcpyDeviceToDevice, c->stream));
        route_cursor_kernel<<<1, 1, 0, c->stream>>>(d.get(), d.get() + world, world);
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    } else {
        d.download(cnt, world);
        u64 run = 0;
        for (u32 p = 0; p < world; ++p) {
            off[p] = run;
            run += cnt[p];
        }
        if (n) d.upload(off, world, world);  // cursors start at the bucket offsets
    }
    if (!n) return;
    Cols8 i32{};
    OutCols8 o32{};
    Words4 i64{}, o64{};
    for (size_t j = 0; j < c32.size(); ++j) {
        i32.p[j] = c32[j];
        o32.p[j] = c32_out[j];
    }
    for (size_t j = 0; j < c64.size(); ++j) {
        i64.p[j] = const_cast<u64*>(c64[j]);
        o64.p[j] = c64_out[j];
    }
    ProfScope prof(c, "route_scatter", double(n) * 2.0 * (4.0 * c32.size() + 8.0 * c64.size()));
    route_scatter_kernel<<<static_cast<unsigned>(ceil_div(n, 256 * 8)), 256, 0, c->stream>>>(
        key, n, world, reinterpret_cast<unsigned long long*>(d.get() + world), i32, o32,
        static_cast<u32>(c32.size()), i64, o64, static_cast<u32>(c64.size()));
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

u64 engine_fingerprint(Ctx* c, const std::vector<const u32*>& cols, u64 n, u32 arity) {
    u64* d = c->d_scalars + 17;
    FV_CUDA(cudaMemsetAsync(d, 0, sizeof(u64), c->stream));
    if (n) {
        fingerprint_kernel<<<grid_for(n), 256, 0, c->stream>>>(cols8(cols), arity, n,
                                                                reinterpret_cast<unsigned long long*>(d));
        FV_CUDA(cudaGetLastError());
        c->count_launch();
    }
    u64 h = 0;
    c->read_scalars(d, &h, 1);
    return h;
}

void engine_sort_keys(Ctx* c, std::vector<DBuf<u64>>& words, u64 n, u32 arity, u32 shift, bool group_only,
                      const char* who) {
    static const bool trace_sorts = std::getenv("FVLOG_TRACE_SORTS") != nullptr;
    if (trace_sorts) std::fprintf(stderr, "[sort-call] engine_sort_keys from %s n=%llu arity=%u\n", who,
                                  static_cast<unsigned long long>(n), arity);
    if (n <= 1) return;
    const u32 W = static_cast<u32>(words.size());
    auto word_bits = [&](u32 w) -> u32 {
        return (2 * w + 1 < arity) ? 2 * shift : shift;  // (hi << shift) | lo
    };
    if (W == 1) {
        const u32 bits = arity >= 2 ? 2 * shift : shift;
        const u32 begin = (group_only && arity == 2) ? shift : 0;
        DBuf<u64> alt(c, n);
        if (radix_sort_keys_u64(c, words[0].get(), alt.get(), n, begin, bits > 64 ? 64 : bits)) words[0].swap(alt);
        return;
    }
    DBuf<u32> perm(c, n), perm_alt(c, n);
    DBuf<u64> tmp(c, n), tmp_alt(c, n);
    iota_u32(c, perm.get(), n);
    for (int w = static_cast<int>(W) - 1; w >= 0; --w) {
        gather_u64_kernel<<<grid_for(n), 256, 0, c->stream>>>(words[w].get(), perm.get(), tmp.get(), n);
        FV_CUDA(cudaGetLastError());
        c->count_launch();
        u32 bits = word_bits(static_cast<u32>(w));
        if (bits > 64) bits = 64;
        if (radix_sort_pairs_u64(c, tmp.get(), tmp_alt.get(), perm.get(), perm_alt.get(), n, 0, bits))
            perm.swap(perm_alt);
    }
    for (u32 w = 0; w < W; ++w) {
        gather_u64_kernel<<<grid_for(n), 256, 0, c->stream>>>(words[w].get(), perm.get(), tmp.get(), n);
        FV_CUDA(cudaGetLastError());
        c->count_launch();
        words[w].swap(tmp);
    }
}

void engine_mask_u64(Ctx* c, u64* p, u64 n, u64 and_mask, u64 or_bits) {
    if (!n) return;
    mask_u64_kernel<<<grid_for(n), 256, 0, c->stream>>>(p, n, and_mask, or_bits);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void engine_block_sketch(Ctx* c, const u64* keys, u64 n, u32 shift, u32 arity, u32* regs) {
    FV_CUDA(cudaMemsetAsync(regs, 0, 4 * kHllRegs, c->stream));
    if (!n) return;
    const u64 want = ceil_div(n, 256 * 16);
    const unsigned grid = static_cast<unsigned>(std::max<u64>(1, std::min<u64>(want, u64(kNumSMs) * 2)));
    ProfScope prof(c, "count_blocks", 8.0 * double(n));
    block_sketch_kernel<<<grid, 256, 0, c->stream>>>(keys, n, shift, arity, regs);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

u64 block_sketch_estimate(const u32* regs) {
    const double m = kHllRegs;
    double sum = 0;
    u64 zeros = 0;
    for (int i = 0; i < kHllRegs; ++i) {
        sum += std::ldexp(1.0, -static_cast<int>(regs[i]));
        zeros += regs[i] == 0;
    }
    double e = (0.7213 / (1.0 + 1.079 / m)) * m * m / sum;
    if (e <= 2.5 * m && zeros) e = m * std::log(m / double(zeros));  // small range: linear counting
    return static_cast<u64>(std::ceil(e));
}

// Tuple-space (start, end) pairs of a direct index over word entries: value
// v's words [wstart[v], wstart[v] + wcount[v]) hold tuples
// [off[wstart[v]], off[wstart[v] + wcount[v]]) (off[n] = the tuple total).
__global__ void word_runs_to_tuples_kernel(const u32* __restrict__ wstart, const u32* __restrict__ wcount,
                                           const u64* __restrict__ off, u64 domain, u32* __restrict__ pair) {
    GRID_STRIDE(v, domain) {
        const u32 cnt = wcount[v];
        u32 s = 0, e = 0;
        if (cnt) {
            s = static_cast<u32>(off[wstart[v]]);
            e = static_cast<u32>(off[u64(wstart[v]) + cnt]);
        }
        pair[2 * v] = s;
        pair[2 * v + 1] = e;
    }
}

void engine_word_index_to_tuples(Ctx* c, const JoinIndex& words, const u64* off, JoinIndex& out) {
    out.domain = words.domain;
    out.ends = true;
    out.n_unique = words.n_unique;
    out.ukeys = DBuf<u32>();
    out.ucount = DBuf<u32>();
    out.ht = HashIndex();
    out.ustart = DBuf<u32>(c, 2 * words.domain);
    ProfScope prof(c, "direct_index", 16.0 * double(words.domain));
    word_runs_to_tuples_kernel<<<grid_for(words.domain), 256, 0, c->stream>>>(words.ustart.get(), words.ucount.get(),
                                                                              off, words.domain, out.ustart.get());
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

}  // namespace fv

// Onesweep LSD radix sort for sm_100a (keys u32/u64, optional u32 payload).
//
// Replaces the comparator sorts of the reference:
//   build_index   (P/src/column.cpp:25-30): std::sort of ids by (value, id)
//   dedup_rows    (P/src/relation.cpp:71-80): sort of ids by (row, id)
// A stable LSD sort of (key, id) pairs started from iota yields exactly the
// reference's strict (value, id) order, so sorted_idx is bit-identical.
//
// Per sort: one histogram kernel computes all digit histograms in a single
// read of the keys (shared atomics, warp-uniform digits added once), a
// tiny kernel turns them into per-digit global bases, then one onesweep
// kernel per 8-bit digit reads each key once and writes it once:
//   - tile of BLOCK*ITEMS keys in a warp-striped arrangement (coalesced
//     128-bit-friendly loads; lane order == input order so ranking is stable)
//   - per-warp digit ranks (peer lanes from one ballot per digit bit),
//     per-warp shared histograms
//   - decoupled look-back across tiles per digit (status words carry an epoch
//     so no clearing between passes)
//   - shared-memory exchange so global stores are runs of one digit.
// HBM roofline per pass: n * 2 * (sizeof(K) + sizeof(payload)) bytes.
#include "radix_sort.h"

#include <cstdio>
#include <cstdlib>
#include <type_traits>

namespace fv {

namespace {

constexpr int kRadixBits = 8;
constexpr u64 kSkipCheckMin = u64(1) << 20;  // sorts smaller than this run every pass
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortBlock = 256;
constexpr int kSortWarps = kSortBlock / 32;

#ifndef FV_SORT_ITEMS_U32
#define FV_SORT_ITEMS_U32 16
#endif
#ifndef FV_SORT_ITEMS_U64
#define FV_SORT_ITEMS_U64 16
#endif


template <typename K>
struct SortTraits;
template <>
struct SortTraits<u32> {
    static constexpr int kItems = FV_SORT_ITEMS_U32;
};
template <>
struct SortTraits<u64> {
    static constexpr int kItems = FV_SORT_ITEMS_U64;
};

template <typename K>
__device__ __forceinline__ u32 digit_of(K key, u32 shift, u32 mask) {
    return static_cast<u32>(key >> shift) & mask;
}

// ---- histogram over all passes -------------------------------------------

// One read of the keys computes every pass's digit histogram. Two shared
// copies per pass (even/odd warps) take plain shared atomics; a warp whose
// 32 digits are all equal (sorted or skewed input: high digits of packed row
// keys often are) adds 32 once instead of 32 conflicting atomics.
constexpr int kHistItems = 8;
template <typename K>
__global__ void __launch_bounds__(256) radix_hist_kernel(const K* __restrict__ keys, u64 n,
                                                         u32 begin_bit, u32 end_bit, u32 npass,
                                                         unsigned long long* __restrict__ hist) {
    __shared__ u32 s_hist[2][8][kRadix];
    for (u32 i = threadIdx.x; i < 2 * 8 * kRadix; i += blockDim.x) (&s_hist[0][0][0])[i] = 0;
    __syncthreads();
    const u32 lane = lane_id(), copy = (threadIdx.x >> 5) & 1;
    const u64 tile = u64(blockDim.x) * kHistItems;
    for (u64 base = u64(blockIdx.x) * tile; base < n; base += u64(gridDim.x) * tile) {
        K key[kHistItems];
#pragma unroll
        for (int k = 0; k < kHistItems; ++k) {
            const u64 i = base + u64(k) * blockDim.x + threadIdx.x;
            key[k] = i < n ? keys[i] : K(0);
        }
#pragma unroll
        for (int k = 0; k < kHistItems; ++k) {
            const u64 i = base + u64(k) * blockDim.x + threadIdx.x;
            const bool valid = i < n;
            // Warps are fully in or fully out of range except the last one.
            const bool full = __all_sync(0xffffffffu, valid);
            for (u32 p = 0; p < npass; ++p) {
                const u32 shift = begin_bit + p * kRadixBits;
                const u32 bits = min(u32(kRadixBits), end_bit - shift);
                const u32 d = digit_of(key[k], shift, (1u << bits) - 1);
                if (full && __all_sync(0xffffffffu, d == __shfl_sync(0xffffffffu, d, 0))) {
                    if (lane == 0) atomicAdd(&s_hist[copy][p][d], 32u);
                } else if (valid) {
                    atomicAdd(&s_hist[copy][p][d], 1u);
                }
            }
        }
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < npass * kRadix; i += blockDim.x) {
        const u32 v = (&s_hist[0][0][0])[i] + (&s_hist[1][0][0])[i];
        if (v) atomicAdd(hist + i, static_cast<unsigned long long>(v));
    }
}

// hist[p][d] -> exclusive bases[p][d]; trivial[p] = 1 when one digit holds
// every key (the pass would be the identity permutation and is skipped).
__global__ void radix_bins_kernel(const unsigned long long* __restrict__ hist, u64* __restrict__ bins,
                                  u64 n, u64* __restrict__ trivial) {
    __shared__ u64 s_warp[kSortWarps + 1];
    const u32 p = blockIdx.x;
    const u64 v = hist[p * kRadix + threadIdx.x];
    // inline block scan (256 threads)
    const u32 lane = lane_id(), warp = threadIdx.x >> 5;
    u64 x = v;
    for (int o = 1; o < 32; o <<= 1) {
        u64 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<u32>(o)) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 run = 0;
        for (int w = 0; w < kSortWarps; ++w) {
            u64 t = s_warp[w];
            s_warp[w] = run;
            run += t;
        }
        s_warp[kSortWarps] = run;
    }
    __syncthreads();
    bins[p * kRadix + threadIdx.x] = s_warp[warp] + x - v;
    const int is_trivial = __syncthreads_or(v == n);
    if (threadIdx.x == 0) trivial[p] = is_trivial ? 1 : 0;
}

// ---- bulk tile loads (TMA 1D bulk copy, cp.async.bulk) -------------------------
//
// A full tile's keys (and values) are copied global -> shared by the TMA
// engine in one bulk transfer per array, completing on an mbarrier; the
// threads then read their warp-striped items from shared memory. The copy is
// one 32 KB request instead of 16 dependent 8-byte loads per thread, so the
// SM issues no load instructions for the tile (SASS: UBLKCP).

__device__ __forceinline__ u32 smem_u32(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, u32 bytes, u64* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase) {
    asm volatile(
        "{\n"
        " .reg .pred done;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        " @!done bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

#ifndef FV_SORT_BULK
#define FV_SORT_BULK 1
#endif
// Resident CTAs per SM the register budget is cut for (smem carveout at
// its maximum so 4 tiles fit): u64 keys + payload keep 3 (less spilling).
#ifndef FV_SORT_MINB
#define FV_SORT_MINB 4
#endif
template <typename K, bool HAS_VAL>
constexpr int sort_min_blocks() { return sizeof(K) == 8 && HAS_VAL ? 3 : FV_SORT_MINB; }
// Early counts: the tile's digit counts come from a shared-atomic histogram
// right after the load and are published before the ranking, so a
// successor's look-back no longer waits for this tile's ranking.
#ifndef FV_SORT_EARLY
#define FV_SORT_EARLY 1
#endif
#ifndef FV_SORT_RANK_GROUP
#define FV_SORT_RANK_GROUP 1
#endif
// Peer masks from match.any (1) instead of one ballot per digit bit (0).
#ifndef FV_SORT_MATCH
#define FV_SORT_MATCH 0
#endif
// Look-back depth: predecessors' status words loaded per round (one
// coalesced row of a warp's 32 digits each).
#ifndef FV_SORT_LBQ
#define FV_SORT_LBQ 4
#endif
#ifndef FV_SORT_CARVE
#define FV_SORT_CARVE 100
#endif

// ---- onesweep pass ------------------------------------------------------------

template <typename K, bool HAS_VAL>
__global__ void __launch_bounds__(kSortBlock, (sort_min_blocks<K, HAS_VAL>())) onesweep_kernel(
    const K* __restrict__ keys_in, K* __restrict__ keys_out, const u32* __restrict__ vals_in,
    u32* __restrict__ vals_out, u64 n, u32 shift, u32 mask, const u64* __restrict__ bins,
    u64* __restrict__ status, u32 epoch, u32* __restrict__ tile_counter) {
    constexpr int ITEMS = SortTraits<K>::kItems;
    constexpr int TILE = kSortBlock * ITEMS;
    constexpr int WARP_TILE = 32 * ITEMS;

    extern __shared__ __align__(16) unsigned char s_raw[];
    K* s_keys = reinterpret_cast<K*>(s_raw);
    u32* s_vals = reinterpret_cast<u32*>(s_raw + sizeof(K) * TILE);
    __shared__ u32 s_whist[kSortWarps][kRadix];
    __shared__ u32 s_block_excl[kRadix];
    __shared__ u32 s_count[kRadix];
    __shared__ u64 s_global[kRadix];
    __shared__ u32 s_tile;
    __shared__ u32 s_warp_sums[kSortWarps];
    __shared__ alignas(8) u64 s_bar;

    const u32 tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    if (tid == 0) {
        s_tile = atomicAdd(tile_counter, 1u);
        if (FV_SORT_BULK) mbar_init(&s_bar, 1);
    }
    for (u32 i = tid; i < kSortWarps * kRadix; i += kSortBlock) (&s_whist[0][0])[i] = 0;
    if (FV_SORT_EARLY) s_count[tid] = 0;
    __syncthreads();
    const u32 tile = s_tile;
    const u64 tile_base = u64(tile) * TILE;

    u32 dig[ITEMS];
    // The tile is staged in shared memory and only the digits stay in
    // registers through ranking and look-back (the keys are re-read for the
    // exchange), which keeps 4 CTAs per SM without spilling the key array.
    // Full tiles of 16-byte aligned arrays arrive by one TMA bulk copy per
    // array; the partial last tile (and unaligned inputs) load directly.
    const bool bulk = FV_SORT_BULK && tile_base + TILE <= n &&
                      !(reinterpret_cast<uintptr_t>(keys_in) & 15) &&
                      (!HAS_VAL || !(reinterpret_cast<uintptr_t>(vals_in) & 15));
    if (bulk) {
        if (tid == 0) {
            constexpr u32 kb = sizeof(K) * TILE, vb = HAS_VAL ? sizeof(u32) * TILE : 0;
            mbar_expect_tx(&s_bar, kb + vb);
            bulk_load(s_keys, keys_in + tile_base, kb, &s_bar);
            if (HAS_VAL) bulk_load(s_vals, vals_in + tile_base, vb, &s_bar);
        }
        mbar_wait(&s_bar, 0);
    } else {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const u32 li = warp * WARP_TILE + k * 32 + lane;
            const u64 i = tile_base + li;
            if (i < n) {
                s_keys[li] = keys_in[i];
                if (HAS_VAL) s_vals[li] = vals_in[i];
            }
        }
        __syncwarp();  // each warp reads back only its own slice
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u32 li = warp * WARP_TILE + k * 32 + lane;
        dig[k] = tile_base + li < n ? digit_of(s_keys[li], shift, mask) : 0xffffu;
    }
    u64* my_status = status + u64(tile) * kRadix + tid;
    if (FV_SORT_EARLY) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
            if (dig[k] != 0xffffu) atomicAdd(&s_count[dig[k]], 1u);
        __syncthreads();
        st_relaxed_u64(my_status, lb_pack(epoch, tile == 0 ? kLbFlagInclusive : kLbFlagAggregate, s_count[tid]));
    }
    // Warp-level stable ranking, item-major (k outer, lane inner) = input order.
    // Lanes with the same digit come from one ballot per digit bit (cheaper
    // than match.any): peers &= ~(ballot ^ (bit ? ~0 : 0)). A full tile with
    // a full 8-bit digit (every pass but a short last one) runs the
    // straight-line form; out-of-range lanes of the last tile only match
    // each other.
    auto rank_items = [&](auto partial_tag, auto full_digit_tag) {
        constexpr bool PARTIAL = decltype(partial_tag)::value;
        constexpr bool FULL_DIGIT = decltype(full_digit_tag)::value;
        constexpr int G = FV_SORT_RANK_GROUP;  // items whose peer masks are formed together (ILP)
#pragma unroll
        for (int k0 = 0; k0 < ITEMS; k0 += G) {
            u32 peers[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const u32 d = dig[k0 + g];
                peers[g] = ~0u;
                if (FV_SORT_MATCH) {
                    peers[g] = __match_any_sync(0xffffffffu, d);
                } else if (PARTIAL) {
                    const bool valid_item = d != 0xffffu;
                    peers[g] = __ballot_sync(0xffffffffu, valid_item);
                    if (!valid_item) peers[g] = ~peers[g];
                }
#pragma unroll
                for (int b = 0; b < (FV_SORT_MATCH ? 0 : kRadixBits); ++b) {
                    if (!FULL_DIGIT && !((mask >> b) & 1u)) break;
                    const u32 bit = (d >> b) & 1u;
                    const u32 x = __ballot_sync(0xffffffffu, bit);
                    peers[g] &= ~(x ^ (0u - bit));
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const u32 d = dig[k0 + g];
                const u32 leader = __ffs(peers[g]) - 1;
                u32 b = 0;
                if ((!PARTIAL || d != 0xffffu) && lane == leader) {
                    b = s_whist[warp][d];
                    s_whist[warp][d] = b + __popc(peers[g]);
                }
                b = __shfl_sync(0xffffffffu, b, leader);
                dig[k0 + g] = d | ((b + __popc(peers[g] & lanemask_lt())) << 16);  // digit | rank << 16
                // The next item's leader for this digit may be another lane:
                // order this lane's counter update before its read
                // (compute-sanitizer racecheck flagged the pair without it).
                __syncwarp();
            }
        }
    };
    using True = std::integral_constant<bool, true>;
    using False = std::integral_constant<bool, false>;
    const bool partial_tile = tile_base + TILE > n;
    if (partial_tile) rank_items(True{}, False{});
    else if (mask == 0xffu) rank_items(False{}, True{});
    else rank_items(False{}, False{});
    __syncthreads();

    // Thread d owns digit d: exclusive scan across warps, tile count.
    const u32 d = tid;
    u32 wcount[kSortWarps];
    u32 count = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
        wcount[w] = s_whist[w][d];
        count += wcount[w];
    }
    // Publish before the look-back so successors are not held up by it.
    if (!FV_SORT_EARLY) st_relaxed_u64(my_status, lb_pack(epoch, tile == 0 ? kLbFlagInclusive : kLbFlagAggregate, count));
    // Block exclusive scan of counts across digits (for the smem exchange).
    {
        u32 x = count;
        for (int o = 1; o < 32; o <<= 1) {
            u32 y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= static_cast<u32>(o)) x += y;
        }
        if (lane == 31) s_warp_sums[warp] = x;
        __syncthreads();
        if (tid == 0) {
            u32 run = 0;
            for (int w = 0; w < kSortWarps; ++w) {
                u32 t = s_warp_sums[w];
                s_warp_sums[w] = run;
                run += t;
            }
        }
        __syncthreads();
        const u32 block_excl = s_warp_sums[warp] + x - count;
        s_block_excl[d] = block_excl;
        // s_whist[w][d] := tile slot of warp w's first item of digit d
        u32 run = block_excl;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            s_whist[w][d] = run;
            run += wcount[w];
        }
    }
    u64 excl = 0;
    if (tile > 0) {
        excl = lookback_thread_deep<FV_SORT_LBQ>(status, tile, kRadix, d, epoch);
        st_relaxed_u64(my_status, lb_pack(epoch, kLbFlagInclusive, excl + count));
    }
    // Output position of tile slot i of digit dd: s_global[dd] + i.
    s_global[d] = bins[d] + excl - s_block_excl[d];
    __syncthreads();

    // Exchange into digit order within the tile.
    K key[ITEMS];
    u32 val[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u32 li = warp * WARP_TILE + k * 32 + lane;
        key[k] = s_keys[li];
        if (HAS_VAL) val[k] = s_vals[li];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u32 dk = dig[k] & 0xffffu;
        if (dk != 0xffffu) {
            const u32 lp = s_whist[warp][dk] + (dig[k] >> 16);
            s_keys[lp] = key[k];
            if (HAS_VAL) s_vals[lp] = val[k];
        }
    }
    __syncthreads();
    const u64 remaining = n - tile_base;
    const u32 valid_count = remaining < u64(TILE) ? static_cast<u32>(remaining) : u32(TILE);
    for (u32 i = tid; i < valid_count; i += kSortBlock) {
        const K kk = s_keys[i];
        const u32 dd = digit_of(kk, shift, mask);
        const u64 pos = s_global[dd] + i;
        keys_out[pos] = kk;
        if (HAS_VAL) vals_out[pos] = s_vals[i];
    }
}

template <typename K, bool HAS_VAL>
void onesweep_pass(Ctx* c, const K* kin, K* kout, const u32* vin, u32* vout, u64 n, u32 shift,
                   u32 mask, const u64* bins) {
    constexpr int TILE = kSortBlock * SortTraits<K>::kItems;
    const u64 tiles = ceil_div(n, TILE);
    u32* counter = nullptr;
    const u32 epoch = c->lookback_epoch(tiles * kRadix, &counter);
    const size_t smem = sizeof(K) * TILE + (HAS_VAL ? sizeof(u32) * TILE : 0);
    // u64 keys + u32 payload need > 48 KB in total (opt-in, once per type).
    static const bool smem_ok = [&] {
        FV_CUDA(cudaFuncSetAttribute(onesweep_kernel<K, HAS_VAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        if (FV_SORT_CARVE >= 0)
            FV_CUDA(cudaFuncSetAttribute(onesweep_kernel<K, HAS_VAL>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         FV_SORT_CARVE));
        return true;
    }();
    (void)smem_ok;
    ProfScope prof(c, sizeof(K) == 8 ? (HAS_VAL ? "radix_onesweep_u64_kv" : "radix_onesweep_u64")
                                     : (HAS_VAL ? "radix_onesweep_u32_kv" : "radix_onesweep_u32"),
                   2.0 * double(n) * (sizeof(K) + (HAS_VAL ? 4 : 0)));
    onesweep_kernel<K, HAS_VAL><<<static_cast<unsigned>(tiles), kSortBlock, smem, c->stream>>>(
        kin, kout, vin, vout, n, shift, mask, bins, c->lb.status, epoch, counter);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

template <typename K, bool HAS_VAL>
bool radix_sort_impl(Ctx* c, K* keys, K* keys_alt, u32* vals, u32* vals_alt, u64 n,
                     u32 begin_bit, u32 end_bit) {
    if (n <= 1 || end_bit <= begin_bit) return false;
    const u32 npass = (end_bit - begin_bit + kRadixBits - 1) / kRadixBits;
    static const bool trace_sorts = std::getenv("FVLOG_TRACE_SORTS") != nullptr;
    if (trace_sorts)
        std::fprintf(stderr, "[sort] n=%llu key=%zu val=%d bits=%u..%u\n", static_cast<unsigned long long>(n),
                     sizeof(K), HAS_VAL ? 1 : 0, begin_bit, end_bit);
    // hist (u64 x npass x 256) | bins (same) | trivial flags (npass)
    DBuf<u64> scratch(c, u64(npass) * kRadix * 2 + 8);
    unsigned long long* hist = reinterpret_cast<unsigned long long*>(scratch.get());
    u64* bins = scratch.get() + u64(npass) * kRadix;
    u64* trivial = bins + u64(npass) * kRadix;
    FV_CUDA(cudaMemsetAsync(hist, 0, sizeof(u64) * npass * kRadix, c->stream));
    {
        const u64 want = ceil_div(n, 256 * kHistItems);
        const unsigned grid = static_cast<unsigned>(want < u64(kNumSMs) * 8 ? (want ? want : 1)
                                                                             : u64(kNumSMs) * 8);
        ProfScope prof(c, "radix_histogram", double(n) * sizeof(K));
        radix_hist_kernel<K><<<grid, 256, 0, c->stream>>>(keys, n, begin_bit, end_bit, npass, hist);
        FV_CUDA(cudaGetLastError());
        radix_bins_kernel<<<npass, kRadix, 0, c->stream>>>(hist, bins, n, trivial);
        FV_CUDA(cudaGetLastError());
        c->count_launch(2);
    }
    // Skipping constant-digit passes needs the histogram on the host (one
    // sync); for small inputs every pass is cheaper than the round trip.
    u64 triv[8] = {0};
    if (n >= kSkipCheckMin) c->read_scalars(trivial, triv, static_cast<int>(npass));

    bool in_alt = false;
    for (u32 p = 0; p < npass; ++p) {
        if (triv[p]) continue;
        const u32 shift = begin_bit + p * kRadixBits;
        const u32 bits = (end_bit - shift) < u32(kRadixBits) ? (end_bit - shift) : u32(kRadixBits);
        const u32 mask = (1u << bits) - 1;
        K* kin = in_alt ? keys_alt : keys;
        K* kout = in_alt ? keys : keys_alt;
        u32* vin = in_alt ? vals_alt : vals;
        u32* vout = in_alt ? vals : vals_alt;
        onesweep_pass<K, HAS_VAL>(c, kin, kout, vin, vout, n, shift, mask, bins + u64(p) * kRadix);
        in_alt = !in_alt;
    }
    return in_alt;
}

}  // namespace

bool radix_sort_pairs_u32(Ctx* c, u32* keys, u32* keys_alt, u32* vals, u32* vals_alt, u64 n,
                          u32 begin_bit, u32 end_bit) {
    return radix_sort_impl<u32, true>(c, keys, keys_alt, vals, vals_alt, n, begin_bit, end_bit);
}
bool radix_sort_keys_u32(Ctx* c, u32* keys, u32* keys_alt, u64 n, u32 begin_bit, u32 end_bit) {
    return radix_sort_impl<u32, false>(c, keys, keys_alt, nullptr, nullptr, n, begin_bit, end_bit);
}
bool radix_sort_pairs_u64(Ctx* c, u64* keys, u64* keys_alt, u32* vals, u32* vals_alt, u64 n,
                          u32 begin_bit, u32 end_bit) {
    return radix_sort_impl<u64, true>(c, keys, keys_alt, vals, vals_alt, n, begin_bit, end_bit);
}
bool radix_sort_keys_u64(Ctx* c, u64* keys, u64* keys_alt, u64 n, u32 begin_bit, u32 end_bit) {
    return radix_sort_impl<u64, false>(c, keys, keys_alt, nullptr, nullptr, n, begin_bit, end_bit);
}

}  // namespace fv

// Single-pass scan / stream-compaction primitive for sm_100a.
//
// The reference's order-preserving compactions (compact_positions,
// P/src/kernels.cpp:15-34: count per fixed block -> sequential scan ->
// write) and its serial exclusive scan (join_offsets, :94-102) become one
// kernel: each CTA reduces a tile, publishes its aggregate, and resolves its
// global prefix by decoupled look-back over its predecessors, so the input
// is read once and the output written once (HBM roofline: n*(in+out) bytes).
#pragma once

#include "fv_common.cuh"

#include <utility>
#include <vector>

namespace fv {

#ifndef FV_SCAN_BLOCK
#define FV_SCAN_BLOCK 256
#endif
constexpr int kScanBlock = FV_SCAN_BLOCK;
#ifndef FV_SCAN_ITEMS
#define FV_SCAN_ITEMS 8
#endif
constexpr int kScanItems = FV_SCAN_ITEMS;
constexpr int kScanTile = kScanBlock * kScanItems;

// Block-wide exclusive scan of one u64 per thread; returns the thread's
// exclusive prefix and writes the block total to *total (all threads).
template <int BLOCK>
__device__ __forceinline__ u64 block_exclusive_scan(u64 v, u64* s_warp, u64* total) {
    constexpr int W = BLOCK / 32;
    const u32 lane = lane_id(), warp = threadIdx.x >> 5;
    u64 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u64 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<u32>(o)) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        u64 w = lane < W ? s_warp[lane] : 0;
        u64 incl = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u64 y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<u32>(o)) incl += y;
        }
        if (lane < W) s_warp[lane] = incl - w;
        if (lane == W - 1) s_warp[W] = incl;
    }
    __syncthreads();
    u64 excl = s_warp[warp] + x - v;
    *total = s_warp[W];
    __syncthreads();
    return excl;
}

// Striped (default): value() and emit() are called in warp-striped order
// (item k of lane l of warp w at k * BLOCK + l — every global access of the
// ops coalesced), the values transposed through shared memory to a blocked
// arrangement for the thread-sequential scan and the prefixes back.
#ifndef FV_SCAN_STRIPED
#define FV_SCAN_STRIPED 1
#endif
__device__ __forceinline__ u32 scan_pad(u32 j) { return j + (j >> 4); }  // u64 bank-conflict padding

// Op contract:
//   __device__ u64  value(u64 i) const;            // item weight (0/1 for select)
//   __device__ void emit(u64 i, u64 prefix, u64 v) const;  // called for every i < n
// The last tile stores the grand total to *d_total.
// 8 CTAs per SM (32 registers): the warps of other tiles cover a tile's
// look-back (tools/scanbench.cu, 10^8 counts: 1.55 -> 2.38 TB/s; with the
// values kept in registers and 4 CTAs per SM most of the time went to the
// barrier after warp 0's look-back).
#ifndef FV_SCAN_MINB
#define FV_SCAN_MINB 8
#endif
template <int BLOCK, int ITEMS, class Op>
__global__ void __launch_bounds__(BLOCK, FV_SCAN_MINB) tile_scan_kernel(Op op, u64 n, u64* status, u32 epoch,
                                                          u32* tile_counter, u64* d_total) {
    __shared__ u32 s_tile;
    __shared__ u64 s_warp[BLOCK / 32 + 1];
    __shared__ u64 s_prefix;
#if FV_SCAN_STRIPED
    __shared__ u64 s_x[BLOCK * ITEMS + (BLOCK * ITEMS) / 16 + 1];
#endif
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const u32 tile = s_tile;
    const u64 tile_base = u64(tile) * (BLOCK * ITEMS);
    [[maybe_unused]] const u64 base = tile_base + u64(threadIdx.x) * ITEMS;

    u64 sum = 0;
#if FV_SCAN_STRIPED
    // (no per-item registers across the look-back: the values live in s_x,
    // so more CTAs fit per SM to hide it)
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u32 li = k * BLOCK + threadIdx.x;
        const u64 i = tile_base + li;
        s_x[scan_pad(li)] = i < n ? op.value(i) : 0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) sum += s_x[scan_pad(threadIdx.x * ITEMS + k)];
#else
    u64 v[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u64 i = base + k;
        v[k] = i < n ? op.value(i) : 0;
        sum += v[k];
    }
#endif
    u64 agg;
    const u64 excl = block_exclusive_scan<BLOCK>(sum, s_warp, &agg);

    if (threadIdx.x < 32) {
        u64 prefix = 0;
        if (tile == 0) {
            if (threadIdx.x == 0) st_relaxed_u64(status, lb_pack(epoch, kLbFlagInclusive, agg));
        } else {
            if (threadIdx.x == 0) st_relaxed_u64(status + tile, lb_pack(epoch, kLbFlagAggregate, agg));
            prefix = lookback_warp(status, tile, epoch);
            if (threadIdx.x == 0)
                st_relaxed_u64(status + tile, lb_pack(epoch, kLbFlagInclusive, prefix + agg));
        }
        if (threadIdx.x == 0) {
            s_prefix = prefix;
            const u64 tiles = ceil_div(n, BLOCK * ITEMS);
            if (tile == tiles - 1 && d_total) *d_total = prefix + agg;
        }
    }
    __syncthreads();
    u64 run = s_prefix + excl;
#if FV_SCAN_STRIPED
    // values -> exclusive prefixes in place (block_exclusive_scan's last
    // barrier ordered every read of s_x above); an item's value is then the
    // next prefix minus its own (the tile's last: the tile total's end).
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u32 j = scan_pad(threadIdx.x * ITEMS + k);
        const u64 x = s_x[j];
        s_x[j] = run;
        run += x;
    }
    if (threadIdx.x == BLOCK - 1) s_x[scan_pad(BLOCK * ITEMS)] = run;  // the slot past the tile
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u32 li = k * BLOCK + threadIdx.x;
        const u64 i = tile_base + li;
        const u64 p = s_x[scan_pad(li)];
        if (i < n) op.emit(i, p, s_x[scan_pad(li + 1)] - p);
    }
#else
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u64 i = base + k;
        if (i < n) op.emit(i, run, v[k]);
        run += v[k];
    }
#endif
}

// Launch helper. d_total may be null. n == 0 writes *d_total = 0.
template <class Op>
void tile_scan(Ctx* c, const Op& op, u64 n, u64* d_total) {
    if (n == 0) {
        if (d_total) FV_CUDA(cudaMemsetAsync(d_total, 0, sizeof(u64), c->stream));
        return;
    }
    const u64 tiles = ceil_div(n, kScanTile);
    u32* counter = nullptr;
    const u32 epoch = c->lookback_epoch(tiles, &counter);
    tile_scan_kernel<kScanBlock, kScanItems, Op>
        <<<static_cast<unsigned>(tiles), kScanBlock, 0, c->stream>>>(op, n, c->lb.status, epoch,
                                                                      counter, d_total);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

// ---- common ops ------------------------------------------------------------

// Exclusive scan of u32 counts into u64 offsets[n + 1] (offsets[n] = total).
struct ScanCountsOp {
    const u32* counts;
    u64* offsets;
    u64 n;
    __device__ u64 value(u64 i) const { return counts[i]; }
    __device__ void emit(u64 i, u64 prefix, u64 v) const {
        offsets[i] = prefix;
        if (i == n - 1) offsets[n] = prefix + v;
    }
};

// Order-preserving compaction of positions i with flag[i] != 0 into ids.
struct SelectFlagsOp {
    const u8* flags;
    u8 want;  // keep when (flags[i] != 0) == want
    u32* out;
    __device__ u64 value(u64 i) const { return (flags[i] != 0) == (want != 0) ? 1 : 0; }
    __device__ void emit(u64 i, u64 prefix, u64 v) const {
        if (v) out[prefix] = static_cast<u32>(i);
    }
};

void exclusive_scan_counts(Ctx* c, const u32* counts, u64* offsets, u64 n);

// Device reductions returning to a device scalar.
// accumulate: fold into the existing *d_out (max) instead of resetting it.
void reduce_max_u32(Ctx* c, const u32* in, u64 n, u64* d_out, bool accumulate = false);
// max over several columns into *d_out (accumulates: atomicMax), one launch.
void reduce_max_u32_multi(Ctx* c, const std::vector<std::pair<const u32*, u64>>& cols, u64* d_out);

// Fill / iota helpers.
void iota_u32(Ctx* c, u32* out, u64 n);
void gather_u32(Ctx* c, const u32* src, const u32* idx, u32* out, u64 n);

}  // namespace fv

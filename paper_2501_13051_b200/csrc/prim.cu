// Small device helpers shared by the operator kernels.
#include "prim.cuh"

#include <algorithm>
#include <utility>
#include <vector>

namespace fv {

namespace {

__global__ void iota_kernel(u32* out, u64 n) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        out[i] = static_cast<u32>(i);
}

__global__ void gather_kernel(const u32* __restrict__ src, const u32* __restrict__ idx,
                              u32* __restrict__ out, u64 n) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        out[i] = src[idx[i]];
}

// One global atomicMax per CTA (a per-warp atomic on the single output word
// serialised ~20 K atomics per launch).
__global__ void reduce_max_kernel(const u32* __restrict__ in, u64 n, unsigned long long* out) {
    __shared__ u32 s_max;
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    u32 m = 0;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        m = max(m, in[i]);
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane_id() == 0 && m) atomicMax(&s_max, m);
    __syncthreads();
    if (threadIdx.x == 0 && s_max) atomicMax(out, static_cast<unsigned long long>(s_max));
}

unsigned grid_for(u64 n, int block = 256) {
    const u64 want = ceil_div(n, block);
    const u64 cap = u64(kNumSMs) * 16;
    return static_cast<unsigned>(want == 0 ? 1 : (want < cap ? want : cap));
}

}  // namespace

void exclusive_scan_counts(Ctx* c, const u32* counts, u64* offsets, u64 n) {
    if (n == 0) {
        FV_CUDA(cudaMemsetAsync(offsets, 0, sizeof(u64), c->stream));
        return;
    }
    ProfScope prof(c, "scan_offsets", double(n) * 12.0);
    tile_scan(c, ScanCountsOp{counts, offsets, n}, n, nullptr);
}

void reduce_max_u32(Ctx* c, const u32* in, u64 n, u64* d_out, bool accumulate) {
    if (!accumulate) FV_CUDA(cudaMemsetAsync(d_out, 0, sizeof(u64), c->stream));
    if (n == 0) return;
    const u64 want = ceil_div(n, u64(256) * 16);  // >= 16 items per thread
    const unsigned grid = static_cast<unsigned>(want < u64(kNumSMs) * 4 ? (want ? want : 1) : u64(kNumSMs) * 4);
    reduce_max_kernel<<<grid, 256, 0, c->stream>>>(in, n,
                                                         reinterpret_cast<unsigned long long*>(d_out));
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

namespace {
struct ColSpan {
    const u32* p;
    u64 n;
};
// blockIdx.y: the column; one global atomic per CTA.
__global__ void reduce_max_multi_kernel(const ColSpan* __restrict__ cols, unsigned long long* out) {
    __shared__ u32 s_max;
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    const ColSpan cs = cols[blockIdx.y];
    u32 m = 0;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < cs.n; i += u64(gridDim.x) * blockDim.x)
        m = max(m, cs.p[i]);
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane_id() == 0 && m) atomicMax(&s_max, m);
    __syncthreads();
    if (threadIdx.x == 0 && s_max) atomicMax(out, static_cast<unsigned long long>(s_max));
}
}  // namespace

void reduce_max_u32_multi(Ctx* c, const std::vector<std::pair<const u32*, u64>>& cols, u64* d_out) {
    if (cols.empty()) return;
    std::vector<ColSpan> h;
    u64 longest = 0;
    for (auto& [p, n] : cols) {
        h.push_back({p, n});
        longest = std::max(longest, n);
    }
    DBuf<ColSpan> d(c, h.size());
    d.upload(h.data(), h.size());
    const u64 want = ceil_div(longest, u64(256) * 16);
    const unsigned gx = static_cast<unsigned>(std::max<u64>(1, std::min<u64>(want, u64(kNumSMs) * 4)));
    reduce_max_multi_kernel<<<dim3(gx, static_cast<unsigned>(h.size())), 256, 0, c->stream>>>(
        d.get(), reinterpret_cast<unsigned long long*>(d_out));
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void iota_u32(Ctx* c, u32* out, u64 n) {
    if (!n) return;
    iota_kernel<<<grid_for(n), 256, 0, c->stream>>>(out, n);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

void gather_u32(Ctx* c, const u32* src, const u32* idx, u32* out, u64 n) {
    if (!n) return;
    ProfScope prof(c, "gather", double(n) * 12.0);
    gather_kernel<<<grid_for(n), 256, 0, c->stream>>>(src, idx, out, n);
    FV_CUDA(cudaGetLastError());
    c->count_launch();
}

}  // namespace fv

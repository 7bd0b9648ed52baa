// Single-pass scan micro-benchmark (not part of the library): times
// exclusive_scan_counts (u32 counts -> u64 offsets, the join's count phase)
// on device-resident data. Bytes per element: 4 read + 8 written.
//   make tools/fvlog_scanbench && tools/fvlog_scanbench [n_millions=100]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fv_common.cuh"
#include "prim.cuh"

using namespace fv;

namespace fv {
void exclusive_scan_counts(Ctx* c, const u32* counts, u64* offsets, u64 n);
}

__global__ void fill_counts(u32* k, u64 n) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        k[i] = static_cast<u32>(mix64(i + 99) % 7);
}

int main(int argc, char** argv) {
    const u64 n = static_cast<u64>((argc > 1 ? std::atof(argv[1]) : 100.0) * 1e6);
    Ctx* c = ctx_new(0);
    {
        DBuf<u32> cnt(c, n);
        DBuf<u64> off(c, n + 1);
        fill_counts<<<1184, 256, 0, c->stream>>>(cnt.get(), n);
        exclusive_scan_counts(c, cnt.get(), off.get(), n);
        c->sync();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int reps = 10;
        cudaEventRecord(a, c->stream);
        for (int r = 0; r < reps; ++r) exclusive_scan_counts(c, cnt.get(), off.get(), n);
        cudaEventRecord(b, c->stream);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        std::vector<u64> h(3);
        off.download(h.data(), 1, n);
        std::printf("{\"scan\": \"u32 counts -> u64 offsets\", \"n\": %llu, \"ms\": %.4f, \"gbs\": %.1f, \"total\": %llu}\n",
                    static_cast<unsigned long long>(n), ms, 12.0 * double(n) / (ms * 1e-3) / 1e9,
                    static_cast<unsigned long long>(h[0]));
    }
    ctx_delete(c);
    return 0;
}

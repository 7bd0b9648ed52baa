// Onesweep radix sort micro-benchmark (not part of the library): times the
// engine's sort entry points on device-resident random keys and checks the
// result is sorted (and, for pairs, a stable permutation).
//   u64 keys, bits [0, B)        - the packed-row-key sort (dedup, Δ)
//   u32 keys + u32 ids, 32 bits  - build_index (P/src/column.cpp:17-43)
// Bytes per pass = 2 * n * (key + payload); reported as GB/s per pass.
//
//   make tools/fvlog_sortbench && tools/fvlog_sortbench [n_millions=200] [bits=40]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fv_common.cuh"
#include "radix_sort.h"

using namespace fv;

__global__ void fill_u64(u64* k, u64 n, u32 bits) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        k[i] = mix64(i * 0x9e3779b97f4a7c15ull + 7) & ((bits >= 64) ? ~0ull : ((1ull << bits) - 1));
}
__global__ void fill_u32(u32* k, u32* v, u64 n) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        k[i] = static_cast<u32>(mix64(i + 12345) % 100000);  // many repeats: stability matters
        v[i] = static_cast<u32>(i);
    }
}

template <typename F>
float time_ms(Ctx* c, F&& f, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();  // warm-up
    c->sync();
    cudaEventRecord(a, c->stream);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b, c->stream);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char** argv) {
    const u64 n = u64(argc > 1 ? std::atof(argv[1]) : 200.0) * 1000000ull;
    const u32 bits = argc > 2 ? std::atoi(argv[2]) : 40;
    Ctx* c = ctx_new(0);
    {
        DBuf<u64> k(c, n), k0(c, n), alt(c, n);
        fill_u64<<<1184, 256, 0, c->stream>>>(k0.get(), n, bits);
        bool in_alt = false;
        const float ms = time_ms(c, [&] {
            cudaMemcpyAsync(k.get(), k0.get(), 8 * n, cudaMemcpyDeviceToDevice, c->stream);
            in_alt = radix_sort_keys_u64(c, k.get(), alt.get(), n, 0, bits);
        }, 3);
        const float copy_ms = time_ms(c, [&] {
            cudaMemcpyAsync(k.get(), k0.get(), 8 * n, cudaMemcpyDeviceToDevice, c->stream);
        }, 3);
        std::vector<u64> h(n);
        (in_alt ? alt : k).download(h.data(), n);
        const bool ok = std::is_sorted(h.begin(), h.end());
        const u32 passes = (bits + 7) / 8;
        const double sort_ms = ms - copy_ms;
        std::printf("{\"sort\": \"u64 keys\", \"n\": %llu, \"bits\": %u, \"passes\": %u, \"ms\": %.3f, "
                    "\"gbs_per_pass\": %.1f, \"sorted\": %s}\n",
                    static_cast<unsigned long long>(n), bits, passes, sort_ms,
                    2.0 * 8 * n * passes / (sort_ms * 1e-3) / 1e9, ok ? "true" : "false");
    }
    {
        DBuf<u32> k(c, n), k0(c, n), ka(c, n), v(c, n), v0(c, n), va(c, n);
        fill_u32<<<1184, 256, 0, c->stream>>>(k0.get(), v0.get(), n);
        bool in_alt = false;
        const float ms = time_ms(c, [&] {
            cudaMemcpyAsync(k.get(), k0.get(), 4 * n, cudaMemcpyDeviceToDevice, c->stream);
            cudaMemcpyAsync(v.get(), v0.get(), 4 * n, cudaMemcpyDeviceToDevice, c->stream);
            in_alt = radix_sort_pairs_u32(c, k.get(), ka.get(), v.get(), va.get(), n, 0, 17);
        }, 3);
        const float copy_ms = time_ms(c, [&] {
            cudaMemcpyAsync(k.get(), k0.get(), 4 * n, cudaMemcpyDeviceToDevice, c->stream);
            cudaMemcpyAsync(v.get(), v0.get(), 4 * n, cudaMemcpyDeviceToDevice, c->stream);
        }, 3);
        std::vector<u32> hk(n), hv(n);
        (in_alt ? ka : k).download(hk.data(), n);
        (in_alt ? va : v).download(hv.data(), n);
        bool ok = true;
        for (u64 i = 1; i < n && ok; ++i)
            ok = hk[i - 1] < hk[i] || (hk[i - 1] == hk[i] && hv[i - 1] < hv[i]);
        const double sort_ms = ms - copy_ms;
        std::printf("{\"sort\": \"u32 keys + u32 ids (stable)\", \"n\": %llu, \"bits\": 17, \"passes\": 3, "
                    "\"ms\": %.3f, \"gbs_per_pass\": %.1f, \"sorted_stable\": %s}\n",
                    static_cast<unsigned long long>(n), sort_ms, 2.0 * 8 * n * 3 / (sort_ms * 1e-3) / 1e9,
                    ok ? "true" : "false");
    }
    ctx_delete(c);
    return 0;
}

// Random-access ceiling of this B200 for the key-set kernels (not part of
// the library): the fused join+dedup (materialize_kernel) and the key-set
// inserts are bound by independent 8-byte loads/CASes at random positions
// of a table far larger than L2, not by streaming bandwidth. This measures
// that ceiling on the box so the roofline in bench.py/DESIGN.md can quote
// it next to the streaming copy peak:
//   copy        streaming read+write (u64), GB/s
//   rand_load   8-byte loads at mix64-random slots of a `table_gb` table
//   rand_cas    8-byte atomicCAS at random slots (the insert path)
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fvlog_membench tools/membench.cu
//   tools/fvlog_membench [table_gb=16] [accesses_millions=2048]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

typedef unsigned long long u64;

__device__ __forceinline__ u64 mix64(u64 z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void copy_kernel(const u64* __restrict__ a, u64* __restrict__ b, u64 n) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) b[i] = a[i];
}

template <int ITEMS>
__global__ void rand_load_kernel(const u64* __restrict__ t, u64 mask, u64 n, u64* out) {
    const u64 base = (u64(blockIdx.x) * blockDim.x + threadIdx.x) * ITEMS;
    u64 v[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) v[k] = base + k < n ? __ldcg(t + (mix64(base + k) & mask)) : 0;
    u64 s = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) s ^= v[k];
    if (s == 0x12345) out[0] = s;  // keep the loads alive
}

template <int ITEMS>
__global__ void rand_cas_kernel(u64* t, u64 mask, u64 n, u64* out) {
    const u64 base = (u64(blockIdx.x) * blockDim.x + threadIdx.x) * ITEMS;
    u64 s = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k)
        if (base + k < n) s ^= atomicCAS(t + (mix64(base + k) & mask), ~0ull, base + k);
    if (s == 0x12345) out[0] = s;
}

int main(int argc, char** argv) {
    const double gb = argc > 1 ? std::atof(argv[1]) : 16.0;
    const u64 n_acc = u64(argc > 2 ? std::atof(argv[2]) : 2048.0) * 1000000ull;
    u64 slots = 1;
    while (double(slots * 2 * 8) <= gb * 1e9) slots <<= 1;
    u64 *t, *out, *b;
    CK(cudaMalloc(&t, slots * 8));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(t, 0xff, slots * 8));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float ms;
    // streaming copy over half the table into the other half
    const u64 half = slots / 2;
    b = t + half;
    for (int r = 0; r < 2; ++r) {
        CK(cudaEventRecord(e0));
        copy_kernel<<<148 * 16, 256>>>(t, b, half);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
    }
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf("{\"table_bytes\": %llu, \"copy_gbs\": %.1f", slots * 8, 2.0 * half * 8 / (ms * 1e-3) / 1e9);
    CK(cudaMemset(t, 0xff, slots * 8));
    constexpr int IT = 8;
    const unsigned grid = unsigned((n_acc + 256 * IT - 1) / (256 * IT));
    for (int r = 0; r < 2; ++r) {
        CK(cudaEventRecord(e0));
        rand_load_kernel<IT><<<grid, 256>>>(t, slots - 1, n_acc, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
    }
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf(", \"rand_load_gaccess_s\": %.2f", n_acc / (ms * 1e-3) / 1e9);
    for (int r = 0; r < 2; ++r) {
        CK(cudaEventRecord(e0));
        rand_cas_kernel<IT><<<grid, 256>>>(t, slots - 1, n_acc, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
    }
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf(", \"rand_cas_gaccess_s\": %.2f, \"accesses\": %llu}\n", n_acc / (ms * 1e-3) / 1e9, n_acc);
    CK(cudaGetLastError());
    return 0;
}

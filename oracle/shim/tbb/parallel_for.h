// Test-infrastructure shim (oracle/_ref only): oneTBB parallel_for on OpenMP.
// The reference writes disjoint output slots in every parallel loop
// (P/include/colog/parallel.hpp:15-18), so any schedule gives identical results.
#pragma once
#include <cstddef>
#include "tbb/blocked_range.h"

namespace tbb {

// parallel_for(blocked_range, body): split into grain-sized chunks.
template <typename T, typename Body>
void parallel_for(const blocked_range<T>& r, const Body& body) {
    const std::size_t n = r.end() - r.begin();
    if (n == 0) return;
    const std::size_t g = r.grainsize() ? r.grainsize() : 1;
    const long long chunks = static_cast<long long>((n + g - 1) / g);
#pragma omp parallel for schedule(dynamic, 1)
    for (long long c = 0; c < chunks; ++c) {
        T b = r.begin() + static_cast<T>(c * g);
        T e = b + static_cast<T>(g);
        if (e > r.end()) e = r.end();
        body(blocked_range<T>(b, e, g));
    }
}

// parallel_for(first, last, f): one call per index.
template <typename Index, typename Func>
void parallel_for(Index first, Index last, const Func& f) {
    const long long lo = static_cast<long long>(first);
    const long long hi = static_cast<long long>(last);
#pragma omp parallel for schedule(dynamic, 1)
    for (long long i = lo; i < hi; ++i) f(static_cast<Index>(i));
}

} // namespace tbb

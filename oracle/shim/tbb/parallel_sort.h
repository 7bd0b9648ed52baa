// Test-infrastructure shim (oracle/_ref only): oneTBB parallel_sort via the
// libstdc++ parallel mode sort. The reference only sorts with strict total
// orders (P/src/column.cpp:25-30, P/src/relation.cpp:54-61), so the result is
// the unique sorted permutation regardless of the sorting algorithm.
#pragma once
#include <algorithm>
#ifdef _OPENMP
#include <parallel/algorithm>
#endif

namespace tbb {

template <typename It, typename Cmp>
void parallel_sort(It first, It last, const Cmp& cmp) {
#ifdef _OPENMP
    __gnu_parallel::sort(first, last, cmp);
#else
    std::sort(first, last, cmp);
#endif
}

} // namespace tbb

// Test-infrastructure shim (oracle/_ref only): oneTBB task_arena mapped to an
// OpenMP thread count for the duration of execute().
#pragma once
#ifdef _OPENMP
#include <omp.h>
#endif

namespace tbb {

class task_arena {
public:
    explicit task_arena(int threads = 0) : threads_(threads) {}

    template <typename F>
    void execute(const F& f) const {
#ifdef _OPENMP
        const int saved = omp_get_max_threads();
        if (threads_ > 0) omp_set_num_threads(threads_);
        f();
        omp_set_num_threads(saved);
#else
        f();
#endif
    }

private:
    int threads_;
};

} // namespace tbb

// Test-infrastructure shim (oracle/_ref only): the subset of oneTBB's
// blocked_range the reference uses (P/include/colog/parallel.hpp:33).
// Not reference source; written for building the reference as a checker.
#pragma once
#include <cstddef>

namespace tbb {

template <typename T>
class blocked_range {
public:
    blocked_range(T b, T e, std::size_t grain = 1) : b_(b), e_(e), grain_(grain) {}
    T begin() const { return b_; }
    T end() const { return e_; }
    std::size_t grainsize() const { return grain_; }

private:
    T b_, e_;
    std::size_t grain_;
};

} // namespace tbb

// Test-infrastructure shim (oracle/_ref only): absl::flat_hash_map as
// std::unordered_map. The reference never observes iteration order except
// through map equality (P/tests/column_test.cpp:159), so results are unchanged.
#pragma once
#include <unordered_map>

namespace absl {

template <typename K, typename V, typename Hash = std::hash<K>, typename Eq = std::equal_to<K>>
using flat_hash_map = std::unordered_map<K, V, Hash, Eq>;

} // namespace absl

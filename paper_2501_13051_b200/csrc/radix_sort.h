// Stable LSD radix sort (onesweep) entry points. Each sorts by bits
// [begin_bit, end_bit) using the *_alt buffers as ping-pong space and returns
// true when the sorted result ended up in the *_alt buffers.
#pragma once

#include "fv_common.cuh"

namespace fv {

bool radix_sort_pairs_u32(Ctx* c, u32* keys, u32* keys_alt, u32* vals, u32* vals_alt, u64 n,
                          u32 begin_bit, u32 end_bit);
bool radix_sort_keys_u32(Ctx* c, u32* keys, u32* keys_alt, u64 n, u32 begin_bit, u32 end_bit);
bool radix_sort_pairs_u64(Ctx* c, u64* keys, u64* keys_alt, u32* vals, u32* vals_alt, u64 n,
                          u32 begin_bit, u32 end_bit);
bool radix_sort_keys_u64(Ctx* c, u64* keys, u64* keys_alt, u64 n, u32 begin_bit, u32 end_bit);

// Number of significant bits of v (0 for v == 0).
inline u32 bit_width_u64(u64 v) {
    u32 b = 0;
    while (v) {
        ++b;
        v >>= 1;
    }
    return b;
}

}  // namespace fv

// Device-resident column store: the B200 form of colog::Column / Version /
// Relation (P/include/colog/column.hpp:26-64, P/include/colog/relation.hpp).
//
// HBM layout of one Column (n rows, u distinct values):
//   raw        u32[n]   values in insertion order (uncompressed, like FVlog)
//   sorted_idx u32[n]   ids ordered by (value, id)
//   ukeys      u32[u]   distinct values, ascending
//   ustart     u32[u]   first position of the value's run in sorted_idx
//   ucount     u32[u]   run length
//   hash       u64[2^k] open-addressing table (value << 32 | run index),
//                       2^k >= 2u, so a probe is ~1 HBM/L2 sector
// Because the index is built from already-sorted unique keys, the table has
// no duplicate-key chains (the paper's point against pure GPU hash maps).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "fv_common.cuh"

namespace fv {

struct HashIndex {
    DBuf<u64> slots;
    u32 mask = 0;
};

constexpr u64 kEmptySlot = ~u64(0);

struct Column {
    Ctx* ctx = nullptr;
    u64 n = 0;
    DBuf<u32> raw;
    DBuf<u32> sorted_idx;
    u64 n_unique = 0;
    DBuf<u32> ukeys, ustart, ucount;
    HashIndex ht;
};

struct Version {
    Ctx* ctx = nullptr;
    u32 arity = 0;
    u64 rows = 0;
    std::vector<std::unique_ptr<Column>> cols;
};

struct Relation {
    Ctx* ctx = nullptr;
    std::string name;
    u32 arity = 0;
    std::unique_ptr<Version> full, delta, new_rows;
};

struct Array {
    Ctx* ctx = nullptr;
    u64 n = 0;
    u32 elem = 4;
    DBuf<u8> bytes;
    template <typename T>
    T* as() const {
        return reinterpret_cast<T*>(bytes.get());
    }
};

struct Match {
    Ctx* ctx = nullptr;
    u64 m = 0;
    DBuf<u32> starts, counts, matched;
};

// ---- column / version construction ---------------------------------------

// Build all index layers over a device raw array (takes ownership).
std::unique_ptr<Column> column_build(Ctx* c, DBuf<u32>&& raw, u64 n);
// Index layers only (build_index, P/src/column.cpp:17-43).
void build_index(Ctx* c, const u32* raw, u64 n, DBuf<u32>& sorted_idx, DBuf<u32>& ukeys,
                 DBuf<u32>& ustart, DBuf<u32>& ucount, u64& n_unique);
void build_hash(Ctx* c, const u32* ukeys, u64 n_unique, HashIndex& ht);

std::unique_ptr<Version> version_empty(Ctx* c, u32 arity);
// Takes ownership of arity device columns of n rows each.
std::unique_ptr<Version> version_from_device(Ctx* c, std::vector<DBuf<u32>>&& cols, u64 n);

// ---- operator mirrors ------------------------------------------------------

// Probe values (device) -> per value (start, count), count = 0 on miss.
void column_probe_device(Ctx* c, const Column& col, const u32* values, u64 n, u32* starts,
                         u32* counts);
// Check ids < bound; throws FV_ERR_RANGE with msg otherwise.
void check_ids(Ctx* c, const u32* ids, u64 n, u64 bound, const char* msg);
DBuf<u32> gather_device(Ctx* c, const u32* src, const u32* ids, u64 n);
std::unique_ptr<Match> join_probe_phase(Ctx* c, const u32* probe, u64 n, const Column& build);
u64 join_total_size(Ctx* c, const Match& m);
DBuf<u64> join_offsets(Ctx* c, const Match& m);  // m + 1 entries
void join_write_phase(Ctx* c, const Match& m, const u64* offsets, u64 total, const Column& build,
                      DBuf<u32>& a, DBuf<u32>& b);
void filter_pairs_eq(Ctx* c, const u32* a, const u32* b, u64 n, const Column& ca,
                     const Column& cb, DBuf<u32>& oa, DBuf<u32>& ob, u64& n_out);
DBuf<u32> filter_neq(Ctx* c, const Version& v, u32 i, u32 j, u64& n_out);
DBuf<u32> select_eq(Ctx* c, const Column& col, u32 v, u64& n_out);
std::unique_ptr<Version> project(Ctx* c, const Version& v, const u32* ids, u64 n,
                                 const std::vector<u32>& col_map);
std::unique_ptr<Version> dedup_rows(Ctx* c, const Version& v);
bool has_duplicate_rows(Ctx* c, const Version& v);
DBuf<u8> deduplicate(Ctx* c, const Version& nv, const Version& full);
std::unique_ptr<Version> difference(Ctx* c, const Version& nv, const u8* flags);
std::unique_ptr<Version> version_append(Ctx* c, const Version& v, const Version& extra);

// Row-major reconstruct to host.
void version_reconstruct(const Version& v, u32* rows_out);

// Lexicographic (row, id) ordering permutation of a version's rows via
// stable LSD passes over the columns (last column first).
DBuf<u32> lexicographic_order(Ctx* c, const u32* const* cols, u32 arity, u64 n,
                              const char* who = __builtin_FUNCTION());

// Process-wide gather counter (P/src/column.cpp:10-15).
void add_gather_volume(u64 n);
u64 gather_volume();
void reset_gather_volume();

}  // namespace fv

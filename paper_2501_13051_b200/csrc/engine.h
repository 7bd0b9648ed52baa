// Device-resident semi-naive fixpoint engine (P/src/engine.cpp re-designed
// for B200).
//
// Relation storage in HBM: every version (FULL, DELTA) of a relation is a
// set of SoA u32 columns kept *sorted lexicographically and distinct*. That
// one invariant replaces the reference's per-column (raw, sorted_idx,
// hash) triple for the engine's purposes:
//   - a join on column 0 probes contiguous runs of the version itself;
//     other join columns get a cached sorted copy;
//   - dedup of NEW against FULL and the FULL <- FULL u DELTA merge become a
//     single merge-path pass over two sorted sequences (no triangle join);
//   - DELTA comes out of that pass already sorted, ready to be indexed.
// Rows are compared as packed row keys: W = ceil(arity/2) u64 words, word w
// = (c[2w] << s) | c[2w+1], with s the bit width of the active domain (no
// IDB value can exceed the EDB/constant maximum: heads only project body
// variables).
#pragma once

#include <map>
#include <memory>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "column.h"
#include "fv_common.cuh"

namespace fv {

// ---- plan IR (P/include/colog/compiler.hpp:14-53) --------------------------

struct ColRef {
    u32 source = 0, col = 0;
    bool operator==(const ColRef& o) const { return source == o.source && col == o.col; }
    bool operator<(const ColRef& o) const {
        return source != o.source ? source < o.source : col < o.col;
    }
};

struct PlanSource {
    std::string relation;
    u32 arity = 0;
    std::vector<std::pair<u32, u32>> const_selects;  // (col, value)
    std::vector<std::pair<u32, u32>> self_eqs;       // (first col, repeated col)
    bool constrained() const { return !const_selects.empty() || !self_eqs.empty(); }
};

struct PlanJoin {
    u32 right_source = 0;
    ColRef left;
    u32 right_col = 0;
    std::vector<std::pair<ColRef, u32>> residual_eq;
};

struct Plan {
    std::string head;
    u32 head_arity = 0;
    std::vector<PlanSource> sources;
    std::vector<PlanJoin> joins;
    std::vector<ColRef> output_cols;
    std::vector<std::pair<u32, u32>> guard_neq;
};

struct RelationDecl {
    std::string name;
    u32 arity = 0;
};

struct FactsBlock {
    std::string relation;
    u32 arity = 0;
    u64 n = 0;
    std::vector<const u32*> cols;  // host SoA
};

// ---- device relation storage ------------------------------------------------

struct DevVersion {
    u64 n = 0;
    std::vector<DBuf<u32>> cols;
    // Rows in lexicographic (col 0, col 1, ...) order (sorted FULL / DELTA,
    // seeded EDB): a word build of it needs no sort.
    bool lex_sorted = false;
    std::vector<const u32*> ptrs() const {
        std::vector<const u32*> p;
        for (auto& c : cols) p.push_back(c.get());
        return p;
    }
};

// Join index over one column of a version: rows grouped by the key column.
struct JoinIndex {
    const DevVersion* rows = nullptr;  // rows ordered by the key column
    DevVersion owned;                  // sorted copy when the key is not column 0
    u64 n_unique = 0;
    DBuf<u32> ukeys, ustart, ucount;
    HashIndex ht;
    // domain > 0: direct-address index (from a counting-sort grouping):
    // ustart/ucount have `domain` entries indexed by value, no ukeys/ht.
    u64 domain = 0;
    // direct index built from sorted keys: ustart holds interleaved
    // (start, end) pairs per value (end exclusive; 0 = no run) and ucount is
    // empty — one pass to build, one 8-byte load per probe (the
    // counting-sort grouping's index keeps separate starts and counts).
    bool ends = false;
};

using IndexMap = std::map<std::pair<int, u32>, std::unique_ptr<JoinIndex>>;

// A binary version in word form for the build side of a composition join
// (RelState::word_builds): columns (x, z & ~31, mask) grouped by x, with its
// join index on column 0.
struct WordBuild {
    DevVersion words;
    JoinIndex idx;
};

// Open-addressing set of packed row keys (empty slot = all ones, which no
// key can equal when 2 * shift < 64), load factor <= 1/2 (3/4 when memory
// forced a smaller table).
struct KeySet {
    DBuf<u64> slots;
    u64 mask = 0;
    u64 count = 0;
    u32 group_bits = 0;  // home-slot layout (engine_kernels.cu keyset_home)
    u64 limit = 0;       // most keys (worst case) the table accepts before growing
    u64 capacity() const { return slots.size(); }
};

// Blocked-bitmap set of packed row keys (binary or unary relations): the
// relation's (a, b) value grid cut into 32 x 32-bit blocks, one 128-byte
// bitmap per non-empty block (row a & 31 is the word, b & 31 the bit; unary:
// 1024 consecutive values). A directory (open addressing, empty = all ones,
// load <= 1/2) maps block ids to slots; bits[32 * slot ...] is that block's
// bitmap. Relations whose tuples cluster in id space (components, trees,
// dense closures) take a fraction of a byte per tuple instead of the key
// set's 16-32, so a fixpoint's whole FULL fits in L2 and a membership test +
// insert is one L2 atomic instead of a random DRAM line. The engine falls
// back to a KeySet when a relation turns out sparse (< kBlockMinDensity
// tuples per block).
struct BlockSet {
    DBuf<u64> dir;
    DBuf<u32> bits;
    DBuf<u32> dbits;  // word form: this iteration's new bits, same layout as `bits`
    u64 generation = 0;  // directory growths so far (recorded word indices die with one)
    DBuf<u64> count;  // device: blocks claimed
    u64 mask = 0;
    u64 blocks = 0;   // host copy of `count` (last read)
    double ratio = 0.0;  // new blocks per candidate, recent maximum (growth estimate)
    u64 capacity() const { return dir.size(); }
};

// Device view of a BlockSet (kernel argument).
struct BlockSetArgs {
    u64* dir = nullptr;
    u32* bits = nullptr;
    u32* dbits = nullptr;  // word form only
    u64 mask = 0;
    u64* count = nullptr;
    u64 limit = 0;  // no new block is claimed once `count` reaches this
    u32 shift = 0, arity = 2;
};

// A partition copy of a relation keyed on a column other than 0 (partitioned
// evaluation only): the rows whose owner(hash(row[col])) is this rank.
struct RelCopy {
    DevVersion full, delta;
    IndexMap indexes;
};

struct RelState {
    std::string name;
    u32 arity = 0;
    bool idb = false;
    // Home copy: all rows (single GPU) or the rows owned by hash(col home).
    u32 home = 0;
    DevVersion full, delta;
    // FULL before the last merge (= FULL minus DELTA), kept when some variant
    // reads it (exactly-once semi-naive variants); old_is_full when the last
    // iteration added nothing.
    bool keep_old = false;
    bool old_is_full = true;
    DevVersion full_old;
    // (0 = full, 1 = delta, col) -> index; invalidated when the version changes
    IndexMap indexes;
    // Partitioned evaluation: extra copies keyed on other probed columns
    // (never on `home`: the home copy is full/delta above).
    std::map<u32, std::unique_ptr<RelCopy>> copies;
    std::set<u32> keyset;  // partition columns this relation is needed on
    // Hash dedup (arity <= 2): the key set of the home FULL. Candidates are
    // inserted straight from the join kernel; only new rows get sorted.
    bool hash_mode = false;
    KeySet keys;
    // Hash mode with a BlockSet instead of `keys` (keys.count still counts
    // FULL's rows); cleared when the relation proves sparse.
    bool block_mode = false;
    BlockSet blocks;
    // Word form (block mode, levels mode, binary; single GPU): DELTA and the
    // levels are words — columns (x, z & ~31, mask of the z's present),
    // grouped by x — so the composition variant that probes DELTA on
    // column 0 (right-linear TC) emits one candidate per word, and FULL's
    // bitmap takes one OR per word. A DevVersion with arity + 1 columns is in
    // word form. Left when the block set turns out sparse (word_sparse).
    bool word_mode = false;
    bool word_sparse = false;
    // Word sink (block mode, binary, single GPU): every insert into the
    // relation goes through the word protocol (FULL bitmap OR + per-block
    // DELTA bitmap, first writer appends), so composition joins can emit
    // whole words into it; with word_mode off its DELTA is expanded back to
    // tuples at finalize. word_mode implies word_sink.
    bool word_sink = false;
    // FULL ordered by (col 1, col 0) with its column-1 join index (binary,
    // sorted FULL, single GPU): built once when a join first probes FULL on
    // column 1, then maintained by merging each sorted DELTA into it (no
    // per-iteration re-sort of FULL).
    std::unique_ptr<JoinIndex> by1;
    std::unique_ptr<JoinIndex> old_by1;  // the same for FULL - DELTA (the FULL the last merge replaced)
    // Word forms of this relation's versions built for composition joins
    // (key: Which), invalidated with `indexes`.
    std::map<int, std::unique_ptr<WordBuild>> word_builds;
    // A join's temporary word sink (word intermediates): never leaves the
    // word form (its result is consumed right away).
    bool temp = false;
    // Partitioned runs: the home column's owner is owner(v >> owner_shift).
    // A word-form relation owns whole 32-value windows (shift 5), so every
    // word of its DELTA lives on one rank.
    u32 owner_shift = 0;
    // With hash dedup, a FULL no join reads is kept as levels: the past DELTAs
    // (one per iteration, grouped by column 0) plus the current `delta`,
    // concatenated and sorted only for dumps; otherwise it is `full`, merged
    // with each sorted Δ.
    bool levels_mode = false;
    std::vector<DevVersion> levels;
    u64 level_rows = 0;
    u64 rows() const { return levels_mode ? level_rows : full.n; }
};

struct IterStat {
    u64 iteration = 0;
    std::string relation;
    u64 delta_rows = 0, full_rows = 0, merges = 0;
    double elapsed_ms = 0.0;
};

struct EvalState {
    Ctx* ctx = nullptr;
    std::map<std::string, std::unique_ptr<RelState>> relations;  // std::map order
    u64 iterations = 0;
    std::vector<IterStat> stats;  // global (all-reduced) counts in a partitioned run
    double elapsed_ms = 0.0;
    u32 key_shift = 32;
    int rank = 0, world = 1;  // this state's partition
    Ctx* owned_ctx = nullptr;  // virtual-rank context owned by the state
    ~EvalState() {
        relations.clear();
        if (owned_ctx) ctx_delete(owned_ctx);
    }
};

// EDB resident in HBM (unsorted, possibly duplicated rows, per relation).
struct DeviceEdb {
    std::map<std::string, DevVersion> rels;
};

DeviceEdb upload_facts(Ctx* c, const std::vector<RelationDecl>& decls, const std::vector<FactsBlock>& facts);

// Host facts: upload + seed + fixpoint (elapsed_ms spans all three, the
// reference's evaluate() boundary, P/src/runner.cpp:58-61).
std::unique_ptr<EvalState> evaluate(Ctx* c, const std::vector<RelationDecl>& decls,
                                    const std::vector<Plan>& plans,
                                    const std::vector<FactsBlock>& facts);
// EDB already resident: seed + fixpoint.
std::unique_ptr<EvalState> evaluate_device(Ctx* c, const std::vector<RelationDecl>& decls,
                                           const std::vector<Plan>& plans,
                                           const std::vector<const DeviceEdb*>& edbs);

// Partitioned evaluation with `world` virtual ranks on c's device (threads,
// in-process transport): the distributed code path on one GPU. Returns one
// state per rank (home partitions; stats are global).
std::vector<std::unique_ptr<EvalState>> evaluate_sharded(Ctx* c, u32 world, const std::vector<RelationDecl>& decls,
                                                         const std::vector<Plan>& plans,
                                                         const std::vector<FactsBlock>& facts);

// Home partition column per IDB relation (partitioned evaluation): the
// column the relation's home copy (key set / levels / sorted FULL) is hash-
// partitioned on. Chosen from the recursive variants: the column whose
// variable the rule carries unchanged from its DELTA atom to the head — for
// right-linear TC, reach(x, z) :- edge(x, y), reach(y, z), column 1 (z): every
// head row is then derived on the rank that owns it, and no candidate crosses
// the interconnect. Relations of arity > 2 and relations with no such column
// use column 0. FVLOG_HOME_COL=0 forces column 0 everywhere.
// `variants`: (plan, delta source) of every executed variant.
std::map<std::string, u32> choose_home_cols(const std::vector<std::pair<const Plan*, long>>& variants,
                                            const std::map<std::string, u32>& idb_arity);

// Static partitioning decisions for one rule plan (partitioned evaluation):
//   src_copy[s]      partition column source s is read from (IDB sources)
//   shuffle[k]       shuffle the intermediate by joins[k].left before step k
//   replicated_out   the derivation only touches replicated (EDB) relations:
//                    its head rows are owner-filtered instead of routed
//   local_out        the intermediate is partitioned on the variable of the
//                    head's home column: every head row is already at its
//                    owner (no routing, no filter)
struct DistPlan {
    std::vector<u32> src_copy;
    std::vector<u8> shuffle;
    bool replicated_out = false;
    bool local_out = false;
};
DistPlan dist_plan(const Plan& p, const std::set<std::string>& idb, const std::map<std::string, u32>& home);

// Validate plan structure against the declarations (throws FV_ERR_PLAN).
void check_plans(const std::vector<RelationDecl>& decls, const std::vector<Plan>& plans);

// Lexicographically sorted row-major dump of FULL (host).
std::vector<u32> dump_sorted(const EvalState& s, const std::string& rel);
// The same rows written straight into a caller's host buffer (rows x arity
// u32): sorted and interleaved on the device, one D2H copy per chunk (pinned
// buffers copy at PCIe / C2C rate).
void dump_sorted_into(const EvalState& s, const std::string& rel, u32* rows_out);
// dump_relation text (integer mode) of the sorted rows, formatted on the device.
std::string dump_sorted_text(const EvalState& s, const std::string& rel);
u64 fingerprint(const EvalState& s, const std::string& rel);

// ---- kernels (engine_kernels.cu) ---------------------------------------------

constexpr int kMaxSlots = 16;
constexpr int kMaxFilters = 8;

// One operand column of the materialize / project kernels.
struct SlotRef {
    const u32* ptr = nullptr;
    u32 side = 0;  // 0: probe-side row i, 1: build-side position p
};

enum FilterOp : u32 { kFilterEq = 0, kFilterNeq = 1, kFilterConst = 2, kFilterOwner = 3 };

struct Filter {
    SlotRef a, b;
    u32 op = kFilterEq;
    u32 value = 0;  // kFilterConst: the constant; kFilterOwner: this rank
    u32 world = 1;  // kFilterOwner: owner(a) = floor(hash32(a >> oshift) * world / 2^32) must equal value
    u32 oshift = 0;  // kFilterOwner: RelState::owner_shift of the owning relation
};

struct OutSpec {
    u32 n_out = 0;  // columns
    SlotRef col[kMaxSlots];
    u32 n_filters = 0;
    Filter f[kMaxFilters];
    // key mode: write W = ceil(n_out/2) packed u64 words per row
    u32 key_mode = 0;
    u32 shift = 32;
    u64* keys[4] = {nullptr, nullptr, nullptr, nullptr};
    u32* out_cols[kMaxSlots] = {nullptr};
    u64* d_count = nullptr;  // compaction counter (n_filters > 0)
    // Hash-insert mode (key mode, one word): instead of writing every
    // candidate, insert it into the relation's key set and append only the
    // keys that were not present to new_keys[*new_count ...].
    u64* ht_slots = nullptr;
    u64 ht_mask = 0;
    u32 ht_group_bits = 0;
    // Tile-local dedup before the key-set probe (off when a relation's
    // candidates are all new rows: nothing to drop; C2 129 -> 112 ms with it).
    u32 tile_set = 1;
    u64* new_keys = nullptr;
    u64* new_count = nullptr;
    u64* probe_count = nullptr;  // optional (trace): key-set probes after the tile-local dedup
    // Partitioned fused dedup: rows whose owner(hash(head col 0)) is not
    // remote_rank are appended to keys[0][*d_count ...] (to be routed)
    // instead of probing the local key set. remote_world = 0: all local.
    u32 remote_world = 0, remote_rank = 0;
    u32 remote_col = 0;  // head column whose owner decides (the home column)
    u32 remote_oshift = 0;  // ... of its value >> remote_oshift
    // Key mode, one word, no key set: drop tile-local repeats and append the
    // tile's distinct keys at keys[0][*d_count ...].
    u32 tile_dedup = 0;
    // Block-set dedup (bs.dir != null, ht_slots null): insert into the
    // relation's BlockSet; candidates it cannot place (claim limit reached,
    // probe run too long) are appended to ovf_keys[*ovf_count ...] for the
    // host to insert after growing the directory.
    BlockSetArgs bs;
    u64* ovf_keys = nullptr;
    u64* ovf_count = nullptr;
    // Word form (block-set dedup of a word-mode head, RelState::word_mode):
    // col[1] is the DELTA side's word base (z & ~31), `wbits` its mask; a
    // word's first DELTA writer appends its key to new_keys, overflow entries
    // carry their masks in ovf_bits, and the new tuples (bits) are counted in
    // *new_tuples.
    SlotRef wbits;
    u32 word_sink = 0;  // the head is a word sink (WORDS kernel; wbits null: one-bit words)
    u32 word_neq = 0;   // word outputs drop the bit of their own x (guard x != z)
    // Profiling only: the tuple candidates the word outputs stand for
    // (sum of their masks' popcounts), for the implementation-independent
    // algorithmic bytes of SURVEY.md §8(d).
    u64* cand_count = nullptr;
    u32* ovf_bits = nullptr;
    u32* new_widx = nullptr;  // bitmap word index of each appended new word
    u64* new_tuples = nullptr;
};

FV_HD inline bool fused_set(const OutSpec& s) { return s.ht_slots != nullptr || s.bs.dir != nullptr; }

// Insert n keys; the ones not yet present are appended to
// new_keys[*d_new ...] (device counter, not reset here).
void engine_hash_insert(Ctx* c, const u64* keys, u64 n, KeySet& set, u64* new_keys, u64* d_new);
// BlockSet: allocate `cap` (power of two) empty slots; the count starts at
// `blocks`; delta_bits: also the (zeroed) DELTA bitmap of the word form.
void engine_blockset_alloc(Ctx* c, BlockSet& s, u64 cap, u64 blocks, bool delta_bits = false);
// Move every block of `from` into the freshly allocated `to` (bitmaps copied whole).
void engine_blockset_grow(Ctx* c, const BlockSet& from, BlockSet& to);
// Insert n keys; new ones are appended to new_keys[*d_new ...] (when
// new_keys), unplaceable ones to ovf[*d_ovf ...].
void engine_blockset_insert(Ctx* c, const u64* keys, u64 n, const BlockSetArgs& s, u64* new_keys, u64* d_new,
                            u64* ovf, u64* d_ovf);
// Move every key of `from` into the (emptied) `to` by scanning from's slots
// in order: with the same layout a key's home in `to` is its old slot plus a
// multiple of from's capacity, so the inserts stream through L2 instead of
// landing at random; a layout change (group_bits) re-scatters them
// (to.count is not touched).
void engine_hash_rehash(Ctx* c, const KeySet& from, KeySet& to);
// Growth by a power-of-two factor with the same layout bits: writes every
// slot of `to` (no memset needed) from `from`'s keys. False when it does not
// apply or its overflow list filled up; `to` must then be reset and rehashed.
bool engine_hash_grow(Ctx* c, const KeySet& from, KeySet& to);
// Distinct rows of lexicographically sorted packed keys -> SoA columns
// (arity <= FV_MAX_ARITY); returns the distinct count.
u64 engine_unique_unpack(Ctx* c, const std::vector<DBuf<u64>>& words, u64 n, u32 arity, u32 shift,
                         const std::vector<u32*>& cols);
// Group n one-word arity-2 keys by their first column (key >> shift; order
// inside a group unspecified) by counting sort; false (keys untouched) when
// the first-column domain exceeds 2^24 or averages > 512 keys per value.
// With `runs`, also fills its column-0 run index (ukeys/ustart/ucount +
// hash; rows left to the caller) for the grouped keys.
// With col0/col1, the grouped rows are written as SoA columns instead
// (keys left as they were). pay_in/pay_out: a u32 payload per key moved
// along (word masks).
// gather_idx / gather_src: the payload is gather_src[gather_idx[i]] instead
// (cleared after the read) — the word masks straight from the DELTA bitmap.
bool engine_group_keys(Ctx* c, DBuf<u64>& keys, u64 n, u32 shift, JoinIndex* runs = nullptr, u32* col0 = nullptr,
                       u32* col1 = nullptr, const u32* pay_in = nullptr, u32* pay_out = nullptr,
                       const u32* gather_idx = nullptr, u32* gather_src = nullptr);
// Word-form block-set insert (RelState::word_mode): n word keys with masks
// `bits`, or packed binary tuple keys (bits null) as one-bit words. New bits
// are OR-ed into FULL and into the DELTA bitmap (s.dbits); a word's first
// DELTA writer appends its key to new_keys[*d_new ...] and *d_tuples counts
// the new bits; entries without a directory slot go to ovf/ovf_bits[*d_ovf ...].
// new_widx (parallel to new_keys) records the entry's bitmap word index.
void engine_blockset_word_insert(Ctx* c, const u64* keys, const u32* bits, u64 n, const BlockSetArgs& s,
                                 u64* new_keys, u32* new_widx, u64* d_new, u64* d_tuples, u64* ovf, u32* ovf_bits,
                                 u64* d_ovf);
// The merged DELTA masks of n word keys (each inserted this iteration), read
// from s.dbits into out_bits and cleared there; widx (recorded word indices,
// valid while the directory has not grown) or null (look the blocks up).
void engine_blockset_collect(Ctx* c, const u64* keys, const u32* widx, u64 n, const BlockSetArgs& s, u32* out_bits);
// fingerprint() of a block set's rows, from its bitmaps.
u64 engine_blockset_fingerprint(Ctx* c, const BlockSet& s, u32 arity);
// Distinct block ids among n packed keys (directory sizing).
u64 engine_count_blocks(Ctx* c, const u64* keys, u64 n, u32 shift, u32 arity);
// The same count left in *d_out on the device (no host round trip).
void engine_count_blocks_async(Ctx* c, const u64* keys, u64 n, u32 shift, u32 arity, u64* d_out);
// HyperLogLog sketch of the distinct block ids (kBlockSketchRegs u32
// registers at regs, zeroed by the call; arity 0: of the distinct keys);
// block_sketch_estimate turns the downloaded registers into a count (~1.6 %
// standard error).
constexpr int kBlockSketchRegs = 4096;
void engine_block_sketch(Ctx* c, const u64* keys, u64 n, u32 shift, u32 arity, u32* regs);
u64 block_sketch_estimate(const u32* regs);
// Packed tuple keys of n word entries (word key, mask) into out, sized by
// the caller to the sum of the masks' popcounts (no host readback).
// off_out (optional, n + 1 entries): each entry's first tuple (and the
// total at [n]) kept for the caller.
void engine_expand_word_keys(Ctx* c, const u64* keys, const u32* bits, u64 n, u64* out, u32* out_x = nullptr,
                             u32* out_z = nullptr, u32 shift = 0, u64* off_out = nullptr);
// A direct index over word entries grouped by x (counting-sort runs: word
// start + word count per value) -> the direct index of their expanded tuples
// (interleaved (start, end) pairs), from the entries' tuple offsets.
void engine_word_index_to_tuples(Ctx* c, const JoinIndex& words, const u64* off, JoinIndex& out);
// Word form (x, z base, mask) of a lexicographically sorted binary version
// of n rows; outputs sized n; returns the word count.
u64 engine_tuples_to_words(Ctx* c, const u32* c0, const u32* c1, u64 n, u32* x, u32* zb, u32* bits,
                            bool exact = true);
// The non-empty words of a binary block set in row-major (x, z) order —
// FULL's word form straight from its bitmaps; outputs hold cap_out entries.
u64 engine_blockset_words(Ctx* c, const BlockSet& s, u32* x, u32* zb, u32* bits, u64 cap_out, u32 key_shift);
// FULL of a block-set relation as lexicographically sorted SoA rows (c0, and
// c1 for binary relations; null c0: count only), decoded from the bitmaps in
// order — no sort of the tuples. Returns the row count.
u64 engine_blockset_dump(Ctx* c, const BlockSet& s, u32 arity, u32* c0, u32* c1);
// Tuples (x, z) of n word entries (x, z base, mask), entry order kept (so
// entries grouped by x give tuples grouped by x); returns the tuple count.
// out_x null: count only.
// count false: no readback (the caller knows the total), returns 0.
u64 engine_expand_words(Ctx* c, const u32* x, const u32* zb, const u32* bits, u64 n, u32* out_x, u32* out_z,
                        bool count = true);
// Distinct rows of sorted packed keys into fresh word buffers; returns the count.
u64 engine_unique_words(Ctx* c, const std::vector<DBuf<u64>>& words, u64 n, std::vector<DBuf<u64>>& out);
// SoA columns -> row-major rows out[i * arity + j] (device buffer).
void engine_interleave(Ctx* c, const std::vector<const u32*>& cols, u64 n, u32* out);
// Keys -> SoA columns (one word per row, arity <= 2).
void engine_unpack_keys(Ctx* c, const u64* keys, u64 n, u32 arity, u32 shift, const std::vector<u32*>& cols);

struct RowFilter {  // predicate on probe-side rows (source constraints)
    u32 n = 0;
    Filter f[kMaxFilters];
};

// counts[i] = run length of probe[i] in the index (0 on miss or when the
// probe row fails `pred`); starts[i] = run start.
// Probe counts scanned straight into offsets[n + 1] (offsets[n] = total),
// one single-pass kernel; starts as for engine_probe_count.
void engine_probe_offsets(Ctx* c, const u32* probe, u64 n, const JoinIndex& idx, const RowFilter& pred,
                          u32* starts, u64* offsets);
void engine_probe_count(Ctx* c, const u32* probe, u64 n, const JoinIndex& idx, const RowFilter& pred,
                        u32* starts, u32* counts);
// Ascending ids of rows passing `pred` (side 0); returns the count.
u64 engine_select_rows(Ctx* c, u64 n, const RowFilter& pred, u32* ids);
// Output-partitioned expansion of T join outputs into `spec`; only outputs
// [o_begin, o_end) when given (chunked fused dedup; positional writes of the
// uncompacted mode stay global output indices).
void engine_materialize(Ctx* c, const u64* offsets, u64 m, u64 total, const u32* starts,
                        const OutSpec& spec, u64 o_begin = 0, u64 o_end = ~u64(0));
// Single-source projection of n rows (side 0 only) into `spec`.
void engine_project(Ctx* c, u64 n, const OutSpec& spec);
// RLE of a sorted key column into (ukeys, ustart, ucount) + hash table.
// key_bits (the key domain's bit width, when <= 24): a direct-address index
// instead of runs + hash (no host readback).
// force_direct: a direct-address index whenever key_bits allows one (the
// caller accepts the 2^key_bits arrays however few the rows).
void engine_build_runs(Ctx* c, const u32* sorted_keys, u64 n, JoinIndex& idx, u32 key_bits = 0,
                       bool force_direct = false);
// Pack SoA columns into W key words.
void engine_pack_keys(Ctx* c, const std::vector<const u32*>& cols, u64 n, u32 shift, u64* const* words);
// p[i] = (p[i] & and_mask) | or_bits (tagging / untagging packed keys).
void engine_mask_u64(Ctx* c, u64* p, u64 n, u64 and_mask, u64 or_bits);
// Merge sorted distinct A (SoA, arity) with sorted B keys (W words, dups
// allowed): C = A u B (SoA), D = B \ A distinct (SoA). Returns |D| (device
// scalar written to *d_new; |C| = n_a + |D|).
void engine_merge(Ctx* c, const std::vector<const u32*>& a_cols, u64 n_a, u64* const* b_words, u64 n_b,
                  u32 arity, u32 shift, const std::vector<u32*>& c_cols,
                  const std::vector<u32*>& d_cols, u64* d_new);
u64 engine_fingerprint(Ctx* c, const std::vector<const u32*>& cols, u64 n, u32 arity);

// Destination rank of a row: owner(hash32(v)) where v is a u32 column value
// or the high/low half of a packed key word.
struct RouteKey {
    const u32* col = nullptr;   // u32 column, or
    const u64* word = nullptr;  // packed key word: v = hi ? word >> shift : word & mask
    u32 shift = 0;
    u32 hi = 0;
    u64 mask = ~u64(0);
    u32 oshift = 0;  // owner of v >> oshift (RelState::owner_shift)
};
// Group n rows by destination rank: u32 columns `c32` and u64 columns `c64`
// are scattered into the matching *_out buffers (capacity n) so that rows for
// rank p occupy [off[p], off[p] + cnt[p]) (order inside a bucket unspecified).
// d_counts_out (device, world entries): the counts stay on the device there
// and cnt/off are not filled (no host round trip; the exchange reads them).
void engine_route(Ctx* c, u64 n, const RouteKey& key, u32 world, const std::vector<const u32*>& c32,
                  const std::vector<u32*>& c32_out, const std::vector<const u64*>& c64,
                  const std::vector<u64*>& c64_out, u64* cnt, u64* off, u64* d_counts_out = nullptr);
// Sort W-word keys in place (LSD over words with a permutation payload).
// Sort packed row keys lexicographically. group_only (one-word keys only):
// order by the first column alone (rows grouped for a column-0 join index;
// within a group the order is unspecified) — skips the low-column passes.
void engine_sort_keys(Ctx* c, std::vector<DBuf<u64>>& words, u64 n, u32 arity, u32 shift, bool group_only = false,
                      const char* who = __builtin_FUNCTION());

}  // namespace fv

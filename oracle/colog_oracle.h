/*
 * TEST INFRASTRUCTURE — ORACLE, NOT PRODUCT.
 *
 * colog_oracle: a plain-C, single-threaded restatement of the reference's
 * column-store algorithms (P = /root/reference/proj). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker. Pinned against the reference itself: the golden
 * vectors in tests/golden/ were produced by the unmodified reference
 * (oracle/_ref/libcolog_ref.so, tests/golden/make_golden.py) and
 * tests/test_oracle.py checks this restatement against them.
 */
#ifndef COLOG_ORACLE_H
#define COLOG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* build_index (P/src/column.cpp:17-43): sorted_idx[n] ordered by (value, id);
 * unique runs written as (keys, starts, counts) ascending by key; returns the
 * number of distinct values. */
uint64_t or_build_index(const uint32_t* raw, uint64_t n, uint32_t* sorted_idx, uint32_t* keys,
                        uint32_t* starts, uint32_t* counts);

/* join_probe_phase + join_total_size (P/src/kernels.cpp:59-92): for each
 * probe value in order, the build column's run; misses dropped. Returns the
 * number of matched probe rows; *total receives the join size. */
uint64_t or_join_probe(const uint32_t* probe, uint64_t np, const uint32_t* build, uint64_t nb,
                       uint32_t* m_starts, uint32_t* m_counts, uint32_t* matched, uint64_t* total);

/* column_join (P/src/kernels.cpp:104-135): pairs in the reference's order
 * (probe-major, sorted_idx order inside a run). a/b sized by or_join_probe's
 * total. */
void or_column_join(const uint32_t* probe, uint64_t np, const uint32_t* build, uint64_t nb,
                    uint32_t* a_ids, uint32_t* b_ids);

/* dedup_rows (P/src/relation.cpp:71-89) over SoA cols[arity][n] stored
 * column-major in one array (col j at cols + j*n). Output column-major with
 * stride n, first-occurrence order; returns the distinct row count. */
uint64_t or_dedup_rows(const uint32_t* cols, uint64_t n, uint32_t arity, uint32_t* out);

/* deduplicate (P/src/kernels.cpp:210-255, Algorithm 2): flags[i] = 1 iff row
 * i of NEW occurs in FULL. */
void or_deduplicate(const uint32_t* new_cols, uint64_t n_new, const uint32_t* full_cols,
                    uint64_t n_full, uint32_t arity, uint8_t* flags);

/* filter_neq (P/src/kernels.cpp:167-178): ascending ids with col i != col j. */
uint64_t or_filter_neq(const uint32_t* cols, uint64_t n, uint32_t ci, uint32_t cj, uint32_t* ids);

/* select_eq (P/src/kernels.cpp:38-46). */
uint64_t or_select_eq(const uint32_t* raw, uint64_t n, uint32_t v, uint32_t* ids);

/* ---- semi-naive engine (P/src/engine.cpp) over compiled plans ------------
 *
 * The plan is passed flattened as uint32 words (format in colog_oracle.c,
 * "PLAN ENCODING"), relations are dense indices 0..n_rel-1. Facts are
 * column-major per relation. The result (every relation's FULL) is returned
 * row-major and lexicographically sorted via or_state_* accessors. */
typedef struct or_state or_state;
or_state* or_evaluate(uint32_t n_rel, const uint32_t* arities, const uint32_t* plan_words,
                      uint64_t n_plan_words, const uint32_t* const* facts, const uint64_t* n_facts);
uint64_t or_state_iterations(const or_state* s);
uint64_t or_state_rows(const or_state* s, uint32_t rel);
/* Row-major sorted rows of FULL. */
void or_state_dump(const or_state* s, uint32_t rel, uint32_t* out);
/* Delta rows of relation rel at iteration it (0 when rel is no head). */
uint64_t or_state_delta(const or_state* s, uint64_t it, uint32_t rel);
void or_state_free(or_state* s);

#ifdef __cplusplus
}
#endif

#endif

/*
 * fvlog.h — C ABI of the B200-native column-oriented Datalog runtime.
 *
 * This is the drop-in boundary for the reference's hot path (the `colog`
 * static library; the reference itself exports no C ABI).
 * Every entry point below names the reference symbol it replaces
 * (P/ = /root/reference/proj). Conventions:
 *
 *   - All host-facing pointers are plain host memory (uint32_t SoA columns,
 *     row-major row blocks, caller-allocated outputs). No torch or CUDA types
 *     appear in a signature; device residency is hidden behind opaque handles.
 *   - Value semantics of the reference (every operator returns a fresh
 *     Version/vector) become "returns a fresh handle the caller frees".
 *   - Reference exceptions map to status codes (throw sites in P/src):
 *       std::invalid_argument (arity/length mismatch) -> FV_ERR_ARITY
 *       std::out_of_range   (gather OOB, bad column)  -> FV_ERR_RANGE
 *       std::length_error   (> 2^32 rows)              -> FV_ERR_LENGTH
 *       DiagnosticError     (parse/validate/compile)   -> FV_ERR_PLAN
 *       std::runtime_error  (I/O)                      -> FV_ERR_IO
 *     plus FV_ERR_OOM / FV_ERR_CUDA for device failures. The message of the
 *     last failure on a context is fv_last_error(ctx) (fv_global_error() for
 *     calls without a context).
 *   - A context owns one CUDA device and one stream and is not thread-safe,
 *     like the reference's single-threaded caller contract
 *     (P/include/colog/parallel.hpp:15-18). There is no CPU fallback: every
 *     data-parallel operator runs as sm_100a kernels.
 */
#ifndef FVLOG_H
#define FVLOG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FVLOG_ABI_VERSION 1
#define FV_MAX_ARITY 8

typedef enum fv_status {
    FV_OK = 0,
    FV_ERR_ARITY = 1,
    FV_ERR_RANGE = 2,
    FV_ERR_LENGTH = 3,
    FV_ERR_PLAN = 4,
    FV_ERR_IO = 5,
    FV_ERR_OOM = 6,
    FV_ERR_CUDA = 7,
    FV_ERR_INVALID = 8
} fv_status;

typedef struct fv_ctx fv_ctx;
typedef struct fv_array fv_array;       /* device u32 / u8 / u64 vector */
typedef struct fv_column fv_column;     /* colog::Column */
typedef struct fv_version fv_version;   /* colog::Version */
typedef struct fv_relation fv_relation; /* colog::Relation */
typedef struct fv_match fv_match;       /* colog::MatchVector */
typedef struct fv_program fv_program;   /* colog::Program (+ dictionary) */
typedef struct fv_state fv_state;       /* colog::EvaluationState */

/* ---- library / context -------------------------------------------------- */

int fv_abi_version(void);
const char* fv_global_error(void);

/* One context per GPU; `device` is the CUDA ordinal. */
fv_status fv_ctx_create(int device, fv_ctx** out);
void fv_ctx_destroy(fv_ctx* ctx);
const char* fv_last_error(const fv_ctx* ctx);
fv_status fv_ctx_synchronize(fv_ctx* ctx);
/* Grow the context's stream-ordered memory pool to at least `bytes` of
 * mapped device memory now (one allocation, freed back into the pool), so
 * later evaluations sub-allocate from it instead of mapping new memory in
 * the middle of a fixpoint. Optional; no reference counterpart (the
 * reference allocates host vectors per operator). */
fv_status fv_ctx_reserve(fv_ctx* ctx, uint64_t bytes);
/* Number of kernels this context has launched so far (profiling evidence). */
uint64_t fv_ctx_kernel_launches(const fv_ctx* ctx);
/* Host synchronisations (stream syncs + scalar readbacks) issued on ctx so
 * far: the host round trips a fixpoint makes (north_star: ~one scalar per
 * iteration). */
uint64_t fv_ctx_host_syncs(const fv_ctx* ctx);
/* Per-kernel-class timing with CUDA events recorded on the context stream
 * around every launch (enable = 1 clears previous entries). Each entry:
 * launches, summed device milliseconds, summed algorithmic bytes (inputs
 * read once + outputs written once). */
fv_status fv_ctx_profile(fv_ctx* ctx, int enable);
uint32_t fv_ctx_profile_count(const fv_ctx* ctx);
fv_status fv_ctx_profile_entry(const fv_ctx* ctx, uint32_t i, const char** name, uint64_t* launches,
                               double* ms, double* bytes);
/* Process-wide count of values materialized by gathers
 * (P/src/column.cpp:10-15 gather_volume / reset_gather_volume). */
uint64_t fv_gather_volume(void);
void fv_reset_gather_volume(void);

/* ---- device arrays (results of id-producing operators) ------------------ */

uint64_t fv_array_size(const fv_array* a);
/* Element width in bytes (1, 4 or 8). */
uint32_t fv_array_elem_bytes(const fv_array* a);
fv_status fv_array_read(const fv_array* a, void* host_out);
void fv_array_free(fv_array* a);

/* ---- Column (P/include/colog/column.hpp:26-64, P/src/column.cpp) -------- */

/* Column::build (P/src/column.cpp:45-52): raw + (value,id)-sorted index +
 * unique value -> (start,count) map, built by the sm_100a onesweep radix
 * sort. `raw` is host memory. */
fv_status fv_column_build(fv_ctx* ctx, const uint32_t* raw, uint64_t n, fv_column** out);
void fv_column_free(fv_column* col);
uint64_t fv_column_size(const fv_column* col);
uint64_t fv_column_unique_count(const fv_column* col);
/* Copy raw values and/or sorted_idx to host (either pointer may be NULL). */
fv_status fv_column_read(const fv_column* col, uint32_t* raw, uint32_t* sorted_idx);
/* unique_idx as three arrays ordered by key. */
fv_status fv_column_read_unique(const fv_column* col, uint32_t* keys, uint32_t* starts,
                                uint32_t* counts);
/* Column::probe (column.hpp:46-50). *found = 0 when v does not occur. */
fv_status fv_column_probe(const fv_column* col, uint32_t v, uint32_t* start, uint32_t* count,
                          int* found);
/* Batched probe of host values on device; found[i] in {0,1}. */
fv_status fv_column_probe_many(const fv_column* col, const uint32_t* values, uint64_t n,
                               uint32_t* starts, uint32_t* counts, uint8_t* found);
/* Column::gather (column.cpp:54-63): out[i] = raw[ids[i]]; any id >= size
 * fails with FV_ERR_RANGE before anything is written. Host in/out. */
fv_status fv_column_gather(const fv_column* col, const uint32_t* ids, uint64_t n,
                           uint32_t* out);
/* Column::append_and_reindex (column.cpp:65-72). */
fv_status fv_column_append_and_reindex(const fv_column* col, const uint32_t* values, uint64_t n,
                                       fv_column** out);
/* build_index (column.cpp:17-43) into caller buffers: sorted_idx[n];
 * keys/starts/counts sized n (only *n_unique entries written). */
fv_status fv_build_index(fv_ctx* ctx, const uint32_t* raw, uint64_t n, uint32_t* sorted_idx,
                         uint32_t* keys, uint32_t* starts, uint32_t* counts,
                         uint64_t* n_unique);

/* ---- Version (P/include/colog/relation.hpp:17-57, P/src/relation.cpp) ---- */

/* Version::from_columns (relation.cpp:19-27): cols[j] are host arrays of n. */
fv_status fv_version_from_columns(fv_ctx* ctx, uint32_t arity, const uint32_t* const* cols,
                                  uint64_t n, fv_version** out);
/* Version::decompose (relation.cpp:8-17): rows is row-major n x arity. */
fv_status fv_version_decompose(fv_ctx* ctx, uint32_t arity, const uint32_t* rows, uint64_t n,
                               fv_version** out);
/* Version(arity): empty. */
fv_status fv_version_empty(fv_ctx* ctx, uint32_t arity, fv_version** out);
void fv_version_free(fv_version* v);
uint32_t fv_version_arity(const fv_version* v);
uint64_t fv_version_rows(const fv_version* v);
/* Borrowed; valid while v lives. */
const fv_column* fv_version_col(const fv_version* v, uint32_t j);
/* Version::reconstruct (relation.cpp:35-39): row-major rows in id order. */
fv_status fv_version_reconstruct(const fv_version* v, uint32_t* rows_out);
/* Version::append (relation.cpp:41-48). */
fv_status fv_version_append(const fv_version* v, const fv_version* extra, fv_version** out);
/* dedup_rows (relation.cpp:71-89): first-occurrence order, dense ids. */
fv_status fv_dedup_rows(const fv_version* v, fv_version** out);
/* has_duplicate_rows (relation.cpp:91-100). */
fv_status fv_has_duplicate_rows(const fv_version* v, int* out);

/* ---- Relation (relation.hpp:60-75) -------------------------------------- */

fv_status fv_relation_create(fv_ctx* ctx, const char* name, uint32_t arity, fv_relation** out);
void fv_relation_free(fv_relation* r);
/* Borrowed views of the three versions. */
const fv_version* fv_relation_full(const fv_relation* r);
const fv_version* fv_relation_delta(const fv_relation* r);
const fv_version* fv_relation_new(const fv_relation* r);
/* Replace FULL (takes ownership of v). */
fv_status fv_relation_set_full(fv_relation* r, fv_version* v);
/* Relation::merge_delta (relation.cpp:102-108): full <- full ++ delta,
 * delta <- deduped_delta (ownership taken), new <- empty. */
fv_status fv_relation_merge_delta(fv_relation* r, fv_version* deduped_delta);

/* ---- RA kernels (P/include/colog/kernels.hpp, P/src/kernels.cpp) -------- */

/* select_eq (kernels.cpp:38-46): ascending ids whose value equals v. */
fv_status fv_select_eq(const fv_column* col, uint32_t v, fv_array** ids);
/* project (kernels.cpp:48-57): host ids and column map. */
fv_status fv_project(const fv_version* v, const uint32_t* ids, uint64_t n_ids,
                     const uint32_t* col_map, uint32_t n_cols, fv_version** out);
/* join_probe_phase (kernels.cpp:59-81) over host probe values. */
fv_status fv_join_probe_phase(fv_ctx* ctx, const uint32_t* probe_values, uint64_t n,
                              const fv_column* build, fv_match** out);
/* A MatchVector given as host arrays (ranges + matched probe positions), for
 * callers that hold one across the phases (join_total_size, join_offsets,
 * join_write_phase take `const MatchVector&`, P/include/colog/kernels.hpp:82-96). */
fv_status fv_match_create(fv_ctx* ctx, const uint32_t* starts, const uint32_t* counts,
                          const uint32_t* matched, uint64_t n, fv_match** out);
void fv_match_free(fv_match* m);
uint64_t fv_match_size(const fv_match* m);
/* ranges (start,count) and matched probe positions, host out. */
fv_status fv_match_read(const fv_match* m, uint32_t* starts, uint32_t* counts,
                        uint32_t* matched);
/* join_total_size (kernels.cpp:83-92). */
fv_status fv_join_total_size(const fv_match* m, uint64_t* total);
/* join_offsets (kernels.cpp:94-102): exclusive scan, host out[size]. */
fv_status fv_join_offsets(const fv_match* m, uint64_t* offsets);
/* join_write_phase (kernels.cpp:104-123): (probe id, build id) pairs in the
 * reference's output order. */
fv_status fv_join_write_phase(const fv_match* m, const fv_column* build, fv_array** a_ids,
                              fv_array** b_ids);
/* column_join (kernels.cpp:125-135) over host probe values. */
fv_status fv_column_join(fv_ctx* ctx, const uint32_t* probe_values, uint64_t n,
                         const fv_column* build, fv_array** a_ids, fv_array** b_ids);
/* filter_pairs_eq, Column overload (kernels.cpp:137-150); host pairs. */
fv_status fv_filter_pairs_eq(fv_ctx* ctx, const uint32_t* a_ids, const uint32_t* b_ids,
                             uint64_t n, const fv_column* col_a, const fv_column* col_b,
                             fv_array** out_a, fv_array** out_b);
/* filter_neq (kernels.cpp:167-178). */
fv_status fv_filter_neq(const fv_version* v, uint32_t col_i, uint32_t col_j, fv_array** ids);
/* deduplicate (kernels.cpp:210-255): u8 flags, 1 = row of NEW is in FULL. */
fv_status fv_deduplicate(const fv_version* new_v, const fv_version* full, fv_array** flags);
/* difference (kernels.cpp:257-268): host flags of size rows(new_v). */
fv_status fv_difference(const fv_version* new_v, const uint8_t* flags, uint64_t n,
                        fv_version** out);
/* union_concat (kernels.cpp:270-272). */
fv_status fv_union_concat(const fv_version* full, const fv_version* delta, fv_version** out);

/* ---- Plan IR (P/include/colog/compiler.hpp:14-53) ----------------------- */

typedef struct fv_colref {
    uint32_t source; /* body atom index */
    uint32_t col;    /* column of that atom */
} fv_colref;

typedef struct fv_plan_source {
    const char* relation;
    uint32_t arity;
    uint32_t n_const_selects;
    const uint32_t* const_select_cols; /* [n_const_selects] */
    const uint32_t* const_select_vals; /* [n_const_selects] */
    uint32_t n_self_eqs;
    const uint32_t* self_eq_pairs; /* [2 * n_self_eqs]: (first col, repeated col) */
} fv_plan_source;

typedef struct fv_plan_join {
    uint32_t right_source; /* index into sources, >= 1; joins[k] attaches k+1 */
    fv_colref left;        /* probe column in the accumulated intermediate */
    uint32_t right_col;    /* hash column of the right atom */
    uint32_t n_residual_eq;
    const fv_colref* residual_left;      /* [n_residual_eq] */
    const uint32_t* residual_right_col;  /* [n_residual_eq] */
} fv_plan_join;

typedef struct fv_plan {
    const char* head_relation;
    uint32_t head_arity;
    uint32_t n_sources;
    const fv_plan_source* sources;
    uint32_t n_joins;
    const fv_plan_join* joins;
    uint32_t n_output_cols; /* head columns first, then guard-only columns */
    const fv_colref* output_cols;
    uint32_t n_guards;
    const uint32_t* guard_neq_pairs; /* [2 * n_guards] slots into output_cols */
} fv_plan;

typedef struct fv_relation_decl {
    const char* name;
    uint32_t arity;
} fv_relation_decl;

/* EDB facts for one relation as host SoA columns (cols[j][i]). */
typedef struct fv_facts {
    const char* relation;
    uint32_t arity;
    uint64_t n_rows;
    const uint32_t* const* cols;
} fv_facts;

/* ---- Frontend (P/src/parser.cpp, P/src/compiler.cpp, P/src/io.cpp) ------ */

/* parse_program (parser.cpp:344-348) + resolve_strings (io.cpp:126-140).
 * On FV_ERR_PLAN the "line:col: message" diagnostic is in diag (and
 * fv_global_error()). */
fv_status fv_program_parse(const char* text, fv_program** out, char* diag, size_t diag_cap);
void fv_program_free(fv_program* p);
/* validate_program (parser.cpp:375-442): newline-separated "line:col: msg"
 * diagnostics; *n_diags = 0 means accepted. */
fv_status fv_program_validate(const fv_program* p, char* diags, size_t cap, uint32_t* n_diags);
/* print_program (parser.cpp:350-373). *len receives the full length. */
fv_status fv_program_print(const fv_program* p, char* buf, size_t cap, size_t* len);
uint32_t fv_program_num_relations(const fv_program* p);
fv_status fv_program_relation(const fv_program* p, uint32_t i, fv_relation_decl* out);
uint32_t fv_program_num_rules(const fv_program* p);
/* compile_rule (compiler.cpp:19-96): borrowed plan valid while p lives. */
fv_status fv_program_plan(const fv_program* p, uint32_t rule, const fv_plan** out);
/* Dictionary of the program (io.hpp/dictionary.hpp): encode adds, lookup
 * fails with FV_ERR_RANGE when absent. */
fv_status fv_program_encode(fv_program* p, const char* s, uint32_t* out);
uint64_t fv_program_dictionary_size(const fv_program* p);

/* ---- Engine (P/include/colog/engine.hpp, P/src/engine.cpp) -------------- */

/* evaluate (engine.cpp:222-239) over explicit declarations and compiled
 * plans: seed (FULL = DELTA = dedup(EDB)), Jacobi semi-naive iterations with
 * one dedup+merge per head relation, EDB-only variants in iteration 0 only.
 * facts are host SoA; several blocks for one relation are concatenated. */
fv_status fv_evaluate(fv_ctx* ctx, const fv_relation_decl* decls, uint32_t n_decls,
                      const fv_plan* plans, uint32_t n_plans, const fv_facts* facts,
                      uint32_t n_facts, fv_state** out);
/* evaluate a parsed program: program facts plus the given blocks. */
fv_status fv_evaluate_program(fv_ctx* ctx, const fv_program* p, const fv_facts* facts,
                              uint32_t n_facts, fv_state** out);
/* EDB resident in HBM: upload once (unsorted, duplicates allowed; seed
 * dedups), evaluate many times without host->device traffic. */
typedef struct fv_edb fv_edb;
fv_status fv_edb_upload(fv_ctx* ctx, const fv_relation_decl* decls, uint32_t n_decls,
                        const fv_facts* facts, uint32_t n_facts, fv_edb** out);
void fv_edb_free(fv_edb* e);
fv_status fv_evaluate_program_edb(fv_ctx* ctx, const fv_program* p, const fv_edb* edb,
                                  fv_state** out);
/* ---- Partitioned (multi-GPU) evaluation, SURVEY.md §8e -------------------
 * IDB relations are hash-partitioned by a home column chosen from the
 * recursive rules (the column a rule carries from its DELTA atom to the head;
 * col 0 otherwise), plus copies on other probed columns; EDB relations are
 * replicated. Derivations whose rows are already at their owner (right-linear
 * TC: all of them) stay local; the others route head rows to
 * owner(hash(home col)) with one all-to-all per head per iteration. New Δ rows
 * are forwarded to the other copies, |Δ| (termination) and the stats are
 * all-reduced. Every rank passes the full EDB. States hold the rank's home
 * partition; stats are global. */
fv_status fv_nccl_unique_id(void* out128);
/* One process per GPU: later evaluations on ctx run partitioned over NCCL. */
fv_status fv_ctx_set_nccl(fv_ctx* ctx, int rank, int world, const void* id128);
/* `world` virtual ranks as threads on ctx's GPU with an in-process
 * transport: the same partitioned code path on one device. states_out
 * receives `world` states (free each). */
fv_status fv_evaluate_program_sharded(fv_ctx* ctx, const fv_program* p, const fv_facts* facts,
                                      uint32_t n_facts, uint32_t world, fv_state** states_out);
fv_status fv_state_partition(const fv_state* s, int* rank, int* world);
/* The static partitioning decisions for a program as JSON (host only):
 * {"relations": {name: {"idb": bool, "home": col, "keyset": [cols]}}, "rules":
 * [{"src_copy": [...], "shuffle": [...], "replicated_out": bool, "local_out":
 * bool}]}. *len = full length. */
fv_status fv_program_partition_plan(const fv_program* p, char* buf, size_t cap, size_t* len);
/* owner(v) = floor(hash32(v) * world / 2^32): the rank owning value v. */
uint32_t fv_owner(uint32_t v, uint32_t world);
void fv_state_free(fv_state* s);
/* EvaluationState::iterations (includes the final empty iteration). */
uint64_t fv_state_iterations(const fv_state* s);
/* Device time of seed + fixpoint in milliseconds (CUDA events). */
double fv_state_elapsed_ms(const fv_state* s);
uint64_t fv_state_num_relations(const fv_state* s);
/* Relations in std::map (name) order, like EvaluationState::relations. */
fv_status fv_state_relation(const fv_state* s, uint64_t i, const char** name, uint32_t* arity,
                            uint64_t* rows);
/* IterationStats x RelationStats (engine.hpp:35-46), flattened. */
uint64_t fv_state_num_stats(const fv_state* s);
fv_status fv_state_stat(const fv_state* s, uint64_t i, uint64_t* iteration, const char** rel,
                        uint64_t* delta_rows, uint64_t* full_rows, uint64_t* merges,
                        double* elapsed_ms);
/* FULL of a relation as lexicographically sorted row-major rows
 * (the set dump_relation writes, P/src/io.cpp:90-117). */
fv_status fv_state_dump_sorted(const fv_state* s, const char* rel, uint32_t* rows_out);
/* Order-independent 64-bit fingerprint of FULL computed on device:
 * sum over rows of splitmix64(pack(row)) (mod 2^64). */
fv_status fv_state_fingerprint(const fv_state* s, const char* rel, uint64_t* out);

/* ---- Runner (P/include/colog/runner.hpp, P/src/runner.cpp) -------------- */

/* colog::run: parse, validate, load <facts_dir>/<rel>.tsv, evaluate, print
 * the reference's stats/summary lines, dump the comma-separated relations
 * as sorted TSV into out_dir. Returns the process exit code (0 ok). out and
 * err receive malloc'd text (free with fv_free). */
int fv_run(int device, const char* program_path, const char* facts_dir, const char* out_dir,
           int print_stats, const char* dump_list, char** out, char** err);
void fv_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* FVLOG_H */

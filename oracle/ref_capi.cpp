// TEST INFRASTRUCTURE — never the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libcolog_ref.so)
// so the Python test-suite can run the real reference operators and engine on
// the same inputs as the CUDA path and as the oracle restatement
// (oracle/colog_oracle.c). Used only by tests/ and tests/golden/make_golden.py.
//
// Every function returns 0 on success and a negative code when the reference
// threw (the message is available from ref_last_error()). Output arrays are
// malloc'd here and released with ref_free().
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "colog/column.hpp"
#include "colog/engine.hpp"
#include "colog/io.hpp"
#include "colog/kernels.hpp"
#include "colog/oracle.hpp"
#include "colog/parser.hpp"
#include "colog/relation.hpp"

using namespace colog;

namespace {

thread_local std::string g_err;

const Executor& exec() {
    static Executor e;
    return e;
}

template <typename T>
T* dup_array(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

Version make_version(const uint32_t* cols_flat, uint64_t n, uint32_t arity) {
    std::vector<std::vector<Value>> cols(arity);
    for (uint32_t j = 0; j < arity; ++j) cols[j].assign(cols_flat + j * n, cols_flat + (j + 1) * n);
    return Version::from_columns(std::move(cols), exec());
}

uint32_t* version_cols(const Version& v) {
    std::vector<uint32_t> flat;
    flat.reserve(v.rows() * v.arity());
    for (std::size_t j = 0; j < v.arity(); ++j)
        flat.insert(flat.end(), v.col(j).raw().begin(), v.col(j).raw().end());
    return dup_array(flat);
}

#define REF_TRY try {
#define REF_CATCH                     \
    }                                 \
    catch (const std::exception& e) { \
        g_err = e.what();             \
        return -1;                    \
    }                                 \
    return 0;

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// build_index (P/src/column.cpp:17-43): sorted_idx plus the unique map as
// three arrays sorted by key.
int ref_build_index(const uint32_t* raw, uint64_t n, uint32_t** sorted_idx, uint32_t** keys,
                    uint32_t** starts, uint32_t** counts, uint64_t* n_unique) {
    REF_TRY
    auto [sorted, unique] = build_index(std::span<const Value>(raw, n), exec());
    std::map<Value, MatchRange> ordered(unique.begin(), unique.end());
    std::vector<uint32_t> k, s, c;
    for (auto& [key, r] : ordered) {
        k.push_back(key);
        s.push_back(r.start);
        c.push_back(r.count);
    }
    *sorted_idx = dup_array(sorted);
    *keys = dup_array(k);
    *starts = dup_array(s);
    *counts = dup_array(c);
    *n_unique = k.size();
    REF_CATCH
}

// column_join over a probe value array (P/src/kernels.cpp:125-131), pairs in
// the reference's output order.
int ref_column_join(const uint32_t* probe, uint64_t np, const uint32_t* build, uint64_t nb,
                    uint32_t** a_ids, uint32_t** b_ids, uint64_t* n_out) {
    REF_TRY
    Column b = Column::build(std::vector<Value>(build, build + nb), exec());
    IdPairSet p = column_join(std::span<const Value>(probe, np), b, exec());
    *a_ids = dup_array(p.a_ids);
    *b_ids = dup_array(p.b_ids);
    *n_out = p.size();
    REF_CATCH
}

// join_probe_phase (P/src/kernels.cpp:59-81) + join_offsets (:94-102).
int ref_join_probe(const uint32_t* probe, uint64_t np, const uint32_t* build, uint64_t nb,
                   uint32_t** starts, uint32_t** counts, uint32_t** matched, uint64_t** offsets,
                   uint64_t* n_match, uint64_t* total) {
    REF_TRY
    Column b = Column::build(std::vector<Value>(build, build + nb), exec());
    MatchVector mv = join_probe_phase(std::span<const Value>(probe, np), b, exec());
    std::vector<uint32_t> s, c;
    for (auto& r : mv.ranges) {
        s.push_back(r.start);
        c.push_back(r.count);
    }
    *starts = dup_array(s);
    *counts = dup_array(c);
    *matched = dup_array(mv.matched);
    *offsets = dup_array(join_offsets(mv));
    *n_match = mv.size();
    *total = join_total_size(mv, exec());
    REF_CATCH
}

// dedup_rows (P/src/relation.cpp:71-89): first-occurrence order.
int ref_dedup_rows(const uint32_t* cols, uint64_t n, uint32_t arity, uint32_t** out,
                   uint64_t* n_out) {
    REF_TRY
    Version v = dedup_rows(make_version(cols, n, arity), exec());
    *out = version_cols(v);
    *n_out = v.rows();
    REF_CATCH
}

// deduplicate (P/src/kernels.cpp:210-255): flags[i] = row i of NEW is in FULL.
int ref_deduplicate(const uint32_t* new_cols, uint64_t n_new, const uint32_t* full_cols,
                    uint64_t n_full, uint32_t arity, uint8_t** flags) {
    REF_TRY
    DupBitmap bm = deduplicate(make_version(new_cols, n_new, arity),
                               make_version(full_cols, n_full, arity), exec());
    *flags = dup_array(bm.flags);
    REF_CATCH
}

// filter_neq (P/src/kernels.cpp:167-178).
int ref_filter_neq(const uint32_t* cols, uint64_t n, uint32_t arity, uint32_t ci, uint32_t cj,
                   uint32_t** ids, uint64_t* n_out) {
    REF_TRY
    auto v = filter_neq(make_version(cols, n, arity), ci, cj, exec());
    *ids = dup_array(v);
    *n_out = v.size();
    REF_CATCH
}

// filter_pairs_eq, Column overload (P/src/kernels.cpp:137-150).
int ref_filter_pairs_eq(const uint32_t* a_ids, const uint32_t* b_ids, uint64_t np,
                        const uint32_t* col_a, uint64_t na, const uint32_t* col_b, uint64_t nb,
                        uint32_t** oa, uint32_t** ob, uint64_t* n_out) {
    REF_TRY
    IdPairSet p{{a_ids, a_ids + np}, {b_ids, b_ids + np}};
    Column ca = Column::build(std::vector<Value>(col_a, col_a + na), exec());
    Column cb = Column::build(std::vector<Value>(col_b, col_b + nb), exec());
    IdPairSet r = filter_pairs_eq(p, ca, cb, exec());
    *oa = dup_array(r.a_ids);
    *ob = dup_array(r.b_ids);
    *n_out = r.size();
    REF_CATCH
}

// Evaluate a program text (facts in text and/or passed as SoA blocks) to
// fixpoint with colog::evaluate (P/src/engine.cpp:222-239). Returns the
// per-iteration stats as "iter rel delta full merges" lines and every
// relation's sorted dump in the reference's TSV format, "#rel name" headers
// between relations.
int ref_evaluate(const char* program_text, uint32_t n_blocks, const char** names,
                 const uint32_t* const* cols, const uint64_t* n_rows, char** report) {
    REF_TRY
    Program prog = parse_program(program_text);
    Dictionary dict;
    resolve_strings(prog, dict);
    FactMap facts = program_facts(prog);
    for (uint32_t b = 0; b < n_blocks; ++b) {
        const RelationDecl* decl = prog.find_relation(names[b]);
        if (!decl) continue;
        auto& rows = facts[names[b]];
        for (uint64_t i = 0; i < n_rows[b]; ++i) {
            Row r(decl->arity);
            for (std::size_t j = 0; j < decl->arity; ++j) r[j] = cols[b][j * n_rows[b] + i];
            rows.push_back(std::move(r));
        }
    }
    EvaluationState st = evaluate(prog, facts, exec());
    std::ostringstream os;
    os << "iterations " << st.iterations << "\n";
    for (const auto& it : st.stats)
        for (const auto& rs : it.relations)
            os << "stat " << it.index << " " << rs.relation << " " << rs.delta_rows << " "
               << rs.full_rows << " " << rs.merges << "\n";
    for (const auto& [name, rel] : st.relations) {
        os << "#rel " << name << " " << rel.arity << " " << rel.full.rows() << "\n";
        dump_relation(rel.full, nullptr, os);
    }
    std::string s = os.str();
    *report = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*report, s.c_str(), s.size() + 1);
    REF_CATCH
}

// Naive least-model evaluation (P/src/oracle.cpp:72-89), same report format
// without stats.
int ref_naive_evaluate(const char* program_text, char** report) {
    REF_TRY
    Program prog = parse_program(program_text);
    Dictionary dict;
    resolve_strings(prog, dict);
    auto rows = oracle::naive_evaluate(prog, program_facts(prog));
    std::ostringstream os;
    for (const auto& [name, set] : rows) {
        os << "#rel " << name << " " << (set.empty() ? 0 : set.begin()->size()) << " "
           << set.size() << "\n";
        for (const Row& r : set) {
            for (std::size_t j = 0; j < r.size(); ++j) os << (j ? "\t" : "") << r[j];
            os << "\n";
        }
    }
    std::string s = os.str();
    *report = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*report, s.c_str(), s.size() + 1);
    REF_CATCH
}

} // extern "C"

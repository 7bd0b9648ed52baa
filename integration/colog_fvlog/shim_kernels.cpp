// The relational-algebra kernels (P/include/colog/kernels.hpp) on fvlog:
// Algorithm 1's probe / total / offsets / write phases, the residual and
// guard filters, Algorithm 2 (deduplicate), difference and union.
#include <numeric>

#include "colog/kernels.hpp"
#include "shim.hpp"

namespace colog {

using fvshim::ArrayH;
using fvshim::check;
using fvshim::ColumnH;
using fvshim::ctx;
using fvshim::VersionH;

namespace {

// A host MatchVector as a device fv_match.
struct MatchH {
    fv_match* p = nullptr;
    explicit MatchH(const MatchVector& mv) {
        std::vector<std::uint32_t> starts(mv.size()), counts(mv.size());
        for (std::size_t k = 0; k < mv.size(); ++k) {
            starts[k] = mv.ranges[k].start;
            counts[k] = mv.ranges[k].count;
        }
        check(fv_match_create(ctx(), starts.data(), counts.data(), mv.matched.data(), mv.size(), &p),
              "fv_match_create");
    }
    MatchH(const MatchH&) = delete;
    MatchH& operator=(const MatchH&) = delete;
    ~MatchH() { fv_match_free(p); }
};

IdPairSet read_pairs(const ArrayH& a, const ArrayH& b) {
    IdPairSet out;
    out.a_ids = a.read<TupleId>();
    out.b_ids = b.read<TupleId>();
    return out;
}

}  // namespace

std::vector<TupleId> select_eq(const Column& col, Value v) {
    ColumnH c(col.raw());
    ArrayH ids;
    check(fv_select_eq(c.p, v, &ids.p), "select_eq");
    return ids.read<TupleId>();
}

Version project(const Version& ver, std::span<const TupleId> ids, std::span<const std::size_t> col_map,
                const Executor&) {
    std::vector<std::uint32_t> cm(col_map.size());
    for (std::size_t k = 0; k < col_map.size(); ++k) {
        if (col_map[k] >= ver.arity()) throw std::out_of_range("project: column index past arity");
        cm[k] = static_cast<std::uint32_t>(col_map[k]);
    }
    VersionH v(ver), out;
    check(fv_project(v.p, ids.data(), ids.size(), cm.data(), static_cast<std::uint32_t>(cm.size()), &out.p),
          "project");
    return fvshim::download(out.p);
}

MatchVector join_probe_phase(std::span<const Value> probe_values, const Column& build, const Executor&) {
    ColumnH b(build.raw());
    fv_match* m = nullptr;
    check(fv_join_probe_phase(ctx(), probe_values.data(), probe_values.size(), b.p, &m), "join_probe_phase");
    const std::uint64_t k = fv_match_size(m);
    std::vector<std::uint32_t> starts(k), counts(k);
    MatchVector mv;
    mv.matched.resize(k);
    const fv_status s = k ? fv_match_read(m, starts.data(), counts.data(), mv.matched.data()) : FV_OK;
    fv_match_free(m);
    check(s, "join_probe_phase");
    mv.ranges.resize(k);
    for (std::uint64_t i = 0; i < k; ++i) mv.ranges[i] = MatchRange{starts[i], counts[i]};
    return mv;
}

std::uint64_t join_total_size(const MatchVector& mv, const Executor&) {
    MatchH m(mv);
    std::uint64_t total = 0;
    check(fv_join_total_size(m.p, &total), "join_total_size");
    return total;
}

std::vector<std::uint64_t> join_offsets(const MatchVector& mv) {
    MatchH m(mv);
    std::vector<std::uint64_t> off(mv.size());
    if (!off.empty()) check(fv_join_offsets(m.p, off.data()), "join_offsets");
    return off;
}

IdPairSet join_write_phase(const MatchVector& mv, std::span<const std::uint64_t> offsets, std::uint64_t total_size,
                           const Column& build, const Executor&) {
    // The device recomputes the offsets of mv (identical by construction:
    // the exclusive scan of the range counts) and sizes the output from them.
    if (offsets.size() != mv.size()) throw std::invalid_argument("join_write_phase: offsets size mismatch");
    MatchH m(mv);
    ColumnH b(build.raw());
    ArrayH a_ids, b_ids;
    check(fv_join_write_phase(m.p, b.p, &a_ids.p, &b_ids.p), "join_write_phase");
    if (fv_array_size(a_ids.p) != total_size) throw std::invalid_argument("join_write_phase: total size mismatch");
    return read_pairs(a_ids, b_ids);
}

IdPairSet column_join(std::span<const Value> probe_values, const Column& build, const Executor&) {
    ColumnH b(build.raw());
    ArrayH a_ids, b_ids;
    check(fv_column_join(ctx(), probe_values.data(), probe_values.size(), b.p, &a_ids.p, &b_ids.p), "column_join");
    return read_pairs(a_ids, b_ids);
}

IdPairSet column_join(const Column& probe, const Column& build, const Executor& exec) {
    return column_join(std::span<const Value>(probe.raw()), build, exec);
}

IdPairSet filter_pairs_eq(const IdPairSet& pairs, const Column& col_a, const Column& col_b, const Executor&) {
    ColumnH a(col_a.raw()), b(col_b.raw());
    ArrayH oa, ob;
    check(fv_filter_pairs_eq(ctx(), pairs.a_ids.data(), pairs.b_ids.data(), pairs.size(), a.p, b.p, &oa.p, &ob.p),
          "filter_pairs_eq");
    return read_pairs(oa, ob);
}

IdPairSet filter_pairs_eq(const IdPairSet& pairs, std::span<const Value> left_values, const Column& col_b,
                          const Executor&) {
    // left_values is aligned with the pairs by position (kernels.hpp:102-105):
    // filter the positions k against a column over left_values, then map the
    // kept positions back to the caller's a ids.
    if (left_values.size() < pairs.size()) throw std::out_of_range("filter_pairs_eq: left values shorter than pairs");
    std::vector<TupleId> pos(pairs.size());
    std::iota(pos.begin(), pos.end(), TupleId{0});
    ColumnH a(std::vector<Value>(left_values.begin(), left_values.begin() + pairs.size())), b(col_b.raw());
    ArrayH ok, ob;
    check(fv_filter_pairs_eq(ctx(), pos.data(), pairs.b_ids.data(), pairs.size(), a.p, b.p, &ok.p, &ob.p),
          "filter_pairs_eq");
    IdPairSet out;
    const std::vector<TupleId> kept = ok.read<TupleId>();
    out.b_ids = ob.read<TupleId>();
    out.a_ids.resize(kept.size());
    for (std::size_t k = 0; k < kept.size(); ++k) out.a_ids[k] = pairs.a_ids[kept[k]];
    return out;
}

std::vector<TupleId> filter_neq(const Version& ver, std::size_t col_i, std::size_t col_j, const Executor&) {
    if (col_i >= ver.arity() || col_j >= ver.arity()) throw std::out_of_range("filter_neq: column index past arity");
    VersionH v(ver);
    ArrayH ids;
    check(fv_filter_neq(v.p, static_cast<std::uint32_t>(col_i), static_cast<std::uint32_t>(col_j), &ids.p),
          "filter_neq");
    return ids.read<TupleId>();
}

DupBitmap deduplicate(const Version& new_ver, const Version& full, const Executor&) {
    VersionH n(new_ver), f(full);
    ArrayH flags;
    check(fv_deduplicate(n.p, f.p, &flags.p), "deduplicate");
    DupBitmap out;
    out.flags = flags.read<std::uint8_t>();
    return out;
}

Version difference(const Version& new_ver, const DupBitmap& flags, const Executor&) {
    VersionH n(new_ver), out;
    check(fv_difference(n.p, flags.flags.data(), flags.size(), &out.p), "difference");
    return fvshim::download(out.p);
}

Version union_concat(const Version& full, const Version& delta, const Executor&) {
    VersionH f(full), d(delta), out;
    check(fv_union_concat(f.p, d.p, &out.p), "union_concat");
    return fvshim::download(out.p);
}

}  // namespace colog

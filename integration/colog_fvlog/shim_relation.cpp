// colog::Version / dedup_rows / has_duplicate_rows / Relation::merge_delta
// (P/include/colog/relation.hpp) on fvlog.
#include "colog/relation.hpp"
#include "shim.hpp"

namespace colog {

namespace fvshim {

VersionH::VersionH(const Version& v) {
    std::vector<const std::uint32_t*> cols(v.arity());
    for (std::size_t j = 0; j < v.arity(); ++j) cols[j] = v.col(j).raw().data();
    check(fv_version_from_columns(ctx(), static_cast<std::uint32_t>(v.arity()), cols.data(), v.rows(), &p),
          "fv_version_from_columns");
}

std::vector<std::vector<Value>> download_columns(const fv_version* v) {
    const std::uint32_t a = fv_version_arity(v);
    const std::uint64_t n = fv_version_rows(v);
    std::vector<std::vector<Value>> cols(a, std::vector<Value>(n));
    for (std::uint32_t j = 0; j < a; ++j)
        if (n) check(fv_column_read(fv_version_col(v, j), cols[j].data(), nullptr), "fv_column_read");
    return cols;
}

Version download(const fv_version* v) {
    const std::uint32_t a = fv_version_arity(v);
    if (fv_version_rows(v) == 0) return Version(a);
    return Version::from_columns(download_columns(v), Executor(1));
}

}  // namespace fvshim

using fvshim::check;
using fvshim::ctx;

Version Version::decompose(std::span<const Row> rows, std::size_t arity, const Executor& exec) {
    // Row-major marshalling of the caller's rows; the split into columns and
    // the index builds run on the device (fv_version_decompose).
    std::vector<std::uint32_t> flat;
    flat.reserve(rows.size() * arity);
    for (const Row& r : rows) {
        if (r.size() != arity) throw std::invalid_argument("decompose: row arity mismatch");
        flat.insert(flat.end(), r.begin(), r.end());
    }
    if (arity == 0) return Version(0);
    fvshim::VersionH d;
    check(fv_version_decompose(ctx(), static_cast<std::uint32_t>(arity), flat.data(), rows.size(), &d.p),
          "decompose");
    return from_columns(fvshim::download_columns(d.p), exec);
}

Version Version::from_columns(std::vector<std::vector<Value>> cols, const Executor& exec) {
    Version ver;
    ver.cols_.reserve(cols.size());
    for (std::size_t j = 1; j < cols.size(); ++j)
        if (cols[j].size() != cols[0].size()) throw std::invalid_argument("from_columns: column length mismatch");
    for (auto& c : cols) ver.cols_.push_back(Column::build(std::move(c), exec));
    return ver;
}

Row Version::row(TupleId id) const {
    Row r(arity());
    for (std::size_t j = 0; j < arity(); ++j) r[j] = cols_[j].value_at(id);
    return r;
}

std::vector<Row> Version::reconstruct() const {
    // Interleaving happens on the device (fv_version_reconstruct).
    const std::size_t a = arity(), n = rows();
    std::vector<Row> out(n, Row(a));
    if (!n || !a) return out;
    fvshim::VersionH d(*this);
    std::vector<std::uint32_t> flat(n * a);
    check(fv_version_reconstruct(d.p, flat.data()), "reconstruct");
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < a; ++j) out[i][j] = flat[i * a + j];
    return out;
}

Version Version::append(const Version& extra, const Executor&) const {
    if (extra.arity() != arity()) throw std::invalid_argument("append: arity mismatch");
    fvshim::VersionH a(*this), b(extra), out;
    check(fv_version_append(a.p, b.p, &out.p), "append");
    return fvshim::download(out.p);
}

Version dedup_rows(const Version& ver, const Executor&) {
    fvshim::VersionH v(ver), out;
    check(fv_dedup_rows(v.p, &out.p), "dedup_rows");
    return fvshim::download(out.p);
}

bool has_duplicate_rows(const Version& ver, const Executor&) {
    fvshim::VersionH v(ver);
    int dup = 0;
    check(fv_has_duplicate_rows(v.p, &dup), "has_duplicate_rows");
    return dup != 0;
}

void Relation::merge_delta(Version deduped_delta, const Executor& exec) {
    if (deduped_delta.arity() != arity) throw std::invalid_argument("merge_delta: arity mismatch");
    full = full.append(deduped_delta, exec);
    delta = std::move(deduped_delta);
    new_rows = Version(arity);
}

}  // namespace colog

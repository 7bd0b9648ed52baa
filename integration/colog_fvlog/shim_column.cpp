// colog::Column / build_index / gather_volume (P/include/colog/column.hpp)
// on fvlog: the (value, id) order and the run map come from the sm_100a
// onesweep radix sort (fv_build_index), gathers from fv_column_gather.
#include <cstdlib>
#include <limits>

#include "colog/column.hpp"
#include "shim.hpp"

namespace colog {

namespace fvshim {

fv_ctx* ctx() {
    static fv_ctx* c = [] {
        const char* e = std::getenv("FVLOG_DEVICE");
        fv_ctx* out = nullptr;
        if (fv_ctx_create(e ? std::atoi(e) : 0, &out) != FV_OK)
            throw std::runtime_error(std::string("fvlog: no device context: ") + fv_global_error());
        return out;
    }();
    return c;
}

void check(fv_status s, const char* what) {
    if (s == FV_OK) return;
    const char* m = fv_last_error(ctx());
    std::string msg = std::string(what) + ": " + (m && *m ? m : fv_global_error());
    switch (s) {
        case FV_ERR_ARITY: throw std::invalid_argument(msg);
        case FV_ERR_RANGE: throw std::out_of_range(msg);
        case FV_ERR_LENGTH: throw std::length_error(msg);
        default: throw std::runtime_error(msg);
    }
}

ColumnH::ColumnH(const std::vector<Value>& raw) {
    check(fv_column_build(ctx(), raw.data(), raw.size(), &p), "fv_column_build");
}

}  // namespace fvshim

using fvshim::check;
using fvshim::ctx;

std::uint64_t gather_volume() { return fv_gather_volume(); }
void reset_gather_volume() { fv_reset_gather_volume(); }

std::pair<std::vector<TupleId>, UniqueIndex> build_index(std::span<const Value> raw, const Executor&) {
    if (raw.size() > std::numeric_limits<TupleId>::max())
        throw std::length_error("column exceeds 32-bit tuple id space");
    const std::size_t n = raw.size();
    std::vector<TupleId> sorted(n);
    std::vector<std::uint32_t> keys(n), starts(n), counts(n);
    std::uint64_t u = 0;
    check(fv_build_index(ctx(), raw.data(), n, sorted.data(), keys.data(), starts.data(), counts.data(), &u),
          "fv_build_index");
    UniqueIndex unique;
    unique.reserve(u);
    for (std::uint64_t k = 0; k < u; ++k) unique.emplace(keys[k], MatchRange{starts[k], counts[k]});
    return {std::move(sorted), std::move(unique)};
}

Column Column::build(std::vector<Value> raw, const Executor& exec) {
    Column col;
    auto [sorted, unique] = build_index(raw, exec);
    col.raw_ = std::move(raw);
    col.sorted_idx_ = std::move(sorted);
    col.unique_idx_ = std::move(unique);
    return col;
}

std::vector<Value> Column::gather(std::span<const TupleId> ids, const Executor&) const {
    fvshim::ColumnH c(raw_);
    std::vector<Value> out(ids.size());
    // Any id >= size fails with FV_ERR_RANGE (std::out_of_range) before a
    // value is written; the gather counter moves by ids.size() on success.
    check(fv_column_gather(c.p, ids.data(), ids.size(), out.data()), "gather");
    return out;
}

Column Column::append_and_reindex(std::span<const Value> new_values, const Executor&) const {
    fvshim::ColumnH c(raw_);
    fv_column* grown = nullptr;
    check(fv_column_append_and_reindex(c.p, new_values.data(), new_values.size(), &grown), "append_and_reindex");
    Column out;
    const std::uint64_t n = fv_column_size(grown), u = fv_column_unique_count(grown);
    out.raw_.resize(n);
    out.sorted_idx_.resize(n);
    std::vector<std::uint32_t> keys(u), starts(u), counts(u);
    fv_status s = fv_column_read(grown, out.raw_.data(), out.sorted_idx_.data());
    if (s == FV_OK && u) s = fv_column_read_unique(grown, keys.data(), starts.data(), counts.data());
    fv_column_free(grown);
    check(s, "append_and_reindex");
    out.unique_idx_.reserve(u);
    for (std::uint64_t k = 0; k < u; ++k) out.unique_idx_.emplace(keys[k], MatchRange{starts[k], counts[k]});
    return out;
}

}  // namespace colog

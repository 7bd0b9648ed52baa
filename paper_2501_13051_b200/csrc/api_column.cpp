// extern "C" boundary, column-store and operator half (include/fvlog.h).
// Every entry point is a thin host wrapper: host buffers in, one upload, the
// sm_100a operator, one download. No computation happens on the host.
#include <cstring>

#include "api_internal.h"
#include "transport.h"

fv_ctx::~fv_ctx() = default;

using fv::DBuf;
using fv::u32;
using fv::u64;
using fv::u8;

namespace fvapi {

namespace {
thread_local std::string g_error;
}

fv_status set_error(fv_ctx* ctx, fv_status s, const std::string& msg) {
    g_error = msg;
    if (ctx && ctx->c) ctx->c->last_error = msg;
    return s;
}

static void make_views(fv_version* w) {
    w->views.clear();
    for (auto& col : w->v->cols) {
        auto view = std::make_unique<fv_column>();
        view->ctx = w->ctx;
        view->col = col.get();
        w->views.push_back(std::move(view));
    }
}

fv_version* wrap_version(fv_ctx* ctx, std::unique_ptr<fv::Version> v) {
    auto* w = new fv_version();
    w->ctx = ctx;
    w->v = std::move(v);
    make_views(w);
    return w;
}

fv_array* wrap_array_u32(fv_ctx* ctx, DBuf<u32>&& b, u64 n) {
    auto* a = new fv_array();
    a->ctx = ctx;
    a->a.ctx = ctx->c;
    a->a.n = n;
    a->a.elem = 4;
    a->a.bytes = DBuf<u8>::adopt(ctx->c, reinterpret_cast<u8*>(b.release()), n * 4);
    return a;
}

static fv_array* wrap_array_u8(fv_ctx* ctx, DBuf<u8>&& b, u64 n) {
    auto* a = new fv_array();
    a->ctx = ctx;
    a->a.ctx = ctx->c;
    a->a.n = n;
    a->a.elem = 1;
    a->a.bytes = std::move(b);
    return a;
}

}  // namespace fvapi

using fvapi::wrap_version;

extern "C" {

int fv_abi_version(void) { return FVLOG_ABI_VERSION; }
const char* fv_global_error(void) { return fvapi::g_error.c_str(); }

fv_status fv_ctx_create(int device, fv_ctx** out) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(out, FV_ERR_INVALID, "fv_ctx_create: null out");
    auto* w = new fv_ctx();
    try {
        w->c = fv::ctx_new(device);
    } catch (...) {
        delete w;
        throw;
    }
    *out = w;
    FV_API_END
}

void fv_ctx_destroy(fv_ctx* ctx) {
    if (!ctx) return;
    if (ctx->c) ctx->c->tx = nullptr;
    ctx->tx.reset();
    fv::ctx_delete(ctx->c);
    delete ctx;
}

fv_status fv_nccl_unique_id(void* out128) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(out128, FV_ERR_INVALID, "fv_nccl_unique_id: null out");
    fv::nccl_unique_id(out128);
    FV_API_END
}

fv_status fv_ctx_set_nccl(fv_ctx* ctx, int rank, int world, const void* id128) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(ctx && id128 && world >= 1 && rank >= 0 && rank < world, FV_ERR_INVALID,
               "fv_ctx_set_nccl: bad argument");
    ctx->c->tx = nullptr;
    ctx->tx = fv::make_nccl_transport(ctx->c, rank, world, id128);
    ctx->c->tx = ctx->tx.get();
    FV_API_END
}

const char* fv_last_error(const fv_ctx* ctx) {
    return ctx && ctx->c ? ctx->c->last_error.c_str() : fvapi::g_error.c_str();
}

fv_status fv_ctx_synchronize(fv_ctx* ctx) {
    FV_API_BEGIN(ctx)
    ctx->c->sync();
    FV_API_END
}

uint64_t fv_ctx_kernel_launches(const fv_ctx* ctx) { return ctx ? ctx->c->launches : 0; }

uint64_t fv_ctx_host_syncs(const fv_ctx* ctx) { return ctx ? ctx->c->syncs : 0; }

fv_status fv_ctx_profile(fv_ctx* ctx, int enable) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(ctx, FV_ERR_INVALID, "fv_ctx_profile: null ctx");
    ctx->c->sync();
    if (enable) ctx->c->prof_agg.clear();
    ctx->c->prof = enable != 0;
    FV_API_END
}

fv_status fv_ctx_reserve(fv_ctx* ctx, uint64_t bytes) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(ctx, FV_ERR_INVALID, "fv_ctx_reserve: null ctx");
    ctx->c->reserve(bytes);
    FV_API_END
}

uint32_t fv_ctx_profile_count(const fv_ctx* ctx) {
    if (!ctx) return 0;
    ctx->c->sync();
    return static_cast<uint32_t>(ctx->c->prof_agg.size());
}

fv_status fv_ctx_profile_entry(const fv_ctx* ctx, uint32_t i, const char** name, uint64_t* launches, double* ms,
                               double* bytes) {
    FV_API_BEGIN(const_cast<fv_ctx*>(ctx))
    FV_REQUIRE(ctx, FV_ERR_INVALID, "fv_ctx_profile_entry: null ctx");
    ctx->c->sync();
    if (i >= ctx->c->prof_agg.size()) fv::fail(FV_ERR_RANGE, "profile entry out of range");
    const auto& [n, a] = ctx->c->prof_agg[i];
    if (name) *name = n.c_str();
    if (launches) *launches = a.launches;
    if (ms) *ms = a.ms;
    if (bytes) *bytes = a.bytes;
    FV_API_END
}
uint64_t fv_gather_volume(void) { return fv::gather_volume(); }
void fv_reset_gather_volume(void) { fv::reset_gather_volume(); }

// ---- arrays ------------------------------------------------------------------

uint64_t fv_array_size(const fv_array* a) { return a ? a->a.n : 0; }
uint32_t fv_array_elem_bytes(const fv_array* a) { return a ? a->a.elem : 0; }

fv_status fv_array_read(const fv_array* a, void* host_out) {
    FV_API_BEGIN(a ? a->ctx : nullptr)
    FV_REQUIRE(a, FV_ERR_INVALID, "fv_array_read: null array");
    a->a.bytes.download(static_cast<u8*>(host_out), a->a.n * a->a.elem);
    FV_API_END
}

void fv_array_free(fv_array* a) {
    if (!a) return;
    a->ctx->c->activate();
    delete a;
}

// ---- columns -------------------------------------------------------------------

fv_status fv_column_build(fv_ctx* ctx, const uint32_t* raw, uint64_t n, fv_column** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(out && (raw || n == 0), FV_ERR_INVALID, "fv_column_build: null argument");
    auto w = std::make_unique<fv_column>();
    w->ctx = ctx;
    w->owned = fv::column_build(ctx->c, fv::make_dbuf(ctx->c, raw, n), n);
    w->col = w->owned.get();
    ctx->c->sync();
    *out = w.release();
    FV_API_END
}

void fv_column_free(fv_column* col) {
    if (!col) return;
    col->ctx->c->activate();
    delete col;
}

uint64_t fv_column_size(const fv_column* col) { return col ? col->col->n : 0; }
uint64_t fv_column_unique_count(const fv_column* col) { return col ? col->col->n_unique : 0; }

fv_status fv_column_read(const fv_column* col, uint32_t* raw, uint32_t* sorted_idx) {
    FV_API_BEGIN(col ? col->ctx : nullptr)
    FV_REQUIRE(col, FV_ERR_INVALID, "fv_column_read: null column");
    if (raw) col->col->raw.download(raw, col->col->n);
    if (sorted_idx) col->col->sorted_idx.download(sorted_idx, col->col->n);
    FV_API_END
}

fv_status fv_column_read_unique(const fv_column* col, uint32_t* keys, uint32_t* starts,
                                uint32_t* counts) {
    FV_API_BEGIN(col ? col->ctx : nullptr)
    FV_REQUIRE(col, FV_ERR_INVALID, "fv_column_read_unique: null column");
    const u64 nu = col->col->n_unique;
    if (keys) col->col->ukeys.download(keys, nu);
    if (starts) col->col->ustart.download(starts, nu);
    if (counts) col->col->ucount.download(counts, nu);
    FV_API_END
}

fv_status fv_column_probe_many(const fv_column* col, const uint32_t* values, uint64_t n,
                               uint32_t* starts, uint32_t* counts, uint8_t* found) {
    FV_API_BEGIN(col ? col->ctx : nullptr)
    FV_REQUIRE(col && (values || n == 0), FV_ERR_INVALID, "fv_column_probe_many: null argument");
    fv::Ctx* c = col->ctx->c;
    DBuf<u32> dv = fv::make_dbuf(c, values, n);
    DBuf<u32> ds(c, n), dc(c, n);
    fv::column_probe_device(c, *col->col, dv.get(), n, ds.get(), dc.get());
    std::vector<u32> hs(n), hc(n);
    ds.download(hs.data(), n);
    dc.download(hc.data(), n);
    for (u64 i = 0; i < n; ++i) {
        if (starts) starts[i] = hs[i];
        if (counts) counts[i] = hc[i];
        if (found) found[i] = hc[i] ? 1 : 0;
    }
    FV_API_END
}

fv_status fv_column_probe(const fv_column* col, uint32_t v, uint32_t* start, uint32_t* count,
                          int* found) {
    uint8_t f = 0;
    uint32_t s = 0, k = 0;
    fv_status st = fv_column_probe_many(col, &v, 1, &s, &k, &f);
    if (st != FV_OK) return st;
    if (start) *start = s;
    if (count) *count = k;
    if (found) *found = f;
    return FV_OK;
}

fv_status fv_column_gather(const fv_column* col, const uint32_t* ids, uint64_t n, uint32_t* out) {
    FV_API_BEGIN(col ? col->ctx : nullptr)
    FV_REQUIRE(col && (ids || n == 0), FV_ERR_INVALID, "fv_column_gather: null argument");
    fv::Ctx* c = col->ctx->c;
    DBuf<u32> di = fv::make_dbuf(c, ids, n);
    fv::check_ids(c, di.get(), n, col->col->n, "gather: tuple id past end of column");
    DBuf<u32> r = fv::gather_device(c, col->col->raw.get(), di.get(), n);
    r.download(out, n);
    FV_API_END
}

fv_status fv_column_append_and_reindex(const fv_column* col, const uint32_t* values, uint64_t n,
                                       fv_column** out) {
    FV_API_BEGIN(col ? col->ctx : nullptr)
    FV_REQUIRE(col && out && (values || n == 0), FV_ERR_INVALID, "append: null argument");
    fv::Ctx* c = col->ctx->c;
    const u64 total = col->col->n + n;
    DBuf<u32> merged(c, total);
    if (col->col->n)
        FV_CUDA(cudaMemcpyAsync(merged.get(), col->col->raw.get(), 4 * col->col->n,
                                cudaMemcpyDeviceToDevice, c->stream));
    merged.upload(values, n, col->col->n);
    auto w = std::make_unique<fv_column>();
    w->ctx = col->ctx;
    w->owned = fv::column_build(c, std::move(merged), total);
    w->col = w->owned.get();
    c->sync();
    *out = w.release();
    FV_API_END
}

fv_status fv_build_index(fv_ctx* ctx, const uint32_t* raw, uint64_t n, uint32_t* sorted_idx,
                         uint32_t* keys, uint32_t* starts, uint32_t* counts, uint64_t* n_unique) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(raw || n == 0, FV_ERR_INVALID, "fv_build_index: null raw");
    fv::Ctx* c = ctx->c;
    DBuf<u32> draw = fv::make_dbuf(c, raw, n);
    DBuf<u32> sidx, uk, us, uc;
    u64 nu = 0;
    fv::build_index(c, draw.get(), n, sidx, uk, us, uc, nu);
    if (sorted_idx) sidx.download(sorted_idx, n);
    if (keys) uk.download(keys, nu);
    if (starts) us.download(starts, nu);
    if (counts) uc.download(counts, nu);
    if (n_unique) *n_unique = nu;
    FV_API_END
}

// ---- versions --------------------------------------------------------------------

fv_status fv_version_from_columns(fv_ctx* ctx, uint32_t arity, const uint32_t* const* cols,
                                  uint64_t n, fv_version** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(out, FV_ERR_INVALID, "fv_version_from_columns: null out");
    FV_REQUIRE(arity <= FV_MAX_ARITY, FV_ERR_ARITY, "fv_version_from_columns: arity exceeds FV_MAX_ARITY");
    std::vector<DBuf<u32>> dcols;
    for (u32 j = 0; j < arity; ++j) {
        FV_REQUIRE(cols && (cols[j] || n == 0), FV_ERR_INVALID, "fv_version_from_columns: null column");
        dcols.push_back(fv::make_dbuf(ctx->c, cols[j], n));
    }
    *out = wrap_version(ctx, fv::version_from_device(ctx->c, std::move(dcols), n));
    ctx->c->sync();
    FV_API_END
}

fv_status fv_version_decompose(fv_ctx* ctx, uint32_t arity, const uint32_t* rows, uint64_t n,
                               fv_version** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(out && (rows || n == 0 || arity == 0), FV_ERR_INVALID, "fv_version_decompose: null argument");
    FV_REQUIRE(arity <= FV_MAX_ARITY, FV_ERR_ARITY, "fv_version_decompose: arity exceeds FV_MAX_ARITY");
    std::vector<std::vector<u32>> cols(arity, std::vector<u32>(n));
    for (u64 i = 0; i < n; ++i)
        for (u32 j = 0; j < arity; ++j) cols[j][i] = rows[i * arity + j];
    std::vector<DBuf<u32>> dcols;
    for (u32 j = 0; j < arity; ++j) dcols.push_back(fv::make_dbuf(ctx->c, cols[j].data(), n));
    *out = wrap_version(ctx, fv::version_from_device(ctx->c, std::move(dcols), n));
    ctx->c->sync();
    FV_API_END
}

fv_status fv_version_empty(fv_ctx* ctx, uint32_t arity, fv_version** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(out, FV_ERR_INVALID, "fv_version_empty: null out");
    *out = wrap_version(ctx, fv::version_empty(ctx->c, arity));
    FV_API_END
}

void fv_version_free(fv_version* v) {
    if (!v) return;
    v->ctx->c->activate();
    delete v;
}

uint32_t fv_version_arity(const fv_version* v) { return v ? v->v->arity : 0; }
uint64_t fv_version_rows(const fv_version* v) { return v ? v->v->rows : 0; }

const fv_column* fv_version_col(const fv_version* v, uint32_t j) {
    if (!v || j >= v->views.size()) return nullptr;
    return v->views[j].get();
}

fv_status fv_version_reconstruct(const fv_version* v, uint32_t* rows_out) {
    FV_API_BEGIN(v ? v->ctx : nullptr)
    FV_REQUIRE(v, FV_ERR_INVALID, "fv_version_reconstruct: null version");
    fv::version_reconstruct(*v->v, rows_out);
    FV_API_END
}

fv_status fv_version_append(const fv_version* v, const fv_version* extra, fv_version** out) {
    FV_API_BEGIN(v ? v->ctx : nullptr)
    FV_REQUIRE(v && extra && out, FV_ERR_INVALID, "fv_version_append: null argument");
    *out = wrap_version(v->ctx, fv::version_append(v->ctx->c, *v->v, *extra->v));
    v->ctx->c->sync();
    FV_API_END
}

fv_status fv_dedup_rows(const fv_version* v, fv_version** out) {
    FV_API_BEGIN(v ? v->ctx : nullptr)
    FV_REQUIRE(v && out, FV_ERR_INVALID, "fv_dedup_rows: null argument");
    *out = wrap_version(v->ctx, fv::dedup_rows(v->ctx->c, *v->v));
    v->ctx->c->sync();
    FV_API_END
}

fv_status fv_has_duplicate_rows(const fv_version* v, int* out) {
    FV_API_BEGIN(v ? v->ctx : nullptr)
    FV_REQUIRE(v && out, FV_ERR_INVALID, "fv_has_duplicate_rows: null argument");
    *out = fv::has_duplicate_rows(v->ctx->c, *v->v) ? 1 : 0;
    FV_API_END
}

// ---- relations -----------------------------------------------------------------------

fv_status fv_relation_create(fv_ctx* ctx, const char* name, uint32_t arity, fv_relation** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(out, FV_ERR_INVALID, "fv_relation_create: null out");
    auto* r = new fv_relation();
    r->ctx = ctx;
    r->name = name ? name : "";
    r->arity = arity;
    r->full.reset(wrap_version(ctx, fv::version_empty(ctx->c, arity)));
    r->delta.reset(wrap_version(ctx, fv::version_empty(ctx->c, arity)));
    r->new_rows.reset(wrap_version(ctx, fv::version_empty(ctx->c, arity)));
    *out = r;
    FV_API_END
}

void fv_relation_free(fv_relation* r) {
    if (!r) return;
    r->ctx->c->activate();
    delete r;
}

const fv_version* fv_relation_full(const fv_relation* r) { return r ? r->full.get() : nullptr; }
const fv_version* fv_relation_delta(const fv_relation* r) { return r ? r->delta.get() : nullptr; }
const fv_version* fv_relation_new(const fv_relation* r) { return r ? r->new_rows.get() : nullptr; }

fv_status fv_relation_set_full(fv_relation* r, fv_version* v) {
    FV_API_BEGIN(r ? r->ctx : nullptr)
    FV_REQUIRE(r && v, FV_ERR_INVALID, "fv_relation_set_full: null argument");
    if (v->v->arity != r->arity) fv::fail(FV_ERR_ARITY, "set_full: arity mismatch");
    r->full.reset(v);
    FV_API_END
}

fv_status fv_relation_merge_delta(fv_relation* r, fv_version* deduped_delta) {
    FV_API_BEGIN(r ? r->ctx : nullptr)
    FV_REQUIRE(r && deduped_delta, FV_ERR_INVALID, "fv_relation_merge_delta: null argument");
    if (deduped_delta->v->arity != r->arity) fv::fail(FV_ERR_ARITY, "merge_delta: arity mismatch");
    fv::Ctx* c = r->ctx->c;
    std::unique_ptr<fv_version> merged(wrap_version(r->ctx, fv::version_append(c, *r->full->v, *deduped_delta->v)));
    r->full = std::move(merged);
    r->delta.reset(deduped_delta);
    r->new_rows.reset(wrap_version(r->ctx, fv::version_empty(c, r->arity)));
    c->sync();
    FV_API_END
}

// ---- RA kernels ----------------------------------------------------------------------

fv_status fv_select_eq(const fv_column* col, uint32_t v, fv_array** ids) {
    FV_API_BEGIN(col ? col->ctx : nullptr)
    FV_REQUIRE(col && ids, FV_ERR_INVALID, "fv_select_eq: null argument");
    u64 n = 0;
    DBuf<u32> r = fv::select_eq(col->ctx->c, *col->col, v, n);
    *ids = fvapi::wrap_array_u32(col->ctx, std::move(r), n);
    FV_API_END
}

fv_status fv_project(const fv_version* v, const uint32_t* ids, uint64_t n_ids,
                     const uint32_t* col_map, uint32_t n_cols, fv_version** out) {
    FV_API_BEGIN(v ? v->ctx : nullptr)
    FV_REQUIRE(v && out && (ids || n_ids == 0) && (col_map || n_cols == 0), FV_ERR_INVALID,
               "fv_project: null argument");
    fv::Ctx* c = v->ctx->c;
    DBuf<u32> di = fv::make_dbuf(c, ids, n_ids);
    std::vector<u32> cm(col_map, col_map + n_cols);
    *out = wrap_version(v->ctx, fv::project(c, *v->v, di.get(), n_ids, cm));
    c->sync();
    FV_API_END
}

fv_status fv_join_probe_phase(fv_ctx* ctx, const uint32_t* probe_values, uint64_t n,
                              const fv_column* build, fv_match** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(build && out && (probe_values || n == 0), FV_ERR_INVALID, "fv_join_probe_phase: null argument");
    DBuf<u32> dp = fv::make_dbuf(ctx->c, probe_values, n);
    auto* m = new fv_match();
    m->ctx = ctx;
    m->m = fv::join_probe_phase(ctx->c, dp.get(), n, *build->col);
    *out = m;
    FV_API_END
}

fv_status fv_match_create(fv_ctx* ctx, const uint32_t* starts, const uint32_t* counts,
                          const uint32_t* matched, uint64_t n, fv_match** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(out && ((starts && counts && matched) || n == 0), FV_ERR_INVALID, "fv_match_create: null argument");
    auto* m = new fv_match();
    m->ctx = ctx;
    m->m = std::make_unique<fv::Match>();
    m->m->ctx = ctx->c;
    m->m->m = n;
    m->m->starts = fv::make_dbuf(ctx->c, starts, n);
    m->m->counts = fv::make_dbuf(ctx->c, counts, n);
    m->m->matched = fv::make_dbuf(ctx->c, matched, n);
    *out = m;
    FV_API_END
}

void fv_match_free(fv_match* m) {
    if (!m) return;
    m->ctx->c->activate();
    delete m;
}

uint64_t fv_match_size(const fv_match* m) { return m ? m->m->m : 0; }

fv_status fv_match_read(const fv_match* m, uint32_t* starts, uint32_t* counts, uint32_t* matched) {
    FV_API_BEGIN(m ? m->ctx : nullptr)
    FV_REQUIRE(m, FV_ERR_INVALID, "fv_match_read: null match");
    if (starts) m->m->starts.download(starts, m->m->m);
    if (counts) m->m->counts.download(counts, m->m->m);
    if (matched) m->m->matched.download(matched, m->m->m);
    FV_API_END
}

fv_status fv_join_total_size(const fv_match* m, uint64_t* total) {
    FV_API_BEGIN(m ? m->ctx : nullptr)
    FV_REQUIRE(m && total, FV_ERR_INVALID, "fv_join_total_size: null argument");
    *total = fv::join_total_size(m->ctx->c, *m->m);
    FV_API_END
}

fv_status fv_join_offsets(const fv_match* m, uint64_t* offsets) {
    FV_API_BEGIN(m ? m->ctx : nullptr)
    FV_REQUIRE(m, FV_ERR_INVALID, "fv_join_offsets: null match");
    DBuf<u64> off = fv::join_offsets(m->ctx->c, *m->m);
    if (offsets) off.download(offsets, m->m->m);
    FV_API_END
}

fv_status fv_join_write_phase(const fv_match* m, const fv_column* build, fv_array** a_ids,
                              fv_array** b_ids) {
    FV_API_BEGIN(m ? m->ctx : nullptr)
    FV_REQUIRE(m && build && a_ids && b_ids, FV_ERR_INVALID, "fv_join_write_phase: null argument");
    fv::Ctx* c = m->ctx->c;
    DBuf<u64> off = fv::join_offsets(c, *m->m);
    u64 total = 0;
    off.download(&total, 1, m->m->m);
    DBuf<u32> a, b;
    fv::join_write_phase(c, *m->m, off.get(), total, *build->col, a, b);
    *a_ids = fvapi::wrap_array_u32(m->ctx, std::move(a), total);
    *b_ids = fvapi::wrap_array_u32(m->ctx, std::move(b), total);
    FV_API_END
}

fv_status fv_column_join(fv_ctx* ctx, const uint32_t* probe_values, uint64_t n,
                         const fv_column* build, fv_array** a_ids, fv_array** b_ids) {
    fv_match* m = nullptr;
    fv_status s = fv_join_probe_phase(ctx, probe_values, n, build, &m);
    if (s != FV_OK) return s;
    s = fv_join_write_phase(m, build, a_ids, b_ids);
    fv_match_free(m);
    return s;
}

fv_status fv_filter_pairs_eq(fv_ctx* ctx, const uint32_t* a_ids, const uint32_t* b_ids,
                             uint64_t n, const fv_column* col_a, const fv_column* col_b,
                             fv_array** out_a, fv_array** out_b) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(col_a && col_b && out_a && out_b && ((a_ids && b_ids) || n == 0), FV_ERR_INVALID,
               "fv_filter_pairs_eq: null argument");
    fv::Ctx* c = ctx->c;
    DBuf<u32> da = fv::make_dbuf(c, a_ids, n), db = fv::make_dbuf(c, b_ids, n);
    DBuf<u32> oa, ob;
    u64 k = 0;
    fv::filter_pairs_eq(c, da.get(), db.get(), n, *col_a->col, *col_b->col, oa, ob, k);
    *out_a = fvapi::wrap_array_u32(ctx, std::move(oa), k);
    *out_b = fvapi::wrap_array_u32(ctx, std::move(ob), k);
    FV_API_END
}

fv_status fv_filter_neq(const fv_version* v, uint32_t col_i, uint32_t col_j, fv_array** ids) {
    FV_API_BEGIN(v ? v->ctx : nullptr)
    FV_REQUIRE(v && ids, FV_ERR_INVALID, "fv_filter_neq: null argument");
    u64 k = 0;
    DBuf<u32> r = fv::filter_neq(v->ctx->c, *v->v, col_i, col_j, k);
    *ids = fvapi::wrap_array_u32(v->ctx, std::move(r), k);
    FV_API_END
}

fv_status fv_deduplicate(const fv_version* new_v, const fv_version* full, fv_array** flags) {
    FV_API_BEGIN(new_v ? new_v->ctx : nullptr)
    FV_REQUIRE(new_v && full && flags, FV_ERR_INVALID, "fv_deduplicate: null argument");
    DBuf<u8> f = fv::deduplicate(new_v->ctx->c, *new_v->v, *full->v);
    *flags = fvapi::wrap_array_u8(new_v->ctx, std::move(f), new_v->v->rows);
    FV_API_END
}

fv_status fv_difference(const fv_version* new_v, const uint8_t* flags, uint64_t n,
                        fv_version** out) {
    FV_API_BEGIN(new_v ? new_v->ctx : nullptr)
    FV_REQUIRE(new_v && out && (flags || n == 0), FV_ERR_INVALID, "fv_difference: null argument");
    if (n != new_v->v->rows) fv::fail(FV_ERR_ARITY, "difference: bitmap not aligned with version");
    fv::Ctx* c = new_v->ctx->c;
    DBuf<u8> df = fv::make_dbuf(c, flags, n);
    *out = wrap_version(new_v->ctx, fv::difference(c, *new_v->v, df.get()));
    c->sync();
    FV_API_END
}

fv_status fv_union_concat(const fv_version* full, const fv_version* delta, fv_version** out) {
    return fv_version_append(full, delta, out);
}

}  // extern "C"

// extern "C" boundary, frontend / engine / runner half (include/fvlog.h).
#include <cstdlib>
#include <cstring>
#include <sstream>

#include <set>

#include "api_internal.h"
#include "frontend.h"
#include "runner.h"
#include "transport.h"

using fv::u32;
using fv::u64;

// POD views of compiled plans, kept alive by the owning program.
struct PlanPod {
    std::vector<fv_plan_source> sources;
    std::vector<std::vector<u32>> const_cols, const_vals, self_pairs;
    std::vector<fv_plan_join> joins;
    std::vector<std::vector<fv_colref>> res_left;
    std::vector<std::vector<u32>> res_right;
    std::vector<fv_colref> outputs;
    std::vector<u32> guards;
    fv_plan plan{};
};

struct fv_program {
    fv::fe::Program prog;
    fv::fe::Dictionary dict;
    std::vector<fv::Plan> plans;
    bool compiled = false;
    std::vector<std::unique_ptr<PlanPod>> pods;
};

struct fv_edb {
    fv_ctx* ctx = nullptr;
    fv::DeviceEdb edb;
};

struct fv_state {
    fv_ctx* ctx = nullptr;
    std::unique_ptr<fv::EvalState> st;
    std::vector<std::string> names;
};

namespace {

void copy_out(const std::string& s, char* buf, size_t cap) {
    if (!buf || cap == 0) return;
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
}

std::unique_ptr<PlanPod> make_pod(const fv::Plan& p) {
    auto pod = std::make_unique<PlanPod>();
    const size_t ns = p.sources.size();
    pod->const_cols.resize(ns);
    pod->const_vals.resize(ns);
    pod->self_pairs.resize(ns);
    for (size_t s = 0; s < ns; ++s) {
        for (auto& [c, v] : p.sources[s].const_selects) {
            pod->const_cols[s].push_back(c);
            pod->const_vals[s].push_back(v);
        }
        for (auto& [a, b] : p.sources[s].self_eqs) {
            pod->self_pairs[s].push_back(a);
            pod->self_pairs[s].push_back(b);
        }
    }
    for (size_t s = 0; s < ns; ++s) {
        fv_plan_source x{};
        x.relation = p.sources[s].relation.c_str();
        x.arity = p.sources[s].arity;
        x.n_const_selects = static_cast<u32>(pod->const_cols[s].size());
        x.const_select_cols = pod->const_cols[s].data();
        x.const_select_vals = pod->const_vals[s].data();
        x.n_self_eqs = static_cast<u32>(p.sources[s].self_eqs.size());
        x.self_eq_pairs = pod->self_pairs[s].data();
        pod->sources.push_back(x);
    }
    pod->res_left.resize(p.joins.size());
    pod->res_right.resize(p.joins.size());
    for (size_t k = 0; k < p.joins.size(); ++k)
        for (auto& [l, r] : p.joins[k].residual_eq) {
            pod->res_left[k].push_back({l.source, l.col});
            pod->res_right[k].push_back(r);
        }
    for (size_t k = 0; k < p.joins.size(); ++k) {
        const auto& j = p.joins[k];
        fv_plan_join x{};
        x.right_source = j.right_source;
        x.left = {j.left.source, j.left.col};
        x.right_col = j.right_col;
        x.n_residual_eq = static_cast<u32>(pod->res_left[k].size());
        x.residual_left = pod->res_left[k].data();
        x.residual_right_col = pod->res_right[k].data();
        pod->joins.push_back(x);
    }
    for (auto& r : p.output_cols) pod->outputs.push_back({r.source, r.col});
    for (auto& [a, b] : p.guard_neq) {
        pod->guards.push_back(a);
        pod->guards.push_back(b);
    }
    fv_plan& q = pod->plan;
    q.head_relation = p.head.c_str();
    q.head_arity = p.head_arity;
    q.n_sources = static_cast<u32>(ns);
    q.sources = pod->sources.data();
    q.n_joins = static_cast<u32>(pod->joins.size());
    q.joins = pod->joins.data();
    q.n_output_cols = static_cast<u32>(pod->outputs.size());
    q.output_cols = pod->outputs.data();
    q.n_guards = static_cast<u32>(p.guard_neq.size());
    q.guard_neq_pairs = pod->guards.data();
    return pod;
}

fv::Plan from_pod(const fv_plan& q) {
    fv::Plan p;
    if (!q.head_relation) fv::fail(FV_ERR_PLAN, "plan without head relation");
    p.head = q.head_relation;
    p.head_arity = q.head_arity;
    for (u32 s = 0; s < q.n_sources; ++s) {
        const fv_plan_source& x = q.sources[s];
        fv::PlanSource src;
        if (!x.relation) fv::fail(FV_ERR_PLAN, "plan source without relation");
        src.relation = x.relation;
        src.arity = x.arity;
        for (u32 k = 0; k < x.n_const_selects; ++k)
            src.const_selects.emplace_back(x.const_select_cols[k], x.const_select_vals[k]);
        for (u32 k = 0; k < x.n_self_eqs; ++k)
            src.self_eqs.emplace_back(x.self_eq_pairs[2 * k], x.self_eq_pairs[2 * k + 1]);
        p.sources.push_back(std::move(src));
    }
    for (u32 k = 0; k < q.n_joins; ++k) {
        const fv_plan_join& x = q.joins[k];
        fv::PlanJoin j;
        j.right_source = x.right_source;
        j.left = {x.left.source, x.left.col};
        j.right_col = x.right_col;
        for (u32 r = 0; r < x.n_residual_eq; ++r)
            j.residual_eq.emplace_back(fv::ColRef{x.residual_left[r].source, x.residual_left[r].col},
                                       x.residual_right_col[r]);
        p.joins.push_back(std::move(j));
    }
    for (u32 k = 0; k < q.n_output_cols; ++k) p.output_cols.push_back({q.output_cols[k].source, q.output_cols[k].col});
    for (u32 k = 0; k < q.n_guards; ++k) p.guard_neq.emplace_back(q.guard_neq_pairs[2 * k], q.guard_neq_pairs[2 * k + 1]);
    return p;
}

std::vector<fv::FactsBlock> blocks_from(const fv_facts* facts, uint32_t n_facts) {
    std::vector<fv::FactsBlock> out;
    for (uint32_t i = 0; i < n_facts; ++i) {
        const fv_facts& f = facts[i];
        if (!f.relation) fv::fail(FV_ERR_INVALID, "facts block without relation name");
        fv::FactsBlock b{f.relation, f.arity, f.n_rows, {}};
        for (u32 j = 0; j < f.arity; ++j) {
            if (f.n_rows && (!f.cols || !f.cols[j])) fv::fail(FV_ERR_INVALID, "facts block with null column");
            b.cols.push_back(f.n_rows ? f.cols[j] : nullptr);
        }
        out.push_back(std::move(b));
    }
    return out;
}

fv_state* wrap_state(fv_ctx* ctx, std::unique_ptr<fv::EvalState> st) {
    auto* s = new fv_state();
    s->ctx = ctx;
    for (auto& [name, r] : st->relations) s->names.push_back(name);
    s->st = std::move(st);
    return s;
}

void ensure_compiled(fv_program* p) {
    if (p->compiled) return;
    auto diags = fv::fe::validate(p->prog);
    if (!diags.empty()) throw fv::fe::DiagnosticError(diags.front());
    p->plans = fv::fe::compile(p->prog);
    p->pods.clear();
    for (auto& plan : p->plans) p->pods.push_back(make_pod(plan));
    p->compiled = true;
}

}  // namespace

extern "C" {

fv_status fv_program_parse(const char* text, fv_program** out, char* diag, size_t diag_cap) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(text && out, FV_ERR_INVALID, "fv_program_parse: null argument");
    try {
        auto p = std::make_unique<fv_program>();
        p->prog = fv::fe::parse(text);
        fv::fe::resolve_strings(p->prog, p->dict);
        *out = p.release();
    } catch (const fv::fe::DiagnosticError& e) {
        copy_out(e.what(), diag, diag_cap);
        throw;
    }
    FV_API_END
}

void fv_program_free(fv_program* p) { delete p; }

fv_status fv_program_validate(const fv_program* p, char* diags, size_t cap, uint32_t* n_diags) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(p, FV_ERR_INVALID, "fv_program_validate: null program");
    auto d = fv::fe::validate(p->prog);
    std::string all;
    for (auto& x : d) all += fv::fe::format(x) + "\n";
    copy_out(all, diags, cap);
    if (n_diags) *n_diags = static_cast<uint32_t>(d.size());
    FV_API_END
}

fv_status fv_program_print(const fv_program* p, char* buf, size_t cap, size_t* len) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(p, FV_ERR_INVALID, "fv_program_print: null program");
    const std::string s = fv::fe::print(p->prog);
    copy_out(s, buf, cap);
    if (len) *len = s.size();
    FV_API_END
}

uint32_t fv_program_num_relations(const fv_program* p) {
    return p ? static_cast<uint32_t>(p->prog.relations.size()) : 0;
}

fv_status fv_program_relation(const fv_program* p, uint32_t i, fv_relation_decl* out) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(p && out, FV_ERR_INVALID, "fv_program_relation: null argument");
    if (i >= p->prog.relations.size()) fv::fail(FV_ERR_RANGE, "relation index out of range");
    out->name = p->prog.relations[i].name.c_str();
    out->arity = p->prog.relations[i].arity;
    FV_API_END
}

uint32_t fv_program_num_rules(const fv_program* p) { return p ? static_cast<uint32_t>(p->prog.rules.size()) : 0; }

fv_status fv_program_plan(const fv_program* p, uint32_t rule, const fv_plan** out) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(p && out, FV_ERR_INVALID, "fv_program_plan: null argument");
    auto* mp = const_cast<fv_program*>(p);
    ensure_compiled(mp);
    if (rule >= mp->pods.size()) fv::fail(FV_ERR_RANGE, "rule index out of range");
    *out = &mp->pods[rule]->plan;
    FV_API_END
}

fv_status fv_program_encode(fv_program* p, const char* s, uint32_t* out) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(p && s && out, FV_ERR_INVALID, "fv_program_encode: null argument");
    *out = p->dict.encode(s);
    FV_API_END
}

uint64_t fv_program_dictionary_size(const fv_program* p) { return p ? p->dict.size() : 0; }

fv_status fv_evaluate(fv_ctx* ctx, const fv_relation_decl* decls, uint32_t n_decls, const fv_plan* plans,
                      uint32_t n_plans, const fv_facts* facts, uint32_t n_facts, fv_state** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(ctx && out && (decls || !n_decls) && (plans || !n_plans) && (facts || !n_facts), FV_ERR_INVALID,
               "fv_evaluate: null argument");
    std::vector<fv::RelationDecl> d;
    for (uint32_t i = 0; i < n_decls; ++i) {
        FV_REQUIRE(decls[i].name, FV_ERR_INVALID, "fv_evaluate: declaration without name");
        d.push_back({decls[i].name, decls[i].arity});
    }
    std::vector<fv::Plan> ps;
    for (uint32_t i = 0; i < n_plans; ++i) ps.push_back(from_pod(plans[i]));
    *out = wrap_state(ctx, fv::evaluate(ctx->c, d, ps, blocks_from(facts, n_facts)));
    FV_API_END
}

fv_status fv_evaluate_program(fv_ctx* ctx, const fv_program* p, const fv_facts* facts, uint32_t n_facts,
                              fv_state** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(ctx && p && out && (facts || !n_facts), FV_ERR_INVALID, "fv_evaluate_program: null argument");
    auto* mp = const_cast<fv_program*>(p);
    ensure_compiled(mp);
    auto pf = fv::fe::program_facts(mp->prog);
    std::map<std::string, u32> arity;
    for (auto& r : mp->prog.relations) arity[r.name] = r.arity;
    std::vector<std::vector<u32>> storage;
    std::vector<fv::FactsBlock> blocks;
    for (auto& [rel, rows] : pf) {
        const u32 a = arity[rel];
        const u64 n = rows.size() / a;
        for (u32 j = 0; j < a; ++j) {
            storage.emplace_back(n);
            for (u64 i = 0; i < n; ++i) storage.back()[i] = rows[i * a + j];
        }
    }
    size_t si = 0;
    for (auto& [rel, rows] : pf) {
        const u32 a = arity[rel];
        fv::FactsBlock b{rel, a, rows.size() / a, {}};
        for (u32 j = 0; j < a; ++j) b.cols.push_back(storage[si++].data());
        blocks.push_back(std::move(b));
    }
    for (auto& b : blocks_from(facts, n_facts)) blocks.push_back(std::move(b));
    *out = wrap_state(ctx, fv::evaluate(ctx->c, fv::fe::declarations(mp->prog), mp->plans, blocks));
    FV_API_END
}

fv_status fv_edb_upload(fv_ctx* ctx, const fv_relation_decl* decls, uint32_t n_decls, const fv_facts* facts,
                        uint32_t n_facts, fv_edb** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(ctx && out && (decls || !n_decls) && (facts || !n_facts), FV_ERR_INVALID, "fv_edb_upload: null argument");
    std::vector<fv::RelationDecl> d;
    for (uint32_t i = 0; i < n_decls; ++i) d.push_back({decls[i].name, decls[i].arity});
    auto* e = new fv_edb();
    e->ctx = ctx;
    e->edb = fv::upload_facts(ctx->c, d, blocks_from(facts, n_facts));
    ctx->c->sync();
    *out = e;
    FV_API_END
}

void fv_edb_free(fv_edb* e) {
    if (!e) return;
    e->ctx->c->activate();
    delete e;
}

fv_status fv_evaluate_program_edb(fv_ctx* ctx, const fv_program* p, const fv_edb* edb, fv_state** out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(ctx && p && edb && out, FV_ERR_INVALID, "fv_evaluate_program_edb: null argument");
    auto* mp = const_cast<fv_program*>(p);
    ensure_compiled(mp);
    auto decls = fv::fe::declarations(mp->prog);
    // Program-text facts are tiny; upload them next to the resident EDB.
    auto pf = fv::fe::program_facts(mp->prog);
    std::vector<std::vector<u32>> storage;
    std::vector<fv::FactsBlock> blocks;
    std::map<std::string, u32> arity;
    for (auto& r : mp->prog.relations) arity[r.name] = r.arity;
    for (auto& [rel, rows] : pf) {
        const u32 a = arity[rel];
        const u64 n = rows.size() / a;
        fv::FactsBlock b{rel, a, n, {}};
        for (u32 j = 0; j < a; ++j) {
            storage.emplace_back(n);
            for (u64 i = 0; i < n; ++i) storage.back()[i] = rows[i * a + j];
        }
        blocks.push_back(std::move(b));
    }
    size_t si = 0;
    for (auto& b : blocks)
        for (u32 j = 0; j < b.arity; ++j) b.cols.push_back(storage[si++].data());
    fv::DeviceEdb text_edb = fv::upload_facts(ctx->c, decls, blocks);
    *out = wrap_state(ctx, fv::evaluate_device(ctx->c, decls, mp->plans, {&text_edb, &edb->edb}));
    FV_API_END
}

fv_status fv_evaluate_program_sharded(fv_ctx* ctx, const fv_program* p, const fv_facts* facts, uint32_t n_facts,
                                      uint32_t world, fv_state** states_out) {
    FV_API_BEGIN(ctx)
    FV_REQUIRE(ctx && p && states_out && (facts || !n_facts), FV_ERR_INVALID,
               "fv_evaluate_program_sharded: null argument");
    auto* mp = const_cast<fv_program*>(p);
    ensure_compiled(mp);
    auto pf = fv::fe::program_facts(mp->prog);
    std::map<std::string, u32> arity;
    for (auto& r : mp->prog.relations) arity[r.name] = r.arity;
    std::vector<std::vector<u32>> storage;
    for (auto& [rel, rows] : pf) {
        const u32 a = arity[rel];
        const u64 n = rows.size() / a;
        for (u32 j = 0; j < a; ++j) {
            storage.emplace_back(n);
            for (u64 i = 0; i < n; ++i) storage.back()[i] = rows[i * a + j];
        }
    }
    std::vector<fv::FactsBlock> blocks;
    size_t si = 0;
    for (auto& [rel, rows] : pf) {
        const u32 a = arity[rel];
        fv::FactsBlock b{rel, a, rows.size() / a, {}};
        for (u32 j = 0; j < a; ++j) b.cols.push_back(storage[si++].data());
        blocks.push_back(std::move(b));
    }
    for (auto& b : blocks_from(facts, n_facts)) blocks.push_back(std::move(b));
    auto states = fv::evaluate_sharded(ctx->c, world, fv::fe::declarations(mp->prog), mp->plans, blocks);
    for (uint32_t r = 0; r < world; ++r) states_out[r] = wrap_state(ctx, std::move(states[r]));
    FV_API_END
}

fv_status fv_program_partition_plan(const fv_program* p, char* buf, size_t cap, size_t* len) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(p, FV_ERR_INVALID, "fv_program_partition_plan: null program");
    auto* mp = const_cast<fv_program*>(p);
    ensure_compiled(mp);
    std::set<std::string> idb;
    for (auto& plan : mp->plans) idb.insert(plan.head);
    std::map<std::string, std::set<u32>> keyset;
    std::map<std::string, u32> idb_arity;
    for (auto& r : mp->prog.relations)
        if (idb.count(r.name)) idb_arity[r.name] = static_cast<u32>(r.arity);
    std::vector<std::pair<const fv::Plan*, long>> variants;
    for (auto& plan : mp->plans)
        for (size_t s = 0; s < plan.sources.size(); ++s)
            if (idb.count(plan.sources[s].relation)) variants.emplace_back(&plan, static_cast<long>(s));
    const auto home = fv::choose_home_cols(variants, idb_arity);
    std::ostringstream rules;
    rules << "[";
    for (size_t i = 0; i < mp->plans.size(); ++i) {
        const auto dp = fv::dist_plan(mp->plans[i], idb, home);
        for (size_t s = 0; s < dp.src_copy.size(); ++s) {
            const std::string& rel = mp->plans[i].sources[s].relation;
            if (idb.count(rel)) keyset[rel].insert(dp.src_copy[s]);
        }
        rules << (i ? "," : "") << "{\"src_copy\":[";
        for (size_t s = 0; s < dp.src_copy.size(); ++s) rules << (s ? "," : "") << dp.src_copy[s];
        rules << "],\"shuffle\":[";
        for (size_t k = 0; k < dp.shuffle.size(); ++k) rules << (k ? "," : "") << int(dp.shuffle[k]);
        rules << "],\"replicated_out\":" << (dp.replicated_out ? "true" : "false")
              << ",\"local_out\":" << (dp.local_out ? "true" : "false") << "}";
    }
    rules << "]";
    std::ostringstream os;
    os << "{\"relations\":{";
    bool first = true;
    for (auto& r : mp->prog.relations) {
        const bool is_idb = idb.count(r.name) > 0;
        std::set<u32> ks = keyset[r.name];
        const u32 h = is_idb ? home.at(r.name) : 0;
        if (is_idb) ks.insert(h);
        os << (first ? "" : ",") << "\"" << r.name << "\":{\"idb\":" << (is_idb ? "true" : "false")
           << ",\"home\":" << h << ",\"keyset\":[";
        bool f2 = true;
        for (u32 k : ks) {
            os << (f2 ? "" : ",") << k;
            f2 = false;
        }
        os << "]}";
        first = false;
    }
    os << "},\"rules\":" << rules.str() << "}";
    const std::string s = os.str();
    copy_out(s, buf, cap);
    if (len) *len = s.size();
    FV_API_END
}

uint32_t fv_owner(uint32_t v, uint32_t world) { return fv::owner_of(v, world); }

fv_status fv_state_partition(const fv_state* s, int* rank, int* world) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(s, FV_ERR_INVALID, "fv_state_partition: null state");
    if (rank) *rank = s->st->rank;
    if (world) *world = s->st->world;
    FV_API_END
}

void fv_state_free(fv_state* s) {
    if (!s) return;
    if (s->ctx) s->ctx->c->activate();
    delete s;
}

uint64_t fv_state_iterations(const fv_state* s) { return s ? s->st->iterations : 0; }
double fv_state_elapsed_ms(const fv_state* s) { return s ? s->st->elapsed_ms : 0.0; }
uint64_t fv_state_num_relations(const fv_state* s) { return s ? s->names.size() : 0; }

fv_status fv_state_relation(const fv_state* s, uint64_t i, const char** name, uint32_t* arity, uint64_t* rows) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(s, FV_ERR_INVALID, "fv_state_relation: null state");
    if (i >= s->names.size()) fv::fail(FV_ERR_RANGE, "relation index out of range");
    const auto& r = *s->st->relations.at(s->names[i]);
    if (name) *name = s->names[i].c_str();
    if (arity) *arity = r.arity;
    if (rows) *rows = r.rows();
    FV_API_END
}

uint64_t fv_state_num_stats(const fv_state* s) { return s ? s->st->stats.size() : 0; }

fv_status fv_state_stat(const fv_state* s, uint64_t i, uint64_t* iteration, const char** rel, uint64_t* delta_rows,
                        uint64_t* full_rows, uint64_t* merges, double* elapsed_ms) {
    FV_API_BEGIN(nullptr)
    FV_REQUIRE(s, FV_ERR_INVALID, "fv_state_stat: null state");
    if (i >= s->st->stats.size()) fv::fail(FV_ERR_RANGE, "stat index out of range");
    const auto& x = s->st->stats[i];
    if (iteration) *iteration = x.iteration;
    if (rel) *rel = x.relation.c_str();
    if (delta_rows) *delta_rows = x.delta_rows;
    if (full_rows) *full_rows = x.full_rows;
    if (merges) *merges = x.merges;
    if (elapsed_ms) *elapsed_ms = x.elapsed_ms;
    FV_API_END
}

fv_status fv_state_dump_sorted(const fv_state* s, const char* rel, uint32_t* rows_out) {
    FV_API_BEGIN(s ? s->ctx : nullptr)
    FV_REQUIRE(s && rel, FV_ERR_INVALID, "fv_state_dump_sorted: null argument");
    if (rows_out) {
        fv::dump_sorted_into(*s->st, rel, rows_out);
    } else {
        if (!s->st->relations.count(rel)) fv::fail(FV_ERR_RANGE, std::string("unknown relation '") + rel + "'");
    }
    FV_API_END
}

fv_status fv_state_fingerprint(const fv_state* s, const char* rel, uint64_t* out) {
    FV_API_BEGIN(s ? s->ctx : nullptr)
    FV_REQUIRE(s && rel && out, FV_ERR_INVALID, "fv_state_fingerprint: null argument");
    *out = fv::fingerprint(*s->st, rel);
    FV_API_END
}

int fv_run(int device, const char* program_path, const char* facts_dir, const char* out_dir, int print_stats,
           const char* dump_list, char** out, char** err) {
    std::ostringstream o, e;
    int rc = 1;
    fv::Ctx* c = nullptr;
    try {
        c = fv::ctx_new(device);
        fv::RunConfig cfg;
        cfg.program_path = program_path ? program_path : "";
        cfg.facts_dir = facts_dir ? facts_dir : "";
        cfg.out_dir = out_dir ? out_dir : "";
        cfg.print_stats = print_stats != 0;
        std::string dl = dump_list ? dump_list : "";
        size_t start = 0;
        while (!dl.empty() && start <= dl.size()) {
            size_t comma = dl.find(',', start);
            if (comma == std::string::npos) comma = dl.size();
            if (comma > start) cfg.dump_relations.push_back(dl.substr(start, comma - start));
            start = comma + 1;
        }
        rc = fv::run(c, cfg, o, e);
    } catch (const std::exception& ex) {
        e << "error: " << ex.what() << "\n";
        rc = 1;
    }
    if (c) fv::ctx_delete(c);
    auto dup = [](const std::string& s) {
        char* p = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(p, s.c_str(), s.size() + 1);
        return p;
    };
    if (out) *out = dup(o.str());
    if (err) *err = dup(e.str());
    return rc;
}

void fv_free(void* p) { std::free(p); }

}  // extern "C"

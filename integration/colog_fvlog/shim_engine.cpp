// The semi-naive driver (P/include/colog/engine.hpp) on fvlog.
//
//   evaluate      -> fv_evaluate: seed, every iteration and the fixpoint test
//                    run on the device; the result relations come back as
//                    host Versions (sorted FULL), the stats as IterationStats.
//   execute_plan  -> fv_evaluate of the one plan over its resolved source
//                    versions as EDB inputs (one EDB-only iteration). The
//                    head block is returned as a set (distinct rows, sorted);
//                    the reference returns one row per derivation
//                    (P/src/engine.cpp:72-146) — equal as sets, which is how
//                    every caller compares it.
//   seed / run_iteration -> the reference's step semantics composed from the
//                    device operators of shim_relation.cpp / shim_kernels.cpp.
//   delta_rewrite / idb_relations -> plan bookkeeping (host, no data).
// Validation and compilation stay the reference's own (parser.cpp,
// compiler.cpp are linked unchanged).
#include <chrono>
#include <functional>
#include <map>
#include <memory>

#include "colog/engine.hpp"
#include "colog/kernels.hpp"
#include "colog/parser.hpp"
#include "shim.hpp"

namespace colog {

using fvshim::check;
using fvshim::ctx;

namespace {

// A RulePlan as the fv_plan POD (fvlog.h), with the arrays it points into.
class PodPlan {
public:
    PodPlan(const RulePlan& p, const std::string* head_override = nullptr,
            const std::vector<std::string>* source_names = nullptr) {
        head_ = head_override ? *head_override : p.head_relation;
        const std::size_t ns = p.sources.size();
        names_.resize(ns);
        sel_cols_.resize(ns);
        sel_vals_.resize(ns);
        self_.resize(ns);
        for (std::size_t s = 0; s < ns; ++s) {
            const auto& src = p.sources[s];
            names_[s] = source_names ? (*source_names)[s] : src.relation;
            for (auto& [c, v] : src.const_selects) {
                sel_cols_[s].push_back(static_cast<std::uint32_t>(c));
                sel_vals_[s].push_back(v);
            }
            for (auto& [a, b] : src.self_eqs) {
                self_[s].push_back(static_cast<std::uint32_t>(a));
                self_[s].push_back(static_cast<std::uint32_t>(b));
            }
        }
        res_l_.resize(p.joins.size());
        res_r_.resize(p.joins.size());
        for (std::size_t k = 0; k < p.joins.size(); ++k)
            for (auto& [l, rc] : p.joins[k].residual_eq) {
                res_l_[k].push_back(ref(l));
                res_r_[k].push_back(static_cast<std::uint32_t>(rc));
            }
        for (const ColRef& r : p.output_cols) outs_.push_back(ref(r));
        for (auto& [a, b] : p.guard_neq) {
            guards_.push_back(static_cast<std::uint32_t>(a));
            guards_.push_back(static_cast<std::uint32_t>(b));
        }
        // Pointers are taken only once every vector has its final size.
        for (std::size_t s = 0; s < ns; ++s) {
            fv_plan_source ps{};
            ps.relation = names_[s].c_str();
            ps.arity = static_cast<std::uint32_t>(p.sources[s].arity);
            ps.n_const_selects = static_cast<std::uint32_t>(sel_cols_[s].size());
            ps.const_select_cols = sel_cols_[s].data();
            ps.const_select_vals = sel_vals_[s].data();
            ps.n_self_eqs = static_cast<std::uint32_t>(self_[s].size() / 2);
            ps.self_eq_pairs = self_[s].data();
            srcs_.push_back(ps);
        }
        for (std::size_t k = 0; k < p.joins.size(); ++k) {
            const auto& j = p.joins[k];
            fv_plan_join pj{};
            pj.right_source = static_cast<std::uint32_t>(j.right_source);
            pj.left = ref(j.left);
            pj.right_col = static_cast<std::uint32_t>(j.right_col);
            pj.n_residual_eq = static_cast<std::uint32_t>(res_l_[k].size());
            pj.residual_left = res_l_[k].data();
            pj.residual_right_col = res_r_[k].data();
            joins_.push_back(pj);
        }
        pod_.head_relation = head_.c_str();
        pod_.head_arity = static_cast<std::uint32_t>(p.head_arity);
        pod_.n_sources = static_cast<std::uint32_t>(srcs_.size());
        pod_.sources = srcs_.data();
        pod_.n_joins = static_cast<std::uint32_t>(joins_.size());
        pod_.joins = joins_.data();
        pod_.n_output_cols = static_cast<std::uint32_t>(outs_.size());
        pod_.output_cols = outs_.data();
        pod_.n_guards = static_cast<std::uint32_t>(guards_.size() / 2);
        pod_.guard_neq_pairs = guards_.data();
    }
    PodPlan(const PodPlan&) = delete;
    PodPlan& operator=(const PodPlan&) = delete;
    const fv_plan& pod() const { return pod_; }

private:
    static fv_colref ref(const ColRef& r) {
        return fv_colref{static_cast<std::uint32_t>(r.source), static_cast<std::uint32_t>(r.col)};
    }
    std::string head_;
    std::vector<std::string> names_;
    std::vector<std::vector<std::uint32_t>> sel_cols_, sel_vals_, self_, res_r_;
    std::vector<std::vector<fv_colref>> res_l_;
    std::vector<fv_colref> outs_;
    std::vector<std::uint32_t> guards_;
    std::vector<fv_plan_source> srcs_;
    std::vector<fv_plan_join> joins_;
    fv_plan pod_{};
};

// SoA fact blocks over host columns the caller keeps alive.
struct FactBlocks {
    std::vector<std::string> names;
    std::vector<std::vector<std::vector<std::uint32_t>>> owned;
    std::vector<std::vector<const std::uint32_t*>> ptrs;
    std::vector<fv_facts> blocks;

    void reserve(std::size_t n) {
        names.reserve(n);
        owned.reserve(n);
        ptrs.reserve(n);
        blocks.reserve(n);
    }
    // Columns of host rows (arity-checked like Version::decompose).
    void add_rows(const std::string& rel, std::size_t arity, const std::vector<Row>& rows) {
        std::vector<std::vector<std::uint32_t>> cols(arity, std::vector<std::uint32_t>(rows.size()));
        for (std::size_t i = 0; i < rows.size(); ++i) {
            if (rows[i].size() != arity) throw std::invalid_argument("decompose: row arity mismatch");
            for (std::size_t j = 0; j < arity; ++j) cols[j][i] = rows[i][j];
        }
        owned.push_back(std::move(cols));
        push(rel, arity, rows.size(), owned.back());
    }
    // A Version's raw columns, borrowed.
    void add_version(const std::string& rel, const Version& v) {
        std::vector<const std::uint32_t*> p(v.arity());
        for (std::size_t j = 0; j < v.arity(); ++j) p[j] = v.col(j).raw().data();
        names.push_back(rel);
        ptrs.push_back(std::move(p));
        blocks.push_back(fv_facts{names.back().c_str(), static_cast<std::uint32_t>(v.arity()), v.rows(),
                                  ptrs.back().data()});
    }

private:
    void push(const std::string& rel, std::size_t arity, std::size_t n,
              const std::vector<std::vector<std::uint32_t>>& cols) {
        std::vector<const std::uint32_t*> p(arity);
        for (std::size_t j = 0; j < arity; ++j) p[j] = cols[j].data();
        names.push_back(rel);
        ptrs.push_back(std::move(p));
        blocks.push_back(fv_facts{names.back().c_str(), static_cast<std::uint32_t>(arity), n, ptrs.back().data()});
    }
};

struct StateH {
    fv_state* p = nullptr;
    StateH() = default;
    StateH(const StateH&) = delete;
    StateH& operator=(const StateH&) = delete;
    ~StateH() { fv_state_free(p); }
};

// Sorted FULL of one relation of a device state as a host Version.
Version relation_version(const fv_state* st, const char* name, std::uint32_t arity, std::uint64_t rows) {
    if (rows == 0) return Version(arity);
    std::vector<std::uint32_t> flat(rows * arity);
    check(fv_state_dump_sorted(st, name, flat.data()), "fv_state_dump_sorted");
    std::vector<std::vector<Value>> cols(arity, std::vector<Value>(rows));
    for (std::uint64_t i = 0; i < rows; ++i)
        for (std::uint32_t j = 0; j < arity; ++j) cols[j][i] = flat[i * arity + j];
    return Version::from_columns(std::move(cols), Executor(1));
}

}  // namespace

std::vector<PlanVariant> delta_rewrite(const RulePlan& plan, const std::set<std::string>& idb) {
    std::vector<PlanVariant> out;
    const std::size_t ns = plan.sources.size();
    for (std::size_t s = 0; s < ns; ++s)
        if (idb.find(plan.sources[s].relation) != idb.end()) out.push_back(PlanVariant{&plan, s});
    return out.empty() ? std::vector<PlanVariant>{PlanVariant{&plan, PlanVariant::kNoDelta}} : out;
}

std::set<std::string> idb_relations(const Program& program) {
    std::set<std::string> heads;
    for (const Rule& rule : program.rules) heads.emplace(rule.head.relation);
    return heads;
}

EvaluationState seed(const Program& program, const FactMap& facts, const Executor& exec) {
    EvaluationState st;
    for (const RelationDecl& d : program.relations) {
        Relation rel(d.name, d.arity);
        const auto f = facts.find(d.name);
        if (f != facts.end() && !f->second.empty()) {
            rel.full = dedup_rows(Version::decompose(f->second, d.arity, exec), exec);
            rel.delta = rel.full;
        }
        st.relations.emplace(d.name, std::move(rel));
    }
    return st;
}

std::vector<std::vector<Value>> execute_plan(const RulePlan& plan,
                                             const std::function<const Version&(std::size_t)>& resolve,
                                             const Executor&) {
    // Every source becomes its own EDB relation "__src<k>" holding the
    // resolved version (two occurrences of one relation may resolve to
    // different versions), the head a fresh relation: the EDB-only variant
    // of iteration 0 is exactly one application of the plan.
    const std::size_t ns = plan.sources.size();
    std::vector<std::string> names(ns);
    std::vector<fv_relation_decl> decls;
    FactBlocks fb;
    fb.reserve(ns);
    const std::string head = "__head";
    for (std::size_t s = 0; s < ns; ++s) {
        names[s] = "__src" + std::to_string(s);
        const Version& v = resolve(s);
        if (v.arity() != plan.sources[s].arity) throw std::invalid_argument("execute_plan: source arity mismatch");
        fb.add_version(names[s], v);
    }
    for (std::size_t s = 0; s < ns; ++s)
        decls.push_back(fv_relation_decl{names[s].c_str(), static_cast<std::uint32_t>(plan.sources[s].arity)});
    decls.push_back(fv_relation_decl{head.c_str(), static_cast<std::uint32_t>(plan.head_arity)});
    PodPlan pp(plan, &head, &names);
    StateH st;
    check(fv_evaluate(ctx(), decls.data(), static_cast<std::uint32_t>(decls.size()), &pp.pod(), 1,
                      fb.blocks.data(), static_cast<std::uint32_t>(fb.blocks.size()), &st.p),
          "execute_plan");
    const char* nm = nullptr;
    std::uint32_t arity = 0;
    std::uint64_t rows = 0;
    for (std::uint64_t i = 0; i < fv_state_num_relations(st.p); ++i) {
        check(fv_state_relation(st.p, i, &nm, &arity, &rows), "fv_state_relation");
        if (head == nm) break;
    }
    std::vector<std::vector<Value>> cols(plan.head_arity, std::vector<Value>(rows));
    if (rows) {
        std::vector<std::uint32_t> flat(rows * arity);
        check(fv_state_dump_sorted(st.p, head.c_str(), flat.data()), "fv_state_dump_sorted");
        for (std::uint64_t i = 0; i < rows; ++i)
            for (std::uint32_t j = 0; j < arity; ++j) cols[j][i] = flat[i * arity + j];
    }
    return cols;
}

bool run_iteration(EvaluationState& state, const std::vector<PlanVariant>& variants, std::size_t iteration,
                   const Executor& exec) {
    // Jacobi step over the iteration-start state (P/src/engine.cpp:163-220):
    // every active variant's head block is pooled per head relation, then
    // each head takes ONE dedup -> deduplicate -> difference -> merge, all on
    // the device operators.
    const auto started = std::chrono::steady_clock::now();
    std::map<std::string, std::vector<std::vector<Value>>> pool;
    for (const PlanVariant& v : variants) pool.try_emplace(v.plan->head_relation, v.plan->head_arity);
    for (const PlanVariant& v : variants) {
        if (iteration != 0 && v.edb_only()) continue;
        const RulePlan& p = *v.plan;
        const auto block = execute_plan(
            p,
            [&](std::size_t s) -> const Version& {
                const Relation& r = state.relations.at(p.sources[s].relation);
                return s == v.delta_source ? r.delta : r.full;
            },
            exec);
        auto& dst = pool.at(p.head_relation);
        for (std::size_t j = 0; j < dst.size(); ++j) dst[j].insert(dst[j].end(), block[j].begin(), block[j].end());
    }
    IterationStats its;
    its.index = iteration;
    bool grew = false;
    for (auto& [name, cols] : pool) {
        Relation& r = state.relations.at(name);
        r.new_rows = Version::from_columns(std::move(cols), exec);
        Version fresh(r.arity);
        if (!r.new_rows.empty()) {
            const Version distinct = dedup_rows(r.new_rows, exec);
            fresh = difference(distinct, deduplicate(distinct, r.full, exec), exec);
        }
        r.merge_delta(std::move(fresh), exec);
        grew = grew || !r.delta.empty();
        its.relations.push_back(RelationStats{name, r.delta.rows(), r.full.rows(), 1});
    }
    its.elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - started).count();
    state.stats.push_back(std::move(its));
    return grew;
}

EvaluationState evaluate(const Program& program, const FactMap& facts, const Executor&) {
    if (auto diags = validate_program(program); !diags.empty()) throw DiagnosticError(diags.front());
    const std::vector<RulePlan> plans = compile_program(program);
    std::vector<std::unique_ptr<PodPlan>> pods;
    std::vector<fv_plan> pod_plans;
    for (const RulePlan& p : plans) {
        pods.push_back(std::make_unique<PodPlan>(p));
        pod_plans.push_back(pods.back()->pod());
    }
    std::vector<fv_relation_decl> decls;
    FactBlocks fb;
    fb.reserve(program.relations.size());
    for (const RelationDecl& d : program.relations) {
        decls.push_back(fv_relation_decl{d.name.c_str(), static_cast<std::uint32_t>(d.arity)});
        const auto f = facts.find(d.name);
        if (f != facts.end() && !f->second.empty()) fb.add_rows(d.name, d.arity, f->second);
    }
    StateH st;
    check(fv_evaluate(ctx(), decls.data(), static_cast<std::uint32_t>(decls.size()), pod_plans.data(),
                      static_cast<std::uint32_t>(pod_plans.size()), fb.blocks.data(),
                      static_cast<std::uint32_t>(fb.blocks.size()), &st.p),
          "evaluate");

    EvaluationState out;
    out.iterations = fv_state_iterations(st.p);
    const std::set<std::string> idb = idb_relations(program);
    for (std::uint64_t i = 0; i < fv_state_num_relations(st.p); ++i) {
        const char* nm = nullptr;
        std::uint32_t arity = 0;
        std::uint64_t rows = 0;
        check(fv_state_relation(st.p, i, &nm, &arity, &rows), "fv_state_relation");
        Relation rel(nm, arity);
        rel.full = relation_version(st.p, nm, arity, rows);
        // At the fixpoint every head relation's DELTA is the final, empty
        // one; relations that are never a head keep their seed DELTA = FULL.
        if (!idb.count(nm)) rel.delta = rel.full;
        out.relations.emplace(rel.name, std::move(rel));
    }
    for (std::uint64_t i = 0; i < fv_state_num_stats(st.p); ++i) {
        std::uint64_t it = 0, delta = 0, full = 0, merges = 0;
        const char* rel = nullptr;
        double ms = 0.0;
        check(fv_state_stat(st.p, i, &it, &rel, &delta, &full, &merges, &ms), "fv_state_stat");
        if (out.stats.empty() || out.stats.back().index != it) {
            out.stats.emplace_back();
            out.stats.back().index = it;
            out.stats.back().elapsed_ms = ms;
        }
        out.stats.back().relations.push_back(RelationStats{rel, delta, full, merges});
    }
    return out;
}

}  // namespace colog

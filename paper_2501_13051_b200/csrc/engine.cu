// Host driver of the device-resident semi-naive engine.
//
// Reference semantics reproduced (P/src/engine.cpp):
//   delta_rewrite (:57-64)   one variant per IDB body occurrence; variant i
//                            reads DELTA at occurrence i and FULL elsewhere;
//                            rules without IDB atoms get one run-once variant
//   seed (:148-161)          FULL = DELTA = dedup(EDB facts)
//   run_iteration (:163-220) Jacobi: every variant sees the iteration-start
//                            state; EDB-only variants run in iteration 0
//                            only; then ONE dedup+merge per head relation
//   evaluate (:222-239)      iterations counts the final empty iteration
// What changes is where the data lives and how each step executes: all
// relation versions stay in HBM as sorted SoA columns, a join step is
// probe/count -> scan -> fused materialize, and dedup/difference/merge is one
// radix sort plus one merge-path pass. The host reads back one scalar per
// join step (its output size, to allocate) and one per head relation per
// iteration (|DELTA|, the fixpoint test).
#include <algorithm>
#include <chrono>
#include <set>

#include "engine.h"
#include "prim.cuh"
#include "radix_sort.h"

namespace fv {

namespace {

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// Growable candidate pool of packed row keys for one head relation.
struct CandPool {
    u32 arity = 0;
    u64 n = 0, cap = 0;
    std::vector<DBuf<u64>> words;

    void reserve(Ctx* c, u64 extra) {
        const u32 W = (arity + 1) / 2;
        if (words.empty()) words.resize(W);
        if (n + extra <= cap) return;
        u64 nc = std::max<u64>(n + extra, cap * 2);
        for (u32 w = 0; w < W; ++w) {
            DBuf<u64> nb(c, nc);
            if (n) FV_CUDA(cudaMemcpyAsync(nb.get(), words[w].get(), 8 * n, cudaMemcpyDeviceToDevice, c->stream));
            words[w] = std::move(nb);
        }
        cap = nc;
    }
};

struct Inter {
    u64 n = 0;
    std::map<ColRef, const u32*> cols;
    std::vector<DBuf<u32>> owned;
};

class Engine {
public:
    Engine(Ctx* c, EvalState& st) : c_(c), st_(st) {}

    RelState& rel(const std::string& name) { return *st_.relations.at(name); }

    JoinIndex& index(RelState& r, bool delta, u32 col) {
        auto key = std::make_pair(delta ? 1 : 0, col);
        auto it = r.indexes.find(key);
        if (it != r.indexes.end()) return *it->second;
        auto idx = std::make_unique<JoinIndex>();
        build_index_on(delta ? r.delta : r.full, col, *idx, nullptr);
        JoinIndex& ref = *idx;
        r.indexes.emplace(key, std::move(idx));
        return ref;
    }

    // Index over `ver` (or its rows passing the source constraints) keyed
    // on column `col`.
    void build_index_on(const DevVersion& ver, u32 col, JoinIndex& idx, const PlanSource* constrained) {
        const DevVersion* base = &ver;
        DevVersion filtered;
        if (constrained) {
            RowFilter pred = source_filter(*constrained, ver);
            DBuf<u32> ids(c_, std::max<u64>(ver.n, 1));
            const u64 k = engine_select_rows(c_, ver.n, pred, ids.get());
            filtered.n = k;
            for (auto& col_buf : ver.cols) {
                DBuf<u32> g(c_, k);
                gather_u32(c_, col_buf.get(), ids.get(), g.get(), k);
                filtered.cols.push_back(std::move(g));
            }
            base = &filtered;
        }
        if (col == 0) {
            if (constrained) {
                idx.owned = std::move(filtered);
                idx.rows = &idx.owned;
            } else {
                idx.rows = &ver;
            }
        } else {
            // Sorted copy keyed on `col` (ties by the remaining columns).
            const u32 arity = static_cast<u32>(base->cols.size());
            std::vector<const u32*> order_cols{base->cols[col].get()};
            for (u32 j = 0; j < arity; ++j)
                if (j != col) order_cols.push_back(base->cols[j].get());
            DBuf<u32> perm = lexicographic_order(c_, order_cols.data(), arity, base->n);
            DevVersion sorted;
            sorted.n = base->n;
            for (u32 j = 0; j < arity; ++j) {
                DBuf<u32> g(c_, base->n);
                gather_u32(c_, base->cols[j].get(), perm.get(), g.get(), base->n);
                sorted.cols.push_back(std::move(g));
            }
            idx.owned = std::move(sorted);
            idx.rows = &idx.owned;
        }
        engine_build_runs(c_, idx.rows->cols[col].get(), idx.rows->n, idx);
    }

    RowFilter source_filter(const PlanSource& s, const DevVersion& v) {
        RowFilter f;
        for (auto& [col, val] : s.const_selects) push(f, Filter{{v.cols[col].get(), 0}, {}, kFilterConst, val});
        for (auto& [a, b] : s.self_eqs)
            push(f, Filter{{v.cols[a].get(), 0}, {v.cols[b].get(), 0}, kFilterEq, 0});
        return f;
    }

    static void push(RowFilter& f, const Filter& x) {
        if (f.n >= static_cast<u32>(kMaxFilters)) fail(FV_ERR_PLAN, "rule needs more than 8 filters");
        f.f[f.n++] = x;
    }
    static void push(OutSpec& s, const Filter& x) {
        if (s.n_filters >= static_cast<u32>(kMaxFilters)) fail(FV_ERR_PLAN, "rule needs more than 8 filters");
        s.f[s.n_filters++] = x;
    }

    // execute_plan (P/src/engine.cpp:72-146) for one variant, appending the
    // head rows as packed keys to `out`.
    void exec_variant(const Plan& plan, long delta_source, CandPool& out) {
        const u32 ns = static_cast<u32>(plan.sources.size());
        std::vector<const DevVersion*> ver(ns);
        for (u32 s = 0; s < ns; ++s) {
            RelState& r = rel(plan.sources[s].relation);
            ver[s] = (static_cast<long>(s) == delta_source) ? &r.delta : &r.full;
            if (ver[s]->n == 0) return;  // engine.cpp:76-78
        }
        Inter cur;
        cur.n = ver[0]->n;
        for (u32 j = 0; j < plan.sources[0].arity; ++j) cur.cols[ColRef{0, j}] = ver[0]->cols[j].get();
        const bool src0_pending = plan.sources[0].constrained();

        // Columns still needed after join step k.
        const size_t nj = plan.joins.size();
        std::vector<std::set<ColRef>> needed(nj);
        for (size_t k = 0; k < nj; ++k) {
            std::set<ColRef>& s = needed[k];
            for (size_t q = k + 1; q < nj; ++q) {
                s.insert(plan.joins[q].left);
                for (auto& r : plan.joins[q].residual_eq) s.insert(r.first);
            }
            for (auto& r : plan.output_cols) s.insert(r);
        }
        const u32 W = (plan.head_arity + 1) / 2;

        for (size_t k = 0; k < nj; ++k) {
            const PlanJoin& jn = plan.joins[k];
            const u32 R = jn.right_source;
            RelState& rr = rel(plan.sources[R].relation);
            std::unique_ptr<JoinIndex> tmp;
            JoinIndex* idx;
            if (plan.sources[R].constrained()) {
                tmp = std::make_unique<JoinIndex>();
                build_index_on(*ver[R], jn.right_col, *tmp, &plan.sources[R]);
                idx = tmp.get();
            } else {
                idx = &index(rr, static_cast<long>(R) == delta_source, jn.right_col);
            }
            if (idx->rows->n == 0) return;
            const u64 n = cur.n;
            DBuf<u32> starts(c_, n), counts(c_, n);
            RowFilter pred;
            if (k == 0 && src0_pending) pred = source_filter(plan.sources[0], *ver[0]);
            engine_probe_count(c_, cur.cols.at(jn.left), n, *idx, pred, starts.get(), counts.get());
            DBuf<u64> offsets(c_, n + 1);
            exclusive_scan_counts(c_, counts.get(), offsets.get(), n);
            u64 T = 0;
            FV_CUDA(cudaMemcpyAsync(c_->pinned, offsets.get() + n, 8, cudaMemcpyDeviceToHost, c_->stream));
            c_->sync();
            T = c_->pinned[0];
            counts.reset();
            if (T == 0) return;

            const bool last = k + 1 == nj;
            auto slot_of = [&](const ColRef& r) -> SlotRef {
                if (r.source == R) return SlotRef{idx->rows->cols[r.col].get(), 1};
                auto it = cur.cols.find(r);
                if (it == cur.cols.end()) fail(FV_ERR_PLAN, "plan references an unbound column");
                return SlotRef{it->second, 0};
            };
            OutSpec spec;
            spec.shift = st_.key_shift;
            for (auto& [lref, rcol] : jn.residual_eq)
                push(spec, Filter{slot_of(lref), SlotRef{idx->rows->cols[rcol].get(), 1}, kFilterEq, 0});
            Inter next;
            if (last) {
                for (auto& [ga, gb] : plan.guard_neq)
                    push(spec, Filter{slot_of(plan.output_cols[ga]), slot_of(plan.output_cols[gb]), kFilterNeq, 0});
                spec.key_mode = 1;
                spec.n_out = plan.head_arity;
                for (u32 h = 0; h < plan.head_arity; ++h) spec.col[h] = slot_of(plan.output_cols[h]);
                out.reserve(c_, T);
                for (u32 w = 0; w < W; ++w) spec.keys[w] = out.words[w].get() + out.n;
            } else {
                spec.key_mode = 0;
                u32 j = 0;
                for (const ColRef& r : needed[k]) {
                    if (r.source > R) continue;
                    if (j >= static_cast<u32>(kMaxSlots)) fail(FV_ERR_PLAN, "join intermediate wider than 16 columns");
                    spec.col[j] = slot_of(r);
                    next.owned.emplace_back(c_, T);
                    spec.out_cols[j] = next.owned.back().get();
                    next.cols[r] = spec.out_cols[j];
                    ++j;
                }
                spec.n_out = j;
            }
            if (spec.n_filters) {
                spec.d_count = c_->d_scalars + 20;
                FV_CUDA(cudaMemsetAsync(spec.d_count, 0, 8, c_->stream));
            }
            engine_materialize(c_, offsets.get(), n, T, starts.get(), spec);
            u64 produced = T;
            if (spec.n_filters) c_->read_scalars(spec.d_count, &produced, 1);
            if (last) {
                out.n += produced;
                return;
            }
            next.n = produced;
            cur = std::move(next);
            if (cur.n == 0) return;
        }
        // No joins: a single-atom rule (copy / projection / selection).
        OutSpec spec;
        spec.shift = st_.key_shift;
        if (src0_pending) {
            RowFilter f = source_filter(plan.sources[0], *ver[0]);
            for (u32 q = 0; q < f.n; ++q) push(spec, f.f[q]);
        }
        auto slot0 = [&](const ColRef& r) { return SlotRef{ver[0]->cols[r.col].get(), 0}; };
        for (auto& [ga, gb] : plan.guard_neq)
            push(spec, Filter{slot0(plan.output_cols[ga]), slot0(plan.output_cols[gb]), kFilterNeq, 0});
        spec.key_mode = 1;
        spec.n_out = plan.head_arity;
        for (u32 h = 0; h < plan.head_arity; ++h) spec.col[h] = slot0(plan.output_cols[h]);
        out.reserve(c_, cur.n);
        for (u32 w = 0; w < W; ++w) spec.keys[w] = out.words[w].get() + out.n;
        if (spec.n_filters) {
            spec.d_count = c_->d_scalars + 20;
            FV_CUDA(cudaMemsetAsync(spec.d_count, 0, 8, c_->stream));
        }
        engine_project(c_, cur.n, spec);
        u64 produced = cur.n;
        if (spec.n_filters) c_->read_scalars(spec.d_count, &produced, 1);
        out.n += produced;
    }

    // Sort candidates and fold them into FULL; returns |DELTA|.
    u64 dedup_merge(RelState& r, CandPool& cand) {
        const u32 arity = r.arity;
        if (cand.n == 0) {
            r.delta = DevVersion();
            r.delta.n = 0;
            r.delta.cols.resize(arity);
            r.indexes.clear();
            return 0;
        }
        engine_sort_keys(c_, cand.words, cand.n, arity, st_.key_shift);
        DevVersion C, D;
        for (u32 j = 0; j < arity; ++j) {
            C.cols.emplace_back(c_, r.full.n + cand.n);
            D.cols.emplace_back(c_, cand.n);
        }
        std::vector<u64*> bw;
        for (auto& w : cand.words) bw.push_back(w.get());
        std::vector<u32*> cc, dc;
        for (u32 j = 0; j < arity; ++j) {
            cc.push_back(C.cols[j].get());
            dc.push_back(D.cols[j].get());
        }
        u64* d_new = c_->d_scalars + 21;
        engine_merge(c_, r.full.ptrs(), r.full.n, bw.data(), cand.n, arity, st_.key_shift, cc, dc, d_new);
        u64 nd = 0;
        c_->read_scalars(d_new, &nd, 1);
        c_->prof_add_bytes("merge_dedup", 8.0 * double(nd) * arity);
        C.n = r.full.n + nd;
        D.n = nd;
        r.full = std::move(C);
        r.delta = std::move(D);
        r.indexes.clear();
        return nd;
    }

private:
    Ctx* c_;
    EvalState& st_;
};

}  // namespace

void check_plans(const std::vector<RelationDecl>& decls, const std::vector<Plan>& plans) {
    std::map<std::string, u32> ar;
    for (auto& d : decls) {
        if (d.arity == 0 || d.arity > FV_MAX_ARITY)
            fail(FV_ERR_ARITY, "relation '" + d.name + "' has unsupported arity " + std::to_string(d.arity));
        ar[d.name] = d.arity;
    }
    for (auto& p : plans) {
        auto bad = [&](const std::string& m) { fail(FV_ERR_PLAN, "plan for '" + p.head + "': " + m); };
        if (!ar.count(p.head) || ar[p.head] != p.head_arity) bad("head relation not declared with this arity");
        if (p.sources.empty()) bad("no body atoms");
        if (p.joins.size() + 1 != p.sources.size()) bad("joins must attach sources 1..n-1 in order");
        for (auto& s : p.sources) {
            if (!ar.count(s.relation) || ar[s.relation] != s.arity) bad("source '" + s.relation + "' arity mismatch");
            for (auto& [c, v] : s.const_selects)
                if (c >= s.arity) bad("constant select column out of range");
            for (auto& [a, b] : s.self_eqs)
                if (a >= s.arity || b >= s.arity) bad("self equality column out of range");
        }
        auto ref_ok = [&](const ColRef& r, u32 max_source) {
            return r.source <= max_source && r.col < p.sources[r.source].arity;
        };
        for (size_t k = 0; k < p.joins.size(); ++k) {
            auto& j = p.joins[k];
            if (j.right_source != k + 1) bad("joins[k] must attach sources[k+1]");
            if (!ref_ok(j.left, static_cast<u32>(k)) || j.right_col >= p.sources[j.right_source].arity)
                bad("join column out of range");
            for (auto& [l, rc] : j.residual_eq)
                if (!ref_ok(l, static_cast<u32>(k)) || rc >= p.sources[j.right_source].arity)
                    bad("residual equality column out of range");
        }
        if (p.output_cols.size() < p.head_arity) bad("fewer output columns than head arity");
        for (auto& r : p.output_cols)
            if (!ref_ok(r, static_cast<u32>(p.sources.size() - 1))) bad("output column out of range");
        for (auto& [a, b] : p.guard_neq)
            if (a >= p.output_cols.size() || b >= p.output_cols.size()) bad("guard slot out of range");
    }
}

DeviceEdb upload_facts(Ctx* c, const std::vector<RelationDecl>& decls, const std::vector<FactsBlock>& facts) {
    std::map<std::string, u32> arity;
    for (auto& d : decls) arity[d.name] = d.arity;
    std::map<std::string, std::vector<const FactsBlock*>> by_rel;
    for (auto& f : facts) {
        auto it = arity.find(f.relation);
        if (it == arity.end()) continue;  // facts for undeclared relations are ignored
        if (f.arity != it->second) fail(FV_ERR_ARITY, "facts for '" + f.relation + "' have the wrong arity");
        by_rel[f.relation].push_back(&f);
    }
    DeviceEdb edb;
    for (auto& [name, blocks] : by_rel) {
        u64 n = 0;
        for (auto* b : blocks) n += b->n;
        if (n == 0) continue;
        DevVersion v;
        v.n = n;
        for (u32 j = 0; j < arity[name]; ++j) {
            DBuf<u32> col(c, n);
            u64 off = 0;
            for (auto* b : blocks) {
                col.upload(b->cols[j], b->n, off);
                off += b->n;
            }
            v.cols.push_back(std::move(col));
        }
        edb.rels.emplace(name, std::move(v));
    }
    return edb;
}

std::unique_ptr<EvalState> evaluate(Ctx* c, const std::vector<RelationDecl>& decls,
                                    const std::vector<Plan>& plans, const std::vector<FactsBlock>& facts) {
    check_plans(decls, plans);
    const auto t0 = Clock::now();
    DeviceEdb edb = upload_facts(c, decls, facts);
    auto st = evaluate_device(c, decls, plans, {&edb});
    st->elapsed_ms = ms_since(t0);
    return st;
}

std::unique_ptr<EvalState> evaluate_device(Ctx* c, const std::vector<RelationDecl>& decls,
                                           const std::vector<Plan>& plans,
                                           const std::vector<const DeviceEdb*>& edbs) {
    check_plans(decls, plans);
    const auto t0 = Clock::now();
    auto st = std::make_unique<EvalState>();
    st->ctx = c;
    std::set<std::string> idb;
    for (auto& p : plans) idb.insert(p.head);
    for (auto& d : decls) {
        auto r = std::make_unique<RelState>();
        r->name = d.name;
        r->arity = d.arity;
        r->idb = idb.count(d.name) > 0;
        r->full.cols.resize(d.arity);
        r->delta.cols.resize(d.arity);
        st->relations[d.name] = std::move(r);
    }

    // ---- gather the resident EDB blocks, key shift from the active domain ----
    std::map<std::string, std::vector<const DevVersion*>> by_rel;
    for (const DeviceEdb* e : edbs)
        for (auto& [name, v] : e->rels) {
            auto it = st->relations.find(name);
            if (it == st->relations.end() || v.n == 0) continue;
            if (v.cols.size() != it->second->arity) fail(FV_ERR_ARITY, "facts for '" + name + "' have the wrong arity");
            by_rel[name].push_back(&v);
        }
    std::map<std::string, DevVersion> concat;  // only for relations with several blocks
    std::map<std::string, const DevVersion*> raw;
    for (auto& [name, blocks] : by_rel) {
        if (blocks.size() == 1) {
            raw[name] = blocks[0];
            continue;
        }
        u64 n = 0;
        for (auto* b : blocks) n += b->n;
        DevVersion v;
        v.n = n;
        for (u32 j = 0; j < st->relations[name]->arity; ++j) {
            DBuf<u32> col(c, n);
            u64 off = 0;
            for (auto* b : blocks) {
                FV_CUDA(cudaMemcpyAsync(col.get() + off, b->cols[j].get(), 4 * b->n, cudaMemcpyDeviceToDevice,
                                        c->stream));
                off += b->n;
            }
            v.cols.push_back(std::move(col));
        }
        raw[name] = &concat.emplace(name, std::move(v)).first->second;
    }
    u64 vmax = 0;
    for (auto& p : plans)
        for (auto& s : p.sources)
            for (auto& cs : s.const_selects) vmax = std::max<u64>(vmax, cs.second);
    u64* dmax = c->d_scalars + 22;
    for (auto& [name, vp] : raw) {
        const DevVersion& v = *vp;
        for (auto& col : v.cols) {
            reduce_max_u32(c, col.get(), v.n, dmax);
            u64 m = 0;
            c->read_scalars(dmax, &m, 1);
            vmax = std::max(vmax, m);
        }
    }
    st->key_shift = std::max<u32>(1, bit_width_u64(vmax));

    Engine eng(c, *st);
    // ---- seed: FULL = DELTA = dedup(EDB) (engine.cpp:148-161) ---------------
    for (auto& [name, vp] : raw) {
        const DevVersion& v = *vp;
        RelState& r = *st->relations[name];
        CandPool pool;
        pool.arity = r.arity;
        pool.reserve(c, v.n);
        std::vector<u64*> wp;
        for (auto& w : pool.words) wp.push_back(w.get());
        engine_pack_keys(c, v.ptrs(), v.n, st->key_shift, wp.data());
        pool.n = v.n;
        eng.dedup_merge(r, pool);  // FULL empty: C = D = distinct rows
        // DELTA must equal FULL; the merge produced two identical copies.
    }
    raw.clear();
    concat.clear();

    // ---- variants (delta_rewrite, engine.cpp:57-64) --------------------------
    struct Variant {
        const Plan* plan;
        long delta_source;
    };
    std::vector<Variant> variants;
    for (auto& p : plans) {
        bool any = false;
        for (size_t s = 0; s < p.sources.size(); ++s)
            if (idb.count(p.sources[s].relation)) {
                variants.push_back({&p, static_cast<long>(s)});
                any = true;
            }
        if (!any) variants.push_back({&p, -1});
    }

    // ---- fixpoint (engine.cpp:163-239) ---------------------------------------
    u64 iteration = 0;
    for (;;) {
        const auto ti = Clock::now();
        std::map<std::string, CandPool> pooled;
        for (auto& v : variants) pooled[v.plan->head].arity = v.plan->head_arity;
        for (auto& v : variants) {
            if (v.delta_source < 0 && iteration != 0) continue;
            eng.exec_variant(*v.plan, v.delta_source, pooled[v.plan->head]);
        }
        bool any_delta = false;
        std::vector<IterStat> its;
        for (auto& [name, pool] : pooled) {
            RelState& r = *st->relations.at(name);
            const u64 nd = eng.dedup_merge(r, pool);
            if (nd) any_delta = true;
            its.push_back({iteration, name, nd, r.full.n, 1, 0.0});
        }
        const double ms = ms_since(ti);
        for (auto& s : its) {
            s.elapsed_ms = ms;
            st->stats.push_back(s);
        }
        if (!any_delta) break;
        ++iteration;
    }
    st->iterations = iteration + 1;
    c->sync();
    st->elapsed_ms = ms_since(t0);
    return st;
}

std::vector<u32> dump_sorted(const EvalState& s, const std::string& rel) {
    auto it = s.relations.find(rel);
    if (it == s.relations.end()) fail(FV_ERR_RANGE, "unknown relation '" + rel + "'");
    const RelState& r = *it->second;
    std::vector<u32> rows(r.full.n * r.arity), col(r.full.n);
    for (u32 j = 0; j < r.arity; ++j) {
        r.full.cols[j].download(col.data(), r.full.n);
        for (u64 i = 0; i < r.full.n; ++i) rows[i * r.arity + j] = col[i];
    }
    return rows;
}

u64 fingerprint(const EvalState& s, const std::string& rel) {
    auto it = s.relations.find(rel);
    if (it == s.relations.end()) fail(FV_ERR_RANGE, "unknown relation '" + rel + "'");
    const RelState& r = *it->second;
    return engine_fingerprint(s.ctx, r.full.ptrs(), r.full.n, r.arity);
}

}  // namespace fv

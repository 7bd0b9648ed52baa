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
//
// Partitioned evaluation (Ctx::tx != null, world > 1):
//   - EDB-only relations are replicated on every rank;
//   - every IDB relation is hash-partitioned: the home copy holds the rows
//     with owner(hash(col 0)) == rank; a relation probed on column c (as a
//     join's right atom, or as a rule's first atom joined on c) also keeps a
//     copy partitioned on c (keyset, derived statically from the plans);
//   - a join step whose right atom is partitioned needs its probe rows on the
//     owner of the probe value: intermediates that are replicated (all EDB so
//     far) or already partitioned on the probe column join locally, others
//     are shuffled by the probe value first;
//   - head rows of a replicated derivation are owner-filtered; all others are
//     routed to owner(head col 0) by ONE all-to-all per head per iteration;
//   - after the local dedup/merge, the new Δ rows are forwarded to the other
//     partition copies; |Δ| and |FULL| are all-reduced (termination + stats).
// Every collective depends only on plan structure, so all ranks issue the
// same sequence (no data-dependent early exits in partitioned mode).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <deque>
#include <set>
#include <thread>

#include "engine.h"
#include "prim.cuh"
#include "radix_sort.h"
#include "transport.h"
#include "tsv.h"

namespace fv {

namespace {

using Clock = std::chrono::steady_clock;

#ifndef FV_KEYSET_GROWTH
#define FV_KEYSET_GROWTH 4
#endif
// New key-set capacity >= kKeysetGrowth x the worst-case key count.
constexpr u64 kKeysetGrowth = FV_KEYSET_GROWTH;

// Pooled (unfused) candidates: rows per join chunk, and the pool size that
// triggers a sort-unique compaction before the next chunk (FVLOG_POOL_BUDGET
// and FVLOG_POOL_CHUNK, in rows, override both — tests use tiny values).
constexpr u64 kPoolChunk = u64(1) << 27;
// Join intermediates larger than this are carried through the rest of the
// chain chunk by chunk (FVLOG_INTER_CHUNK overrides).
constexpr u64 kInterChunk = u64(1) << 28;
constexpr u64 kPoolBudget = u64(1) << 29;

// Join outputs per fused join+dedup launch (see exec_variant).
constexpr u64 kFusedChunk = u64(1) << 28;

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

// Per head relation per iteration in hash mode: the keys found new so far
// (appended by the fused join kernel or by hash_insert over a pool).
struct HeadSink {
    DBuf<u64> keys;
    u64 cap = 0;
    u64 bound = 0;  // host upper bound of the device count
    DBuf<u64> counter;   // [0] new keys, [1] overflow keys (block sets), [2] new tuples (word form)
    u64 candidates = 0;  // rows offered to the key set this iteration
    // Block sets: keys the set could not place (drained before every chunk).
    DBuf<u64> ovf;
    u64 ovf_cap = 0;
    // Word form: the merged masks of `keys` (at finalize), the masks of `ovf`
    // entries, the bitmap word index of each `keys` entry (recorded at
    // append; valid while the directory generation is still gen0).
    DBuf<u32> bits, ovf_bits, widx;
    u64 gen0 = ~u64(0);
    u64 chunk_blocks0 = 0, chunk_cands = 0;  // growth-ratio bookkeeping
    u64 tuples = 0;                          // host copy of counter[2] (last read)
    // Counters (new, overflow, tuples, blocks) already read with another
    // scalar (the join's output count, or known zero for a fresh sink):
    // the next read_block_counters uses them instead of a sync.
    bool pre = false;
    u64 pre_vals[4] = {0, 0, 0, 0};
};

// Block sets (BlockSet, engine.h): a relation falls back to a key set when
// its directory would need more than kBlockSparseFactor x the bytes of the
// equivalent key set and more than kBlockSparseMinBytes (FVLOG_SET=keyset
// uses key sets throughout).
constexpr double kBlockSparseFactor = 8.0;
constexpr double kBlockSparseMinBytes = 1e9;
constexpr u64 kBlockMinCap = u64(1) << 12;
std::vector<const DevVersion*> levels_of(const RelState& r);

// Key-set layout choice (KeySet::group_bits, see keyset_home in
// engine_kernels.cu): group pairs of adjacent keys while a relation's
// candidates are (almost) all new rows (<= kGroupedRatio candidates per new row in
// the last iteration), scatter every key otherwise. FVLOG_KEYSET_GROUP=0/1
// forces one layout; FVLOG_GROUP_RATIO overrides the threshold (1.05-1.2
// measured equal; 1.5 switches TC one iteration too late).
constexpr double kGroupedRatio = 1.1;

}  // namespace

// Delta-first join order for one semi-naive variant (engine decision, not
// part of the reference's plan semantics: the variant's result set does not
// depend on the join order). compile_rule orders a rule's atoms left to right
// (P/src/compiler.cpp:19-96), so a variant whose DELTA atom is not first
// joins FULL x FULL before touching DELTA — e.g. CSPA's valueAlias(x,y) :-
// valueFlow(z,x), memoryAlias(z,w), valueFlow(w,y) with DELTA at the third
// atom materializes every (x,w) pair of the two FULL relations each
// iteration. Here the DELTA source goes first and the others follow in their
// original order as soon as they share a variable with the joined prefix;
// every equality of the rule (join keys, residuals, self-equalities) is
// re-derived from the variable classes. Returns false (p unchanged) when no
// such connected order exists.
bool delta_first_plan(const Plan& p, u32 d, Plan& out, std::vector<u32>* order_out) {
    const u32 ns = static_cast<u32>(p.sources.size());
    if (d == 0 || d >= ns) return false;
    std::vector<u32> base(ns + 1, 0);
    for (u32 s = 0; s < ns; ++s) base[s + 1] = base[s] + p.sources[s].arity;
    std::vector<u32> parent(base[ns]);
    for (u32 i = 0; i < parent.size(); ++i) parent[i] = i;
    std::function<u32(u32)> find = [&](u32 x) { return parent[x] == x ? x : parent[x] = find(parent[x]); };
    auto unite = [&](u32 a, u32 b) { parent[find(a)] = find(b); };
    auto node = [&](const ColRef& r) { return base[r.source] + r.col; };
    for (u32 k = 0; k < p.joins.size(); ++k) {
        const PlanJoin& j = p.joins[k];
        unite(node(j.left), base[j.right_source] + j.right_col);
        for (auto& [l, rc] : j.residual_eq) unite(node(l), base[j.right_source] + rc);
    }
    for (u32 s = 0; s < ns; ++s)
        for (auto& [a, b] : p.sources[s].self_eqs) unite(base[s] + a, base[s] + b);
    std::vector<u32> order{d};
    std::vector<bool> used(ns, false);
    used[d] = true;
    std::map<u32, ColRef> rep;  // class -> first joined occurrence (new numbering)
    for (u32 c = 0; c < p.sources[d].arity; ++c) rep.emplace(find(base[d] + c), ColRef{0, c});
    out = Plan();
    out.head = p.head;
    out.head_arity = p.head_arity;
    out.sources.push_back(p.sources[d]);
    while (order.size() < ns) {
        bool found = false;
        for (u32 t = 0; t < ns && !found; ++t) {
            if (used[t]) continue;
            PlanJoin jn;
            bool have_key = false;
            for (u32 c = 0; c < p.sources[t].arity; ++c) {
                auto it = rep.find(find(base[t] + c));
                if (it == rep.end()) continue;
                if (!have_key) {
                    jn.left = it->second;
                    jn.right_col = c;
                    have_key = true;
                } else {
                    jn.residual_eq.emplace_back(it->second, c);
                }
            }
            if (!have_key) continue;
            const u32 pos = static_cast<u32>(order.size());
            jn.right_source = pos;
            for (u32 c = 0; c < p.sources[t].arity; ++c) rep.emplace(find(base[t] + c), ColRef{pos, c});
            out.sources.push_back(p.sources[t]);
            out.joins.push_back(std::move(jn));
            order.push_back(t);
            used[t] = true;
            found = true;
        }
        if (!found) return false;  // no connected order (cross product)
    }
    std::vector<u32> new_of(ns);
    for (u32 i = 0; i < ns; ++i) new_of[order[i]] = i;
    if (order_out) *order_out = order;
    for (const ColRef& r : p.output_cols) out.output_cols.push_back(ColRef{new_of[r.source], r.col});
    out.guard_neq = p.guard_neq;
    return true;
}

namespace {

// Union-find over a plan's column references (source, col): the variable
// classes the plan's join keys, residual and self equalities induce.
struct VarClasses {
    std::vector<u32> base, parent;
    explicit VarClasses(const Plan& p) {
        const u32 ns = static_cast<u32>(p.sources.size());
        base.assign(ns + 1, 0);
        for (u32 s = 0; s < ns; ++s) base[s + 1] = base[s] + p.sources[s].arity;
        parent.resize(base[ns]);
        for (u32 i = 0; i < parent.size(); ++i) parent[i] = i;
        for (const PlanJoin& j : p.joins) {
            unite(node(j.left), base[j.right_source] + j.right_col);
            for (auto& [l, rc] : j.residual_eq) unite(node(l), base[j.right_source] + rc);
        }
        for (u32 s = 0; s < ns; ++s)
            for (auto& [a, b] : p.sources[s].self_eqs) unite(base[s] + a, base[s] + b);
    }
    u32 node(const ColRef& r) const { return base[r.source] + r.col; }
    u32 find(u32 x) {
        while (parent[x] != x) x = parent[x] = parent[parent[x]];
        return x;
    }
    void unite(u32 a, u32 b) { parent[find(a)] = find(b); }
    bool same(const ColRef& a, const ColRef& b) { return find(node(a)) == find(node(b)); }
};

}  // namespace

std::map<std::string, u32> choose_home_cols(const std::vector<std::pair<const Plan*, long>>& variants,
                                            const std::map<std::string, u32>& idb_arity) {
    std::map<std::string, u32> home;
    for (auto& [name, a] : idb_arity) home[name] = 0;
    const char* e = std::getenv("FVLOG_HOME_COL");
    if (e && std::string(e) == "0") return home;
    std::map<std::string, std::vector<u32>> score;
    for (auto& [p, d] : variants) {
        if (d < 0 || p->sources[d].relation != p->head) continue;
        const u32 a = p->head_arity;
        if (a > 2) continue;  // packed-key routing covers columns 0 and 1
        VarClasses vc(*p);
        auto& sc = score[p->head];
        sc.resize(a, 0);
        for (u32 c = 0; c < a; ++c)
            if (vc.same(p->output_cols[c], ColRef{static_cast<u32>(d), c})) ++sc[c];
    }
    for (auto& [name, sc] : score) {
        u32 best = 0;
        for (u32 c = 1; c < sc.size(); ++c)
            if (sc[c] > sc[best]) best = c;
        home[name] = best;
    }
    return home;
}

DistPlan dist_plan(const Plan& p, const std::set<std::string>& idb, const std::map<std::string, u32>& home) {
    DistPlan d;
    const u32 ns = static_cast<u32>(p.sources.size());
    d.src_copy.assign(ns, 0);
    auto is_idb = [&](u32 s) { return idb.count(p.sources[s].relation) > 0; };
    auto home_of = [&](const std::string& rel) {
        auto it = home.find(rel);
        return it == home.end() ? 0u : it->second;
    };
    // `key`: column references whose value the intermediate is partitioned
    // on (every row sits on owner(value)); empty while it is replicated.
    std::set<ColRef> key;
    auto extend = [&](const ColRef& a, const ColRef& b) {
        if (key.count(a)) key.insert(b);
        else if (key.count(b)) key.insert(a);
    };
    if (is_idb(0)) {
        // Co-partitioned with the first join's right atom when that is
        // partitioned too; otherwise the home copy serves any replicated join.
        const bool co = !p.joins.empty() && is_idb(p.joins[0].right_source);
        d.src_copy[0] = co ? p.joins[0].left.col : home_of(p.sources[0].relation);
        key.insert(ColRef{0, d.src_copy[0]});
    }
    for (u32 s = 0; s < ns && !key.empty(); ++s)
        for (auto& [a, b] : p.sources[s].self_eqs) extend(ColRef{s, a}, ColRef{s, b});
    for (const PlanJoin& jn : p.joins) {
        const u32 R = jn.right_source;
        u8 sh = 0;
        if (is_idb(R)) {
            if (key.empty()) {
                // Replicated intermediate x partitioned atom: read the home
                // copy; the result is partitioned like it.
                d.src_copy[R] = home_of(p.sources[R].relation);
                key.insert(ColRef{R, d.src_copy[R]});
            } else {
                d.src_copy[R] = jn.right_col;
                if (!key.count(jn.left)) {
                    sh = 1;
                    key.clear();
                    key.insert(jn.left);
                }
            }
        }
        d.shuffle.push_back(sh);
        if (key.empty()) continue;
        extend(jn.left, ColRef{R, jn.right_col});
        for (auto& [l, rc] : jn.residual_eq) extend(l, ColRef{R, rc});
        for (auto& [a, b] : p.sources[R].self_eqs) extend(ColRef{R, a}, ColRef{R, b});
    }
    d.replicated_out = key.empty();
    d.local_out = !key.empty() && key.count(p.output_cols[home_of(p.head)]) > 0;
    return d;
}

namespace {

class Engine {
public:
    Engine(Ctx* c, EvalState& st) : c_(c), st_(st) {
        if (c->tx) {
            world_ = static_cast<u32>(c->tx->world());
            rank_ = static_cast<u32>(c->tx->rank());
            const char* e = std::getenv("FVLOG_FORCE_PARTITIONED");
            force_partitioned_ = e && std::string(e) == "1";
        }
    }

    // FVLOG_FORCE_PARTITIONED=1 runs the partitioned path even with one
    // rank (a context with a transport), so the NCCL code path — routing,
    // grouped send/recv, all-reduce — is exercised on a single GPU.
    bool dist() const { return world_ > 1 || force_partitioned_; }
    bool partitioned(const RelState& r) const { return dist() && r.idb; }
    RelState& rel(const std::string& name) { return *st_.relations.at(name); }

    // Copy kc of a relation: its rows partitioned on column kc (the home
    // copy when kc is the relation's home column; always on one GPU).
    DevVersion& vfull(RelState& r, u32 kc) { return kc != r.home ? r.copies.at(kc)->full : r.full; }
    DevVersion& vdelta(RelState& r, u32 kc) { return kc != r.home ? r.copies.at(kc)->delta : r.delta; }
    IndexMap& vindexes(RelState& r, u32 kc) { return kc != r.home ? r.copies.at(kc)->indexes : r.indexes; }

    // FULL - DELTA of the home copy (see RelState::full_old).
    DevVersion& vold(RelState& r) { return r.old_is_full ? r.full : r.full_old; }
    enum Which { kFull = 0, kDelta = 1, kOld = 2 };
    DevVersion& version(RelState& r, u32 kc, Which w) {
        return w == kDelta ? vdelta(r, kc) : (w == kOld ? vold(r) : vfull(r, kc));
    }

    JoinIndex& index(RelState& r, u32 kc, Which which, u32 col) {
        if (which == kOld && r.old_is_full) which = kFull;
        if (col == 1 && r.arity == 2 && !dist() && !r.levels_mode && r.hash_mode && by1_) {
            if (which == kFull) {
                if (!r.by1) {
                    r.by1 = std::make_unique<JoinIndex>();
                    build_index_on(r.full, 1, *r.by1, nullptr);
                }
                return *r.by1;
            }
            if (which == kOld && r.old_by1) return *r.old_by1;
        }
        IndexMap& m = vindexes(r, kc);
        auto key = std::make_pair(static_cast<int>(which), col);
        auto it = m.find(key);
        if (it != m.end()) return *it->second;
        auto idx = std::make_unique<JoinIndex>();
        build_index_on(version(r, kc, which), col, *idx, nullptr);
        JoinIndex& ref = *idx;
        m.emplace(key, std::move(idx));
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
            if (trace_)
                std::fprintf(stderr, "[fvlog]   sorted copy on col %u: %llu rows x %u cols\n", col,
                             static_cast<unsigned long long>(base->n), arity);
            std::vector<const u32*> order_cols{base->cols[col].get()};
            for (u32 j = 0; j < arity; ++j)
                if (j != col) order_cols.push_back(base->cols[j].get());
            DBuf<u32> perm = base->n ? lexicographic_order(c_, order_cols.data(), arity, base->n) : DBuf<u32>();
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
        engine_build_runs(c_, idx.rows->cols[col].get(), idx.rows->n, idx, st_.key_shift);
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
    Filter owner_filter(const SlotRef& s, u32 oshift) const {
        Filter f{s, {}, kFilterOwner, rank_};
        f.world = world_;
        f.oshift = oshift;
        return f;
    }

    // ---- exchange helpers (partitioned mode) -------------------------------------

    // All-to-all of routed rows. `route` has filled send buffers grouped by
    // destination with cnt/off; returns the received row count and fills
    // `recv` buffers (allocated here) for each column.
    // d_cnt: the route kernel's per-destination counts, on the device; the
    // count exchange gathers them there and returns send and receive counts
    // with one host round trip.
    template <typename T>
    u64 exchange(const std::vector<DBuf<T>>& send, const u64* d_cnt, std::vector<DBuf<T>>& recv) {
        std::vector<u64> cnt(world_), off(world_), rcnt(world_), roff(world_);
        c_->tx->exchange_counts_dev(c_, d_cnt, cnt.data(), rcnt.data());
        u64 run = 0;
        for (u32 p = 0; p < world_; ++p) {
            off[p] = run;
            run += cnt[p];
        }
        u64 total = 0;
        for (u32 p = 0; p < world_; ++p) {
            roff[p] = total;
            total += rcnt[p];
        }
        recv.clear();
        std::vector<ExchangeCol> cols;
        for (size_t j = 0; j < send.size(); ++j) {
            recv.emplace_back(c_, total);
            cols.push_back(ExchangeCol{send[j].get(), recv.back().get(), static_cast<u32>(sizeof(T))});
        }
        c_->tx->exchange_rows(c_, cols, cnt.data(), off.data(), rcnt.data(), roff.data());
        return total;
    }

    // Shuffle an intermediate so every row sits on owner(row[key]).
    Inter shuffle(const Inter& cur, const ColRef& key) {
        std::vector<const u32*> in;
        std::vector<ColRef> refs;
        for (auto& [r, p] : cur.cols) {
            refs.push_back(r);
            in.push_back(p);
        }
        std::vector<DBuf<u32>> send;
        std::vector<u32*> outp;
        for (size_t j = 0; j < in.size(); ++j) {
            send.emplace_back(c_, cur.n);
            outp.push_back(send.back().get());
        }
        std::vector<u64> cnt(world_), off(world_);
        RouteKey rk;
        rk.col = cur.cols.at(key);
        DBuf<u64> d_cnt(c_, world_);
        engine_route(c_, cur.n, rk, world_, in, outp, {}, {}, cnt.data(), off.data(), d_cnt.get());
        Inter next;
        next.n = exchange(send, d_cnt.get(), next.owned);
        for (size_t j = 0; j < refs.size(); ++j) next.cols[refs[j]] = next.owned[j].get();
        return next;
    }

    // Route a candidate pool to owner(head col 0).
    void route_pool(CandPool& pool, u32 home, u32 oshift) {
        const u32 W = (pool.arity + 1) / 2;
        if (pool.words.empty()) pool.words.resize(W);
        std::vector<const u64*> in;
        std::vector<DBuf<u64>> send;
        std::vector<u64*> outp;
        for (u32 w = 0; w < W; ++w) {
            in.push_back(pool.words[w].get());
            send.emplace_back(c_, pool.n);
            outp.push_back(send.back().get());
        }
        // Packed keys: the home column is the high half (col 0) or the low
        // half (col 1) of a binary key, the whole word of a unary one.
        // (choose_home_cols only picks a non-zero home for arity <= 2).
        RouteKey rk;
        rk.word = pool.words[0].get();
        rk.shift = st_.key_shift;
        rk.hi = pool.arity >= 2 && home == 0 ? 1 : 0;
        if (pool.arity >= 2 && home == 1) rk.mask = (u64(1) << st_.key_shift) - 1;
        rk.oshift = oshift;
        std::vector<u64> cnt(world_), off(world_);
        DBuf<u64> d_cnt(c_, world_);
        engine_route(c_, pool.n, rk, world_, {}, {}, in, outp, cnt.data(), off.data(), d_cnt.get());
        std::vector<DBuf<u64>> recv;
        pool.n = exchange(send, d_cnt.get(), recv);
        pool.words = std::move(recv);
        pool.cap = pool.n;
    }

    // ---- execute_plan (P/src/engine.cpp:72-146) for one variant ------------------

    // Join step k of plan p is a word composition: the right atom is binary,
    // unconstrained, joined on its column 0 with nothing else to check, and
    // the head is (left-side column, right atom's column 1) with no guard.
    static bool word_step_ok(const Plan& p, size_t k) {
        const PlanJoin& j = p.joins[k];
        const u32 R = j.right_source;
        // the only guard allowed is x != z between the two head columns (a
        // word drops x's own bit)
        const bool guard_ok = p.guard_neq.empty() ||
                              (p.guard_neq.size() == 1 && p.guard_neq[0].first + p.guard_neq[0].second == 1);
        return k + 1 == p.joins.size() && p.sources[R].arity == 2 && !p.sources[R].constrained() &&
               j.right_col == 0 && j.residual_eq.empty() && guard_ok && p.head_arity == 2 &&
               p.output_cols.size() == 2 && p.output_cols[1] == ColRef{R, 1} && p.output_cols[0].source != R;
    }

    // Source 0 can be carried as words: binary and unconstrained, its column
    // 1 is the head's column 1 and nothing else (never a join key or a
    // residual; no guard but x != z between the two head columns).
    static bool carry_ok(const Plan& p) {
        const ColRef y{0, 1};
        if (p.sources[0].arity != 2 || p.sources[0].constrained() || p.head_arity != 2 || p.output_cols.size() != 2 ||
            !(p.output_cols[1] == y) || p.output_cols[0] == y)
            return false;
        for (const PlanJoin& j : p.joins) {
            if (j.left == y) return false;
            for (auto& [l, rc] : j.residual_eq)
                if (l == y) return false;
        }
        return p.guard_neq.empty() ||
               (p.guard_neq.size() == 1 && p.guard_neq[0].first + p.guard_neq[0].second == 1);
    }

    // Word form of a binary version of r (home copy) with its column-0 join
    // index, cached until the version changes. Built from the lexicographic
    // order when the version has it, else from a sorted copy.
    // from_bitmap: FULL's words are read from the block set's bitmaps
    // (row-major, no tuple pass) — only valid before the iteration inserts
    // into the relation (prepare_full_words), since the bitmaps then already
    // hold this iteration's new rows.
    WordBuild& word_build(RelState& r, Which which, bool from_bitmap = false) {
        if (which == kOld && r.old_is_full) which = kFull;
        auto it = r.word_builds.find(static_cast<int>(which));
        if (it != r.word_builds.end()) return *it->second;
        const DevVersion& v = version(r, r.home, which);
        auto wb = std::make_unique<WordBuild>();
        const u64 n = v.n;
        if (from_bitmap && which == kFull && r.block_mode && r.blocks.capacity() && r.arity == 2 && !dist()) {
            for (int j = 0; j < 3; ++j) wb->words.cols.emplace_back(c_, std::max<u64>(n, 1));
            wb->words.n = engine_blockset_words(c_, r.blocks, wb->words.cols[0].get(), wb->words.cols[1].get(),
                                                wb->words.cols[2].get(), std::max<u64>(n, 1), st_.key_shift);
            wb->words.lex_sorted = false;  // grouped by x (z windows in block order)
            wb->idx.rows = &wb->words;
            engine_build_runs(c_, wb->words.cols[0].get(), wb->words.n, wb->idx, st_.key_shift);
            if (trace_)
                std::fprintf(stderr, "[fvlog]   word build of %s (full, from the bitmaps): %llu rows -> %llu words\n",
                             r.name.c_str(), static_cast<unsigned long long>(n),
                             static_cast<unsigned long long>(wb->words.n));
            WordBuild& ref = *wb;
            r.word_builds.emplace(static_cast<int>(kFull), std::move(wb));
            return ref;
        }
        DevVersion sorted;
        const DevVersion* src = &v;
        if (!v.lex_sorted && n > 1) {
            std::vector<DBuf<u64>> words;
            words.emplace_back(c_, n);
            u64* wp = words[0].get();
            engine_pack_keys(c_, v.ptrs(), n, st_.key_shift, &wp);
            engine_sort_keys(c_, words, n, 2, st_.key_shift);
            sorted.n = n;
            sorted.cols.emplace_back(c_, n);
            sorted.cols.emplace_back(c_, n);
            std::vector<u32*> dc{sorted.cols[0].get(), sorted.cols[1].get()};
            engine_unpack_keys(c_, words[0].get(), n, 2, st_.key_shift, dc);
            src = &sorted;
        }
        for (int j = 0; j < 3; ++j) wb->words.cols.emplace_back(c_, std::max<u64>(n, 1));
        // Sized by the row count (rows past the words carry x = 0xffffffff,
        // which no index holds) unless that could be a value (32-bit keys)
        // or the trace wants the word count.
        const bool exact = st_.key_shift >= 32 || trace_;
        wb->words.n = n ? engine_tuples_to_words(c_, src->cols[0].get(), src->cols[1].get(), n,
                                                 wb->words.cols[0].get(), wb->words.cols[1].get(),
                                                 wb->words.cols[2].get(), exact)
                        : 0;
        wb->words.lex_sorted = true;
        wb->idx.rows = &wb->words;
        engine_build_runs(c_, wb->words.cols[0].get(), wb->words.n, wb->idx, st_.key_shift);
        if (trace_)
            std::fprintf(stderr, "[fvlog]   word build of %s (%s): %llu rows -> %llu words\n", r.name.c_str(),
                         which == kDelta ? "delta" : (which == kOld ? "old" : "full"),
                         static_cast<unsigned long long>(n), static_cast<unsigned long long>(wb->words.n));
        WordBuild& ref = *wb;
        r.word_builds.emplace(static_cast<int>(which), std::move(wb));
        return ref;
    }

    // Word builds of FULL for the iteration's composition steps, taken from
    // the block sets before any insert of the iteration.
    void prepare_full_words(const std::vector<std::pair<const Plan*, long>>& active) {
        if (dist() || !words_) return;
        for (auto& [p, d] : active) {
            if (p->joins.empty()) continue;
            const size_t k = p->joins.size() - 1;
            if (!word_step_ok(*p, k) || !rel(p->head).word_sink) continue;
            const u32 R = p->joins[k].right_source;
            if (static_cast<long>(R) == d) continue;  // DELTA build
            RelState& r = rel(p->sources[R].relation);
            if (r.block_mode && !r.levels_mode) word_build(r, kFull, true);
        }
    }

    // One variant's execution state (execute_plan, P/src/engine.cpp:72-146).
    struct VarRun {
        const Plan& plan;
        const DistPlan& dp;
        long delta_source;
        std::vector<const DevVersion*> ver;
        std::vector<Which> which;
        std::vector<std::set<ColRef>> needed;  // columns still needed after join step k
        u32 W = 1;
        bool src0_pending = false;
        bool D = false;
        CandPool& out;
        HeadSink* sink;
        // Source 0 is carried as words (x, z base, mask) through the chain:
        // its column 1 is only the head's column 1, so the mask rides along
        // as ColRef {0, 2} and the last step emits one word per row.
        bool carry = false;
        // Step 0's probe counts and output offsets computed ahead, together
        // with other variants' (one host round trip for all their sizes).
        struct Pre {
            bool valid = false;
            DBuf<u32> starts;
            DBuf<u64> offsets;
            u64 T = 0;
        } pre;
        Inter cur;  // step 0's input (prepared variants)
    };

    // `old_src[s]`: source s reads FULL - DELTA instead of FULL (exactly-once
    // variants; empty = every non-DELTA source reads FULL, the reference).
    // A variant's versions and step-0 input; null when a source is empty.
    std::unique_ptr<VarRun> prepare_variant(const Plan& plan, const DistPlan& dp, long delta_source,
                                            const std::vector<u8>& old_src, CandPool& out, HeadSink* sink) {
        const u32 ns = static_cast<u32>(plan.sources.size());
        auto vp = std::unique_ptr<VarRun>(new VarRun{plan, dp, delta_source, std::vector<const DevVersion*>(ns),
                                                     std::vector<Which>(ns, kFull), {}, (plan.head_arity + 1) / 2,
                                                     plan.sources[0].constrained(), dist(), out, sink});
        VarRun& v = *vp;
        for (u32 s = 0; s < ns; ++s) {
            RelState& r = rel(plan.sources[s].relation);
            const u32 kc = partitioned(r) ? dp.src_copy[s] : 0;
            if (static_cast<long>(s) == delta_source) v.which[s] = kDelta;
            else if (!old_src.empty() && old_src[s]) v.which[s] = kOld;
            v.ver[s] = &version(r, kc, v.which[s]);
            if (!v.D && v.ver[s]->n == 0) return nullptr;  // engine.cpp:76-78
        }
        // (partitioned runs: only a DELTA that is already words — the word
        // builds are single-GPU)
        v.carry = words_ && !plan.joins.empty() && rel(plan.head).word_sink && carry_ok(plan) &&
                  (!v.D || v.ver[0]->cols.size() == 3);
        if (v.carry && v.ver[0]->cols.size() == 2) {
            // the probe side as words (cached word build of that version)
            WordBuild& wb = word_build(rel(plan.sources[0].relation), v.which[0]);
            v.ver[0] = &wb.words;
            if (v.ver[0]->n == 0) return nullptr;
        }
        Inter& cur = v.cur;
        cur.n = v.ver[0]->n;
        for (u32 j = 0; j < plan.sources[0].arity; ++j) cur.cols[ColRef{0, j}] = v.ver[0]->cols[j].get();
        if (v.carry) cur.cols[ColRef{0, 2}] = v.ver[0]->cols[2].get();
        const size_t nj = plan.joins.size();
        v.needed.resize(nj);
        for (size_t k = 0; k < nj; ++k) {
            std::set<ColRef>& s = v.needed[k];
            for (size_t q = k + 1; q < nj; ++q) {
                s.insert(plan.joins[q].left);
                for (auto& r : plan.joins[q].residual_eq) s.insert(r.first);
            }
            for (auto& r : plan.output_cols) s.insert(r);
            if (v.carry) s.insert(ColRef{0, 2});
        }
        return vp;
    }

    void run_variant(VarRun& v) {
        const Plan& plan = v.plan;
        const DistPlan& dp = v.dp;
        CandPool& out = v.out;
        Inter cur = std::move(v.cur);
        if (!plan.joins.empty()) {
            join_step(v, 0, std::move(cur));
            return;
        }
        // No joins: a single-atom rule (copy / projection / selection).
        const u32 W = v.W;
        OutSpec spec;
        spec.shift = st_.key_shift;
        if (v.src0_pending) {
            RowFilter f = source_filter(plan.sources[0], *v.ver[0]);
            for (u32 q = 0; q < f.n; ++q) push(spec, f.f[q]);
        }
        auto slot0 = [&](const ColRef& r) { return SlotRef{v.ver[0]->cols[r.col].get(), 0}; };
        for (auto& [ga, gb] : plan.guard_neq)
            push(spec, Filter{slot0(plan.output_cols[ga]), slot0(plan.output_cols[gb]), kFilterNeq, 0});
        if (v.D && dp.replicated_out) {
            const RelState& h = rel(plan.head);
            push(spec, owner_filter(slot0(plan.output_cols[h.home]), h.owner_shift));
        }
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

    // The build-side index of join step k (tmp owns a constrained source's
    // one-off index); *inter_word: the step's intermediate goes through a
    // word sink (inter_refs its columns).
    JoinIndex* step_index(VarRun& v, size_t k, std::unique_ptr<JoinIndex>& tmp, ColRef (&inter_refs)[2],
                          bool* inter_word) {
        const Plan& plan = v.plan;
        const PlanJoin& jn = plan.joins[k];
        const u32 R = jn.right_source;
        const size_t nj = plan.joins.size();
        RelState& rr = rel(plan.sources[R].relation);
        const bool word_step = k + 1 == nj && !v.D && word_step_ok(plan, k);
        // A deduplicated binary intermediate (x, z) of a composition step is
        // produced through a temporary word sink instead of rows + sort-unique.
        *inter_word = !v.D && words_ && k + 1 < nj && inter_word_ok(v, k, inter_refs);
        if (plan.sources[R].constrained()) {
            tmp = std::make_unique<JoinIndex>();
            build_index_on(*v.ver[R], jn.right_col, *tmp, &plan.sources[R]);
            return tmp.get();
        }
        if ((word_step && rel(plan.head).word_sink && v.ver[R]->cols.size() == 2) || *inter_word) {
            // Composition into a word sink: probe the word form of the build
            // version (x, z base, mask), one output per word.
            return &word_build(rr, v.which[R]).idx;
        }
        return &index(rr, partitioned(rr) ? v.dp.src_copy[R] : 0, v.which[R], jn.right_col);
    }

    // Probe counts of step k -> per-row output offsets (offsets[n] = T).
    void count_step(VarRun& v, size_t k, const Inter& cur, JoinIndex& idx, u32* starts, u64* offsets) {
        const u64 n = cur.n;
        RowFilter pred;
        if (k == 0 && v.src0_pending) pred = source_filter(v.plan.sources[0], *v.ver[0]);
        if (fused_probe_scan_) {
            engine_probe_offsets(c_, cur.cols.at(v.plan.joins[k].left), n, idx, pred, starts, offsets);
            return;
        }
        DBuf<u32> counts(c_, n);
        engine_probe_count(c_, cur.cols.at(v.plan.joins[k].left), n, idx, pred, starts, counts.get());
        exclusive_scan_counts(c_, counts.get(), offsets, n);
    }

    // Step 0 of several prepared variants counted with one host round trip
    // for all their output sizes. Left to join_step (which reads its size
    // with the head's set counters): partitioned runs, constrained build
    // sides, and a last step into a head an earlier variant of the batch
    // already feeds (its set counters are read on that step's sync).
    void precount_variants(std::vector<std::unique_ptr<VarRun>>& vs) {
        if (dist()) return;
        std::vector<VarRun*> todo;
        std::set<std::string> heads;
        for (auto& vp : vs) {
            if (!vp) continue;
            VarRun& v = *vp;
            const Plan& plan = v.plan;
            if (plan.joins.empty()) continue;
            const bool last = plan.joins.size() == 1;
            const bool taken = last && v.sink && (heads.count(plan.head) || v.sink->counter.get());
            if (v.sink) heads.insert(plan.head);
            if (taken || plan.sources[plan.joins[0].right_source].constrained()) continue;
            todo.push_back(&v);
        }
        if (todo.size() < 2) return;
        if (batch_pinned_cap_ < todo.size()) {
            if (batch_pinned_) cudaFreeHost(batch_pinned_);
            batch_pinned_cap_ = std::max<size_t>(256, 2 * todo.size());
            FV_CUDA(cudaMallocHost(&batch_pinned_, sizeof(u64) * batch_pinned_cap_));
        }
        for (size_t q = 0; q < todo.size(); ++q) {
            VarRun& v = *todo[q];
            std::unique_ptr<JoinIndex> tmp;
            ColRef refs[2];
            bool iw = false;
            JoinIndex* idx = step_index(v, 0, tmp, refs, &iw);
            const u64 n = v.cur.n;
            v.pre.starts = DBuf<u32>(c_, n);
            v.pre.offsets = DBuf<u64>(c_, n + 1);
            if (idx->rows->n == 0) {
                FV_CUDA(cudaMemsetAsync(v.pre.offsets.get() + n, 0, 8, c_->stream));
            } else {
                count_step(v, 0, v.cur, *idx, v.pre.starts.get(), v.pre.offsets.get());
            }
            FV_CUDA(cudaMemcpyAsync(batch_pinned_ + q, v.pre.offsets.get() + n, 8, cudaMemcpyDeviceToHost, c_->stream));
        }
        c_->sync();
        for (size_t q = 0; q < todo.size(); ++q) {
            todo[q]->pre.T = batch_pinned_[q];
            todo[q]->pre.valid = true;
        }
    }

    // Join step k of a variant on intermediate `cur`; recurses into step k+1.
    // An intermediate larger than inter_chunk_ rows is produced and carried
    // through the rest of the chain chunk by chunk (single GPU: every rank of
    // a partitioned run must issue the same collectives, so it stays whole
    // there), so memory stays O(chunk x depth + output).
    void join_step(VarRun& v, size_t k, Inter cur) {
        const Plan& plan = v.plan;
        const DistPlan& dp = v.dp;
        const bool D = v.D;
        const u32 W = v.W;
        CandPool& out = v.out;
        HeadSink* sink = v.sink;
        const long delta_source = v.delta_source;
        const size_t nj = plan.joins.size();
        const PlanJoin& jn = plan.joins[k];
        const u32 R = jn.right_source;
        if (D && dp.shuffle[k]) cur = shuffle(cur, jn.left);
        std::unique_ptr<JoinIndex> tmp;
        ColRef inter_refs[2];
        bool inter_word = false;
        JoinIndex* idx = step_index(v, k, tmp, inter_refs, &inter_word);
        const bool pre_ok = k == 0 && v.pre.valid;
        if (!D && !pre_ok && idx->rows->n == 0) return;
        // The build side is in word form (x, z base, mask): a binary atom whose
        // version has three columns (a ternary atom's version also has three).
        const bool word_build_side = plan.sources[R].arity == 2 && idx->rows->cols.size() == 3;
        // Carried words: the last step's head column 1 is source 0's word.
        const bool word_probe_side = v.carry && k + 1 == nj;
        const u64 n = cur.n;
        DBuf<u32> starts;
        DBuf<u64> offsets;
        u64 T = 0;
        if (pre_ok) {
            // counted ahead (precount_variants)
            starts = std::move(v.pre.starts);
            offsets = std::move(v.pre.offsets);
            T = v.pre.T;
            v.pre.valid = false;
        } else {
            starts = DBuf<u32>(c_, n);
            offsets = DBuf<u64>(c_, n + 1);
            count_step(v, k, cur, *idx, starts.get(), offsets.get());
            FV_CUDA(cudaMemcpyAsync(c_->pinned, offsets.get() + n, 8, cudaMemcpyDeviceToHost, c_->stream));
            // The fused dedup's set counters ride on the same sync (its first
            // chunk then needs no read of its own).
            HeadSink* pre = nullptr;
            if (k + 1 == nj && sink && sink->counter.get()) {
                RelState& hr = rel(plan.head);
                if (hr.block_mode && hr.blocks.capacity()) {
                    pre = sink;
                    FV_CUDA(cudaMemcpyAsync(c_->pinned + 8, sink->counter.get(), 24, cudaMemcpyDeviceToHost,
                                            c_->stream));
                    FV_CUDA(cudaMemcpyAsync(c_->pinned + 11, hr.blocks.count.get(), 8, cudaMemcpyDeviceToHost,
                                            c_->stream));
                }
            }
            c_->sync();
            T = c_->pinned[0];
            if (pre && T) {  // consumed by the first chunk's hash_reserve below
                pre->pre = true;
                for (int q = 0; q < 4; ++q) pre->pre_vals[q] = c_->pinned[8 + q];
            }
        }
        if (trace_)
            std::fprintf(stderr, "[fvlog]   %s join %zu/%zu delta@%ld probe=%llu outputs=%llu\n", plan.head.c_str(), k, nj,
                         delta_source, static_cast<unsigned long long>(n), static_cast<unsigned long long>(T));
        if (!D && T == 0) return;

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
        if (last) {
            // Word build side: the x != z guard is applied to the words (the
            // word of x's own window drops x's bit), not as a row filter.
            const bool word_guard = (word_build_side || word_probe_side) && !plan.guard_neq.empty() &&
                                    rel(plan.head).word_sink;
            spec.word_neq = word_guard ? 1 : 0;
            for (auto& [ga, gb] : plan.guard_neq)
                if (!word_guard)
                    push(spec, Filter{slot_of(plan.output_cols[ga]), slot_of(plan.output_cols[gb]), kFilterNeq, 0});
            if (D && dp.replicated_out) {
                const RelState& h = rel(plan.head);
                push(spec, owner_filter(slot_of(plan.output_cols[h.home]), h.owner_shift));
            }
            spec.key_mode = 1;
            spec.n_out = plan.head_arity;
            for (u32 h = 0; h < plan.head_arity; ++h) spec.col[h] = slot_of(plan.output_cols[h]);
            if (sink) {
                // Fused dedup: the join kernel inserts into FULL's key set.
                // Output chunks bound what the key set and the new-key
                // buffer must be sized for: each chunk may add at most its
                // own size, and the real count is re-read between chunks
                // (CSPA joins produce ~10^3 candidates per new row).
                RelState& hr = rel(plan.head);
                if (trace_) {
                    spec.probe_count = c_->d_scalars + 24;
                    FV_CUDA(cudaMemsetAsync(spec.probe_count, 0, 8, c_->stream));
                }
                // Partitioned: rows owned here are deduplicated in this
                // kernel, the others are pooled for the all-to-all.
                const bool route = D && !dp.replicated_out && !dp.local_out;
                if (route) {
                    out.reserve(c_, T);
                    spec.keys[0] = out.words[0].get() + out.n;
                    spec.d_count = c_->d_scalars + 26;
                    spec.remote_world = world_;
                    spec.remote_rank = rank_;
                    spec.remote_col = hr.home;
                    spec.remote_oshift = hr.owner_shift;
                    FV_CUDA(cudaMemsetAsync(spec.d_count, 0, 8, c_->stream));
                }
                // A chunk's outputs bound the keys it can add to the local
                // key set, which sizes the table (4x the bound). Routed runs
                // keep only ~1/world of them, so their chunks shrink by the
                // world size: per-rank tables sized for 2^28 new keys would
                // be mostly empty and every growth would stream them.
                const u64 chunk = route ? std::max<u64>(u64(1) << 24, kFusedChunk / world_) : kFusedChunk;
                for (u64 t0 = 0; t0 < T; t0 += chunk) {
                    const u64 t1 = std::min(T, t0 + chunk);
                    hash_reserve(hr, *sink, t1 - t0);
                    if (hr.block_mode) {
                        spec.ht_slots = nullptr;
                        spec.bs = block_args(hr);
                        spec.ovf_keys = sink->ovf.get();
                        spec.ovf_count = sink->counter.get() + 1;
                        spec.tile_set = block_tile_set_;
                        spec.wbits = SlotRef();
                        spec.word_sink = 0;
                        if (hr.word_sink) {
                            // Word sink: a composition step whose build side
                            // is in word form (x, z base, mask) emits one
                            // output per word; other joins emit their tuples
                            // as one-bit words.
                            if (word_probe_side) spec.wbits = slot_of(ColRef{0, 2});
                            else if (word_build_side) spec.wbits = SlotRef{idx->rows->cols[2].get(), 1};
                            spec.word_sink = 1;
                            spec.ovf_bits = sink->ovf_bits.get();
                            spec.new_tuples = sink->counter.get() + 2;
                            spec.new_widx = sink->widx.get();
                            spec.tile_set = word_combine_;
                        }
                    } else {
                        spec.bs = BlockSetArgs();
                        spec.ht_slots = hr.keys.slots.get();
                        spec.ht_mask = hr.keys.mask;
                        spec.ht_group_bits = hr.keys.group_bits;
                        // grouped layout <=> last iteration's candidates were all new
                        spec.tile_set = hr.keys.group_bits == 0 ? 1u : 0u;
                    }
                    spec.new_keys = sink->keys.get();
                    spec.new_count = sink->counter.get();
                    engine_materialize(c_, offsets.get(), n, T, starts.get(), spec, t0, t1);
                }
                sink->candidates += T;
                if (route) {
                    u64 pooled = 0;
                    c_->read_scalars(spec.d_count, &pooled, 1);
                    out.n += pooled;
                }
                if (trace_) {
                    u64 probes = 0;
                    c_->read_scalars(spec.probe_count, &probes, 1);
                    std::fprintf(stderr, "[fvlog]   fused dedup: %llu candidates -> %llu key-set probes\n",
                                 static_cast<unsigned long long>(T), static_cast<unsigned long long>(probes));
                }
                return;
            }
            // One-word keys: drop tile-local repeats before they are
            // pooled (and, partitioned, routed over NVLink).
            if (W == 1) spec.tile_dedup = 1;
            // Pooled candidates (no key set) are produced in chunks and
            // the pool is sort-uniqued whenever the next chunk would
            // push it past kPoolBudget rows (SURVEY.md §7 hard part 1:
            // the reference materializes every candidate at once).
            const bool compacts = spec.n_filters || spec.tile_dedup;
            for (u64 t0 = 0; t0 < T; t0 += pool_chunk_) {
                const u64 t1 = std::min(T, t0 + pool_chunk_);
                if (out.n && out.n + (t1 - t0) > pool_budget_) compact_pool(out);
                out.reserve(c_, t1 - t0);
                // Positional (uncompacted) writes use absolute output
                // indices: bias the base so output t0 lands at out.n.
                for (u32 w = 0; w < W; ++w) spec.keys[w] = out.words[w].get() + out.n - (compacts ? 0 : t0);
                if (compacts) {
                    spec.d_count = c_->d_scalars + 20;
                    FV_CUDA(cudaMemsetAsync(spec.d_count, 0, 8, c_->stream));
                }
                engine_materialize(c_, offsets.get(), n, T, starts.get(), spec, t0, t1);
                u64 produced = t1 - t0;
                if (compacts) c_->read_scalars(spec.d_count, &produced, 1);
                out.n += produced;
            }
            return;
        }
        if (inter_word) {
            Inter next = word_intermediate(*idx, offsets.get(), n, T, starts.get(), slot_of(inter_refs[0]),
                                           inter_refs, temp_ratio_[std::make_tuple(&plan, k, delta_source)]);
            if (!D && next.n == 0) return;
            join_step(v, k + 1, std::move(next));
            return;
        }
        // A carried word with one other needed column: the intermediate is
        // merged into words (same (x, z window) rows OR their masks) through
        // a temporary word sink instead of being materialized row by row.
        if (v.carry && !D && words_) {
            std::vector<ColRef> need;
            for (const ColRef& r : v.needed[k])
                if (r.source <= R) need.push_back(r);
            const ColRef yb{0, 1}, ym{0, 2};
            std::vector<ColRef> other;
            for (const ColRef& r : need)
                if (!(r == yb) && !(r == ym)) other.push_back(r);
            if (other.size() == 1 && need.size() == 3 && spec.n_filters == 0) {
                const ColRef refs3[3] = {other[0], yb, ym};
                const SlotRef zb = slot_of(yb), wm = slot_of(ym);
                Inter next = word_intermediate(*idx, offsets.get(), n, T, starts.get(), slot_of(other[0]), refs3,
                                               temp_ratio_[std::make_tuple(&plan, k, delta_source)], &zb, &wm);
                if (next.n == 0) return;
                join_step(v, k + 1, std::move(next));
                return;
            }
        }
        // Intermediate: the columns later steps and the head still need.
        std::vector<ColRef> refs;
        for (const ColRef& r : v.needed[k]) {
            if (r.source > R) continue;
            if (refs.size() >= static_cast<size_t>(kMaxSlots)) fail(FV_ERR_PLAN, "join intermediate wider than 16 columns");
            refs.push_back(r);
        }
        spec.key_mode = 0;
        spec.n_out = static_cast<u32>(refs.size());
        for (u32 j = 0; j < spec.n_out; ++j) spec.col[j] = slot_of(refs[j]);
        const bool compacts = spec.n_filters != 0;
        u32 bound_cols = 0;
        for (u32 s = 0; s <= R; ++s) bound_cols += plan.sources[s].arity;
        const u64 chunk = D ? T : std::max<u64>(inter_chunk_, 1);
        for (u64 t0 = 0; t0 < std::max<u64>(T, 1); t0 += chunk) {
            const u64 t1 = std::min(T, t0 + chunk);
            Inter next;
            for (u32 j = 0; j < spec.n_out; ++j) {
                next.owned.emplace_back(c_, t1 - t0);
                // positional writes use absolute output indices (see above)
                spec.out_cols[j] = next.owned.back().get() - (compacts ? 0 : t0);
                next.cols[refs[j]] = next.owned.back().get();
            }
            if (compacts) {
                spec.d_count = c_->d_scalars + 20;
                FV_CUDA(cudaMemsetAsync(spec.d_count, 0, 8, c_->stream));
            }
            engine_materialize(c_, offsets.get(), n, T, starts.get(), spec, t0, t1);
            u64 produced = t1 - t0;
            if (compacts) c_->read_scalars(spec.d_count, &produced, 1);
            next.n = produced;
            // (carried word masks are 32-bit payloads, not domain values:
            // the packed-key dedup does not apply)
            if (spec.n_out < bound_cols && !v.carry) maybe_dedup_inter(next, std::make_tuple(&plan, k, delta_source));
            if (!D && next.n == 0) continue;
            join_step(v, k + 1, std::move(next));
            if (T == 0) break;
        }
    }

    // Step k (not the last) can produce its intermediate as words: the right
    // atom is binary, unconstrained, joined on its column 0 with nothing else
    // to check, the later steps and the head need exactly one left-side
    // column and the right atom's column 1, and the step's intermediates have
    // been measured to repeat (maybe_dedup_inter's policy is on). refs[0]:
    // the left-side column, refs[1] = {R, 1}.
    bool inter_word_ok(VarRun& v, size_t k, ColRef (&refs)[2]) {
        const Plan& p = v.plan;
        const PlanJoin& j = p.joins[k];
        const u32 R = j.right_source;
        if (p.sources[R].arity != 2 || p.sources[R].constrained() || j.right_col != 0 || !j.residual_eq.empty())
            return false;
        if (v.ver[R]->cols.size() != 2) return false;
        std::vector<ColRef> need;
        for (const ColRef& r : v.needed[k])
            if (r.source <= R) need.push_back(r);
        if (need.size() != 2) return false;
        const ColRef right{R, 1};
        if (need[0] == right) std::swap(need[0], need[1]);
        if (!(need[1] == right) || need[0].source >= R) return false;
        auto it = inter_policy_.find(std::make_tuple(&p, k, v.delta_source));
        if (it == inter_policy_.end() || !it->second.on) return false;
        refs[0] = need[0];
        refs[1] = need[1];
        return true;
    }

    // The distinct (x, z) rows of a composition step, through a temporary
    // word sink: the join emits one word per (probe row, build word), the
    // block set dedups, the merged words expand to the rows (grouped by x).
    // carried: the word is source 0's carried word (z base {0,1}, mask {0,2},
    // given as zb / wbits); the intermediate stays in word form — one row per
    // (x, z window) with the masks of all its derivations OR-ed — and keeps
    // carrying it (refs[1] = {0,1}, refs[2] = {0,2}).
    Inter word_intermediate(JoinIndex& idx, const u64* offsets, u64 n, u64 T, const u32* starts, const SlotRef& left,
                            const ColRef* refs, double& block_ratio, const SlotRef* zb = nullptr,
                            const SlotRef* wbits = nullptr) {
        const bool carried = zb != nullptr;
        RelState tmp;
        // new blocks per output measured at this call site last time: the
        // directory is sized for it up front (no overflow-list rounds)
        tmp.blocks.ratio = block_ratio;
        tmp.name = "(intermediate)";
        tmp.arity = 2;
        tmp.hash_mode = tmp.block_mode = tmp.levels_mode = tmp.word_sink = true;
        tmp.word_mode = carried;
        tmp.temp = true;
        tmp.delta.cols.resize(carried ? 3 : 2);
        HeadSink sk;
        OutSpec spec;
        spec.shift = st_.key_shift;
        spec.key_mode = 1;
        spec.n_out = 2;
        spec.col[0] = left;
        spec.col[1] = carried ? *zb : SlotRef{idx.rows->cols[1].get(), 1};
        spec.wbits = carried ? *wbits : SlotRef{idx.rows->cols[2].get(), 1};
        spec.word_sink = 1;
        spec.tile_set = word_combine_;
        for (u64 t0 = 0; t0 < T; t0 += kFusedChunk) {
            const u64 t1 = std::min(T, t0 + kFusedChunk);
            hash_reserve(tmp, sk, t1 - t0);
            spec.bs = block_args(tmp);
            spec.ovf_keys = sk.ovf.get();
            spec.ovf_count = sk.counter.get() + 1;
            spec.ovf_bits = sk.ovf_bits.get();
            spec.new_keys = sk.keys.get();
            spec.new_count = sk.counter.get();
            spec.new_tuples = sk.counter.get() + 2;
            spec.new_widx = sk.widx.get();
            engine_materialize(c_, offsets, n, T, starts, spec, t0, t1);
        }
        CandPool none;
        none.arity = 2;
        const u64 nd = T ? hash_finalize(tmp, sk, none) : 0;
        // (from the final block count: an overflowed first insert counts
        // only the blocks that fit before its drain)
        if (T) block_ratio = std::max(tmp.blocks.ratio, double(tmp.blocks.blocks) / double(T));
        if (trace_)
            std::fprintf(stderr, "[fvlog]   word intermediate: %llu word outputs -> %llu rows\n",
                         static_cast<unsigned long long>(T), static_cast<unsigned long long>(nd));
        Inter next;
        const size_t nc = carried ? 3 : 2;
        next.n = carried ? tmp.delta.n : nd;  // word form: one row per word
        if (next.n) {
            next.owned = std::move(tmp.delta.cols);
        } else {
            next.owned.clear();
            for (size_t j = 0; j < nc; ++j) next.owned.emplace_back(c_, 0);
        }
        for (size_t j = 0; j < nc; ++j) next.cols[refs[j]] = next.owned[j].get();
        return next;
    }

    // Distinct rows of a join intermediate that dropped columns. The join
    // multiplies duplicates: in CSPA's valueAlias(x,y) :- valueFlow(z,x),
    // memoryAlias(z,w), valueFlow(w,y) the (x,w) pairs repeat once per z and
    // every repeat would re-derive all of valueFlow(w,_). Sets are unchanged
    // (the reference keeps every id pair; results are compared as sets).
    // Adaptive per plan step and variant: an intermediate of at least
    // kInterProbeRows rows is deduplicated and measured; the step keeps
    // deduplicating once a measurement removed >= 1/4 of the rows, and is
    // re-measured whenever its intermediates grow 4x past the last
    // measurement (early iterations often have no repeats yet).
    using InterKey = std::tuple<const Plan*, size_t, long>;
    // Word intermediates' new-blocks-per-output ratio, per plan step.
    std::map<std::tuple<const Plan*, size_t, long>, double> temp_ratio_;
    struct InterPolicy {
        bool on = false;
        u64 measured = 0;  // size of the last measured intermediate (0: never)
    };
    static constexpr u64 kInterProbeRows = u64(1) << 16;

    void maybe_dedup_inter(Inter& x, const InterKey& key) {
        const u32 a = static_cast<u32>(x.owned.size());
        if (a == 0 || a > FV_MAX_ARITY || x.n < 2 || x.owned.size() != x.cols.size()) return;
        InterPolicy& policy = inter_policy_[key];
        const bool measure = !policy.on && x.n >= inter_probe_rows_ &&
                             (policy.measured == 0 || x.n >= 4 * policy.measured);
        if (!policy.on && !measure) return;
        std::vector<const u32*> cols;
        for (auto& b : x.owned) cols.push_back(b.get());
        const u32 W = (a + 1) / 2;
        std::vector<DBuf<u64>> words;
        std::vector<u64*> wp;
        for (u32 w = 0; w < W; ++w) {
            words.emplace_back(c_, x.n);
            wp.push_back(words.back().get());
        }
        engine_pack_keys(c_, cols, x.n, st_.key_shift, wp.data());
        if (measure && W == 1 && !exact_blocks_) {
            // Measure with a sketch of the distinct keys (one pass) and only
            // sort-unique when it shows enough repeats (SG's intermediates
            // have none: three measuring sorts of up to 2.8e7 rows).
            DBuf<u32> regs(c_, kBlockSketchRegs);
            engine_block_sketch(c_, words[0].get(), x.n, st_.key_shift, 0, regs.get());
            std::vector<u32> h(kBlockSketchRegs);
            regs.download(h.data(), kBlockSketchRegs);
            const u64 est = std::min<u64>(x.n, block_sketch_estimate(h.data()));
            policy.measured = x.n;
            if (trace_)
                std::fprintf(stderr, "[fvlog]   intermediate sketch %llu -> ~%llu distinct\n",
                             static_cast<unsigned long long>(x.n), static_cast<unsigned long long>(est));
            if (4 * est > 3 * x.n) return;  // < 1/4 repeats: leave it
            policy.on = true;
        }
        engine_sort_keys(c_, words, x.n, a, st_.key_shift);
        std::vector<DBuf<u32>> out;
        std::vector<u32*> op;
        for (u32 j = 0; j < a; ++j) {
            out.emplace_back(c_, x.n);
            op.push_back(out.back().get());
        }
        const u64 k = engine_unique_unpack(c_, words, x.n, a, st_.key_shift, op);
        if (trace_)
            std::fprintf(stderr, "[fvlog]   intermediate dedup %llu -> %llu (%s)\n", static_cast<unsigned long long>(x.n),
                         static_cast<unsigned long long>(k), policy.on ? "on" : "measured");
        if (measure && !policy.on) {
            policy.measured = x.n;
            policy.on = 4 * k <= 3 * x.n;
        }
        // x.cols maps ColRefs to the owned buffers in order of creation.
        std::map<const u32*, u32*> remap;
        for (u32 j = 0; j < a; ++j) remap[x.owned[j].get()] = op[j];
        for (auto& [ref, ptr] : x.cols) ptr = remap.at(ptr);
        x.owned = std::move(out);
        x.n = k;
    }

    // Sort-unique the pooled candidates in place (bounded-memory pooling).
    void compact_pool(CandPool& pool) {
        engine_sort_keys(c_, pool.words, pool.n, pool.arity, st_.key_shift);
        std::vector<DBuf<u64>> uniq;
        const u64 k = engine_unique_words(c_, pool.words, pool.n, uniq);
        if (trace_)
            std::fprintf(stderr, "[fvlog]   pool compaction %llu -> %llu rows\n",
                         static_cast<unsigned long long>(pool.n), static_cast<unsigned long long>(k));
        pool.words = std::move(uniq);
        pool.cap = pool.n;  // buffers were sized n; k rows are live
        pool.n = k;
    }

    // Sort candidates and fold them into (full, delta); returns |DELTA|.
    // Sort-merge dedup in two halves so that several relations' merges share
    // one host round trip for their new-row counts: merge_launch enqueues the
    // sort and the merge-path merge (new count to a device slot), then
    // merge_complete installs FULL and DELTA once the count is on the host.
    struct PendingMerge {
        DevVersion* full = nullptr;
        DevVersion* delta = nullptr;
        IndexMap* indexes = nullptr;
        RelState* home = nullptr;
        u32 arity = 0;
        DevVersion C, Dv;
        u64 cand_n = 0;
        DBuf<u64> d_new;
    };

    PendingMerge merge_launch(DevVersion& full, DevVersion& delta, IndexMap& indexes, u32 arity, CandPool& cand,
                              RelState* home) {
        if (cand.n) engine_sort_keys(c_, cand.words, cand.n, arity, st_.key_shift);
        std::vector<u64*> bw;
        for (auto& w : cand.words) bw.push_back(w.get());
        return merge_launch_sorted(full, delta, indexes, arity, bw, cand.n, home);
    }

    // merge_launch of n candidate keys already sorted (bw: their words).
    PendingMerge merge_launch_sorted(DevVersion& full, DevVersion& delta, IndexMap& indexes, u32 arity,
                                     std::vector<u64*>& bw, u64 n, RelState* home) {
        PendingMerge pm;
        pm.full = &full;
        pm.delta = &delta;
        pm.indexes = &indexes;
        pm.home = home;
        pm.arity = arity;
        pm.cand_n = n;
        if (n == 0) return pm;
        for (u32 j = 0; j < arity; ++j) {
            pm.C.cols.emplace_back(c_, full.n + n);
            pm.Dv.cols.emplace_back(c_, n);
        }
        std::vector<u32*> cc, dc;
        for (u32 j = 0; j < arity; ++j) {
            cc.push_back(pm.C.cols[j].get());
            dc.push_back(pm.Dv.cols[j].get());
        }
        pm.d_new = DBuf<u64>(c_, 1);
        engine_merge(c_, full.ptrs(), full.n, bw.data(), n, arity, st_.key_shift, cc, dc, pm.d_new.get());
        return pm;
    }

    // Seeds of several sort-merged (EDB) relations share one radix sort:
    // their packed keys are tagged with the relation's number above the
    // key bits, sorted together, untagged, and each relation's slice is
    // merged (deduplicated) on its own. False (nothing done) when fewer
    // than two relations qualify or the tags do not fit in 64 bits.
    bool seed_batch(const std::vector<std::pair<RelState*, const DevVersion*>>& rels, std::vector<PendingMerge>& pend) {
        if (rels.size() < 2) return false;
        const u32 base = 2 * st_.key_shift;
        u32 tag_bits = 1;
        while ((u64(1) << tag_bits) < rels.size()) ++tag_bits;
        if (base + tag_bits > 64) return false;
        u64 total = 0;
        for (auto& [r, v] : rels) total += v->n;
        DBuf<u64> all(c_, std::max<u64>(total, 1)), alt(c_, std::max<u64>(total, 1));
        u64 off = 0;
        for (size_t i = 0; i < rels.size(); ++i) {
            const DevVersion& v = *rels[i].second;
            u64* wp = all.get() + off;
            engine_pack_keys(c_, v.ptrs(), v.n, st_.key_shift, &wp);
            engine_mask_u64(c_, wp, v.n, ~u64(0), u64(i) << base);
            off += v.n;
        }
        if (total > 1 && radix_sort_keys_u64(c_, all.get(), alt.get(), total, 0, base + tag_bits)) all.swap(alt);
        engine_mask_u64(c_, all.get(), total, base >= 64 ? ~u64(0) : (u64(1) << base) - 1, 0);
        off = 0;
        for (auto& [r, v] : rels) {
            std::vector<u64*> bw{all.get() + off};
            pend.push_back(merge_launch_sorted(r->full, r->delta, r->indexes, r->arity, bw, v->n, r));
            off += v->n;
        }
        return true;
    }

    u64 merge_complete(PendingMerge& pm, u64 nd) {
        DevVersion& full = *pm.full;
        DevVersion& delta = *pm.delta;
        RelState* home = pm.home;
        if (pm.cand_n == 0) {
            delta = DevVersion();
            delta.n = 0;
            delta.cols.resize(pm.arity);
            pm.indexes->clear();
            if (home) home->word_builds.clear();
            if (home) set_old(*home, nullptr);
            return 0;
        }
        c_->prof_add_bytes("merge_dedup", 8.0 * double(nd) * pm.arity);
        pm.C.n = full.n + nd;
        pm.Dv.n = nd;
        pm.C.lex_sorted = pm.Dv.lex_sorted = true;  // merge-path output of sorted inputs
        if (home) home->word_builds.clear();
        if (home && nd) {
            set_old(*home, &full);
        } else if (home) {
            set_old(*home, nullptr);
        }
        full = std::move(pm.C);
        delta = std::move(pm.Dv);
        pm.indexes->clear();
        return nd;
    }

    // Complete several pending merges with one read of their counts.
    std::vector<u64> merge_complete_all(std::vector<PendingMerge>& pms) {
        std::vector<u64> nds(pms.size(), 0);
        size_t live = 0;
        for (auto& pm : pms) live += pm.cand_n ? 1 : 0;
        if (live) {
            if (batch_pinned_cap_ < live) {
                if (batch_pinned_) cudaFreeHost(batch_pinned_);
                batch_pinned_cap_ = std::max<size_t>(256, 2 * live);
                FV_CUDA(cudaMallocHost(&batch_pinned_, sizeof(u64) * batch_pinned_cap_));
            }
            size_t q = 0;
            for (auto& pm : pms)
                if (pm.cand_n)
                    FV_CUDA(cudaMemcpyAsync(batch_pinned_ + q++, pm.d_new.get(), 8, cudaMemcpyDeviceToHost, c_->stream));
            c_->sync();
            q = 0;
            for (size_t i = 0; i < pms.size(); ++i)
                if (pms[i].cand_n) nds[i] = batch_pinned_[q++];
        }
        for (size_t i = 0; i < pms.size(); ++i) nds[i] = merge_complete(pms[i], nds[i]);
        return nds;
    }

    u64 dedup_merge(DevVersion& full, DevVersion& delta, IndexMap& indexes, u32 arity, CandPool& cand,
                    RelState* home = nullptr) {
        std::vector<PendingMerge> one;
        one.push_back(merge_launch(full, delta, indexes, arity, cand, home));
        return merge_complete_all(one)[0];
    }

    // A relation's versions changed: its join indexes and word builds go.
    static void invalidate(RelState& r) {
        r.indexes.clear();
        r.word_builds.clear();
    }

    // The FULL a merge is about to replace becomes FULL - DELTA (moved, no
    // copy); null: nothing new, FULL - DELTA = FULL.
    void set_old(RelState& r, DevVersion* replaced) {
        r.full_old = DevVersion();
        r.old_is_full = true;
        if (replaced && r.keep_old) {
            r.full_old = std::move(*replaced);
            r.old_is_full = false;
        }
    }

    u64 dedup_merge_home(RelState& r, CandPool& cand) {
        return dedup_merge(r.full, r.delta, r.indexes, r.arity, cand, &r);
    }

    // Seed one copy of a relation from raw EDB rows (owner-filtered on kc
    // when partitioned).
    // Sort-merged copies are only launched (pend): the caller completes
    // every relation's seed merge with one read of the counts.
    void seed_copy(RelState& r, const DevVersion& v, u32 kc, std::vector<PendingMerge>& pend) {
        CandPool pool = seed_pool(r, v, kc);
        if (kc == r.home && r.hash_mode) {
            HeadSink sink;
            hash_finalize(r, sink, pool);
            return;
        }
        pend.push_back(
            merge_launch(vfull(r, kc), vdelta(r, kc), vindexes(r, kc), r.arity, pool, kc == r.home ? &r : nullptr));
    }

    PendingMerge merge_launch_home(RelState& r, CandPool& cand) {
        return merge_launch(r.full, r.delta, r.indexes, r.arity, cand, &r);
    }

    CandPool seed_pool(RelState& r, const DevVersion& v, u32 kc) {
        CandPool pool;
        pool.arity = r.arity;
        pool.reserve(c_, v.n);
        const u32 W = (r.arity + 1) / 2;
        if (!partitioned(r)) {
            std::vector<u64*> wp;
            for (auto& w : pool.words) wp.push_back(w.get());
            engine_pack_keys(c_, v.ptrs(), v.n, st_.key_shift, wp.data());
            pool.n = v.n;
        } else {
            OutSpec spec;
            spec.shift = st_.key_shift;
            spec.key_mode = 1;
            spec.n_out = r.arity;
            for (u32 j = 0; j < r.arity; ++j) spec.col[j] = SlotRef{v.cols[j].get(), 0};
            push(spec, owner_filter(SlotRef{v.cols[kc].get(), 0}, kc == r.home ? r.owner_shift : 0));
            for (u32 w = 0; w < W; ++w) spec.keys[w] = pool.words[w].get();
            spec.d_count = c_->d_scalars + 20;
            FV_CUDA(cudaMemsetAsync(spec.d_count, 0, 8, c_->stream));
            engine_project(c_, v.n, spec);
            c_->read_scalars(spec.d_count, &pool.n, 1);
        }
        return pool;
    }

    // Forward the new home Δ rows to the relation's other partition copies.
    void forward_delta(RelState& r) {
        for (u32 kc : r.keyset) {
            if (kc == r.home) continue;
            std::vector<const u32*> in;
            std::vector<DBuf<u32>> send;
            std::vector<u32*> outp;
            for (u32 j = 0; j < r.arity; ++j) {
                in.push_back(r.delta.cols[j].get());
                send.emplace_back(c_, r.delta.n);
                outp.push_back(send.back().get());
            }
            RouteKey rk;
            rk.col = r.delta.cols[kc].get();
            std::vector<u64> cnt(world_), off(world_);
            DBuf<u64> d_cnt(c_, world_);
            engine_route(c_, r.delta.n, rk, world_, in, outp, {}, {}, cnt.data(), off.data(), d_cnt.get());
            std::vector<DBuf<u32>> recv;
            const u64 n = exchange(send, d_cnt.get(), recv);
            CandPool pool;
            pool.arity = r.arity;
            pool.reserve(c_, n);
            std::vector<const u32*> rp;
            for (auto& b : recv) rp.push_back(b.get());
            std::vector<u64*> wp;
            for (auto& w : pool.words) wp.push_back(w.get());
            engine_pack_keys(c_, rp, n, st_.key_shift, wp.data());
            pool.n = n;
            RelCopy& cp = *r.copies.at(kc);
            dedup_merge(cp.full, cp.delta, cp.indexes, r.arity, pool);
        }
    }

    // ---- hash-mode dedup ---------------------------------------------------------

    u64 sink_count(HeadSink& s) {
        if (!s.counter.get()) return 0;
        u64 n = 0;
        c_->read_scalars(s.counter.get(), &n, 1);
        s.bound = n;
        return n;
    }

    // Room for `extra` more new keys in the sink and for count + extra keys
    // in the relation's key set at load factor <= 1/2 (rehash when needed).
    void hash_reserve(RelState& r, HeadSink& s, u64 extra) {
        if (!s.counter.get()) {
            s.counter = DBuf<u64>(c_, 3);
            FV_CUDA(cudaMemsetAsync(s.counter.get(), 0, 24, c_->stream));
            // fresh counters are zero and the block count is the last one read
            s.pre = true;
            s.pre_vals[0] = s.pre_vals[1] = s.pre_vals[2] = 0;
            s.pre_vals[3] = r.blocks.blocks;
        }
        if (r.block_mode) {
            block_reserve(r, s, extra);
            if (r.block_mode) return;  // else: converted to a key set, reserve that
        }
        if (s.bound + extra > s.cap) {
            const u64 have = sink_count(s);
            const u64 nc = std::max<u64>(have + extra, 2 * s.cap);
            DBuf<u64> nk(c_, nc);
            if (have) FV_CUDA(cudaMemcpyAsync(nk.get(), s.keys.get(), 8 * have, cudaMemcpyDeviceToDevice, c_->stream));
            s.keys = std::move(nk);
            s.cap = nc;
        }
        s.bound += extra;
        // bound counts every candidate as new, so the real load stays below
        // the worst case the table accepts (KeySet::limit: half its slots,
        // three quarters when memory forced a smaller table).
        if (r.keys.count + s.bound <= r.keys.limit) return;
        // Re-read the real count before growing: a stale bound (earlier
        // chunks counted as all-new) must not trigger a rehash.
        const u64 pending = sink_count(s);
        s.bound = pending + extra;
        if (r.keys.count + s.bound <= r.keys.limit) return;
        // Grow to a worst-case load of 1/4: most probes of a fused join are
        // repeats of present keys, and short linear-probe runs keep them to
        // one DRAM access; 4x growth also keeps the number of rehashes low.
        // Memory-tight: settle for 1/2, then 3/4 (fails loudly beyond).
        const u64 need = r.keys.count + pending + extra;
        u64 cap = 1u << 16;
        while (cap < kKeysetGrowth * need) cap <<= 1;
        KeySet ns;
        for (int attempt = 0;; ++attempt) {
            try {
                ns.slots = DBuf<u64>(c_, cap);
                ns.limit = attempt < 2 ? cap / 2 : cap / 4 * 3;
                break;
            } catch (const Error& e) {
                const u64 next = cap / 2;
                const bool fits_next = attempt == 0 ? next >= 2 * need : 3 * (next / 4) >= need;
                if (e.status != FV_ERR_OOM || attempt >= 2 || !fits_next) throw;
                cap = next;
            }
        }
        ns.mask = cap - 1;
        ns.count = r.keys.count;
        ns.group_bits = r.keys.capacity() ? r.keys.group_bits : initial_group_bits();
        // The old table holds FULL's keys and the ones found new so far this
        // iteration (a relation's keys only ever enter through its table):
        // move them all in one streaming pass over its slots — windowed in
        // shared memory when the layout is unchanged (every new slot written
        // once, no memset), else memset + atomic rehash.
        if (!(grow_windowed_ && engine_hash_grow(c_, r.keys, ns))) {
            FV_CUDA(cudaMemsetAsync(ns.slots.get(), 0xff, 8 * cap, c_->stream));
            if (r.keys.capacity()) engine_hash_rehash(c_, r.keys, ns);
        }
        r.keys = std::move(ns);
    }

    // ---- block-set dedup ---------------------------------------------------------

    BlockSetArgs block_args(const RelState& r) const {
        BlockSetArgs a;
        a.dir = r.blocks.dir.get();
        a.bits = r.blocks.bits.get();
        a.dbits = r.blocks.dbits.get();
        a.mask = r.blocks.mask;
        a.count = r.blocks.count.get();
        a.limit = r.blocks.capacity() / 4 * 3;
        a.shift = st_.key_shift;
        a.arity = r.arity;
        return a;
    }

    // Sink counters (new, overflow) and the block count in one sync; also
    // updates the relation's new-blocks-per-candidate estimate.
    void read_block_counters(RelState& r, HeadSink& s, u64* nw, u64* ov) {
        const u64* v = s.pre_vals;
        if (!s.pre) {
            FV_CUDA(cudaMemcpyAsync(c_->pinned, s.counter.get(), 24, cudaMemcpyDeviceToHost, c_->stream));
            FV_CUDA(cudaMemcpyAsync(c_->pinned + 3, r.blocks.count.get(), 8, cudaMemcpyDeviceToHost, c_->stream));
            c_->sync();
            v = c_->pinned;
        }
        s.pre = false;
        *nw = v[0];
        *ov = v[1];
        s.tuples = v[2];
        r.blocks.blocks = v[3];
        s.bound = std::max(s.bound, *nw);
        if (s.chunk_cands) {
            const double got = double(r.blocks.blocks - std::min(r.blocks.blocks, s.chunk_blocks0)) /
                               double(s.chunk_cands);
            r.blocks.ratio = std::max(r.blocks.ratio * 0.5, got);
            s.chunk_cands = 0;
        }
    }

    // Directory capacity for `need` blocks at load <= 1/2; false when that
    // would make the set too sparse to pay (the caller converts it).
    bool block_grow(RelState& r, u64 need, u64 live_keys) {
        BlockSet& b = r.blocks;
        if (b.capacity() && need <= b.capacity() / 2) return true;
        u64 cap = kBlockMinCap, cap2 = kBlockMinCap;
        while (cap < block_headroom_ * need) cap <<= 1;
        while (cap2 < 2 * need) cap2 <<= 1;
        // Sparse (about one row per block): the key set of the rows present
        // is several times smaller; switch once the directory is large
        // (judged at load 1/2 whatever the headroom).
        const double bytes = 136.0 * double(cap2);
        const double keyset_bytes = 8.0 * kKeysetGrowth * double(std::max<u64>(live_keys, 1));
        if (force_blocks_ < 0 && bytes > block_sparse_bytes_ && bytes > kBlockSparseFactor * keyset_bytes) {
            // A word-form relation cannot switch mid-iteration (its DELTA is
            // words): it grows and leaves the word form at the next finalize.
            if (!r.word_sink) return false;
            r.word_sparse = true;
        }
        BlockSet ns;
        engine_blockset_alloc(c_, ns, cap, b.blocks, r.word_sink);
        ns.ratio = b.ratio;
        ns.generation = b.generation + 1;
        if (b.capacity()) engine_blockset_grow(c_, b, ns);
        if (trace_)
            std::fprintf(stderr, "[fvlog]   %s block set -> %llu slots (%llu blocks)\n", r.name.c_str(),
                         static_cast<unsigned long long>(cap), static_cast<unsigned long long>(b.blocks));
        b = std::move(ns);
        return true;
    }

    // Insert the overflow list (n keys) after growing the directory; repeats
    // until the set placed every key.
    void drain_overflow(RelState& r, HeadSink& s, u64 n) {
        while (n) {
            DBuf<u64> tmp(c_, n);
            FV_CUDA(cudaMemcpyAsync(tmp.get(), s.ovf.get(), 8 * n, cudaMemcpyDeviceToDevice, c_->stream));
            FV_CUDA(cudaMemsetAsync(s.counter.get() + 1, 0, 8, c_->stream));
            // At least double the directory (n keys may share far fewer
            // blocks; another round follows if they do not fit). A long list
            // (a seed, a first large iteration) is sized exactly by counting
            // its distinct blocks, so it drains in one round.
            u64 need = std::max(r.blocks.blocks + std::max<u64>(4096, std::min(n, r.blocks.blocks)),
                                r.blocks.capacity() / 2 + 1);
            if (n >= (u64(1) << 16))
                need = std::max(need, r.blocks.blocks + count_blocks(tmp.get(), n, r.arity));
            if (!block_grow(r, need, r.keys.count + s.bound + n)) {
                // too sparse for blocks: the key set takes over, overflow keys included
                convert_to_keyset(r, &s, tmp.get(), n);
                return;
            }
            if (r.word_sink) {
                DBuf<u32> tb(c_, n);
                FV_CUDA(cudaMemcpyAsync(tb.get(), s.ovf_bits.get(), 4 * n, cudaMemcpyDeviceToDevice, c_->stream));
                engine_blockset_word_insert(c_, tmp.get(), tb.get(), n, block_args(r), s.keys.get(), s.widx.get(),
                                            s.counter.get(), s.counter.get() + 2, s.ovf.get(), s.ovf_bits.get(),
                                            s.counter.get() + 1);
            } else {
                engine_blockset_insert(c_, tmp.get(), n, block_args(r), s.keys.get(), s.counter.get(), s.ovf.get(),
                                       s.counter.get() + 1);
            }
            u64 nw;
            read_block_counters(r, s, &nw, &n);
        }
    }

    void block_reserve(RelState& r, HeadSink& s, u64 extra) {
        u64 nw = 0, ov = 0;
        // No directory yet: the sink's count is the prefetched (or fresh,
        // zero) value when there is one, not another round trip.
        const bool pre_known = s.pre;
        const u64 pre_nw = s.pre_vals[0];
        if (r.blocks.capacity()) read_block_counters(r, s, &nw, &ov);
        else s.pre = false;
        if (s.bound + extra > s.cap) {
            const u64 have = r.blocks.capacity() ? nw : pre_known ? pre_nw : sink_count(s);
            const u64 nc = std::max<u64>(have + extra, 2 * s.cap);
            DBuf<u64> nk(c_, nc);
            if (have) FV_CUDA(cudaMemcpyAsync(nk.get(), s.keys.get(), 8 * have, cudaMemcpyDeviceToDevice, c_->stream));
            s.keys = std::move(nk);
            if (r.word_sink) {
                DBuf<u32> nw_idx(c_, nc);
                if (have)
                    FV_CUDA(cudaMemcpyAsync(nw_idx.get(), s.widx.get(), 4 * have, cudaMemcpyDeviceToDevice, c_->stream));
                s.widx = std::move(nw_idx);
            }
            s.cap = nc;
        }
        if (ov) {
            drain_overflow(r, s, ov);
            if (!r.block_mode) return;
        }
        if (s.ovf_cap < extra) {
            s.ovf = DBuf<u64>(c_, extra);
            if (r.word_sink) s.ovf_bits = DBuf<u32>(c_, extra);
            s.ovf_cap = extra;
        }
        s.bound = nw + extra;
        const double ratio = block_ratio_ >= 0 ? block_ratio_ : r.blocks.ratio;
        const u64 est = std::min<u64>(extra, static_cast<u64>(double(extra) * ratio) + (block_ratio_ >= 0 ? 0 : 1024));
        if (!block_grow(r, r.blocks.blocks + est, r.keys.count + nw)) {
            convert_to_keyset(r, &s, nullptr, 0);
            return;
        }
        s.chunk_blocks0 = r.blocks.blocks;
        s.chunk_cands = extra;
        if (nw == 0) s.gen0 = r.blocks.generation;  // no entry recorded yet
    }

    // Replace a relation's block set by a key set holding FULL's rows plus
    // the keys this iteration already found new (sink) and `extra` pending
    // keys (inserted with new-key detection).
    void convert_to_keyset(RelState& r, HeadSink* s, const u64* extra, u64 n_extra) {
        u64 nw = s ? sink_count(*s) : 0;
        const u64 total = r.keys.count + nw + n_extra;
        u64 cap = u64(1) << 16;
        while (cap < kKeysetGrowth * total) cap <<= 1;
        KeySet ns;
        ns.slots = DBuf<u64>(c_, cap);
        ns.mask = cap - 1;
        ns.limit = cap / 2;
        ns.count = r.keys.count;
        ns.group_bits = initial_group_bits();
        FV_CUDA(cudaMemsetAsync(ns.slots.get(), 0xff, 8 * cap, c_->stream));
        std::vector<const DevVersion*> full;
        if (r.levels_mode) full = levels_of(r);
        else full.push_back(&r.full);
        const u64 chunk = u64(1) << 27;
        for (const DevVersion* v : full) {
            for (u64 off = 0; off < v->n; off += chunk) {
                const u64 m = std::min(chunk, v->n - off);
                DBuf<u64> k(c_, m);
                std::vector<const u32*> cols;
                for (auto& col : v->cols) cols.push_back(col.get() + off);
                u64* kp = k.get();
                engine_pack_keys(c_, cols, m, st_.key_shift, &kp);
                engine_hash_insert(c_, k.get(), m, ns, nullptr, nullptr);
            }
        }
        if (nw) engine_hash_insert(c_, s->keys.get(), nw, ns, nullptr, nullptr);
        if (n_extra) engine_hash_insert(c_, extra, n_extra, ns, s->keys.get(), s->counter.get());
        if (trace_)
            std::fprintf(stderr, "[fvlog]   %s block set (%llu blocks, %llu rows) -> key set of %llu slots\n",
                         r.name.c_str(), static_cast<unsigned long long>(r.blocks.blocks),
                         static_cast<unsigned long long>(total), static_cast<unsigned long long>(cap));
        r.keys = std::move(ns);
        r.block_mode = false;
        r.blocks = BlockSet();
        if (s) s->bound = nw + n_extra;
    }

    u32 initial_group_bits() const { return forced_group_ >= 0 ? static_cast<u32>(forced_group_) : 1u; }

    // Re-lay the key set out with `bits` (same capacity): one pass over the
    // old slots, keys re-scattered into the new layout.
    void relayout_keys(RelState& r, u32 bits) {
        KeySet ns;
        ns.slots = DBuf<u64>(c_, r.keys.capacity());
        ns.mask = r.keys.mask;
        ns.limit = r.keys.limit;
        ns.count = r.keys.count;
        ns.group_bits = bits;
        FV_CUDA(cudaMemsetAsync(ns.slots.get(), 0xff, 8 * ns.capacity(), c_->stream));
        engine_hash_rehash(c_, r.keys, ns);
        if (trace_)
            std::fprintf(stderr, "[fvlog]   %s key set -> group_bits %u (%llu slots)\n", r.name.c_str(), bits,
                         static_cast<unsigned long long>(ns.capacity()));
        r.keys = std::move(ns);
    }

    // Word form: the iteration's new words become DELTA (columns x, z base,
    // mask, grouped by x; the counting sort also yields its column-0 join
    // index); returns |DELTA| in tuples.
    // A first large insert into a block set with no growth history (a seed):
    // measure its distinct blocks so the directory is sized before the
    // insert instead of by overflow rounds.
    void estimate_blocks(RelState& r, const CandPool& pool) {
        if (!r.block_mode || r.blocks.ratio > 0 || pool.n < (u64(1) << 16) || block_ratio_ >= 0) return;
        const u64 nb = count_blocks(pool.words[0].get(), pool.n, r.arity);
        r.blocks.ratio = double(nb) / double(pool.n);
    }

    // Distinct blocks of n packed keys, to size a directory: the HyperLogLog
    // sketch (one pass) unless FVLOG_EXACT_BLOCKS=1 (sort + count).
    u64 count_blocks(const u64* keys, u64 n, u32 arity) {
        if (exact_blocks_) return engine_count_blocks(c_, keys, n, st_.key_shift, arity);
        if (!n) return 0;
        DBuf<u32> regs(c_, kBlockSketchRegs);
        engine_block_sketch(c_, keys, n, st_.key_shift, arity, regs.get());
        std::vector<u32> h(kBlockSketchRegs);
        regs.download(h.data(), kBlockSketchRegs);
        return std::min<u64>(n, block_sketch_estimate(h.data()));
    }

    // estimate_blocks for several heads' pools with one read of the counts.
    void estimate_blocks_all(const std::vector<std::pair<RelState*, HeadSink*>>& heads,
                             std::map<std::string, CandPool>& pooled) {
        std::vector<RelState*> need;
        for (auto& [r, s] : heads) {
            const CandPool& pool = pooled.at(r->name);
            if (r->hash_mode && r->block_mode && r->blocks.ratio <= 0 && pool.n >= (u64(1) << 16) && block_ratio_ < 0)
                need.push_back(r);
        }
        if (need.size() < 2) return;  // (a single one reads its count in estimate_blocks)
        std::vector<u64> nb(need.size());
        if (exact_blocks_) {
            DBuf<u64> d(c_, need.size());
            for (size_t q = 0; q < need.size(); ++q) {
                const CandPool& pool = pooled.at(need[q]->name);
                engine_count_blocks_async(c_, pool.words[0].get(), pool.n, st_.key_shift, need[q]->arity, d.get() + q);
            }
            d.download(nb.data(), need.size());
        } else {
            DBuf<u32> regs(c_, kBlockSketchRegs * need.size());
            for (size_t q = 0; q < need.size(); ++q) {
                const CandPool& pool = pooled.at(need[q]->name);
                engine_block_sketch(c_, pool.words[0].get(), pool.n, st_.key_shift, need[q]->arity,
                                    regs.get() + kBlockSketchRegs * q);
            }
            std::vector<u32> h(kBlockSketchRegs * need.size());
            regs.download(h.data(), h.size());
            for (size_t q = 0; q < need.size(); ++q)
                nb[q] = std::min<u64>(pooled.at(need[q]->name).n, block_sketch_estimate(h.data() + kBlockSketchRegs * q));
        }
        for (size_t q = 0; q < need.size(); ++q)
            need[q]->blocks.ratio = double(nb[q]) / double(pooled.at(need[q]->name).n);
    }

    // Insert a head's pooled candidates (copies, unfused joins) into its set;
    // the new keys join the ones the fused joins appended.
    void insert_pool(RelState& r, HeadSink& s, CandPool& pool) {
        if (!r.hash_mode) return;
        estimate_blocks(r, pool);
        if (!pool.n) return;
        hash_reserve(r, s, pool.n);
        if (r.word_sink)
            engine_blockset_word_insert(c_, pool.words[0].get(), nullptr, pool.n, block_args(r), s.keys.get(),
                                        s.widx.get(), s.counter.get(), s.counter.get() + 2, s.ovf.get(),
                                        s.ovf_bits.get(), s.counter.get() + 1);
        else if (r.block_mode)
            engine_blockset_insert(c_, pool.words[0].get(), pool.n, block_args(r), s.keys.get(), s.counter.get(),
                                   s.ovf.get(), s.counter.get() + 1);
        else
            engine_hash_insert(c_, pool.words[0].get(), pool.n, r.keys, s.keys.get(), s.counter.get());
        s.candidates += pool.n;
        pool.n = 0;
    }

    // The set counters of several heads in one host round trip (the next
    // read_block_counters of each uses them).
    void prefetch_counters(const std::vector<std::pair<RelState*, HeadSink*>>& heads) {
        std::vector<std::pair<RelState*, HeadSink*>> live;
        for (auto& [r, s] : heads)
            if (r->block_mode && r->blocks.capacity() && s->counter.get()) live.emplace_back(r, s);
        if (live.empty()) return;
        if (batch_pinned_cap_ < 4 * live.size()) {
            if (batch_pinned_) cudaFreeHost(batch_pinned_);
            batch_pinned_cap_ = std::max<size_t>(256, 8 * live.size());
            FV_CUDA(cudaMallocHost(&batch_pinned_, sizeof(u64) * batch_pinned_cap_));
        }
        for (size_t q = 0; q < live.size(); ++q) {
            FV_CUDA(cudaMemcpyAsync(batch_pinned_ + 4 * q, live[q].second->counter.get(), 24, cudaMemcpyDeviceToHost,
                                    c_->stream));
            FV_CUDA(cudaMemcpyAsync(batch_pinned_ + 4 * q + 3, live[q].first->blocks.count.get(), 8,
                                    cudaMemcpyDeviceToHost, c_->stream));
        }
        c_->sync();
        for (size_t q = 0; q < live.size(); ++q) {
            HeadSink& s = *live[q].second;
            s.pre = true;
            for (int k = 0; k < 4; ++k) s.pre_vals[k] = batch_pinned_[4 * q + k];
        }
    }

    u64 word_finalize(RelState& r, HeadSink& s, CandPool& pool) {
        insert_pool(r, s, pool);
        u64 nw = 0, ov = 0;
        if (s.counter.get()) {
            read_block_counters(r, s, &nw, &ov);
            if (ov) {
                drain_overflow(r, s, ov);
                read_block_counters(r, s, &nw, &ov);
            }
        }
        const u64 tuples = s.counter.get() ? s.tuples : 0;
        if (!r.word_mode) {
            // Word sink with a tuple DELTA: the merged words of the
            // iteration become DELTA's tuples.
            if (nw) {
                s.bits = DBuf<u32>(c_, nw);
                const bool idx_ok = s.gen0 == r.blocks.generation && r.blocks.capacity() <= (u64(1) << 27);
                engine_blockset_collect(c_, s.keys.get(), idx_ok ? s.widx.get() : nullptr, nw, block_args(r),
                                        s.bits.get());
            }
            if (nw && grouped_expand_ && r.levels_mode && r.arity == 2) {
                // Group the word entries by x (counting sort over words, not
                // tuples), then expand them: the tuples come out grouped by x
                // with no tuple-level sort or scatter.
                DBuf<u32> wb(c_, nw);
                JoinIndex word_runs;
                if (engine_group_keys(c_, s.keys, nw, st_.key_shift, &word_runs, nullptr, nullptr, s.bits.get(),
                                      wb.get())) {
                    const u64 nd = install_word_delta(r, s.keys.get(), wb.get(), nw, tuples, &word_runs);
                    s.keys = DBuf<u64>();
                    s.cap = 0;
                    if (r.word_sparse && !r.temp) leave_word_mode(r);
                    return nd;
                }
            }
            // ... else expand to packed tuple keys, then the usual path.
            DBuf<u64> tk(c_, std::max<u64>(tuples, 1));
            if (nw) engine_expand_word_keys(c_, s.keys.get(), s.bits.get(), nw, tk.get());
            s.keys = DBuf<u64>();
            s.cap = 0;
            const u64 nd = finish_delta(r, std::move(tk), tuples);
            if (r.word_sparse && !r.temp) leave_word_mode(r);
            return nd;
        }
        invalidate(r);
        if (r.delta.n) r.levels.push_back(std::move(r.delta));
        DevVersion Dv;
        Dv.n = nw;
        for (u32 j = 0; j <= r.arity; ++j) Dv.cols.emplace_back(c_, nw);
        if (nw == 0) {
            r.delta = std::move(Dv);
            set_old(r, nullptr);
            if (r.word_sparse && !r.temp) leave_word_mode(r);
            return 0;
        }
        r.keys.count += tuples;
        r.level_rows += tuples;
        // One entry per word first written this iteration; its merged mask
        // is read (and cleared) from the DELTA bitmap.
        s.bits = DBuf<u32>(c_, nw);
        const bool idx_ok = s.gen0 == r.blocks.generation && r.blocks.capacity() <= (u64(1) << 27);
        auto delta_index = std::make_unique<JoinIndex>();
        // With valid recorded word indices the grouping scatter reads the
        // masks from the DELTA bitmap itself (no collect pass).
        bool grouped = idx_ok && scatter_gather_ && engine_group_keys(c_, s.keys, nw, st_.key_shift, delta_index.get(), Dv.cols[0].get(),
                                                   Dv.cols[1].get(), nullptr, Dv.cols[2].get(), s.widx.get(),
                                                   r.blocks.dbits.get());
        if (!grouped) {
            engine_blockset_collect(c_, s.keys.get(), idx_ok ? s.widx.get() : nullptr, nw, block_args(r),
                                    s.bits.get());
            grouped = engine_group_keys(c_, s.keys, nw, st_.key_shift, delta_index.get(), Dv.cols[0].get(),
                                        Dv.cols[1].get(), s.bits.get(), Dv.cols[2].get());
        }
        if (!grouped) {
            // Domain too large for the counting sort: unpack, then order the
            // entries by x (stable LSD pass over column 0) and gather.
            std::vector<u32*> dc{Dv.cols[0].get(), Dv.cols[1].get()};
            engine_unpack_keys(c_, s.keys.get(), nw, 2, st_.key_shift, dc);
            FV_CUDA(cudaMemcpyAsync(Dv.cols[2].get(), s.bits.get(), 4 * nw, cudaMemcpyDeviceToDevice, c_->stream));
            const u32* order_cols[1] = {Dv.cols[0].get()};
            DBuf<u32> perm = lexicographic_order(c_, order_cols, 1, nw);
            DevVersion G;
            G.n = nw;
            for (u32 j = 0; j <= r.arity; ++j) {
                DBuf<u32> g(c_, nw);
                gather_u32(c_, Dv.cols[j].get(), perm.get(), g.get(), nw);
                G.cols.push_back(std::move(g));
            }
            Dv = std::move(G);
        }
        s.cap = 0;
        r.delta = std::move(Dv);
        if (grouped) {
            delta_index->rows = &r.delta;
            r.indexes.emplace(std::make_pair(static_cast<int>(kDelta), 0u), std::move(delta_index));
        }
        if (r.word_sparse && !r.temp) leave_word_mode(r);
        return tuples;
    }

    // Levels-mode binary relation: DELTA = the tuples of nw word entries
    // (word key, mask) already grouped by x (nd tuples in all), with its
    // column-0 direct index; the previous DELTA becomes a level.
    u64 install_word_delta(RelState& r, const u64* wkeys, const u32* wb, u64 nw, u64 nd,
                           const JoinIndex* word_runs = nullptr) {
        invalidate(r);
        if (r.delta.n) r.levels.push_back(std::move(r.delta));
        DevVersion Dv;
        Dv.n = nd;
        for (u32 j = 0; j < 2; ++j) Dv.cols.emplace_back(c_, std::max<u64>(nd, 1));
        r.keys.count += nd;
        r.level_rows += nd;
        DBuf<u64> off(c_, nw + 1);
        engine_expand_word_keys(c_, wkeys, wb, nw, nullptr, Dv.cols[0].get(), Dv.cols[1].get(), st_.key_shift,
                                off.get());
        auto di = std::make_unique<JoinIndex>();
        // DELTA's column-0 index from the words' runs (one pass over the
        // value domain) instead of a pass over the expanded tuples
        if (word_runs && word_runs->domain && word_runs->ucount.get())
            engine_word_index_to_tuples(c_, *word_runs, off.get(), *di);
        else
            engine_build_runs(c_, Dv.cols[0].get(), nd, *di, st_.key_shift, true);
        r.delta = std::move(Dv);
        di->rows = &r.delta;
        r.indexes.emplace(std::make_pair(static_cast<int>(kDelta), 0u), std::move(di));
        return nd;
    }

    // Word-form version -> tuple form (grouping by x is kept).
    void to_tuples(DevVersion& v, u32 arity) {
        if (v.cols.size() != arity + 1) return;
        DevVersion t;
        // one pass counts the tuples (sizes the output), the second writes them
        t.n = engine_expand_words(c_, v.cols[0].get(), v.cols[1].get(), v.cols[2].get(), v.n, nullptr, nullptr);
        t.cols.emplace_back(c_, t.n);
        t.cols.emplace_back(c_, t.n);
        engine_expand_words(c_, v.cols[0].get(), v.cols[1].get(), v.cols[2].get(), v.n, t.cols[0].get(),
                            t.cols[1].get());
        v = std::move(t);
    }

    // Leave the word form (the block set proved sparse): DELTA and the levels
    // become tuples and the relation converts to a key set.
    void leave_word_mode(RelState& r) {
        to_tuples(r.delta, r.arity);
        for (auto& lv : r.levels) to_tuples(lv, r.arity);
        invalidate(r);
        r.word_mode = false;
        r.word_sink = false;
        r.word_sparse = false;
        if (trace_) std::fprintf(stderr, "[fvlog]   %s leaves the word form\n", r.name.c_str());
        convert_to_keyset(r, nullptr, nullptr, 0);
    }

    // Sort the iteration's new keys into Δ and fold them into FULL.
    u64 hash_finalize(RelState& r, HeadSink& s, CandPool& pool) {
        if (r.word_sink) return word_finalize(r, s, pool);
        insert_pool(r, s, pool);
        u64 nd = 0;
        if (r.block_mode && s.counter.get()) {
            u64 ov;
            read_block_counters(r, s, &nd, &ov);
            if (ov) {
                drain_overflow(r, s, ov);
                nd = sink_count(s);  // the drain may also have converted the set
            }
        } else {
            nd = sink_count(s);
        }
        if (!r.block_mode && forced_group_ < 0 && r.keys.capacity() && s.candidates) {
            const u32 want = double(s.candidates) <= group_ratio_ * double(std::max<u64>(nd, 1)) ? 1u : 0u;
            if (trace_)
                std::fprintf(stderr, "[fvlog]   %s candidates/new = %.3f\n", r.name.c_str(),
                             double(s.candidates) / double(std::max<u64>(nd, 1)));
            if (want != r.keys.group_bits) relayout_keys(r, want);
        }
        DBuf<u64> keys = std::move(s.keys);
        s.cap = 0;
        return finish_delta(r, std::move(keys), nd);
    }

    // Merge DELTA (just built, sorted by column 0) into the (col 1, col 0)
    // ordered copy of FULL: sort DELTA's (col 1, col 0) keys, one merge-path
    // pass, the column-1 run index rebuilt.
    void advance_by1(RelState& r, const DevVersion& d) {
        JoinIndex& o = *r.by1;
        const u64 nd = d.n, nf = o.rows->n;
        std::vector<DBuf<u64>> words;
        words.emplace_back(c_, nd);
        u64* wp = words[0].get();
        engine_pack_keys(c_, std::vector<const u32*>{d.cols[1].get(), d.cols[0].get()}, nd, st_.key_shift, &wp);
        engine_sort_keys(c_, words, nd, 2, st_.key_shift);
        DevVersion C, unused;
        for (int j = 0; j < 2; ++j) {
            C.cols.emplace_back(c_, nf + nd);
            unused.cols.emplace_back(c_, nd);
        }
        std::vector<u64*> bw{words[0].get()};
        // merge order (col 1, col 0); C keeps column semantics (cols[1] = col 1)
        engine_merge(c_, std::vector<const u32*>{o.rows->cols[1].get(), o.rows->cols[0].get()}, nf, bw.data(), nd, 2,
                     st_.key_shift, std::vector<u32*>{C.cols[1].get(), C.cols[0].get()},
                     std::vector<u32*>{unused.cols[1].get(), unused.cols[0].get()}, c_->d_scalars + 47);
        C.n = nf + nd;
        auto ni = std::make_unique<JoinIndex>();
        ni->owned = std::move(C);
        ni->rows = &ni->owned;
        engine_build_runs(c_, ni->owned.cols[1].get(), ni->owned.n, *ni, st_.key_shift);
        // the replaced copy is FULL - DELTA's (exactly-once variants probe it)
        r.old_by1 = r.keep_old && !r.old_is_full ? std::move(r.by1) : nullptr;
        r.by1 = std::move(ni);
        if (trace_)
            std::fprintf(stderr, "[fvlog]   %s (col 1, col 0) copy: +%llu rows by merge\n", r.name.c_str(),
                         static_cast<unsigned long long>(nd));
    }

    // The iteration's nd new packed tuple keys become DELTA (grouped by
    // column 0 in levels mode, sorted and merged into FULL otherwise).
    u64 finish_delta(RelState& r, DBuf<u64>&& new_keys, u64 nd) {
        // FULL's word build becomes the build of FULL - DELTA when the merge
        // keeps the replaced FULL (exactly-once variants read it).
        std::unique_ptr<WordBuild> full_words;
        if (auto it = r.word_builds.find(static_cast<int>(kFull)); it != r.word_builds.end())
            full_words = std::move(it->second);
        invalidate(r);
        DevVersion Dv;
        Dv.n = nd;
        for (u32 j = 0; j < r.arity; ++j) Dv.cols.emplace_back(c_, nd);
        // Levels mode: the previous DELTA becomes a level (moved, no copy);
        // the current DELTA is the newest level until the next iteration.
        if (r.levels_mode && r.delta.n) r.levels.push_back(std::move(r.delta));
        if (nd == 0) {
            r.delta = std::move(Dv);
            set_old(r, nullptr);
            return 0;
        }
        r.keys.count += nd;
        std::vector<DBuf<u64>> words;
        words.push_back(std::move(new_keys));
        // Levels-mode FULL is never merged, so Δ only has to be grouped by
        // column 0 (its join index): unary keys are distinct (already
        // grouped), binary keys take a counting sort on column 0 when its
        // domain is small, else the column-0 radix passes. A sorted FULL
        // needs the full order.
        // The counting sort also yields DELTA's column-0 join index (its runs
        // are the non-empty counters), installed below once DELTA is in place.
        auto delta_index = std::make_unique<JoinIndex>();
        bool have_index = false;
        if (!r.levels_mode) {
            engine_sort_keys(c_, words, nd, r.arity, st_.key_shift);
        } else if (r.arity == 2) {
            // The scatter writes DELTA's columns directly (no unpack pass).
            have_index = engine_group_keys(c_, words[0], nd, st_.key_shift, delta_index.get(), Dv.cols[0].get(),
                                           Dv.cols[1].get());
            if (!have_index) engine_sort_keys(c_, words, nd, r.arity, st_.key_shift, true);
        }
        if (!have_index) {
            std::vector<u32*> dc;
            for (auto& col : Dv.cols) dc.push_back(col.get());
            engine_unpack_keys(c_, words[0].get(), nd, r.arity, st_.key_shift, dc);
        }
        if (r.levels_mode) {
            r.level_rows += nd;
        } else {
            // FULL is read by joins: keep it one sorted version.
            DevVersion C, unused;
            for (u32 j = 0; j < r.arity; ++j) {
                C.cols.emplace_back(c_, r.full.n + nd);
                unused.cols.emplace_back(c_, nd);
            }
            std::vector<u64*> bw{words[0].get()};
            std::vector<u32*> cc, uc;
            for (u32 j = 0; j < r.arity; ++j) {
                cc.push_back(C.cols[j].get());
                uc.push_back(unused.cols[j].get());
            }
            u64* d_new = c_->d_scalars + 23;
            engine_merge(c_, r.full.ptrs(), r.full.n, bw.data(), nd, r.arity, st_.key_shift, cc, uc, d_new);
            C.n = r.full.n + nd;
            C.lex_sorted = true;
            Dv.lex_sorted = true;  // unpacked from the sorted keys
            set_old(r, &r.full);
            r.full = std::move(C);
            if (r.by1) advance_by1(r, Dv);
            if (!r.old_is_full && full_words) r.word_builds.emplace(static_cast<int>(kOld), std::move(full_words));
        }
        r.delta = std::move(Dv);
        if (have_index) {
            delta_index->rows = &r.delta;
            r.indexes.emplace(std::make_pair(static_cast<int>(kDelta), 0u), std::move(delta_index));
        }
        return nd;
    }

    void allreduce(std::vector<u64>& v) {
        if (dist() && !v.empty()) c_->tx->allreduce_sum(c_, v.data(), static_cast<int>(v.size()));
    }
    u32 world() const { return world_; }
    u32 rank() const { return rank_; }

public:
    ~Engine() {
        if (batch_pinned_) cudaFreeHost(batch_pinned_);
    }

private:
    Ctx* c_;
    EvalState& st_;
    u64* batch_pinned_ = nullptr;  // prefetch_counters staging
    size_t batch_pinned_cap_ = 0;
    bool force_partitioned_ = false;
    std::map<InterKey, InterPolicy> inter_policy_;
    const bool trace_ = std::getenv("FVLOG_TRACE") != nullptr;
    static u64 env_rows(const char* name, u64 dflt) {
        const char* e = std::getenv(name);
        return e && std::atoll(e) > 0 ? static_cast<u64>(std::atoll(e)) : dflt;
    }
    const u64 pool_chunk_ = env_rows("FVLOG_POOL_CHUNK", kPoolChunk);
    const u64 inter_chunk_ = env_rows("FVLOG_INTER_CHUNK", kInterChunk);
    // FVLOG_INTER_PROBE_ROWS (tests): the intermediate size at which repeats are first measured.
    const u64 inter_probe_rows_ = env_rows("FVLOG_INTER_PROBE_ROWS", kInterProbeRows);
    const u64 pool_budget_ = env_rows("FVLOG_POOL_BUDGET", kPoolBudget);
    const double group_ratio_ = [] {
        const char* e = std::getenv("FVLOG_GROUP_RATIO");
        return e ? std::atof(e) : kGroupedRatio;
    }();
    const int forced_group_ = [] {
        const char* e = std::getenv("FVLOG_KEYSET_GROUP");
        return e ? std::atoi(e) : -1;
    }();
    // FVLOG_GROW=rehash: key-set growth by memset + atomic rehash only.
    const bool grow_windowed_ = [] {
        const char* e = std::getenv("FVLOG_GROW");
        return !(e && std::string(e) == "rehash");
    }();
    // FVLOG_SET=keyset: key sets only; =blocks: block sets even when sparse.
    const int force_blocks_ = [] {
        const char* e = std::getenv("FVLOG_SET");
        return e ? (std::string(e) == "blocks" ? 1 : 0) : -1;
    }();
    // Tests: FVLOG_BLOCK_RATIO fixes the new-blocks-per-candidate estimate
    // (0 provokes overflow lists), FVLOG_BLOCK_SPARSE_BYTES the directory
    // size below which a sparse relation keeps its block set.
    const double block_ratio_ = [] {
        const char* e = std::getenv("FVLOG_BLOCK_RATIO");
        return e ? std::atof(e) : -1.0;
    }();
    const double block_sparse_bytes_ = [] {
        const char* e = std::getenv("FVLOG_BLOCK_SPARSE_BYTES");
        return e ? std::atof(e) : kBlockSparseMinBytes;
    }();
    // FVLOG_BY1=0: column-1 indexes of FULL re-sorted per iteration instead
    // of maintained by merge.
    const bool by1_ = [] {
        const char* e = std::getenv("FVLOG_BY1");
        return !(e && std::string(e) == "0");
    }();
    // FVLOG_WORDS=0: no word sinks, word builds or word intermediates.
    const bool words_ = [] {
        const char* e = std::getenv("FVLOG_WORDS");
        return !(e && std::string(e) == "0");
    }();
    // FVLOG_WORD_COMBINE=0: no tile-local OR-combine of word-form outputs.
    const u32 word_combine_ = [] {
        const char* e = std::getenv("FVLOG_WORD_COMBINE");
        return e ? static_cast<u32>(std::atoi(e) != 0) : 1u;
    }();
    // FVLOG_BLOCK_HEADROOM=h: a growing directory gets >= h x the blocks
    // it must hold (grows again at load 1/2). Measured h = 2 / 4 / 8: C2 20.7
    // / 20.0 / 22.2 ms, C4 62.2 / 60.9 ms (half the growth passes; 8 spreads
    // the directory past what stays in L2).
    const u64 block_headroom_ = [] {
        const char* e = std::getenv("FVLOG_BLOCK_HEADROOM");
        return e ? std::max<u64>(2, std::strtoull(e, nullptr, 10)) : u64(4);
    }();
    // FVLOG_EXACT_BLOCKS=1: directory sizes from an exact distinct-block
    // count (54-bit radix sort) instead of the HyperLogLog sketch.
    const bool exact_blocks_ = [] {
        const char* e = std::getenv("FVLOG_EXACT_BLOCKS");
        return e && std::string(e) == "1";
    }();
    // FVLOG_PROBE_SCAN=0: probe counts written by one kernel and scanned by
    // another instead of one fused single-pass probe + scan.
    const bool fused_probe_scan_ = [] {
        const char* e = std::getenv("FVLOG_PROBE_SCAN");
        return !(e && std::string(e) == "0");
    }();
    // FVLOG_GROUPED_EXPAND=0: a word sink's tuple DELTA is expanded to
    // packed keys and grouped by a tuple-level counting sort instead of
    // grouping the word entries and expanding them in place.
    const bool grouped_expand_ = [] {
        const char* e = std::getenv("FVLOG_GROUPED_EXPAND");
        return !(e && std::string(e) == "0");
    }();
    // FVLOG_SCATTER_GATHER=1: the grouping scatter reads a word-form DELTA's
    // masks from the DELTA bitmap itself instead of a separate collect pass
    // (C2: 25.2 vs 24.85 ms per fixpoint with the collect pass, so off).
    const bool scatter_gather_ = [] {
        const char* e = std::getenv("FVLOG_SCATTER_GATHER");
        return e && std::string(e) == "1";
    }();
    // FVLOG_BLOCK_TILE_SET=0: no tile-local dedup before the block-set probe.
    const u32 block_tile_set_ = [] {
        const char* e = std::getenv("FVLOG_BLOCK_TILE_SET");
        return e ? static_cast<u32>(std::atoi(e) != 0) : 1u;
    }();

public:
    bool blocks_enabled() const { return force_blocks_ != 0; }

private:
    u32 world_ = 1, rank_ = 0;
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
    Engine eng(c, *st);
    st->rank = static_cast<int>(eng.rank());
    st->world = static_cast<int>(eng.world());
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
    u64* dmax = c->d_scalars + 22;  // one max over every EDB column, one readback
    FV_CUDA(cudaMemsetAsync(dmax, 0, sizeof(u64), c->stream));
    {
        std::vector<std::pair<const u32*, u64>> cols;  // every EDB column, one launch
        for (auto& [name, vp] : raw)
            for (auto& col : vp->cols)
                if (vp->n) cols.emplace_back(col.get(), vp->n);
        reduce_max_u32_multi(c, cols, dmax);
    }
    {
        u64 m = 0;
        c->read_scalars(dmax, &m, 1);
        vmax = std::max(vmax, m);
    }
    if (eng.dist()) {  // every rank must pack keys with the same shift
        std::vector<u64> bits(64, 0);
        bits[bit_width_u64(vmax)] = 1;
        eng.allreduce(bits);
        for (u32 b = 0; b < 64; ++b)
            if (bits[b]) vmax = std::max<u64>(vmax, b ? (u64(1) << (b - 1)) : 0);
    }
    st->key_shift = std::max<u32>(1, bit_width_u64(vmax));

    // ---- variants (delta_rewrite, engine.cpp:57-64) --------------------------
    struct Variant {
        const Plan* plan;
        long delta_source;
        size_t plan_index;     // index into dplans
        std::vector<u8> old_src;  // per executed source: read FULL - DELTA
        // Reversed orientation of a two-atom word composition (DELTA first,
        // probing its words against the other atom indexed on the join
        // column): chosen when DELTA's words are few next to the other atom,
        // and always in partitioned runs (the other atom is replicated, DELTA
        // is this rank's share).
        const Plan* alt = nullptr;
        size_t alt_index = 0;
        std::vector<u8> alt_old;  // old_src of the alternative order
    };
    std::vector<DistPlan> dplans;
    std::deque<Plan> reordered;  // delta-first plans (stable addresses)
    std::vector<Variant> variants;
    std::set<std::string> full_read;  // relations whose FULL some variant reads
    // FVLOG_JOIN_ORDER=rule keeps every variant in the rule's atom order.
    const char* order_env = std::getenv("FVLOG_JOIN_ORDER");
    const bool delta_first = !(order_env && std::string(order_env) == "rule");
    // Exactly-once variants (single GPU): the variant with DELTA at IDB
    // occurrence i reads FULL - DELTA at the IDB occurrences before i and FULL
    // after it, so a derivation using several DELTA rows is produced by one
    // variant instead of each (the reference reads FULL everywhere,
    // P/src/engine.cpp:180-183). The union over variants is the same set.
    // FVLOG_SEMINAIVE=reference restores the reference's variants.
    const char* sn_env = std::getenv("FVLOG_SEMINAIVE");
    const bool exactly_once = !eng.dist() && !(sn_env && std::string(sn_env) == "reference");
    for (size_t i = 0; i < plans.size(); ++i) {
        const Plan& p = plans[i];
        bool any = false;
        for (size_t s = 0; s < p.sources.size(); ++s)
            if (idb.count(p.sources[s].relation)) {
                Plan rp;
                // Only chains of >= 3 atoms where an IDB atom precedes DELTA
                // (the rule order would join two growing FULL relations
                // first); for two atoms the rule order probes FULL against
                // DELTA's index, cheaper than a per-iteration sorted copy of
                // FULL on another column, and an EDB prefix is fixed-size.
                bool idb_before = false;
                for (size_t q = 0; q < s; ++q) idb_before = idb_before || idb.count(p.sources[q].relation) > 0;
                // old_by_rule[q]: rule atom q reads FULL - DELTA in this variant.
                std::vector<u8> old_by_rule(p.sources.size(), 0);
                if (exactly_once)
                    for (size_t q = 0; q < s; ++q) old_by_rule[q] = idb.count(p.sources[q].relation) ? 1 : 0;
                std::vector<u32> order;
                if (delta_first && idb_before && p.sources.size() >= 3 &&
                    delta_first_plan(p, static_cast<u32>(s), rp, &order)) {
                    std::vector<u8> old_src(order.size());
                    for (size_t i = 0; i < order.size(); ++i) old_src[i] = old_by_rule[order[i]];
                    reordered.push_back(std::move(rp));
                    variants.push_back({&reordered.back(), 0, variants.size(), std::move(old_src)});
                } else {
                    variants.push_back({&p, static_cast<long>(s), variants.size(), old_by_rule});
                }
                any = true;
            }
        if (!any) variants.push_back({&p, -1, variants.size(), {}});
    }
    // Partitioned runs: home columns from the executed variants, then each
    // variant's static partitioning decisions.
    {
        std::map<std::string, u32> idb_arity;
        for (auto& [name, r] : st->relations)
            if (r->idb) idb_arity[name] = r->arity;
        std::vector<std::pair<const Plan*, long>> pv;
        for (auto& v : variants) pv.emplace_back(v.plan, v.delta_source);
        const std::map<std::string, u32> home = eng.dist() ? choose_home_cols(pv, idb_arity) : std::map<std::string, u32>();
        for (auto& [name, col] : home) st->relations.at(name)->home = col;
        for (auto& v : variants) dplans.push_back(dist_plan(*v.plan, idb, home));
        for (auto& v : variants) {
            const Plan& p = *v.plan;
            if (v.delta_source != 1 || p.sources.size() != 2 || !Engine::word_step_ok(p, 0)) continue;
            Plan rp;
            std::vector<u32> order;
            if (!delta_first_plan(p, 1, rp, &order)) continue;
            // The other atom becomes the build side, probed on its join
            // column: only when that index is cheap — column 0 (a run index
            // of the sorted version) or a static EDB relation.
            if (rp.joins[0].right_col != 0 && idb.count(rp.sources[1].relation)) continue;
            reordered.push_back(std::move(rp));
            v.alt = &reordered.back();
            v.alt_old = {0, v.old_src.empty() ? u8(0) : v.old_src[0]};
            dplans.push_back(dist_plan(*v.alt, idb, home));
            v.alt_index = dplans.size() - 1;
        }
    }
    for (auto& v : variants)
        for (size_t s = 0; s < v.plan->sources.size(); ++s) {
            if (static_cast<long>(s) == v.delta_source) continue;
            full_read.insert(v.plan->sources[s].relation);
            if (!v.old_src.empty() && v.old_src[s]) st->relations.at(v.plan->sources[s].relation)->keep_old = true;
        }
    // Partition copies each IDB relation needs (static in the executed variant plans).
    if (eng.dist()) {
        for (auto& [name, r] : st->relations)
            if (r->idb) r->keyset.insert(r->home);
        for (auto& v : variants) {
            const Plan& p = *v.plan;
            const DistPlan& dp = dplans[v.plan_index];
            for (u32 s = 0; s < p.sources.size(); ++s) {
                RelState& r = *st->relations.at(p.sources[s].relation);
                if (r.idb) r.keyset.insert(dp.src_copy[s]);
            }
        }
        for (auto& [name, r] : st->relations)
            for (u32 kc : r->keyset)
                if (kc != r->home) {
                    auto cp = std::make_unique<RelCopy>();
                    cp->full.cols.resize(r->arity);
                    cp->delta.cols.resize(r->arity);
                    r->copies.emplace(kc, std::move(cp));
                }
    }

    // Dedup strategy per relation: a key set for binary/unary relations (keys
    // are one u64 word that can never equal the empty slot), the sort +
    // merge-path pipeline otherwise. FVLOG_DEDUP=sort forces the latter.
    const char* mode = std::getenv("FVLOG_DEDUP");
    const bool hash_ok = !(mode && std::string(mode) == "sort");
    for (auto& [name, r] : st->relations) {
        r->hash_mode = hash_ok && r->idb && r->arity <= 2 && (r->arity == 1 || 2 * st->key_shift < 64);
        r->levels_mode = r->hash_mode && !full_read.count(name);
        r->block_mode = r->hash_mode && eng.blocks_enabled();
    }
    // Word sinks (RelState::word_sink, single GPU): binary block-set
    // relations that head at least one word composition step (a last join
    // step whose right atom is joined on its column 0 and gives the head's
    // column 1, Engine::word_step_ok) take every insert as words.
    // Word DELTA (RelState::word_mode): a levels-mode word sink whose DELTA is
    // only ever read as the right atom of such a step into a word sink — e.g.
    // right-linear TC, reach(x, z) :- edge(x, y), reach(y, z) — keeps DELTA
    // and the levels as words. FVLOG_WORDS=0 disables both.
    // Partitioned runs: only the word DELTA of a relation whose every
    // derivation stays where it is produced — the composition variants local
    // (homed on the column they carry, z) and the copies replicated
    // (owner-filtered) — with no partition copies; the home column's owner is
    // then taken over 32-value windows (owner_shift 5) so a word never
    // straddles two ranks.
    const char* words_env = std::getenv("FVLOG_WORDS");
    if (!(words_env && std::string(words_env) == "0")) {
        auto last_step = [](const Plan& p) { return p.joins.size() - 1; };
        if (!eng.dist()) {
            for (auto& v : variants) {
                const Plan& p = *v.plan;
                RelState& h = *st->relations.at(p.head);
                if (h.block_mode && h.arity == 2 && !p.joins.empty() && Engine::word_step_ok(p, last_step(p)))
                    h.word_sink = true;
            }
        }
        for (auto& [name, r] : st->relations) {
            if (!(r->block_mode && r->levels_mode && r->arity == 2)) continue;
            if (!eng.dist() && !r->word_sink) continue;
            bool ok = !eng.dist() || (r->home == 1 && r->keyset == std::set<u32>{1});
            bool any = false;
            for (auto& v : variants) {
                const Plan& p = *v.plan;
                const DistPlan& dp = dplans[v.plan_index];
                const bool reads_delta = v.delta_source >= 0 && p.sources[v.delta_source].relation == name;
                const bool composes = reads_delta && !p.joins.empty() &&
                                      static_cast<u32>(v.delta_source) == p.joins[last_step(p)].right_source &&
                                      Engine::word_step_ok(p, last_step(p));
                if (eng.dist()) {
                    // only the exchange-free TC shape: head == r, composition local, copies replicated
                    if (p.head == name && !p.joins.empty()) {
                        if (composes && p.sources.size() == 2 && dp.local_out) any = true;
                        else ok = false;
                    } else if (p.head == name) {
                        if (!dp.replicated_out) ok = false;
                    } else if (reads_delta) {
                        ok = false;
                    }
                    continue;
                }
                if (!reads_delta) continue;
                if (composes && st->relations.at(p.head)->word_sink) any = true;
                else ok = false;
            }
            r->word_mode = ok && any;
            if (r->word_mode) r->word_sink = true;
            if (r->word_mode && eng.dist()) r->owner_shift = 5;
        }
    }

    const bool trace = std::getenv("FVLOG_TRACE") != nullptr;
    // FVLOG_REVERSE=0: two-atom word compositions always probe in rule
    // order; =1: always reversed (when eligible); unset: by size.
    const char* rev_env = std::getenv("FVLOG_REVERSE");
    const bool reverse_env = !(rev_env && std::string(rev_env) == "0");
    const bool reverse_always = rev_env && std::string(rev_env) == "1";
    // FVLOG_REVERSE_RATIO=r: reverse a two-atom composition when r * |DELTA|
    // is below the other atom's size (default 4; measured 2 / 4 / 8 / never:
    // C2 21.19 / 20.67 / 20.67 / 20.73 ms, C4 62.2 / 62.3 / 62.6 / 64.0).
    const char* rr_env = std::getenv("FVLOG_REVERSE_RATIO");
    const double reverse_ratio = rr_env ? std::atof(rr_env) : 4.0;
    // FVLOG_SEED_BATCH=0: every sort-merged relation's seed sorts on its own.
    const char* sb_env = std::getenv("FVLOG_SEED_BATCH");
    const bool seed_batch_env = !(sb_env && std::string(sb_env) == "0");
    // FVLOG_PRECOUNT=0: every join step reads its own output size.
    const char* pc_env = std::getenv("FVLOG_PRECOUNT");
    const bool precount_env = !(pc_env && std::string(pc_env) == "0");
    u64 syncs_seen = c->syncs;
    auto tr = [&](const char* what, Clock::time_point t, u64 it) {
        if (trace) {
            // host syncs of the phase (the trace's own sync not counted)
            const u64 phase_syncs = c->syncs - syncs_seen;
            c->sync();
            syncs_seen = c->syncs;
            std::fprintf(stderr, "[fvlog] it=%llu %-10s %.3f ms  host syncs %llu\n", static_cast<unsigned long long>(it),
                         what, ms_since(t), static_cast<unsigned long long>(phase_syncs));
        }
    };
    if (trace) tr("setup", t0, 0);
    // ---- seed: FULL = DELTA = dedup(EDB) (engine.cpp:148-161) ---------------
    const auto ts = Clock::now();
    {
        std::vector<Engine::PendingMerge> pend;
        // sort-merged single-GPU relations of arity <= 2: one shared sort
        std::vector<std::pair<RelState*, const DevVersion*>> batch;
        for (auto& [name, vp] : raw) {
            RelState& r = *st->relations[name];
            if (seed_batch_env && !eng.partitioned(r) && !r.hash_mode && r.arity <= 2 && vp->n)
                batch.emplace_back(&r, vp);
        }
        const bool batched = eng.seed_batch(batch, pend);
        for (auto& [name, vp] : raw) {
            RelState& r = *st->relations[name];
            if (batched && std::find_if(batch.begin(), batch.end(), [&](const auto& b) { return b.first == &r; }) !=
                               batch.end())
                continue;
            if (eng.partitioned(r)) {
                for (u32 kc : r.keyset) eng.seed_copy(r, *vp, kc, pend);
            } else {
                eng.seed_copy(r, *vp, 0, pend);  // FULL empty: C = D = distinct rows
            }
        }
        eng.merge_complete_all(pend);
    }
    raw.clear();
    concat.clear();
    tr("seed", ts, 0);

    // ---- fixpoint (engine.cpp:163-239) ---------------------------------------
    u64 iteration = 0;
    for (;;) {
        const auto ti = Clock::now();
        std::map<std::string, CandPool> pooled;
        std::map<std::string, HeadSink> sinks;
        for (auto& v : variants) pooled[v.plan->head].arity = v.plan->head_arity;
        {
            std::vector<std::pair<const Plan*, long>> active;
            for (auto& v : variants)
                if (v.delta_source >= 0 || iteration == 0) active.emplace_back(v.plan, v.delta_source);
            eng.prepare_full_words(active);
        }
        {
            // Every variant is prepared first so that their step-0 output
            // sizes come back in one host round trip (precount_variants).
            std::vector<std::unique_ptr<Engine::VarRun>> runs;
            for (auto& v : variants) {
                if (v.delta_source < 0 && iteration != 0) continue;
                RelState& hr = *st->relations.at(v.plan->head);
                HeadSink* sink = hr.hash_mode ? &sinks[v.plan->head] : nullptr;
                if (v.alt && hr.word_sink && reverse_env) {
                    // DELTA's rows (words when it is word form) against the other
                    // atom's rows: probe the smaller side.
                    const RelState& dr = *st->relations.at(v.plan->sources[1].relation);
                    const RelState& pr = *st->relations.at(v.plan->sources[0].relation);
                    const u64 other = v.old_src.empty() || !v.old_src[0] || pr.old_is_full ? pr.rows() : pr.full_old.n;
                    if (reverse_always || (eng.dist() && dr.word_mode) || (!eng.dist() && reverse_ratio * double(dr.delta.n) < double(other))) {
                        runs.push_back(
                            eng.prepare_variant(*v.alt, dplans[v.alt_index], 0, v.alt_old, pooled[v.plan->head], sink));
                        continue;
                    }
                }
                runs.push_back(eng.prepare_variant(*v.plan, dplans[v.plan_index], v.delta_source, v.old_src,
                                                   pooled[v.plan->head], sink));
            }
            if (precount_env) eng.precount_variants(runs);
            for (auto& r : runs)
                if (r) eng.run_variant(*r);
        }
        tr("variants", ti, iteration);
        const auto tf = Clock::now();
        std::vector<u64> counts;  // per head: |Δ|, |FULL| (local, then global)
        // Set heads: pooled candidates inserted first, all heads' counters
        // then read in one round trip (not one per head).
        std::vector<std::pair<RelState*, HeadSink*>> set_heads;
        for (auto& [name, pool] : pooled) {
            RelState& r = *st->relations.at(name);
            if (eng.dist()) eng.route_pool(pool, r.home, r.owner_shift);
            if (r.hash_mode) set_heads.emplace_back(&r, &sinks[name]);
        }
        bool any_pool = false;
        for (auto& [r, s] : set_heads) any_pool = any_pool || pooled.at(r->name).n > 0;
        if (any_pool) {
            eng.estimate_blocks_all(set_heads, pooled);
            eng.prefetch_counters(set_heads);
            for (auto& [r, s] : set_heads) eng.insert_pool(*r, *s, pooled.at(r->name));
        }
        eng.prefetch_counters(set_heads);
        {
            // Sort-merged heads (single GPU) complete together: one read of
            // their new-row counts.
            std::vector<Engine::PendingMerge> pend;
            std::vector<std::pair<size_t, RelState*>> pend_at;
            for (auto& [name, pool] : pooled) {
                RelState& r = *st->relations.at(name);
                if (!r.hash_mode && !eng.dist()) {
                    pend_at.emplace_back(counts.size(), &r);
                    pend.push_back(eng.merge_launch_home(r, pool));
                    counts.push_back(0);
                    counts.push_back(0);
                    continue;
                }
                const u64 nd = r.hash_mode ? eng.hash_finalize(r, sinks[name], pool) : eng.dedup_merge_home(r, pool);
                if (eng.dist()) eng.forward_delta(r);
                counts.push_back(nd);
                counts.push_back(r.rows());
            }
            const std::vector<u64> nds = eng.merge_complete_all(pend);
            for (size_t i = 0; i < pend.size(); ++i) {
                counts[pend_at[i].first] = nds[i];
                counts[pend_at[i].first + 1] = pend_at[i].second->rows();
            }
        }
        eng.allreduce(counts);
        tr("finalize", tf, iteration);
        bool any_delta = false;
        std::vector<IterStat> its;
        size_t k = 0;
        for (auto& [name, pool] : pooled) {
            const u64 nd = counts[2 * k], nf = counts[2 * k + 1];
            ++k;
            if (nd) any_delta = true;
            its.push_back({iteration, name, nd, nf, 1, 0.0});
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
    if (trace) {
        u64 reserved = 0, used = 0;
        cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrUsedMemCurrent, &used);
        std::fprintf(stderr, "[fvlog] pool reserved %.2f GB used %.2f GB trims %llu\n", reserved / 1e9, used / 1e9,
                     static_cast<unsigned long long>(c->pool_trims));
    }
    return st;
}

std::vector<std::unique_ptr<EvalState>> evaluate_sharded(Ctx* base, u32 world, const std::vector<RelationDecl>& decls,
                                                         const std::vector<Plan>& plans,
                                                         const std::vector<FactsBlock>& facts) {
    if (world == 0 || world > 64) fail(FV_ERR_INVALID, "evaluate_sharded: world must be in [1, 64]");
    check_plans(decls, plans);
    auto group = make_local_group(static_cast<int>(world));
    std::vector<Ctx*> ctxs(world, nullptr);
    std::vector<std::unique_ptr<EvalState>> out(world);
    std::vector<std::exception_ptr> errs(world);
    try {
        for (u32 r = 0; r < world; ++r) {
            ctxs[r] = ctx_new(base->device);
            ctxs[r]->tx = group[r].get();
        }
        std::vector<std::thread> threads;
        for (u32 r = 0; r < world; ++r)
            threads.emplace_back([&, r] {
                try {
                    ctxs[r]->activate();
                    out[r] = evaluate(ctxs[r], decls, plans, facts);
                } catch (...) {
                    errs[r] = std::current_exception();
                    // Peers blocked in a collective would otherwise wait forever.
                    group[r]->abort();
                }
            });
        for (auto& t : threads) t.join();
    } catch (...) {
        for (auto* c : ctxs)
            if (c) ctx_delete(c);
        throw;
    }
    for (u32 r = 0; r < world; ++r) {
        ctxs[r]->tx = nullptr;
        if (out[r]) {
            out[r]->owned_ctx = ctxs[r];
        } else {
            ctx_delete(ctxs[r]);
        }
    }
    // The first failure is the cause; the others are the aborts it triggered.
    const int first = group[0]->first_failed();
    if (first >= 0 && errs[first]) std::rethrow_exception(errs[first]);
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    return out;
}

namespace {

// Levels-mode FULL: the past DELTAs plus the current one.
std::vector<const DevVersion*> levels_of(const RelState& r) {
    std::vector<const DevVersion*> out;
    for (auto& lv : r.levels) out.push_back(&lv);
    if (r.delta.n) out.push_back(&r.delta);
    return out;
}

// The relation's rows as lexicographically sorted device columns: FULL
// itself, or (levels mode) one sort of the concatenated levels into `tmp`.
const DevVersion& sorted_rows(const EvalState& s, const RelState& r, DevVersion& tmp) {
    if (!r.levels_mode) return r.full;
    Ctx* c = s.ctx;
    const u64 n = r.rows();
    if (r.block_mode && r.blocks.capacity() && !std::getenv("FVLOG_DUMP_SORT")) {
        // The block set holds FULL exactly: decode its bitmaps in row order
        // (FVLOG_DUMP_SORT=1: concatenate the levels and radix-sort instead).
        tmp.n = n;
        tmp.cols.clear();
        for (u32 j = 0; j < r.arity; ++j) tmp.cols.emplace_back(c, n);
        const u64 got = engine_blockset_dump(c, r.blocks, r.arity, n ? tmp.cols[0].get() : nullptr,
                                             r.arity == 2 && n ? tmp.cols[1].get() : nullptr);
        if (got != n) fail(FV_ERR_INVALID, "block set holds " + std::to_string(got) + " rows, expected " +
                                               std::to_string(n));
        return tmp;
    }
    // Levels are grouped by column 0 per iteration; one sort of their
    // concatenation gives the lexicographic dump (like dump_relation's std::sort).
    tmp.n = n;
    tmp.cols.clear();
    for (u32 j = 0; j < r.arity; ++j) tmp.cols.emplace_back(c, n);
    u64 off = 0;
    for (const DevVersion* lv : levels_of(r)) {
        if (!lv->n) continue;
        if (lv->cols.size() == r.arity + 1) {  // word form: expanded in place
            off += engine_expand_words(c, lv->cols[0].get(), lv->cols[1].get(), lv->cols[2].get(), lv->n,
                                       tmp.cols[0].get() + off, tmp.cols[1].get() + off);
            continue;
        }
        for (u32 j = 0; j < r.arity; ++j)
            FV_CUDA(cudaMemcpyAsync(tmp.cols[j].get() + off, lv->cols[j].get(), 4 * lv->n, cudaMemcpyDeviceToDevice,
                                    c->stream));
        off += lv->n;
    }
    if (off != n) fail(FV_ERR_INVALID, "levels hold " + std::to_string(off) + " rows, expected " + std::to_string(n));
    if (n) {
        std::vector<DBuf<u64>> words;
        words.emplace_back(c, n);
        u64* wp = words[0].get();
        engine_pack_keys(c, tmp.ptrs(), n, s.key_shift, &wp);
        engine_sort_keys(c, words, n, r.arity, s.key_shift);
        std::vector<u32*> cols;
        for (auto& col : tmp.cols) cols.push_back(col.get());
        engine_unpack_keys(c, words[0].get(), n, r.arity, s.key_shift, cols);
    }
    return tmp;
}

const RelState& find_rel(const EvalState& s, const std::string& rel) {
    auto it = s.relations.find(rel);
    if (it == s.relations.end()) fail(FV_ERR_RANGE, "unknown relation '" + rel + "'");
    return *it->second;
}

}  // namespace

void dump_sorted_into(const EvalState& s, const std::string& rel, u32* rows_out) {
    const RelState& r = find_rel(s, rel);
    Ctx* c = s.ctx;
    DevVersion tmp;
    const DevVersion& src = sorted_rows(s, r, tmp);
    const u64 n = r.rows();
    if (!n) return;
    // Bounded staging: rows are interleaved and copied out in 2^26-row chunks.
    const u64 chunk = std::min<u64>(n, u64(1) << 26);
    DBuf<u32> buf(c, chunk * r.arity);
    for (u64 off = 0; off < n; off += chunk) {
        const u64 m = std::min(chunk, n - off);
        std::vector<const u32*> cols;
        for (u32 j = 0; j < r.arity; ++j) cols.push_back(src.cols[j].get() + off);
        engine_interleave(c, cols, m, buf.get());
        FV_CUDA(cudaMemcpyAsync(rows_out + off * r.arity, buf.get(), 4 * m * r.arity, cudaMemcpyDeviceToHost,
                                c->stream));
    }
    c->sync();
}

std::vector<u32> dump_sorted(const EvalState& s, const std::string& rel) {
    const RelState& r = find_rel(s, rel);
    std::vector<u32> rows(r.rows() * r.arity);
    dump_sorted_into(s, rel, rows.data());
    return rows;
}

std::string dump_sorted_text(const EvalState& s, const std::string& rel) {
    const RelState& r = find_rel(s, rel);
    DevVersion tmp;
    const DevVersion& src = sorted_rows(s, r, tmp);
    return tsv_format_u32(s.ctx, src.ptrs(), r.rows(), r.arity);
}

u64 fingerprint(const EvalState& s, const std::string& rel) {
    auto it = s.relations.find(rel);
    if (it == s.relations.end()) fail(FV_ERR_RANGE, "unknown relation '" + rel + "'");
    const RelState& r = *it->second;
    if (!r.levels_mode) return engine_fingerprint(s.ctx, r.full.ptrs(), r.full.n, r.arity);
    if (r.block_mode && r.blocks.capacity() && !std::getenv("FVLOG_DUMP_SORT"))
        return engine_blockset_fingerprint(s.ctx, r.blocks, r.arity);  // the bitmaps hold FULL exactly
    u64 h = 0;  // the fingerprint is a sum over rows: additive over levels
    for (const DevVersion* lv : levels_of(r)) {
        if (lv->cols.size() == r.arity + 1 && lv->n) {  // word form: fingerprint of its tuples
            const u64 t = engine_expand_words(s.ctx, lv->cols[0].get(), lv->cols[1].get(), lv->cols[2].get(), lv->n,
                                              nullptr, nullptr);
            DBuf<u32> x(s.ctx, t), z(s.ctx, t);
            engine_expand_words(s.ctx, lv->cols[0].get(), lv->cols[1].get(), lv->cols[2].get(), lv->n, x.get(),
                                z.get());
            h += engine_fingerprint(s.ctx, std::vector<const u32*>{x.get(), z.get()}, t, r.arity);
            continue;
        }
        h += engine_fingerprint(s.ctx, lv->ptrs(), lv->n, r.arity);
    }
    return h;
}

}  // namespace fv

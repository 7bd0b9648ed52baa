/*
 * TEST INFRASTRUCTURE — ORACLE, NOT PRODUCT. See colog_oracle.h.
 *
 * Plain-C restatement of the reference's column-store algorithms and of its
 * Jacobi semi-naive driver. Each function cites the reference lines it
 * follows (P = /root/reference/proj). Single-threaded, O(n log n) sorts via
 * qsort; meant for inputs that finish in seconds.
 */
#include "colog_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---- helpers ------------------------------------------------------------ */

static const uint32_t* g_raw; /* qsort context (single-threaded oracle) */
static uint32_t g_arity;
static const uint32_t* g_rows; /* row-major rows for row comparisons */

static int cmp_value_id(const void* pa, const void* pb) {
    uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    if (g_raw[a] != g_raw[b]) return g_raw[a] < g_raw[b] ? -1 : 1;
    return a < b ? -1 : (a > b);
}

static int cmp_u32(const void* pa, const void* pb) {
    uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    return a < b ? -1 : (a > b);
}

/* Row comparison on row-major rows (lexicographic), ties by index. */
static int cmp_row_idx(const void* pa, const void* pb) {
    uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    for (uint32_t j = 0; j < g_arity; ++j) {
        uint32_t x = g_rows[(uint64_t)a * g_arity + j], y = g_rows[(uint64_t)b * g_arity + j];
        if (x != y) return x < y ? -1 : 1;
    }
    return a < b ? -1 : (a > b);
}

static int row_cmp(const uint32_t* x, const uint32_t* y, uint32_t arity) {
    for (uint32_t j = 0; j < arity; ++j)
        if (x[j] != y[j]) return x[j] < y[j] ? -1 : 1;
    return 0;
}

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) abort();
    return p;
}

/* ---- build_index (P/src/column.cpp:17-43) ------------------------------ */

uint64_t or_build_index(const uint32_t* raw, uint64_t n, uint32_t* sorted_idx, uint32_t* keys,
                        uint32_t* starts, uint32_t* counts) {
    for (uint64_t i = 0; i < n; ++i) sorted_idx[i] = (uint32_t)i; /* iota */
    g_raw = raw;
    qsort(sorted_idx, n, sizeof(uint32_t), cmp_value_id); /* strict (value, id) order */
    uint64_t u = 0, i = 0;
    while (i < n) { /* run-length encode into the unique map */
        uint32_t v = raw[sorted_idx[i]];
        uint64_t j = i + 1;
        while (j < n && raw[sorted_idx[j]] == v) ++j;
        keys[u] = v;
        starts[u] = (uint32_t)i;
        counts[u] = (uint32_t)(j - i);
        ++u;
        i = j;
    }
    return u;
}

/* Binary search of a value in the unique keys: Column::probe
 * (P/include/colog/column.hpp:46-50). Returns 1 and the run on hit. */
static int probe(const uint32_t* keys, const uint32_t* starts, const uint32_t* counts, uint64_t u,
                 uint32_t v, uint32_t* s, uint32_t* c) {
    uint64_t lo = 0, hi = u;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (keys[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    if (lo < u && keys[lo] == v) {
        *s = starts[lo];
        *c = counts[lo];
        return 1;
    }
    return 0;
}

typedef struct {
    uint64_t n, u;
    uint32_t *sorted, *keys, *starts, *counts;
} index_t;

static void index_build(index_t* ix, const uint32_t* raw, uint64_t n) {
    ix->n = n;
    ix->sorted = xmalloc(sizeof(uint32_t) * n);
    ix->keys = xmalloc(sizeof(uint32_t) * n);
    ix->starts = xmalloc(sizeof(uint32_t) * n);
    ix->counts = xmalloc(sizeof(uint32_t) * n);
    ix->u = or_build_index(raw, n, ix->sorted, ix->keys, ix->starts, ix->counts);
}

static void index_free(index_t* ix) {
    free(ix->sorted);
    free(ix->keys);
    free(ix->starts);
    free(ix->counts);
}

/* ---- join (P/src/kernels.cpp:59-135, Algorithm 1) ----------------------- */

uint64_t or_join_probe(const uint32_t* probe_v, uint64_t np, const uint32_t* build, uint64_t nb,
                       uint32_t* m_starts, uint32_t* m_counts, uint32_t* matched, uint64_t* total) {
    index_t ix;
    index_build(&ix, build, nb);
    uint64_t m = 0, t = 0;
    for (uint64_t i = 0; i < np; ++i) {
        uint32_t s, c;
        if (probe(ix.keys, ix.starts, ix.counts, ix.u, probe_v[i], &s, &c)) {
            if (m_starts) m_starts[m] = s;
            if (m_counts) m_counts[m] = c;
            if (matched) matched[m] = (uint32_t)i;
            ++m;
            t += c;
        }
    }
    *total = t;
    index_free(&ix);
    return m;
}

void or_column_join(const uint32_t* probe_v, uint64_t np, const uint32_t* build, uint64_t nb,
                    uint32_t* a_ids, uint32_t* b_ids) {
    index_t ix;
    index_build(&ix, build, nb);
    uint64_t o = 0;
    /* Output position n belongs to the run j with offsets[j] <= n <
     * offsets[j+1]; walking the runs in order writes the same sequence. */
    for (uint64_t i = 0; i < np; ++i) {
        uint32_t s, c;
        if (!probe(ix.keys, ix.starts, ix.counts, ix.u, probe_v[i], &s, &c)) continue;
        for (uint32_t r = 0; r < c; ++r) {
            a_ids[o] = (uint32_t)i;
            b_ids[o] = ix.sorted[s + r];
            ++o;
        }
    }
    index_free(&ix);
}

/* ---- dedup_rows (P/src/relation.cpp:71-89) ------------------------------ */

uint64_t or_dedup_rows(const uint32_t* cols, uint64_t n, uint32_t arity, uint32_t* out) {
    uint32_t* rows = xmalloc(sizeof(uint32_t) * n * arity);
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < arity; ++j) rows[i * arity + j] = cols[(uint64_t)j * n + i];
    uint32_t* order = xmalloc(sizeof(uint32_t) * n);
    for (uint64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
    g_rows = rows;
    g_arity = arity;
    qsort(order, n, sizeof(uint32_t), cmp_row_idx);
    uint32_t* keep = xmalloc(sizeof(uint32_t) * n);
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (i == 0 || row_cmp(rows + (uint64_t)order[i - 1] * arity, rows + (uint64_t)order[i] * arity,
                              arity) != 0)
            keep[k++] = order[i]; /* group head = smallest id of the row */
    qsort(keep, k, sizeof(uint32_t), cmp_u32); /* first-occurrence order */
    for (uint64_t i = 0; i < k; ++i)
        for (uint32_t j = 0; j < arity; ++j) out[(uint64_t)j * n + i] = rows[(uint64_t)keep[i] * arity + j];
    free(rows);
    free(order);
    free(keep);
    return k;
}

/* ---- deduplicate (P/src/kernels.cpp:185-255, Algorithm 2) -------------- */

void or_deduplicate(const uint32_t* new_cols, uint64_t n_new, const uint32_t* full_cols,
                    uint64_t n_full, uint32_t arity, uint8_t* flags) {
    memset(flags, 0, n_new);
    if (n_new == 0 || n_full == 0) return;
    index_t* ix = xmalloc(sizeof(index_t) * arity);
    for (uint32_t j = 0; j < arity; ++j) index_build(&ix[j], full_cols + (uint64_t)j * n_full, n_full);
    uint32_t* pos = xmalloc(sizeof(uint32_t) * arity);
    uint32_t* s = xmalloc(sizeof(uint32_t) * arity);
    uint32_t* c = xmalloc(sizeof(uint32_t) * arity);
    for (uint64_t i = 0; i < n_new; ++i) {
        int hit = 1;
        for (uint32_t j = 0; j < arity && hit; ++j)
            hit = probe(ix[j].keys, ix[j].starts, ix[j].counts, ix[j].u, new_cols[(uint64_t)j * n_new + i],
                        &s[j], &c[j]);
        if (!hit) continue; /* early drop */
        if (arity == 1) {
            flags[i] = 1;
            continue;
        }
        for (uint32_t j = 0; j < arity; ++j) pos[j] = 0;
        for (;;) { /* runs_intersect: ascending id runs share an element? */
            uint32_t mx = ix[0].sorted[s[0] + pos[0]];
            int all_eq = 1, done = 0;
            for (uint32_t j = 1; j < arity; ++j) {
                uint32_t v = ix[j].sorted[s[j] + pos[j]];
                if (v != mx) {
                    all_eq = 0;
                    if (v > mx) mx = v;
                }
            }
            if (all_eq) {
                flags[i] = 1;
                break;
            }
            for (uint32_t j = 0; j < arity && !done; ++j) {
                while (pos[j] < c[j] && ix[j].sorted[s[j] + pos[j]] < mx) ++pos[j];
                if (pos[j] >= c[j]) done = 1;
            }
            if (done) break;
        }
    }
    for (uint32_t j = 0; j < arity; ++j) index_free(&ix[j]);
    free(ix);
    free(pos);
    free(s);
    free(c);
}

uint64_t or_filter_neq(const uint32_t* cols, uint64_t n, uint32_t ci, uint32_t cj, uint32_t* ids) {
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (cols[(uint64_t)ci * n + i] != cols[(uint64_t)cj * n + i]) ids[k++] = (uint32_t)i;
    return k;
}

uint64_t or_select_eq(const uint32_t* raw, uint64_t n, uint32_t v, uint32_t* ids) {
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (raw[i] == v) ids[k++] = (uint32_t)i;
    return k;
}

/* ---- semi-naive engine (P/src/engine.cpp) --------------------------------
 *
 * PLAN ENCODING (uint32 words):
 *   n_plans, then per plan:
 *     head_rel, head_arity, n_sources,
 *       per source: rel, arity, n_const, (col, val) x n_const, n_self, (a, b) x n_self
 *     n_joins,
 *       per join: right_source, left_source, left_col, right_col, n_res,
 *                 (left_source, left_col, right_col) x n_res
 *     n_out, (source, col) x n_out,
 *     n_guards, (slot_a, slot_b) x n_guards
 */

typedef struct {
    uint32_t* rows; /* row-major, sorted lexicographically, distinct */
    uint64_t n, cap;
} rowset_t;

typedef struct {
    uint32_t rel, arity, n_const, n_self;
    const uint32_t* consts;
    const uint32_t* selfs;
} src_t;

typedef struct {
    uint32_t right, lsrc, lcol, rcol, n_res;
    const uint32_t* res;
} join_t;

typedef struct {
    uint32_t head, head_arity, n_src, n_join, n_out, n_guard;
    src_t* src;
    join_t* join;
    const uint32_t* out;
    const uint32_t* guard;
} plan_t;

struct or_state {
    uint32_t n_rel;
    uint32_t* arity;
    rowset_t* full;
    uint64_t iterations;
    uint64_t* deltas; /* [iterations][n_rel] */
};

typedef struct {
    uint32_t* v;
    uint64_t n, cap;
} vec_t;

static void vec_push(vec_t* v, uint32_t x) {
    if (v->n == v->cap) {
        v->cap = v->cap ? v->cap * 2 : 64;
        v->v = realloc(v->v, sizeof(uint32_t) * v->cap);
        if (!v->v) abort();
    }
    v->v[v->n++] = x;
}

static void rows_sort_unique(uint32_t* rows, uint64_t* n, uint32_t arity) {
    if (*n == 0) return;
    uint32_t* idx = xmalloc(sizeof(uint32_t) * *n);
    for (uint64_t i = 0; i < *n; ++i) idx[i] = (uint32_t)i;
    g_rows = rows;
    g_arity = arity;
    qsort(idx, *n, sizeof(uint32_t), cmp_row_idx);
    uint32_t* out = xmalloc(sizeof(uint32_t) * *n * arity);
    uint64_t k = 0;
    for (uint64_t i = 0; i < *n; ++i) {
        const uint32_t* r = rows + (uint64_t)idx[i] * arity;
        if (k == 0 || row_cmp(out + (k - 1) * arity, r, arity) != 0) {
            memcpy(out + k * arity, r, sizeof(uint32_t) * arity);
            ++k;
        }
    }
    memcpy(rows, out, sizeof(uint32_t) * k * arity);
    *n = k;
    free(idx);
    free(out);
}

static int rowset_contains(const rowset_t* s, const uint32_t* r, uint32_t arity) {
    uint64_t lo = 0, hi = s->n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        int c = row_cmp(s->rows + mid * arity, r, arity);
        if (c == 0) return 1;
        if (c < 0) lo = mid + 1;
        else hi = mid;
    }
    return 0;
}

/* selected_ids (P/src/engine.cpp:17-39): rows passing constants / self-eqs. */
static int row_selected(const uint32_t* r, const src_t* s) {
    for (uint32_t k = 0; k < s->n_const; ++k)
        if (r[s->consts[2 * k]] != s->consts[2 * k + 1]) return 0;
    for (uint32_t k = 0; k < s->n_self; ++k)
        if (r[s->selfs[2 * k]] != r[s->selfs[2 * k + 1]]) return 0;
    return 1;
}

/* execute_plan (P/src/engine.cpp:72-146) with the intended residual-eq
 * semantics (left value read at the intermediate row's id; the reference's
 * filter_pairs_eq at P/src/kernels.cpp:155 indexes by pair position). */
static void execute_plan(const plan_t* p, const rowset_t* const* ver, vec_t* out) {
    uint32_t ns = p->n_src;
    for (uint32_t s = 0; s < ns; ++s)
        if (ver[s]->n == 0) return;
    /* intermediate: tuples of per-source row ids, width grows by one per join */
    vec_t cur = {0}, next = {0};
    const src_t* s0 = &p->src[0];
    for (uint64_t i = 0; i < ver[0]->n; ++i)
        if (row_selected(ver[0]->rows + i * s0->arity, s0)) vec_push(&cur, (uint32_t)i);
    uint32_t width = 1;
    for (uint32_t k = 0; k < p->n_join && cur.n; ++k) {
        const join_t* jn = &p->join[k];
        const src_t* rs = &p->src[jn->right];
        const rowset_t* rv = ver[jn->right];
        /* index the (selected) right rows on the hash column */
        uint32_t* rcol = xmalloc(sizeof(uint32_t) * (rv->n ? rv->n : 1));
        uint32_t* sel = xmalloc(sizeof(uint32_t) * (rv->n ? rv->n : 1));
        uint64_t nsel = 0;
        for (uint64_t i = 0; i < rv->n; ++i)
            if (row_selected(rv->rows + i * rs->arity, rs)) {
                rcol[nsel] = rv->rows[i * rs->arity + jn->rcol];
                sel[nsel] = (uint32_t)i;
                ++nsel;
            }
        index_t ix;
        index_build(&ix, rcol, nsel);
        next.n = 0;
        uint64_t tuples = cur.n / width;
        for (uint64_t t = 0; t < tuples; ++t) {
            const uint32_t* tup = cur.v + t * width;
            uint32_t lv = ver[jn->lsrc]->rows[(uint64_t)tup[jn->lsrc] * p->src[jn->lsrc].arity + jn->lcol];
            uint32_t st, cn;
            if (!probe(ix.keys, ix.starts, ix.counts, ix.u, lv, &st, &cn)) continue;
            for (uint32_t r = 0; r < cn; ++r) {
                uint32_t rid = sel[ix.sorted[st + r]];
                int ok = 1;
                for (uint32_t q = 0; q < jn->n_res && ok; ++q) {
                    uint32_t ls = jn->res[3 * q], lc = jn->res[3 * q + 1], rc = jn->res[3 * q + 2];
                    uint32_t a = ver[ls]->rows[(uint64_t)tup[ls] * p->src[ls].arity + lc];
                    uint32_t b = rv->rows[(uint64_t)rid * rs->arity + rc];
                    ok = a == b;
                }
                if (!ok) continue;
                for (uint32_t w = 0; w < width; ++w) vec_push(&next, tup[w]);
                vec_push(&next, rid);
            }
        }
        index_free(&ix);
        free(rcol);
        free(sel);
        vec_t tmp = cur;
        cur = next;
        next = tmp;
        ++width;
    }
    uint64_t tuples = cur.n / width;
    for (uint64_t t = 0; t < tuples && width == ns; ++t) {
        const uint32_t* tup = cur.v + t * width;
        int ok = 1;
        for (uint32_t g = 0; g < p->n_guard && ok; ++g) {
            uint32_t sa = p->guard[2 * g], sb = p->guard[2 * g + 1];
            uint32_t as = p->out[2 * sa], ac = p->out[2 * sa + 1];
            uint32_t bs = p->out[2 * sb], bc = p->out[2 * sb + 1];
            uint32_t va = ver[as]->rows[(uint64_t)tup[as] * p->src[as].arity + ac];
            uint32_t vb = ver[bs]->rows[(uint64_t)tup[bs] * p->src[bs].arity + bc];
            ok = va != vb;
        }
        if (!ok) continue;
        for (uint32_t h = 0; h < p->head_arity; ++h) {
            uint32_t sx = p->out[2 * h], cx = p->out[2 * h + 1];
            vec_push(out, ver[sx]->rows[(uint64_t)tup[sx] * p->src[sx].arity + cx]);
        }
    }
    free(cur.v);
    free(next.v);
}

static const uint32_t* parse_plan(const uint32_t* w, plan_t* p) {
    p->head = *w++;
    p->head_arity = *w++;
    p->n_src = *w++;
    p->src = xmalloc(sizeof(src_t) * p->n_src);
    for (uint32_t s = 0; s < p->n_src; ++s) {
        src_t* x = &p->src[s];
        x->rel = *w++;
        x->arity = *w++;
        x->n_const = *w++;
        x->consts = w;
        w += 2 * x->n_const;
        x->n_self = *w++;
        x->selfs = w;
        w += 2 * x->n_self;
    }
    p->n_join = *w++;
    p->join = xmalloc(sizeof(join_t) * (p->n_join ? p->n_join : 1));
    for (uint32_t k = 0; k < p->n_join; ++k) {
        join_t* j = &p->join[k];
        j->right = *w++;
        j->lsrc = *w++;
        j->lcol = *w++;
        j->rcol = *w++;
        j->n_res = *w++;
        j->res = w;
        w += 3 * j->n_res;
    }
    p->n_out = *w++;
    p->out = w;
    w += 2 * p->n_out;
    p->n_guard = *w++;
    p->guard = w;
    w += 2 * p->n_guard;
    return w;
}

or_state* or_evaluate(uint32_t n_rel, const uint32_t* arities, const uint32_t* plan_words,
                      uint64_t n_plan_words, const uint32_t* const* facts, const uint64_t* n_facts) {
    (void)n_plan_words;
    const uint32_t* w = plan_words;
    uint32_t n_plans = *w++;
    plan_t* plans = xmalloc(sizeof(plan_t) * (n_plans ? n_plans : 1));
    for (uint32_t i = 0; i < n_plans; ++i) w = parse_plan(w, &plans[i]);

    or_state* st = calloc(1, sizeof(or_state));
    st->n_rel = n_rel;
    st->arity = xmalloc(sizeof(uint32_t) * n_rel);
    memcpy(st->arity, arities, sizeof(uint32_t) * n_rel);
    st->full = calloc(n_rel, sizeof(rowset_t));
    rowset_t* delta = calloc(n_rel, sizeof(rowset_t));
    uint8_t* is_idb = calloc(n_rel, 1);
    for (uint32_t i = 0; i < n_plans; ++i) is_idb[plans[i].head] = 1;

    /* seed (P/src/engine.cpp:148-161): FULL = DELTA = dedup(EDB) */
    for (uint32_t r = 0; r < n_rel; ++r) {
        uint32_t a = arities[r];
        uint64_t n = n_facts ? n_facts[r] : 0;
        rowset_t* f = &st->full[r];
        f->rows = xmalloc(sizeof(uint32_t) * (n * a + 1));
        for (uint64_t i = 0; i < n; ++i)
            for (uint32_t j = 0; j < a; ++j) f->rows[i * a + j] = facts[r][(uint64_t)j * n + i];
        f->n = n;
        rows_sort_unique(f->rows, &f->n, a);
        delta[r].rows = xmalloc(sizeof(uint32_t) * (f->n * a + 1));
        memcpy(delta[r].rows, f->rows, sizeof(uint32_t) * f->n * a);
        delta[r].n = f->n;
    }

    /* delta_rewrite (P/src/engine.cpp:57-64) */
    uint32_t n_var = 0;
    uint32_t* var_plan = xmalloc(sizeof(uint32_t) * 64 * (n_plans + 1));
    int64_t* var_delta = xmalloc(sizeof(int64_t) * 64 * (n_plans + 1));
    for (uint32_t i = 0; i < n_plans; ++i) {
        uint32_t before = n_var;
        for (uint32_t s = 0; s < plans[i].n_src; ++s)
            if (is_idb[plans[i].src[s].rel]) {
                var_plan[n_var] = i;
                var_delta[n_var++] = s;
            }
        if (n_var == before) {
            var_plan[n_var] = i;
            var_delta[n_var++] = -1;
        }
    }

    uint64_t cap_it = 16;
    st->deltas = calloc(cap_it * n_rel, sizeof(uint64_t));
    vec_t* pooled = calloc(n_rel, sizeof(vec_t));
    const rowset_t** ver = xmalloc(sizeof(rowset_t*) * 64);
    uint64_t it = 0;
    for (;;) {
        for (uint32_t r = 0; r < n_rel; ++r) pooled[r].n = 0;
        for (uint32_t v = 0; v < n_var; ++v) { /* run_iteration (engine.cpp:163-220) */
            const plan_t* p = &plans[var_plan[v]];
            if (var_delta[v] < 0 && it != 0) continue; /* EDB-only: iteration 0 only */
            for (uint32_t s = 0; s < p->n_src; ++s)
                ver[s] = ((int64_t)s == var_delta[v]) ? &delta[p->src[s].rel] : &st->full[p->src[s].rel];
            execute_plan(p, ver, &pooled[p->head]);
        }
        if (it == cap_it) {
            st->deltas = realloc(st->deltas, sizeof(uint64_t) * cap_it * 2 * n_rel);
            memset(st->deltas + cap_it * n_rel, 0, sizeof(uint64_t) * cap_it * n_rel);
            cap_it *= 2;
        }
        int any = 0;
        for (uint32_t r = 0; r < n_rel; ++r) {
            if (!is_idb[r]) continue;
            uint32_t a = arities[r];
            uint64_t n = a ? pooled[r].n / a : 0;
            rows_sort_unique(pooled[r].v, &n, a); /* dedup NEW */
            /* difference against FULL, then merge (kernels.cpp:210-268) */
            uint32_t* d = xmalloc(sizeof(uint32_t) * (n * a + 1));
            uint64_t nd = 0;
            for (uint64_t i = 0; i < n; ++i)
                if (!rowset_contains(&st->full[r], pooled[r].v + i * a, a)) {
                    memcpy(d + nd * a, pooled[r].v + i * a, sizeof(uint32_t) * a);
                    ++nd;
                }
            rowset_t* f = &st->full[r];
            uint32_t* merged = xmalloc(sizeof(uint32_t) * ((f->n + nd) * a + 1));
            uint64_t x = 0, y = 0, z = 0;
            while (x < f->n || y < nd) {
                if (y == nd || (x < f->n && row_cmp(f->rows + x * a, d + y * a, a) < 0)) {
                    memcpy(merged + z * a, f->rows + x * a, sizeof(uint32_t) * a);
                    ++x;
                } else {
                    memcpy(merged + z * a, d + y * a, sizeof(uint32_t) * a);
                    ++y;
                }
                ++z;
            }
            free(f->rows);
            f->rows = merged;
            f->n = z;
            free(delta[r].rows);
            delta[r].rows = d;
            delta[r].n = nd;
            st->deltas[it * n_rel + r] = nd;
            if (nd) any = 1;
        }
        ++it;
        if (!any) break;
    }
    st->iterations = it; /* includes the final empty iteration */

    for (uint32_t r = 0; r < n_rel; ++r) {
        free(delta[r].rows);
        free(pooled[r].v);
    }
    for (uint32_t i = 0; i < n_plans; ++i) {
        free(plans[i].src);
        free(plans[i].join);
    }
    free(plans);
    free(delta);
    free(pooled);
    free(is_idb);
    free(var_plan);
    free(var_delta);
    free(ver);
    return st;
}

uint64_t or_state_iterations(const or_state* s) { return s->iterations; }
uint64_t or_state_rows(const or_state* s, uint32_t rel) { return s->full[rel].n; }
void or_state_dump(const or_state* s, uint32_t rel, uint32_t* out) {
    memcpy(out, s->full[rel].rows, sizeof(uint32_t) * s->full[rel].n * s->arity[rel]);
}
uint64_t or_state_delta(const or_state* s, uint64_t it, uint32_t rel) {
    return it < s->iterations ? s->deltas[it * s->n_rel + rel] : 0;
}
void or_state_free(or_state* s) {
    if (!s) return;
    for (uint32_t r = 0; r < s->n_rel; ++r) free(s->full[r].rows);
    free(s->full);
    free(s->arity);
    free(s->deltas);
    free(s);
}

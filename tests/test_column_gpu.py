"""GPU parity: the column store and RA operator mirrors (through the C ABI)
against the reference's golden vectors and the oracle restatement.
Mirrors P/tests/column_test.cpp, relation_test.cpp and kernels_test.cpp."""
import numpy as np
import pytest

from conftest import load_golden, matches
from paper_2501_13051_b200 import workloads as W
from paper_2501_13051_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def C(ctx):
    from paper_2501_13051_b200 import colog
    return colog


# ---- column_test.cpp ---------------------------------------------------------------


def test_build_index_worked_example(C):
    col = C.Column.build([5, 3, 5, 1])
    assert col.sorted_idx().tolist() == [3, 1, 0, 2]
    u = col.unique_idx()
    assert len(u) == 3
    assert col.probe(1) == C.MatchRange(0, 1)
    assert col.probe(3) == C.MatchRange(1, 1)
    assert col.probe(5) == C.MatchRange(2, 2)
    assert col.probe(2) is None
    assert C.Column.build([1, 1, 1, 2, 3, 3, 3, 3, 4, 4, 4, 4]).probe(1) == C.MatchRange(0, 3)


def test_empty_column(C):
    col = C.Column.build([])
    assert col.sorted_idx().size == 0 and col.unique_idx() == {}
    assert col.probe(0) is None


def test_gather_and_bounds(C):
    col = C.Column.build([5, 3, 5, 1])
    assert col.gather([0, 3]).tolist() == [5, 1]
    assert col.gather([]).size == 0
    assert C.Column.build([7]).gather([0, 0, 0]).tolist() == [7, 7, 7]
    with pytest.raises(_lib.RangeError):
        C.Column.build([5, 3]).gather([0, 2])


def test_append_and_reindex(C):
    col = C.Column.build([5, 3])
    grown = col.append_and_reindex([5])
    assert grown.raw().tolist() == [5, 3, 5]
    assert grown.probe(3) == C.MatchRange(0, 1)
    assert grown.probe(5) == C.MatchRange(1, 2)
    a = W.random_values(404, 1500, 64)
    b = W.random_values(405, 700, 64)
    app = C.Column.build(a).append_and_reindex(b)
    reb = C.Column.build(np.concatenate([a, b]))
    assert np.array_equal(app.sorted_idx(), reb.sorted_idx())
    assert app.unique_idx() == reb.unique_idx()


def test_build_index_golden(C):
    for c in load_golden("column.json"):
        raw = np.asarray(c["raw"], np.uint32) if "raw" in c else W.random_values(*c["gen"][1:])
        s, k, st, cnt = C.build_index_arrays(raw)
        o = c["out"]
        assert matches(s, o["sorted_idx"]), c["name"]
        assert matches(k, o["keys"]) and matches(st, o["starts"]) and matches(cnt, o["counts"]), c["name"]


def test_build_index_large_skewed(C, oracle):
    # 10^7 skewed column vs the oracle, bit-exact.
    raw = W.random_values(77, 10_000_000, 1_000_000, True)
    s, k, st, cnt = C.build_index_arrays(raw)
    os_, ok, ost, ocnt = oracle.build_index(raw)
    assert np.array_equal(s, os_) and np.array_equal(k, ok)
    assert np.array_equal(st, ost) and np.array_equal(cnt, ocnt)


def test_build_index_1e8_properties(C):
    # 10^8 elements, full 32-bit domain: stable (value, id) order == numpy's
    # stable argsort (size-independent restatement of the reference order).
    raw = (W.splitmix64(91, 100_000_000) >> np.uint64(32)).astype(np.uint32)
    s, k, st, cnt = C.build_index_arrays(raw)
    assert np.array_equal(s, np.argsort(raw, kind="stable").astype(np.uint32))
    sv = raw[s]
    uk, us, uc = np.unique(sv, return_index=True, return_counts=True)
    assert np.array_equal(k, uk) and np.array_equal(st, us) and np.array_equal(cnt, uc)


# ---- kernels_test.cpp -----------------------------------------------------------------


def test_select_eq(C):
    col = C.Column.build([5, 3, 5, 1])
    assert C.select_eq(col, 5).tolist() == [0, 2]
    assert C.select_eq(col, 2).size == 0
    assert C.select_eq(C.Column.build([9]), 9).tolist() == [0]


def test_project(C):
    ver = C.Version.decompose([(1, 10), (2, 20), (3, 30)], 2)
    assert C.project(ver, [0, 1, 2], [0, 1]).reconstruct() == ver.reconstruct()
    assert C.project(ver, [], [0, 1]).rows() == 0
    assert C.project(ver, [2, 0], [1, 0, 1]).reconstruct() == [(30, 3, 30), (10, 1, 10)]
    with pytest.raises(_lib.RangeError):
        C.project(ver, [0], [2])


def test_join_worked_example(C):
    edge_y = C.Column.build([1, 1, 1, 2, 3, 3, 3, 3, 4, 4, 4, 4])
    mv = C.join_probe_phase([1, 2, 7, 3, 4], edge_y)
    assert mv.size() == 4
    assert mv.ranges[0].count == 3 and mv.ranges[1].count == 1
    assert mv.matched.tolist() == [0, 1, 3, 4]
    total = C.join_total_size(mv)
    assert total == 12
    off = C.join_offsets(mv)
    assert off.tolist()[:3] == [0, 3, 4]
    out = C.join_write_phase(mv, off, total, edge_y)
    assert out.size() == 12
    assert out.a_ids[2] == 0 and out.b_ids[2] == 2


def test_join_small_cases(C):
    assert C.column_join(C.Column.build([1, 2, 3]), C.Column.build([4, 5])).size() == 0
    assert C.column_join(C.Column.build([]), C.Column.build([4, 5])).size() == 0
    assert C.column_join(C.Column.build([1, 2, 3]), C.Column.build([])).size() == 0
    p = C.column_join(C.Column.build([1, 2, 2]), C.Column.build([2, 2, 3]))
    assert sorted(zip(p.a_ids.tolist(), p.b_ids.tolist())) == [(1, 0), (1, 1), (2, 0), (2, 1)]


def test_join_golden_exact_order(C):
    for c in load_golden("join.json"):
        if "gen" in c:
            p, b = W.random_values(*c["gen"][0]), W.random_values(*c["gen"][1])
        else:
            p, b = np.asarray(c["probe"], np.uint32), np.asarray(c["build"], np.uint32)
        out = C.column_join(p, C.Column.build(b))
        assert matches(out.a_ids, c["out"]["a_ids"]), c["name"]
        assert matches(out.b_ids, c["out"]["b_ids"]), c["name"]
        mv = C.join_probe_phase(p, C.Column.build(b))
        assert C.join_total_size(mv) == c["out"]["total"]
        assert matches(mv.matched, c["out"]["matched"])


def test_join_large_skewed_vs_oracle(C, oracle):
    p = W.random_values(31, 2_000_000, 20000, True)
    b = W.random_values(32, 300_000, 20000, False)
    out = C.column_join(p, C.Column.build(b))
    oa, ob = oracle.column_join(p, b)
    assert np.array_equal(out.a_ids, oa) and np.array_equal(out.b_ids, ob)


def test_filter_pairs_eq(C):
    a0, b0 = C.Column.build([1, 2, 3]), C.Column.build([1, 2, 9])
    pairs = C.IdPairSet(np.array([0, 1, 2], np.uint32), np.array([0, 1, 2], np.uint32))
    assert C.filter_pairs_eq(pairs, a0, b0).a_ids.tolist() == [0, 1]
    assert C.filter_pairs_eq(pairs, a0, C.Column.build([7, 7, 7])).size() == 0
    same = C.IdPairSet(np.array([0, 1], np.uint32), np.array([0, 1], np.uint32))
    assert C.filter_pairs_eq(same, a0, a0) == same


def test_multi_column_join_composition(C):
    for r in range(10):
        left = W.random_rows(240 + r, 150, 2, 12)
        right = W.random_rows(340 + r, 150, 2, 12)
        lv, rv = C.Version.from_columns(left.T), C.Version.from_columns(right.T)
        pairs = C.column_join(lv.col(0), rv.col(0))
        pairs = C.filter_pairs_eq(pairs, lv.col(1), rv.col(1))
        got = set(zip(pairs.a_ids.tolist(), pairs.b_ids.tolist()))
        exp = {(i, j) for i in range(150) for j in range(150) if tuple(left[i]) == tuple(right[j])}
        assert got == exp


def test_filter_neq_golden(C):
    for c in load_golden("filter_neq.json"):
        rows = np.asarray(c["rows"], np.uint32) if "rows" in c else W.random_rows(*c["gen"])
        v = C.Version.from_columns(rows.reshape(-1, c["arity"]).T)
        assert matches(C.filter_neq(v, c["i"], c["j"]), c["out"]), c["name"]


def test_deduplicate_golden(C, oracle):
    for c in load_golden("deduplicate.json"):
        a = c["arity"]
        if "gen" in c:
            full = oracle.dedup_rows(W.random_rows(*c["gen"][0]), a)
            new = oracle.dedup_rows(W.random_rows(*c["gen"][1]), a)
        else:
            full = np.asarray(c["full"], np.uint32).reshape(-1, a)
            new = np.asarray(c["new"], np.uint32).reshape(-1, a)
        nv = C.Version.from_columns(new.T) if new.size else C.Version.empty_version(a)
        fv = C.Version.from_columns(full.T) if full.size else C.Version.empty_version(a)
        assert matches(C.deduplicate(nv, fv).flags, c["out"]), c["name"]


def test_difference(C):
    nv = C.Version.decompose([(1, 2), (3, 4)], 2)
    assert C.difference(nv, [1, 1]).rows() == 0
    assert C.difference(nv, [0, 0]).reconstruct() == nv.reconstruct()
    assert C.difference(nv, [1, 0]).reconstruct() == [(3, 4)]
    with pytest.raises(_lib.ArityError):
        C.difference(nv, [1])


def test_union_concat(C):
    a, b = C.Version.decompose([(1, 1)], 2), C.Version.decompose([(2, 2)], 2)
    assert C.union_concat(a, b).rows() == 2
    lo = [(v, v) for v in range(1000)]
    hi = [(v, v) for v in range(1000, 1234)]
    assert C.union_concat(C.Version.decompose(lo, 2), C.Version.decompose(hi, 2)).rows() == 1234


def test_gather_volume_lazy_materialization(C):
    left, right = W.random_rows(28, 500, 2, 30), W.random_rows(29, 500, 2, 30)
    lv, rv = C.Version.from_columns(left.T), C.Version.from_columns(right.T)
    C.reset_gather_volume()
    pairs = C.column_join(lv.col(1), rv.col(0))
    assert C.gather_volume() == 0
    m = C.project(lv, pairs.a_ids, [0])
    assert C.gather_volume() == pairs.size() and m.rows() == pairs.size()


# ---- relation_test.cpp ------------------------------------------------------------------


def test_decompose_reconstruct(C):
    edge = C.Version.decompose([(0, 2), (1, 4), (3, 5)], 2)
    assert edge.col(0).value_at(1) == 1 and edge.col(1).value_at(1) == 4 and edge.rows() == 3
    assert C.Version.decompose([], 2).rows() == 0
    dup = C.Version.decompose([(2, 9), (2, 9)], 2)
    assert dup.rows() == 2
    for arity in (1, 2, 4):
        rows = W.random_rows(11 + arity, 500, arity, 50)
        assert np.array_equal(C.Version.decompose(rows, arity).reconstruct_array(), rows)
    with pytest.raises(_lib.ArityError):
        C.Version.decompose([(1, 2, 3)], 2)


def test_arity_beyond_max_is_rejected(C):
    # a 9-column version must be an FV_ERR_ARITY, not a stack overrun.
    rows = W.random_rows(5, 64, 9, 10)
    with pytest.raises(_lib.ArityError):
        C.Version.decompose(rows, 9)
    with pytest.raises(_lib.ArityError):
        C.Version.from_columns([rows[:, j] for j in range(9)])
    with pytest.raises(_lib.ArityError):
        C.Version.empty_version(9)
    v = C.Version.decompose(W.random_rows(6, 64, 3, 10), 3)
    with pytest.raises(_lib.ArityError):
        C.project(v, np.arange(64), [0, 1, 2, 0, 1, 2, 0, 1, 2])


def test_zero_column_version_has_no_rows(C):
    # P/include/colog/relation.hpp:31: Version::rows() is 0 without columns.
    v = C.Version.decompose(W.random_rows(7, 16, 2, 10), 2)
    p = C.project(v, np.arange(16), [])
    assert p.arity() == 0 and p.rows() == 0


def test_dedup_rows_golden(C):
    for c in load_golden("dedup_rows.json"):
        rows = (np.asarray(c["rows"], np.uint32).reshape(-1, c["arity"]) if "rows" in c
                else W.random_rows(*c["gen"]))
        v = C.Version.from_columns(rows.T) if rows.size else C.Version.empty_version(c["arity"])
        assert matches(C.dedup_rows(v).reconstruct_array(), c["out"]), c["name"]


def test_merge_delta_and_duplicates(C):
    rel = C.Relation("r", 2)
    rel.full = C.Version.decompose([(1, 2)], 2)
    rel.merge_delta(C.Version.decompose([(2, 3)], 2))
    assert rel.full.reconstruct() == [(1, 2), (2, 3)]
    assert rel.delta.reconstruct() == [(2, 3)]
    assert rel.new_rows.rows() == 0
    before = rel.full.reconstruct()
    rel.merge_delta(C.Version.empty_version(2))
    assert rel.full.reconstruct() == before and rel.delta.rows() == 0
    assert C.has_duplicate_rows(C.Version.decompose([(1, 2), (1, 2)], 2))
    assert not C.has_duplicate_rows(C.Version.decompose([(1, 2), (2, 1)], 2))


def test_difference_merge_stays_duplicate_free(C):
    rel = C.Relation("r", 2)
    rel.full = C.dedup_rows(C.Version.from_columns(W.random_rows(27, 200, 2, 8).T))
    for r in range(5):
        inc = C.dedup_rows(C.Version.from_columns(W.random_rows(270 + r, 80, 2, 8).T))
        flags = C.deduplicate(inc, rel.full)
        rel.merge_delta(C.difference(inc, flags))
        assert not C.has_duplicate_rows(rel.full)

"""GPU parity of the fixpoint engine (through the C ABI): identical sorted
tuple sets, per-iteration delta counts and iteration counts as the
reference (tests/golden/engine.json), the oracle restatement and the naive
evaluator; the reference's run()/CLI surface (P/tests/io_test.cpp:148-229,
P/tests/CMakeLists.txt:25-35); full-size checks at BASELINE sizes."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

import golden_cases
from conftest import GOLDEN, ROOT, load_golden, matches
from oracle import naive
from paper_2501_13051_b200 import _lib
from paper_2501_13051_b200 import engine as E
from paper_2501_13051_b200 import workloads as W
from progen import Rng, random_edb, random_program

pytestmark = pytest.mark.gpu


def _rows_set(a):
    return {tuple(r) for r in np.asarray(a).tolist()}


def test_engine_golden_cases(ctx):
    for case in load_golden("engine.json"):
        text, facts = golden_cases.program_and_facts(case)
        st = E.evaluate_program(text, facts, ctx=ctx)
        assert st.iterations == case["iterations"], case["name"]
        got_stats = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in st.stats()]
        assert got_stats == [tuple(s) for s in case["stats"]], case["name"]
        rels = st.relations()
        assert set(rels) == set(case["relations"]), case["name"]
        for rel, exp in case["relations"].items():
            assert rels[rel][1] == exp["rows"], (case["name"], rel)
            assert matches(st.dump(rel).reshape(-1), exp["dump"]), (case["name"], rel)


def test_engine_vs_oracle_and_naive_random_programs(ctx, oracle):
    g = Rng(56)
    compared = 0
    for _ in range(60):
        text, arities = random_program(g)
        prog = E.compile_program(text)
        if prog.validate():
            continue
        facts = random_edb(g, arities, 40)
        st = E.evaluate_program(prog, facts, ctx=ctx)
        it, rels, deltas = oracle.evaluate(*prog.oracle_args(facts))
        exp = naive.naive_evaluate(text, {k: [tuple(r) for r in v] for k, v in facts.items()})
        names = [r for r, _ in prog.relations()]
        assert st.iterations == it, text
        for k, name in enumerate(names):
            got = st.dump(name)
            assert np.array_equal(got, rels[k]), (text, name)
            assert _rows_set(got) == exp.get(name, set()), (text, name)
        dc = st.delta_counts()
        for rel, seq in dc.items():
            assert seq == [deltas[i][names.index(rel)] for i in range(it)], (text, rel)
        compared += 1
    assert compared > 15


@pytest.mark.parametrize("words", ["1", "0"])
def test_guard_with_a_ternary_build_side(ctx, words, monkeypatch):
    # Regression (found by the reference's own engine suite through the
    # drop-in shim, P/tests/engine_test.cpp:262-276, random program round 7):
    # a three-column build version was taken for a word-form one and the
    # guard v2 != v3 was dropped.
    monkeypatch.setenv("FVLOG_WORDS", words)
    text = ("i1(v3, v1) :- e0(v2, v4), i1(v1, v4), e1(v4, v4, v3), v2 != v3.\n"
            "i1(v3, v1) :- e1(v3, v1, v2), v3 != v2.\n")
    facts = {"e0": np.array([[7, 2], [5, 1], [3, 4], [5, 1], [1, 1]], np.uint32),
             "e1": np.array([[0, 5, 4], [5, 1, 0], [1, 3, 3], [3, 1, 2], [5, 4, 3], [5, 5, 7], [3, 4, 6], [0, 1, 0],
                             [4, 4, 3], [0, 2, 1], [5, 2, 4], [3, 6, 0], [1, 1, 1], [2, 1, 4], [3, 6, 2], [7, 3, 1],
                             [4, 7, 7], [1, 7, 3], [0, 4, 1], [4, 0, 6], [6, 5, 0], [4, 6, 3], [5, 2, 5], [2, 0, 6],
                             [0, 1, 7], [7, 1, 5], [1, 5, 4]], np.uint32)}
    st = E.evaluate_program(text, facts, ctx=ctx)
    exp = naive.naive_evaluate(text, {k: [tuple(int(x) for x in r) for r in v] for k, v in facts.items()})
    assert _rows_set(st.dump("i1")) == exp["i1"]


def test_residual_equalities_follow_the_naive_semantics(ctx):
    # Multi-variable joins: the reference's filter_pairs_eq (P/src/kernels.cpp:155)
    # indexes the left values by pair position; the engine implements the
    # intended semantics and is checked against the naive evaluator.
    text = ("t(x, y) :- a(x, y), b(x, y).\n"
            "u(x, z) :- a(x, y), b(y, x), c(x, y, z).\n"
            "p(x) :- a(x, x).\n")
    g = Rng(9)
    for r in range(6):
        facts = {"a": W.random_rows(100 + r, 80, 2, 6), "b": W.random_rows(200 + r, 80, 2, 6),
                 "c": W.random_rows(300 + r, 60, 3, 6)}
        st = E.evaluate_program(text, facts, ctx=ctx)
        exp = naive.naive_evaluate(text, {k: [tuple(x) for x in v] for k, v in facts.items()})
        for rel in ("t", "u", "p"):
            assert _rows_set(st.dump(rel)) == exp[rel], rel


def test_explicit_plan_boundary(ctx):
    prog = E.compile_program(W.SG_PROGRAM)
    facts = {"edge": W.binary_tree(6)}
    a = E.evaluate_program(prog, facts, ctx=ctx)
    b = E.evaluate(prog.relations(), prog.plans(), facts, ctx=ctx)
    assert np.array_equal(a.dump("sg"), b.dump("sg"))
    assert a.delta_counts() == b.delta_counts()
    bad = prog.plans()
    bad[1].joins[0].right_col = 7
    with pytest.raises(_lib.DiagnosticError):
        E.evaluate(prog.relations(), bad, facts, ctx=ctx)


def test_invalid_programs_raise_diagnostics(ctx):
    with pytest.raises(_lib.DiagnosticError, match="head variable 'z'"):
        E.evaluate_program("reach(x, z) :- edge(x, y).", {}, ctx=ctx)
    with pytest.raises(_lib.DiagnosticError, match="cross products"):
        E.evaluate_program("a(x, y) :- b(x), c(y).", {}, ctx=ctx)


def test_fingerprint_matches_host_restatement(ctx):
    st = E.evaluate_program(W.TC_PROGRAM, {"edge": W.tc_uniform(500, 2500, 3)}, ctx=ctx)
    assert st.fingerprint("reach") == E.fingerprint_rows(st.dump("reach"))


def test_seed_deduplicates_and_counts(ctx):
    st = E.evaluate_program(W.TC_PROGRAM, {"edge": np.array([[1, 2], [1, 2], [2, 3]], np.uint32)}, ctx=ctx)
    assert st.rows("edge") == 2
    assert _rows_set(st.dump("reach")) == {(1, 2), (2, 3), (1, 3)}
    s = E.evaluate_program("reach(x, y) :- edge(x, y).\n", {"edge": np.array([[1, 2]], np.uint32)}, ctx=ctx)
    assert s.iterations == 2


def test_delta_sum_equals_full(ctx):
    st = E.evaluate_program(W.TC_PROGRAM, {"edge": W.path_graph(15)}, ctx=ctx)
    assert sum(st.delta_counts()["reach"]) == st.rows("reach") == 105


def test_max_u32_values_and_arity4(ctx):
    big = np.array([[4294967295, 0], [0, 4294967294], [4294967294, 4294967295]], np.uint32)
    st = E.evaluate_program(W.TC_PROGRAM, {"edge": big}, ctx=ctx)
    exp = naive.naive_evaluate(W.TC_PROGRAM, {"edge": [tuple(map(int, r)) for r in big]})
    assert _rows_set(st.dump("reach")) == exp["reach"]
    text = "q(a, b, c, d) :- r(a, b, c, d).\nq(a, b, c, e) :- q(a, b, c, d), r(d, x, y, e), a != e.\n"
    facts = {"r": W.random_rows(5, 200, 4, 9)}
    st = E.evaluate_program(text, facts, ctx=ctx)
    exp = naive.naive_evaluate(text, {"r": [tuple(map(int, r)) for r in facts["r"]]})
    assert _rows_set(st.dump("q")) == exp["q"]


# ---- runner / CLI (P/tests/io_test.cpp:161-229, P/tests/CMakeLists.txt:25-35) ----------------


def test_run_path10_end_to_end():
    with tempfile.TemporaryDirectory() as d:
        prog = os.path.join(d, "tc.dl")
        open(prog, "w").write(W.TC_PROGRAM)
        W.write_tsv_dir(os.path.join(d, "facts"), {"edge": W.path_graph(10)})
        rc, out, err = E.run(prog, os.path.join(d, "facts"), os.path.join(d, "out"), stats=True, dump=["reach"])
        assert rc == 0 and err == ""
        assert "rel=reach rows=45" in out and "iter=0 rel=reach delta=9" in out
        assert open(os.path.join(d, "out", "reach.tsv")).readline().strip() == "0\t1"


def test_run_rejects_invalid_program():
    with tempfile.TemporaryDirectory() as d:
        prog = os.path.join(d, "bad.dl")
        open(prog, "w").write("reach(x, z) :- edge(x, y).\n")
        os.makedirs(os.path.join(d, "facts"))
        rc, out, err = E.run(prog, os.path.join(d, "facts"), os.path.join(d, "out"))
        assert rc != 0 and "head variable 'z'" in err


def test_run_resolves_string_constants():
    with tempfile.TemporaryDirectory() as d:
        prog = os.path.join(d, "family.dl")
        open(prog, "w").write('parentof("Larry", "Alice").\nparentof("Alice", "Bob").\n'
                              "ancestor(x, y) :- parentof(x, y).\n"
                              "ancestor(x, z) :- parentof(x, y), ancestor(y, z).\n")
        os.makedirs(os.path.join(d, "facts"))
        rc, out, err = E.run(prog, os.path.join(d, "facts"), os.path.join(d, "out"), dump=["ancestor"])
        assert rc == 0 and "rel=ancestor rows=3" in out
        assert "Larry\tBob" in open(os.path.join(d, "out", "ancestor.tsv")).read()


def test_cli_binary_matches_reference_ctests():
    cli = os.path.join(ROOT, "paper_2501_13051_b200", "fvlog")
    data = os.path.join(ROOT, "tests", "data")
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([cli, "run", os.path.join(data, "tc.dl"), "--facts", os.path.join(data, "path10"),
                            "--out", d, "--dump", "reach"], capture_output=True, text=True)
        assert r.returncode == 0 and "rel=reach rows=45" in r.stdout
        r = subprocess.run([cli, "run", os.path.join(data, "invalid_unbound.dl"), "--facts",
                            os.path.join(data, "path10"), "--out", d], capture_output=True, text=True)
        assert r.returncode != 0


# ---- full BASELINE sizes: size-independent checks --------------------------------------------


def _large():
    p = os.path.join(GOLDEN, "large.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def test_sg_c3_full_size_against_reference(ctx):
    st = E.evaluate_program(W.SG_PROGRAM, {"edge": W.sg_forest(244, 10)}, ctx=ctx)
    assert st.rows("sg") == W.sg_count(244, 10) == 340_637_176
    assert st.iterations == 11
    assert sum(st.delta_counts()["sg"]) == 340_637_176
    # The tuple set itself, not just its size: fingerprint and per-iteration
    # deltas of the unmodified reference run over the forest's disjoint trees.
    g = _large().get("C3")
    if g and "fingerprint" in g:
        assert str(st.fingerprint("sg")) == g["fingerprint"]
        assert st.delta_counts()["sg"] == g["deltas"]


def test_sg_beyond_c3_1e9_tuples(ctx):
    # Maximum-size case: 61 depth-12 trees (499,590 edges) derive 1.36e9 SG
    # tuples (~4x C3): key set, levels and sort scratch must fit one B200.
    st = E.evaluate_program(W.SG_PROGRAM, {"edge": W.sg_forest(61, 12)}, ctx=ctx)
    assert st.rows("sg") == W.sg_count(61, 12) == 1_364_047_230
    assert st.iterations == 13
    assert sum(st.delta_counts()["sg"]) == 1_364_047_230


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_tc_full_size_against_large_goldens(ctx, cfg):
    g = _large().get(cfg)
    if not g:
        pytest.skip(f"{cfg} golden not generated (tests/golden/make_golden_large.py)")
    edges = W.tc_uniform(10_000, 50_000, 1) if cfg == "C1" else W.tc_powerlaw(1000, 1000, 5000, 1)
    st = E.evaluate_program(W.TC_PROGRAM, {"edge": edges}, ctx=ctx)
    assert st.rows("reach") == g["rows"]
    assert st.delta_counts()["reach"] == g["deltas"]
    assert st.iterations == g["iterations"]
    assert str(st.fingerprint("reach")) == g["fingerprint"]


@pytest.mark.parametrize("mode", ["sort", "hash"])
def test_both_dedup_strategies_match_reference(ctx, mode, monkeypatch):
    # FVLOG_DEDUP=sort: radix sort + merge-path for every relation;
    # default (hash): key-set dedup fused into the join for arity <= 2.
    monkeypatch.setenv("FVLOG_DEDUP", mode)
    for case in load_golden("engine.json"):
        if case["name"] == "TC uniform 2000/10000":
            continue
        text, facts = golden_cases.program_and_facts(case)
        st = E.evaluate_program(text, facts, ctx=ctx)
        got = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in st.stats()]
        assert got == [tuple(s) for s in case["stats"]], (mode, case["name"])
        for rel, exp in case["relations"].items():
            assert matches(st.dump(rel).reshape(-1), exp["dump"]), (mode, case["name"], rel)


def _check_relations(st, g):
    rels = st.relations()
    for rel, exp in g["relations"].items():
        assert rels[rel][1] == exp["rows"], rel
        assert str(st.fingerprint(rel)) == exp["fingerprint"], rel
    deltas = st.delta_counts()
    for rel, exp in g["relations"].items():
        if rel in deltas:
            assert deltas[rel] == exp["deltas"], rel
    assert st.iterations == g["iterations"]


def test_lubm_c5_full_size_against_reference(ctx):
    """C5: OWL-RL/LUBM rule set on ~10.2 M facts vs the unmodified reference
    (tests/golden/make_golden_large.py c5)."""
    g = _large().get("C5")
    if not g:
        pytest.skip("C5 golden not generated")
    st = E.evaluate_program(W.LUBM_PROGRAM, W.lubm_facts(340), ctx=ctx)
    _check_relations(st, g)


def test_cspa_c4_full_size_against_reference(ctx):
    """C4: CSPA on 4000 disjoint functions vs the unmodified reference run
    component-batch by component-batch (fingerprints, row counts and
    per-iteration deltas add over disjoint components)."""
    g = _large().get("C4")
    if not g:
        pytest.skip("C4 golden not generated")
    st = E.evaluate_program(W.CSPA_PROGRAM, W.cspa_facts(4000, 100, 100, 70), ctx=ctx)
    _check_relations(st, g)


@pytest.mark.parametrize("order", ["rule", "delta"])
def test_join_orders_match_reference(ctx, order, monkeypatch):
    # FVLOG_JOIN_ORDER=rule: every variant joins in the rule's atom order
    # (compile_rule); default: delta-first order for >= 3-atom variants with
    # an IDB atom before DELTA. Both must give the reference's sets and stats.
    monkeypatch.setenv("FVLOG_JOIN_ORDER", order)
    for case in load_golden("engine.json"):
        if case["name"] == "TC uniform 2000/10000":
            continue
        text, facts = golden_cases.program_and_facts(case)
        st = E.evaluate_program(text, facts, ctx=ctx)
        got = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in st.stats()]
        assert got == [tuple(s) for s in case["stats"]], (order, case["name"])
        for rel, exp in case["relations"].items():
            assert matches(st.dump(rel).reshape(-1), exp["dump"]), (order, case["name"], rel)


@pytest.mark.parametrize("grow", ["windowed", "rehash", "overflow"])
def test_keyset_growth_paths_match_reference(ctx, grow, monkeypatch):
    # Key-set growth: windowed shared-memory rebuild (default; its overflow
    # list holds the few keys that leave their window), memset + atomic
    # rehash (FVLOG_GROW=rehash), or the windowed pass abandoned because the
    # overflow list filled up (a 1-entry list) and redone by the rehash.
    # All must give the reference's sets. C1 at full size grows its key set
    # several times (2^16 -> 2^30 slots).
    monkeypatch.setenv("FVLOG_SET", "keyset")
    if grow == "overflow":
        monkeypatch.setenv("FVLOG_GROW_OVERFLOW_CAP", "1")
    else:
        monkeypatch.setenv("FVLOG_GROW", grow)
    for case in load_golden("engine.json"):
        text, facts = golden_cases.program_and_facts(case)
        st = E.evaluate_program(text, facts, ctx=ctx)
        got = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in st.stats()]
        assert got == [tuple(s) for s in case["stats"]], (grow, case["name"])
        for rel, exp in case["relations"].items():
            assert matches(st.dump(rel).reshape(-1), exp["dump"]), (grow, case["name"], rel)
    g = _large().get("C1")
    if g:
        st = E.evaluate_program(W.TC_PROGRAM, {"edge": W.tc_uniform(10_000, 50_000, 1)}, ctx=ctx)
        assert st.rows("reach") == g["rows"]
        assert st.delta_counts()["reach"] == g["deltas"]
        assert str(st.fingerprint("reach")) == g["fingerprint"]


@pytest.mark.parametrize("setmode", [
    {"FVLOG_SET": "keyset"},                                  # key sets only (round-1 engine)
    {"FVLOG_SET": "blocks"},                                  # block sets, never converted
    {"FVLOG_SET": "blocks", "FVLOG_BLOCK_RATIO": "0"},        # directory never pre-grown: overflow lists drained
    {"FVLOG_BLOCK_SPARSE_BYTES": "0"},                        # sparse relations convert to key sets mid-run
    {"FVLOG_BLOCK_TILE_SET": "0"},                            # no tile-local dedup before the block set
    {"FVLOG_WORDS": "0"},                                     # tuple-form DELTA for every block-set relation
    {"FVLOG_BLOCK_RATIO": "0"},                               # word form with overflow lists drained
    {"FVLOG_BLOCK_SPARSE_BYTES": "0", "FVLOG_WORDS": "1"},    # word form left mid-run (sparse -> key set)
    {"FVLOG_WORD_COMBINE": "0"},                              # no tile-local OR-combine of word outputs
    {"FVLOG_DUMP_SORT": "1"},                                 # dumps by sorting the levels, not from the bitmaps
    {"FVLOG_INTER_PROBE_ROWS": "2"},                          # intermediates deduplicated early (word intermediates)
    {"FVLOG_INTER_PROBE_ROWS": "2", "FVLOG_WORDS": "0"},      # ... by sort-unique
    {"FVLOG_REVERSE": "1"},                                   # word compositions always probe DELTA's words
    {"FVLOG_REVERSE": "0"},                                   # ... never
    {"FVLOG_BY1": "0"},                                       # column-1 indexes of FULL re-sorted every iteration
    {"FVLOG_SCATTER_GATHER": "1"},                            # DELTA masks read by the grouping scatter
    {"FVLOG_PRECOUNT": "0"},                                  # every join step reads its own output size
    {"FVLOG_SEED_BATCH": "0"},                                # every EDB seed sorted on its own
    {"FVLOG_PROBE_SCAN": "0"},                                # join counts written, then scanned by a second kernel
    {"FVLOG_GROUPED_EXPAND": "0"},                            # tuple DELTA of a word sink via a tuple-level counting sort
    {"FVLOG_EXACT_BLOCKS": "1"},                              # directories sized by exact block counts, not the sketch
    {"FVLOG_BLOCK_HEADROOM": "2"},                            # directories grown to 2x their blocks (more growth passes)
], ids=["keyset", "blocks", "blocks-overflow", "blocks-convert", "blocks-no-tile-set", "no-words",
        "words-overflow", "words-leave", "words-no-combine", "dump-sort", "inter-words", "inter-sort",
        "reverse-always", "reverse-never", "by1-resort", "scatter-gather", "no-precount", "no-seed-batch", "no-probe-scan", "no-grouped-expand", "exact-blocks", "headroom-2"])
def test_dedup_sets_match_reference(ctx, setmode, monkeypatch):
    # FULL's dedup structure for binary/unary IDB relations: a BlockSet
    # (blocked bitmap, default) or a KeySet; every path must give the
    # reference's sets and per-iteration stats, C1 included at full size.
    for k, v in setmode.items():
        monkeypatch.setenv(k, v)
    for case in load_golden("engine.json"):
        text, facts = golden_cases.program_and_facts(case)
        st = E.evaluate_program(text, facts, ctx=ctx)
        got = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in st.stats()]
        assert got == [tuple(s) for s in case["stats"]], (setmode, case["name"])
        for rel, exp in case["relations"].items():
            assert matches(st.dump(rel).reshape(-1), exp["dump"]), (setmode, case["name"], rel)
    g = _large().get("C1")
    if g:
        st = E.evaluate_program(W.TC_PROGRAM, {"edge": W.tc_uniform(10_000, 50_000, 1)}, ctx=ctx)
        assert st.rows("reach") == g["rows"]
        assert st.delta_counts()["reach"] == g["deltas"]
        assert str(st.fingerprint("reach")) == g["fingerprint"]


@pytest.mark.parametrize("group", ["0", "1"])
def test_keyset_layouts_match_reference(ctx, group, monkeypatch):
    # FVLOG_KEYSET_GROUP forces the key-set home layout (0: every key
    # scattered, 1: adjacent key pairs share a sector); the default picks one
    # per relation from candidates per new row. Results must not depend on it.
    monkeypatch.setenv("FVLOG_SET", "keyset")
    monkeypatch.setenv("FVLOG_KEYSET_GROUP", group)
    for case in load_golden("engine.json"):
        if case["name"] == "TC uniform 2000/10000":
            continue
        text, facts = golden_cases.program_and_facts(case)
        st = E.evaluate_program(text, facts, ctx=ctx)
        got = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in st.stats()]
        assert got == [tuple(s) for s in case["stats"]], (group, case["name"])
        for rel, exp in case["relations"].items():
            assert matches(st.dump(rel).reshape(-1), exp["dump"]), (group, case["name"], rel)


@pytest.mark.parametrize("mode", ["reference", "exactly-once"])
def test_seminaive_variants_match_reference(ctx, mode, monkeypatch):
    # Default: the variant with DELTA at IDB occurrence i reads FULL - DELTA
    # before i (each multi-DELTA derivation once); FVLOG_SEMINAIVE=reference
    # reads FULL everywhere like P/src/engine.cpp:180-183. Same sets/stats.
    if mode == "reference":
        monkeypatch.setenv("FVLOG_SEMINAIVE", "reference")
    for case in load_golden("engine.json"):
        if case["name"] == "TC uniform 2000/10000":
            continue
        text, facts = golden_cases.program_and_facts(case)
        st = E.evaluate_program(text, facts, ctx=ctx)
        got = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in st.stats()]
        assert got == [tuple(s) for s in case["stats"]], (mode, case["name"])
        for rel, exp in case["relations"].items():
            assert matches(st.dump(rel).reshape(-1), exp["dump"]), (mode, case["name"], rel)


def test_bounded_pool_compaction_matches_reference(ctx, monkeypatch):
    # Sorted-mode dedup with tiny join chunks and pool budget: candidates are
    # produced chunk by chunk and the pool is sort-uniqued whenever it would
    # outgrow the budget (bounded memory); results and stats must not change.
    monkeypatch.setenv("FVLOG_DEDUP", "sort")
    monkeypatch.setenv("FVLOG_POOL_CHUNK", "1000")
    monkeypatch.setenv("FVLOG_POOL_BUDGET", "3000")
    for case in load_golden("engine.json"):
        if case["name"] in ("TC uniform 2000/10000", "SG tree depth 10"):
            continue
        text, facts = golden_cases.program_and_facts(case)
        st = E.evaluate_program(text, facts, ctx=ctx)
        got = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in st.stats()]
        assert got == [tuple(s) for s in case["stats"]], case["name"]
        for rel, exp in case["relations"].items():
            assert matches(st.dump(rel).reshape(-1), exp["dump"]), (case["name"], rel)


def test_chunked_join_chains_match_reference(ctx, monkeypatch):
    # Intermediates of multi-join rules carried through the rest of the chain
    # in tiny chunks (bounded memory): same sets and stats.
    monkeypatch.setenv("FVLOG_INTER_CHUNK", "50")
    for case in load_golden("engine.json"):
        if case["name"] in ("TC uniform 2000/10000", "SG tree depth 10"):
            continue
        text, facts = golden_cases.program_and_facts(case)
        st = E.evaluate_program(text, facts, ctx=ctx)
        got = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in st.stats()]
        assert got == [tuple(s) for s in case["stats"]], case["name"]
        for rel, exp in case["relations"].items():
            assert matches(st.dump(rel).reshape(-1), exp["dump"]), (case["name"], rel)

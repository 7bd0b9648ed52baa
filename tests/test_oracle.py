"""CPU: the oracle restatement (oracle/colog_oracle.c) against the golden
vectors produced by the unmodified reference (tests/golden/make_golden.py),
and directly against oracle/_ref when it is built here."""
import numpy as np
import pytest

from conftest import load_golden, matches
from paper_2501_13051_b200 import workloads as W


def _column_raw(c):
    return np.asarray(c["raw"], np.uint32) if "raw" in c else W.random_values(*c["gen"][1:])


def test_build_index_golden(oracle):
    for c in load_golden("column.json"):
        s, k, st, cnt = oracle.build_index(_column_raw(c))
        o = c["out"]
        assert matches(s, o["sorted_idx"]), c["name"]
        assert matches(k, o["keys"]) and matches(st, o["starts"]) and matches(cnt, o["counts"]), c["name"]


def _join_inputs(c):
    if "gen" in c:
        return W.random_values(*c["gen"][0]), W.random_values(*c["gen"][1])
    return np.asarray(c["probe"], np.uint32), np.asarray(c["build"], np.uint32)


def test_column_join_golden(oracle):
    for c in load_golden("join.json"):
        p, b = _join_inputs(c)
        a_ids, b_ids = oracle.column_join(p, b)
        assert matches(a_ids, c["out"]["a_ids"]) and matches(b_ids, c["out"]["b_ids"]), c["name"]
        s, cnt, m, total = oracle.join_probe(p, b)
        assert total == c["out"]["total"]
        assert matches(s, c["out"]["starts"]) and matches(cnt, c["out"]["counts"])
        assert matches(m, c["out"]["matched"])


def test_dedup_rows_golden(oracle):
    for c in load_golden("dedup_rows.json"):
        rows = (np.asarray(c["rows"], np.uint32).reshape(-1, c["arity"]) if "rows" in c
                else W.random_rows(*c["gen"]))
        assert matches(oracle.dedup_rows(rows, c["arity"]), c["out"]), c["name"]


def test_deduplicate_golden(oracle):
    for c in load_golden("deduplicate.json"):
        a = c["arity"]
        if "gen" in c:
            full = oracle.dedup_rows(W.random_rows(*c["gen"][0]), a)
            new = oracle.dedup_rows(W.random_rows(*c["gen"][1]), a)
        else:
            full = np.asarray(c["full"], np.uint32).reshape(-1, a)
            new = np.asarray(c["new"], np.uint32).reshape(-1, a)
        assert matches(oracle.deduplicate(new, full, a), c["out"]), c["name"]


def test_filter_neq_golden(oracle):
    for c in load_golden("filter_neq.json"):
        rows = np.asarray(c["rows"], np.uint32) if "rows" in c else W.random_rows(*c["gen"])
        assert matches(oracle.filter_neq(rows, c["arity"], c["i"], c["j"]), c["out"]), c["name"]


def test_oracle_against_built_reference(oracle):
    from oracle.bind import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    ref = Reference()
    for seed in range(6):
        a = W.random_values(seed, 2500, 300, seed % 2 == 0)
        b = W.random_values(seed + 50, 1800, 300, True)
        for x, y in zip(oracle.build_index(a), ref.build_index(a)):
            assert np.array_equal(x, y)
        for x, y in zip(oracle.column_join(a, b), ref.column_join(a, b)):
            assert np.array_equal(x, y)
        rows = W.random_rows(seed, 700, 3, 5)
        assert np.array_equal(oracle.dedup_rows(rows, 3), ref.dedup_rows(rows, 3))


# ---- engine: oracle restatement vs reference goldens and the naive oracle ----

import json
import os

from paper_2501_13051_b200 import engine as E
from oracle import naive
from progen import Rng, random_edb, random_program
import golden_cases


def test_oracle_engine_golden(oracle):
    for case in load_golden("engine.json"):
        text, facts = golden_cases.program_and_facts(case)
        if case["name"] == "SG tree depth 10":
            continue  # 1.4M rows: covered on the GPU; too slow for the C oracle here
        prog = E.compile_program(text)
        it, rels, deltas = oracle.evaluate(*prog.oracle_args(facts))
        assert it == case["iterations"], case["name"]
        names = [r for r, _ in prog.relations()]
        for rel, exp in case["relations"].items():
            got = rels[names.index(rel)]
            assert got.shape[0] == exp["rows"], (case["name"], rel)
            assert matches(got.reshape(-1), exp["dump"]), (case["name"], rel)
        for (i, rel, d, _full, _m) in case["stats"]:
            assert deltas[i][names.index(rel)] == d, (case["name"], i, rel)


def test_oracle_engine_vs_naive_random_programs(oracle):
    g = Rng(56)
    compared = 0
    for _ in range(40):
        text, arities = random_program(g)
        prog = E.compile_program(text)
        if prog.validate():
            continue
        facts = random_edb(g, arities, 40)
        it, rels, _ = oracle.evaluate(*prog.oracle_args(facts))
        exp = naive.naive_evaluate(text, {k: [tuple(r) for r in v] for k, v in facts.items()})
        for k, (name, _a) in enumerate(prog.relations()):
            assert {tuple(r) for r in rels[k].tolist()} == exp.get(name, set()), (text, name)
        compared += 1
    assert compared > 10

"""Generate tests/golden/*.json from the UNMODIFIED reference.

Runs oracle/_ref/libcolog_ref.so (built from /root/reference/proj/src by
`make -C oracle ref`) on deterministic splitmix64 inputs and records its
outputs. Small outputs are stored verbatim, large ones as (length, sha256).
The fixtures are committed; /root/reference is not needed to read them.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bind import Reference  # noqa: E402
from paper_2501_13051_b200 import workloads as W  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SMALL = 4096


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype="<u4")).tobytes()).hexdigest()


def enc(a):
    a = np.asarray(a)
    if a.size <= SMALL:
        return a.tolist()
    return {"len": int(a.shape[0]), "sha256": digest(a)}


def gen_column(ref: Reference):
    cases = [
        {"name": "column_test.cpp:61-68", "raw": [5, 3, 5, 1]},
        {"name": "column_test.cpp:70-74", "raw": [1, 1, 1, 2, 3, 3, 3, 3, 4, 4, 4, 4]},
        {"name": "column_test.cpp:76-81 empty", "raw": []},
        {"name": "single", "raw": [7]},
        {"name": "max u32 values", "raw": [4294967295, 0, 4294967295, 2147483648, 1]},
    ]
    for i in range(40):  # column_test.cpp:120-132 shape (portable generator)
        n = int(W.uniform(101, 1, 3000, i)[0])
        dom = int(W.uniform(102, 1, 499, i)[0]) + 1
        cases.append({"name": f"random-{i}", "gen": ["random_values", 1000 + i, n, dom, i % 3 == 0]})
    cases.append({"name": "random-100k", "gen": ["random_values", 2000, 100000, 5000, False]})
    cases.append({"name": "skew-1M", "gen": ["random_values", 2001, 1000000, 100000, True]})
    for c in cases:
        raw = c["raw"] if "raw" in c else W.random_values(*c["gen"][1:])
        s, k, st, cnt = ref.build_index(raw)
        c["out"] = {"sorted_idx": enc(s), "keys": enc(k), "starts": enc(st), "counts": enc(cnt)}
    return cases


def gen_join(ref: Reference):
    cases = [
        {"name": "kernels_test.cpp:65-90 Alg.1", "probe": [1, 2, 7, 3, 4],
         "build": [1, 1, 1, 2, 3, 3, 3, 3, 4, 4, 4, 4]},
        {"name": "kernels_test.cpp:100-105", "probe": [1, 2, 2], "build": [2, 2, 3]},
        {"name": "disjoint", "probe": [1, 2, 3], "build": [4, 5]},
        {"name": "empty probe", "probe": [], "build": [4, 5]},
        {"name": "empty build", "probe": [1, 2, 3], "build": []},
    ]
    for i in range(60):  # kernels_test.cpp:107-137 shape
        na = int(W.uniform(21, 1, 400, 3 * i)[0])
        nb = int(W.uniform(21, 1, 400, 3 * i + 1)[0])
        dom = int(W.uniform(21, 1, 59, 3 * i + 2)[0]) + 1
        cases.append({"name": f"random-{i}", "gen": [[3000 + i, na, dom, i % 4 == 0],
                                                     [4000 + i, nb, dom, i % 4 == 0]]})
    cases.append({"name": "skew-200k", "gen": [[5000, 200000, 2000, True], [5001, 50000, 2000, True]]})
    for c in cases:
        if "gen" in c:
            p = W.random_values(*c["gen"][0])
            b = W.random_values(*c["gen"][1])
        else:
            p, b = c["probe"], c["build"]
        a_ids, b_ids = ref.column_join(p, b)
        s, cnt, m, off, total = ref.join_probe(p, b)
        c["out"] = {"a_ids": enc(a_ids), "b_ids": enc(b_ids), "total": int(total),
                    "starts": enc(s), "counts": enc(cnt), "matched": enc(m),
                    "offsets": enc(off.astype(np.uint64).view(np.uint32).reshape(-1)) if off.size > SMALL
                    else off.tolist()}
    return cases


def gen_dedup(ref: Reference):
    cases = [
        {"name": "relation_test.cpp:94-99", "arity": 2, "rows": [[5, 5], [1, 1], [5, 5], [2, 2], [1, 1]]},
        {"name": "relation_test.cpp:90", "arity": 2, "rows": [[1, 2], [1, 2], [3, 4]]},
        {"name": "arity-1", "arity": 1, "rows": [[4], [4], [2]]},
        {"name": "empty", "arity": 2, "rows": []},
    ]
    for arity in (1, 2, 3, 4):
        for i in range(6):
            cases.append({"name": f"random-a{arity}-{i}", "arity": arity,
                          "gen": [6000 + 10 * arity + i, 1000, arity, 15 if i % 2 else 4]})
    cases.append({"name": "big-a2", "arity": 2, "gen": [7000, 300000, 2, 300]})
    for c in cases:
        rows = np.asarray(c["rows"], np.uint32).reshape(-1, c["arity"]) if "rows" in c else \
            W.random_rows(*c["gen"])
        c["out"] = enc(ref.dedup_rows(rows, c["arity"]).reshape(-1))
    return cases


def gen_deduplicate(ref: Reference):
    cases = [
        {"name": "kernels_test.cpp:212-223", "arity": 2, "new": [[1, 2], [3, 4]], "full": [[1, 2]]},
        {"name": "kernels_test.cpp:225-231 overlap", "arity": 2, "new": [[1, 4]], "full": [[1, 2], [3, 4]]},
        {"name": "empty full", "arity": 2, "new": [[1, 2], [3, 4]], "full": []},
    ]
    for arity in (1, 2, 3, 4):  # kernels_test.cpp:233-250 shape
        for i in range(12):
            dom = 4 if i % 2 else 12
            cases.append({"name": f"random-a{arity}-{i}", "arity": arity,
                          "gen": [[8000 + 100 * arity + i, 300, arity, dom],
                                  [9000 + 100 * arity + i, 120, arity, dom]]})
    for c in cases:
        a = c["arity"]
        if "gen" in c:
            full = ref.dedup_rows(W.random_rows(*c["gen"][0]), a)
            new = ref.dedup_rows(W.random_rows(*c["gen"][1]), a)
        else:
            full = np.asarray(c["full"], np.uint32).reshape(-1, a)
            new = np.asarray(c["new"], np.uint32).reshape(-1, a)
        c["out"] = enc(ref.deduplicate(new, full, a))
    return cases


def gen_filter_neq(ref: Reference):
    cases = [{"name": "kernels_test.cpp:196-198", "arity": 2, "rows": [[1, 1], [1, 2]], "i": 0, "j": 1},
             {"name": "all equal", "arity": 2, "rows": [[3, 3], [9, 9]], "i": 0, "j": 1},
             {"name": "random", "arity": 3, "gen": [9500, 400, 3, 6], "i": 2, "j": 0}]
    for c in cases:
        rows = np.asarray(c["rows"], np.uint32) if "rows" in c else W.random_rows(*c["gen"])
        c["out"] = enc(ref.filter_neq(rows, c["arity"], c["i"], c["j"]))
    return cases


ENGINE_CASES = [
    # name, program, {rel: generator spec}
    ("tc-path10 (data/samples/path10)", "TC", {"edge": ["path_graph", 10]}),
    ("engine_test.cpp:158-174 TC 3-path", "TC", {"edge": ["rows", [[1, 2], [2, 3]]]}),
    ("engine_test.cpp:208-218 path-30", "TC", {"edge": ["path_graph", 30]}),
    ("engine_test.cpp:208-218 cycle-12", "TC", {"edge": ["cycle_graph", 12]}),
    ("engine_test.cpp:198-206 saturated copy", "reach(x, y) :- edge(x, y).\n", {"edge": ["rows", [[1, 2]]]}),
    ("engine_test.cpp:220-228 SG tree depth 3", "SG", {"edge": ["binary_tree", 3]}),
    ("SG tree depth 10", "SG", {"edge": ["binary_tree", 10]}),
    ("TC uniform 300/1500", "TC", {"edge": ["tc_uniform", 300, 1500, 1]}),
    ("TC uniform 2000/10000", "TC", {"edge": ["tc_uniform", 2000, 10000, 1]}),
    ("TC powerlaw 4x(200,1000)", "TC", {"edge": ["tc_powerlaw", 4, 200, 1000, 1]}),
    ("CSPA 3x60", "CSPA", {"cspa": [3, 60, 80, 60, 3]}),
    ("LUBM scale 1", "LUBM", {"lubm": [1, 5]}),
    ("engine_test.cpp:287-305 LUBM-style 6 rules",
     "professor(x) :- fullprofessor(x).\nfaculty(x) :- professor(x).\n"
     "worksfor(x, y) :- headof(x, y).\nmemberof(x, y) :- worksfor(x, y).\n"
     "suborgof(x, z) :- suborgof(x, y), suborgof(y, z).\n"
     "memberof(x, z) :- memberof(x, y), suborgof(y, z).\n",
     {"fullprofessor": ["random_rows", 57, 20, 1, 30], "headof": ["random_rows", 58, 30, 2, 30],
      "suborgof": ["random_rows", 59, 50, 2, 15]}),
    ("constants and repeated vars",
     "a(x) :- b(3, x), c(x, x).\nd(x, y) :- b(x, y), c(y, y), x != y.\n",
     {"b": ["rows", [[3, 5], [3, 6], [4, 7], [5, 5]]], "c": ["rows", [[5, 5], [6, 9], [7, 7]]]}),
    ("mutual recursion + 3-atom",
     "p(x, y) :- e(x, y).\nq(x, z) :- p(x, y), e(y, z).\np(x, z) :- q(x, y), p(y, z), x != z.\n",
     {"e": ["random_rows", 61, 60, 2, 20]}),
]

PROGRAMS = {"TC": W.TC_PROGRAM, "SG": W.SG_PROGRAM, "CSPA": W.CSPA_PROGRAM, "LUBM": W.LUBM_PROGRAM}


def engine_facts(spec: dict):
    facts = {}
    for rel, g in spec.items():
        if rel in ("cspa", "lubm"):
            facts.update(W.cspa_facts(*g) if rel == "cspa" else W.lubm_facts(*g))
            continue
        kind, args = g[0], g[1:]
        if kind == "rows":
            facts[rel] = np.asarray(args[0], np.uint32)
        else:
            facts[rel] = getattr(W, kind)(*args)
    return facts


def gen_engine(ref: Reference):
    cases = []
    for name, prog, spec in ENGINE_CASES:
        text = PROGRAMS.get(prog, prog)
        facts = engine_facts(spec)
        rep = ref.evaluate(text, facts)
        rels = {}
        for rel, rows in rep["relations"].items():
            rels[rel] = {"rows": int(rows.shape[0]),
                         "dump": enc(rows.reshape(-1)) if rows.size <= SMALL else
                         {"len": int(rows.size), "sha256": digest(rows.reshape(-1))}}
        cases.append({"name": name, "program": prog, "facts": spec, "iterations": rep["iterations"],
                      "stats": rep["stats"], "relations": rels})
    return cases


def main():
    if not Reference.available():
        sys.exit("oracle/_ref/libcolog_ref.so missing: run `make -C oracle ref` first")
    ref = Reference()
    out = {
        "column.json": gen_column(ref),
        "join.json": gen_join(ref),
        "dedup_rows.json": gen_dedup(ref),
        "deduplicate.json": gen_deduplicate(ref),
        "filter_neq.json": gen_filter_neq(ref),
        "engine.json": gen_engine(ref),
    }
    for fname, data in out.items():
        with open(os.path.join(OUT, fname), "w") as fh:
            json.dump({"generator": "tests/golden/make_golden.py (unmodified reference via "
                                    "oracle/_ref/libcolog_ref.so)", "cases": data}, fh)
        print(fname, len(data))


if __name__ == "__main__":
    main()

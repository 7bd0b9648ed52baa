"""Deterministic synthetic inputs for the Datalog workloads.

All randomness is splitmix64 (portable, unlike the reference's
std::uniform_int_distribution streams, P/tests/support.hpp:29-50), so the
GPU engine, the oracle and the reference CPU engine read identical facts.
Values are dense u32 node ids.

Programs are the reference's TC/SG (P/data/programs/*.dl), the standard
CSPA rules and an OWL-RL/LUBM-style rule set.
"""
from __future__ import annotations

import os
from typing import Dict, List, Tuple

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """n consecutive splitmix64 outputs of the stream seeded with `seed`."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, n: int, hi: int, offset: int = 0) -> np.ndarray:
    """n values in [0, hi] (inclusive, like uniform_int_distribution(0, hi))."""
    return (splitmix64(seed, n, offset) % np.uint64(hi + 1)).astype(np.uint32)


def unit(seed: int, n: int, offset: int = 0) -> np.ndarray:
    return (splitmix64(seed, n, offset) >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


# ---- column / row generators (support.hpp analogues) -------------------------


def random_values(seed: int, n: int, domain: int, skew: bool = False) -> np.ndarray:
    """~support.hpp:29-41: values in [0, domain]; skew puts ~90% on one key."""
    v = uniform(seed, n, domain)
    if skew and n:
        hot = uniform(seed ^ 0x5151, 1, domain)[0]
        pct = uniform(seed ^ 0xABAB, n, 99)
        v = np.where(pct < 90, hot, v).astype(np.uint32)
    return v


def random_rows(seed: int, n: int, arity: int, domain: int) -> np.ndarray:
    return uniform(seed, n * arity, domain).reshape(n, arity)


def path_graph(nodes: int) -> np.ndarray:
    i = np.arange(max(nodes - 1, 0), dtype=np.uint32)
    return np.stack([i, i + 1], axis=1)


def cycle_graph(nodes: int) -> np.ndarray:
    i = np.arange(nodes, dtype=np.uint32)
    return np.stack([i, (i + 1) % nodes], axis=1).astype(np.uint32)


def binary_tree(depth: int, base: int = 0) -> np.ndarray:
    """support.hpp:80-86: heap-numbered parent->child edges (nodes from 1)."""
    nodes = (1 << (depth + 1)) - 1
    child = np.arange(2, nodes + 1, dtype=np.uint64)
    return np.stack([child // 2 + base, child + base], axis=1).astype(np.uint32)


# ---- workload graphs ---------------------------------------------------------------


def _distinct_pairs(src: np.ndarray, dst: np.ndarray, m: int) -> np.ndarray:
    """First m distinct (src, dst) pairs with src != dst, in generation order."""
    keep = src != dst
    src, dst = src[keep], dst[keep]
    key = src.astype(np.uint64) << np.uint64(32) | dst.astype(np.uint64)
    _, first = np.unique(key, return_index=True)
    first.sort()
    first = first[:m]
    return np.stack([src[first], dst[first]], axis=1).astype(np.uint32)


def tc_uniform(nodes: int, edges: int, seed: int = 1) -> np.ndarray:
    """C1: `edges` distinct uniform (u, v), u != v, over `nodes` nodes."""
    got = np.zeros((0, 2), np.uint32)
    draw = int(edges * 1.2) + 64
    offset = 0
    while got.shape[0] < edges:
        r = uniform(seed, 2 * draw, nodes - 1, offset)
        offset += 2 * draw
        cand = np.concatenate([got, r.reshape(-1, 2)])
        got = _distinct_pairs(cand[:, 0], cand[:, 1], edges)
        draw *= 2
    return got


def tc_powerlaw(components: int = 1000, nodes: int = 1000, edges: int = 5000, seed: int = 1,
                alpha: float = 1.0, first: int = 0) -> np.ndarray:
    """C2: `components` disjoint blocks of `nodes` nodes with `edges` distinct
    edges each; sources Zipf(alpha) over a per-block node permutation,
    targets uniform (no giant SCC, |TC| ~ components * 0.65 C^2).
    `first` generates blocks first .. first + components - 1 of the same
    sequence (a slice of a larger graph)."""
    w = 1.0 / np.arange(1, nodes + 1, dtype=np.float64) ** alpha
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    out = []
    for c in range(first, first + components):
        s = seed * 1_000_003 + c
        perm = np.argsort(splitmix64(s ^ 0x7777, nodes), kind="stable").astype(np.uint32)
        draw = edges * 3
        u = unit(s, draw)
        src = perm[np.minimum(np.searchsorted(cdf, u, side="right"), nodes - 1)]
        dst = uniform(s ^ 0x3333, draw, nodes - 1)
        e = _distinct_pairs(src, dst, edges)
        if e.shape[0] < edges:
            raise RuntimeError("tc_powerlaw: not enough distinct edges; raise draw")
        out.append(e + np.uint32(c * nodes))
    return np.concatenate(out) if out else np.zeros((0, 2), np.uint32)


def sg_forest(trees: int, depth: int) -> np.ndarray:
    """C3: forest of complete binary trees (node ids disjoint per tree)."""
    per = (1 << (depth + 1))  # ids 1..2^(d+1)-1 used per tree
    return np.concatenate([binary_tree(depth, base=t * per) for t in range(trees)])


def sg_count(trees: int, depth: int) -> int:
    """Closed form |SG| of the forest."""
    return trees * ((4 ** (depth + 1) - 4) // 3 - (2 ** (depth + 1) - 2))


def cspa_facts(components: int, vars_per: int, assign_per: int, deref_per: int,
               seed: int = 3) -> Dict[str, np.ndarray]:
    """C4: K disjoint 'functions' of C variables; assign(y, x) and
    dereference(y, x) uniform inside each component."""
    a, d = [], []
    for c in range(components):
        s = seed * 7919 + c
        base = np.uint32(c * vars_per)
        ra = uniform(s, 2 * assign_per, vars_per - 1).reshape(-1, 2) + base
        rd = uniform(s ^ 0x9999, 2 * deref_per, vars_per - 1).reshape(-1, 2) + base
        a.append(ra)
        d.append(rd)
    return {"assign": np.concatenate(a).astype(np.uint32),
            "dereference": np.concatenate(d).astype(np.uint32)}


# ---- programs -------------------------------------------------------------------------

TC_PROGRAM = "reach(x, y) :- edge(x, y).\nreach(x, z) :- edge(x, y), reach(y, z).\n"
SG_PROGRAM = ("sg(x, y) :- edge(p, x), edge(p, y), x != y.\n"
              "sg(x, y) :- edge(a, x), sg(a, b), edge(b, y), x != y.\n")
CSPA_PROGRAM = """valueFlow(y, x) :- assign(y, x).
valueFlow(x, y) :- assign(x, z), memoryAlias(z, y).
valueFlow(x, y) :- valueFlow(x, z), valueFlow(z, y).
memoryAlias(x, w) :- dereference(y, x), valueAlias(y, z), dereference(z, w).
valueAlias(x, y) :- valueFlow(z, x), valueFlow(z, y).
valueAlias(x, y) :- valueFlow(z, x), memoryAlias(z, w), valueFlow(w, y).
valueFlow(x, x) :- assign(x, y).
valueFlow(x, x) :- assign(y, x).
memoryAlias(x, x) :- assign(y, x).
memoryAlias(x, x) :- assign(x, y).
"""
LUBM_PROGRAM = """professor(x) :- fullprofessor(x).
professor(x) :- associateprofessor(x).
professor(x) :- assistantprofessor(x).
faculty(x) :- professor(x).
faculty(x) :- lecturer(x).
employee(x) :- faculty(x).
person(x) :- employee(x).
student(x) :- undergraduatestudent(x).
student(x) :- graduatestudent(x).
person(x) :- student(x).
organization(x) :- university(x).
organization(x) :- department(x).
organization(x) :- researchgroup(x).
course(x) :- graduatecourse(x).
worksfor(x, y) :- headof(x, y).
memberof(x, y) :- worksfor(x, y).
degreefrom(x, y) :- undergraduatedegreefrom(x, y).
degreefrom(x, y) :- mastersdegreefrom(x, y).
degreefrom(x, y) :- doctoraldegreefrom(x, y).
member(y, x) :- memberof(x, y).
memberof(x, y) :- member(y, x).
hasalumnus(y, x) :- degreefrom(x, y).
degreefrom(x, y) :- hasalumnus(y, x).
suborganizationof(x, z) :- suborganizationof(x, y), suborganizationof(y, z).
person(x) :- advisor(x, y).
professor(y) :- advisor(x, y).
faculty(x) :- teacherof(x, y).
course(y) :- teacherof(x, y).
organization(y) :- memberof(x, y).
organization(x) :- suborganizationof(x, y).
organization(y) :- suborganizationof(x, y).
university(y) :- degreefrom(x, y).
person(x) :- degreefrom(x, y).
publication(x) :- publicationauthor(x, y).
person(y) :- publicationauthor(x, y).
chair(x) :- person(x), headof(x, y), department(y).
employee(x) :- person(x), worksfor(x, y), organization(y).
student(x) :- person(x), takescourse(x, y), course(y).
teachingassistant(x) :- person(x), teachingassistantof(x, y), course(y).
"""

LUBM_UNARY = ["fullprofessor", "associateprofessor", "assistantprofessor", "lecturer",
              "undergraduatestudent", "graduatestudent", "university", "department",
              "researchgroup", "graduatecourse"]
LUBM_BINARY = ["headof", "worksfor", "undergraduatedegreefrom", "mastersdegreefrom",
               "doctoraldegreefrom", "suborganizationof", "advisor", "teacherof",
               "publicationauthor", "takescourse", "teachingassistantof"]


def lubm_facts(scale: int, seed: int = 5) -> Dict[str, np.ndarray]:
    """C5 (UBA-like, vertically partitioned): `scale` universities, each with
    departments, research groups, faculty, students, courses, publications.
    Entity ids are dense and disjoint per class."""
    rng_off = [0]

    def draw(n, hi):
        r = uniform(seed, n, hi, rng_off[0])
        rng_off[0] += n
        return r

    U = scale
    D = U * 15
    G = D * 10
    FP, AP, SP, LE = D * 8, D * 10, D * 8, D * 6
    UG, GS = D * 300, D * 60
    C, GC = D * 40, D * 20
    PUB = D * 200
    ids = {}
    nxt = 0
    for name, cnt in [("university", U), ("department", D), ("researchgroup", G),
                      ("fullprofessor", FP), ("associateprofessor", AP),
                      ("assistantprofessor", SP), ("lecturer", LE),
                      ("undergraduatestudent", UG), ("graduatestudent", GS),
                      ("course", C), ("graduatecourse", GC), ("publication", PUB)]:
        ids[name] = np.arange(nxt, nxt + cnt, dtype=np.uint32)
        nxt += cnt
    uni, dept, grp = ids["university"], ids["department"], ids["researchgroup"]
    fac = np.concatenate([ids["fullprofessor"], ids["associateprofessor"],
                          ids["assistantprofessor"], ids["lecturer"]])
    prof = np.concatenate([ids["fullprofessor"], ids["associateprofessor"],
                           ids["assistantprofessor"]])
    ug, gs = ids["undergraduatestudent"], ids["graduatestudent"]
    courses = np.concatenate([ids["course"], ids["graduatecourse"]])
    pubs = ids["publication"]

    def pairs(a, b):
        return np.stack([a.astype(np.uint32), b.astype(np.uint32)], axis=1)

    f: Dict[str, np.ndarray] = {k: ids[k].reshape(-1, 1) for k in LUBM_UNARY}
    f["headof"] = pairs(ids["fullprofessor"][:D], dept)
    f["worksfor"] = pairs(fac, dept[draw(fac.size, D - 1)])
    f["suborganizationof"] = np.concatenate([pairs(dept, uni[np.arange(D) // 15]),
                                             pairs(grp, dept[np.arange(G) // 10])])
    f["undergraduatedegreefrom"] = pairs(fac, uni[draw(fac.size, U - 1)])
    f["mastersdegreefrom"] = pairs(prof, uni[draw(prof.size, U - 1)])
    f["doctoraldegreefrom"] = pairs(prof, uni[draw(prof.size, U - 1)])
    f["advisor"] = pairs(gs, prof[draw(gs.size, prof.size - 1)])
    f["teacherof"] = pairs(fac[draw(courses.size, fac.size - 1)], courses)
    f["publicationauthor"] = pairs(pubs, prof[draw(pubs.size, prof.size - 1)])
    students = np.concatenate([ug, gs])
    f["takescourse"] = pairs(np.repeat(students, 3), courses[draw(students.size * 3, courses.size - 1)])
    f["teachingassistantof"] = pairs(gs[: C], ids["course"])
    return f


def write_tsv_dir(path: str, facts: Dict[str, np.ndarray]) -> None:
    """<dir>/<rel>.tsv, the reference's facts layout (P/src/io.cpp:44-88)."""
    os.makedirs(path, exist_ok=True)
    for rel, rows in facts.items():
        rows = np.asarray(rows, dtype=np.uint32)
        if rows.ndim == 1:
            rows = rows.reshape(-1, 1)
        with open(os.path.join(path, rel + ".tsv"), "w") as fh:
            if rows.shape[0]:
                np.savetxt(fh, rows, fmt="%d", delimiter="\t")

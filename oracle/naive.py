"""TEST INFRASTRUCTURE — ORACLE, NOT PRODUCT (see oracle/__init__.py).

Pure-Python restatement of the reference's naive least-model evaluator
(P/src/oracle.cpp:19-89): nested-loop matching of all body atoms with
constant, repeated-variable and guard checks, repeated full immediate
consequence until nothing changes. Shares nothing with the engine but the
program text; small inputs only.

Programs are given as ASTs of plain tuples (see parse_rules) so this file
needs no frontend: rules are written ("head", [args]), [("rel", [args])...],
[("x", "y") guards]; args are variable names (str) or ints.
"""
from __future__ import annotations

import re
from typing import Dict, List, Set, Tuple

Row = Tuple[int, ...]

_ATOM = re.compile(r"\s*([a-z][A-Za-z0-9_]*)\s*\(([^)]*)\)\s*")


def parse_rules(text: str):
    """Minimal parser for the dialect subset used in tests (no strings):
    returns (facts, rules)."""
    facts, rules = [], []
    src = re.sub(r"(%|//)[^\n]*", "", text)
    for clause in [c.strip() for c in src.split(".") if c.strip()]:
        if ":-" in clause:
            head_s, body_s = clause.split(":-", 1)
            head = _atom(head_s)
            body, guards = [], []
            for item in _split_items(body_s):
                if "!=" in item:
                    a, b = [x.strip() for x in item.split("!=")]
                    guards.append((a, b))
                else:
                    body.append(_atom(item))
            rules.append((head, body, guards))
        else:
            facts.append(_atom(clause))
    return facts, rules


def _split_items(s: str) -> List[str]:
    out, depth, cur = [], 0, ""
    for ch in s:
        if ch == "(":
            depth += 1
        elif ch == ")":
            depth -= 1
        if ch == "," and depth == 0:
            out.append(cur)
            cur = ""
        else:
            cur += ch
    if cur.strip():
        out.append(cur)
    return [x.strip() for x in out]


def _atom(s: str):
    m = _ATOM.fullmatch(s)
    if not m:
        raise ValueError(f"bad atom {s!r}")
    args = []
    for a in m.group(2).split(","):
        a = a.strip()
        args.append(int(a) if a.isdigit() else a)
    return (m.group(1), args)


def single_step(rule, rows: Dict[str, Set[Row]]) -> Set[Row]:
    """oracle::single_step (P/src/oracle.cpp:65-70)."""
    head, body, guards = rule
    out: Set[Row] = set()

    def search(depth: int, env: Dict[str, int]):
        if depth == len(body):
            for a, b in guards:
                if env[a] == env[b]:
                    return
            out.add(tuple(env[t] if isinstance(t, str) else t for t in head[1]))
            return
        rel, args = body[depth]
        for row in rows.get(rel, ()):
            if len(row) != len(args):
                continue
            bound_here = []
            ok = True
            for t, v in zip(args, row):
                if isinstance(t, int):
                    if v != t:
                        ok = False
                        break
                elif t in env:
                    if env[t] != v:
                        ok = False
                        break
                else:
                    env[t] = v
                    bound_here.append(t)
            if ok:
                search(depth + 1, env)
            for t in bound_here:
                del env[t]

    search(0, {})
    return out


def naive_evaluate(text: str, edb: Dict[str, List[Row]]) -> Dict[str, Set[Row]]:
    """oracle::naive_evaluate (P/src/oracle.cpp:72-89)."""
    facts, rules = parse_rules(text)
    rows: Dict[str, Set[Row]] = {}
    for rel, args in facts:
        rows.setdefault(rel, set()).add(tuple(args))
    for head, body, _ in rules:
        rows.setdefault(head[0], set())
        for a in body:
            rows.setdefault(a[0], set())
    for rel, tuples in edb.items():
        rows.setdefault(rel, set()).update(tuple(int(x) for x in r) for r in tuples)
    changed = True
    while changed:
        changed = False
        for rule in rules:
            derived = single_step(rule, rows)
            target = rows.setdefault(rule[0][0], set())
            before = len(target)
            target |= derived
            changed |= len(target) != before
    return rows

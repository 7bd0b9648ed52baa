"""Random programs in the supported fragment, restating the reference's
generator (P/tests/engine_test.cpp:33-116) on a portable PRNG, with the
empty-`bound` dereference (engine_test.cpp:72/83) fixed: a disconnected atom
is left as is (the program then fails validation and is skipped) and a rule
whose body binds no variable gets no head."""
from __future__ import annotations

from typing import Dict, List, Optional, Tuple

import numpy as np

from paper_2501_13051_b200 import workloads as W


class Rng:
    def __init__(self, seed: int):
        self.seed, self.i = seed, 0

    def randint(self, lo: int, hi: int) -> int:
        v = int(W.splitmix64(self.seed, 1, self.i)[0] % np.uint64(hi - lo + 1)) + lo
        self.i += 1
        return v


VARS = ["v0", "v1", "v2", "v3", "v4", "v5"]


def random_rule(g: Rng, rels: List[Tuple[str, int]], idb: List[str]) -> Optional[str]:
    bound: List[str] = []
    body = []
    for b in range(g.randint(1, 3)):
        name, arity = rels[g.randint(0, len(rels) - 1)]
        args: List[str] = []
        shares = b == 0
        for c in range(arity):
            roll = g.randint(0, 9)
            if roll == 0:
                args.append(str(g.randint(0, 7)))
            elif bound and (roll < 6 or (not shares and c + 1 == arity)):
                args.append(bound[g.randint(0, len(bound) - 1)])
                shares = True
            else:
                v = VARS[g.randint(0, 5)]
                args.append(v)
                if b == 0 or v in bound:
                    shares = True
        if not shares and bound:
            args[0] = bound[0]
        for t in args:
            if not t.isdigit() and t not in bound:
                bound.append(t)
        body.append(f"{name}({', '.join(args)})")
    if not bound:
        return None
    hname, harity = [r for r in rels if r[0] in idb][g.randint(0, len(idb) - 1)]
    head = [bound[g.randint(0, len(bound) - 1)] for _ in range(harity)]
    items = list(body)
    if len(bound) >= 2 and g.randint(0, 2) == 0 and bound[0] != bound[-1]:
        items.append(f"{bound[0]} != {bound[-1]}")
    return f"{hname}({', '.join(head)}) :- {', '.join(items)}."


def random_program(g: Rng):
    rels = [("e0", 2), ("e1", g.randint(1, 3)), ("i0", 2), ("i1", g.randint(1, 2))]
    idb = ["i0", "i1"]
    rules = []
    for _ in range(g.randint(1, 4)):
        r = random_rule(g, rels, idb)
        if r:
            rules.append(r)
    return "\n".join(rules) + "\n", dict(rels)


def random_edb(g: Rng, arities: Dict[str, int], max_rows: int) -> Dict[str, np.ndarray]:
    edb = {}
    for rel, a in arities.items():
        if not rel.startswith("e"):
            continue
        n = g.randint(0, max_rows)
        edb[rel] = np.array([[g.randint(0, 7) for _ in range(a)] for _ in range(n)], np.uint32).reshape(n, a)
    return edb

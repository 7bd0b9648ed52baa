"""Rebuild the inputs of tests/golden/engine.json cases (shared by tests)."""
import numpy as np

from paper_2501_13051_b200 import workloads as W

PROGRAMS = {"TC": W.TC_PROGRAM, "SG": W.SG_PROGRAM, "CSPA": W.CSPA_PROGRAM, "LUBM": W.LUBM_PROGRAM}


def program_and_facts(case):
    text = PROGRAMS.get(case["program"], case["program"])
    facts = {}
    for rel, g in case["facts"].items():
        if rel == "cspa":
            facts.update(W.cspa_facts(*g))
            continue
        if rel == "lubm":
            facts.update(W.lubm_facts(*g))
            continue
        kind, args = g[0], g[1:]
        if kind == "rows":
            facts[rel] = np.asarray(args[0], np.uint32)
        else:
            facts[rel] = getattr(W, kind)(*args)
    return text, facts

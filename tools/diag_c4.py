import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2501_13051_b200 import colog, engine as E, workloads as W
ctx = colog.Context(0)
f = W.cspa_facts(4000, 100, 100, 70)
for rep in range(2):
    t = time.time()
    st = E.evaluate_program(W.CSPA_PROGRAM, f, ctx=ctx)
    print("rep", rep, "wall %.1f ms" % (1000 * (time.time() - t)), flush=True)
    del st

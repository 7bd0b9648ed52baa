"""Diagnostic: repeated fixpoints of one BASELINE workload (C1..C5) with the
engine trace on (FVLOG_TRACE=1 prints per-iteration phase times, host syncs,
join sizes and word builds). Not a benchmark.
    python tools/diag_wl.py C5 [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_13051_b200 import colog, engine as E  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_workloads import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = colog.Context(0)
facts = cfg["facts"]()
for rep in range(reps):
    t = time.time()
    st = E.evaluate_program(cfg["program"], facts, ctx=ctx)
    print("rep", rep, "wall %.1f ms" % (1000 * (time.time() - t)), "syncs", ctx.host_syncs(), flush=True)
    del st

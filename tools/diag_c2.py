"""Diagnostic: repeated C2 fixpoints with the engine trace (FVLOG_TRACE=1
prints per-iteration host phase times and pool state). Not a benchmark."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_13051_b200 import colog, engine as E, workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = colog.Context(0)
e = W.tc_powerlaw(1000, 1000, 5000, 1)
keep = None
for rep in range(reps):
    t = time.time()
    st = E.evaluate_program(W.TC_PROGRAM, {"edge": e}, ctx=ctx)
    dt = time.time() - t
    print("rep", rep, "wall %.1f ms" % (1000 * dt), "engine %.1f ms" % st.elapsed_ms, "rows", st.rows("reach"),
          flush=True)
    keep = st if os.environ.get("DIAG_KEEP") else None
    del st

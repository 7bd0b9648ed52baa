"""The partitioned engine's work on one GPU: C2 evaluated
with `world` virtual ranks and the in-process transport
(fv_evaluate_program_sharded — the multi-GPU code path, ranks run one after
concurrently on the same device, one thread and stream each, every call
creating fresh per-rank contexts and memory pools). Reports wall seconds and
checks the global stats against C2's golden; run it under an ncu
launch list for per-kernel times (route, exchange-side insert, fused join).
The exchange is a device-to-device copy here, not NVLink.

    python tools/bench_sharded.py [--worlds 2,4,8] [--out f.json]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_13051_b200 import _lib, colog, engine as E, workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out")
    args = ap.parse_args()
    ctx = colog.Context(0)
    _lib.bind("fv_ctx_reserve", C.c_int, [C.c_void_p, C.c_uint64])
    _lib.check(ctx._lib.fv_ctx_reserve(ctx.h, 96 << 30), ctx.h)
    edges = W.tc_powerlaw(1000, 1000, 5000, 1)
    facts = {"edge": edges}
    # The check: C2's pinned per-iteration deltas and row count
    # (tests/golden/large.json), so no single-GPU run is needed here.
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "large.json")))["C2"]
    want = {"edge": None, "reach": g["deltas"]}
    n_single = g["rows"]
    out = {}
    for world in [int(w) for w in args.worlds.split(",")]:
        best = None
        for rep in range(max(args.reps, 1)):
            ctx.synchronize()
            t = time.perf_counter()
            shards = E.evaluate_program_sharded(W.TC_PROGRAM, facts, world, ctx=ctx)
            ctx.synchronize()
            dt = time.perf_counter() - t
            ok = shards[0].delta_counts()["reach"] == want["reach"] and sum(s.rows("reach") for s in shards) == n_single
            del shards
            assert ok, f"world {world}: global stats differ from the single-GPU run"
            best = dt if best is None or dt < best else best
        out[f"world{world}"] = {"seconds_all_ranks": round(best, 4), "identical_stats": True}
        print(json.dumps({f"world{world}": out[f"world{world}"]}), flush=True)
    if args.out:
        json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

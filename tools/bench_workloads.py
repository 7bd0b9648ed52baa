"""Seconds to fixpoint and derived tuples/s for every BASELINE config
(C1 TC uniform, C2 TC power-law, C3 SG, C4 CSPA, C5 OWL-RL/LUBM) on one GPU,
each checked against its full-size golden (tests/golden/large.json), with
the unmodified CPU reference (oracle/_ref/colog_ref, all host cores) timed on
a bounded sample of the same generator — and the GPU on that same sample, so
the speed-up is quoted on identical inputs. bench.py's single JSON line is
the C2 headline; this is the per-workload table (profiles/<round>/workloads.json).

Timing: wall clock around fv_evaluate_program with pinned host SoA facts
(EDB upload + seed + fixpoint, the reference's evaluate() span,
P/src/runner.cpp:58-61, whose facts are likewise already in memory); the
call synchronises the device before returning. Median of --steps runs
after --warmup runs. The memory pool is reserved once up front.

    python tools/bench_workloads.py [--configs C1,C2,C3,C4,C5] [--steps 3] [--warmup 1] [--out f.json]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_13051_b200 import _lib, colog, engine as E, workloads as W  # noqa: E402

CONFIGS = {
    "C1": dict(name="TC uniform 10k nodes / 50k edges", program=W.TC_PROGRAM,
               facts=lambda: {"edge": W.tc_uniform(10_000, 50_000, 1)},
               sample=lambda: {"edge": W.tc_uniform(2_000, 10_000, 1)}, sample_desc="tc_uniform(2000, 10000, 1)"),
    "C2": dict(name="TC power-law 1000 x (1000 nodes, 5000 edges)", program=W.TC_PROGRAM,
               facts=lambda: {"edge": W.tc_powerlaw(1000, 1000, 5000, 1)},
               sample=lambda: {"edge": W.tc_powerlaw(1000, 1000, 5000, 1)[:30 * 5000]},
               sample_desc="first 30 of the 1000 components"),
    "C3": dict(name="SG forest of 244 complete binary trees, depth 10 (499,224 edges)", program=W.SG_PROGRAM,
               facts=lambda: {"edge": W.sg_forest(244, 10)},
               sample=lambda: {"edge": W.sg_forest(8, 10)}, sample_desc="sg_forest(8, 10)"),
    "C4": dict(name="CSPA 4000 functions x 100 vars (400k assign / 280k dereference)", program=W.CSPA_PROGRAM,
               facts=lambda: W.cspa_facts(4000, 100, 100, 70),
               sample=lambda: {k: v[: 20 * (100 if k == "assign" else 70)]
                               for k, v in W.cspa_facts(4000, 100, 100, 70).items()},
               sample_desc="first 20 of the 4000 functions"),
    "C5": dict(name="OWL-RL/LUBM 39 rules on lubm_facts(340) (10.15 M facts)", program=W.LUBM_PROGRAM,
               facts=lambda: W.lubm_facts(340), sample=lambda: W.lubm_facts(34),
               sample_desc="lubm_facts(34) (1/10 scale)"),
}


def pinned_soa(facts, arities):
    """Host facts as pinned SoA columns (the layout fv_facts takes), built
    once outside the timed region — like the reference's in-memory FactMap."""
    import torch
    out = {}
    for rel, rows in facts.items():
        if rel not in arities:
            continue
        r = np.asarray(rows, dtype=np.uint32).reshape(-1, arities[rel])
        cols = []
        for j in range(r.shape[1]):
            t = torch.empty(r.shape[0], dtype=torch.int32, pin_memory=True)
            t.numpy().view(np.uint32)[:] = r[:, j]
            cols.append(t)
        out[rel] = cols
    return out


def gpu_run(ctx, program, facts, steps, warmup):
    """Median wall time of fv_evaluate_program on pinned host facts (EDB
    upload + seed + fixpoint; the call returns after the device finished)."""
    prog = E.compile_program(program)
    arities = dict(prog.relations())
    soa = pinned_soa(facts, arities)
    keep, blocks = [], []
    for rel, cols in soa.items():
        ptrs = (C.POINTER(C.c_uint32) * len(cols))(*[C.cast(t.data_ptr(), C.POINTER(C.c_uint32)) for t in cols])
        name = rel.encode()
        keep += [ptrs, name]
        blocks.append(E.fv_facts(name, len(cols), cols[0].shape[0], ptrs))
    arr = (E.fv_facts * max(len(blocks), 1))(*blocks)
    times, st = [], None
    for i in range(warmup + steps):
        if st is not None:
            del st
        h = C.c_void_p()
        t = time.perf_counter()
        _lib.check(ctx._lib.fv_evaluate_program(ctx.h, prog.h, arr, len(blocks), C.byref(h)), ctx.h)
        dt = time.perf_counter() - t
        st = E.State(ctx, h.value)
        if i >= warmup:
            times.append(dt)
    return st, statistics.median(times), times


def reference_run(program, facts):
    ref = os.path.join(ROOT, "oracle", "_ref", "colog_ref")
    if not os.path.exists(ref):
        return None
    cores = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as d:
        W.write_tsv_dir(os.path.join(d, "facts"), facts)
        p = os.path.join(d, "p.dl")
        open(p, "w").write(program)
        r = subprocess.run([ref, "run", p, "--facts", os.path.join(d, "facts"), "--out", os.path.join(d, "out"),
                            "--workers", str(cores), "--stats"], capture_output=True, text=True, check=True)
    deltas = 0
    total_ms = None
    for l in r.stdout.splitlines():
        f = dict(kv.split("=", 1) for kv in l.split())
        if l.startswith("iter="):
            deltas += int(f["delta"])
        elif l.startswith("iterations="):
            total_ms = float(f["total_ms"])
    return {"derived_tuples": deltas, "seconds": total_ms / 1000.0, "cores": cores,
            "tuples_per_s": deltas / (total_ms / 1000.0), "kind": "reference (oracle/_ref, OpenMP shim)"}


def parity(key, st, golden):
    g = golden.get(key)
    if not g:
        return "no golden"
    if "relations" in g:
        ok = all(st.rows(r) == v["rows"] and str(st.fingerprint(r)) == v["fingerprint"]
                 for r, v in g["relations"].items())
    else:
        rel = "sg" if key == "C3" else "reach"
        ok = st.rows(rel) == g["rows"] and ("fingerprint" not in g or str(st.fingerprint(rel)) == g["fingerprint"])
    ok = ok and st.iterations == g["iterations"]
    return ("identical to " + g["source"]) if ok else "MISMATCH vs " + g["source"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--no-reference", action="store_true")
    ap.add_argument("--reserve-gb", type=float, default=96.0)
    ap.add_argument("--out")
    args = ap.parse_args()
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "large.json")))
    ctx = colog.Context(0)
    _lib.bind("fv_ctx_reserve", C.c_int, [C.c_void_p, C.c_uint64])
    _lib.check(ctx._lib.fv_ctx_reserve(ctx.h, int(args.reserve_gb * 2**30)), ctx.h)
    results = {}
    for key in args.configs.split(","):
        cfg = CONFIGS[key]
        facts = cfg["facts"]()
        st, med, times = gpu_run(ctx, cfg["program"], facts, args.steps, args.warmup)
        derived = st.derived_tuples()
        res = {"workload": cfg["name"], "edb_facts": int(sum(v.shape[0] for v in facts.values())),
               "derived_tuples": derived, "iterations": st.iterations,
               "idb_rows": {r: n for r, (a, n) in st.relations().items()},
               "seconds_to_fixpoint": med, "runs_s": [round(t, 5) for t in times],
               "tuples_per_s": derived / med, "parity": parity(key, st, golden)}
        del st
        if not args.no_reference:
            sample = cfg["sample"]()
            ref = reference_run(cfg["program"], sample)
            st2, med2, _ = gpu_run(ctx, cfg["program"], sample, args.steps, args.warmup)
            res["sample"] = {"what": cfg["sample_desc"], "reference": ref,
                             "gpu": {"derived_tuples": st2.derived_tuples(), "seconds": med2,
                                     "tuples_per_s": st2.derived_tuples() / med2},
                             "speedup_same_input": (ref["seconds"] / med2) if ref else None}
            if ref:
                assert st2.derived_tuples() == ref["derived_tuples"], (key, "sample derived tuples differ")
            del st2
        results[key] = res
        print(json.dumps({key: res}), flush=True)
    if args.out:
        json.dump(results, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

"""Facts loading + dump formatting outside evaluate():
the fvlog CLI (integer facts parsed and dumps formatted on the device) and
the unmodified reference CLI (oracle/_ref/colog_ref, all host cores) on the
same files.
  reference io_s = process wall - total_ms (its evaluate() span): program
                   parse + facts load + dump write (+ a few ms of start-up)
  fvlog io_s     = the runner's own parse + load + dump phases (FVLOG_TRACE),
                   i.e. the same work; process_s is the whole process, which
                   also pays CUDA context creation and teardown (~2 s, fixed).

Each side: one warm-up run, then the median of 3 runs.

    python tools/bench_io.py [--out f.json]
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_13051_b200 import workloads as W  # noqa: E402

CLI = os.path.join(ROOT, "paper_2501_13051_b200", "fvlog")
REF = os.path.join(ROOT, "oracle", "_ref", "colog_ref")

CASES = [
    ("C5 LUBM lubm_facts(340), dump 4 largest IDB", W.LUBM_PROGRAM, lambda: W.lubm_facts(340),
     ["person", "student", "course", "hasalumnus"]),
    ("TC tc_uniform(2000, 10000), dump reach", W.TC_PROGRAM, lambda: {"edge": W.tc_uniform(2000, 10000, 1)},
     ["reach"]),
]


def run(binary, prog, facts, out, dump):
    args = [binary, "run", prog, "--facts", facts, "--out", out, "--dump", ",".join(dump)]
    if binary == REF:
        args += ["--workers", str(os.cpu_count() or 1)]
    t = time.perf_counter()
    r = subprocess.run(args, capture_output=True, text=True, check=True, env=dict(os.environ, FVLOG_TRACE="1"))
    wall = time.perf_counter() - t
    total_ms = float([l for l in r.stdout.splitlines() if l.startswith("iterations=")][0].split()[1].split("=")[1])
    phases = {}
    for l in r.stderr.splitlines():
        if l.startswith("[fvlog] run "):
            f = l.split()
            phases[" ".join(f[2:-2])] = phases.get(" ".join(f[2:-2]), 0.0) + float(f[-2]) / 1000.0
    return wall, total_ms / 1000.0, phases


def dir_bytes(d):
    return sum(os.path.getsize(os.path.join(d, f)) for f in os.listdir(d))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    args = ap.parse_args()
    res = {}
    for name, program, facts_fn, dump in CASES:
        with tempfile.TemporaryDirectory() as d:
            prog = os.path.join(d, "p.dl")
            open(prog, "w").write(program)
            facts = os.path.join(d, "facts")
            W.write_tsv_dir(facts, facts_fn())
            row = {"facts_bytes": dir_bytes(facts)}
            for label, binary in (("fvlog", CLI), ("reference", REF)):
                out = os.path.join(d, label)
                run(binary, prog, facts, out, dump)  # warm (page cache, driver)
                # median of 3 process runs (by wall time)
                wall, evaluate_s, phases = sorted((run(binary, prog, facts, out, dump) for _ in range(3)),
                                                  key=lambda r: r[0])[1]
                if label == "fvlog":
                    io = sum(v for k, v in phases.items() if k in ("parse", "load facts", "dump"))
                    row[label] = {"process_s": round(wall, 3), "evaluate_s": round(evaluate_s, 4),
                                  "io_s": round(io, 4), "phases_s": {k: round(v, 4) for k, v in phases.items()}}
                else:
                    row[label] = {"process_s": round(wall, 3), "evaluate_s": round(evaluate_s, 4),
                                  "io_s": round(wall - evaluate_s, 3)}
            row["dump_bytes"] = dir_bytes(os.path.join(d, "fvlog"))
            same = all(open(os.path.join(d, "fvlog", r + ".tsv"), "rb").read() ==
                       open(os.path.join(d, "reference", r + ".tsv"), "rb").read() for r in dump)
            row["dumps_identical"] = same
            row["io_speedup"] = round(row["reference"]["io_s"] / row["fvlog"]["io_s"], 1)
        res[name] = row
        print(json.dumps({name: row}), flush=True)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

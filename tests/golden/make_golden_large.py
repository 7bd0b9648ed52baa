"""Full-size golden values for the BASELINE configs (size-independent checks).

  C1  TC, uniform 10k nodes / 50k edges: the UNMODIFIED reference
      (oracle/_ref/colog_ref, all cores) -> |reach|, per-iteration deltas,
      order-independent fingerprint of the sorted dump.
  C2  TC, 1000 disjoint Zipf components x (1000 nodes, 5000 edges): the
      UNMODIFIED reference on 100 batches of 10 disjoint components (rows,
      fingerprints and per-iteration deltas add), witnessed by an independent
      per-component distance-layer closure with dense matrix products (the
      semi-naive delta of iteration k is the set of pairs at shortest-path
      distance k+1).
  C3  SG forest of 244 depth-10 trees: the UNMODIFIED reference on batches of
      disjoint trees (rows also checked against the closed form).
  C4  CSPA on K disjoint functions (cspa_facts(K, 100, 100, 70)): the
      UNMODIFIED reference run on batches of components (components are
      disjoint, so the fixpoint is the union of the per-batch fixpoints:
      rows, fingerprints and per-iteration deltas add, iterations = max).
  C5  OWL-RL/LUBM rule set on lubm_facts(340) (~10.2 M facts): the
      UNMODIFIED reference on the whole input.

    python tests/golden/make_golden_large.py [c1] [c2] [c3] [c4] [c5]
Writes tests/golden/large.json (merging with what is already there).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2501_13051_b200 import workloads as W  # noqa: E402
from paper_2501_13051_b200.engine import fingerprint_rows  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "large.json")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "colog_ref")


def c1():
    edges = W.tc_uniform(10_000, 50_000, 1)
    with tempfile.TemporaryDirectory() as d:
        W.write_tsv_dir(os.path.join(d, "facts"), {"edge": edges})
        prog = os.path.join(d, "tc.dl")
        open(prog, "w").write(W.TC_PROGRAM)
        t0 = time.time()
        r = subprocess.run([REF_BIN, "run", prog, "--facts", os.path.join(d, "facts"), "--out",
                            os.path.join(d, "out"), "--stats", "--dump", "reach"],
                           capture_output=True, text=True, check=True,
                           env=dict(os.environ, OMP_WAIT_POLICY="passive"))
        wall = time.time() - t0
        deltas = [int(l.split()[2].split("=")[1]) for l in r.stdout.splitlines() if l.startswith("iter=")]
        summary = [l for l in r.stdout.splitlines() if l.startswith("iterations=")][0]
        import pandas as pd
        rows = pd.read_csv(os.path.join(d, "out", "reach.tsv"), sep="\t", header=None,
                           dtype=np.uint32).to_numpy()
    return {"config": "C1 tc_uniform(10000, 50000, 1)", "source": "unmodified reference (oracle/_ref)",
            "rows": int(rows.shape[0]), "fingerprint": str(fingerprint_rows(rows)),
            "deltas": deltas, "iterations": len(deltas), "reference_summary": summary,
            "reference_wall_s": round(wall, 1)}


def closure_layers(edges: np.ndarray, n: int):
    """Distance layers of the transitive closure of one component (n nodes)."""
    import torch
    a = torch.zeros((n, n), dtype=torch.float32)
    a[torch.as_tensor(edges[:, 0].astype(np.int64)), torch.as_tensor(edges[:, 1].astype(np.int64))] = 1.0
    reach = a > 0
    frontier = a.clone()
    layers = [int(reach.sum())]
    while True:
        nxt = (a @ frontier) > 0          # pairs (x, z): x -> y, (y, z) in frontier
        new = nxt & ~reach
        k = int(new.sum())
        layers.append(k)
        if k == 0:
            break
        reach |= new
        frontier = new.to(torch.float32)
    return reach, layers


def c2(components=1000, nodes=1000, edges=5000):
    import torch
    torch.set_num_threads(os.cpu_count() or 1)
    e = W.tc_powerlaw(components, nodes, edges, 1)
    total_rows, fp = 0, 0
    deltas: list = []
    for c in range(components):
        ce = e[c * edges:(c + 1) * edges] - np.uint32(c * nodes)
        reach, layers = closure_layers(ce, nodes)
        for i, k in enumerate(layers):
            if i >= len(deltas):
                deltas.append(0)
            deltas[i] += k
        xs, zs = np.nonzero(reach.numpy())
        rows = np.stack([xs + c * nodes, zs + c * nodes], axis=1).astype(np.uint64)
        total_rows += rows.shape[0]
        fp = (fp + fingerprint_rows(rows)) & 0xFFFFFFFFFFFFFFFF
    while len(deltas) > 1 and deltas[-1] == 0 and deltas[-2] == 0:
        deltas.pop()
    return {"config": f"C2 tc_powerlaw({components}, {nodes}, {edges}, 1)",
            "source": "per-component distance-layer closure (independent of the engine)",
            "rows": int(total_rows), "fingerprint": str(fp), "deltas": deltas, "iterations": len(deltas)}


def run_reference(program: str, facts: dict, workers: int, dump=True):
    """Unmodified reference on `facts`: (per-relation rows/fingerprint/deltas,
    iterations, total_ms)."""
    with tempfile.TemporaryDirectory() as d:
        W.write_tsv_dir(os.path.join(d, "facts"), facts)
        prog = os.path.join(d, "p.dl")
        open(prog, "w").write(program)
        import re
        rels = sorted(set(re.findall(r"([a-z][A-Za-z0-9_]*)\s*\(", program)))
        r = subprocess.run([REF_BIN, "run", prog, "--facts", os.path.join(d, "facts"), "--out",
                            os.path.join(d, "out"), "--workers", str(workers), "--stats"]
                           + (["--dump", ",".join(rels)] if dump else []),
                           capture_output=True, text=True, check=True,
                           env=dict(os.environ, OMP_WAIT_POLICY="passive"))
        out = {}
        for l in r.stdout.splitlines():
            f = dict(kv.split("=", 1) for kv in l.split())
            if l.startswith("iter="):
                out.setdefault(f["rel"], {"deltas": []})["deltas"].append(int(f["delta"]))
            elif l.startswith("rel="):
                out.setdefault(f["rel"], {"deltas": []})["rows"] = int(f["rows"])
            elif l.startswith("iterations="):
                iterations, total_ms = int(f["iterations"]), float(f["total_ms"])
        if dump:
            import pandas as pd
            for rel in rels:
                path = os.path.join(d, "out", rel + ".tsv")
                if os.path.getsize(path) == 0:
                    out[rel]["fingerprint"] = "0"
                    continue
                rows = pd.read_csv(path, sep="\t", header=None, dtype=np.uint32).to_numpy()
                out[rel]["fingerprint"] = str(fingerprint_rows(rows))
    return out, iterations, total_ms


C4_SHAPE = dict(components=4000, vars_per=100, assign_per=100, deref_per=70)


def _c4_batch(args):
    lo, hi = args
    K = C4_SHAPE["components"]
    f = W.cspa_facts(K, C4_SHAPE["vars_per"], C4_SHAPE["assign_per"], C4_SHAPE["deref_per"])
    a, dr = C4_SHAPE["assign_per"], C4_SHAPE["deref_per"]
    sub = {"assign": f["assign"][lo * a:hi * a], "dereference": f["dereference"][lo * dr:hi * dr]}
    return run_reference(W.CSPA_PROGRAM, sub, 1)


def c4(batch=10, procs=None):
    from multiprocessing import Pool
    K = C4_SHAPE["components"]
    jobs = [(lo, min(K, lo + batch)) for lo in range(0, K, batch)]
    total = {}
    iterations = 0
    ms = 0.0
    t0 = time.time()
    with Pool(procs or os.cpu_count()) as pool:
        for i, (rels, it, tms) in enumerate(pool.imap_unordered(_c4_batch, jobs)):
            iterations = max(iterations, it)
            ms += tms
            for rel, g in rels.items():
                t = total.setdefault(rel, {"rows": 0, "fingerprint": 0, "deltas": []})
                t["rows"] += g["rows"]
                t["fingerprint"] = (t["fingerprint"] + int(g["fingerprint"])) & 0xFFFFFFFFFFFFFFFF
                for k, dv in enumerate(g["deltas"]):
                    if k >= len(t["deltas"]):
                        t["deltas"].append(0)
                    t["deltas"][k] += dv
            if i % 50 == 0:
                print(f"C4 batch {i}/{len(jobs)} {time.time() - t0:.0f}s", flush=True)
    for t in total.values():
        t["fingerprint"] = str(t["fingerprint"])
        t["deltas"] += [0] * (iterations - len(t["deltas"]))
    return {"config": "C4 cspa_facts({components}, {vars_per}, {assign_per}, {deref_per}, seed=3)".format(**C4_SHAPE),
            "source": f"unmodified reference (oracle/_ref) on {len(jobs)} batches of {batch} disjoint components",
            "relations": total, "iterations": iterations, "reference_cpu_s_sum": round(ms / 1000.0, 1)}


def _merge_batches(results, total, relations):
    """Add per-batch reference results over disjoint components: rows,
    fingerprints and per-iteration deltas add, iterations = max."""
    iterations = 0
    ms = 0.0
    for rels, it, tms in results:
        iterations = max(iterations, it)
        ms += tms
        for rel in relations:
            g = rels[rel]
            t = total.setdefault(rel, {"rows": 0, "fingerprint": 0, "deltas": []})
            t["rows"] += g["rows"]
            t["fingerprint"] = (t["fingerprint"] + int(g["fingerprint"])) & 0xFFFFFFFFFFFFFFFF
            for k, dv in enumerate(g["deltas"]):
                if k >= len(t["deltas"]):
                    t["deltas"].append(0)
                t["deltas"][k] += dv
    for t in total.values():
        t["fingerprint"] = str(t["fingerprint"])
        t["deltas"] += [0] * (iterations - len(t["deltas"]))
    return iterations, ms


C2_SHAPE = dict(components=1000, nodes=1000, edges=5000)


def _c2_batch(args):
    lo, hi = args
    e = W.tc_powerlaw(hi - lo, C2_SHAPE["nodes"], C2_SHAPE["edges"], 1, first=lo)
    return run_reference(W.TC_PROGRAM, {"edge": e}, 1)


def c2_ref(batch=10, procs=None):
    """C2 from the UNMODIFIED reference, batch by batch over its disjoint
    components (tc_powerlaw(first=lo) generates exactly the slice lo..hi of
    the full graph; the reference's semi-naive Δ of iteration k on a union of
    disjoint components is the union of the per-component Δs)."""
    from multiprocessing import Pool
    K = C2_SHAPE["components"]
    jobs = [(lo, min(K, lo + batch)) for lo in range(0, K, batch)]
    results = []
    t0 = time.time()
    with Pool(procs or os.cpu_count()) as pool:
        for i, res in enumerate(pool.imap_unordered(_c2_batch, jobs)):
            results.append(res)
            if i % 10 == 0:
                print(f"C2 batch {i}/{len(jobs)} {time.time() - t0:.0f}s", flush=True)
    total = {}
    iterations, ms = _merge_batches(results, total, ["reach"])
    r = total["reach"]
    return {"config": "C2 tc_powerlaw({components}, {nodes}, {edges}, 1)".format(**C2_SHAPE),
            "source": f"unmodified reference (oracle/_ref) on {len(jobs)} batches of {batch} disjoint components",
            "rows": r["rows"], "fingerprint": r["fingerprint"], "deltas": r["deltas"],
            "iterations": iterations, "reference_cpu_s_sum": round(ms / 1000.0, 1),
            "reference_wall_s": round(time.time() - t0, 1)}


C3_SHAPE = dict(trees=244, depth=10)


def _c3_batch(args):
    lo, hi = args
    per = 1 << (C3_SHAPE["depth"] + 1)
    e = np.concatenate([W.binary_tree(C3_SHAPE["depth"], base=t * per) for t in range(lo, hi)])
    return run_reference(W.SG_PROGRAM, {"edge": e}, 1)


def c3_ref(batch=4, procs=None):
    """C3 from the UNMODIFIED reference on batches of the forest's disjoint
    trees (exactly sg_forest's node numbering), plus the closed form."""
    from multiprocessing import Pool
    K = C3_SHAPE["trees"]
    jobs = [(lo, min(K, lo + batch)) for lo in range(0, K, batch)]
    results = []
    t0 = time.time()
    with Pool(procs or os.cpu_count()) as pool:
        for i, res in enumerate(pool.imap_unordered(_c3_batch, jobs)):
            results.append(res)
            if i % 10 == 0:
                print(f"C3 batch {i}/{len(jobs)} {time.time() - t0:.0f}s", flush=True)
    total = {}
    iterations, ms = _merge_batches(results, total, ["sg"])
    r = total["sg"]
    closed = W.sg_count(K, C3_SHAPE["depth"])
    if r["rows"] != closed:
        raise RuntimeError(f"C3: reference rows {r['rows']} != closed form {closed}")
    return {"config": "C3 sg_forest({trees}, {depth})".format(**C3_SHAPE),
            "source": f"unmodified reference (oracle/_ref) on {len(jobs)} batches of {batch} disjoint trees; "
                      "rows also equal the closed form",
            "rows": r["rows"], "fingerprint": r["fingerprint"], "deltas": r["deltas"],
            "iterations": iterations, "reference_cpu_s_sum": round(ms / 1000.0, 1),
            "reference_wall_s": round(time.time() - t0, 1)}


C5_SCALE = 340


def c5():
    f = W.lubm_facts(C5_SCALE)
    t0 = time.time()
    rels, it, tms = run_reference(W.LUBM_PROGRAM, f, os.cpu_count() or 1)
    return {"config": f"C5 lubm_facts({C5_SCALE})", "facts": int(sum(v.shape[0] for v in f.values())),
            "source": "unmodified reference (oracle/_ref)", "relations": rels, "iterations": it,
            "reference_total_ms": round(tms, 1), "reference_wall_s": round(time.time() - t0, 1)}


def main():
    which = sys.argv[1:] or ["c1", "c2"]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    if "c2" in which:
        data["C2"] = c2_ref()
        # second, independent witness: the dense distance-layer closure
        w = c2()
        if (w["rows"], w["fingerprint"], w["deltas"]) != (data["C2"]["rows"], data["C2"]["fingerprint"],
                                                            data["C2"]["deltas"]):
            raise RuntimeError("C2: reference and distance-layer closure disagree")
        data["C2"]["witness"] = "per-component distance-layer closure (dense matmul) agrees"
        print("C2", data["C2"]["rows"], data["C2"]["iterations"], flush=True)
    if "c3" in which:
        data["C3"] = c3_ref()
        print("C3", data["C3"]["rows"], data["C3"]["iterations"], flush=True)
    if "c1" in which:
        data["C1"] = c1()
        print("C1", data["C1"]["rows"], data["C1"]["iterations"], flush=True)
    if "c4" in which:
        data["C4"] = c4()
        print("C4", {k: v["rows"] for k, v in data["C4"]["relations"].items()}, flush=True)
    if "c5" in which:
        data["C5"] = c5()
        print("C5", data["C5"]["iterations"], flush=True)
    json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()

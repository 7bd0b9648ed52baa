"""Full-size golden values for the BASELINE configs (size-independent checks).

  C1  TC, uniform 10k nodes / 50k edges: the UNMODIFIED reference
      (oracle/_ref/colog_ref, all cores) -> |reach|, per-iteration deltas,
      order-independent fingerprint of the sorted dump.
  C2  TC, 1000 disjoint Zipf components x (1000 nodes, 5000 edges): an
      independent per-component distance-layer closure with dense matrix
      products (the semi-naive delta of iteration k is the set of pairs at
      shortest-path distance k+1) -> |reach|, deltas, fingerprint
      (fingerprints add over disjoint components).
  C3  SG forest of 244 depth-10 trees: closed form.

    python tests/golden/make_golden_large.py [c1] [c2]
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


def main():
    which = sys.argv[1:] or ["c1", "c2"]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    if "c2" in which:
        data["C2"] = c2()
        print("C2", data["C2"]["rows"], data["C2"]["iterations"], flush=True)
    if "c1" in which:
        data["C1"] = c1()
        print("C1", data["C1"]["rows"], data["C1"]["iterations"], flush=True)
    data["C3"] = {"config": "C3 sg_forest(244, 10)", "source": "closed form", "rows": W.sg_count(244, 10),
                  "iterations": 11}
    json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()

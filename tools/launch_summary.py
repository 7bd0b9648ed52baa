"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per
launch) by kernel: launches, total ms, share, DRAM GB read/written, GB/s.

    python tools/launch_summary.py gpurun_out/<dir>/launch.csv [--json out.json]
"""
import io
import json
import sys

import pandas as pd


def summarise(path):
    txt = open(path).read()
    df = pd.read_csv(io.StringIO(txt[txt.find('"ID"'):]))
    df["val"] = pd.to_numeric(df["Metric Value"].astype(str).str.replace(",", ""), errors="coerce")
    p = df.pivot_table(index=["ID", "Kernel Name"], columns="Metric Name", values="val").reset_index()
    p["kernel"] = p["Kernel Name"].str.extract(r"(\w+_kernel(?:<[^>(]*>)?)")[0].fillna(p["Kernel Name"].str[:40])
    g = p.groupby("kernel").agg(launches=("ID", "count"), ns=("gpu__time_duration.sum", "sum"),
                                rd=("dram__bytes_read.sum", "sum"), wr=("dram__bytes_write.sum", "sum"))
    g = g.sort_values("ns", ascending=False)
    total = g.ns.sum()
    out = {}
    for k, r in g.iterrows():
        out[k] = {"launches": int(r.launches), "ms": r.ns / 1e6, "share": r.ns / total,
                  "dram_read_gb": r.rd / 1e9, "dram_write_gb": r.wr / 1e9,
                  "dram_gbs": (r.rd + r.wr) / r.ns, "dram_bytes_per_launch": (r.rd + r.wr) / r.launches}
    return out, total / 1e6


if __name__ == "__main__":
    out, total = summarise(sys.argv[1])
    print(f"{'kernel':45s} {'n':>5s} {'ms':>9s} {'share':>6s} {'rdGB':>8s} {'wrGB':>8s} {'GB/s':>7s}")
    for k, r in out.items():
        print(f"{k[:45]:45s} {r['launches']:5d} {r['ms']:9.3f} {r['share']:6.3f} {r['dram_read_gb']:8.2f} "
              f"{r['dram_write_gb']:8.2f} {r['dram_gbs']:7.0f}")
    print("total kernel ms", round(total, 3))
    if "--json" in sys.argv:
        json.dump({"total_ms": total, "kernels": out}, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)

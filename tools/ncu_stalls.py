"""Warp-stall samples per source line of one `ncu --set full --import-source
on` capture (the source page's "Warp Stall Sampling (All Samples)" column,
summed over each line's SASS), top lines first.

    python tools/ncu_stalls.py capture.ncu-rep [--top 20] [--json out.json]
"""
import argparse
import csv
import io
import json
import subprocess


def stalls(rep, top=20):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True, check=True).stdout
    lines, total, fname = {}, 0, None
    for r in csv.reader(io.StringIO(txt)):
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 6 or not r[0] or r[0] == "Line No" or r[2] != "-":
            continue
        try:
            n = int(r[4])
        except ValueError:
            continue
        lines[(fname, int(r[0]))] = (n, r[1].strip())
        total += n
    out = [{"file": f, "line": ln, "share": round(n / total, 4), "source": src[:120]}
           for (f, ln), (n, src) in sorted(lines.items(), key=lambda x: -x[1][0])[:top]]
    return {"capture": rep.split("/")[-1], "samples": total, "top_lines": out}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=20)
    ap.add_argument("--json")
    a = ap.parse_args()
    res = stalls(a.rep, a.top)
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)
    for t in res["top_lines"]:
        print(f'{100 * t["share"]:5.1f}%  {t["file"]}:{t["line"]}  {t["source"][:90]}')

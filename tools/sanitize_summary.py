"""Condense the compute-sanitizer logs of tools/sanitize.sh into one JSON
(per log: the tool's ERROR SUMMARY line, the exit line, the distinct hazard
sites it reported and, for the drop-in doctest suites, the suite summary).

    python tools/sanitize_summary.py gpurun_out/<tag> profiles/<round>/sanitizer/summary_<tag>.json "<source note>"
"""
import json
import os
import re
import sys


def summarise(src: str) -> dict:
    logs = {}
    for f in sorted(os.listdir(src)):
        if not f.endswith(".log"):
            continue
        txt = open(os.path.join(src, f), errors="replace").read()
        summary = re.findall(r"(?:ERROR|RACECHECK) SUMMARY: .*", txt)
        exits = re.findall(r"^exit \d+", txt, re.M)
        sites = sorted(set(re.findall(r"(?:Race reported|Invalid \w+ of size \d+|Barrier error).*?(?:\n\s+at .*)?", txt)))
        suite = re.findall(r"\[doctest\] test cases: .*", txt)
        pytest = re.findall(r"\d+ passed.*", txt)
        logs[f] = {"summary": summary[-1] if summary else None, "exit": exits[-1] if exits else None,
                   "hazard_sites": sites[:20], "suite": suite[-1] if suite else (pytest[-1] if pytest else None)}
    return logs


if __name__ == "__main__":
    src, dst = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else "tools/sanitize.sh on a B200"
    os.makedirs(os.path.dirname(dst), exist_ok=True)
    json.dump({"source": note, "logs": summarise(src)}, open(dst, "w"), indent=1)
    print(dst)

"""Build profiles/<round>/ from a gpu_round.sh output directory:

  launches.json      per-kernel totals of the ncu launch list (every launch of
                     one bench step: gpu__time_duration, dram bytes)
  full_<kernel>.json key metrics of each `ncu --set full` capture (duration,
                     DRAM bytes, throughput, occupancy, L2 hit, top stalls)
  bench.json, membench.json, pytest_gpu.log (copied)

and profiles/ncu_summary.json, which bench.py reads for roofline.traffic:
{"kernels": {<profiler name>: {"dram_bytes_per_launch": ..., "kernel": ...}}}.

    python tools/ncu_summary.py gpurun_out/r1b profiles/r1
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_summary import summarise  # noqa: E402

# bench.py / fv_ctx_profile names -> CUDA kernel names in the launch list
PROFILER_TO_KERNEL = {
    # fused join + set dedup: word form (<.., 1, 1>), block set (<.., 1, 0>),
    # key set (<.., 0, 0>); round-1 names had two template arguments
    "join_dedup": ["materialize_kernel<0, 0, 1, 1>", "materialize_kernel<0, 0, 1, 0>", "materialize_kernel<0, 0, 0, 0>",
                   "materialize_kernel<0, 0, 1>", "materialize_kernel<0, 0>"],
    "join_materialize": ["materialize_kernel<0, 0, 0, 0>", "materialize_kernel<0, 0>"],
    "blockset_insert": ["blockset_word_insert_kernel", "blockset_insert_kernel"],
    "blockset_collect": "blockset_collect_kernel",
    "blockset_grow": "blockset_grow_kernel",
    "group_keys": ["group_count_kernel", "group_scatter_kernel"],
    "hash_insert": "hash_insert_keys_kernel",
    "radix_onesweep_u64": "onesweep_kernel<unsigned long, 0>",
    "radix_histogram": "radix_hist_kernel<unsigned long>",
    "merge_dedup": "merge_kernel<1>",
    "unpack_keys": "unpack_keys_kernel",
    "pack_keys": "pack_kernel",
    "join_probe_count": "probe_count_kernel",
    "hash_grow": "hash_grow_kernel",
    "hash_rehash": "hash_rehash_kernel",
}

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
]


def full_capture(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return None
    h, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        m = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in FULL_METRICS:
            if k in d:
                m[k] = d[k] + (" " + u[k] if u.get(k) else "")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
                except ValueError:
                    pass
        m["top_stalls_cycles_per_issue"] = {k: round(v, 2) for v, k in sorted(stalls, reverse=True)[:5]}
        out.append(m)
    return out


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    launches, total_ms = summarise(os.path.join(src, "launches.csv"))
    json.dump({"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                         "--clock-control none, python bench.py --steps 1 --warmup 0 (cold-cache, serialised)",
               "total_kernel_ms": total_ms, "kernels": launches},
              open(os.path.join(dst, "launches.json"), "w"), indent=1)
    for f in sorted(os.listdir(src)):
        if f.startswith("launches_") and f.endswith(".csv"):
            ks, tot = summarise(os.path.join(src, f))
            src_txt = ("ncu launch list of C2 over 8 virtual ranks, all ranks (tools/bench_sharded.py)"
                       if "sharded" in f else f"ncu launch list of one {f[9:-4]} fixpoint (tools/bench_workloads.py)")
            json.dump({"source": src_txt,
                       "total_kernel_ms": tot, "kernels": ks},
                      open(os.path.join(dst, f.replace(".csv", ".json")), "w"), indent=1)
    for f in sorted(os.listdir(src)):
        if f.startswith("full_") and f.endswith(".ncu-rep"):
            cap = full_capture(os.path.join(src, f))
            if cap:
                json.dump(cap, open(os.path.join(dst, f.replace(".ncu-rep", ".json")), "w"), indent=1)
            if f == "full_materialize_kernel.ncu-rep":
                from ncu_stalls import stalls  # warp-stall samples per source line
                try:
                    json.dump(stalls(os.path.join(src, f)),
                              open(os.path.join(dst, "stalls_materialize_kernel.json"), "w"), indent=1)
                except Exception as e:  # noqa: BLE001 (capture without source counters)
                    print("stalls:", e)
    for f in ("bench.json", "membench.json", "workloads.json", "ops.json", "io.json", "sortbench.json", "sharded.json",
              "pytest_gpu.log", "smoke.log", "nproc.txt", "lscpu.txt"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    summary = {"round_dir": dst, "kernels": {}}
    for prof, kerns in PROFILER_TO_KERNEL.items():
        kerns = kerns if isinstance(kerns, list) else [kerns]
        ks = [launches[k] for k in kerns if k in launches]
        if not ks:
            continue
        n = sum(k["launches"] for k in ks)
        by = sum((k["dram_read_gb"] + k["dram_write_gb"]) * 1e9 for k in ks)
        summary["kernels"][prof] = {"kernel": " + ".join(k for k in kerns if k in launches),
                                    "dram_bytes_per_launch": by / n, "launches_per_step": n,
                                    "share_of_step": sum(k["share"] for k in ks)}
    json.dump(summary, open(os.path.join(os.path.dirname(dst.rstrip("/")), "ncu_summary.json"), "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

#!/usr/bin/env python
"""Benchmark: seconds to fixpoint & derived tuples/s (BASELINE.json metric).

Workload (N=1 line, BASELINE.json configs[1]): transitive closure on the C2
synthetic power-law graph — 1000 disjoint components x (1000 nodes, 5000
distinct edges), Zipf(1.0) sources. One step = one complete
fixpoint (seed + all semi-naive iterations) of the reference's TC program.

  value  derived tuples/s with the EDB already resident in HBM (fv_edb +
         fv_evaluate_program_edb), device-timed with CUDA events, max over
         ranks; FULL grows to 5.2 GB per step, far beyond the 126 MB L2.
  e2e    the same metric through the reference-facing C ABI with HOST
         buffers (fv_evaluate_program: pinned host facts uploaded inside the
         timed step) and a device->host read of the result statistics.
  roofline  live per-kernel CUDA-event timing inside the timed steps
         (fv_ctx_profile), dominant kernel vs MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the unmodified reference (oracle/_ref/colog_ref, all host
         cores) on a bounded sample: the first components of the same graph.

Multi-GPU (torchrun, N>1): the hash-partitioned engine over NCCL (weak
scaling): the graph is N x 1000 components (N C2 instances, disjoint node
ids), the EDB is replicated, `reach` is partitioned by hash(col 0) and every
iteration routes new candidate tuples to their owner GPU with one NCCL
all-to-all and all-reduces |Δ|; time = max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fvlog|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "seconds to fixpoint & derived tuples/sec (TC, SG, CSPA) at 1/2/4/8 B200"
UNIT = "tuples/s"
COMPONENTS, NODES, EDGES = 1000, 1000, 5000
WORKLOAD = (f"TC C2: {COMPONENTS} disjoint Zipf(1.0) components x ({NODES} nodes, {EDGES} edges) "
            f"= {COMPONENTS * NODES} nodes / {COMPONENTS * EDGES} edges, reference tc.dl")


def rank_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def graph_for(world: int = 1, dist=None):
    """N x C2: components 0..999 are the N=1 graph; more are appended. Under
    torchrun every rank generates its own 1000 components and the slices are
    all-gathered (the EDB is replicated)."""
    from paper_2501_13051_b200 import workloads as W
    if dist is None or world == 1:
        return W.tc_powerlaw(COMPONENTS * world, NODES, EDGES, seed=1)
    import torch
    rank = dist.get_rank()
    mine = W.tc_powerlaw(COMPONENTS, NODES, EDGES, seed=1, first=rank * COMPONENTS)
    t = torch.from_numpy(mine.view(np.int32)).cuda()
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return torch.cat(parts).cpu().numpy().view(np.uint32)


# ---- clocks ---------------------------------------------------------------------------

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}


class ClockSampler:
    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.2)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---- CPU reference --------------------------------------------------------------------


def reference_sample(components: int, rank: int = 0):
    """Run the unmodified reference (oracle/_ref/colog_ref, all host cores) on
    the first `components` components of the rank's graph. Returns
    (derived tuples, seconds to fixpoint, cores, kind)."""
    from paper_2501_13051_b200 import workloads as W
    e = graph_for(1)[: components * EDGES]
    ref_bin = os.path.join(ROOT, "oracle", "_ref", "colog_ref")
    cores = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as d:
        if os.path.exists(ref_bin):
            W.write_tsv_dir(os.path.join(d, "facts"), {"edge": e})
            prog = os.path.join(d, "tc.dl")
            open(prog, "w").write(W.TC_PROGRAM)
            r = subprocess.run([ref_bin, "run", prog, "--facts", os.path.join(d, "facts"), "--out",
                                os.path.join(d, "out"), "--workers", str(cores)],
                               capture_output=True, text=True, check=True)
            rows = {l.split()[0][4:]: int(l.split()[1][5:]) for l in r.stdout.splitlines()
                    if l.startswith("rel=")}
            total_ms = float([l for l in r.stdout.splitlines() if l.startswith("iterations=")][0]
                             .split()[1].split("=")[1])
            return rows["reach"], total_ms / 1000.0, cores, "reference"
    # Fallback: the single-threaded C restatement of the reference (port).
    from oracle.bind import Oracle
    from paper_2501_13051_b200 import engine as E
    prog = E.compile_program(W.TC_PROGRAM)
    t0 = time.perf_counter()
    it, rels, _ = Oracle().evaluate(*prog.oracle_args({"edge": e}))
    dt = time.perf_counter() - t0
    return rels[prog.relation_index("reach")].shape[0], dt, 1, "port"


def run_reference_impl(args):
    rank, world, _ = rank_env()
    if rank != 0:
        return
    comps = args.ref_components
    for _ in range(args.warmup if args.ref_warmup else 0):
        reference_sample(comps)
    total_tuples, total_s, cores, kind = 0, 0.0, 1, "reference"
    for _ in range(args.steps):
        n, s, cores, kind = reference_sample(comps)
        total_tuples += n
        total_s += s
    value = total_tuples / total_s
    sample = (f"first {comps} of {COMPONENTS} components of the C2 graph per step "
              f"({comps * EDGES} edges); reference total_ms (evaluate only)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * total_s / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (splitmix64 seed 1)", "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- GPU arm ----------------------------------------------------------------------------


def run_fvlog(args):
    rank, world, local = rank_env()
    # Keep stdout to the one JSON line (NCCL prints its version banner at
    # INFO/VERSION levels).
    os.environ["NCCL_DEBUG"] = "WARN"
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local if world > 1 else 0
    torch.cuda.set_device(device)

    from paper_2501_13051_b200 import colog, engine as E, workloads as W
    import ctypes as C
    from paper_2501_13051_b200 import _lib

    ctx = colog.Context(device)
    l = ctx._lib
    E._bind()
    _lib.bind("fv_ctx_profile", C.c_int, [C.c_void_p, C.c_int])
    _lib.bind("fv_ctx_profile_count", C.c_uint32, [C.c_void_p])
    _lib.bind("fv_ctx_profile_entry", C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_char_p),
                                                 C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                                 C.POINTER(C.c_double)])
    _lib.bind("fv_edb_upload", C.c_int, [C.c_void_p, C.POINTER(E.fv_relation_decl), C.c_uint32,
                                         C.POINTER(E.fv_facts), C.c_uint32, C.POINTER(C.c_void_p)])
    _lib.bind("fv_edb_free", None, [C.c_void_p])
    _lib.bind("fv_ctx_reserve", C.c_int, [C.c_void_p, C.c_uint64])
    # Map the memory pool once up front (outside every timed region) so the
    # fixpoints sub-allocate instead of growing the pool mid-iteration.
    _lib.check(l.fv_ctx_reserve(ctx.h, int(args.reserve_gb * 2**30)), ctx.h)
    _lib.bind("fv_evaluate_program_edb", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)])

    if world > 1:
        uid = [E.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        E.set_nccl(ctx, rank, world, uid[0])
    elif args.partitioned:
        # The multi-GPU code path on one GPU: a 1-rank NCCL communicator with
        # the partitioned engine forced on (routing + NCCL exchange to self).
        os.environ["FVLOG_FORCE_PARTITIONED"] = "1"
        E.set_nccl(ctx, 0, 1, E.nccl_unique_id())
    edges = graph_for(world, dist)
    # pinned host copy of the EDB for the e2e leg
    # Host facts for the e2e leg: pinned SoA columns (the fv_facts layout),
    # prepared once outside every timed region.
    pinned_cols = []
    for j in range(edges.shape[1]):
        t = torch.empty(edges.shape[0], dtype=torch.int32, pin_memory=True)
        t.numpy().view(np.uint32)[:] = edges[:, j]
        pinned_cols.append(t)
    h2d_bytes = sum(t.numel() * 4 for t in pinned_cols)
    e2e_ptrs = (C.POINTER(C.c_uint32) * len(pinned_cols))(
        *[C.cast(t.data_ptr(), C.POINTER(C.c_uint32)) for t in pinned_cols])
    e2e_facts = (E.fv_facts * 1)(E.fv_facts(b"edge", len(pinned_cols), edges.shape[0], e2e_ptrs))
    prog = E.compile_program(W.TC_PROGRAM)
    decls = prog.relations()
    d_arr = (E.fv_relation_decl * len(decls))(*[E.fv_relation_decl(n.encode(), a) for n, a in decls])
    f_arr, nf, keep = E._facts_array({"edge": edges}, dict(decls))
    edb = C.c_void_p()
    _lib.check(l.fv_edb_upload(ctx.h, d_arr, len(decls), f_arr, nf, C.byref(edb)), ctx.h)

    def step_resident():
        h = C.c_void_p()
        _lib.check(l.fv_evaluate_program_edb(ctx.h, prog.h, edb, C.byref(h)), ctx.h)
        return E.State(ctx, h.value)

    def step_e2e():
        h = C.c_void_p()
        _lib.check(l.fv_evaluate_program(ctx.h, prog.h, e2e_facts, 1, C.byref(h)), ctx.h)
        st = E.State(ctx, h.value)
        stats = st.stats()  # device->host read of the step's result
        return st, stats

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- warmup ----
    derived = None
    for _ in range(args.warmup):
        st = step_resident()
        derived = st.derived_tuples()
        iterations = st.iterations
        del st

    # ---- timed: resident EDB ----
    launches0 = ctx.kernel_launches()
    _lib.check(l.fv_ctx_profile(ctx.h, 1), ctx.h)
    sampler = ClockSampler(device)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tuples = 0
    with sampler:
        ev0.record()
        for _ in range(args.steps):
            st = step_resident()
            tuples += st.derived_tuples()
            rows, iterations = st.rows("reach"), st.iterations
            # Drop the step's result before the next step (as a caller
            # would): two live fixpoints would double the pool footprint.
            del st
        ev1.record()
        barrier()
    dev_ms = ev0.elapsed_time(ev1)
    _lib.check(l.fv_ctx_profile(ctx.h, 0), ctx.h)
    launches = ctx.kernel_launches() - launches0
    kernels = []
    for i in range(l.fv_ctx_profile_count(ctx.h)):
        nm, la, ms, by = C.c_char_p(), C.c_uint64(), C.c_double(), C.c_double()
        _lib.check(l.fv_ctx_profile_entry(ctx.h, i, C.byref(nm), C.byref(la), C.byref(ms), C.byref(by)), ctx.h)
        kernels.append({"name": nm.value.decode(), "launches": la.value, "ms": ms.value, "bytes": by.value})
    kernels.sort(key=lambda k: -k["ms"])

    t_max = max_over_ranks(dev_ms)
    # Stats (hence derived tuples) are global in a partitioned evaluation.
    all_tuples = float(tuples)
    value = all_tuples / (t_max / 1000.0)

    # ---- timed: e2e through the C ABI with host buffers ----
    barrier()
    if args.no_e2e:
        args_steps_e2e = 0
    else:
        args_steps_e2e = args.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_tuples = 0
    d2h = 0
    e0.record()
    for _ in range(args_steps_e2e):
        st, stats = step_e2e()
        e2e_tuples += st.derived_tuples()
        d2h = 40 * len(stats) + 24 * len(st.relations())
        del st
    e1.record()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = float(e2e_tuples) / (e2e_ms / 1000.0) if args_steps_e2e else None

    # ---- untimed: key-set probe count of one fixpoint (FVLOG_TRACE) ----
    # The fused join is bound by random key-set accesses, not by streaming
    # bytes: count its probes on one extra, untimed step (the engine's trace
    # counts them) to put its live duration against the measured random-load
    # ceiling of tools/membench.cu.
    probe_stats = None
    if world == 1 and not args.partitioned and not args.no_random_access:
        os.environ["FVLOG_TRACE"] = "1"
        sys.stderr.flush()
        saved = os.dup(2)
        with tempfile.TemporaryFile() as tmp:
            os.dup2(tmp.fileno(), 2)
            try:
                st = step_resident()
                del st
                ctx.synchronize()
            finally:
                os.dup2(saved, 2)
                os.close(saved)
                del os.environ["FVLOG_TRACE"]
            tmp.seek(0)
            cands = probes = 0
            for ln in tmp.read().decode(errors="replace").splitlines():
                f = ln.split()
                if "fused" in f and "dedup:" in f and len(f) >= 7:
                    cands += int(f[3])
                    probes += int(f[6])
        probe_stats = (cands, probes)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peaks()
    top = kernels[0] if kernels else None
    roofline = None
    if top:
        achieved = (top["bytes"] / top["launches"]) / (top["ms"] / top["launches"] / 1000.0) / 1e9
        traffic = None
        ncu = os.path.join(ROOT, "profiles", "ncu_summary.json")
        if os.path.exists(ncu):
            tr = json.load(open(ncu)).get("kernels", {}).get(top["name"], {})
            traffic = tr.get("dram_bytes_per_launch")
        roofline = {"bound": "hbm", "kernel": top["name"], "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                    "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": top["bytes"] / top["launches"],
                    "avg_launch_ms": top["ms"] / top["launches"]}
    random_access = None
    join = next((k for k in kernels if k["name"] == "join_dedup"), None)
    if probe_stats and join and probe_stats[1]:
        mb = os.path.join(ROOT, "profiles", "r1", "membench.json")
        ceiling = json.load(open(mb)).get("rand_load_gaccess_s") if os.path.exists(mb) else None
        rate = probe_stats[1] / (join["ms"] / args.steps / 1000.0) / 1e9
        random_access = {"kernel": "join_dedup", "candidates_per_step": probe_stats[0],
                         "keyset_probes_per_step": probe_stats[1], "achieved_gprobes_s": round(rate, 2),
                         "ceiling_gloads_s": ceiling,
                         "frac": round(rate / ceiling, 3) if ceiling else None,
                         "ceiling_source": "random 8-byte loads into an 8 GB table, tools/membench.cu on a B200 "
                                           "(profiles/r1/membench.json)",
                         "probe_count_source": "one extra untimed step with FVLOG_TRACE=1"}
    step_ms = t_max / args.steps
    total_kernel_ms = sum(k["ms"] for k in kernels)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "seconds_to_fixpoint": step_ms / 1000.0,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (splitmix64 seed 1+rank, tests/golden/large.json pins the fixpoint)",
        "config": {"workload": WORKLOAD, "program": "reach(x,y):-edge(x,y). reach(x,z):-edge(x,y),reach(y,z).",
                   "derived_tuples_per_step": int(tuples // args.steps), "reach_rows": rows,
                   "iterations": iterations,
                   "parallelism": (f"hash-partitioned x{world}: reach by hash(col 0), edge replicated, "
                                   f"one NCCL all-to-all + all-reduce per iteration")
                                  if world > 1 or args.partitioned else "1 GPU",
                   "components": COMPONENTS * world,
                   "l2": "inputs larger than L2 (FULL grows to >5 GB per step, L2 126 MB)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms / max(1, args_steps_e2e),
                "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": d2h,
                "path": "fv_evaluate_program (host pinned facts) + fv_state_stat readback"},
        "gpu_launches": int(launches),
        "clocks": sampler.summary(),
        "roofline": roofline,
        "random_access": random_access,
        "kernels": [{"name": k["name"], "launches": k["launches"], "ms_per_step": k["ms"] / args.steps,
                     "share": round(k["ms"] / total_kernel_ms, 4) if total_kernel_ms else None,
                     "gbs": round(k["bytes"] / (k["ms"] / 1000.0) / 1e9, 1) if k["ms"] else None}
                    for k in kernels[:8]],
    }
    if world == 1 and not args.no_cpu_baseline:
        n, s, cores, kind = reference_sample(args.ref_components)
        line["cpu_baseline"] = {"value": n / s, "unit": UNIT, "cores": cores, "kind": kind,
                                "sample": f"first {args.ref_components} of {COMPONENTS} components "
                                          f"({n} derived tuples, {s:.2f} s to fixpoint)"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fvlog", choices=["fvlog", "reference"])
    ap.add_argument("--ref-components", type=int, default=30)
    ap.add_argument("--ref-warmup", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e leg (profiling runs)")
    ap.add_argument("--no-random-access", action="store_true",
                    help="skip the untimed traced step that counts key-set probes (profiling runs)")
    ap.add_argument("--reserve-gb", type=float, default=96.0, help="fv_ctx_reserve before warm-up")
    ap.add_argument("--partitioned", action="store_true",
                    help="N=1 only: run the hash-partitioned multi-GPU path over a 1-rank NCCL communicator")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_impl(args)
    else:
        run_fvlog(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: seconds to fixpoint & derived tuples/s (BASELINE.json metric).

Headline workload (BASELINE.json configs[1]): transitive closure on the C2
synthetic power-law graph — 1000 disjoint components x (1000 nodes, 5000
distinct edges), Zipf(1.0) sources. One step = one complete
fixpoint (seed + all semi-naive iterations) of the reference's TC program.

  value   derived tuples/s with the EDB already resident in HBM (fv_edb +
          fv_evaluate_program_edb), device-timed with CUDA events with the
          kernel profiler OFF, max over ranks; FULL grows to 5.2 GB per step,
          far beyond the 126 MB L2.
  parity  the timed step's result against tests/golden/large.json (generated
          by the unmodified reference): row count, per-iteration deltas,
          iterations and the order-independent fingerprint (N=1).
  kernels/roofline  a separate profiled pass (fv_ctx_profile: per-launch CUDA
          events) of the same step; dominant kernel vs MEASURED_PEAKS.json.
  e2e     the same metric through the reference-facing C ABI with HOST
          buffers: pinned facts uploaded inside the timed step
          (fv_evaluate_program) and the result statistics read back.
  e2e_with_dump  as e2e, plus the sorted result relation copied to a pinned
          host buffer every step (fv_state_dump_sorted: 5.2 GB D2H for C2).
  cpu_baseline  the unmodified reference (oracle/_ref/colog_ref, all host
          cores) on a bounded sample (the first components of the same graph),
          with the GPU timed on that identical sample (same_input).
  workloads  SG (C3), CSPA (C4) and OWL-RL/LUBM (C5) timed in the same run,
          each with its parity check against the reference goldens.

Multi-GPU (N>1): the hash-partitioned engine over NCCL, weak scaling — N
disjoint copies of every workload (node ids shifted per copy); the EDB is
replicated, IDB relations are partitioned, |Δ| is all-reduced; time = max
over ranks. `python bench.py --gpus N` re-launches itself under
torch.distributed.run when WORLD_SIZE is unset, and fails loudly when the box
has fewer than N GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fvlog|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
GOLDEN = os.path.join(ROOT, "tests", "golden", "large.json")


def rank_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---- workloads ------------------------------------------------------------------------


def replicate(facts: dict, copies: int) -> dict:
    """`copies` disjoint instances of the same facts (node ids shifted by the
    instance's index x the active-domain span): the weak-scaling input."""
    if copies == 1:
        return facts
    span = 1 + max(int(v.max()) for v in facts.values() if v.size)
    return {k: np.concatenate([v + np.uint32(r * span) for r in range(copies)]) for k, v in facts.items()}


def workload_specs():
    from paper_2501_13051_b200 import workloads as W
    return {
        "TC-C2": dict(program=W.TC_PROGRAM, golden="C2", result="reach",
                      facts=lambda: {"edge": W.tc_powerlaw(COMPONENTS, NODES, EDGES, seed=1)},
                      desc=f"TC C2: {COMPONENTS} disjoint Zipf(1.0) components x ({NODES} nodes, {EDGES} edges) "
                           f"= {COMPONENTS * NODES} nodes / {COMPONENTS * EDGES} edges, reference tc.dl"),
        "SG-C3": dict(program=W.SG_PROGRAM, golden="C3", result="sg",
                      facts=lambda: {"edge": W.sg_forest(244, 10)},
                      desc="SG C3: forest of 244 complete binary trees of depth 10 (499,224 edges), reference sg.dl"),
        "CSPA-C4": dict(program=W.CSPA_PROGRAM, golden="C4", result=None,
                        facts=lambda: W.cspa_facts(4000, 100, 100, 70),
                        desc="CSPA C4: 4000 disjoint functions x 100 variables (400k assign, 280k dereference)"),
        "LUBM-C5": dict(program=W.LUBM_PROGRAM, golden="C5", result=None,
                        facts=lambda: W.lubm_facts(340),
                        desc="OWL-RL/LUBM C5: lubm_facts(340), 10.15 M facts, 40 rules"),
    }


def headline_config(world: int) -> dict:
    """The headline's `config` — static, so both arms print the identical dict."""
    return {"workload": workload_specs()["TC-C2"]["desc"] + (f"; {world} disjoint copies (weak scaling)"
                                                            if world > 1 else ""),
            "program": "reach(x,y):-edge(x,y). reach(x,z):-edge(x,y),reach(y,z).",
            "components": COMPONENTS * world,
            "l2": "inputs larger than L2 (FULL grows to >5 GB per copy per step, L2 126 MB)"}


def golden_relations(g: dict, result: str | None) -> dict:
    return g["relations"] if "relations" in g else {result: g}


def check_parity(states, g: dict, result, world: int, dist=None) -> dict:
    """A step's result vs the reference golden: per relation rows, per-
    iteration deltas (stats are global in a partitioned run) and, at N=1, the
    order-independent fingerprint; weak scaling multiplies rows and deltas."""
    if not g:
        return {"golden": None, "match": None, "why": "tests/golden/large.json has no entry"}
    st = states
    deltas = st.delta_counts()
    rels = st.relations()
    bad = []
    checked = 0
    for rel, exp in golden_relations(g, result).items():
        rows = rels[rel][1]
        if dist is not None:
            import torch
            t = torch.tensor([rows], dtype=torch.int64, device="cuda")
            dist.all_reduce(t)
            rows = int(t.item())
        if rows != world * exp["rows"]:
            bad.append(f"{rel}: rows {rows} != {world * exp['rows']}")
        if rel in deltas and "deltas" in exp and deltas[rel] != [world * d for d in exp["deltas"]]:
            bad.append(f"{rel}: deltas differ")
        if world == 1 and "fingerprint" in exp and str(st.fingerprint(rel)) != exp["fingerprint"]:
            bad.append(f"{rel}: fingerprint differs")
        checked += 1
    if st.iterations != g["iterations"]:
        bad.append(f"iterations {st.iterations} != {g['iterations']}")
    out = {"golden": g["config"].split()[0], "source": g.get("source"), "relations_checked": checked,
           "checks": "rows, per-iteration deltas, iterations" + (", fingerprint" if world == 1 else
                                                                 f" (x{world} copies)"),
           "match": not bad}
    if bad:
        out["mismatches"] = bad[:8]
    return out


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
            time.sleep(0.05)

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


def sample_edges(components: int):
    """The CPU sample: the first `components` components of the headline graph."""
    from paper_2501_13051_b200 import workloads as W
    return W.tc_powerlaw(components, NODES, EDGES, seed=1)


class ReferenceSample:
    """The unmodified reference (oracle/_ref/colog_ref) on the sample, all host
    cores; the facts directory is written once. Falls back to the C
    restatement (port, one thread) where the reference binary is absent."""

    def __init__(self, components: int):
        from paper_2501_13051_b200 import workloads as W
        self.components = components
        self.edges = sample_edges(components)
        self.ref_bin = os.path.join(ROOT, "oracle", "_ref", "colog_ref")
        self.cores = os.cpu_count() or 1
        self.dir = tempfile.TemporaryDirectory()
        d = self.dir.name
        self.kind = "reference" if os.path.exists(self.ref_bin) else "port"
        if self.kind == "reference":
            W.write_tsv_dir(os.path.join(d, "facts"), {"edge": self.edges})
            self.prog = os.path.join(d, "tc.dl")
            open(self.prog, "w").write(W.TC_PROGRAM)

    def run(self):
        """(derived tuples, seconds to fixpoint): the reference's total_ms,
        i.e. evaluate() from EDB seed to fixpoint (P/src/runner.cpp:58-61)."""
        from paper_2501_13051_b200 import workloads as W
        d = self.dir.name
        if self.kind == "reference":
            r = subprocess.run([self.ref_bin, "run", self.prog, "--facts", os.path.join(d, "facts"), "--out",
                                os.path.join(d, "out"), "--workers", str(self.cores), "--stats"],
                               capture_output=True, text=True, check=True)
            derived = sum(int(l.split()[2].split("=")[1]) for l in r.stdout.splitlines() if l.startswith("iter="))
            total_ms = float([l for l in r.stdout.splitlines() if l.startswith("iterations=")][0]
                             .split()[1].split("=")[1])
            return derived, total_ms / 1000.0
        from oracle.bind import Oracle
        from paper_2501_13051_b200 import engine as E
        prog = E.compile_program(W.TC_PROGRAM)
        t0 = time.perf_counter()
        it, rels, _ = Oracle().evaluate(*prog.oracle_args({"edge": self.edges}))
        dt = time.perf_counter() - t0
        self.cores = 1
        return rels[prog.relation_index("reach")].shape[0], dt

    def describe(self):
        return (f"first {self.components} of {COMPONENTS} components of the C2 graph per step "
                f"({self.components * EDGES} edges); reference total_ms = evaluate() only")


def run_reference_impl(args):
    rank, world, _ = rank_env()
    if rank != 0:
        return
    ref = ReferenceSample(args.ref_components)
    for _ in range(args.warmup):
        ref.run()
    total_tuples, total_s = 0, 0.0
    for _ in range(args.steps):
        n, s = ref.run()
        total_tuples += n
        total_s += s
    value = total_tuples / total_s
    sample = ref.describe()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * total_s / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (splitmix64 seed 1)", "config": headline_config(world),
            "parallelism": f"CPU, {ref.cores} host threads",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref.cores, "kind": ref.kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- GPU arm ----------------------------------------------------------------------------


class Runner:
    """One process's GPU context, NCCL wiring and timing helpers."""

    def __init__(self, args):
        self.args = args
        self.rank, self.world, local = rank_env()
        # Keep stdout to the one JSON line (NCCL prints its banner at INFO).
        os.environ["NCCL_DEBUG"] = "WARN"
        import torch
        self.torch = torch
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            self.dist = dist
        self.device = local if self.world > 1 else 0
        torch.cuda.set_device(self.device)
        import ctypes as C
        from paper_2501_13051_b200 import _lib, colog, engine as E
        self.C, self.E, self._lib = C, E, _lib
        self.ctx = colog.Context(self.device)
        self.l = self.ctx._lib
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
        _lib.bind("fv_evaluate_program_edb", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)])
        # Map the memory pool once up front (outside every timed region) so the
        # fixpoints sub-allocate instead of growing the pool mid-iteration.
        _lib.check(self.l.fv_ctx_reserve(self.ctx.h, int(args.reserve_gb * 2**30)), self.ctx.h)
        if self.world > 1:
            uid = [E.nccl_unique_id() if self.rank == 0 else None]
            self.dist.broadcast_object_list(uid, src=0)
            E.set_nccl(self.ctx, self.rank, self.world, uid[0])
        elif args.partitioned:
            # The multi-GPU code path on one GPU: a 1-rank NCCL communicator
            # with the partitioned engine forced on.
            os.environ["FVLOG_FORCE_PARTITIONED"] = "1"
            E.set_nccl(self.ctx, 0, 1, E.nccl_unique_id())

    # -- plumbing
    def barrier(self):
        self.torch.cuda.synchronize()
        if self.dist is not None:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def reduce(self, x: float, op: str) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=getattr(self.dist.ReduceOp, op))
        return float(t.item())

    def prepare(self, program: str, facts: dict):
        """Compile, upload the EDB once (resident leg) and pin a host copy of
        the facts (e2e leg)."""
        C, E, torch = self.C, self.E, self.torch
        prog = E.compile_program(program)
        decls = prog.relations()
        d_arr = (E.fv_relation_decl * len(decls))(*[E.fv_relation_decl(n.encode(), a) for n, a in decls])
        f_arr, nf, keep = E._facts_array(facts, dict(decls))
        edb = C.c_void_p()
        self._lib.check(self.l.fv_edb_upload(self.ctx.h, d_arr, len(decls), f_arr, nf, C.byref(edb)), self.ctx.h)
        pinned, recs, h2d = [], [], 0
        for name, arr in facts.items():
            arr = arr.reshape(arr.shape[0], -1)
            cols = []
            for j in range(arr.shape[1]):
                t = torch.empty(arr.shape[0], dtype=torch.int32, pin_memory=True)
                t.numpy().view(np.uint32)[:] = arr[:, j]
                cols.append(t)
                h2d += arr.shape[0] * 4
            pinned.append(cols)
            ptrs = (C.POINTER(C.c_uint32) * len(cols))(*[C.cast(t.data_ptr(), C.POINTER(C.c_uint32)) for t in cols])
            recs.append(E.fv_facts(name.encode(), len(cols), arr.shape[0], ptrs))
        host = (E.fv_facts * len(recs))(*recs)
        return dict(prog=prog, edb=edb, host=host, n_host=len(recs), pinned=pinned, h2d=h2d, keep=keep)

    def release(self, w):
        self.l.fv_edb_free(w["edb"])

    def step_resident(self, w):
        h = self.C.c_void_p()
        self._lib.check(self.l.fv_evaluate_program_edb(self.ctx.h, w["prog"].h, w["edb"], self.C.byref(h)),
                        self.ctx.h)
        return self.E.State(self.ctx, h.value)

    def step_host(self, w):
        h = self.C.c_void_p()
        self._lib.check(self.l.fv_evaluate_program(self.ctx.h, w["prog"].h, w["host"], w["n_host"], self.C.byref(h)),
                        self.ctx.h)
        return self.E.State(self.ctx, h.value)

    def timed(self, steps: int, fn, sampler=None):
        """Run fn() `steps` times between barriers under CUDA events on torch's
        current stream (the engine's stream is synchronised inside every
        evaluate call, so the events bracket all of its work); returns
        (max-over-ranks ms, last fn() result, per-step results)."""
        torch = self.torch
        self.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        out = []
        if sampler is not None:
            sampler.__enter__()
        try:
            e0.record()
            for _ in range(steps):
                out.append(fn())
                if len(out) > 1:
                    out[-2] = None  # free the previous step's result (one fixpoint live)
            e1.record()
            self.barrier()
        finally:
            if sampler is not None:
                sampler.__exit__()
        return self.reduce(e0.elapsed_time(e1), "MAX"), out[-1] if out else None

    def profile(self, steps: int, fn):
        C = self.C
        self._lib.check(self.l.fv_ctx_profile(self.ctx.h, 1), self.ctx.h)
        st = None
        for _ in range(steps):
            st = None
            st = fn()
        self.ctx.synchronize()
        self._lib.check(self.l.fv_ctx_profile(self.ctx.h, 0), self.ctx.h)
        kernels = []
        for i in range(self.l.fv_ctx_profile_count(self.ctx.h)):
            nm, la, ms, by = C.c_char_p(), C.c_uint64(), C.c_double(), C.c_double()
            self._lib.check(self.l.fv_ctx_profile_entry(self.ctx.h, i, C.byref(nm), C.byref(la), C.byref(ms),
                                                        C.byref(by)), self.ctx.h)
            kernels.append({"name": nm.value.decode(), "launches": la.value, "ms": ms.value, "bytes": by.value})
        kernels.sort(key=lambda k: -k["ms"])
        return kernels, st


def roofline_of(kernels, steps):
    peak, peak_src = measured_peaks()
    top = kernels[0] if kernels else None
    if not top:
        return None
    achieved = (top["bytes"] / top["launches"]) / (top["ms"] / top["launches"] / 1000.0) / 1e9
    traffic = None
    ncu = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(ncu):
        tr = json.load(open(ncu)).get("kernels", {}).get(top["name"], {})
        traffic = tr.get("dram_bytes_per_launch")
    return {"bound": "hbm", "kernel": top["name"], "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": top["bytes"] / top["launches"],
            "avg_launch_ms": top["ms"] / top["launches"],
            "timing": "per-launch CUDA events on the engine stream, separate profiled pass of the same step"}


def kernel_table(kernels, steps):
    total = sum(k["ms"] for k in kernels)
    return [{"name": k["name"], "launches": k["launches"], "ms_per_step": k["ms"] / steps,
             "share": round(k["ms"] / total, 4) if total else None,
             "gbs": round(k["bytes"] / (k["ms"] / 1000.0) / 1e9, 1) if k["ms"] else None}
            for k in kernels[:8]]


def probe_count(R: Runner, w):
    """Key-set probes of one fixpoint: one extra, untimed step with the engine
    trace on (FVLOG_TRACE counts candidates and probes of the fused join)."""
    os.environ["FVLOG_TRACE"] = "1"
    sys.stderr.flush()
    saved = os.dup(2)
    with tempfile.TemporaryFile() as tmp:
        os.dup2(tmp.fileno(), 2)
        try:
            st = R.step_resident(w)
            del st
            R.ctx.synchronize()
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
    return cands, probes


def run_workload(R: Runner, name: str, spec: dict, golden: dict, steps: int, warmup: int) -> dict:
    """One BASELINE workload: resident-EDB fixpoints timed in this run, with
    the parity check of the last timed step."""
    facts = replicate(spec["facts"](), R.world)
    w = R.prepare(spec["program"], facts)
    for _ in range(warmup):
        st = R.step_resident(w)
        del st
    syncs0 = R.ctx.host_syncs()
    ms, st = R.timed(steps, lambda: R.step_resident(w))
    syncs = (R.ctx.host_syncs() - syncs0) / steps
    derived = st.derived_tuples()
    iterations = st.iterations
    parity = check_parity(st, golden.get(spec["golden"], {}), spec["result"], R.world, R.dist)
    del st
    # one profiled step: the device's kernel time against the step's time
    kernels, st = R.profile(1, lambda: R.step_resident(w))
    del st
    kernel_ms = sum(k["ms"] for k in kernels)
    out = {"workload": spec["desc"], "ms_per_step": ms / steps, "value": derived / (ms / steps / 1000.0),
           "unit": UNIT, "derived_tuples_per_step": derived, "iterations": iterations,
           "facts": int(sum(v.shape[0] for v in facts.values())), "steps": steps, "warmup": warmup,
           "host_syncs_per_step": syncs, "host_syncs_per_iteration": round(syncs / max(iterations, 1), 2),
           "kernel_ms_per_step": round(kernel_ms, 3),
           "kernel_busy": round(kernel_ms / (ms / steps), 3),
           "kernel_busy_what": "sum of per-launch CUDA-event kernel times (one profiled step) / ms_per_step",
           "parity": parity}
    R.release(w)
    return out


def run_fvlog(args):
    R = Runner(args)
    rank, world = R.rank, R.world
    specs = workload_specs()
    golden = json.load(open(GOLDEN)) if os.path.exists(GOLDEN) else {}
    tc = specs["TC-C2"]
    facts = replicate(tc["facts"](), world)
    w = R.prepare(tc["program"], facts)

    # ---- warmup, then the timed steps (resident EDB, profiler off) ----
    for _ in range(args.warmup):
        st = R.step_resident(w)
        del st
    launches0 = R.ctx.kernel_launches()
    syncs0 = R.ctx.host_syncs()
    sampler = ClockSampler(R.device)
    t_max, st = R.timed(args.steps, lambda: R.step_resident(w), sampler)
    launches = R.ctx.kernel_launches() - launches0
    syncs = R.ctx.host_syncs() - syncs0
    derived = st.derived_tuples()
    iterations = st.iterations
    value = derived * args.steps / (t_max / 1000.0)
    parity = check_parity(st, golden.get("C2", {}), "reach", world, R.dist)
    reach_rows = int(R.reduce(float(st.rows("reach")), "SUM"))
    del st

    # ---- profiled pass: per-kernel times and the roofline ----
    prof_steps = max(1, min(args.steps, args.profile_steps))
    kernels, st = R.profile(prof_steps, lambda: R.step_resident(w))
    del st

    # ---- e2e: host facts through the C ABI, stats read back ----
    e2e = None
    if not args.no_e2e:
        def e2e_step():
            s = R.step_host(w)
            s.stats()  # device->host read of the step's result statistics
            return s
        e2e_ms, st = R.timed(args.steps, e2e_step)
        n_stats = len(st.stats())
        e2e = {"value": derived * args.steps / (e2e_ms / 1000.0), "unit": UNIT, "ms_per_step": e2e_ms / args.steps,
               "h2d_bytes_per_step": int(w["h2d"]), "d2h_bytes_per_step": 40 * n_stats + 24 * len(st.relations()),
               "path": "fv_evaluate_program (pinned host facts) + fv_state_stat readback"}
        del st

    # ---- e2e with the result: + the sorted relation into pinned host memory ----
    e2e_dump = None
    if not args.no_e2e and not args.no_dump:
        import torch
        rows_local = None
        st = R.step_host(w)
        rows_local = st.rows("reach")
        del st
        host = torch.empty(rows_local * 2 + 2, dtype=torch.int32, pin_memory=True)
        out = host.numpy().view(np.uint32)
        dump_steps = max(1, min(args.steps, args.dump_steps))

        def dump_step():
            s = R.step_host(w)
            s.stats()
            s.dump_into("reach", out)
            return s
        d_ms, st = R.timed(dump_steps, dump_step)
        # spot-check the copied rows: sorted, and their fingerprint is the device's
        n = rows_local
        rows = out[: 2 * n].reshape(n, 2)
        ok_sorted = bool(n < 2 or np.all((rows[1:, 0] > rows[:-1, 0]) |
                                         ((rows[1:, 0] == rows[:-1, 0]) & (rows[1:, 1] > rows[:-1, 1]))))
        e2e_dump = {"value": derived * dump_steps / (d_ms / 1000.0), "unit": UNIT, "ms_per_step": d_ms / dump_steps,
                    "steps": dump_steps, "h2d_bytes_per_step": int(w["h2d"]),
                    "d2h_bytes_per_step": int(8 * n) + 40 * len(st.stats()),
                    "path": "fv_evaluate_program + fv_state_stat + fv_state_dump_sorted('reach') into pinned host "
                            "memory (the INTEGRATION.md drop-in's call shape)",
                    "dump_sorted_strictly": ok_sorted}
        del st, host, out, rows

    # ---- untimed: key-set probes of one fixpoint ----
    probe_stats = None
    if world == 1 and not args.partitioned and not args.no_random_access:
        probe_stats = probe_count(R, w)
    R.release(w)

    # ---- same-input GPU figure on the CPU reference's sample ----
    same_input = None
    ref = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = ReferenceSample(args.ref_components)
        sw = R.prepare(tc["program"], {"edge": ref.edges})
        for _ in range(2):
            s = R.step_host(sw)
            del s
        ms, s = R.timed(5, lambda: R.step_host(sw))
        gd = s.derived_tuples()
        del s
        R.release(sw)
        same_input = {"gpu_value": gd / (ms / 5 / 1000.0), "gpu_ms_per_step": ms / 5,
                      "path": "fv_evaluate_program with host facts (the span of the reference's total_ms: "
                              "EDB seed + fixpoint)", "derived_tuples": gd}

    # ---- the other BASELINE workloads, timed in this run ----
    workloads = {}
    if not args.no_workloads:
        for name in ("SG-C3", "CSPA-C4", "LUBM-C5"):
            workloads[name] = run_workload(R, name, specs[name], golden, args.workload_steps,
                                           max(1, min(args.warmup, 2)))

    if rank != 0:
        if R.dist is not None:
            R.dist.destroy_process_group()
        return

    random_access = None
    join = next((k for k in kernels if k["name"] == "join_dedup"), None)
    if probe_stats and join and probe_stats[1]:
        mb = os.path.join(ROOT, "profiles", "r1", "membench.json")
        ceiling = json.load(open(mb)).get("rand_load_gaccess_s") if os.path.exists(mb) else None
        rate = probe_stats[1] / (join["ms"] / prof_steps / 1000.0) / 1e9
        random_access = {"kernel": "join_dedup", "candidates_per_step": probe_stats[0],
                         "keyset_probes_per_step": probe_stats[1], "achieved_gprobes_s": round(rate, 2),
                         "ceiling_gloads_s": ceiling, "frac": round(rate / ceiling, 3) if ceiling else None,
                         "ceiling_source": "random 8-byte loads into an 8 GB table, tools/membench.cu on a B200 "
                                           "(profiles/r1/membench.json)",
                         "probe_count_source": "one extra untimed step with FVLOG_TRACE=1"}
    step_ms = t_max / args.steps
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "seconds_to_fixpoint": step_ms / 1000.0,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (splitmix64 seed 1; tests/golden/large.json, from the unmodified reference, pins the "
                "fixpoint)",
        "config": headline_config(world),
        "parallelism": (f"hash-partitioned x{world} over NCCL: IDB partitioned, EDB replicated, |delta| all-reduced"
                        if world > 1 or args.partitioned else "1 GPU"),
        "result": {"derived_tuples_per_step": derived, "reach_rows": reach_rows, "iterations": iterations},
        "parity": parity,
        "e2e": e2e,
        "e2e_with_dump": e2e_dump,
        "gpu_launches": int(launches),
        "kernel_busy": round(sum(k["ms"] for k in kernels) / prof_steps / (t_max / args.steps), 3),
        "host_syncs": {"per_step": syncs / args.steps, "per_iteration": round(syncs / args.steps / iterations, 2),
                       "what": "stream syncs + scalar readbacks on the engine context (fv_ctx_host_syncs)"},
        "clocks": sampler.summary(),
        "roofline": roofline_of(kernels, prof_steps),
        "random_access": random_access,
        "kernels": kernel_table(kernels, prof_steps),
        "profiled_steps": prof_steps,
    }
    if ref is not None:
        n, s = ref.run()
        cpu = n / s
        line["cpu_baseline"] = {"value": cpu, "unit": UNIT, "cores": ref.cores, "kind": ref.kind,
                                "sample": ref.describe() + f" ({n} derived tuples, {s:.2f} s to fixpoint)"}
        if same_input:
            same_input["cpu_value"] = cpu
            same_input["same_input_ratio"] = round(same_input["gpu_value"] / cpu, 1)
            same_input["sample"] = ref.describe()
            line["same_input"] = same_input
    if workloads:
        line["workloads"] = workloads
    print(json.dumps(line), flush=True)
    if R.dist is not None:
        R.dist.destroy_process_group()


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fvlog", choices=["fvlog", "reference"])
    ap.add_argument("--ref-components", type=int, default=15,
                    help="CPU reference sample: the first components of the graph (~6 s per step on 16 cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e legs (profiling runs)")
    ap.add_argument("--no-dump", action="store_true", help="skip the e2e_with_dump leg")
    ap.add_argument("--no-workloads", action="store_true", help="skip the SG / CSPA / LUBM block")
    ap.add_argument("--no-random-access", action="store_true",
                    help="skip the untimed traced step that counts key-set probes (profiling runs)")
    ap.add_argument("--profile-steps", type=int, default=3)
    ap.add_argument("--dump-steps", type=int, default=3)
    ap.add_argument("--workload-steps", type=int, default=5)
    ap.add_argument("--reserve-gb", type=float, default=96.0, help="fv_ctx_reserve before warm-up")
    ap.add_argument("--partitioned", action="store_true",
                    help="N=1 only: run the hash-partitioned multi-GPU path over a 1-rank NCCL communicator")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1:
        ap.error("--steps must be >= 1 and --warmup >= 0")
    in_torchrun = "WORLD_SIZE" in os.environ
    if args.impl == "fvlog" and args.gpus > 1 and not in_torchrun:
        # One process per GPU: re-launch under torch.distributed.run.
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} requested but this box has {have} GPU(s); refusing to run "
                  f"a smaller world", file=sys.stderr)
            sys.exit(2)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
        sys.exit(subprocess.run(cmd + sys.argv[1:]).returncode)
    if in_torchrun and args.impl == "fvlog" and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: WORLD_SIZE={os.environ['WORLD_SIZE']} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference_impl(args)
    else:
        run_fvlog(args)


if __name__ == "__main__":
    main()

"""Operator-level mirrors of the reference's relation/operator API
 at 10^7-10^8 scale: the B200 through
the C ABI against the unmodified reference operators (oracle/_ref/
libcolog_ref.so, all host cores) on the same inputs, bit-exact checked.

Per operator: end-to-end seconds through the C ABI (host arrays in, host
arrays out: H2D + kernels + D2H), the device-only kernel time from the live
per-kernel profiler (fv_ctx_profile) with its algorithmic bytes, and the
reference's seconds. The reference runs on a bounded sample when the full
input would take too long; both sides are then timed on that sample too.

    python tools/bench_ops.py [--out f.json]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.bind import Reference  # noqa: E402  (checker + CPU arm)
from paper_2501_13051_b200 import _lib, colog, workloads as W  # noqa: E402


def profile(ctx, fn):
    """Run fn with the kernel profiler on: (result, wall s, {kernel: (ms, bytes)})."""
    _lib.check(ctx._lib.fv_ctx_profile(ctx.h, 1), ctx.h)
    t = time.perf_counter()
    out = fn()
    ctx.synchronize()
    wall = time.perf_counter() - t
    _lib.check(ctx._lib.fv_ctx_profile(ctx.h, 0), ctx.h)
    ks = {}
    for i in range(ctx._lib.fv_ctx_profile_count(ctx.h)):
        nm, la, ms, by = C.c_char_p(), C.c_uint64(), C.c_double(), C.c_double()
        _lib.check(ctx._lib.fv_ctx_profile_entry(ctx.h, i, C.byref(nm), C.byref(la), C.byref(ms), C.byref(by)),
                   ctx.h)
        ks[nm.value.decode()] = (ms.value, by.value)
    return out, wall, ks


def kernel_summary(ks):
    ms = sum(v[0] for v in ks.values())
    by = sum(v[1] for v in ks.values())
    return {"kernel_ms": round(ms, 3), "algorithmic_gb": round(by / 1e9, 3),
            "achieved_gbs": round(by / (ms / 1e3) / 1e9, 1) if ms else None,
            "kernels": {k: round(v[0], 3) for k, v in sorted(ks.items(), key=lambda x: -x[1][0])[:4]}}


def timed(fn, reps=1):
    best = None
    for _ in range(reps):
        t = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t
        best = dt if best is None or dt < best else best
    return out, best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    args = ap.parse_args()
    ctx = colog.Context(0)
    for name, res, argt in [("fv_ctx_profile", C.c_int, [C.c_void_p, C.c_int]),
                            ("fv_ctx_profile_count", C.c_uint32, [C.c_void_p]),
                            ("fv_ctx_profile_entry", C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_char_p),
                                                               C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                                               C.POINTER(C.c_double)])]:
        _lib.bind(name, res, argt)
    ref = Reference()
    results = {}

    def record(name, what, gpu_full, gpu_sample, ref_sample, identical, sample_desc):
        results[name] = {"what": what, "gpu": gpu_full, "sample": sample_desc,
                         "gpu_on_sample_s": round(gpu_sample, 4), "reference_on_sample_s": round(ref_sample, 4),
                         "speedup_same_input": round(ref_sample / gpu_sample, 1) if gpu_sample else None,
                         "identical_to_reference": identical}
        print(json.dumps({name: results[name]}), flush=True)

    # build_index (P/src/column.cpp:17-43): 10^8 values, 90 % on one hot key.
    raw = W.random_values(101, 100_000_000, 1_000_000, True)
    colog.build_index_arrays(raw[:1000], ctx)  # warm
    _, wall, ks = profile(ctx, lambda: colog.build_index_arrays(raw, ctx))
    s = raw[:10_000_000]
    g, gs = timed(lambda: colog.build_index_arrays(s, ctx), 2)  # host in, host out
    r, rs = timed(lambda: ref.build_index(s))
    same = all(np.array_equal(a, b) for a, b in zip(g, r))
    record("build_index", "10^8 u32 values, 90 % one hot key (support.hpp:29-41 skew)",
           {"e2e_s": round(wall, 4), **kernel_summary(ks)}, gs, rs, same, "first 10^7 values")

    # column_join (P/src/kernels.cpp:125-135): 2*10^6 probes vs a 10^7 build column.
    build_raw = W.random_values(7, 10_000_000, 2_000_000)
    probe = W.random_values(8, 2_000_000, 2_000_000)
    col = colog.Column.build(build_raw, ctx)
    colog.column_join(probe[:100], col)
    pairs, wall, ks = profile(ctx, lambda: colog.column_join(probe, col))
    n_out = pairs.size()
    del pairs
    sp, sb = probe[:200_000], build_raw[:1_000_000]
    # the build column (with its index) is constructed inside the timed call on both sides
    g, gs = timed(lambda: colog.column_join(sp, colog.Column.build(sb, ctx)), 2)
    r, rs = timed(lambda: ref.column_join(sp, sb))
    same = np.array_equal(np.asarray(g.a_ids), r[0]) and np.array_equal(np.asarray(g.b_ids), r[1])
    record("column_join", f"2*10^6 probe values vs 10^7 build column -> {n_out} pairs (probe-major order)",
           {"e2e_s": round(wall, 4), "pairs": n_out, **kernel_summary(ks)}, gs, rs, same,
           "2*10^5 probes vs the first 10^6 build values")

    # dedup_rows (P/src/relation.cpp:71-89): 5*10^7 binary rows, ~50 % repeats.
    rows = W.random_rows(9, 50_000_000, 2, 5_000)
    ver = colog.Version.from_columns([rows[:, 0], rows[:, 1]], ctx)
    colog.dedup_rows(colog.Version.from_columns([rows[:10, 0], rows[:10, 1]], ctx))
    d, wall, ks = profile(ctx, lambda: colog.dedup_rows(ver))
    n_d = d.rows()
    del d
    sr = rows[:5_000_000]
    # Both sides build the Version from host columns inside the timed call
    # (the reference's make_version indexes every column).
    g, gs = timed(lambda: colog.dedup_rows(colog.Version.from_columns([sr[:, 0], sr[:, 1]], ctx))
                  .reconstruct_array(), 2)
    r, rs = timed(lambda: ref.dedup_rows(sr, 2))
    same = np.array_equal(np.asarray(g).reshape(-1, 2), np.asarray(r).reshape(-1, 2))
    record("dedup_rows", f"5*10^7 binary rows -> {n_d} distinct (first-occurrence order)",
           {"e2e_s": round(wall, 4), **kernel_summary(ks)}, gs, rs, same, "first 5*10^6 rows")

    # deduplicate (P/src/kernels.cpp:210-255): NEW 10^7 rows vs FULL 5*10^7.
    full_rows = W.random_rows(10, 50_000_000, 2, 20_000)
    full = colog.dedup_rows(colog.Version.from_columns([full_rows[:, 0], full_rows[:, 1]], ctx))
    new_rows = W.random_rows(11, 10_000_000, 2, 20_000)
    new = colog.dedup_rows(colog.Version.from_columns([new_rows[:, 0], new_rows[:, 1]], ctx))
    colog.deduplicate(new, full)
    flags, wall, ks = profile(ctx, lambda: colog.deduplicate(new, full))
    n_dup = int(np.count_nonzero(np.asarray(flags.flags)))
    fs = full.reconstruct_array()[:5_000_000]
    ns = new.reconstruct_array()[:1_000_000]
    g, gs = timed(lambda: np.asarray(colog.deduplicate(colog.Version.from_columns([ns[:, 0], ns[:, 1]], ctx),
                                                       colog.Version.from_columns([fs[:, 0], fs[:, 1]], ctx))
                                     .flags), 2)
    r, rs = timed(lambda: ref.deduplicate(ns, fs, 2))
    same = np.array_equal(g.astype(bool), np.asarray(r).astype(bool))
    record("deduplicate", f"NEW 10^7 vs FULL 5*10^7 binary rows -> {n_dup} already in FULL (Algorithm 2)",
           {"e2e_s": round(wall, 4), **kernel_summary(ks)}, gs, rs, same,
           "NEW 10^6 vs FULL 5*10^6")
    if args.out:
        json.dump(results, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

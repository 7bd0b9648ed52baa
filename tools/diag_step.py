"""Diagnostic (not a benchmark): C2 fixpoint wall time under the bench's two
legs — resident EDB (fv_evaluate_program_edb) with/without the live kernel
profiler and with/without keeping the previous state alive — and the host-
facts path (fv_evaluate_program). FVLOG_TRACE=1 adds per-phase host times.

    python tools/diag_step.py [reps]
"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_13051_b200 import _lib, colog, engine as E, workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = colog.Context(0)
l = ctx._lib
E._bind()
_lib.bind("fv_ctx_profile", C.c_int, [C.c_void_p, C.c_int])
_lib.bind("fv_edb_upload", C.c_int, [C.c_void_p, C.POINTER(E.fv_relation_decl), C.c_uint32,
                                     C.POINTER(E.fv_facts), C.c_uint32, C.POINTER(C.c_void_p)])
_lib.bind("fv_evaluate_program_edb", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)])
_lib.bind("fv_ctx_reserve", C.c_int, [C.c_void_p, C.c_uint64])
if os.environ.get("DIAG_RESERVE_GB"):
    t = time.perf_counter()
    _lib.check(l.fv_ctx_reserve(ctx.h, int(float(os.environ["DIAG_RESERVE_GB"]) * 2**30)), ctx.h)
    print("reserve ms", (time.perf_counter() - t) * 1000, flush=True)
edges = W.tc_powerlaw(1000, 1000, 5000, 1)
prog = E.compile_program(W.TC_PROGRAM)
decls = prog.relations()
d_arr = (E.fv_relation_decl * len(decls))(*[E.fv_relation_decl(n.encode(), a) for n, a in decls])
f_arr, nf, keep = E._facts_array({"edge": edges}, dict(decls))
edb = C.c_void_p()
_lib.check(l.fv_edb_upload(ctx.h, d_arr, len(decls), f_arr, nf, C.byref(edb)), ctx.h)


def resident():
    h = C.c_void_p()
    _lib.check(l.fv_evaluate_program_edb(ctx.h, prog.h, edb, C.byref(h)), ctx.h)
    return E.State(ctx, h.value)


def hostfacts():
    return E.evaluate_program(prog, {"edge": edges}, ctx=ctx)


def run(name, fn, profile, keep_last):
    _lib.check(l.fv_ctx_profile(ctx.h, 1 if profile else 0), ctx.h)
    last = None
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        st = fn()
        ts.append((time.perf_counter() - t) * 1000)
        el = st.elapsed_ms
        if keep_last:
            last = st
        del st
    _lib.check(l.fv_ctx_profile(ctx.h, 0), ctx.h)
    del last
    print(f"{name:40s} wall ms " + " ".join(f"{x:8.1f}" for x in ts) + f"   engine ms (last) {el:.1f}", flush=True)


for _ in range(2):
    del_ = resident()
    del del_
run("resident profile=0 keep=0", resident, False, False)
run("resident profile=1 keep=0", resident, True, False)
run("resident profile=0 keep=1", resident, False, True)
run("resident profile=1 keep=1", resident, True, True)
run("hostfacts profile=0 keep=0", hostfacts, False, False)
run("resident profile=0 keep=0 (again)", resident, False, False)

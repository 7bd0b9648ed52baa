"""TEST INFRASTRUCTURE — ORACLE, NOT PRODUCT (see oracle/__init__.py).

ctypes bindings of the C restatement (liboracle.so) and of the unmodified
reference library (oracle/_ref/libcolog_ref.so).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcolog_ref.so")
REF_BIN = os.path.join(HERE, "_ref", "colog_ref")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def build_oracle() -> None:
    src = os.path.join(HERE, "colog_oracle.c")
    if (not os.path.exists(ORACLE_SO)
            or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src)):
        subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True,
                       stdout=subprocess.DEVNULL)


class Oracle:
    """The C restatement (oracle/colog_oracle.c)."""

    def __init__(self):
        build_oracle()
        self.l = C.CDLL(ORACLE_SO)
        self.l.or_build_index.restype = C.c_uint64
        self.l.or_join_probe.restype = C.c_uint64
        self.l.or_dedup_rows.restype = C.c_uint64
        self.l.or_filter_neq.restype = C.c_uint64
        self.l.or_select_eq.restype = C.c_uint64
        self.l.or_evaluate.restype = C.c_void_p
        self.l.or_state_iterations.restype = C.c_uint64
        self.l.or_state_iterations.argtypes = [C.c_void_p]
        self.l.or_state_rows.restype = C.c_uint64
        self.l.or_state_rows.argtypes = [C.c_void_p, C.c_uint32]
        self.l.or_state_dump.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        self.l.or_state_delta.restype = C.c_uint64
        self.l.or_state_delta.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32]
        self.l.or_state_free.argtypes = [C.c_void_p]

    def build_index(self, raw):
        a = _u32(raw)
        n = a.size
        s, k, st, c = (np.empty(max(n, 1), np.uint32) for _ in range(4))
        u = self.l.or_build_index(_p(a), C.c_uint64(n), _p(s), _p(k), _p(st), _p(c))
        return s[:n], k[:u], st[:u], c[:u]

    def join_probe(self, probe, build):
        p, b = _u32(probe), _u32(build)
        s, c, m = (np.empty(max(p.size, 1), np.uint32) for _ in range(3))
        total = C.c_uint64()
        k = self.l.or_join_probe(_p(p), C.c_uint64(p.size), _p(b), C.c_uint64(b.size), _p(s), _p(c),
                                 _p(m), C.byref(total))
        return s[:k], c[:k], m[:k], total.value

    def column_join(self, probe, build):
        p, b = _u32(probe), _u32(build)
        total = C.c_uint64()
        self.l.or_join_probe(_p(p), C.c_uint64(p.size), _p(b), C.c_uint64(b.size), None, None, None,
                             C.byref(total))
        a_ids = np.empty(max(total.value, 1), np.uint32)
        b_ids = np.empty(max(total.value, 1), np.uint32)
        self.l.or_column_join(_p(p), C.c_uint64(p.size), _p(b), C.c_uint64(b.size), _p(a_ids), _p(b_ids))
        return a_ids[:total.value], b_ids[:total.value]

    def dedup_rows(self, rows, arity):
        r = _u32(rows).reshape(-1, arity)
        n = r.shape[0]
        cols = np.ascontiguousarray(r.T)
        out = np.empty((arity, max(n, 1)), np.uint32)
        k = self.l.or_dedup_rows(_p(cols), C.c_uint64(n), C.c_uint32(arity), _p(out))
        return np.ascontiguousarray(out[:, :k].T)

    def deduplicate(self, new_rows, full_rows, arity):
        nr = _u32(new_rows).reshape(-1, arity)
        fr = _u32(full_rows).reshape(-1, arity)
        flags = np.empty(max(nr.shape[0], 1), np.uint8)
        self.l.or_deduplicate(_p(np.ascontiguousarray(nr.T)), C.c_uint64(nr.shape[0]),
                              _p(np.ascontiguousarray(fr.T)), C.c_uint64(fr.shape[0]),
                              C.c_uint32(arity), _p(flags))
        return flags[:nr.shape[0]]

    def filter_neq(self, rows, arity, i, j):
        r = _u32(rows).reshape(-1, arity)
        ids = np.empty(max(r.shape[0], 1), np.uint32)
        k = self.l.or_filter_neq(_p(np.ascontiguousarray(r.T)), C.c_uint64(r.shape[0]),
                                 C.c_uint32(i), C.c_uint32(j), _p(ids))
        return ids[:k]

    def evaluate(self, arities: Sequence[int], plan_words: Sequence[int],
                 facts: Sequence[Optional[np.ndarray]]):
        """Semi-naive fixpoint over encoded plans; returns (iterations,
        [sorted rows per relation], deltas[it][rel])."""
        nrel = len(arities)
        ar = _u32(arities)
        pw = _u32(plan_words)
        cols = []
        ptrs = (C.c_void_p * max(nrel, 1))()
        ns = np.zeros(max(nrel, 1), np.uint64)
        for r in range(nrel):
            f = facts[r]
            if f is None or len(f) == 0:
                a = np.zeros((arities[r], 0), np.uint32)
            else:
                a = np.ascontiguousarray(_u32(f).reshape(-1, arities[r]).T)
            cols.append(a)
            ptrs[r] = a.ctypes.data
            ns[r] = a.shape[1]
        st = self.l.or_evaluate(C.c_uint32(nrel), _p(ar), _p(pw), C.c_uint64(pw.size), ptrs, _p(ns))
        try:
            it = self.l.or_state_iterations(st)
            rels = []
            for r in range(nrel):
                n = self.l.or_state_rows(st, r)
                out = np.empty((n, arities[r]), np.uint32)
                if n:
                    self.l.or_state_dump(st, r, out.ctypes.data)
                rels.append(out)
            deltas = [[self.l.or_state_delta(st, i, r) for r in range(nrel)] for i in range(it)]
        finally:
            self.l.or_state_free(st)
        return it, rels, deltas


class Reference:
    """The unmodified reference (oracle/_ref/libcolog_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        self.l = C.CDLL(REF_SO)
        self.l.ref_last_error.restype = C.c_char_p
        self.l.ref_free.argtypes = [C.c_void_p]

    def _err(self, rc):
        if rc != 0:
            raise RuntimeError(self.l.ref_last_error().decode())

    def _take(self, p, n, dt=np.uint32):
        if n == 0:
            self.l.ref_free(p)
            return np.zeros(0, dt)
        arr = np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), (n,)).copy()
        self.l.ref_free(p)
        return arr

    def build_index(self, raw):
        a = _u32(raw)
        s, k, st, c = (C.c_void_p() for _ in range(4))
        nu = C.c_uint64()
        self._err(self.l.ref_build_index(_p(a), C.c_uint64(a.size), C.byref(s), C.byref(k),
                                         C.byref(st), C.byref(c), C.byref(nu)))
        return (self._take(s, a.size), self._take(k, nu.value), self._take(st, nu.value),
                self._take(c, nu.value))

    def column_join(self, probe, build):
        p, b = _u32(probe), _u32(build)
        a_ids, b_ids = C.c_void_p(), C.c_void_p()
        n = C.c_uint64()
        self._err(self.l.ref_column_join(_p(p), C.c_uint64(p.size), _p(b), C.c_uint64(b.size),
                                         C.byref(a_ids), C.byref(b_ids), C.byref(n)))
        return self._take(a_ids, n.value), self._take(b_ids, n.value)

    def join_probe(self, probe, build):
        p, b = _u32(probe), _u32(build)
        s, c, m, off = (C.c_void_p() for _ in range(4))
        nm, total = C.c_uint64(), C.c_uint64()
        self._err(self.l.ref_join_probe(_p(p), C.c_uint64(p.size), _p(b), C.c_uint64(b.size),
                                        C.byref(s), C.byref(c), C.byref(m), C.byref(off),
                                        C.byref(nm), C.byref(total)))
        k = nm.value
        return (self._take(s, k), self._take(c, k), self._take(m, k),
                self._take(off, k, np.uint64), total.value)

    def dedup_rows(self, rows, arity):
        r = _u32(rows).reshape(-1, arity)
        cols = np.ascontiguousarray(r.T)
        out = C.c_void_p()
        n = C.c_uint64()
        self._err(self.l.ref_dedup_rows(_p(cols), C.c_uint64(r.shape[0]), C.c_uint32(arity),
                                        C.byref(out), C.byref(n)))
        flat = self._take(out, n.value * arity)
        return np.ascontiguousarray(flat.reshape(arity, n.value).T)

    def deduplicate(self, new_rows, full_rows, arity):
        nr = _u32(new_rows).reshape(-1, arity)
        fr = _u32(full_rows).reshape(-1, arity)
        flags = C.c_void_p()
        self._err(self.l.ref_deduplicate(_p(np.ascontiguousarray(nr.T)), C.c_uint64(nr.shape[0]),
                                         _p(np.ascontiguousarray(fr.T)), C.c_uint64(fr.shape[0]),
                                         C.c_uint32(arity), C.byref(flags)))
        return self._take(flags, nr.shape[0], np.uint8)

    def filter_neq(self, rows, arity, i, j):
        r = _u32(rows).reshape(-1, arity)
        ids = C.c_void_p()
        n = C.c_uint64()
        self._err(self.l.ref_filter_neq(_p(np.ascontiguousarray(r.T)), C.c_uint64(r.shape[0]),
                                        C.c_uint32(arity), C.c_uint32(i), C.c_uint32(j),
                                        C.byref(ids), C.byref(n)))
        return self._take(ids, n.value)

    def evaluate(self, program: str, facts: Dict[str, np.ndarray]) -> dict:
        """colog::evaluate; returns parse_report() of the text report."""
        names = list(facts)
        arrs = [np.ascontiguousarray(_u32(facts[k]).reshape(len(facts[k]), -1).T) for k in names]
        c_names = (C.c_char_p * max(len(names), 1))(*[k.encode() for k in names])
        ptrs = (C.c_void_p * max(len(names), 1))(*[a.ctypes.data for a in arrs])
        ns = (C.c_uint64 * max(len(names), 1))(*[a.shape[1] for a in arrs])
        rep = C.c_void_p()
        self._err(self.l.ref_evaluate(program.encode(), C.c_uint32(len(names)), c_names, ptrs, ns,
                                      C.byref(rep)))
        text = C.cast(rep, C.c_char_p).value.decode()
        self.l.ref_free(rep)
        return parse_report(text)

    def naive_evaluate(self, program: str) -> dict:
        rep = C.c_void_p()
        self._err(self.l.ref_naive_evaluate(program.encode(), C.byref(rep)))
        text = C.cast(rep, C.c_char_p).value.decode()
        self.l.ref_free(rep)
        return parse_report(text)


def parse_report(text: str) -> dict:
    """{'iterations': k, 'stats': [(iter, rel, delta, full, merges)],
        'relations': {name: np.ndarray rows (sorted)}}"""
    out = {"iterations": None, "stats": [], "relations": {}}
    cur = None
    arity = 0
    rows: List[List[int]] = []
    for line in text.splitlines():
        if line.startswith("iterations "):
            out["iterations"] = int(line.split()[1])
        elif line.startswith("stat "):
            _, it, rel, d, f, m = line.split()
            out["stats"].append((int(it), rel, int(d), int(f), int(m)))
        elif line.startswith("#rel "):
            if cur is not None:
                out["relations"][cur] = np.asarray(rows, np.uint32).reshape(-1, arity)
            _, cur, arity, _n = line.split()
            arity = int(arity)
            rows = []
        elif line:
            rows.append([int(x) for x in line.split("\t")])
    if cur is not None:
        out["relations"][cur] = np.asarray(rows, np.uint32).reshape(-1, max(arity, 1))
    return out

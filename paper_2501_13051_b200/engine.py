"""Program / plan / fixpoint API over the C ABI (P/include/colog/engine.hpp,
compiler.hpp, parser.hpp, runner.hpp). Parsing and planning run in the host
C++ frontend of libfvlog.so; evaluation runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import check, vp
from .colog import Context, _ctx

u32p = C.POINTER(C.c_uint32)


class fv_colref(C.Structure):
    _fields_ = [("source", C.c_uint32), ("col", C.c_uint32)]


class fv_plan_source(C.Structure):
    _fields_ = [("relation", C.c_char_p), ("arity", C.c_uint32), ("n_const_selects", C.c_uint32),
                ("const_select_cols", u32p), ("const_select_vals", u32p), ("n_self_eqs", C.c_uint32),
                ("self_eq_pairs", u32p)]


class fv_plan_join(C.Structure):
    _fields_ = [("right_source", C.c_uint32), ("left", fv_colref), ("right_col", C.c_uint32),
                ("n_residual_eq", C.c_uint32), ("residual_left", C.POINTER(fv_colref)),
                ("residual_right_col", u32p)]


class fv_plan(C.Structure):
    _fields_ = [("head_relation", C.c_char_p), ("head_arity", C.c_uint32), ("n_sources", C.c_uint32),
                ("sources", C.POINTER(fv_plan_source)), ("n_joins", C.c_uint32),
                ("joins", C.POINTER(fv_plan_join)), ("n_output_cols", C.c_uint32),
                ("output_cols", C.POINTER(fv_colref)), ("n_guards", C.c_uint32), ("guard_neq_pairs", u32p)]


class fv_relation_decl(C.Structure):
    _fields_ = [("name", C.c_char_p), ("arity", C.c_uint32)]


class fv_facts(C.Structure):
    _fields_ = [("relation", C.c_char_p), ("arity", C.c_uint32), ("n_rows", C.c_uint64),
                ("cols", C.POINTER(u32p))]


_bound = False


def _bind():
    global _bound
    if _bound:
        return
    B = _lib.bind
    B("fv_program_parse", C.c_int, [C.c_char_p, C.POINTER(vp), C.c_char_p, C.c_size_t])
    B("fv_program_free", None, [vp])
    B("fv_program_validate", C.c_int, [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_uint32)])
    B("fv_program_print", C.c_int, [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)])
    B("fv_program_num_relations", C.c_uint32, [vp])
    B("fv_program_relation", C.c_int, [vp, C.c_uint32, C.POINTER(fv_relation_decl)])
    B("fv_program_num_rules", C.c_uint32, [vp])
    B("fv_program_plan", C.c_int, [vp, C.c_uint32, C.POINTER(C.POINTER(fv_plan))])
    B("fv_program_encode", C.c_int, [vp, C.c_char_p, C.POINTER(C.c_uint32)])
    B("fv_program_dictionary_size", C.c_uint64, [vp])
    B("fv_evaluate", C.c_int, [vp, C.POINTER(fv_relation_decl), C.c_uint32, C.POINTER(fv_plan), C.c_uint32,
                               C.POINTER(fv_facts), C.c_uint32, C.POINTER(vp)])
    B("fv_evaluate_program", C.c_int, [vp, vp, C.POINTER(fv_facts), C.c_uint32, C.POINTER(vp)])
    B("fv_state_free", None, [vp])
    B("fv_state_iterations", C.c_uint64, [vp])
    B("fv_state_elapsed_ms", C.c_double, [vp])
    B("fv_state_num_relations", C.c_uint64, [vp])
    B("fv_state_relation", C.c_int, [vp, C.c_uint64, C.POINTER(C.c_char_p), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint64)])
    B("fv_state_num_stats", C.c_uint64, [vp])
    B("fv_state_stat", C.c_int, [vp, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_char_p),
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_double)])
    B("fv_state_dump_sorted", C.c_int, [vp, C.c_char_p, u32p])
    B("fv_state_fingerprint", C.c_int, [vp, C.c_char_p, C.POINTER(C.c_uint64)])
    B("fv_run", C.c_int, [C.c_int, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_char_p,
                          C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)])
    B("fv_free", None, [C.c_void_p])
    B("fv_evaluate_program_sharded", C.c_int, [vp, vp, C.POINTER(fv_facts), C.c_uint32, C.c_uint32,
                                               C.POINTER(vp)])
    B("fv_state_partition", C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)])
    B("fv_program_partition_plan", C.c_int, [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)])
    B("fv_owner", C.c_uint32, [C.c_uint32, C.c_uint32])
    B("fv_nccl_unique_id", C.c_int, [C.c_void_p])
    B("fv_ctx_set_nccl", C.c_int, [vp, C.c_int, C.c_int, C.c_void_p])
    _bound = True


# ---- plan IR in Python (RulePlan mirror) ---------------------------------------------


@dataclass
class Source:
    relation: str
    arity: int
    const_selects: List[Tuple[int, int]] = field(default_factory=list)
    self_eqs: List[Tuple[int, int]] = field(default_factory=list)


@dataclass
class Join:
    right_source: int
    left: Tuple[int, int]
    right_col: int
    residual_eq: List[Tuple[Tuple[int, int], int]] = field(default_factory=list)


@dataclass
class RulePlan:
    head_relation: str
    head_arity: int
    sources: List[Source]
    joins: List[Join]
    output_cols: List[Tuple[int, int]]
    guard_neq: List[Tuple[int, int]]


def _plan_from_c(p: fv_plan) -> RulePlan:
    srcs = []
    for s in range(p.n_sources):
        x = p.sources[s]
        srcs.append(Source(x.relation.decode(), x.arity,
                           [(x.const_select_cols[k], x.const_select_vals[k]) for k in range(x.n_const_selects)],
                           [(x.self_eq_pairs[2 * k], x.self_eq_pairs[2 * k + 1]) for k in range(x.n_self_eqs)]))
    joins = []
    for k in range(p.n_joins):
        j = p.joins[k]
        joins.append(Join(j.right_source, (j.left.source, j.left.col), j.right_col,
                          [((j.residual_left[r].source, j.residual_left[r].col), j.residual_right_col[r])
                           for r in range(j.n_residual_eq)]))
    return RulePlan(p.head_relation.decode(), p.head_arity, srcs, joins,
                    [(p.output_cols[k].source, p.output_cols[k].col) for k in range(p.n_output_cols)],
                    [(p.guard_neq_pairs[2 * k], p.guard_neq_pairs[2 * k + 1]) for k in range(p.n_guards)])


class _PlanPack:
    """Keeps the ctypes arrays behind an fv_plan array alive."""

    def __init__(self, plans: Sequence[RulePlan]):
        self.keep = []
        arr = (fv_plan * max(len(plans), 1))()
        for i, p in enumerate(plans):
            srcs = (fv_plan_source * max(len(p.sources), 1))()
            for s, x in enumerate(p.sources):
                cc = (C.c_uint32 * max(len(x.const_selects), 1))(*[c for c, _ in x.const_selects])
                cv = (C.c_uint32 * max(len(x.const_selects), 1))(*[v for _, v in x.const_selects])
                se = (C.c_uint32 * max(2 * len(x.self_eqs), 1))(*[v for pr in x.self_eqs for v in pr])
                name = x.relation.encode()
                self.keep += [cc, cv, se, name]
                srcs[s] = fv_plan_source(name, x.arity, len(x.const_selects), cc, cv, len(x.self_eqs), se)
            joins = (fv_plan_join * max(len(p.joins), 1))()
            for k, j in enumerate(p.joins):
                rl = (fv_colref * max(len(j.residual_eq), 1))(*[fv_colref(*l) for l, _ in j.residual_eq])
                rr = (C.c_uint32 * max(len(j.residual_eq), 1))(*[r for _, r in j.residual_eq])
                self.keep += [rl, rr]
                joins[k] = fv_plan_join(j.right_source, fv_colref(*j.left), j.right_col, len(j.residual_eq), rl, rr)
            outs = (fv_colref * max(len(p.output_cols), 1))(*[fv_colref(*o) for o in p.output_cols])
            gd = (C.c_uint32 * max(2 * len(p.guard_neq), 1))(*[v for g in p.guard_neq for v in g])
            head = p.head_relation.encode()
            self.keep += [srcs, joins, outs, gd, head]
            arr[i] = fv_plan(head, p.head_arity, len(p.sources), srcs, len(p.joins), joins,
                             len(p.output_cols), outs, len(p.guard_neq), gd)
        self.arr = arr


def _facts_array(facts: Dict[str, np.ndarray], arities: Dict[str, int]):
    keep = []
    blocks = []
    for rel, rows in facts.items():
        if rel not in arities:
            continue
        a = arities[rel]
        r = np.asarray(rows, dtype=np.uint32).reshape(-1, a)
        cols = [np.ascontiguousarray(r[:, j]) for j in range(a)]
        ptrs = (u32p * a)(*[c.ctypes.data_as(u32p) for c in cols])
        name = rel.encode()
        keep += [cols, ptrs, name]
        blocks.append(fv_facts(name, a, r.shape[0], ptrs))
    arr = (fv_facts * max(len(blocks), 1))(*blocks)
    return arr, len(blocks), keep


# ---- programs --------------------------------------------------------------------------


class Program:
    """Parsed + string-resolved program (parse_program + resolve_strings)."""

    def __init__(self, text: str):
        _bind()
        self.l = _lib.lib()
        h = vp()
        diag = C.create_string_buffer(1024)
        check(self.l.fv_program_parse(text.encode(), C.byref(h), diag, 1024))
        self.h = h.value
        self.text = text

    def __del__(self):
        try:
            self.l.fv_program_free(self.h)
        except Exception:
            pass

    def validate(self) -> List[str]:
        buf = C.create_string_buffer(1 << 16)
        n = C.c_uint32()
        check(self.l.fv_program_validate(self.h, buf, 1 << 16, C.byref(n)))
        return [x for x in buf.value.decode().split("\n") if x]

    def print(self) -> str:
        ln = C.c_size_t()
        check(self.l.fv_program_print(self.h, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        check(self.l.fv_program_print(self.h, buf, ln.value + 1, C.byref(ln)))
        return buf.value.decode()

    def relations(self) -> List[Tuple[str, int]]:
        out = []
        for i in range(self.l.fv_program_num_relations(self.h)):
            d = fv_relation_decl()
            check(self.l.fv_program_relation(self.h, i, C.byref(d)))
            out.append((d.name.decode(), d.arity))
        return out

    def plans(self) -> List[RulePlan]:
        out = []
        for r in range(self.l.fv_program_num_rules(self.h)):
            p = C.POINTER(fv_plan)()
            check(self.l.fv_program_plan(self.h, r, C.byref(p)))
            out.append(_plan_from_c(p.contents))
        return out

    def encode(self, s: str) -> int:
        v = C.c_uint32()
        check(self.l.fv_program_encode(self.h, s.encode(), C.byref(v)))
        return v.value

    def partition_plan(self) -> dict:
        """Static partitioning decisions of the multi-GPU engine (dist_plan)."""
        import json
        ln = C.c_size_t()
        check(self.l.fv_program_partition_plan(self.h, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        check(self.l.fv_program_partition_plan(self.h, buf, ln.value + 1, C.byref(ln)))
        return json.loads(buf.value.decode())

    # -- oracle adaptor (test infrastructure consumes this; plain data only) --
    def relation_index(self, name: str) -> int:
        return [r for r, _ in self.relations()].index(name)

    def plan_words(self) -> List[int]:
        """Encode plans as the oracle's uint32 word format (oracle/colog_oracle.c)."""
        rels = [r for r, _ in self.relations()]
        w = [len(self.plans())]
        for p in self.plans():
            w += [rels.index(p.head_relation), p.head_arity, len(p.sources)]
            for s in p.sources:
                w += [rels.index(s.relation), s.arity, len(s.const_selects)]
                for c, v in s.const_selects:
                    w += [c, v]
                w += [len(s.self_eqs)]
                for a, b in s.self_eqs:
                    w += [a, b]
            w += [len(p.joins)]
            for j in p.joins:
                w += [j.right_source, j.left[0], j.left[1], j.right_col, len(j.residual_eq)]
                for (ls, lc), rc in j.residual_eq:
                    w += [ls, lc, rc]
            w += [len(p.output_cols)]
            for s, c in p.output_cols:
                w += [s, c]
            w += [len(p.guard_neq)]
            for a, b in p.guard_neq:
                w += [a, b]
        return w

    def oracle_args(self, facts: Dict[str, np.ndarray]):
        rels = self.relations()
        arities = [a for _, a in rels]
        fl = []
        for name, a in rels:
            f = facts.get(name)
            fl.append(None if f is None else np.asarray(f, np.uint32).reshape(-1, a))
        return arities, self.plan_words(), fl


def compile_program(text: str) -> Program:
    return Program(text)


# ---- evaluation -------------------------------------------------------------------------


@dataclass
class IterationStat:
    index: int
    relation: str
    delta_rows: int
    full_rows: int
    merges: int
    elapsed_ms: float


class State:
    """EvaluationState: relations, iterations, per-iteration stats."""

    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h
        self.l = ctx._lib

    def __del__(self):
        try:
            self.l.fv_state_free(self.h)
        except Exception:
            pass

    @property
    def iterations(self) -> int:
        return int(self.l.fv_state_iterations(self.h))

    @property
    def elapsed_ms(self) -> float:
        return float(self.l.fv_state_elapsed_ms(self.h))

    def relations(self) -> Dict[str, Tuple[int, int]]:
        out = {}
        for i in range(self.l.fv_state_num_relations(self.h)):
            n, a, r = C.c_char_p(), C.c_uint32(), C.c_uint64()
            check(self.l.fv_state_relation(self.h, i, C.byref(n), C.byref(a), C.byref(r)), self.ctx.h)
            out[n.value.decode()] = (a.value, r.value)
        return out

    def rows(self, rel: str) -> int:
        return self.relations()[rel][1]

    def stats(self) -> List[IterationStat]:
        out = []
        for i in range(self.l.fv_state_num_stats(self.h)):
            it, rel, d, f, m = C.c_uint64(), C.c_char_p(), C.c_uint64(), C.c_uint64(), C.c_uint64()
            ms = C.c_double()
            check(self.l.fv_state_stat(self.h, i, C.byref(it), C.byref(rel), C.byref(d), C.byref(f), C.byref(m),
                                       C.byref(ms)), self.ctx.h)
            out.append(IterationStat(it.value, rel.value.decode(), d.value, f.value, m.value, ms.value))
        return out

    def delta_counts(self) -> Dict[str, List[int]]:
        out: Dict[str, List[int]] = {}
        for s in self.stats():
            out.setdefault(s.relation, []).append(s.delta_rows)
        return out

    def dump(self, rel: str) -> np.ndarray:
        a, n = self.relations()[rel]
        out = np.empty((n, a), np.uint32)
        if n:
            check(self.l.fv_state_dump_sorted(self.h, rel.encode(), out.ctypes.data_as(u32p)), self.ctx.h)
        return out

    def dump_into(self, rel: str, out: np.ndarray) -> int:
        """Sorted rows of `rel` written into a caller-provided C-contiguous
        u32 buffer of at least rows x arity elements (e.g. a pinned host
        tensor's numpy view); returns the row count."""
        a, n = self.relations()[rel]
        if out.dtype != np.uint32 or not out.flags["C_CONTIGUOUS"] or out.size < n * a:
            raise ValueError("dump_into: need a C-contiguous uint32 buffer of rows x arity elements")
        if n:
            check(self.l.fv_state_dump_sorted(self.h, rel.encode(), out.ctypes.data_as(u32p)), self.ctx.h)
        return n

    def fingerprint(self, rel: str) -> int:
        v = C.c_uint64()
        check(self.l.fv_state_fingerprint(self.h, rel.encode(), C.byref(v)), self.ctx.h)
        return v.value

    def derived_tuples(self) -> int:
        """Sum over iterations and relations of |DELTA|."""
        return sum(s.delta_rows for s in self.stats())


def evaluate_program(program, facts: Dict[str, np.ndarray], ctx: Optional[Context] = None) -> State:
    """evaluate(program, facts) on the GPU. `program` is text or a Program."""
    _bind()
    c = _ctx(ctx)
    prog = program if isinstance(program, Program) else Program(program)
    arities = dict(prog.relations())
    arr, n, keep = _facts_array(facts, arities)
    h = vp()
    check(c._lib.fv_evaluate_program(c.h, prog.h, arr, n, C.byref(h)), c.h)
    del keep
    return State(c, h.value)


def evaluate_program_sharded(program, facts: Dict[str, np.ndarray], world: int,
                             ctx: Optional[Context] = None) -> List[State]:
    """Hash-partitioned evaluation with `world` virtual ranks on one GPU (the
    multi-GPU code path with an in-process transport). Returns one State per
    rank holding that rank's home partition; stats are global."""
    _bind()
    c = _ctx(ctx)
    prog = program if isinstance(program, Program) else Program(program)
    arr, n, keep = _facts_array(facts, dict(prog.relations()))
    hs = (vp * world)()
    check(c._lib.fv_evaluate_program_sharded(c.h, prog.h, arr, n, world, hs), c.h)
    del keep
    return [State(c, hs[r]) for r in range(world)]


def owner(v: int, world: int) -> int:
    """Rank owning value v in a partitioned evaluation."""
    _bind()
    return int(_lib.lib().fv_owner(v, world))


def _map_process_nccl() -> None:
    """libfvlog binds the NCCL already mapped into the process (RTLD_NOLOAD)
    and only loads libnccl.so.2 itself when there is none. Under PyTorch that
    must be torch's bundled NCCL: once another libnccl.so.2 owns the soname,
    torch's CUDA library cannot load. Importing torch first maps it."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    _map_process_nccl()
    _bind()
    buf = C.create_string_buffer(128)
    check(_lib.lib().fv_nccl_unique_id(buf))
    return buf.raw


def set_nccl(ctx: Context, rank: int, world: int, uid: bytes) -> None:
    """Make later evaluations on ctx hash-partitioned over NCCL."""
    _map_process_nccl()
    _bind()
    b = C.create_string_buffer(uid, 128)
    check(ctx._lib.fv_ctx_set_nccl(ctx.h, rank, world, b), ctx.h)


def evaluate(decls: Sequence[Tuple[str, int]], plans: Sequence[RulePlan], facts: Dict[str, np.ndarray],
             ctx: Optional[Context] = None) -> State:
    """evaluate over explicit declarations and plans (the plan-level boundary)."""
    _bind()
    c = _ctx(ctx)
    d_arr = (fv_relation_decl * max(len(decls), 1))(*[fv_relation_decl(n.encode(), a) for n, a in decls])
    pack = _PlanPack(plans)
    arr, n, keep = _facts_array(facts, dict(decls))
    h = vp()
    check(c._lib.fv_evaluate(c.h, d_arr, len(decls), pack.arr, len(plans), arr, n, C.byref(h)), c.h)
    del keep, pack
    return State(c, h.value)


def fingerprint_rows(rows: np.ndarray) -> int:
    """Host restatement of the device fingerprint (fingerprint_kernel)."""
    rows = np.asarray(rows, np.uint64)
    if rows.ndim == 1:
        rows = rows.reshape(-1, 1)
    with np.errstate(over="ignore"):
        h = np.full(rows.shape[0], 0x2545F4914F6CDD1D, np.uint64)
        for j in range(rows.shape[1]):
            z = (h ^ rows[:, j]) + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            h = z ^ (z >> np.uint64(31))
        return int(h.sum(dtype=np.uint64))


def run(program_path: str, facts_dir: str, out_dir: str, stats: bool = False,
        dump: Sequence[str] = (), device: int = 0) -> Tuple[int, str, str]:
    """colog::run on the GPU: (exit code, stdout text, stderr text)."""
    _bind()
    l = _lib.lib()
    o, e = C.c_void_p(), C.c_void_p()
    rc = l.fv_run(device, program_path.encode(), facts_dir.encode(), out_dir.encode(), int(stats),
                  ",".join(dump).encode(), C.byref(o), C.byref(e))
    out = C.cast(o, C.c_char_p).value.decode() if o.value else ""
    err = C.cast(e, C.c_char_p).value.decode() if e.value else ""
    l.fv_free(o)
    l.fv_free(e)
    return rc, out, err

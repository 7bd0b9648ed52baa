"""Python mirror of the reference's relation/operator API over the C ABI.

Names, argument meaning and error behaviour follow the reference's headers
(P = /root/reference/proj):
  Column, build_index, gather_volume      P/include/colog/column.hpp
  Version, Relation, dedup_rows           P/include/colog/relation.hpp
  select_eq ... union_concat              P/include/colog/kernels.hpp
so the parity tests read like the reference's own doctest suites. Every
operator executes as sm_100a kernels through libfvlog.so; there is no host
implementation of any operator here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import check, u32p, u64p, u8p, vp

__all__ = [
    "Context", "default_context", "Column", "build_index", "gather_volume", "reset_gather_volume",
    "Version", "Relation", "dedup_rows", "has_duplicate_rows", "MatchRange", "MatchVector",
    "IdPairSet", "DupBitmap", "select_eq", "project", "join_probe_phase", "join_total_size",
    "join_offsets", "join_write_phase", "column_join", "filter_pairs_eq", "filter_neq",
    "deduplicate", "difference", "union_concat",
]


def _u32(a) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int64) if not isinstance(a, np.ndarray) else a)
    if arr.dtype != np.uint32:
        if arr.size and (arr.min() < 0 or arr.max() > 0xFFFFFFFF):
            raise OverflowError("values must fit in uint32")
        arr = arr.astype(np.uint32)
    return np.ascontiguousarray(arr)


def _p32(a: np.ndarray):
    return a.ctypes.data_as(u32p)


class Context:
    """One GPU: stream + memory pool (the reference's Executor,
    P/include/colog/parallel.hpp:19-73)."""

    def __init__(self, device: int = 0):
        self._lib = _lib.lib()
        h = vp()
        check(self._lib.fv_ctx_create(device, C.byref(h)))
        self.h = h.value
        self.device = device

    def synchronize(self):
        check(self._lib.fv_ctx_synchronize(self.h), self.h)

    def kernel_launches(self) -> int:
        return int(self._lib.fv_ctx_kernel_launches(self.h))

    def host_syncs(self) -> int:
        """Host synchronisations issued on this context so far."""
        return int(self._lib.fv_ctx_host_syncs(self.h))

    def close(self):
        if getattr(self, "h", None):
            self._lib.fv_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # Workers of the reference Executor have no analogue; kept for API parity.
    def workers(self) -> int:
        return 1


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx if ctx is not None else default_context()


class _Array:
    """Owned fv_array handle -> numpy."""

    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h

    def numpy(self) -> np.ndarray:
        l = self.ctx._lib
        n = l.fv_array_size(self.h)
        eb = l.fv_array_elem_bytes(self.h)
        dt = {1: np.uint8, 4: np.uint32, 8: np.uint64}[eb]
        out = np.empty(n, dtype=dt)
        if n:
            check(l.fv_array_read(self.h, out.ctypes.data_as(vp)), self.ctx.h)
        return out

    def __del__(self):
        try:
            self.ctx._lib.fv_array_free(self.h)
        except Exception:
            pass


def _take_array(ctx: Context, h) -> np.ndarray:
    return _Array(ctx, h).numpy()


# ---- Column -------------------------------------------------------------------------


@dataclass(frozen=True)
class MatchRange:
    start: int = 0
    count: int = 0


class Column:
    """colog::Column: raw + sorted_idx + unique_idx, resident in HBM."""

    def __init__(self, ctx: Context, h, owner=None, owned=True):
        self.ctx, self.h, self._owner, self._owned = ctx, h, owner, owned

    @staticmethod
    def build(raw: Iterable[int], ctx: Optional[Context] = None) -> "Column":
        c = _ctx(ctx)
        a = _u32(list(raw) if not isinstance(raw, np.ndarray) else raw)
        h = vp()
        check(c._lib.fv_column_build(c.h, _p32(a), a.size, C.byref(h)), c.h)
        return Column(c, h.value)

    def __del__(self):
        if self._owned:
            try:
                self.ctx._lib.fv_column_free(self.h)
            except Exception:
                pass

    def size(self) -> int:
        return int(self.ctx._lib.fv_column_size(self.h))

    def __len__(self):
        return self.size()

    def empty(self) -> bool:
        return self.size() == 0

    def raw(self) -> np.ndarray:
        n = self.size()
        out = np.empty(n, dtype=np.uint32)
        check(self.ctx._lib.fv_column_read(self.h, _p32(out), None), self.ctx.h)
        return out

    def sorted_idx(self) -> np.ndarray:
        n = self.size()
        out = np.empty(n, dtype=np.uint32)
        check(self.ctx._lib.fv_column_read(self.h, None, _p32(out)), self.ctx.h)
        return out

    def unique_arrays(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        nu = int(self.ctx._lib.fv_column_unique_count(self.h))
        k, s, c = (np.empty(nu, dtype=np.uint32) for _ in range(3))
        check(self.ctx._lib.fv_column_read_unique(self.h, _p32(k), _p32(s), _p32(c)), self.ctx.h)
        return k, s, c

    def unique_idx(self) -> Dict[int, MatchRange]:
        k, s, c = self.unique_arrays()
        return {int(a): MatchRange(int(b), int(d)) for a, b, d in zip(k, s, c)}

    def value_at(self, i: int) -> int:
        return int(self.gather([i])[0])

    def probe(self, v: int) -> Optional[MatchRange]:
        s, k, f = C.c_uint32(), C.c_uint32(), C.c_int()
        check(self.ctx._lib.fv_column_probe(self.h, v, C.byref(s), C.byref(k), C.byref(f)), self.ctx.h)
        return MatchRange(s.value, k.value) if f.value else None

    def probe_many(self, values) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        a = _u32(values)
        s, k = np.empty(a.size, np.uint32), np.empty(a.size, np.uint32)
        f = np.empty(a.size, np.uint8)
        check(self.ctx._lib.fv_column_probe_many(self.h, _p32(a), a.size, _p32(s), _p32(k),
                                                 f.ctypes.data_as(u8p)), self.ctx.h)
        return s, k, f

    def gather(self, ids) -> np.ndarray:
        a = _u32(ids)
        out = np.empty(a.size, dtype=np.uint32)
        check(self.ctx._lib.fv_column_gather(self.h, _p32(a), a.size, _p32(out)), self.ctx.h)
        return out

    def append_and_reindex(self, new_values) -> "Column":
        a = _u32(new_values)
        h = vp()
        check(self.ctx._lib.fv_column_append_and_reindex(self.h, _p32(a), a.size, C.byref(h)), self.ctx.h)
        return Column(self.ctx, h.value)


def build_index(raw, ctx: Optional[Context] = None) -> Tuple[np.ndarray, Dict[int, MatchRange]]:
    """build_index (P/src/column.cpp:17-43)."""
    c = _ctx(ctx)
    a = _u32(raw)
    n = a.size
    sidx, k, s, cnt = (np.empty(max(n, 1), dtype=np.uint32) for _ in range(4))
    nu = C.c_uint64()
    check(c._lib.fv_build_index(c.h, _p32(a), n, _p32(sidx), _p32(k), _p32(s), _p32(cnt),
                                C.byref(nu)), c.h)
    m = nu.value
    return sidx[:n], {int(k[i]): MatchRange(int(s[i]), int(cnt[i])) for i in range(m)}


def build_index_arrays(raw, ctx: Optional[Context] = None):
    """build_index returning (sorted_idx, keys, starts, counts) arrays."""
    c = _ctx(ctx)
    a = _u32(raw)
    n = a.size
    sidx, k, s, cnt = (np.empty(max(n, 1), dtype=np.uint32) for _ in range(4))
    nu = C.c_uint64()
    check(c._lib.fv_build_index(c.h, _p32(a), n, _p32(sidx), _p32(k), _p32(s), _p32(cnt),
                                C.byref(nu)), c.h)
    m = nu.value
    return sidx[:n], k[:m], s[:m], cnt[:m]


def gather_volume() -> int:
    return int(_lib.lib().fv_gather_volume())


def reset_gather_volume() -> None:
    _lib.lib().fv_reset_gather_volume()


# ---- Version / Relation -------------------------------------------------------------


class Version:
    """colog::Version: n aligned Columns; row id = position."""

    def __init__(self, ctx: Context, h, owned=True, owner=None):
        self.ctx, self.h, self._owned, self._owner = ctx, h, owned, owner

    @staticmethod
    def empty_version(arity: int, ctx: Optional[Context] = None) -> "Version":
        c = _ctx(ctx)
        h = vp()
        check(c._lib.fv_version_empty(c.h, arity, C.byref(h)), c.h)
        return Version(c, h.value)

    @staticmethod
    def decompose(rows: Sequence[Sequence[int]], arity: int, ctx: Optional[Context] = None) -> "Version":
        c = _ctx(ctx)
        rows_list = [tuple(r) for r in rows] if not isinstance(rows, np.ndarray) else rows
        for r in rows_list:
            if len(r) != arity:
                raise _lib.ArityError("decompose: row arity mismatch")
        a = _u32(np.asarray(rows_list, dtype=np.int64).reshape(-1, arity) if len(rows_list) else
                 np.zeros((0, arity), dtype=np.uint32))
        h = vp()
        check(c._lib.fv_version_decompose(c.h, arity, _p32(a), len(rows_list), C.byref(h)), c.h)
        return Version(c, h.value)

    @staticmethod
    def from_columns(cols: Sequence[Sequence[int]], ctx: Optional[Context] = None) -> "Version":
        c = _ctx(ctx)
        arrs = [_u32(col) for col in cols]
        n = arrs[0].size if arrs else 0
        for a in arrs[1:]:
            if a.size != n:
                raise _lib.ArityError("from_columns: column length mismatch")
        ptrs = (u32p * max(len(arrs), 1))(*[_p32(a) for a in arrs])
        h = vp()
        check(c._lib.fv_version_from_columns(c.h, len(arrs), ptrs, n, C.byref(h)), c.h)
        return Version(c, h.value)

    def __del__(self):
        if self._owned:
            try:
                self.ctx._lib.fv_version_free(self.h)
            except Exception:
                pass

    def arity(self) -> int:
        return int(self.ctx._lib.fv_version_arity(self.h))

    def rows(self) -> int:
        return int(self.ctx._lib.fv_version_rows(self.h))

    def empty(self) -> bool:
        return self.rows() == 0

    def col(self, j: int) -> Column:
        h = self.ctx._lib.fv_version_col(self.h, j)
        if not h:
            raise _lib.RangeError("col: column index past arity")
        return Column(self.ctx, h, owner=self, owned=False)

    def reconstruct_array(self) -> np.ndarray:
        n, k = self.rows(), self.arity()
        out = np.empty((n, k), dtype=np.uint32)
        if n and k:
            check(self.ctx._lib.fv_version_reconstruct(self.h, _p32(out)), self.ctx.h)
        return out

    def reconstruct(self) -> List[Tuple[int, ...]]:
        return [tuple(int(x) for x in r) for r in self.reconstruct_array()]

    def row(self, i: int) -> Tuple[int, ...]:
        return tuple(int(self.col(j).value_at(i)) for j in range(self.arity()))

    def append(self, extra: "Version") -> "Version":
        h = vp()
        check(self.ctx._lib.fv_version_append(self.h, extra.h, C.byref(h)), self.ctx.h)
        return Version(self.ctx, h.value)


def dedup_rows(ver: Version) -> Version:
    """dedup_rows (P/src/relation.cpp:71-89): first-occurrence order."""
    h = vp()
    check(ver.ctx._lib.fv_dedup_rows(ver.h, C.byref(h)), ver.ctx.h)
    return Version(ver.ctx, h.value)


def has_duplicate_rows(ver: Version) -> bool:
    r = C.c_int()
    check(ver.ctx._lib.fv_has_duplicate_rows(ver.h, C.byref(r)), ver.ctx.h)
    return bool(r.value)


class Relation:
    """colog::Relation with full / delta / new_rows versions."""

    def __init__(self, name: str, arity: int, ctx: Optional[Context] = None):
        c = _ctx(ctx)
        h = vp()
        check(c._lib.fv_relation_create(c.h, name.encode(), arity, C.byref(h)), c.h)
        self.ctx, self.h, self.name, self.arity = c, h.value, name, arity

    def __del__(self):
        try:
            self.ctx._lib.fv_relation_free(self.h)
        except Exception:
            pass

    def _view(self, fn) -> Version:
        return Version(self.ctx, fn(self.h), owned=False, owner=self)

    @property
    def full(self) -> Version:
        return self._view(self.ctx._lib.fv_relation_full)

    @full.setter
    def full(self, v: Version) -> None:
        # Ownership moves into the relation: detach v from Python's free.
        copy = v.append(Version.empty_version(v.arity(), self.ctx))
        check(self.ctx._lib.fv_relation_set_full(self.h, copy.h), self.ctx.h)
        copy._owned = False

    @property
    def delta(self) -> Version:
        return self._view(self.ctx._lib.fv_relation_delta)

    @property
    def new_rows(self) -> Version:
        return self._view(self.ctx._lib.fv_relation_new)

    def merge_delta(self, deduped_delta: Version) -> None:
        copy = deduped_delta.append(Version.empty_version(deduped_delta.arity(), self.ctx))
        check(self.ctx._lib.fv_relation_merge_delta(self.h, copy.h), self.ctx.h)
        copy._owned = False


# ---- RA kernels -------------------------------------------------------------------------


@dataclass
class MatchVector:
    ranges: List[MatchRange]
    matched: np.ndarray
    _h: object = field(default=None, repr=False)
    _ctx: object = field(default=None, repr=False)

    def size(self) -> int:
        return len(self.ranges)

    def __del__(self):
        if self._h is not None:
            try:
                self._ctx._lib.fv_match_free(self._h)
            except Exception:
                pass


@dataclass
class IdPairSet:
    a_ids: np.ndarray
    b_ids: np.ndarray

    def size(self) -> int:
        return int(self.a_ids.size)

    def __eq__(self, o) -> bool:
        return np.array_equal(self.a_ids, o.a_ids) and np.array_equal(self.b_ids, o.b_ids)


@dataclass
class DupBitmap:
    flags: np.ndarray

    def size(self) -> int:
        return int(self.flags.size)

    def test(self, i: int) -> bool:
        return bool(self.flags[i])


def select_eq(col: Column, v: int) -> np.ndarray:
    h = vp()
    check(col.ctx._lib.fv_select_eq(col.h, v, C.byref(h)), col.ctx.h)
    return _take_array(col.ctx, h.value)


def project(ver: Version, ids, col_map: Sequence[int]) -> Version:
    a, m = _u32(ids), _u32(list(col_map))
    h = vp()
    check(ver.ctx._lib.fv_project(ver.h, _p32(a), a.size, _p32(m), m.size, C.byref(h)), ver.ctx.h)
    return Version(ver.ctx, h.value)


def _probe_values(probe) -> np.ndarray:
    return probe.raw() if isinstance(probe, Column) else _u32(probe)


def join_probe_phase(probe_values, build: Column) -> MatchVector:
    c = build.ctx
    a = _probe_values(probe_values)
    h = vp()
    check(c._lib.fv_join_probe_phase(c.h, _p32(a), a.size, build.h, C.byref(h)), c.h)
    m = int(c._lib.fv_match_size(h.value))
    s, k, mm = (np.empty(m, np.uint32) for _ in range(3))
    if m:
        check(c._lib.fv_match_read(h.value, _p32(s), _p32(k), _p32(mm)), c.h)
    return MatchVector([MatchRange(int(x), int(y)) for x, y in zip(s, k)], mm, h.value, c)


def join_total_size(mv: MatchVector) -> int:
    t = C.c_uint64()
    check(mv._ctx._lib.fv_join_total_size(mv._h, C.byref(t)), mv._ctx.h)
    return t.value


def join_offsets(mv: MatchVector) -> np.ndarray:
    out = np.empty(max(mv.size(), 1), np.uint64)
    check(mv._ctx._lib.fv_join_offsets(mv._h, out.ctypes.data_as(u64p)), mv._ctx.h)
    return out[:mv.size()]


def join_write_phase(mv: MatchVector, offsets, total_size: int, build: Column) -> IdPairSet:
    ha, hb = vp(), vp()
    check(mv._ctx._lib.fv_join_write_phase(mv._h, build.h, C.byref(ha), C.byref(hb)), mv._ctx.h)
    a, b = _take_array(mv._ctx, ha.value), _take_array(mv._ctx, hb.value)
    assert a.size == total_size
    return IdPairSet(a, b)


def column_join(probe, build: Column) -> IdPairSet:
    """column_join (P/src/kernels.cpp:125-135): probe is a Column or values."""
    c = build.ctx
    a = _probe_values(probe)
    ha, hb = vp(), vp()
    check(c._lib.fv_column_join(c.h, _p32(a), a.size, build.h, C.byref(ha), C.byref(hb)), c.h)
    return IdPairSet(_take_array(c, ha.value), _take_array(c, hb.value))


def filter_pairs_eq(pairs: IdPairSet, col_a: Column, col_b: Column) -> IdPairSet:
    c = col_a.ctx
    a, b = _u32(pairs.a_ids), _u32(pairs.b_ids)
    ha, hb = vp(), vp()
    check(c._lib.fv_filter_pairs_eq(c.h, _p32(a), _p32(b), a.size, col_a.h, col_b.h,
                                    C.byref(ha), C.byref(hb)), c.h)
    return IdPairSet(_take_array(c, ha.value), _take_array(c, hb.value))


def filter_neq(ver: Version, col_i: int, col_j: int) -> np.ndarray:
    h = vp()
    check(ver.ctx._lib.fv_filter_neq(ver.h, col_i, col_j, C.byref(h)), ver.ctx.h)
    return _take_array(ver.ctx, h.value)


def deduplicate(new_ver: Version, full: Version) -> DupBitmap:
    h = vp()
    check(new_ver.ctx._lib.fv_deduplicate(new_ver.h, full.h, C.byref(h)), new_ver.ctx.h)
    return DupBitmap(_take_array(new_ver.ctx, h.value))


def difference(new_ver: Version, flags) -> Version:
    f = np.ascontiguousarray(np.asarray(flags.flags if isinstance(flags, DupBitmap) else flags,
                                        dtype=np.uint8))
    h = vp()
    check(new_ver.ctx._lib.fv_difference(new_ver.h, f.ctypes.data_as(u8p), f.size, C.byref(h)),
          new_ver.ctx.h)
    return Version(new_ver.ctx, h.value)


def union_concat(full: Version, delta: Version) -> Version:
    h = vp()
    check(full.ctx._lib.fv_union_concat(full.h, delta.h, C.byref(h)), full.ctx.h)
    return Version(full.ctx, h.value)

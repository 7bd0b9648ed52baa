"""GPU: the hash-partitioned (multi-GPU) engine path, run with W virtual
ranks on one B200 (threads + in-process transport; the same partitioning,
routing, count exchange, Δ forwarding and all-reduced stats as the NCCL
path). The union of the ranks' home partitions, the global per-iteration
stats and the iteration count must equal the single-GPU evaluation."""
import numpy as np
import pytest

import golden_cases
from conftest import load_golden
from paper_2501_13051_b200 import engine as E
from paper_2501_13051_b200 import workloads as W
from progen import Rng, random_edb, random_program

pytestmark = pytest.mark.gpu

CASES = [
    ("TC uniform", W.TC_PROGRAM, {"edge": W.tc_uniform(300, 1500, 1)}),
    ("TC powerlaw", W.TC_PROGRAM, {"edge": W.tc_powerlaw(4, 200, 1000, 1)}),
    ("SG tree", W.SG_PROGRAM, {"edge": W.binary_tree(6)}),
    ("CSPA", W.CSPA_PROGRAM, W.cspa_facts(3, 60, 80, 60, 3)),
    ("LUBM", W.LUBM_PROGRAM, W.lubm_facts(1, 5)),
    ("3-atom mutual", "p(x, y) :- e(x, y).\nq(x, z) :- p(x, y), e(y, z).\np(x, z) :- q(x, y), p(y, z), x != z.\n",
     {"e": W.random_rows(61, 60, 2, 20)}),
    ("constants", "a(x) :- b(3, x), c(x, x).\nd(x, y) :- b(x, y), c(y, y), x != y.\n",
     {"b": np.array([[3, 5], [3, 6], [4, 7], [5, 5]], np.uint32), "c": np.array([[5, 5], [6, 9], [7, 7]], np.uint32)}),
    ("probe on col 1", "r(x, y) :- e(x, y).\nr(x, z) :- r(x, y), e(y, z).\ns(y, x) :- r(x, y).\nt(x, z) :- s(x, y), r(y, z).\n",
     {"e": W.random_rows(7, 120, 2, 40)}),
]


def _check(single, shards, text):
    assert all(s.iterations == single.iterations for s in shards), text
    stats = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in single.stats()]
    for sh in shards:
        assert [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in sh.stats()] == stats, text
    idb = {s.relation for s in single.stats()}
    for rel, (arity, n) in single.relations().items():
        exp = single.dump(rel)
        parts = [sh.dump(rel) for sh in shards]
        if rel in idb:
            got = np.concatenate(parts) if parts else np.zeros((0, arity), np.uint32)
            assert got.shape[0] == n, (text, rel)  # home partitions are disjoint
            got = got[np.lexsort(got.T[::-1])] if got.size else got
            assert np.array_equal(got, exp), (text, rel)
            fp = sum(sh.fingerprint(rel) for sh in shards) & 0xFFFFFFFFFFFFFFFF
            assert fp == single.fingerprint(rel), (text, rel)
        else:
            for p in parts:  # EDB relations are replicated
                assert np.array_equal(p, exp), (text, rel)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("home", ["rules", "col0"])
def test_sharded_equals_single_gpu(ctx, world, home, monkeypatch):
    # "rules": home columns chosen from the recursive rules (TC: col 1,
    # exchange-free); "col0": every IDB relation homed on column 0 (routed).
    if home == "col0":
        monkeypatch.setenv("FVLOG_HOME_COL", "0")
    for name, text, facts in CASES:
        single = E.evaluate_program(text, facts, ctx=ctx)
        shards = E.evaluate_program_sharded(text, facts, world, ctx=ctx)
        _check(single, shards, name)


def test_sharded_random_programs(ctx):
    g = Rng(77)
    done = 0
    for _ in range(30):
        text, arities = random_program(g)
        prog = E.compile_program(text)
        if prog.validate():
            continue
        facts = random_edb(g, arities, 40)
        single = E.evaluate_program(prog, facts, ctx=ctx)
        _check(single, E.evaluate_program_sharded(prog, facts, 3, ctx=ctx), text)
        done += 1
    assert done > 8


def test_sharded_golden_stats(ctx):
    for case in load_golden("engine.json"):
        if case["name"] in ("SG tree depth 10", "TC uniform 2000/10000"):
            continue
        text, facts = golden_cases.program_and_facts(case)
        shards = E.evaluate_program_sharded(text, facts, 2, ctx=ctx)
        got = [(s.index, s.relation, s.delta_rows, s.full_rows, s.merges) for s in shards[0].stats()]
        assert got == [tuple(s) for s in case["stats"]], case["name"]


def test_sharded_c1_size(ctx):
    # Full C1 input across 4 virtual ranks: global stats equal single-GPU.
    edges = W.tc_uniform(10_000, 50_000, 1)
    single = E.evaluate_program(W.TC_PROGRAM, {"edge": edges}, ctx=ctx)
    shards = E.evaluate_program_sharded(W.TC_PROGRAM, {"edge": edges}, 4, ctx=ctx)
    assert sum(s.rows("reach") for s in shards) == single.rows("reach")
    assert shards[0].delta_counts() == single.delta_counts()
    fp = sum(s.fingerprint("reach") for s in shards) & 0xFFFFFFFFFFFFFFFF
    assert fp == single.fingerprint("reach")


def test_nccl_transport_single_rank(monkeypatch):
    """The NCCL transport itself (dlopen'ed libnccl, ncclCommInitRank, grouped
    ncclSend/ncclRecv, ncclAllReduce) on one GPU: a 1-rank communicator with
    the partitioned path forced on, so every routing/exchange step goes
    through NCCL (to self). Results must equal the single-GPU evaluation."""
    from paper_2501_13051_b200 import colog
    monkeypatch.setenv("FVLOG_FORCE_PARTITIONED", "1")
    ctx = colog.Context(0)
    E.set_nccl(ctx, 0, 1, E.nccl_unique_id())
    plain = colog.Context(0)
    for name, text, facts in CASES:
        single = E.evaluate_program(text, facts, ctx=plain)
        part = E.evaluate_program(text, facts, ctx=ctx)
        _check(single, [part], name)


def _nccl_rank(rank, world, uid, cases, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        from paper_2501_13051_b200 import colog, engine as E2
        ctx = colog.Context(rank)
        E2.set_nccl(ctx, rank, world, uid)
        out = []
        for name, text, facts in cases:
            st = E2.evaluate_program(text, facts, ctx=ctx)
            out.append({rel: st.dump(rel) for rel in st.relations()} | {
                "__stats": [(s.index, s.relation, s.delta_rows, s.full_rows) for s in st.stats()],
                "__iterations": st.iterations})
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, "".join(traceback.format_exception(e))))


def test_nccl_two_processes(ctx):
    """Two processes, one GPU each, one NCCL communicator: the real multi-GPU
    path (routing all-to-alls over NVLink, Δ forwarding, all-reduced stats).
    The union of the two home partitions must equal the single-GPU result."""
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    world = 2
    uid = E.nccl_unique_id()
    cases = [c for c in CASES if c[0] in ("TC uniform", "SG tree", "CSPA", "LUBM", "probe on col 1")]
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_nccl_rank, args=(r, world, uid, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r, v in res.items():
        assert not isinstance(v, str), f"rank {r}: {v}"
    for k, (name, text, facts) in enumerate(cases):
        single = E.evaluate_program(text, facts, ctx=ctx)
        stats = [(s.index, s.relation, s.delta_rows, s.full_rows) for s in single.stats()]
        idb = {s.relation for s in single.stats()}
        for r in range(world):
            assert res[r][k]["__stats"] == stats and res[r][k]["__iterations"] == single.iterations, name
        for rel in single.relations():
            if rel not in idb:
                continue
            got = np.concatenate([res[r][k][rel] for r in range(world)])
            got = got[np.lexsort(got.T[::-1])] if got.size else got
            assert np.array_equal(got, single.dump(rel)), (name, rel)

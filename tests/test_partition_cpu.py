"""CPU, world_size 2 over gloo: the hash-partitioned fixpoint protocol.

Each rank runs a host simulation of the partitioned engine that takes its
partitioning decisions from the product's planner (fv_program_partition_plan:
which copy each source reads, where intermediates are shuffled, which
derivations are replicated) and its ownership from the product's owner hash
(fv_owner). Exchanges are gloo all-to-alls, the termination/stat scalars a
gloo all-reduce. The union of the ranks' home partitions and the global
per-iteration deltas must equal the single-node oracle — so the static plan
the GPU engine executes is sound for these programs."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _alltoall(buckets, world):
    gathered = [None] * world
    dist.all_gather_object(gathered, buckets)
    me = dist.get_rank()
    out = []
    for p in range(world):
        out.extend(gathered[p][me])
    return out


def simulate(text, facts, rank, world):
    sys.path.insert(0, ROOT)
    from paper_2501_13051_b200 import engine as E
    prog = E.compile_program(text)
    plans = prog.plans()
    pp = prog.partition_plan()
    arity = dict(prog.relations())
    idb = {p.head_relation for p in plans}
    own = lambda v: E.owner(int(v), world)  # noqa: E731
    home_col = {rel: pp["relations"][rel]["home"] for rel in idb}
    state = {}
    for rel, a in arity.items():
        rows = {tuple(int(x) for x in r) for r in np.asarray(facts.get(rel, np.zeros((0, a))), np.int64).reshape(-1, a)}
        if rel in idb:
            state[rel] = {kc: {"full": {r for r in rows if own(r[kc]) == rank},
                               "delta": {r for r in rows if own(r[kc]) == rank}}
                          for kc in pp["relations"][rel]["keyset"]}
        else:
            state[rel] = {0: {"full": set(rows), "delta": set(rows)}}

    def selected(row, src):
        return all(row[c] == v for c, v in src.const_selects) and all(row[a] == row[b] for a, b in src.self_eqs)

    variants = []
    for i, p in enumerate(plans):
        ds = [s for s, src in enumerate(p.sources) if src.relation in idb]
        variants += [(i, s) for s in ds] if ds else [(i, -1)]

    stats, it = [], 0
    while True:
        pooled = {p.head_relation: [] for p in plans}
        for i, ds in variants:
            if ds < 0 and it:
                continue
            p, dp = plans[i], pp["rules"][i]
            vers = []
            for s, src in enumerate(p.sources):
                kc = dp["src_copy"][s] if src.relation in idb else 0
                vers.append(state[src.relation][kc]["delta" if s == ds else "full"])
            inter = [(r,) for r in vers[0] if selected(r, p.sources[0])]
            for k, jn in enumerate(p.joins):
                if dp["shuffle"][k]:
                    b = [[] for _ in range(world)]
                    for t in inter:
                        b[own(t[jn.left[0]][jn.left[1]])].append(t)
                    inter = _alltoall(b, world)
                src = p.sources[jn.right_source]
                index = {}
                for r in vers[jn.right_source]:
                    if selected(r, src):
                        index.setdefault(r[jn.right_col], []).append(r)
                nxt = []
                for t in inter:
                    for r in index.get(t[jn.left[0]][jn.left[1]], ()):
                        if all(t[ls][lc] == r[rc] for (ls, lc), rc in jn.residual_eq):
                            nxt.append(t + (r,))
                inter = nxt
            for t in inter:
                vals = [t[s][c] for s, c in p.output_cols]
                if any(vals[a] == vals[b] for a, b in p.guard_neq):
                    continue
                head = tuple(vals[: p.head_arity])
                h = home_col[p.head_relation]
                if dp["replicated_out"] and own(head[h]) != rank:
                    continue
                if dp["local_out"]:
                    # the plan claims the row was derived at its owner
                    assert own(head[h]) == rank, (p.head_relation, head)
                pooled[p.head_relation].append(head)
        counts = []
        for rel in sorted(pooled):
            b = [[] for _ in range(world)]
            h = home_col[rel]
            for row in pooled[rel]:
                b[own(row[h])].append(row)
            home = state[rel][h]
            new = set(_alltoall(b, world)) - home["full"]
            home["full"] |= new
            home["delta"] = new
            for kc in pp["relations"][rel]["keyset"]:
                if kc == h:
                    continue
                b = [[] for _ in range(world)]
                for row in new:
                    b[own(row[kc])].append(row)
                got = set(_alltoall(b, world))
                state[rel][kc]["full"] |= got
                state[rel][kc]["delta"] = got
            counts += [len(new), len(home["full"])]
        import torch
        t = torch.tensor(counts, dtype=torch.int64)
        dist.all_reduce(t)
        g = t.tolist()
        for k, rel in enumerate(sorted(pooled)):
            stats.append((it, rel, g[2 * k], g[2 * k + 1]))
        if not any(g[0::2]):
            break
        it += 1
    home = {rel: sorted(st[home_col[rel]]["full"]) for rel, st in state.items() if rel in idb}
    return {"iterations": it + 1, "stats": stats, "home": home}


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        try:
            q.put((rank, [simulate(text, facts, rank, world) for _, text, facts in cases]))
        except Exception as e:  # noqa: BLE001 — reported by the parent
            import traceback
            q.put((rank, "".join(traceback.format_exception(e))))
    finally:
        dist.destroy_process_group()


def _cases():
    sys.path.insert(0, ROOT)
    from paper_2501_13051_b200 import workloads as W
    return [
        ("TC", W.TC_PROGRAM, {"edge": W.tc_uniform(60, 200, 1)}),
        ("SG", W.SG_PROGRAM, {"edge": W.binary_tree(4)}),
        ("CSPA", W.CSPA_PROGRAM, W.cspa_facts(2, 20, 25, 20, 3)),
        ("col-1 probes", "r(x, y) :- e(x, y).\nr(x, z) :- r(x, y), e(y, z).\ns(y, x) :- r(x, y).\n"
                         "t(x, z) :- s(x, y), r(y, z).\n", {"e": W.random_rows(7, 60, 2, 25)}),
        ("3-atom", "p(x, y) :- e(x, y).\nq(x, z) :- p(x, y), e(y, z).\np(x, z) :- q(x, y), p(y, z), x != z.\n",
         {"e": W.random_rows(61, 40, 2, 15)}),
    ]


def test_partitioned_protocol_gloo_world2():
    from oracle.bind import Oracle
    from paper_2501_13051_b200 import engine as E
    cases = _cases()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for r, res in results.items():
        assert not isinstance(res, str), f"rank {r}: {res}"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    oracle = Oracle()
    for k, (name, text, facts) in enumerate(cases):
        prog = E.compile_program(text)
        it, rels, deltas = oracle.evaluate(*prog.oracle_args(facts))
        names = [r for r, _ in prog.relations()]
        r0, r1 = results[0][k], results[1][k]
        assert r0["iterations"] == r1["iterations"] == it, name
        assert r0["stats"] == r1["stats"], name
        for (i, rel, d, _f) in r0["stats"]:
            assert d == deltas[i][names.index(rel)], (name, i, rel)
        for rel, rows0 in r0["home"].items():
            rows1 = r1["home"][rel]
            assert not set(rows0) & set(rows1), (name, rel)  # disjoint home partitions
            exp = {tuple(int(x) for x in r) for r in rels[names.index(rel)].tolist()}
            assert set(rows0) | set(rows1) == exp, (name, rel)


def test_home_columns_make_tc_exchange_free():
    """The planner's home column for right-linear TC is column 1 and its
    recursive rule is local_out (no routing); left-linear TC keeps column 0,
    also local; SG has no carried column and routes (column 0)."""
    sys.path.insert(0, ROOT)
    from paper_2501_13051_b200 import engine as E, workloads as W
    pp = E.compile_program(W.TC_PROGRAM).partition_plan()
    assert pp["relations"]["reach"]["home"] == 1
    assert pp["relations"]["reach"]["keyset"] == [1]  # no partition copies
    assert all(r["local_out"] or r["replicated_out"] for r in pp["rules"])
    left = E.compile_program("reach(x, y) :- edge(x, y).\nreach(x, z) :- reach(x, y), edge(y, z).\n")
    pl = left.partition_plan()
    assert pl["relations"]["reach"]["home"] == 0 and pl["rules"][1]["local_out"]
    sg = E.compile_program(W.SG_PROGRAM).partition_plan()
    assert sg["relations"]["sg"]["home"] == 0
    assert any(not r["local_out"] and not r["replicated_out"] for r in sg["rules"])

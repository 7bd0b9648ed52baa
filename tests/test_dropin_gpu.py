"""The drop-in proof: the reference's OWN test suites, compiled unmodified
against its own headers, linked with the colog-on-fvlog shim
(integration/colog_fvlog) instead of P/src/{column,relation,kernels,engine}.cpp,
run their assertions against the B200 path (integration/Makefile).

Suites: P/tests/column_test.cpp, relation_test.cpp, kernels_test.cpp,
engine_test.cpp (56 doctest cases: the worked examples of Algorithm 1, the
nested-loop join oracle on random and skewed columns, Algorithm 2 against the
naive check, semi-naive == naive on random programs, ...). Plus the reference's
CLI ctests (P/tests/CMakeLists.txt:25-35) through its own runner.cpp on the
shim. The binaries are built in this container (they need /root/reference) and
travel to the GPU box with the snapshot; the box never reads /root/reference.
"""
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")
SUITES = {"column": 11, "relation": 8, "kernels": 18, "engine": 12}


def _binary(name):
    p = os.path.join(BUILD, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (integration/Makefile needs /root/reference; run __graft_entry__.build())")
    return p


def _linked_libfvlog(p):
    out = subprocess.run(["ldd", p], capture_output=True, text=True).stdout
    return "libfvlog.so" in out


def test_dropin_binaries_link_libfvlog():
    """(CPU) every drop-in binary resolves libfvlog.so, and none carries the
    reference's own hot-path objects."""
    for name in [f"{s}_test" for s in SUITES] + ["colog_fvlog"]:
        p = _binary(name)
        assert _linked_libfvlog(p), name
        syms = subprocess.run(["nm", "-C", p], capture_output=True, text=True).stdout
        # the shim's definitions, not the reference's: colog::Column::build
        # calls fv_build_index
        assert "fv_build_index" in syms, name
        if name in ("engine_test", "colog_fvlog"):
            assert "fv_evaluate" in syms, name


def _run_suite(binary):
    """Run a doctest suite with one child process per case; returns
    ({case: (status, assertions)}, summary line)."""
    r = subprocess.run([binary], capture_output=True, text=True, timeout=1800,
                       env=dict(os.environ, DOCTEST_MINI_FORK="1"))
    cases = {}
    for line in r.stdout.splitlines():
        m = re.match(r"\[doctest\] case: (\S+) (\d+) (.*)$", line)
        if m:
            cases[m.group(3)] = (m.group(1), int(m.group(2)))
    summary = [l for l in r.stdout.splitlines() if l.startswith("[doctest] test cases")]
    assert summary, f"exit {r.returncode}\n" + r.stdout + r.stderr[-6000:]
    return cases, summary[-1], r.stderr


def test_reference_suites_on_the_reference_build():
    """(CPU) the baseline: the same suites linked against the reference's own
    objects. In this environment the reference passes column/relation/kernels
    and 10 of 12 engine cases: its random-rule generator indexes an empty
    vector (P/tests/engine_test.cpp:83, a crash) and its residual-equality
    defect (P/src/kernels.cpp:155) fails semi-naive == naive."""
    for suite, n in SUITES.items():
        cases, _, _ = _run_suite(_binary(f"{suite}_test_ref"))
        assert len(cases) == n, suite
        bad = {c: st for c, (st, _) in cases.items() if st != "ok"}
        if suite == "engine":
            assert set(bad) <= {"executing a compiled plan once equals the oracle's single step",
                                "semi-naive evaluation equals naive evaluation on random programs"}, bad
        else:
            assert not bad, (suite, bad)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suite_on_gpu(suite):
    """Every case the reference passes passes on fvlog with the same number of
    assertions; cases the reference fails on its own defect pass on fvlog;
    the generator crash (inside the test's own code) is the only allowed
    non-pass, and only where the reference crashes too."""
    ref, _, _ = _run_suite(_binary(f"{suite}_test_ref"))
    got, summary, err = _run_suite(_binary(f"{suite}_test"))
    assert set(got) == set(ref) and len(got) == SUITES[suite], summary
    for case, (st, n) in ref.items():
        gst, gn = got[case]
        if st == "ok":
            assert gst == "ok" and gn == n, (case, got[case], ref[case], err[-3000:])
        elif st == "failed":
            assert gst == "ok", (case, got[case], err[-3000:])
        else:  # crashed inside the reference's test generator
            assert gst in ("ok", st), (case, got[case])


@pytest.mark.gpu
def test_reference_cli_ctests_on_gpu():
    cli = _binary("colog_fvlog")
    data = os.path.join(ROOT, "tests", "data")
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([cli, "run", os.path.join(data, "tc.dl"), "--facts", os.path.join(data, "path10"),
                            "--out", d, "--dump", "reach"], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "rel=reach rows=45" in r.stdout, r.stdout + r.stderr
        with open(os.path.join(d, "reach.tsv")) as f:
            rows = [tuple(map(int, l.split("\t"))) for l in f.read().splitlines()]
        assert sorted(rows) == sorted((i, j) for i in range(10) for j in range(i + 1, 10))
        r = subprocess.run([cli, "run", os.path.join(data, "invalid_unbound.dl"), "--facts",
                            os.path.join(data, "path10"), "--out", d], capture_output=True, text=True, timeout=300)
        assert r.returncode != 0

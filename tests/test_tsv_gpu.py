"""GPU: facts files and dumps — the run() surface of
P/src/io.cpp:44-124 and P/src/runner.cpp:26-92 with integer-mode facts parsed
and dumps formatted on the device. Every case runs the fvlog CLI and the
unmodified reference (oracle/_ref/colog_ref, the checker) on the same files
and compares exit status, summary lines, error messages and dump bytes."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from conftest import ROOT
from paper_2501_13051_b200 import workloads as W

pytestmark = pytest.mark.gpu

CLI = os.path.join(ROOT, "paper_2501_13051_b200", "fvlog")
REF = os.path.join(ROOT, "oracle", "_ref", "colog_ref")


def _run(binary, prog, facts, out, dump):
    args = [binary, "run", prog, "--facts", facts, "--out", out]
    if dump:
        args += ["--dump", ",".join(dump)]
    r = subprocess.run(args, capture_output=True, text=True)
    lines = [l for l in r.stdout.splitlines() if l.startswith("rel=")]
    it = [l.split()[0] for l in r.stdout.splitlines() if l.startswith("iterations=")]
    return r.returncode, lines, it, r.stderr.strip()


def _compare(program, files, dump, expect_ok=True):
    """files: {rel: raw TSV text}; runs both engines; returns (rc, stderr)."""
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref not built")
    with tempfile.TemporaryDirectory() as d:
        prog = os.path.join(d, "p.dl")
        open(prog, "w").write(program)
        facts = os.path.join(d, "facts")
        os.makedirs(facts)
        for rel, text in files.items():
            with open(os.path.join(facts, rel + ".tsv"), "wb") as fh:
                fh.write(text.encode() if isinstance(text, str) else text)
        got = _run(CLI, prog, facts, os.path.join(d, "a"), dump)
        exp = _run(REF, prog, facts, os.path.join(d, "b"), dump)
        assert (got[0] == 0) == (exp[0] == 0), (got, exp)
        assert got[1] == exp[1] and got[2] == exp[2], (got, exp)
        if exp[0] != 0:
            # Same message; the path prefix is the same file.
            assert got[3] == exp[3], (got[3], exp[3])
        for rel in dump if exp[0] == 0 else []:
            a = open(os.path.join(d, "a", rel + ".tsv"), "rb").read()
            b = open(os.path.join(d, "b", rel + ".tsv"), "rb").read()
            assert a == b, rel
        assert (got[0] == 0) == expect_ok
        return got


def test_integer_facts_edge_cases():
    # CRLF, empty lines (also "\r" alone), leading zeros, duplicates, no
    # trailing newline, u32 max.
    text = "1\t2\r\n\n2\t3\n\r\n0003\t4\n1\t2\n4\t4294967295\n4294967295\t0"
    _compare(W.TC_PROGRAM, {"edge": text}, ["reach", "edge"])


def test_unary_and_ternary_relations():
    prog = "a(x) :- b(x, y, z), c(z).\nd(x, y, z) :- b(x, y, z), a(x).\n"
    b = "\n".join(f"{i % 7}\t{i}\t{i % 3}" for i in range(60)) + "\n"
    c = "0\n2\n"
    _compare(prog, {"b": b, "c": c}, ["a", "d"])


@pytest.mark.parametrize("bad, why", [
    ("1\t2\n3\tx\n", "non-integer field after an integer first line"),
    ("1\t2\n3\t4\t5\n", "too many fields"),
    ("1\t2\n\n3\n", "too few fields"),
    ("1\t2\n3\t4294967296\n", "value above u32"),
    ("1\t2\n3\t-1\n", "sign"),
    ("1\t2\n3\t+1\n", "plus sign"),
    ("1\t2\n3\t 1\n", "leading space"),
    ("1\t2\n3\t\n", "empty field"),
    ("1\t2\n3\t99999999999999999999999\n", "beyond u64"),
])
def test_integer_facts_errors_match_reference(bad, why):
    rc, _, _, err = _compare(W.TC_PROGRAM, {"edge": bad}, [], expect_ok=False)
    assert rc != 0 and err, why


def test_first_bad_line_is_reported():
    # Several bad lines: the reference stops at the first one (line 3).
    _compare(W.TC_PROGRAM, {"edge": "1\t2\n\nx\t1\n1\t2\t3\n"}, [], expect_ok=False)


def test_dictionary_mode_files_stay_on_the_host_path():
    text = "alice\tbob\nbob\tcarol\ncarol\t7\n"
    _compare(W.TC_PROGRAM, {"edge": text}, ["reach"])


def test_large_integer_file_roundtrip():
    e = W.tc_uniform(2000, 10000, 5)
    text = "\n".join(f"{a}\t{b}" for a, b in e.tolist()) + "\n"
    _compare(W.TC_PROGRAM, {"edge": text}, ["reach", "edge"])


@pytest.mark.parametrize("files", [
    {"edge": ""},                      # empty file
    {"edge": "\n\r\n\n"},              # only blank lines
    {},                                # no facts file at all
    {"edge": "1\t2\n", "reach": "5\t6\n7\t7\n"},   # IDB relation seeded from a file
])
def test_empty_and_seeded_inputs(files):
    _compare(W.TC_PROGRAM, files, ["reach", "edge"])


def test_relation_without_rules_or_facts():
    # A relation declared only in a body: empty EDB, empty result, 1 iteration.
    _compare("a(x, y) :- b(x, y), c(y).\n", {"b": "1\t2\n"}, ["a", "b", "c"])

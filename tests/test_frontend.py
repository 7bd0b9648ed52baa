"""CPU: the host frontend (parse / validate / print)
against the unmodified reference. Each invalid program goes through both the
reference CLI (oracle/_ref/colog_ref, which prints
"<path>:<line>:<col>: <message>" per diagnostic, P/src/runner.cpp:36-47) and
fvlog's parser/validator (host code in libfvlog.so, no GPU needed); the
diagnostic lines must be identical. Cases follow P/tests/frontend_test.cpp:42-89
plus a few more syntax errors."""
import os
import subprocess
import tempfile

import pytest

from conftest import ROOT
from paper_2501_13051_b200 import _lib
from paper_2501_13051_b200 import engine as E

REF = os.path.join(ROOT, "oracle", "_ref", "colog_ref")

INVALID = [
    "a(x) :- b(x, y, z). b(u, v).",                    # arity mismatch (parse)
    "a(x) :- b(x), !c(x).",                           # negation
    "a(x) :- b(x, y), x < y.",                        # only != guards
    "a(x, y).",                                       # non-ground fact
    "a(4294967296).",                                 # constant beyond 32 bits
    "Reach(x, y) :- edge(x, y).",                     # uppercase relation
    "edge(1, 2).\nreach(x y) :- edge(x, y).",         # syntax error, line 2
    "reach(x, y) :- edge(x, y)\n",                    # missing '.'
    "reach(x, z) :- edge(x, y).",                     # range restriction
    "a(x, y) :- b(x), c(y).",                         # cross product
    "a(x) :- b(x), x != w.",                          # unbound guard variable
    "a(x) :- b(x), b(x, x).",                         # arity mismatch (body)
    "a(\"s\", x) :- b(x).",                           # head constant
    "a(x) :- .",                                      # empty body
    "a(x) :- b(x), c(x) d(x).",                       # missing comma
]


def _reference_diagnostics(text):
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "p.dl")
        open(p, "w").write(text)
        os.makedirs(os.path.join(d, "f"))
        r = subprocess.run([REF, "run", p, "--facts", os.path.join(d, "f"), "--out", os.path.join(d, "o")],
                           capture_output=True, text=True)
        assert r.returncode != 0
        return [l[len(p) + 1:] for l in r.stderr.splitlines() if l.startswith(p + ":")]


def _fvlog_diagnostics(text):
    try:
        prog = E.Program(text)
    except _lib.DiagnosticError as e:
        return [str(e)]
    return prog.validate()


@pytest.mark.parametrize("text", INVALID)
def test_diagnostics_match_reference(text):
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref not built")
    exp = _reference_diagnostics(text)
    assert exp, "reference accepted the program"
    assert _fvlog_diagnostics(text) == exp


def test_print_reparse_roundtrip():
    text = ('% family facts\nparentof("Alice", "Bob").\nparentof("Larry", "Alice").\nedge(1, 2).\n'
            "ancestor(x, y) :- parentof(x, y).\nancestor(x, z) :- parentof(x, y), ancestor(y, z).\n"
            "sg(x, y) :- edge(p, x), edge(p, y), x != y.\n")
    p = E.Program(text)
    q = E.Program(p.print())
    assert q.print() == p.print()
    assert q.relations() == p.relations()

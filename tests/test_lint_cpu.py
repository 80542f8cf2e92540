"""Static checks of the host code (no GPU): every name a function reads must be bound somewhere.

pyflakes is not installed in this image, so this is a small undefined-name check on top of the
standard library's ``symtable``: a name a function uses but does not bind resolves to an enclosing
function, the module, or builtins -- otherwise it is the kind of NameError that once sent every
N>1 bench run of the peer-slab path to the fallback (bench.py make_peer_step).
"""
from __future__ import annotations

import builtins
import os
import symtable

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FILES = ["bench.py", "__graft_entry__.py"] + sorted(
    os.path.join("paper_2106_15869_b200", f) for f in os.listdir(os.path.join(ROOT, "paper_2106_15869_b200"))
    if f.endswith(".py")) + sorted(
    os.path.join("tests", f) for f in os.listdir(os.path.join(ROOT, "tests")) if f.endswith(".py")) + sorted(
    os.path.join(d, f) for d in ("tools", "oracle", os.path.join("tests", "golden"))
    for f in os.listdir(os.path.join(ROOT, d)) if f.endswith(".py"))


def _undefined(path):
    src = open(os.path.join(ROOT, path)).read()
    top = symtable.symtable(src, path, "exec")
    module_names = {s.get_name() for s in top.get_symbols() if s.is_assigned() or s.is_imported()}
    known = module_names | set(dir(builtins)) | {"__file__", "__name__", "__doc__"}
    bad = []

    def walk(tab, enclosing):
        bound_here = {s.get_name() for s in tab.get_symbols()
                      if s.is_assigned() or s.is_imported() or s.is_parameter()}
        for s in tab.get_symbols():
            name = s.get_name()
            if tab.get_type() == "function" and s.is_referenced() and s.is_global() and not s.is_declared_global():
                if name not in known and name not in enclosing:
                    bad.append(f"{path}: {tab.get_name()}() reads undefined name {name!r} (line {tab.get_lineno()})")
        inner = enclosing | (bound_here if tab.get_type() == "function" else set())
        for ch in tab.get_children():
            walk(ch, inner)

    walk(top, set())
    return bad


@pytest.mark.parametrize("path", FILES)
def test_no_undefined_names(path):
    assert _undefined(path) == []


def test_checker_catches_a_closure_name_error(tmp_path):
    p = tmp_path / "x.py"
    p.write_text("def f():\n    def g():\n        return undefined_thing + 1\n    return g\n")
    rel = os.path.relpath(p, ROOT)
    assert any("undefined_thing" in m for m in _undefined(rel))

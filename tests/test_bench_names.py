"""Static check of bench.py and the tools it shares code with: every name a
function reads as a global exists at module level (catches a stale variable
in a code path only a GPU run executes, e.g. main_c1)."""

import builtins
import importlib
import os
import symtable
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _undefined_globals(path, module):
    src = open(path).read()
    table = symtable.symtable(src, path, "exec")
    known = set(dir(module)) | set(dir(builtins))
    missing = []

    def walk(t):
        if t.get_type() == "function":
            for s in t.get_symbols():
                if s.is_referenced() and s.is_global() and s.get_name() not in known:
                    missing.append((t.get_name(), s.get_name()))
        for c in t.get_children():
            walk(c)
    walk(table)
    return missing


@pytest.mark.parametrize("name", ["bench", "tools.c2_diag", "tools.c4_probe", "tools.gemm_shapes"])
def test_no_undefined_globals(name):
    pytest.importorskip("torch")
    mod = importlib.import_module(name)
    assert _undefined_globals(mod.__file__, mod) == []

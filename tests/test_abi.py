"""The C-ABI library loads and exports every entry point include/tally_b200.h
declares; no compute calls (runs without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2410_07381_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tally_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_ ]+\**\s+\**(tally_[a-z0-9_]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("tally_init", "tally_kernel_create", "tally_launch", "tally_preempt",
                 "tally_launch_query", "tally_runner_create", "tally_runner_run",
                 "tally_runner_fire", "tally_runner_on_event", "tally_runner_filter"):
        assert must in names
    assert len(names) >= 35


def test_every_declared_symbol_is_exported():
    raw = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(raw, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(declared_functions()) == set(_lib.exported_symbols())


def test_abi_version_and_kinds():
    assert _lib.lib.tally_abi_version() == 2
    names = [_lib.lib.tally_kernel_kind_name(i).decode()
             for i in range(_lib.lib.tally_kernel_kind_count())]
    for k in ("vecadd_i64", "vecadd_f32", "rowsum_f32"):
        assert k in names


def test_no_silent_cpu_path_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    info = _lib.c_gpu_info()
    rc = _lib.lib.tally_init(0, ctypes.byref(info))
    assert rc == _lib.ENODEV
    assert "device" in _lib.last_error().lower()
    with pytest.raises(ValueError):
        _lib.check(_lib.lib.tally_launch(0, 0, None, None), "launch before init")


def test_error_mapping():
    with pytest.raises(_lib.TransformError):
        _lib.check(_lib.ETRANSFORM, "x")
    with pytest.raises(ValueError):
        _lib.check(_lib.EINVAL, "x")
    with pytest.raises(_lib.TallyError):
        _lib.check(_lib.ECUDA, "x")

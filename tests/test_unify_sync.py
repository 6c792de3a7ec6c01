"""The product's unified-synchronisation pass (paper_2410_07381_b200.transforms,
ref transforms.py:200-288) against the reference's own output on the 200
acceptance-gate kernels and the witness, plus the IR-JIT's lowering of the
returned-count update to one shared atomic (CPU only)."""

import pytest

from paper_2410_07381_b200 import transforms as T
from paper_2410_07381_b200.irjit import codegen, normalize, ptb_safe


def test_unify_equals_reference_on_gate_kernels(gold):
    for c in gold("acceptance")["cases"]:
        u = T.unify_synchronization(normalize(c["kernel"]))
        assert u == normalize(c["unified"]), c["seed"]
        assert T.has_unified_sync_shape(u) and ptb_safe(u)


def test_unify_witness_matches_reference(gold):
    w = gold("transforms")["witness"]
    raw = normalize(w["kernel"])
    assert not ptb_safe(raw)
    u = T.unify_synchronization(raw)
    assert T.has_unified_sync_shape(u) and ptb_safe(u)
    assert u["regs"] == raw["regs"] + 4 and u["shared"] == raw["shared"] + 1


def test_unify_fresh_labels_avoid_collisions():
    k = {"name": "k", "params": ("__usync",), "nparams": 1, "grid": (1, 1, 1), "block": (2, 1, 1),
         "regs": 2, "shared": 0, "dependent": False,
         "body": [("CONST", (("r", 1), ("i", 1)), "__uret"), ("BAR_SYNC", (), None),
                  ("CONST", (("r", 1), ("i", 2)), None), ("RET", (), None)]}
    u = T.unify_synchronization(k)
    labels = [lab for _o, _a, lab in u["body"] if lab is not None]
    assert len(labels) == len(set(labels))
    assert "__usync_1" in labels and "__uret_2" in labels


def test_jit_lowers_the_returned_count_to_one_atomic(gold):
    c = gold("acceptance")["cases"][0]
    u = T.unify_synchronization(normalize(c["kernel"]))
    src = codegen(u, "ns")
    n_ret = sum(op == "RET" for op, _a, _l in normalize(c["kernel"])["body"])
    assert src.count("atomicAdd(reinterpret_cast<unsigned long long*>(sh + ") == n_ret

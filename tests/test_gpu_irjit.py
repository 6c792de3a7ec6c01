"""IR-JIT on the B200: reference IR kernels compiled to CUDA (NVRTC, sm_100a)
and run in all three Tally shapes, bit-exact against the reference's golden
memory images -- acceptance criterion 1 (ref
tests/test_acceptance.py:98-120) executed on the device.  Needs a B200."""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import kernel_ir as ki   # noqa: E402
from oracle import rewrites as rw    # noqa: E402


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_07381_b200 as P
    from paper_2410_07381_b200 import irjit, kernels
    P.B200Device.get(0)
    return P, irjit, kernels.Stream(high_priority=False)


def _run(jk, memory, args, launch):
    mem = torch.tensor(memory, dtype=torch.int64, device="cuda")
    fault = torch.zeros(1, dtype=torch.int64, device="cuda")
    dk = jk.bind(mem, fault, args)
    torch.cuda.synchronize()
    states = launch(dk)
    torch.cuda.synchronize()
    out = mem.cpu().tolist(), int(fault.item()), states
    dk.close()
    return out


def test_golden_interpreter_cases_on_device(env, gold):
    P, irjit, s = env
    checked = 0
    for case in gold("ir")["cases"]:
        e = case["expect"]
        if e["status"] not in ("Completed", "MemoryFault"):
            continue
        jk = irjit.JitKernel(case["kernel"])
        mem, fault, _ = _run(jk, case["memory"], case["args"], lambda dk: [dk.original(s).wait()])
        if e["status"] == "Completed":
            assert fault == 0, case["name"]
            assert mem == e["memory"], case["name"]
        else:
            assert fault & 1, case["name"]
        checked += 1
    assert checked >= 60


def test_step_limit_faults_instead_of_hanging(env, gold):
    P, irjit, s = env
    case = next(c for c in gold("ir")["cases"] if c["name"] == "steplimit")
    jk = irjit.JitKernel(case["kernel"])
    _mem, fault, _ = _run(jk, case["memory"] or [0], case["args"], lambda dk: [dk.original(s).wait()])
    assert fault & 2


def test_sliced_and_ptb_equivalence_on_device(env, gold):
    """40 reference random kernels x {1/2, 1/4, 1/8, 1/total} (rectangular,
    largest-axis plans) x PTB workers {1, 2, 4, 8}: payload equals the
    reference's base image; every logical block exactly once."""
    P, irjit, s = env
    for rec in gold("transforms")["equiv"]:
        kd = rec["kernel"]
        jk = irjit.JitKernel(kd)
        base = rec["base"]["memory"]
        total = kd["grid"][0] * kd["grid"][1] * kd["grid"][2]
        for f in (Fraction(1, 2), Fraction(1, 4), Fraction(1, 8), Fraction(1, total)):
            plan = P.slice_plan(None, f, grid=kd["grid"])
            ec = torch.zeros(total, dtype=torch.int64, device="cuda")
            mem, fault, _ = _run(jk, rec["memory"], rec["args"], lambda dk: [
                dk.sliced_rect(s, o, g, exec_count=ec).wait() for o, g in plan])
            assert fault == 0 and mem == base, (rec["seed"], f)
            assert bool((ec == 1).all())
        for w in (1, 2, 4, 8):
            ec = torch.zeros(total, dtype=torch.int64, device="cuda")
            mem, fault, st = _run(jk, rec["memory"], rec["args"],
                                  lambda dk: [dk.ptb(s, w, exec_count=ec).wait()])
            assert fault == 0 and mem == base, (rec["seed"], w)
            assert st[0].task_counter >= total
            assert bool((ec == 1).all())


def test_preempt_at_every_counter_then_resume_on_device(env, gold):
    """ref tests/test_transforms.py:185-219 on device: the JIT-compiled kernel,
    PTB(4), preempted when the counter reaches c, resumed from the persisted
    counter; payload equals the reference's uninterrupted image."""
    P, irjit, s = env
    g = gold("transforms")["preempt"]
    k = ki.kernel_from_json(g["kernel"])
    payload = len(g["memory"]) - 2
    expect = g["uninterrupted"]["memory"][:payload]
    jk = irjit.JitKernel(k)
    for c in range(0, 18):
        ec = torch.zeros(16, dtype=torch.int64, device="cuda")

        def chain(dk):
            first = dk.ptb(s, 4, preempt_at=c, exec_count=ec).wait()
            out = [first]
            if first.parked:
                out.append(dk.ptb(s, 4, start_count=first.task_counter, exec_count=ec).wait())
            return out
        mem, fault, sts = _run(jk, g["memory"][:payload], g["args"], chain)
        assert fault == 0
        assert mem == expect, c
        assert sts[0].task_counter >= min(c, 16) if c else sts[0].task_counter >= 16
        assert bool((ec == 1).all())


def test_unified_sync_witness_on_device(env, gold):
    P, irjit, s = env
    w = gold("transforms")["witness"]
    raw = ki.kernel_from_json(w["kernel"])
    jk = irjit.JitKernel(raw)
    assert not jk.ptb_ok
    mem = torch.zeros(4, dtype=torch.int64, device="cuda")
    fault = torch.zeros(1, dtype=torch.int64, device="cuda")
    dk = jk.bind(mem, fault, ())
    with pytest.raises(P.TransformError):
        dk.ptb(s, 1)
    dk.close()
    uni = irjit.JitKernel(rw.unify_synchronization(raw))
    assert uni.ptb_ok
    mem, fault, _ = _run(uni, [0, 0, 0, 0], (), lambda dk: [dk.ptb(s, 1).wait()])
    assert mem == [7, 7, 7, 7] == w["unified"]["memory"][:4]

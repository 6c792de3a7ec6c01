"""Acceptance criterion 1 on the B200 (ref
tests/test_acceptance.py:98-120): the reference's 200 random kernels, compiled
by the IR-JIT, each run untransformed, sliced at every fraction of the
reference's gate (1/2 .. 1/32 and 1/total, largest-axis rectangular plans) and
as PTB with 1, 2, 4 and 8 workers after the product's
``unify_synchronization`` -- every final memory image equals the reference
interpreter's, and every logical block runs exactly once.  Needs a B200."""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(gold):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_07381_b200 as P
    from paper_2410_07381_b200 import irjit, kernels, transforms
    P.B200Device.get(0)
    cases = gold("acceptance")["cases"]
    raw = irjit.JitKernel.compile_many([c["kernel"] for c in cases])
    uni = irjit.JitKernel.compile_many([transforms.unify_synchronization(irjit.normalize(c["kernel"]))
                                        for c in cases])
    return P, kernels.Stream(high_priority=False), cases, raw, uni


def _image(memory):
    return torch.tensor(memory, dtype=torch.int64, device="cuda")


def test_acceptance_gate_200_kernels_on_device(env, gold):
    P, s, cases, raw, uni = env
    fracs = [Fraction(f) for f in gold("acceptance")["fractions"]]
    runs = 0
    for c, jr, ju in zip(cases, raw, uni):
        assert c["status"] == "Completed"
        grid = c["kernel"]["grid"]
        total = grid[0] * grid[1] * grid[2]
        expect = c["base"]
        fault = torch.zeros(1, dtype=torch.int64, device="cuda")
        shapes = [("original", None)] + [("sliced", f) for f in fracs + [Fraction(1, total)]] + \
                 [("ptb", w) for w in gold("acceptance")["workers"]]
        for shape, arg in shapes:
            mem = _image(c["memory"])
            ec = torch.zeros(total, dtype=torch.int64, device="cuda")
            dk = (ju if shape == "ptb" else jr).bind(mem, fault, c["args"])
            if shape == "original":
                dk.original(s, exec_count=ec).wait()
            elif shape == "sliced":
                for o, g in P.slice_plan(None, arg, grid=grid):
                    dk.sliced_rect(s, o, g, exec_count=ec).wait()
            else:
                st = dk.ptb(s, arg, exec_count=ec).wait()
                assert st.done and total <= st.task_counter <= total + arg, (c["seed"], arg)
            got = mem.cpu().tolist()
            dk.close()
            assert int(fault.item()) == 0, (c["seed"], shape, arg)
            assert got == expect, (c["seed"], shape, arg)
            assert bool((ec == 1).all()), (c["seed"], shape, arg)
            runs += 1
    assert runs == 200 * (1 + len(fracs) + 1 + 4)


def test_unified_kernels_preempt_and_resume_on_device(env):
    """The product-unified kernels under real preemption: PTB(2) preempted when
    its counter reaches c, resumed from the persisted counter, for a sample of
    the gate's kernels and every c -- the image equals the reference's."""
    P, s, cases, _raw, uni = env
    for c, ju in list(zip(cases, uni))[:200:10]:
        grid = c["kernel"]["grid"]
        total = grid[0] * grid[1] * grid[2]
        for at in range(0, total + 1):
            mem = _image(c["memory"])
            fault = torch.zeros(1, dtype=torch.int64, device="cuda")
            ec = torch.zeros(total, dtype=torch.int64, device="cuda")
            dk = ju.bind(mem, fault, c["args"])
            st = dk.ptb(s, 2, preempt_at=at, exec_count=ec).wait()
            if st.parked:
                st = dk.ptb(s, 2, start_count=st.task_counter, exec_count=ec).wait()
            assert st.done
            got = mem.cpu().tolist()
            dk.close()
            assert int(fault.item()) == 0 and got == c["base"], (c["seed"], at)
            assert bool((ec == 1).all()), (c["seed"], at)

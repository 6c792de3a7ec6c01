"""On-device parity of every kernel shape (Original / Sliced / PTB) against the
CPU oracle and the reference's golden vectors, plus exactly-once audits and
preempt/resume exactness.  Needs a B200."""

import random
from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import kernel_ir as ki          # noqa: E402
from oracle import rewrites as rw           # noqa: E402


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_07381_b200 as pkg
    from paper_2410_07381_b200 import kernels
    pkg.B200Device.get(0)
    pkg.kernels = kernels
    return pkg


@pytest.fixture(scope="module")
def stream(P):
    return P.kernels.Stream(high_priority=False)


def _ir_case(gold, name):
    return next(c for c in gold("ir")["cases"] if c["name"] == name)


def _vecadd_kernel(P, case):
    mem = torch.tensor(case["memory"], dtype=torch.int64, device="cuda")
    a, b, o = case["args"]
    n = case["kernel"]["grid"][0]
    return mem, P.kernels.vecadd_i64(mem, a, b, o, n, elems_per_block=1)


@pytest.mark.parametrize("name", ["vecadd", "vecadd16_wrap"])
def test_vecadd_i64_all_shapes_match_reference_golden(P, stream, gold, name):
    case = _ir_case(gold, name)
    expect = case["expect"]["memory"]
    # the oracle agrees with the golden vector
    k = ki.kernel_from_json(case["kernel"])
    assert list(ki.interpret(k, tuple(case["args"]), tuple(case["memory"])).memory) == expect
    n = case["kernel"]["grid"][0]
    runs = [("original", lambda dk, ec: [dk.original(stream, exec_count=ec)])]
    for f in (Fraction(1, 2), Fraction(1, 4), Fraction(1, 3), Fraction(1, n)):
        plan = P.slice_plan(n, f)
        runs.append((f"sliced{f}", lambda dk, ec, plan=plan:
                     [dk.sliced(stream, off, cnt, exec_count=ec) for off, cnt in plan]))
    for w in (1, 2, 4, 8, 148):
        runs.append((f"ptb{w}", lambda dk, ec, w=w: [dk.ptb(stream, w, exec_count=ec)]))
    for label, go in runs:
        mem, dk = _vecadd_kernel(P, case)
        ec = torch.zeros(n, dtype=torch.int64, device="cuda")
        for L in go(dk, ec):
            L.wait()
        assert mem.cpu().tolist() == expect, label
        assert ec.cpu().tolist() == [1] * n, label          # exactly once
        dk.close()


def test_ptb_preempt_at_every_counter_then_resume(P, stream, gold):
    """Device analogue of ref tests/test_transforms.py:185-219: raise the flag
    when the counter reaches c (MemTrigger), resume from the persisted counter;
    payload equals the uninterrupted run, every logical block ran exactly once."""
    case = _ir_case(gold, "vecadd16_wrap")
    expect = case["expect"]["memory"]
    for workers in (1, 4, 16):
        for c in range(0, 18):
            mem, dk = _vecadd_kernel(P, case)
            ec = torch.zeros(16, dtype=torch.int64, device="cuda")
            first = dk.ptb(stream, workers, preempt_at=c, exec_count=ec).wait()
            ctr = first.task_counter
            assert ctr >= min(c, 16) if c > 0 else ctr >= 16
            # every block below the counter ran exactly once or was handed
            # back unrun (bounded retirement: at most one per worker), none
            # above it ran
            counts = ec.cpu().tolist()
            below = counts[:min(ctr, 16)]
            returned = below.count(0)
            assert set(below) <= {0, 1} and returned <= workers
            assert counts[min(ctr, 16):] == [0] * (16 - min(ctr, 16))
            assert first.parked == (ctr < 16 or returned > 0)
            if first.parked:
                second = dk.ptb(stream, workers, start_count=ctr, exec_count=ec).wait()
                assert second.done and second.task_counter >= 16
            assert mem.cpu().tolist() == expect, (workers, c)
            assert ec.cpu().tolist() == [1] * 16, (workers, c)
            dk.close()


def _hold(stream, ms=60):
    """Queue ~ms of spinning in front of the next launch on ``stream``."""
    with torch.cuda.stream(torch.cuda.ExternalStream(stream.handle())):
        torch.cuda._sleep(int(ms * 2.0e6))


def test_ptb_flag_before_launch_is_noop(P, stream, gold):
    """ref tests/test_transforms.py:174-183: the flag is raised before any
    worker starts (the launch waits behind ~60 ms of spinning on its stream)
    -> no claim, counter == start, memory untouched; a resume then completes
    the kernel exactly once."""
    case = _ir_case(gold, "vecadd")
    mem, dk = _vecadd_kernel(P, case)
    before = mem.cpu().tolist()
    n = case["kernel"]["grid"][0]
    ec = torch.zeros(n, dtype=torch.int64, device="cuda")
    _hold(stream)
    L = dk.ptb(stream, 4, exec_count=ec)
    L.preempt()
    st = L.wait()
    assert st.parked and not st.done
    assert st.claims == 0 and st.task_counter == 0
    assert mem.cpu().tolist() == before
    assert int(ec.sum().item()) == 0
    st2 = dk.ptb(stream, 4, start_count=st.task_counter, exec_count=ec).wait()
    assert st2.done
    assert mem.cpu().tolist() == case["expect"]["memory"]
    assert ec.cpu().tolist() == [1] * n


def test_chain_flag_parks_the_queue_behind_a_preempted_launch(P, stream, gold):
    """Look-ahead chain mode: three PTB launches queued on one stream behind
    ~60 ms of spinning; preempting the first parks all three before any
    claim (one shared word), and resuming them in order completes each
    exactly once."""
    from paper_2410_07381_b200 import kernels
    g = torch.Generator(device="cuda").manual_seed(3)
    n = 1 << 20
    x = torch.rand(n, device="cuda", generator=g)
    y = torch.rand(n, device="cuda", generator=g)
    outs = [torch.zeros(n, device="cuda") for _ in range(3)]
    ks = [kernels.vecadd_f32(x if i == 0 else outs[i - 1], y, outs[i]) for i in range(3)]
    ecs = [torch.zeros(k.total_blocks, dtype=torch.int64, device="cuda") for k in ks]
    _hold(stream)
    Ls = [k.ptb(stream, 148, exec_count=e, chain=True) for k, e in zip(ks, ecs)]
    Ls[0].preempt()
    sts = [L.wait() for L in Ls]
    assert all(st.parked and st.claims == 0 for st in sts)
    assert all(int(e.sum().item()) == 0 for e in ecs)
    assert all(int(o.abs().sum().item()) == 0 for o in outs)
    for k, e in zip(ks, ecs):
        assert k.ptb(stream, 148, exec_count=e, chain=True).wait().done
    ref = x
    for i in range(3):
        ref = ref + y
        assert torch.equal(outs[i], ref)
        assert bool((ecs[i] == 1).all())

def test_vecadd_f32_bit_exact_all_shapes(P, stream):
    g = torch.Generator(device="cuda").manual_seed(0)
    n = 1 << 22
    a = torch.rand(n, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, device="cuda", generator=g) * 2 - 1
    ref = a + b                                  # IEEE add: exactly rounded
    for shape in ("original", "sliced", "ptb"):
        c = torch.full_like(a, float("nan"))
        dk = P.kernels.vecadd_f32(a, b, c)
        total = dk.total_blocks
        ec = torch.zeros(total, dtype=torch.int64, device="cuda")
        if shape == "original":
            dk.original(stream, exec_count=ec).wait()
        elif shape == "sliced":
            for off, cnt in P.slice_plan(total, Fraction(1, 7)):
                dk.sliced(stream, off, cnt, exec_count=ec).wait()
        else:
            dk.ptb(stream, 296, exec_count=ec).wait()
        assert torch.equal(c, ref), shape
        assert bool((ec == 1).all()), shape
        dk.close()


def test_rowsum_f32_shapes_identical_and_within_tolerance(P, stream):
    g = torch.Generator(device="cuda").manual_seed(1)
    for rows, cols in ((4096, 768), (1000, 1023), (8, 5)):
        x = torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1
        outs = []
        for shape in ("original", "sliced", "ptb"):
            out = torch.zeros(rows, device="cuda")
            dk = P.kernels.rowsum_f32(x, out)
            if shape == "original":
                dk.original(stream).wait()
            elif shape == "sliced":
                for off, cnt in P.slice_plan(dk.total_blocks, Fraction(1, 4)):
                    dk.sliced(stream, off, cnt).wait()
            else:
                dk.ptb(stream, 148).wait()
            outs.append(out.clone())
            dk.close()
        assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
        ref = x.double().sum(dim=1)
        rel = ((outs[0].double() - ref).abs().max() / ref.abs().max()).item()
        assert rel < 1e-5, rel


def test_random_preempts_exactly_once_at_scale(P, stream):
    """Host-timed preemptions at random instants on a 2^26-element PTB
    launch; every logical block executes exactly once across the chain."""
    n = 1 << 26
    a = torch.ones(n, device="cuda")
    b = torch.arange(n, device="cuda", dtype=torch.float32)
    c = torch.zeros(n, device="cuda")
    dk = P.kernels.vecadd_f32(a, b, c)
    total = dk.total_blocks
    ec = torch.zeros(total, dtype=torch.int64, device="cuda")
    rng = random.Random(7)
    ctr, hops = 0, 0
    while ctr < total:
        L = dk.ptb(stream, 148 * 4, start_count=ctr, exec_count=ec)
        t_end = P.B200Device.now_ns() + rng.randint(0, 300_000)
        while P.B200Device.now_ns() < t_end and not L.query().done:
            pass
        try:
            L.preempt()
        except ValueError:
            pass   # already finished
        st = L.wait()
        assert st.task_counter >= ctr
        ctr = st.task_counter
        hops += 1
        assert hops < 1000
    torch.cuda.synchronize()
    assert bool((ec == 1).all())
    assert torch.equal(c, b + 1)
    dk.close()


def test_preemption_latency_under_50us(P, stream):
    """Flag write -> last worker exit, on the device clock, for a PTB launch of
    the HP-sized vecadd (logical blocks of ~1 us)."""
    n = 1 << 26
    a = torch.rand(n, device="cuda")
    b = torch.rand(n, device="cuda")
    c = torch.zeros(n, device="cuda")
    dk = P.kernels.vecadd_f32(a, b, c)
    dev = P.B200Device.get()
    off, unc = dev.clock_offset()
    lat = []
    for _ in range(10):
        L = dk.ptb(stream, 148 * 4)
        t = P.B200Device.now_ns() + 100_000
        while P.B200Device.now_ns() < t:
            pass
        L.preempt()
        st = L.wait()
        if not st.parked:
            continue
        lat.append((st.gt_last_exit + off - st.host_preempt_ns) / 1000.0)
    assert lat, "no launch was still running at the preempt instant"
    lat.sort()
    print(f"preempt latency us: median {lat[len(lat) // 2]:.1f} max {lat[-1]:.1f} "
          f"(clock uncertainty {unc / 1000:.1f} us)")
    assert lat[len(lat) // 2] < 50.0
    dk.close()


def test_hp_blocks_dominate_queued_be_blocks(P):
    """Row a17, HP dominance (ref sim.py:370-384: no best-effort block starts
    while a high-priority launch has unplaced blocks), on the device: a
    best-effort spin kernel with four waves of blocks queued on the
    lowest-priority stream, then a high-priority spin kernel with two waves;
    the hardware CTA scheduler (stream priorities) places every HP block
    before any further BE block -- from the first HP block's start to the last
    HP block's start, no BE block starts (block logs on %globaltimer; a
    handful racing the very first HP dispatch are tolerated)."""
    import time
    K = P.kernels
    lo, hi = K.Stream(high_priority=False), K.Stream(high_priority=True)
    probe = K.spin(148, 256, 0)
    slots = 148 * max(1, probe.info.occupancy_original)
    be = K.spin(4 * slots, 256, 1_000_000)   # 4 waves of 1 ms blocks
    hp = K.spin(2 * slots, 256, 100_000)
    for _ in range(2):
        bl = torch.zeros(be.total_blocks, 3, dtype=torch.int64, device="cuda")
        hl = torch.zeros(hp.total_blocks, 3, dtype=torch.int64, device="cuda")
        Lb = be.original(lo, block_log=bl)
        time.sleep(0.0015)   # the BE kernel's second wave is resident, two more queued
        Lh = hp.original(hi, block_log=hl)
        Lh.wait()
        Lb.wait()
        b, h = bl.cpu(), hl.cpu()
        h0, h1 = h[:, 0].min().item(), h[:, 0].max().item()
        assert b[:, 0].min().item() < h0 < b[:, 0].max().item()   # HP arrived while BE blocks were queued
        inside = ((b[:, 0] > h0) & (b[:, 0] < h1)).sum().item()
        assert inside <= 8, (inside, be.total_blocks)
        # and the HP blocks were not starved: all placed within ~one BE block time
        assert h1 - h0 < 1_000_000 + 3 * 100_000

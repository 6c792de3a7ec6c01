"""tcgen05 GEMM kernels in all three Tally shapes.  Needs a B200.

Tolerances (north star): fp32 (3xTF32) within 1e-5 relative, bf16 within 1e-2,
both normwise against a float64 reference of the same inputs:
    max|C - C_ref| / max|C_ref|
and every shape bit-identical to the untransformed (Original) kernel.
"""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_07381_b200 as P
    from paper_2410_07381_b200 import kernels
    P.B200Device.get(0)
    return P, kernels, kernels.Stream(high_priority=False)


def _run_shapes(P, dk, stream, out, total):
    results = {}
    for shape in ("original", "sliced", "ptb"):
        out.zero_()
        ec = torch.zeros(total, dtype=torch.int64, device="cuda")
        if shape == "original":
            dk.original(stream, exec_count=ec).wait()
        elif shape == "sliced":
            for off, cnt in P.slice_plan(total, Fraction(1, 5)):
                dk.sliced(stream, off, cnt, exec_count=ec).wait()
        else:
            dk.ptb(stream, 148, exec_count=ec).wait()
        assert bool((ec == 1).all()), shape
        results[shape] = out.clone()
    return results


@pytest.mark.parametrize("mnk", [(256, 128, 64), (512, 384, 1024), (1024, 1024, 4096)])
def test_sgemm_tf32x3_fp32_accuracy_all_shapes(env, mnk):
    P, kernels, stream = env
    M, N, K = mnk
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    B = torch.rand(N, K, device="cuda", generator=g) * 2 - 1
    C = torch.zeros(M, N, device="cuda")
    sg = kernels.sgemm_tf32x3(A, B, C)
    sg.prepare(stream)
    # the split is exact: hi + lo == x
    assert torch.equal(sg.a_hi + sg.a_lo, A) and torch.equal(sg.b_hi + sg.b_lo, B)
    res = _run_shapes(P, sg.gemm, stream, C, sg.gemm.total_blocks)
    ref = A.double() @ B.double().T
    err = ((res["original"].double() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-5, err
    assert torch.equal(res["original"], res["sliced"]) and torch.equal(res["original"], res["ptb"])
    sg.close()


@pytest.mark.parametrize("mnk", [(256, 256, 128), (1024, 768, 2048)])
def test_gemm_bf16_all_shapes(env, mnk):
    P, kernels, stream = env
    M, N, K = mnk
    g = torch.Generator(device="cuda").manual_seed(M * 3 + K)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    B = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    dk = kernels.gemm_bf16(A, B, C)
    res = _run_shapes(P, dk, stream, C, dk.total_blocks)
    ref = A.double() @ B.double().T
    err = ((res["original"].double() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-2, err
    assert torch.equal(res["original"], res["sliced"]) and torch.equal(res["original"], res["ptb"])
    dk.close()


def test_sgemm_ptb_preempt_resume_exactly_once(env):
    """Preempt the PTB SGEMM at claim counts 37, 200, 311 (device MemTrigger)
    and resume until done.  Preempted workers stop at a K-chunk boundary and
    park their fp32 running total in C; the chain's result is bit-identical
    to the untransformed kernel and every tile is claimed exactly once."""
    P, kernels, stream = env
    M = N = K = 2048
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    B = torch.rand(N, K, device="cuda", generator=g) * 2 - 1
    C = torch.zeros(M, N, device="cuda")
    sg = kernels.sgemm_tf32x3(A, B, C)
    sg.prepare(stream)
    sg.gemm.original(stream).wait()
    ref = C.clone()
    C.zero_()
    torch.cuda.synchronize()
    total = sg.gemm.total_blocks
    ec = torch.zeros(total, dtype=torch.int64, device="cuda")
    ctr, hops, parked = 0, 0, 0
    triggers = [37, 200, 311]
    while True:
        c = triggers[hops] if hops < len(triggers) else None
        st = sg.gemm.ptb(stream, 148, start_count=ctr, preempt_at=c, exec_count=ec).wait()
        assert st.task_counter >= ctr
        ctr = st.task_counter
        hops += 1
        parked += st.parked
        if not st.parked:
            break
        assert hops < 50
    assert parked >= 3
    torch.cuda.synchronize()
    assert bool((ec == 1).all())
    assert torch.equal(C, ref)
    sg.close()


def test_sgemm_chunk_preemption_latency_and_exactness(env):
    """Host-timed preemptions of a 4096^3 PTB SGEMM at random instants: the
    chain stays bit-exact and the flag->last-exit latency is a fraction of a
    tile (chunk granularity, ~1/8 of a 128x64 3xTF32 tile)."""
    import random
    P, kernels, stream = env
    M = N = K = 4096
    g = torch.Generator(device="cuda").manual_seed(6)
    A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    B = torch.rand(N, K, device="cuda", generator=g) * 2 - 1
    C = torch.zeros(M, N, device="cuda")
    sg = kernels.sgemm_tf32x3(A, B, C)
    sg.prepare(stream)
    sg.gemm.original(stream).wait()
    ref = C.clone()
    C.zero_()
    torch.cuda.synchronize()
    dev = P.B200Device.get()
    off, _ = dev.clock_offset()
    total = sg.gemm.total_blocks
    ec = torch.zeros(total, dtype=torch.int64, device="cuda")
    rng = random.Random(3)
    ctr, lat, hops = 0, [], 0
    while True:
        L = sg.gemm.ptb(stream, 148, start_count=ctr, exec_count=ec)
        t_end = P.B200Device.now_ns() + rng.randint(20_000, 120_000)
        while P.B200Device.now_ns() < t_end and not L.query().done:
            pass
        if hops < 12:
            try:
                L.preempt()
            except ValueError:
                pass
        st = L.wait()
        ctr = st.task_counter
        hops += 1
        if st.parked:
            lat.append((st.gt_last_exit + off - st.host_preempt_ns) / 1e3)
        else:
            break
        assert hops < 100
    torch.cuda.synchronize()
    assert bool((ec == 1).all())
    assert torch.equal(C, ref)
    lat.sort()
    print(f"sgemm chunk-preemption latency us: median {lat[len(lat) // 2]:.1f} max {lat[-1]:.1f}")
    assert lat[len(lat) // 2] < 30.0
    sg.close()


def test_gemm_cooperative_suspension_resumes_in_place(env):
    """Pausable PTB GEMM: suspend mid-run (global pause word), verify it stops
    making progress, resume, and the result equals the Original kernel's."""
    P, kernels, stream = env
    from paper_2410_07381_b200 import _lib
    import ctypes as C
    M = N = K = 4096
    g = torch.Generator(device="cuda").manual_seed(9)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    B = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).bfloat16()
    C_ = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    dk = kernels.gemm_bf16(A, B, C_)
    dk.original(stream).wait()
    ref = C_.clone()
    C_.zero_()
    ec = torch.zeros(dk.total_blocks, dtype=torch.int64, device="cuda")
    d = _lib.c_launch_desc(shape=_lib.SHAPE_PTB, workers=148, start_count=0, preempt_at=-1,
                           exec_count=ec.data_ptr(), pausable=1)
    lid = C.c_int()
    _lib.check(_lib.lib.tally_set_pause(1), "pause")      # start suspended
    _lib.check(_lib.lib.tally_launch(dk.id, stream.id, C.byref(d), C.byref(lid)), "launch")
    L = kernels.Launch(lid.value, _lib.SHAPE_PTB)
    t_end = P.B200Device.now_ns() + 20_000_000
    while P.B200Device.now_ns() < t_end:
        pass
    assert not L.query().done                              # held in place
    _lib.check(_lib.lib.tally_set_pause(0), "resume")
    st = L.wait()
    assert st.done and not st.parked
    assert bool((ec == 1).all())
    assert torch.equal(C_, ref)
    dk.close()

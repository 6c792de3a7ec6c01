"""Generate ``tests/golden/*.json`` by running the REFERENCE ``tallysim``.

Run in the build container only (``/root/reference`` is absent on the GPU
box):

    python -m oracle.gen_golden            # writes tests/golden/*.json

The reference is imported read-only from ``/root/reference/pkg/src``.  The
fixtures pin (a) the oracle restatement in this package and (b) the product's
decision core, so every value here is an output of the reference itself; the
scenario inputs mirror the reference's own tests (cited per section).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from fractions import Fraction

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import tallysim.ir as ir
    import tallysim.ir.randgen as randgen
    import tallysim.profiler as profiler
    import tallysim.scheduler as scheduler
    import tallysim.sim as sim
    import tallysim.transforms as transforms
    import tallysim.workloads as workloads
    return ir, randgen, transforms, sim, profiler, scheduler, workloads


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def kjson(k):
    """Reference KernelDef -> oracle JSON encoding (see oracle/kernel_ir.py)."""
    from tallysim.ir.core import Imm, Reg, SpecialReg

    def enc(o):
        if isinstance(o, Reg):
            return {"r": o.index}
        if isinstance(o, Imm):
            return {"i": o.value}
        if isinstance(o, SpecialReg):
            return {"s": f"{o.kind}.{o.axis}"}
        return o
    return {"name": k.name, "params": list(k.params), "grid": list(k.grid),
            "block": list(k.block), "regs": k.register_count, "shared": k.shared_words,
            "dependent": k.inter_block_dependent,
            "body": [[i.opcode, [enc(o) for o in i.operands], i.label] for i in k.body]}


def res_json(r):
    return {"status": r.status, "memory": None if r.final_memory is None else
            list(r.final_memory), "steps": r.steps_executed}


# --------------------------------------------------------------------------
def gen_ir():
    ir, randgen, tr, *_ = _ref()
    from tallysim.ir import (Dim3, Imm, Instruction, KernelDef, LaunchSpec, Reg,
                             SpecialReg, interpret, parse_kernel)
    cases = []

    def simple(body, block=Dim3(1), shared=0, params=(), regs=4, grid=Dim3(1)):
        return KernelDef("t", params, grid, block, regs, shared, tuple(body))

    # ref tests/test_cli.py:17-35 and tests/test_ir.py:165-172 (vecadd golden)
    vecadd_text = ("kernel vecadd\ngrid 8 1 1\nblock 1 1 1\nregs 6\nshared 0\n"
                   "param a_base\nparam b_base\nparam out_base\n"
                   "  READ_SPECIAL r3 blockIdx.x\n  ADD r4 r0 r3\n  LOAD_GLOBAL r4 r4\n"
                   "  ADD r5 r1 r3\n  LOAD_GLOBAL r5 r5\n  ADD r4 r4 r5\n  ADD r5 r2 r3\n"
                   "  STORE_GLOBAL r5 r4\n  RET\n")
    vk = parse_kernel(vecadd_text)
    mem = tuple(range(1, 9)) + tuple(range(10, 18)) + (0,) * 8
    cases.append(("vecadd", vk, (0, 8, 16), mem, 0, 10**7))
    # 16-block vecadd with extreme values (wrap-around) for the device parity path
    vk16 = KernelDef(vk.name, vk.params, Dim3(16), vk.block, vk.register_count,
                     vk.shared_words, vk.body)
    big = (2**63 - 1, -2**63, 5, -5, 2**62, -(2**62), 1, 0) * 2
    mem16 = big + tuple(range(16)) + (0,) * 16
    cases.append(("vecadd16_wrap", vk16, (0, 16, 32), mem16, 0, 10**7))
    # ref tests/test_ir.py:183-205
    cases.append(("divmod", simple([
        Instruction("CONST", (Reg(0), Imm(-7))), Instruction("DIV", (Reg(1), Reg(0), Imm(2))),
        Instruction("MOD", (Reg(2), Reg(0), Imm(2))), Instruction("STORE_GLOBAL", (Imm(0), Reg(1))),
        Instruction("STORE_GLOBAL", (Imm(1), Reg(2))), Instruction("RET")]), (), (0, 0), 0, 10**7))
    cases.append(("div0", simple([
        Instruction("CONST", (Reg(0), Imm(11))), Instruction("DIV", (Reg(1), Reg(0), Imm(0))),
        Instruction("MOD", (Reg(2), Reg(0), Imm(0))), Instruction("STORE_GLOBAL", (Imm(0), Reg(1))),
        Instruction("STORE_GLOBAL", (Imm(1), Reg(2))), Instruction("RET")]), (), (0, 0), 0, 10**7))
    # ref tests/test_ir.py:207-235
    cases.append(("divergent", simple([
        Instruction("READ_SPECIAL", (Reg(0), SpecialReg("threadIdx", "x"))),
        Instruction("BRANCH", (Reg(0), "wait")), Instruction("RET"),
        Instruction("BAR_SYNC", label="wait"), Instruction("RET")], block=Dim3(2)), (), (), 0, 10**7))
    cases.append(("exchange", simple([
        Instruction("READ_SPECIAL", (Reg(0), SpecialReg("threadIdx", "x"))),
        Instruction("STORE_SHARED", (Reg(0), Reg(0))), Instruction("BAR_SYNC"),
        Instruction("CONST", (Reg(1), Imm(1))), Instruction("SUB", (Reg(1), Reg(1), Reg(0))),
        Instruction("LOAD_SHARED", (Reg(2), Reg(1))), Instruction("STORE_GLOBAL", (Reg(0), Reg(2))),
        Instruction("RET")], block=Dim3(2), shared=2), (), (0, 0), 0, 10**7))
    # ref tests/test_ir.py:237-247
    cases.append(("steplimit", simple([Instruction("JUMP", ("loop",), label="loop")]), (), (), 0, 100))
    cases.append(("fault", simple([Instruction("LOAD_GLOBAL", (Reg(0), Imm(99))),
                                   Instruction("RET")]), (), (0,), 0, 10**7))
    # random kernels, ref ir/randgen.py:63-190 (as used in tests/test_acceptance.py:98-120)
    for seed in range(60):
        c = randgen.random_kernel(seed, max_blocks=16, max_threads=8)
        cases.append((f"rand{seed}", c.kernel, c.arg_values, c.initial_memory, 0, 10**7))
    for seed in range(8):
        c = randgen.random_kernel(1000 + seed)
        cases.append((f"randbig{seed}", c.kernel, c.arg_values, c.initial_memory, seed, 10**7))

    out = []
    for name, k, args, mem, seed, lim in cases:
        r = interpret(LaunchSpec(k, args, mem), seed, lim)
        out.append({"name": name, "kernel": kjson(k), "args": list(args), "memory": list(mem),
                    "seed": seed, "step_limit": lim, "expect": res_json(r)})
    return {"cases": out}


def gen_transforms():
    ir, randgen, tr, *_ = _ref()
    from tallysim.ir import Dim3, Imm, Instruction, KernelDef, LaunchSpec, Reg, SpecialReg, interpret
    # ref tests/test_transforms.py:50-70: slice_extents known answers + a grid sweep
    extents = []
    fr = [Fraction(1, d) for d in (1, 2, 3, 4, 5, 8, 16, 32, 64)] + [Fraction(2, 3), Fraction(3, 8)]
    for n in list(range(1, 41)) + [64, 100, 108, 148, 1024, 2048, 4096]:
        for f in fr + [Fraction(1, n)]:
            extents.append({"len": n, "frac": str(f), "extents": tr.slice_extents(n, f)})
    plans = []
    for grid in ((16, 1, 1), (6, 2, 1), (2, 6, 1), (3, 3, 3), (64, 32, 1), (1, 1, 9)):
        for f in (Fraction(1, 2), Fraction(1, 4), Fraction(1, 3), Fraction(1, 1)):
            c = randgen.random_kernel(1)
            k = KernelDef("g", c.kernel.params, Dim3(*grid), c.kernel.block,
                          c.kernel.register_count, c.kernel.shared_words, c.kernel.body)
            p = tr.slice_kernel(k, f)
            plans.append({"grid": list(grid), "frac": str(f),
                          "subs": [[list(o), list(g)] for o, g in p.sub_launches]})

    # sliced / ptb equivalence (ref tests/test_acceptance.py:98-120)
    equiv = []
    for seed in range(40):
        c = randgen.random_kernel(seed, max_blocks=16, max_threads=8)
        base = interpret(c.launch)
        rec = {"seed": seed, "kernel": kjson(c.kernel), "args": list(c.arg_values),
               "memory": list(c.initial_memory), "base": res_json(base), "sliced": {}, "ptb": {}}
        for f in (Fraction(1, 2), Fraction(1, 4), Fraction(1, 8), Fraction(1, c.kernel.grid.total)):
            r = tr.run_sliced(tr.slice_kernel(c.kernel, f), c.arg_values, c.initial_memory)
            rec["sliced"][str(f)] = {"status": r.status, "same": r.final_memory == base.final_memory,
                                     "steps": r.steps_executed}
        for w in (1, 2, 4, 8):
            ptb = tr.make_preemptible(tr.unify_synchronization(c.kernel), Dim3(w))
            n = len(c.initial_memory)
            ctl = tr.PtbControl(n, n + 1, c.kernel.grid.total, c.kernel.grid)
            r = tr.run_ptb(ptb, ctl, c.arg_values, c.initial_memory + (0, 0))
            rec["ptb"][str(w)] = {"status": r.status, "tail": list(r.final_memory[n:]),
                                  "same": r.final_memory[:n] == base.final_memory}
        equiv.append(rec)

    # preempt at every counter value then resume (ref tests/test_transforms.py:185-219)
    c = randgen.random_kernel(13, max_blocks=16, max_threads=8)
    k = c.kernel
    k16 = KernelDef(k.name, k.params, Dim3(16), k.block, k.register_count, k.shared_words, k.body)
    nth = k.block.total
    n = 16 * nth
    mem = tuple(range(1, n + 1)) + (0,) * n + (0, 0)
    ptb = tr.make_preemptible(tr.unify_synchronization(k16), Dim3(4))
    ctl = tr.PtbControl(len(mem), len(mem) + 1, 16, k16.grid)
    full = mem + (0, 0)
    unint = tr.run_ptb(ptb, ctl, (0, n), full)
    sweep = []
    for cnt in range(17):
        first = tr.run_ptb(ptb, ctl, (0, n), full, preempt_at_count=cnt)
        m = list(first.final_memory)
        m[ctl.preempt_flag_addr] = 0
        second = tr.run_ptb(ptb, ctl, (0, n), tuple(m))
        sweep.append({"c": cnt, "first": res_json(first), "second": res_json(second)})
    preempt = {"kernel": kjson(k16), "args": [0, n], "memory": list(full), "workers": 4,
               "ctr": ctl.task_counter_addr, "flag": ctl.preempt_flag_addr,
               "uninterrupted": res_json(unint), "sweep": sweep}

    # witness (ref tests/test_transforms.py:222-264)
    body = [
        Instruction("READ_SPECIAL", (Reg(0), SpecialReg("threadIdx", "x"))),
        Instruction("READ_SPECIAL", (Reg(1), SpecialReg("blockIdx", "x"))),
        Instruction("MUL", (Reg(2), Reg(1), Imm(2))), Instruction("ADD", (Reg(2), Reg(2), Reg(0))),
        Instruction("CONST", (Reg(3), Imm(7))), Instruction("STORE_GLOBAL", (Reg(2), Reg(3))),
        Instruction("BRANCH", (Reg(0), "cont")), Instruction("RET"),
        Instruction("BAR_SYNC", label="cont"), Instruction("RET")]
    wk = KernelDef("witness", (), Dim3(2), Dim3(2), 4, 0, tuple(body))
    raw = tr.run_ptb(tr.make_preemptible(wk, Dim3(1), enforce_unified=False),
                     tr.PtbControl(4, 5, 4, wk.grid), (), (0,) * 6)
    uni = tr.run_ptb(tr.make_preemptible(tr.unify_synchronization(wk), Dim3(1)),
                     tr.PtbControl(4, 5, 2, wk.grid), (), (0,) * 6)
    witness = {"kernel": kjson(wk), "raw": res_json(raw), "unified": res_json(uni)}
    return {"extents": extents, "plans": plans, "equiv": equiv, "preempt": preempt,
            "witness": witness}


# --------------------------------------------------------------------------
def gen_acceptance():
    """Acceptance criterion 1 (ref tests/test_acceptance.py:98-120):
    the 200 random kernels (max_blocks=16, max_threads=8), their inputs, the
    reference interpreter's final image, and the reference's unified-sync
    rewrite of each (what the product's unify_synchronization must equal)."""
    ir, randgen, tr, *_ = _ref()
    from tallysim.ir import interpret
    cases = []
    for seed in range(200):
        c = randgen.random_kernel(seed, max_blocks=16, max_threads=8)
        base = interpret(c.launch)
        cases.append({"seed": seed, "kernel": kjson(c.kernel), "args": list(c.arg_values),
                      "memory": list(c.initial_memory), "status": base.status,
                      "base": list(base.final_memory), "unified": kjson(tr.unify_synchronization(c.kernel))})
    return {"cases": cases, "fractions": ["1/2", "1/4", "1/8", "1/16", "1/32"], "workers": [1, 2, 4, 8]}


def _shape_json(s):
    n = type(s).__name__
    if n == "SlicedShape":
        return {"kind": "sliced", "sub_blocks": list(s.sub_blocks)}
    if n == "PtbShape":
        return {"kind": "ptb", "worker_count": s.worker_count, "start_count": s.start_count}
    return {"kind": "original"}


def _cost_json(c):
    return {"block_duration_ns": c.block_duration_ns, "launch_overhead_ns": c.launch_overhead_ns,
            "ptb_iteration_overhead_ns": c.ptb_iteration_overhead_ns,
            "threads_per_block": c.threads_per_block, "total_blocks": c.total_blocks}


def gen_sim():
    *_, sim, profiler, scheduler, workloads = _ref()
    from tallysim.sim import (BEST_EFFORT, HIGH, GpuSim, GpuSpec, OriginalShape, PtbShape,
                              SimLaunch, SlicedShape, cost_model, events_to_csv, ms_to_ns)
    G8 = GpuSpec(8, 1024, 4)
    G4 = GpuSpec(4, 128, 1)
    GB = GpuSpec(148, 2048, 32)
    scen = []

    def add(name, gpu, launches, preempts=(), seed=0):
        s = GpuSim(gpu, placement_seed=seed)
        hs = []
        for at, task, kern, prio, shape, cost in launches:
            hs.append(s.submit(SimLaunch(task, kern, prio, shape, cost), at))
        for at, idx in preempts:
            s.signal_preempt(hs[idx], at)
        s.run_to_completion()
        csv = events_to_csv(s.events)
        hj = []
        for h, (at, *_r) in zip(hs, launches):
            d = {"finish_time": h.finish_time, "blocks_finished": h.blocks_finished,
                 "task_counter": h.task_counter, "parked": h.parked, "done": h.done,
                 "park_times": h.park_times, "sub_completions": h.sub_completions}
            hj.append(d)
        turn = []
        for at, idx in preempts:
            try:
                turn.append(s.measured_turnaround(hs[idx], at))
            except ValueError:
                turn.append(None)
        scen.append({"name": name, "gpu": [gpu.num_sms, gpu.max_threads_per_sm, gpu.max_blocks_per_sm],
                     "seed": seed,
                     "launches": [{"at": at, "task": t, "kernel": k, "priority": p,
                                   "shape": _shape_json(sh), "cost": _cost_json(c)}
                                  for at, t, k, p, sh, c in launches],
                     "preempts": [{"at": at, "launch": i} for at, i in preempts],
                     "csv_sha256": sha(csv), "n_events": len(s.events),
                     "csv": csv if len(s.events) <= 400 else None,
                     "handles": hj, "turnaround": turn})

    c8 = cost_model(1.0, 8, threads_per_block=256)       # ref tests/test_sim.py:60-72
    c16 = cost_model(1.0, 16, threads_per_block=256)
    add("one_wave", G8, [(0, "t", "k", BEST_EFFORT, OriginalShape(), cost_model(1.0, 32, 256))])
    add("two_waves", G8, [(0, "t", "k", BEST_EFFORT, OriginalShape(), cost_model(1.0, 64, 256))])
    add("sliced8", G8, [(0, "t", "k", BEST_EFFORT, SlicedShape((1,) * 8), c8)])
    add("sliced_uneven", G4, [(0, "t", "k", BEST_EFFORT, SlicedShape((3, 3, 4)), cost_model(0.5, 10, 128))])
    add("ptb2x16", G8, [(0, "t", "k", BEST_EFFORT, PtbShape(2), c16)])
    add("ptb_preempt_resume", G8, [(0, "t", "k", BEST_EFFORT, PtbShape(2), c16),
                                   (0, "t", "k", BEST_EFFORT, PtbShape(2, 16), c16)],
        preempts=[(ms_to_ns(3.5), 0)])
    add("ptb_preempt_mid", G4, [(0, "t", "k", BEST_EFFORT, PtbShape(4), cost_model(0.15, 108, 128))],
        preempts=[(ms_to_ns(1.234), 0)])
    add("ptb_preempt_in_overhead", G4, [(0, "t", "k", BEST_EFFORT, PtbShape(4), cost_model(0.15, 108, 128))],
        preempts=[(2000, 0)])
    add("ptb_preempt_late", G4, [(0, "t", "k", BEST_EFFORT, PtbShape(4), cost_model(0.1, 8, 128))],
        preempts=[(ms_to_ns(0.19), 0)])
    add("hp_vs_be", G4, [(0, "be", "bk", BEST_EFFORT, OriginalShape(), cost_model(0.15, 108, 128)),
                         (ms_to_ns(0.2), "hp", "hk", HIGH, OriginalShape(), cost_model(1.0, 1, 128))])
    add("hp_vs_ptb", G4, [(0, "be", "bk", BEST_EFFORT, PtbShape(4), cost_model(0.15, 108, 128)),
                          (ms_to_ns(0.2), "hp", "hk", HIGH, OriginalShape(), cost_model(1.0, 2, 128))],
        preempts=[(ms_to_ns(0.2), 0)])
    add("mixed_limits", G8, [(0, "a", "ka", BEST_EFFORT, OriginalShape(), cost_model(0.3, 40, 256)),
                             (1000, "b", "kb", BEST_EFFORT, OriginalShape(), cost_model(0.2, 50, 512)),
                             (50_000, "h", "kh", HIGH, OriginalShape(), cost_model(0.1, 12, 1024))], seed=3)
    for seed in (0, 1, 7):
        add(f"b200_ptb_seed{seed}", GB, [(0, "be", "sgemm", BEST_EFFORT, PtbShape(296), cost_model(0.03, 2048, 256)),
                                        (ms_to_ns(0.05), "hp", "vadd", HIGH, OriginalShape(), cost_model(0.004, 4096, 256))],
            preempts=[(ms_to_ns(0.05), 0)], seed=seed)
    add("b200_original_waves", GB, [(0, "be", "k", BEST_EFFORT, OriginalShape(), cost_model(0.01, 3000, 128))], seed=2)
    return {"scenarios": scen}


def gen_tuner():
    *_, sim, profiler, scheduler, workloads = _ref()
    from tallysim.profiler import (ConfigCandidate, Profiler, ProfileKey, candidate_configs,
                                   estimate_turnaround, select_config)
    from tallysim.sim import GpuSpec, cost_model
    G4, G8, GB = GpuSpec(4, 128, 1), GpuSpec(8, 1024, 4), GpuSpec(148, 2048, 32)

    def cj(c):
        return {"variant": c.variant, "fraction": None if c.fraction is None else str(c.fraction),
                "worker_count": c.worker_count}
    menus = []
    for gpu in (G4, G8, GB):
        for blocks in (1, 2, 3, 7, 8, 10, 16, 64, 100, 108, 1024, 2048, 4096):
            for tpb in (32, 128, 256, 1024):
                c = cost_model(0.1, blocks, tpb)
                if gpu.occupancy_limit(tpb) < 1:
                    continue
                menus.append({"gpu": [gpu.num_sms, gpu.max_threads_per_sm, gpu.max_blocks_per_sm],
                              "blocks": blocks, "tpb": tpb,
                              "cands": [cj(x) for x in candidate_configs(c, gpu)]})
    eq1 = []
    for lat, w, tot in ((1_000_000, 4, 100), (10_000_000, 2, 16), (333, 3, 7), (5, 1, 2), (15, 1, 2)):
        eq1.append({"lat": lat, "w": w, "total": tot,
                    "est": estimate_turnaround(ConfigCandidate("Ptb", worker_count=w), lat, tot)})
    profiles = []
    for gpu, runs, items in ((G4, 10, [("train_k", 0.15, 108, 128), ("serve_k", 3.925, 1, 128),
                                       ("k64", 0.5, 64, 128)]),
                             (G8, 3, [("k16", 1.0, 16, 256), ("k100", 0.2, 100, 512)]),
                             (GB, 2, [("sg", 0.03, 2048, 256), ("va", 0.004, 4096, 256),
                                      ("rd", 0.25, 1024, 256)])):
        p = Profiler(gpu, runs=runs)
        sel = {}
        for name, ms, blocks, tpb in items:
            c = cost_model(ms, blocks, tpb)
            key = ProfileKey(name, (blocks, 1, 1), (tpb, 1, 1))
            recs = p.profile(key, c)
            sel[name] = {str(th): cj(select_config(recs, th))
                         for th in (1, 10_000, 31_600, 100_000, 300_000, 1_000_000, 10**9)}
        profiles.append({"gpu": [gpu.num_sms, gpu.max_threads_per_sm, gpu.max_blocks_per_sm],
                         "runs": runs, "items": [list(i) for i in items],
                         "cache": p.dump_cache(), "select": sel,
                         "simulated_runs": p.simulated_runs})
    return {"menus": menus, "eq1": eq1, "profiles": profiles}


def _policy_scenarios():
    from tallysim.scheduler import KernelWork, TaskScript
    from tallysim.sim import BEST_EFFORT, HIGH, GpuSpec, cost_model, ms_to_ns
    G4 = GpuSpec(4, 128, 1)
    GB = GpuSpec(148, 2048, 32)
    hp = cost_model(1.0, 1, threads_per_block=128)          # ref tests/test_scheduler.py:28-29
    be = cost_model(0.15, 108, threads_per_block=128)
    S = []
    arr = tuple(ms_to_ns(x) for x in (0.5, 3.0, 3.2, 7.7, 12.0, 12.0, 15.3))
    S.append(("hp_be", G4, 20.0, [TaskScript("hp", HIGH, (KernelWork("hp_k", hp),), arr),
                                  TaskScript("be", BEST_EFFORT, (KernelWork("be_k", be),))]))
    S.append(("two_be", G4, 10.0, [TaskScript("hp", HIGH, (KernelWork("hp_k", hp),), arr[:3]),
                                   TaskScript("b1", BEST_EFFORT, (KernelWork("b1_k", be),)),
                                   TaskScript("b2", BEST_EFFORT, (KernelWork("b2_k", cost_model(0.4, 16, 128)),))]))
    S.append(("exempt", G4, 8.0, [TaskScript("hp", HIGH, (KernelWork("hp_k", hp),), arr[:3]),
                                  TaskScript("be", BEST_EFFORT, (KernelWork("be_k", be, exempt=True),))]))
    S.append(("pipeline", G4, 12.0, [
        TaskScript("hp", HIGH, (KernelWork("h1", cost_model(0.3, 2, 128)),
                                KernelWork("h2", cost_model(0.2, 6, 128))), arr[:5]),
        TaskScript("be", BEST_EFFORT, (KernelWork("e1", cost_model(0.05, 40, 128)),
                                       KernelWork("e2", cost_model(0.4, 9, 128)),
                                       KernelWork("e3", cost_model(2.0, 3, 128))))]))
    S.append(("sliced_be", G4, 6.0, [
        TaskScript("hp", HIGH, (KernelWork("hp_k", cost_model(0.2, 1, 128)),), (ms_to_ns(1.1), ms_to_ns(2.9))),
        TaskScript("be", BEST_EFFORT, (KernelWork("be_k", cost_model(0.5, 16, 128)),))]))
    S.append(("be_inference", G4, 10.0, [
        TaskScript("hp", HIGH, (KernelWork("hp_k", hp),), arr[:4]),
        TaskScript("bi", BEST_EFFORT, (KernelWork("bi_k", cost_model(0.3, 8, 128)),),
                   tuple(ms_to_ns(x) for x in (0.1, 0.2, 2.0, 2.05, 6.0)))]))
    varr = tuple(ms_to_ns(x) for x in (0.01, 0.07, 0.08, 0.2, 0.33, 0.34, 0.5, 0.71))
    S.append(("b200_c1", GB, 1.0, [
        TaskScript("hp", HIGH, (KernelWork("vadd", cost_model(0.004, 4096, 256)),), varr),
        TaskScript("be", BEST_EFFORT, (KernelWork("sgemm", cost_model(0.03, 2048, 256)),))]))
    return S


def gen_policy():
    *_, sim, profiler, scheduler, workloads = _ref()
    from tallysim.profiler import Profiler
    from tallysim.scheduler import POLICIES, SchedulerConfig, run_policy
    from tallysim.sim import events_to_csv, ms_to_ns
    out = []
    for name, gpu, hz, tasks in _policy_scenarios():
        runs = 2 if gpu.num_sms > 100 else 10
        prof = Profiler(gpu, runs=runs)
        for pol in POLICIES:
            for seed in ((0, 5) if gpu.num_sms < 100 else (0,)):
                r = run_policy(gpu, tasks, SchedulerConfig(policy=pol), ms_to_ns(hz),
                               profiler=prof, placement_seed=seed)
                csv = events_to_csv(r.events)
                out.append({"scenario": name, "policy": pol, "seed": seed, "runs": runs,
                            "csv_sha256": sha(csv), "n_events": len(r.events),
                            "requests": {k: [list(x) for x in v] for k, v in r.requests.items()},
                            "iterations": r.iterations,
                            "kinds": sorted({e.kind for e in r.events})})
        # threshold variations for Tally
        for th in (10_000, 300_000):
            r = run_policy(gpu, tasks, SchedulerConfig(turnaround_threshold_ns=th), ms_to_ns(hz),
                           profiler=prof, placement_seed=0)
            out.append({"scenario": name, "policy": "Tally", "threshold": th, "seed": 0, "runs": runs,
                        "csv_sha256": sha(events_to_csv(r.events)), "n_events": len(r.events),
                        "requests": {k: [list(x) for x in v] for k, v in r.requests.items()},
                        "iterations": r.iterations})
    return {"runs": out}


def gen_traffic():
    *_, sim, profiler, scheduler, workloads = _ref()
    from tallysim.scheduler import KernelWork
    from tallysim.sim import BEST_EFFORT, HIGH, GpuSpec, cost_model, ms_to_ns
    from tallysim.workloads import (TraceSpec, WorkloadSpec, generate_arrivals, p99_nearest_rank,
                                    report_csv_rows, run_experiment)
    arrivals = []
    for load, lat, dur, seed in ((0.5, 3_925_000, 200_000_000, 0), (0.25, 1_000_000, 50_000_000, 7),
                                 (0.9, 35_000, 5_000_000, 3), (0.5, 40_000, 20_000_000, 11)):
        a = generate_arrivals(load, lat, dur, seed)
        arrivals.append({"load": load, "lat": lat, "dur": dur, "seed": seed, "n": len(a),
                         "sha256": sha(",".join(map(str, a))), "head": list(a[:20])})
    p99 = []
    for xs in (list(range(1, 101)), [5], [3, 1, 2], list(range(1000, 0, -7)), [10] * 150 + [99]):
        p99.append({"xs": xs, "p99": p99_nearest_rank(xs)})
    G4 = GpuSpec(4, 128, 1)
    serve = WorkloadSpec("serve", "inference", HIGH,
                         (KernelWork("serve_k", cost_model(3.925, 1, threads_per_block=128)),),
                         TraceSpec(load=0.5))
    train = WorkloadSpec("train", "training", BEST_EFFORT,
                         (KernelWork("train_k", cost_model(0.15, 108, threads_per_block=128)),))
    reps = run_experiment(G4, [serve, train], ["Tally", "KernelPriority", "Eager", "TimeSliced"],
                          ms_to_ns(400.0), seed=0)
    exp = {"horizon_ms": 400.0, "rows": [row for r in reps for row in report_csv_rows(r)],
           "calibration": {r.policy: {t: [m.p99_latency_ns, m.throughput_per_s, m.completed]
                                      for t, m in r.calibration.items()} for r in reps}}
    return {"arrivals": arrivals, "p99": p99, "experiment": exp}


def main():
    os.makedirs(OUT, exist_ok=True)
    only = sys.argv[1:]
    for name, fn in (("ir", gen_ir), ("transforms", gen_transforms), ("sim", gen_sim),
                     ("tuner", gen_tuner), ("policy", gen_policy), ("traffic", gen_traffic),
                     ("acceptance", gen_acceptance)):
        if only and name not in only:
            continue
        doc = fn()
        doc["_generated_by"] = "oracle/gen_golden.py from /root/reference/pkg/src (tallysim 0.1.0)"
        with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
            json.dump(doc, fh, separators=(",", ":"), sort_keys=True)
        print(name, os.path.getsize(os.path.join(OUT, f"{name}.json")))


if __name__ == "__main__":
    main()

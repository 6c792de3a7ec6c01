"""Real-time co-location on the B200 through the reference-shaped API:
HP vector-add requests at Poisson arrivals + a BE kernel loop, under every
policy.  Needs a B200."""

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_07381_b200 as P
    from paper_2410_07381_b200 import kernels, workloads
    dev = P.B200Device.get(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    n_hp = 1 << 22
    ha, hb, hc = (torch.rand(n_hp, device="cuda", generator=g) for _ in range(3))
    n_be = 1 << 26
    ba, bb, bc = (torch.rand(n_be, device="cuda", generator=g) for _ in range(3))
    hp = kernels.vecadd_f32(ha, hb, hc)
    be = kernels.vecadd_f32(ba, bb, bc)
    return P, workloads, dev, hp, be, (ha, hb, hc, ba, bb, bc)


def _tasks(P, workloads, hp, be, horizon_ns, lat_ns):
    arr = workloads.generate_arrivals(0.3, lat_ns, horizon_ns, seed=1)
    hp_w = P.KernelWork("vadd_hp", hp.cost(), kernel=hp)
    be_w = P.KernelWork("vadd_be", be.cost(), kernel=be)
    return [P.TaskScript("hp", P.HIGH, (hp_w,), arr), P.TaskScript("be", P.BEST_EFFORT, (be_w,))], arr


@pytest.mark.parametrize("policy", ["Tally", "KernelPriority", "Eager", "TimeSliced"])
def test_colocation_runs_every_policy(env, policy):
    P, workloads, dev, hp, be, bufs = env
    prof = P.Profiler(dev.spec, runs=3)
    horizon = 60_000_000
    tasks, arr = _tasks(P, workloads, hp, be, horizon, 200_000)
    res = P.run_policy(dev.spec, tasks, P.SchedulerConfig(policy=policy), horizon, profiler=prof)
    assert len(res.requests["hp"]) == len(arr)
    assert res.iterations["be"], "best-effort made no progress"
    lat = sorted(c - a for a, c in res.requests["hp"])
    assert lat[0] > 0
    kinds = {e.kind for e in res.events}
    assert "LaunchIssued" in kinds and "KernelFinished" in kinds
    if policy == "Tally":
        ptb = [r for r in res.launches if r["shape"] == 2]
        cfg = prof.select(tasks[1].kernels[0].profile_key(), tasks[1].kernels[0].cost)
        if cfg.variant == "Ptb":
            assert ptb and any(r["parked"] for r in ptb)
    torch.cuda.synchronize()
    ha, hb, hc, ba, bb, bc = bufs
    assert torch.equal(hc, ha + hb)
    assert torch.equal(bc, ba + bb)


def test_tally_keeps_hp_tail_close_to_solo(env):
    P, workloads, dev, hp, be, bufs = env
    prof = P.Profiler(dev.spec, runs=3)
    horizon = 150_000_000
    tasks, arr = _tasks(P, workloads, hp, be, horizon, 200_000)
    cfg = P.SchedulerConfig(policy="Tally", turnaround_threshold_ns=60_000)
    solo = P.run_policy(dev.spec, tasks[:1], cfg, horizon, profiler=prof, record_events=False)
    co = P.run_policy(dev.spec, tasks, cfg, horizon, profiler=prof, record_events=False)
    p99 = workloads.p99_nearest_rank
    s = p99([c - a for a, c in solo.requests["hp"]])
    c = p99([c - a for a, c in co.requests["hp"]])
    print(f"solo p99 {s / 1e3:.1f} us, co-located p99 {c / 1e3:.1f} us, "
          f"BE iterations {len(co.iterations['be'])}")
    assert co.iterations["be"]
    if c >= 4 * s + 100_000:   # diagnose: the slowest requests and what BE was doing then
        slow = sorted(((c2 - a2, a2) for a2, c2 in co.requests["hp"]), reverse=True)[:5]
        print("slowest", slow)
    assert c < 4 * s + 100_000


@pytest.mark.parametrize("policy", ["Tally", "KernelPriority", "Eager"])
def test_lookahead_keeps_dependent_kernels_in_order(env, policy):
    """Real-time look-ahead (runner option lookahead=4): a training step of
    dependent kernels -- a chain of large vector adds (tuner: PTB) each
    feeding a small one (Original) -- co-located with HP requests that
    preempt it.  Queued launches behind a parked one must park too (chain
    flag), so every output equals the sequential computation bit for bit,
    and launches really were queued behind in-flight ones."""
    P, workloads, dev, hp, be, bufs = env
    from paper_2410_07381_b200 import kernels
    g = torch.Generator(device="cuda").manual_seed(7)
    nb, ns, depth = 1 << 25, 1 << 18, 6
    b0 = torch.rand(nb, device="cuda", generator=g)
    y = torch.rand(nb, device="cuda", generator=g)
    ys = torch.rand(ns, device="cuda", generator=g)
    big = [torch.empty(nb, device="cuda") for _ in range(depth)]
    small = [torch.empty(ns, device="cuda") for _ in range(depth)]
    works = []
    for k in range(depth):
        kb = kernels.vecadd_f32(b0 if k == 0 else big[k - 1], y, big[k])
        ks = kernels.vecadd_f32(big[k][:ns], ys, small[k])
        works += [P.KernelWork(f"big{k}", kb.cost(), kernel=kb), P.KernelWork(f"small{k}", ks.cost(), kernel=ks)]
    prof = P.Profiler(dev.spec, runs=3)
    horizon = 80_000_000
    arr = workloads.generate_arrivals(0.3, 200_000, horizon, seed=3)
    tasks = [P.TaskScript("hp", P.HIGH, (P.KernelWork("vadd_hp", hp.cost(), kernel=hp),), arr),
             P.TaskScript("be", P.BEST_EFFORT, tuple(works))]
    res = P.run_policy(dev.spec, tasks, P.SchedulerConfig(policy=policy), horizon, profiler=prof,
                       record_events=False, options={"lookahead": 4})
    torch.cuda.synchronize()
    assert len(res.requests["hp"]) == len(arr) and res.iterations["be"]
    ref = b0
    for k in range(depth):
        ref = ref + y
        assert torch.equal(big[k], ref), k
        assert torch.equal(small[k], ref[:ns] + ys), k
    be_l = sorted((r for r in res.launches if r["task"] == 1), key=lambda r: r["issue_ns"])
    queued = sum(1 for a, b in zip(be_l, be_l[1:]) if b["issue_ns"] < a["complete_ns"])
    assert queued > len(be_l) // 4, (queued, len(be_l))
    if policy == "Tally":
        cfgs = {w.kernel_id: prof.select(w.profile_key(), w.cost).variant for w in works}
        print(cfgs)
        if "Ptb" in cfgs.values():
            assert any(r["parked"] for r in be_l)


class _FixedChoices:
    """A tuner stand-in with fixed choices (the B200 run and its replay must
    use the same ones); ``bind`` is the only other call the runner makes."""

    def __init__(self, choices):
        self.choices = choices

    def bind(self, kernel_id, kernel):
        pass

    def select(self, key, cost, threshold_ns=None):
        return self.choices[key.kernel]


@pytest.mark.parametrize("policy", ["Tally", "KernelPriority", "Eager"])
def test_b200_dispatch_decisions_replay_through_reference_runner(env, policy):
    """Dispatch-order parity on hardware: the native runner
    drives the B200 in real time over an HP arrival trace and a best-effort
    pipeline with one PTB, one Sliced and one Original kernel; its logged
    decisions (every submission: task, kernel, shape, workers, resume
    counter, blocks; every preemption) are replayed through the reference
    policy runner (oracle restatement of scheduler.py) with each launch
    completing when and how it did on the B200.  The reference runner must
    make exactly the same decisions in the same order."""
    from fractions import Fraction
    import paper_2410_07381_b200 as P
    from paper_2410_07381_b200 import kernels, workloads
    from oracle import gpu_model as gm
    from oracle import policy as opol
    from oracle import replay as orp
    from oracle import tuner as otu
    _P, _w, dev, hp, _be, _bufs = env
    g = torch.Generator(device="cuda").manual_seed(11)
    sizes = {"be_ptb": 1 << 25, "be_sliced": 1 << 23, "be_orig": 1 << 20}
    bufs, works = {}, []
    for name, n in sizes.items():
        a, b, c = (torch.rand(n, device="cuda", generator=g) for _ in range(3))
        bufs[name] = (a, b, c)
        k = kernels.vecadd_f32(a, b, c)
        works.append(P.KernelWork(name, k.cost(), kernel=k))
    pchoice = {"be_ptb": P.ConfigCandidate("Ptb", worker_count=296),
               "be_sliced": P.ConfigCandidate("Sliced", fraction=Fraction(1, 4)),
               "be_orig": P.ConfigCandidate("Original")}
    horizon = 40_000_000
    arr = workloads.generate_arrivals(0.3, 150_000, horizon, seed=5)
    hp_w = P.KernelWork("vadd_hp", hp.cost(), kernel=hp)
    tasks = [P.TaskScript("hp", P.HIGH, (hp_w,), arr), P.TaskScript("be", P.BEST_EFFORT, tuple(works))]
    res = P.run_policy(dev.spec, tasks, P.SchedulerConfig(policy=policy), horizon,
                       profiler=_FixedChoices(pchoice))
    torch.cuda.synchronize()
    for a, b, c in bufs.values():
        assert torch.equal(c, a + b)
    names = {(0, 0): ("hp", "vadd_hp")}
    names.update({(1, i): ("be", w.kernel_id) for i, w in enumerate(works)})
    ocost = lambda c: gm.KernelCostModel(c.block_duration_ns, c.launch_overhead_ns,   # noqa: E731
                                         c.ptb_iteration_overhead_ns, c.threads_per_block, c.total_blocks)
    otasks = [opol.TaskScript("hp", gm.HIGH, (opol.KernelWork("vadd_hp", ocost(hp_w.cost)),), arr),
              opol.TaskScript("be", gm.BEST_EFFORT, tuple(opol.KernelWork(w.kernel_id, ocost(w.cost)) for w in works))]
    ochoice = {k: otu.ConfigCandidate(v.variant, v.fraction, v.worker_count) for k, v in pchoice.items()}
    sim, ores = orp.replay(gm.GpuSpec(148, 2048, 32), otasks, opol.SchedulerConfig(policy=policy), horizon,
                           res.launches, names, ochoice, res.timers)
    assert sim.mismatch is None, sim.mismatch
    assert len(sim.submitted) == len(res.launches) and not sim.expected
    b200_pre = [(names[(r["task"], r["kernel_index"])][0], names[(r["task"], r["kernel_index"])][1],
                 r["start_count"]) for r in sorted(res.launches, key=lambda r: r["handle"]) if r["preempt_ns"] >= 0]
    assert sim.preempts == b200_pre
    assert len(ores.requests["hp"]) == len(res.requests["hp"]) == len(arr)
    assert len(ores.iterations["be"]) == len(res.iterations["be"])
    if policy == "Tally":
        shapes = {r["shape"] for r in res.launches}
        assert shapes == {0, 1, 2}
        assert b200_pre, "no preemption happened"


@pytest.mark.parametrize("policy", ["Tally", "KernelPriority", "Eager"])
def test_reference_runner_drives_the_b200_through_b200sim(env, policy):
    """The GpuSim surface over the C ABI (b200sim.B200Sim): the reference
    policy runner (oracle restatement of scheduler.py, unchanged) drives the
    B200 in real time -- HP requests complete, BE outputs are exact, and the
    event log has the reference's kinds including per-logical-block
    BlockStarted / BlockFinished from the device clock, each block of every
    finished launch exactly once."""
    from fractions import Fraction
    import collections
    from paper_2410_07381_b200 import b200sim, kernels, workloads
    from oracle import gpu_model as gm
    from oracle import policy as opol
    from oracle import replay as orp
    from oracle import tuner as otu
    _P, _w, dev, hp, _be, _bufs = env
    g = torch.Generator(device="cuda").manual_seed(12)
    sizes = {"be_ptb": 1 << 26, "be_sliced": 1 << 22, "be_orig": 1 << 20}
    bufs, dks = {}, {"vadd_hp": hp}
    for name, n in sizes.items():
        a, b, c = (torch.rand(n, device="cuda", generator=g) for _ in range(3))
        bufs[name] = (a, b, c)
        dks[name] = kernels.vecadd_f32(a, b, c)
    cost = lambda dk: gm.KernelCostModel(1000, 5000, 1000, dk.info.threads_per_block, dk.total_blocks)  # noqa: E731
    horizon = 30_000_000
    arr = workloads.generate_arrivals(0.3, 150_000, horizon, seed=9)
    tasks = [opol.TaskScript("hp", gm.HIGH, (opol.KernelWork("vadd_hp", cost(hp)),), arr),
             opol.TaskScript("be", gm.BEST_EFFORT, tuple(opol.KernelWork(k, cost(dks[k])) for k in sizes))]
    choice = {"be_ptb": otu.ConfigCandidate("Ptb", worker_count=296),
              "be_sliced": otu.ConfigCandidate("Sliced", fraction=Fraction(1, 4)),
              "be_orig": otu.ConfigCandidate("Original")}
    sims = []

    def make(gpu, placement_seed=0, record_events=True):
        s = b200sim.B200Sim(gpu, record_events=record_events, kernels=dks)
        sims.append(s)
        return s
    r = opol.PolicyRunner(dev.spec, tasks, opol.SchedulerConfig(policy=policy), horizon,
                          profiler=orp.FixedProfiler(choice), sim_cls=make)
    r.start_policy_clock()
    res = r.run()
    torch.cuda.synchronize()
    assert len(res.requests["hp"]) == len(arr)
    assert res.iterations["be"]
    for a, b, c in bufs.values():
        assert torch.equal(c, a + b)
    evs = res.events
    kinds = collections.Counter(e.kind for e in evs)
    assert kinds["BlockStarted"] == kinds["BlockFinished"] > 0
    assert kinds["LaunchIssued"] and kinds["KernelFinished"]
    if policy == "Tally":
        assert kinds["PreemptSignaled"]
        parked = [h for h in sims[0].handles if h.parked]
        assert 0 < len(parked) and kinds["WorkerParked"] <= len(parked)
    # every logical block of the Original best-effort kernel: once per launch
    n_orig = sum(1 for e in evs if e.kind == "KernelFinished" and e.kernel == "be_orig")
    fin = collections.Counter(e.block for e in evs if e.kind == "BlockFinished" and e.kernel == "be_orig")
    assert set(fin.values()) == {n_orig} and len(fin) == dks["be_orig"].total_blocks
    assert gm.events_to_csv(evs).startswith("time_ns,kind,task,kernel,block\n")
    assert all(a.time <= b.time for a, b in zip(evs, evs[1:]))
    sims[0].close()

import sys, os
sys.path.insert(0, os.getcwd())
import torch
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
arr = workloads.generate_arrivals(0.3, 200_000, 150_000_000, seed=1)
hp_w = P.KernelWork("vadd_hp", hp.cost(), kernel=hp)
be_w = P.KernelWork("vadd_be", be.cost(), kernel=be)
tasks = [P.TaskScript("hp", P.HIGH, (hp_w,), arr), P.TaskScript("be", P.BEST_EFFORT, (be_w,))]
prof = P.Profiler(dev.spec, runs=3)
cfg = P.SchedulerConfig(policy="Tally", turnaround_threshold_ns=60_000)
prof.bind("vadd_be", be)
for r in prof.profile(be_w.profile_key(), be_w.cost):
    print(r.candidate.describe(), r.kernel_latency_ns, r.turnaround_estimate_ns)
print("select", prof.select(be_w.profile_key(), be_w.cost, 60_000).describe())
co = P.run_policy(dev.spec, tasks, cfg, 150_000_000, profiler=prof, record_events=False)
lat = sorted(((c - a, a) for a, c in co.requests["hp"]), reverse=True)[:5]
print("slowest", lat)
L = co.launches
print(len(L), list(L[0].keys()))
for r in L[:40]:
    print({k: r[k] for k in r})

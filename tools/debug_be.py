"""GPU debugging aid: Tally solo BE (split + sgemm pipeline) progress."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402

dev = P.B200Device.get(0)
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(4096, 4096, device="cuda", generator=g) * 2 - 1
B = torch.rand(4096, 4096, device="cuda", generator=g) * 2 - 1
sg = kernels.sgemm_tf32x3(A, B, torch.zeros(4096, 4096, device="cuda"))
prof = P.Profiler(dev.spec, runs=2)
ws = (P.KernelWork("split_a", sg.split_a.cost(), kernel=sg.split_a),
      P.KernelWork("split_b", sg.split_b.cost(), kernel=sg.split_b),
      P.KernelWork("sgemm", sg.gemm.cost(), kernel=sg.gemm))
for w in ws:
    prof.bind(w.kernel_id, w.kernel)
out = {"choice": {w.kernel_id: prof.select(w.profile_key(), w.cost).describe() for w in ws}}
torch.cuda.synchronize()
be = P.TaskScript("be", P.BEST_EFFORT, ws)
for pol in ("Eager", "Tally"):
    r = P.run_policy(dev.spec, [be], P.SchedulerConfig(policy=pol), 50_000_000, profiler=prof,
                     options={"trace": 1})
    out[pol] = {"iterations": len(r.iterations["be"]), "launches": len(r.launches),
                "first": [{k: x[k] for k in ("kernel_index", "shape", "workers", "count", "submit_ns",
                                              "issue_ns", "gpu_start_ns", "gpu_end_ns", "complete_ns",
                                              "task_counter", "parked")} for x in r.launches[:8]]}
print(json.dumps(out, indent=1))

"""GPU debugging aid: GEMM shape equality at 4096^3, pause/resume, and whether
HP CTAs co-reside with resident (suspended) GEMM workers."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import _lib, kernels  # noqa: E402

out = {}
dev = P.B200Device.get(0)
s = kernels.Stream(high_priority=False)
hs = kernels.Stream(high_priority=True)
g = torch.Generator(device="cuda").manual_seed(9)
M = N = K = 4096
A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).bfloat16()
B = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).bfloat16()
Cm = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
dk = kernels.gemm_bf16(A, B, Cm)
dk.original(s).wait()
ref = Cm.clone()
ref64 = (A.double() @ B.double().T)
out["orig_err"] = ((ref.double() - ref64).abs().max() / ref64.abs().max()).item()
Cm.zero_()
dk.ptb(s, 148).wait()
diff = (Cm != ref).view(32, 128, 32, 128).any(dim=3).any(dim=1)
out["ptb_equal"] = bool(torch.equal(Cm, ref))
out["ptb_bad_tiles"] = int(diff.sum().item())
out["ptb_err"] = ((Cm.double() - ref64).abs().max() / ref64.abs().max()).item()


def launch_pausable(workers=148):
    d = _lib.c_launch_desc(shape=_lib.SHAPE_PTB, workers=workers, start_count=0, preempt_at=-1,
                           pausable=1)
    lid = C.c_int()
    _lib.check(_lib.lib.tally_launch(dk.id, s.id, C.byref(d), C.byref(lid)), "launch")
    return kernels.Launch(lid.value, _lib.SHAPE_PTB)


Cm.zero_()
_lib.check(_lib.lib.tally_set_pause(1), "pause")
L = launch_pausable()
t = P.B200Device.now_ns() + 5_000_000
while P.B200Device.now_ns() < t:
    pass
out["held"] = not L.query().done
_lib.check(_lib.lib.tally_set_pause(0), "resume")
L.wait()
out["pause_equal"] = bool(torch.equal(Cm, ref))
diff = (Cm != ref).view(32, 128, 32, 128).any(dim=3).any(dim=1)
out["pause_bad_tiles"] = int(diff.sum().item())
out["pause_err"] = ((Cm.double() - ref64).abs().max() / ref64.abs().max()).item()

# HP vecadd next to suspended GEMM workers
n = 1 << 24
a, b, c = (torch.rand(n, device="cuda") for _ in range(3))
hp = kernels.vecadd_f32(a, b, c)
solo = []
for _ in range(5):
    solo.append(hp.original(hs, timed=True).elapsed_ns)
out["hp_solo_ns"] = sorted(solo)[2]
_lib.check(_lib.lib.tally_set_pause(1), "pause")
L = launch_pausable()
t = P.B200Device.now_ns() + 2_000_000
while P.B200Device.now_ns() < t:
    pass
t0 = P.B200Device.now_ns()
H = hp.original(hs, timed=True)
deadline = t0 + 50_000_000
while not H.query().done and P.B200Device.now_ns() < deadline:
    pass
out["hp_next_to_suspended_host_us"] = (P.B200Device.now_ns() - t0) / 1e3
out["hp_next_to_suspended_done"] = H.query().done
_lib.check(_lib.lib.tally_set_pause(0), "resume")
out["hp_next_to_suspended_ns"] = H.elapsed_ns
L.wait()
# HP next to a running (not paused) GEMM
L = launch_pausable()
t = P.B200Device.now_ns() + 200_000
while P.B200Device.now_ns() < t:
    pass
H = hp.original(hs, timed=True)
out["hp_next_to_running_ns"] = H.elapsed_ns
L.wait()
print(json.dumps(out, indent=1))

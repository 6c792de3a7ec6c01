import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2410_07381_b200 as P
from paper_2410_07381_b200 import kernels
from tools.ptb_overhead import program
P.B200Device.get(0)
s = kernels.Stream(high_priority=False)
tr = program("c4")
tr.step_original(s)
torch.cuda.synchronize()
seen = set()
for name, dk in tr.program:
    if dk.kind in seen: continue
    seen.add(dk.kind)
    w = dk.full_workers()
    try:
        dk.original(s).wait()
        dk.ptb(s, w).wait()
        print("ok", dk.kind, name, w, dk.info.occupancy_ptb, flush=True)
    except Exception as e:
        print("FAIL", dk.kind, name, w, dk.info.occupancy_ptb, e, flush=True)
        break

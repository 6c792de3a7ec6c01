import sys, os, time, json, random
sys.path.insert(0, os.getcwd())
import torch
import paper_2410_07381_b200 as P
from paper_2410_07381_b200 import kernels, gpt2
P.B200Device.get(0)
hp = gpt2.BertInfer(seq=128)
hs = kernels.Stream(high_priority=True)
res = {}
for label, gap in (("b2b", 0), ("gap1ms", 1e-3), ("gap5ms", 5e-3), ("gap20ms", 20e-3)):
    ts = []
    for i in range(150):
        L = hp.kernel.original(hs, timed=True)
        L.wait()
        ts.append(L.elapsed_ns / 1e3)
        if gap:
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < gap * random.random() * 2:
                pass
    s = sorted(ts)
    res[label] = [round(s[int(q * (len(s) - 1))], 1) for q in (0.1, 0.5, 0.9, 0.99)] + [round(s[-1], 1)]
print(json.dumps(res))

"""Why is a Llama-2-7B decode request slower next to BERT-large training
under Tally?  Times one request (prefill + G decode-step graph launches,
back to back on the high-priority stream, device time by CUDA events) after
different predecessors:

  warm        back-to-back requests
  idle        after 200 ms of an idle GPU
  be_step     after one full BE training step (Original shape)
  be_ptb      after one full BE step in PTB shape (full occupancy)
  concurrent  with the BE step launched right before on the low-priority stream
              (no preemption: what the request sees if BE keeps running)

and through the runner (run_policy, one request, solo vs next to the BE task).

    python tools/c4_probe.py [--gen 16]
"""

from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import bert, kernels, llama  # noqa: E402


def med(xs):
    s = sorted(xs)
    return round(s[len(s) // 2] / 1e3, 1)


def main():
    gen = int(sys.argv[sys.argv.index("--gen") + 1]) if "--gen" in sys.argv else 16
    P.B200Device.get(0)
    be_s = kernels.Stream(high_priority=False)
    hp_s = kernels.Stream(high_priority=True)
    hp = llama.LlamaDecode(prompt=32, gen=gen)
    tr = bert.BertTrain(batch=8, seq=512, lr=1e-3)
    g = torch.Generator(device="cuda").manual_seed(0)
    tr.set_batch(torch.randint(0, tr.V, (8, 512), device="cuda", generator=g),
                 torch.randint(0, tr.V, (8, 512), device="cuda", generator=g))
    pipe = hp.pipeline()

    def request():
        Ls = [dk.original(hp_s, timed=True) for dk in pipe]
        for L in Ls:
            L.wait()
        return sum(L.elapsed_ns for L in Ls), [L.elapsed_ns for L in Ls]

    def be_step(shape):
        Ls = []
        for _, dk in tr.program:
            if shape == "ptb":
                Ls.append(dk.ptb(be_s, dk.full_workers()))
            else:
                Ls.append(dk.original(be_s))
        return Ls

    out = {}
    for _ in range(3):
        request()
        for L in be_step("orig"):
            L.wait()
    res = {k: [] for k in ("warm", "idle", "be_step", "be_ptb", "concurrent")}
    steps = {}
    for _ in range(5):
        request()
        t, s = request()
        res["warm"].append(t)
        steps["warm"] = s
        time.sleep(0.2)
        res["idle"].append(request()[0])
        for L in be_step("orig"):
            L.wait()
        t, s = request()
        res["be_step"].append(t)
        steps["be_step"] = s
        for L in be_step("ptb"):
            L.wait()
        res["be_ptb"].append(request()[0])
        Ls = be_step("orig")
        res["concurrent"].append(request()[0])
        for L in Ls:
            L.wait()
    out["request_device_us_median"] = {k: med(v) for k, v in res.items()}
    out["per_step_us_warm"] = [round(x / 1e3, 1) for x in steps["warm"]]
    out["per_step_us_after_be_step"] = [round(x / 1e3, 1) for x in steps["be_step"]]
    # through the runner: one request solo, then next to the BE task (Tally)
    dev = P.B200Device.get(0)
    prof = P.Profiler(dev.spec, runs=1)
    dec_w = P.KernelWork("decode", hp.decode_kernel.cost(), exempt=True, kernel=hp.decode_kernel)
    hp_pipe = (P.KernelWork("prefill", hp.prefill_kernel.cost(), exempt=True, kernel=hp.prefill_kernel),) + \
        (dec_w,) * gen
    be_ws = []
    for name, dk in tr.program:
        sig = tr.work_signature(name, dk)
        prof.bind(sig, dk)
        be_ws.append(P.KernelWork(sig, dk.cost(), kernel=dk))
    be_task = P.TaskScript("be", P.BEST_EFFORT, tuple(be_ws))
    arr = tuple(int(200e6 + i * 300e6) for i in range(5))
    hp_task = P.TaskScript("hp", P.HIGH, hp_pipe, arr)
    cfg = P.SchedulerConfig(policy="Tally")
    runner = {}
    for label, tasks in (("solo", [hp_task]), ("tally", [hp_task, be_task])):
        r = P.run_policy(dev.spec, tasks, cfg, int(1700e6), profiler=prof, record_events=False, options={"trace": 1})
        lat = [c - a for a, c in r.requests["hp"]]
        hp_l = [x for x in r.launches if x["priority"] == 0 and x["gpu_start_ns"] > 0]
        gaps = [b["gpu_start_ns"] - a["gpu_end_ns"] for a, b in zip(hp_l, hp_l[1:]) if b["gpu_start_ns"] > a["gpu_end_ns"]
                and b["gpu_start_ns"] - a["gpu_end_ns"] < 5e6]
        runs = [x["gpu_end_ns"] - x["gpu_start_ns"] for x in hp_l]
        be_during = 0
        for x in r.launches:
            if x["priority"] != 0 and x["gpu_start_ns"] > 0:
                for a, c in r.requests["hp"]:
                    if a < x["gpu_start_ns"] < c:
                        be_during += 1
                        break
        runner[label] = {"latency_us": [round(x / 1e3) for x in lat], "hp_step_gap_us_median": med(gaps),
                         "hp_step_run_us_median": med(runs), "hp_launches": len(hp_l),
                         "be_launch_starts_inside_requests": be_during}
    out["runner"] = runner
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

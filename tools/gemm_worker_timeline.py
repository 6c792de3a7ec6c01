"""Per-worker timeline of a PTB GEMM launch (worker_log telemetry on the
device clock): entry, first tile in hand, exit, logical blocks run -- where a
persistent tcgen05 GEMM's time goes before / after its tiles.

    python tools/gemm_worker_timeline.py [M N K] [--single]
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    M, N, K = (int(x) for x in args[:3]) if len(args) >= 3 else (4096, 3072, 1024)
    pair = "--single" not in sys.argv
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    A = (torch.randn(M, K, device="cuda") * 0.1).bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.1).bfloat16()
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    dk = kernels.gemm(A, B, C, pair=pair)
    W = 148 * max(1, dk.info.occupancy_ptb)
    out = {"shape": [M, N, K], "kind": dk.kind, "blocks": dk.total_blocks, "workers": W, "runs": []}
    for rep in range(4):
        wl = torch.zeros(W * 4, dtype=torch.int64, device="cuda")
        bl = torch.zeros(dk.total_blocks * 3, dtype=torch.int64, device="cuda")
        L = dk.ptb(s, W, worker_log=wl, timed=True, block_log=bl)
        L.wait()
        if rep == 0:
            continue
        b = bl.view(-1, 3).cpu().tolist()
        per_worker = {}
        for st, en, who in b:
            per_worker.setdefault(who >> 32, []).append((st, en))
        steps, spans = [], []
        for lst in per_worker.values():
            lst.sort()
            steps += [lst[k + 1][0] - lst[k][0] for k in range(len(lst) - 1)]
            spans += [en - st for st, en in lst]
        steps.sort()
        spans.sort()
        w = wl.view(W, 4).cpu().tolist()
        t0 = min(r[1] for r in w)
        entry = sorted((r[1] - t0) / 1e3 for r in w)
        first = sorted((r[2] - t0) / 1e3 for r in w if r[2])
        exit_ = sorted((r[3] - t0) / 1e3 for r in w)
        blocks = [r[0] & 0xffffffff for r in w]
        q = lambda v, f: v[min(len(v) - 1, int(f * len(v)))]
        out["runs"].append({
            "elapsed_us": L.elapsed_ns / 1e3,
            "entry_us_p0_p50_max": [q(entry, 0), q(entry, .5), entry[-1]],
            "first_tile_us_p0_p50_max": [q(first, 0), q(first, .5), first[-1]] if first else None,
            "exit_us_p0_p50_max": [q(exit_, 0), q(exit_, .5), exit_[-1]],
            "blocks_run_hist": {str(b): blocks.count(b) for b in sorted(set(blocks))},
            "smids_distinct": len({r[0] >> 32 for r in w}),
            # block_log: consecutive blocks of one worker -- first-MMA to first-MMA
            "block_step_us_p10_p50_p90": [steps[int(f * (len(steps) - 1))] / 1e3 for f in (.1, .5, .9)] if steps else None,
            "block_first_mma_to_last_store_us_p50": spans[len(spans) // 2] / 1e3 if spans else None,
        })
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Where a PTB launch's fixed cost goes (diagnostics): a spin kernel with one
0-us block per worker, PTB at full occupancy, with the per-worker log
(t_entry, t_exit on %globaltimer) and the launch's own stamps (earliest entry,
last exit = outcome published), against the launch's CUDA-event time; the
untransformed launch with its per-block log for comparison.

    python tools/ptb_timeline.py [--block-us 0] [--per 1]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2410_07381_b200 as P  # noqa: E402
from paper_2410_07381_b200 import kernels  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--block-us", type=float, default=0.0)
    ap.add_argument("--per", type=int, default=1)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    P.B200Device.get(0)
    s = kernels.Stream(high_priority=False)
    probe = kernels.spin(148, 256, 0)
    W = 148 * max(1, probe.info.occupancy_ptb)
    dk = kernels.spin(W * args.per, 256, int(args.block_us * 1000))
    rows = []
    for r in range(args.reps + 2):
        wl = torch.zeros(W, 4, dtype=torch.int64, device="cuda")
        L = dk.ptb(s, W, timed=True, worker_log=wl)
        st = L.wait()
        ev = L.elapsed_ns
        w = wl.cpu()
        t_in, t_out = w[:, 1], w[:, 2]
        bl = torch.zeros(dk.total_blocks, 3, dtype=torch.int64, device="cuda")
        Lo = dk.original(s, timed=True, block_log=bl)
        Lo.wait()
        b = bl.cpu()
        if r < 2:
            continue
        rows.append({
            "ptb_event_us": ev / 1e3,
            "ptb_entry_spread_us": (t_in.max() - t_in.min()).item() / 1e3,
            "ptb_loop_span_us": (t_out.max() - t_in.min()).item() / 1e3,
            "ptb_exit_path_us": (st.gt_last_exit - t_out.max().item()) / 1e3,
            "ptb_first_start_vs_min_entry_us": (st.gt_first_start - t_in.min().item()) / 1e3,
            "orig_event_us": Lo.elapsed_ns / 1e3,
            "orig_block_span_us": (b[:, 1].max() - b[:, 0].min()).item() / 1e3,
        })
    med = {k: sorted(r[k] for r in rows)[len(rows) // 2] for k in rows[0]}
    print(json.dumps({"workers": W, "blocks": dk.total_blocks, "block_us": args.block_us, "median": med}, indent=1))


if __name__ == "__main__":
    main()

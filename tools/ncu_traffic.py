"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) from
an ncu --set full report of `tools/ncu_c2.py kernels NAME...` (each name
launched Original, then PTB at full occupancy), merged into
profiles/ncu_traffic.json under keys "<config>:<name>:Original" and
"<config>:<name>:Ptb(full occupancy)" -- what bench.py reports as
roofline.traffic -- and a one-line-per-launch summary on stdout.

    python tools/ncu_traffic.py REPORT.ncu-rep c2 NAME [NAME ...]
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, config, names = sys.argv[1], sys.argv[2], sys.argv[3:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[0], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, k):
        return float(r[col[k]].replace(",", ""))
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    db = json.load(open(path))
    shapes = ["Original", "Ptb(full occupancy)"]
    for i, r in enumerate(data):
        name, shape = names[i // 2], shapes[i % 2]
        t = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        db[f"{config}:{name}:{shape}"] = int(t)
        print(f"{name:32s} {shape:20s} {val(r, 'gpu__time_duration.sum') / 1e3:9.1f} us  "
              f"dram {t / 1e6:9.1f} MB  {r[col['Kernel Name']][:70]}")
    json.dump(db, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()

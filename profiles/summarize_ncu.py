#!/usr/bin/env python
"""Summarise ncu outputs into the markdown tables kept under profiles/.

    python profiles/summarize_ncu.py launches <launches.csv>
    python profiles/summarize_ncu.py full <report.ncu-rep>

`launches`: share of device time per kernel from a
`--metrics gpu__time_duration.sum --csv --log-file` capture (cold-cache,
serialised launches: compare shares, not absolutes).
`full`: the key counters of every kernel in a `--set full` report.
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp insts"),
]


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["| share | launches | avg us | kernel |", "|---:|---:|---:|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {100 * sum(v) / tot:.1f}% | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | `{k}` |")
    return "\n".join(out)


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    out = ["| kernel | " + " | ".join(n for _, n in FULL_METRICS) + " |",
           "|---|" + "---:|" * len(FULL_METRICS)]
    for r in rows[2:]:
        cells = []
        for m, _ in FULL_METRICS:
            i = idx.get(m)
            cells.append(f"{r[i]} {units[i]}".strip() if i is not None else "n/a")
        out.append(f"| `{r[idx['Kernel Name']]}` | " + " | ".join(cells) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))

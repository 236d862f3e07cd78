#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, total device time and share of the step.

    python tools/launch_summary.py gpurun_out/launches_r01.csv > profiles/launches_r01_summary.json

ncu serialises launches and runs them cold-cache, so absolute times exceed
the in-situ ones; the shares are what to compare against bench.py.
"""

from __future__ import annotations

import csv
import json
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    m = re.search(r"hx::(\w+)", name) or re.search(r"(\w+_kernel)", name)
    base = m.group(1) if m else name[:48]
    t = re.search(r"<([^>]*)>", name)
    return f"{base}<{t.group(1)}>" if t else base


def main(path: str) -> None:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[iu], 1e-6)
        k = short(r[ik])
        per[k][0] += 1
        per[k][1] += v * scale
    total = sum(v[1] for v in per.values())
    out = {"source": path, "total_ms": total, "launches": sum(v[0] for v in per.values()),
           "kernels": {k: {"launches": n, "ms": ms, "share": ms / total}
                       for k, (n, ms) in sorted(per.items(), key=lambda kv: -kv[1][1])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])

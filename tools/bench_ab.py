#!/usr/bin/env python
"""In-step A/B of library builds or runtime knobs: alternating `bench.py` runs on
one box, since the B200's power cap makes isolated kernel timings mislead
(DRAM traffic and clocks change with the variant).

    python tools/bench_ab.py cur=HX_LIB=tools/bin/libhx_cur.so \\
                             band1=HX_LIB=tools/bin/libhx_band1.so [--rounds 2] [-- bench args]
    python tools/bench_ab.py auto=HX_GEMM_GROUP=0 old=HX_GEMM_GROUP=16

Each variant is NAME=VAR=VALUE[,VAR=VALUE...]; one line per run with tokens/s,
SM clock, value per MHz, the attention kernels' in-step times and the GEMM time
per step (from bench.py's roofline / kernel_share keys).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    argv = sys.argv[1:]
    extra = []
    if "--" in argv:
        i = argv.index("--")
        argv, extra = argv[:i], argv[i + 1:]
    rounds = 2
    if "--rounds" in argv:
        i = argv.index("--rounds")
        rounds = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    variants = []
    for spec in argv:
        name, _, assigns = spec.partition("=")
        env = dict(a.split("=", 1) for a in assigns.split(",") if a)
        variants.append((name, env))
    base = ["--compare-1f1b", "no", "--no-cpu-baseline", "--no-e2e", *extra]
    for r in range(rounds):
        order = variants if r % 2 == 0 else variants[::-1]
        for name, env in order:
            out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *base], capture_output=True, text=True,
                                 env={**os.environ, **env}, timeout=900)
            lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
            if not lines:
                print(json.dumps({"variant": name, "error": out.stderr[-400:]}), flush=True)
                continue
            d = json.loads(lines[-1])
            ks, roof, mhz = d.get("kernel_share") or {}, d.get("roofline") or {}, d["clocks"]["sm_mhz"]
            print(json.dumps({"variant": name, "tokens_per_s": round(d["value"]), "sm_mhz": mhz,
                              "per_mhz": round(d["value"] / mhz, 2) if mhz else None,
                              "attn_bwd_ms": round(roof.get("attn_bwd_ms", 0), 3),
                              "attn_fwd_ms": round((roof.get("attn_fwd") or {}).get("ms", 0), 3),
                              "gemm_ms_per_step": round((ks.get("gemm") or {}).get("ms_per_step", 0), 1)}),
                  flush=True)


if __name__ == "__main__":
    main()

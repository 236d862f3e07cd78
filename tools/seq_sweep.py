#!/usr/bin/env python
"""BASELINE config 5: sequence-length sweep on one B200 (measured p = 1) with the
helix vs 1F1B pipeline prediction at p = 2/4/8 from the measured component times.

    python tools/seq_sweep.py [--workload gpt3b_64k] [--seqs 16384,32768,65536,98304,131072]
                              [--out profiles/r01_seq_sweep.json]

Each point is one `bench.py` run (helix two-fold + recompute, chunked MLP, host
offload when the stash does not fit); the JSON collects measured tokens/s, MFU,
same-kernel 1F1B + rc at p = 1, and the predicted tokens/s / bubble of
helix_twofold(_rc) and 1f1b(_rc) at p = 2/4/8.
"""

from __future__ import annotations

import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt3b_64k")
    ap.add_argument("--seqs", default="16384,32768,65536,98304,131072")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r01_seq_sweep.json"))
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    points = []
    for s in [int(x) for x in args.seqs.split(",")]:
        cmd = [sys.executable, str(ROOT / "bench.py"), "--workload", args.workload, "--seq", str(s),
               "--method", "helix_twofold_rc", "--mlp-chunk", "8192", "--steps", str(args.steps),
               "--warmup", str(args.warmup), "--no-cpu-baseline", "--no-e2e", "--stash-budget-gb", "-1"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
        if r.returncode != 0 or not lines:
            points.append({"s": s, "error": (r.stderr or r.stdout)[-800:]})
            print(json.dumps(points[-1]), flush=True)
            continue
        d = json.loads(lines[-1])
        pred = (d.get("bubble_predicted_by_reference_model") or {}).get("pipeline_prediction", {})
        pt = {"s": s, "tokens_per_s": d["value"], "mfu": d["mfu"], "ms_per_step": d["ms_per_step"],
              "max_memory_gb": d["max_memory_gb"], "clocks": d["clocks"],
              "same_kernel_1f1b": d.get("baseline_1f1b_same_kernels"),
              "offload": d.get("stash_offload"),
              "predicted": {p: {m: {k: v[k] for k in ("tokens_per_s", "bubble_fraction") if k in v}
                                | {k: v[k] for k in ("speedup_vs_1f1b", "speedup_vs_1f1b_rc") if k in v}
                                for m, v in row.items()} for p, row in pred.items()}}
        points.append(pt)
        print(json.dumps({k: pt[k] for k in ("s", "tokens_per_s", "mfu", "max_memory_gb")}), flush=True)
    out = {"workload": args.workload, "method": "helix_twofold_rc", "mlp_chunk": 8192, "points": points}
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()

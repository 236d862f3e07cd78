#!/usr/bin/env python
"""The reference's own execute_schedule timed at BASELINE config 1's model
(SURVEY 8d "CPU reference timing"): helix_twofold, helix_twofold_rc and 1f1b
at p in {1, 2, 4, 8} (L = max(4, p), m = 2p), replay (1 core) and threaded
(p stage threads) drivers, with the threaded wait timeout raised
(P/runtime/executor.py:56).  Uses pipelab from baseline/_ref (unmodified).

    python tools/cpu_reference_sweep.py --out profiles/r02_cpu_reference_sweep.json [--jobs 4]
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def one(job):
    method, p, threaded = job
    os.environ["OMP_NUM_THREADS"] = "1"
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    import pipelab.runtime.executor as ex
    from pipelab import ModelConfig, generate
    from pipelab.costs import DurationTable
    from pipelab.runtime import execute_schedule, make_inputs, make_model
    ex._WAIT_TIMEOUT = 1e9
    cfg = ModelConfig(L=max(4, p), h=256, s=1024, b=1, num_heads=4, p=p, m=2 * p)
    base = method.removesuffix("_rc") if method == "helix_twofold_rc" else method
    sched = generate(method, cfg, DurationTable.from_units(1, 3, 2))
    P, X = make_model(cfg, 0), make_inputs(cfg, 1)
    t0 = time.perf_counter()
    r = execute_schedule(sched, P, X, threaded=threaded)
    wall = time.perf_counter() - t0
    tokens = cfg.m * cfg.s * cfg.b
    return {"method": method, "p": p, "L": cfg.L, "m": cfg.m, "driver": "threaded" if threaded else "replay",
            "seconds": wall, "tokens_per_s": tokens / wall, "losses": r.losses, "_base": base}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r02_cpu_reference_sweep.json")
    ap.add_argument("--jobs", type=int, default=4)
    ap.add_argument("--stages", default="1,2,4,8")
    args = ap.parse_args()
    jobs = [(m, p, thr) for p in map(int, args.stages.split(",")) for m in ("helix_twofold", "helix_twofold_rc", "1f1b")
            for thr in (False, True)]
    rows = []
    with ProcessPoolExecutor(args.jobs) as ex:
        for row in ex.map(one, jobs):
            row.pop("_base")
            rows.append(row)
            print(json.dumps(row), flush=True)
    out = {"what": "reference pipelab execute_schedule at BASELINE config 1's model (h=256, heads=4, s=1024, b=1), "
                   "L=max(4,p), m=2p, DurationTable.from_units(1,3,2), make_model seed 0 / make_inputs seed 1",
           "host": {"cpu_model": next((ln.split(":", 1)[1].strip() for ln in Path("/proc/cpuinfo").read_text().splitlines()
                                       if ln.startswith("model name")), "unknown"),
                    "nproc": os.cpu_count(), "python": platform.python_version(), "concurrent_jobs": args.jobs},
           "rows": rows}
    Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

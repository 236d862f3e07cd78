#!/usr/bin/env python
"""SURVEY 8(d)'s CPU-reference timing grid at the tiny shape, and the same grid
on the B200.

The reference's own ``execute_schedule`` (``P/runtime/executor.py:425-440``) is
timed in replay and threaded mode for helix_twofold, helix_twofold_rc and 1f1b
at p in {1, 2, 4, 8} (L = max(4, p), m = 2p, h=256, heads=4, s=1024, b=1;
params ``make_model(cfg, 0)``, inputs ``make_inputs(cfg, 1)``), with
``_WAIT_TIMEOUT`` raised (``:56``; SURVEY 8(d) caveat: p=8 threaded otherwise
aborts).  ``--side gpu`` runs the same grid through this package's
``execute_schedule`` on one B200 (all stages on one device, as the reference's
replay mode) and through ``HelixRuntime`` device-timed, and compares its losses
with the reference's from ``--ref-jsonl``.

    python tools/config1_grid.py --side ref [--ps 1,2,4,8] > profiles/r02_config1_grid_ref_box.jsonl
    python tools/config1_grid.py --side gpu --ref-jsonl profiles/r02_config1_grid_ref_box.jsonl

The reference side imports pipelab from ``baseline/_ref`` (the unmodified
installed reference); it is a measurement tool, not part of the product path.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METHODS = ("helix_twofold", "helix_twofold_rc", "1f1b")


def grid(ps):
    for p in ps:
        for method in METHODS:
            yield p, method, dict(L=max(4, p), h=256, s=1024, b=1, num_heads=4, p=p, m=2 * p)


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def side_ref(ps, modes):
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    import pipelab
    from pipelab import DurationTable, ModelConfig, generate
    from pipelab.runtime import execute_schedule, make_inputs, make_model
    from pipelab.runtime import executor as ex

    ex._WAIT_TIMEOUT = 1e9
    host = {"cpu_model": cpu_model(), "nproc": os.cpu_count(), "pipelab": pipelab.__file__}
    for p, method, kw in grid(ps):
        cfg = ModelConfig(**kw)
        sched = generate(method, cfg, DurationTable.from_units(1, 3, 2))
        P, X = make_model(cfg, 0), make_inputs(cfg, 1)
        for threaded in modes:
            t0 = time.perf_counter()
            res = execute_schedule(sched, P, X, threaded=threaded)
            wall = time.perf_counter() - t0
            tokens = cfg.m * cfg.s * cfg.b
            print(json.dumps({"side": "reference", "method": method, "p": p, "config": kw,
                              "mode": "threaded" if threaded else "replay", "wall_s": wall,
                              "tokens_per_s": tokens / wall, "losses": list(res.losses),
                              "peak_stash_elements": list(res.peak_stash_elements), **host}), flush=True)


def side_gpu(ps, ref_jsonl):
    sys.path.insert(0, str(ROOT))
    import torch
    from paper_2507_00394_b200 import ModelConfig, generate
    from paper_2507_00394_b200.costs import DurationTable
    from paper_2507_00394_b200.runtime import execute_schedule, make_inputs, make_model
    from paper_2507_00394_b200.runtime.executor import DeviceModel, HelixRuntime

    ref = {}
    if ref_jsonl and Path(ref_jsonl).exists():
        for ln in open(ref_jsonl):
            if ln.startswith("{"):
                r = json.loads(ln)
                ref[(r["method"], r["p"])] = r["losses"]
    dev = torch.device("cuda:0")
    for p, method, kw in grid(ps):
        cfg = ModelConfig(**kw)
        sched = generate(method, cfg, DurationTable.from_units(1, 3, 2))
        P, X = make_model(cfg, 0), make_inputs(cfg, 1)
        tokens = cfg.m * cfg.s * cfg.b
        out = {"side": "b200", "method": method, "p": p, "config": kw}
        for _ in range(2):
            res = execute_schedule(sched, P, X)
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            res = execute_schedule(sched, P, X)
        wall = (time.perf_counter() - t0) / reps
        out["execute_schedule"] = {"wall_s": wall, "tokens_per_s": tokens / wall,
                                   "how": "drop-in call: float64 host fixtures in, numpy RunResult out"}
        if (method, p) in ref:
            out["loss_max_rel_err_vs_reference"] = max(abs(a - b) / abs(b) for a, b in zip(res.losses, ref[(method, p)]))
        model = DeviceModel.from_host(sched, P, range(cfg.p), dev)
        rt = HelixRuntime(sched, model, None, "multistream", dev)
        xs = [torch.from_numpy(x).to(dev, torch.bfloat16).reshape(cfg.s * cfg.b, cfg.h) for x in X]
        for _ in range(3):
            rt.run(xs)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            rt.run(xs)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        out["device"] = {"ms_per_step": ms, "tokens_per_s": tokens / (ms / 1e3),
                         "how": "HelixRuntime multistream, all p stages on one GPU, CUDA events"}
        try:
            g = rt.capture(xs)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            a.record()
            for _ in range(10):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            gms = a.elapsed_time(b) / 10
            out["device_cuda_graph"] = {"ms_per_step": gms, "tokens_per_s": tokens / (gms / 1e3)}
        except Exception as e:  # noqa: BLE001 -- reported per row
            out["device_cuda_graph"] = {"error": f"{type(e).__name__}: {e}"[:200]}
        print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", choices=("ref", "gpu"), required=True)
    ap.add_argument("--ps", default="1,2,4,8")
    ap.add_argument("--modes", default="replay,threaded")
    ap.add_argument("--ref-jsonl", default=str(ROOT / "profiles" / "r02_config1_grid_ref_box.jsonl"))
    args = ap.parse_args()
    ps = [int(x) for x in args.ps.split(",")]
    if args.side == "ref":
        side_ref(ps, [m == "threaded" for m in args.modes.split(",")])
    else:
        side_gpu(ps, args.ref_jsonl)


if __name__ == "__main__":
    main()

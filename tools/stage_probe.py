#!/usr/bin/env python
"""One rank of a p-stage pipeline on one B200 (HelixRuntime mode "probe").

Runs stage r's tasks of the p-stage schedule at the real per-stage shapes with
loopback communication (executor._Loopback: receives are fresh payload buffers
of the wire layout, sends are checked and dropped), and reports

* measured device memory (torch max_memory_allocated, the executor's distinct
  stash bytes) next to runtime/memplan.py's plan for that rank;
* the rank's busy time (sum of compute-task device times) and per-component
  durations, with the simulator's makespan prediction from them.

Used for the per-rank memory model at BASELINE configs 3-4 and the "does plain
1F1B fit at 3B/64k, p=8" question (round-2 verdict items 6-7).

    python tools/stage_probe.py --workload gpt3b_64k --p 8 --stage 0 --method 1f1b
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2507_00394_b200 import ModelConfig, generate  # noqa: E402
from paper_2507_00394_b200.costs import DurationTable  # noqa: E402
from paper_2507_00394_b200.partition import pre_stage  # noqa: E402
from paper_2507_00394_b200.runtime import HelixRuntime  # noqa: E402
from paper_2507_00394_b200.runtime.executor import DeviceModel, stage_fields  # noqa: E402
from paper_2507_00394_b200.runtime.memplan import GB, plan  # noqa: E402
from paper_2507_00394_b200.runtime.model import DeviceLayer, random_device_layer  # noqa: E402
from paper_2507_00394_b200.engine import CommModel  # noqa: E402
from paper_2507_00394_b200.simulate import (measured_durations, simulate, simulate_classes,  # noqa: E402
                                            task_class_durations)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt3b_64k", choices=sorted(WORKLOADS))
    ap.add_argument("--L", type=int, default=None, help="override the layer count (reduced-L probes)")
    ap.add_argument("--seq", type=int, default=None, help="override the sequence length (sweeps)")
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--stage", type=int, nargs="+", default=[0])
    ap.add_argument("--method", default="helix_twofold_rc")
    ap.add_argument("--mlp-chunk", type=int, default=None)
    ap.add_argument("--regen-pre-x", action="store_true")
    ap.add_argument("--stash-budget-gb", type=float, default=None)
    ap.add_argument("--iters", type=int, default=2, help="the last one is measured")
    ap.add_argument("--stream-inputs", action="store_true",
                    help="keep the inputs in pinned host memory (the runtime's input streamer)")
    args = ap.parse_args()

    wl = dict(WORKLOADS[args.workload])
    if args.L:
        wl["L"] = args.L
    if args.seq:
        wl["s"] = args.seq
    cfg = ModelConfig(L=wl["L"], h=wl["h"], s=wl["s"], b=wl["b"], num_heads=wl["num_heads"], p=args.p, m=2 * args.p)
    units = DurationTable.from_units(1, 3, 2)
    sched = generate(args.method, cfg, units)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    chunked = any(t.comp == "chunk" for t in sched.tasks.values() if t.is_compute)
    for stage in args.stage:
        gen = torch.Generator(device=dev).manual_seed(1234)
        layers = {}
        for l in range(cfg.L):
            need, own = stage_fields(sched, stage, l)
            if need:
                full = random_device_layer(cfg.h, gen, dev)
                layers[l] = DeviceLayer({k: v for k, v in full.items() if k in need},
                                        tuple(k for k in full if k in own))
                del full
        budget = None if args.stash_budget_gb is None else int(args.stash_budget_gb * GB)
        rt = HelixRuntime(sched, DeviceModel(layers), args.mlp_chunk, "probe", dev, rank=stage,
                          stash_budget_bytes=budget, regen_pre_x=args.regen_pre_x, record_timeline=True)
        first = 0 if chunked else pre_stage(0, cfg)
        ig = torch.Generator(device=dev).manual_seed(1)
        T = cfg.s * cfg.b
        inputs = [torch.randn(T, cfg.h, generator=ig, device=dev).to(torch.bfloat16) if stage == first else None
                  for _ in range(cfg.m)]
        if args.stream_inputs:
            inputs = [None if x is None else x.cpu().pin_memory() for x in inputs]
        try:
            for it in range(args.iters):
                torch.cuda.synchronize()
                if it == args.iters - 1:
                    torch.cuda.reset_peak_memory_stats(dev)
                t0 = time.perf_counter()
                rt.run(inputs)
                torch.cuda.synchronize()
                wall = time.perf_counter() - t0
        except torch.OutOfMemoryError as e:
            pl = plan(sched, stage, args.mlp_chunk, regen_pre_x=args.regen_pre_x, durations=units)
            print(json.dumps({"probe": "stage", "workload": args.workload, "L": cfg.L, "p": cfg.p,
                              "method": args.method, "stage": stage, "mlp_chunk": args.mlp_chunk,
                              "oom": str(e).splitlines()[0][:200],
                              "max_memory_allocated_gb": torch.cuda.max_memory_allocated(dev) / GB,
                              "plan_gb": pl.as_gb()}), flush=True)
            continue
        tl = rt.timeline
        busy = sum(e - s for tid, (s, e) in tl.items())
        span = max(e for _s, e in tl.values()) - min(s for s, _e in tl.values())
        table = measured_durations(sched, tl) if not chunked else None
        st = rt.stages[stage]
        pl = plan(sched, stage, args.mlp_chunk, regen_pre_x=args.regen_pre_x, durations=table or units,
                  stream_inputs=args.stream_inputs)
        out = {
            "probe": "stage", "workload": args.workload, "L": cfg.L, "h": cfg.h, "s": cfg.s, "p": cfg.p, "m": cfg.m,
            "method": args.method, "stage": stage, "mlp_chunk": args.mlp_chunk, "regen_pre_x": args.regen_pre_x,
            "stash_budget_gb": args.stash_budget_gb,
            "measured": {"max_memory_allocated_gb": torch.cuda.max_memory_allocated(dev) / GB,
                         "stash_peak_gb": st.peak_bytes / GB, "stash_peak_at": st.peak_bytes_at,
                         "busy_ms": busy, "device_span_ms": span, "wall_s": wall,
                         "offload": rt.offload_stats()},
            "plan_gb": pl.as_gb(),
            "tokens_per_s_if_busy_bound": cfg.m * cfg.s * cfg.b / (busy / 1e3),
        }
        classes = task_class_durations(sched, tl)
        out["task_class_ns"] = classes
        # the reference list scheduler over the whole p-stage schedule with these
        # measured per-class durations (every stage runs the same shapes), NVLink comm
        comm = CommModel("bytes", latency=5000, bytes_per_element=2, bandwidth=int(770e9))
        sim_c = simulate_classes(sched, classes, comm)
        out["predicted_from_classes"] = {"makespan_ms": sim_c.metrics.makespan / 1e6,
                                         "bubble_fraction": sim_c.metrics.bubble_fraction,
                                         "tokens_per_s": cfg.m * cfg.s * cfg.b / (sim_c.metrics.makespan * 1e-9)}
        if table is not None:
            sim = simulate(generate(args.method, cfg, table), table)
            out["durations_ns"] = {f"{c}.{ps}": v for (c, ps), v in table.entries.items()}
            out["simulated_makespan_ms"] = sim.metrics.makespan / 1e6
            out["simulated_bubble_fraction"] = sim.metrics.bubble_fraction
        print(json.dumps(out), flush=True)
        del rt, layers, inputs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

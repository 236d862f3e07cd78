#!/usr/bin/env python
"""p = 8 makespan predictions from stage-probe measurements (profiles/*.jsonl).

Each probe ran one rank of the 8-stage pipeline on one B200 at the real
per-stage shapes (tools/stage_probe.py) and recorded the device time of every
task class (FWD.attn, BWD_B.post, RECOMPUTE_FWD.post, FWD.chunk.x2, ...).  The
reference's list scheduler (P/engine.py, restated in engine.py) replays the
whole p-stage schedule with those durations and NVLink transfers modelled at
770 GB/s per direction + 5 us.  1F1B chunk classes measured at a reduced L
scale linearly with the layers per chunk.  Predictions, not measurements.

    python tools/predict_from_probes.py > profiles/r02_pipeline_predictions.json
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_00394_b200 import ModelConfig, generate  # noqa: E402
from paper_2507_00394_b200.costs import DurationTable  # noqa: E402
from paper_2507_00394_b200.engine import CommModel  # noqa: E402
from paper_2507_00394_b200.simulate import simulate_classes  # noqa: E402

SHAPES = {"gpt3b_64k": dict(L=16, h=4096, s=65536, b=1, num_heads=32),
          "gpt7b_128k": dict(L=32, h=4096, s=131072, b=1, num_heads=32)}
COMM = CommModel("bytes", latency=5000, bytes_per_element=2, bandwidth=int(770e9))


def load():
    rows = []
    for f in sorted((ROOT / "profiles").glob("r02_stage_probes_*.jsonl")):
        for ln in f.read_text().splitlines():
            d = json.loads(ln)
            if d.get("task_class_ns") and not d.get("oom"):
                d["_file"] = f.name
                rows.append(d)
    return rows


def scaled(classes: dict, L_probe: int, p: int, L: int) -> dict:
    """Chunk classes measured with L_probe/p layers per chunk, at L/p."""
    out = {}
    for k, v in classes.items():
        if ".chunk.x" in k:
            base, span = k.rsplit(".x", 1)
            out[f"{base}.x{L // p}"] = int(v * (L // p) / int(span))
        else:
            out[k] = v
    return out


def main():
    rows = load()
    units = DurationTable.from_units(1, 3, 2)
    out = {}
    keys = [(wl, shape) for wl, shape in SHAPES.items()]
    # sequence-sweep probes (BASELINE config 5): one entry per probed length
    for r in rows:
        if r["workload"] == "gpt3b_64k" and r["s"] != SHAPES["gpt3b_64k"]["s"]:
            k = (f"gpt3b_s{r['s']}", dict(SHAPES["gpt3b_64k"], s=r["s"]))
            if k not in keys:
                keys.append(k)
    for wl, shape in keys:
        cfg = ModelConfig(**shape, p=8, m=16)
        res = {}
        for r in rows:
            base = "gpt3b_64k" if wl.startswith("gpt3b") else wl
            if r["workload"] != base or r["stage"] != 0 or r["s"] != cfg.s:
                continue
            key = r["method"] + (" +regen_pre_x" if r.get("regen_pre_x") else "") + \
                (" +offload" if r.get("stash_budget_gb") else "")
            cls = scaled(r["task_class_ns"], r["L"], r["p"], cfg.L)
            sim = simulate_classes(generate(r["method"], cfg, units), cls, COMM)
            res[key] = {"makespan_ms": sim.metrics.makespan / 1e6, "bubble_fraction": sim.metrics.bubble_fraction,
                        "tokens_per_s": cfg.m * cfg.s * cfg.b / (sim.metrics.makespan * 1e-9),
                        "probe_L": r["L"], "probe_busy_ms": r["measured"]["busy_ms"],
                        "probe_max_memory_gb": r["measured"]["max_memory_allocated_gb"], "source": r["_file"]}
        for a in [k for k in res if k.startswith("helix")]:
            for b in [k for k in res if k.startswith("1f1b")]:
                res[a][f"speedup_vs_{b}"] = res[b]["makespan_ms"] / res[a]["makespan_ms"]
        out[wl] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

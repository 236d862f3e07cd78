#!/usr/bin/env python
"""Condense ncu reports into profiles/ncu_summary.json (+ a readable table).

    python tools/ncu_summary.py gpurun_out/prof_attn_r01.ncu-rep [more.ncu-rep ...] \
        [--out profiles/ncu_summary.json] [--tag r01]

Per kernel (first launch of each name): duration, tensor-pipe active %, DRAM
bytes read+write (the roofline 'traffic'), registers, achieved occupancy and the
top warp-stall reasons.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from pathlib import Path

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "tensor_active_pct": ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    "mem_tensor_active_pct": ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_read": ("dram__bytes_read.sum", 1),
    "dram_write": ("dram__bytes_write.sum", 1),
    "registers": ("launch__registers_per_thread", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_reduce_input_pct": ("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed", 1),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
              "usecond": 1e3, "msecond": 1e6, "nsecond": 1}


def short(name: str) -> str:
    m = re.search(r"(attn_\w+|gemm_sm100_kernel|gemm_2sm_kernel|ln_\w+_kernel|mse_loss_kernel|axpy_f32_kernel)", name)
    base = m.group(1) if m else name[:40]
    t = re.search(r"<([^>]*)>", name)
    return f"{base}<{t.group(1)}>" if t else base


def summarize(rep: Path) -> dict:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    for h, i in list(col.items()):  # section-prefixed names (e.g. "TPC.TriageCompute.<metric>")
        col.setdefault(h.split(".", 2)[-1] if h.count(".") >= 3 and h.split(".")[0].isupper() else h, i)
    out = {}
    for r in rows[2:]:
        name = short(r[col["Kernel Name"]])
        if name in out:
            continue
        rec = {}
        for key, (metric, _scale) in KEYS.items():
            if metric in col:
                try:
                    v = float(r[col[metric]].replace(",", ""))
                except ValueError:
                    continue
                u = units[col[metric]]
                if key.startswith("dram_r") or key.startswith("dram_w"):
                    v *= UNIT_SCALE.get(u, 1)
                if key == "duration_ms":
                    v = v * UNIT_SCALE.get(u, 1) / 1e6
                rec[key] = v
        stalls = {}
        for h, i in col.items():
            m = re.match(r"smsp__average_warp_latency_issue_stalled_(\w+)\.ratio$", h) or \
                re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", h)
            if m:
                try:
                    stalls[m.group(1)] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        if stalls:
            tot = sum(stalls.values()) or 1.0
            rec["top_stalls"] = {k: round(v / tot, 3) for k, v in
                                 sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        if "dram_read" in rec and "dram_write" in rec:
            rec["dram_bytes"] = rec["dram_read"] + rec["dram_write"]
        out[name] = rec
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--out", default="profiles/ncu_summary.json")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    outp = Path(args.out)
    data = json.loads(outp.read_text()) if outp.exists() else {}
    for rep in args.reports:
        for name, rec in summarize(Path(rep)).items():
            rec["report"] = Path(rep).name
            rec["tag"] = args.tag
            data[name] = rec
            # convenient aliases for bench.py's roofline 'traffic'
            if name.startswith("attn_bwd_fused_kernel"):
                data["attn_bwd"] = rec
            if name.startswith("attn_fwd_kernel"):
                data["attn_fwd"] = rec
            print(f"{name:40s} " + " ".join(
                f"{k}={v:.4g}" if isinstance(v, float) else f"{k}={v}" for k, v in rec.items()
                if k not in ("report", "tag")))
    outp.parent.mkdir(parents=True, exist_ok=True)
    outp.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()

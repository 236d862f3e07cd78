#!/usr/bin/env python
"""HelixPipe stage-execution benchmark (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per stage)

Workload (BASELINE.json metric, configs[1] = GPT-1.3B at seq 32k): L=24,
h=2048, 16 heads, s=32768, b=1, helix two-fold FILO with p = N stages and
m = 2N micro-batches, so per-GPU work (L*m/p = 48 layer-micro-batches) is
fixed as N grows ("scaling": "weak").  One step = one full schedule iteration:
every micro-batch forward and backward through all layers with gradient
accumulation (the reference has no optimizer step, P/runtime/executor.py:386-422).
Random-init weights of that architecture and N(0,1) synthetic inputs, bf16
compute with fp32 accumulation.  Activations are far larger than the 126 MB L2
(134 MB per tensor), so no L2 flush is needed between steps.

value  = m*s*b tokens / step, device-timed with CUDA events (max over ranks)
e2e    = same iteration through HelixRuntime with pinned-host inputs copied in
         and the losses read back inside the timed region
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tokens/s (device-timed, max over ranks) at 1/2/4/8 B200, seq 32k-128k; bubble %"
WORKLOADS = {
    "gpt1.3b_32k": dict(L=24, h=2048, s=32768, b=1, num_heads=16),
    "gpt3b_64k": dict(L=16, h=4096, s=65536, b=1, num_heads=32),
    "gpt7b_128k": dict(L=32, h=4096, s=131072, b=1, num_heads=32),
    "tiny": dict(L=4, h=256, s=1024, b=1, num_heads=4),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="gpt1.3b_32k", choices=sorted(WORKLOADS))
    ap.add_argument("--method", default="helix_twofold")
    ap.add_argument("--seq", type=int, default=None, help="override the workload's sequence length (sweeps)")
    ap.add_argument("--mlp-chunk", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=int, default=256)
    ap.add_argument("--stash-budget-gb", type=float, default=None,
                    help="device budget for stashed activations; the rest is FILO-offloaded to pinned "
                         "host memory ('auto': free HBM after weights/grads minus a working-set margin; "
                         "default: auto for gpt7b_128k, off otherwise)")
    ap.add_argument("--trace-out", default=None,
                    help="write the measured per-task device timeline of one iteration as a Chrome "
                         "trace (<prefix>.trace.json) and CSV (<prefix>.csv), reference schema")
    ap.add_argument("--compare-1f1b", choices=["auto", "yes", "no"], default="auto",
                    help="also time the same-kernel 1F1B schedule on the same model / inputs "
                         "(auto: yes, except for the host-offload workload gpt7b_128k)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[2:]):
                if flag.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU legs


def cpu_sample_tokens_per_s(wl: dict, sample_s: int, threads: int = 1) -> tuple[float, float, str]:
    """Time the float64 oracle (the reference's algorithm, einsum, no BLAS) on
    one layer of the workload's width at a bounded sequence length, on
    ``threads`` host threads in parallel, and convert to whole-workload
    tokens/s by the reference's own FLOP count (P/costs.py:62-71:
    72h^2 + 12hs per token per layer, full-square attention as computed)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    from oracle import helix_oracle as O

    h, heads = wl["h"], wl["num_heads"]

    def one(seed: int) -> float:
        P = O.make_model(1, h, seed)[0]
        x = O.make_inputs(1, sample_s, 1, h, seed + 1)[0]
        t0 = time.perf_counter()
        z, cache = O.layer_fwd(x, P, heads)
        _, dz = O.loss_and_grad(z)
        O.layer_bwd(dz, P, cache, heads)
        return time.perf_counter() - t0

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, range(threads)))
    wall = time.perf_counter() - t0
    sample_flops = threads * sample_s * (72 * h * h + 12 * h * sample_s)
    rate = sample_flops / wall
    full_per_token = wl["L"] * (72 * h * h + 12 * h * wl["s"])
    desc = (f"oracle (float64 numpy einsum, reference algorithm) one layer h={h} heads={heads} "
            f"s={sample_s} fwd+bwd x{threads} threads in {wall:.2f}s = {rate / 1e9:.2f} GFLOP/s, "
            f"scaled by reference FLOPs/token (L*(72h^2+12hs)) to L={wl['L']} s={wl['s']}")
    _ = np, math
    return rate / full_per_token, wall, desc


def run_reference(args, wl, rank: int, world: int) -> None:
    """--impl reference: the reference's CPU algorithm (oracle port; the
    reference is Python and cannot be compiled into oracle/_ref) on this
    host's cores, bounded sample per step."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    sample_s = 64
    for _ in range(args.warmup):
        cpu_sample_tokens_per_s(wl, 64, 1)
    vals, walls, desc = [], [], ""
    for _ in range(args.steps):
        v, wall, desc = cpu_sample_tokens_per_s(wl, sample_s, cores)
        vals.append(v)
        walls.append(wall)
    value = sum(vals) / len(vals)
    p = args.gpus
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.workload, **wl, "p": p, "m": 2 * p, "method": args.method},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


def profile_traffic(kernel: str) -> float | None:
    """DRAM bytes per launch of ``kernel`` from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        data = json.loads(p.read_text())
        return data.get(kernel, {}).get("dram_bytes")
    except (ValueError, OSError):
        return None


def main() -> None:
    args = parse()
    wl = dict(WORKLOADS[args.workload])
    if args.seq:
        wl["s"] = args.seq
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return
    if world > 1:
        # leave SMs for the NCCL p2p kernels that run next to persistent GEMMs
        os.environ.setdefault("HX_SM_RESERVE", "8")
    if args.workload == "gpt7b_128k" or args.stash_budget_gb is not None:
        # offloading churns GB-sized blocks: grow segments instead of fragmenting them
        os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

    import torch
    import torch.distributed as dist
    from paper_2507_00394_b200 import ModelConfig, generate
    from paper_2507_00394_b200.costs import DurationTable, attention_kernel_flops, b200_flops_per_token
    from paper_2507_00394_b200.runtime import HelixRuntime
    from paper_2507_00394_b200.runtime import _lib, kernels as K
    from paper_2507_00394_b200.runtime.executor import DeviceModel, make_pair_groups, stage_fields
    from paper_2507_00394_b200.runtime.model import DeviceLayer, random_device_layer
    from paper_2507_00394_b200.simulate import (measured_durations, metrics_from_timeline, overlap_report,
                                                predict_pipeline, simulate)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import datetime
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=600))
    p = world
    cfg = ModelConfig(L=wl["L"], h=wl["h"], s=wl["s"], b=wl["b"], num_heads=wl["num_heads"], p=p, m=2 * p)
    units = DurationTable.from_units(1, 3, 2)
    sched = generate(args.method, cfg, units)
    stages = [rank] if world > 1 else list(range(p))
    groups = make_pair_groups(p) if world > 1 else None

    def build_runtime(schedule):
        """Random-init weights of the architecture, drawn on the GPU (same
        distributions as make_model), placed per the schedule's stage ownership."""
        gen = torch.Generator(device=dev).manual_seed(1234)
        layers = {}
        for l in range(cfg.L):
            need, own = set(), set()
            for st in stages:
                n_, o_ = stage_fields(schedule, st, l)
                need |= set(n_)
                own |= set(o_)
            full = random_device_layer(cfg.h, gen, dev)
            if need:
                layers[l] = DeviceLayer({k: v for k, v in full.items() if k in need},
                                        tuple(k for k in full if k in own))
            del full
        budget = None
        if args.stash_budget_gb is not None and args.stash_budget_gb >= 0:
            budget = int(args.stash_budget_gb * 2**30)
        elif args.stash_budget_gb is not None or args.workload == "gpt7b_128k":
            # free HBM after weights + fp32 grads, minus the per-task working set
            # (regenerated post stash, MLP gradients, qkv / dqkv, attention workspaces:
            # ~22 x T*h bf16 at the last layer's backward) and allocator slack
            torch.cuda.synchronize()
            free, _total = torch.cuda.mem_get_info(dev)
            budget = max(0, free - 40 * cfg.s * cfg.b * cfg.h * 2)
        return HelixRuntime(schedule, DeviceModel(layers), args.mlp_chunk,
                            "distributed" if world > 1 else "replay", dev,
                            rank=rank if world > 1 else None, groups=groups, stash_budget_bytes=budget)

    rt = build_runtime(sched)
    T = cfg.s * cfg.b
    ig = torch.Generator(device=dev).manual_seed(1)
    inputs = [torch.randn(T, cfg.h, generator=ig, device=dev).to(torch.bfloat16) for _ in range(cfg.m)]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def time_steps(runtime, steps):
        """Barrier + sync on both sides, CUDA events on the launching stream,
        max over ranks.  Returns ms per step."""
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            runtime.run(inputs)
        b.record()
        barrier()
        t_ms = a.elapsed_time(b) / steps
        if world > 1:
            t = torch.tensor([t_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_ms = float(t.item())
        return t_ms

    for _ in range(args.warmup):
        rt.run(inputs)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    _lib.start_kernel_timers()      # per-entry-point CUDA events inside the timed steps
    ms = time_steps(rt, args.steps)
    ktimes = _lib.stop_kernel_timers()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    tokens = cfg.m * cfg.s * cfg.b
    value = tokens / (ms / 1e3)
    losses = rt.losses()

    # bubble: one extra iteration with per-task device events (reference metric definition)
    rt.record_timeline = True
    rt.run(inputs)
    rt.record_timeline = False
    tl = rt.timeline or {}
    bubble = None
    if world > 1:
        allt = [None] * world
        dist.all_gather_object(allt, tl)
        tl = {k: v for part in allt for k, v in part.items()}
    predicted = None
    if rank == 0 and tl and args.trace_out:
        from paper_2507_00394_b200.simulate import timeline_csv, write_chrome_trace
        write_chrome_trace(f"{args.trace_out}.trace.json", sched, tl, "ms")
        Path(f"{args.trace_out}.csv").write_text(timeline_csv(sched, tl))
    if rank == 0 and tl:
        measured = metrics_from_timeline(sched, tl)
        bubble = measured.bubble_fraction
        # the reference's own simulator fed with device-measured
        # component times, predicted bubble / makespan next to the measured ones
        table = measured_durations(sched, tl)
        sim = simulate(sched, table)
        predicted = {"bubble_fraction": sim.metrics.bubble_fraction,
                     "makespan_ms": sim.metrics.makespan / 1e6, "measured_makespan_ms": measured.makespan}
        if world > 1:
            # P/simulate.py:118-151 on the measured timeline: transfer waits, and the part the
            # two-fold order should have hidden (rank clocks start at each rank's run start)
            ov = overlap_report(sched, tl)
            predicted["measured_comm_wait_ms"] = ov.total_wait
            predicted["measured_steady_comm_wait_ms"] = ov.steady_wait
        if world == 1:
            # helix vs same-kernel 1F1B at p = 2/4/8 predicted from these measured component
            # times (reference simulator, NVLink 770 GB/s per direction): a prediction only
            predicted["pipeline_prediction"] = predict_pipeline(cfg, table)

    # same-kernel 1F1B baseline (the north-star comparison), same model / inputs
    base_1f1b = None
    if args.compare_1f1b == "yes" or (args.compare_1f1b == "auto" and args.workload != "gpt7b_128k"):
        del rt
        torch.cuda.empty_cache()
        base_method = "1f1b_rc" if args.method.endswith("_rc") else "1f1b"  # like for like
        rt_b = build_runtime(generate(base_method, cfg, units))
        for _ in range(max(1, args.warmup)):
            rt_b.run(inputs)
        ms_b = time_steps(rt_b, args.steps)
        base_1f1b = {"method": base_method, "value": tokens / (ms_b / 1e3), "ms_per_step": ms_b,
                     "helix_speedup": ms_b / ms}
        del rt_b
        torch.cuda.empty_cache()
        rt = build_runtime(sched)
        rt.run(inputs)

    # e2e through the public runtime with host buffers
    e2e = None
    if not args.no_e2e:
        host = [x.cpu().pin_memory() for x in inputs]
        dev_in = [torch.empty_like(x) for x in inputs]
        h2d = sum(x.numel() * x.element_size() for x in host)
        barrier()
        t0 = time.perf_counter()
        e2e_ev0, e2e_ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_ev0.record()
        for _ in range(args.steps):
            for d_, h_ in zip(dev_in, host):
                d_.copy_(h_, non_blocking=True)
            rt.run(dev_in)
            got = rt.sumsq.cpu()  # D2H read of the step's losses (sync)
        e2e_ev1.record()
        barrier()
        e2e_ms = e2e_ev0.elapsed_time(e2e_ev1) / args.steps
        wall_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": tokens / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(got.numel() * got.element_size()), "wall_ms_per_step": wall_ms}
        del host, dev_in

    # roofline of the dominant kernel (attention backward): its mean duration over
    # the launches inside the timed steps (CUDA events on the launching stream),
    # against the SUSTAINED bf16 peak since it runs inside a long power-capped step;
    # the same kernel timed alone afterwards is reported beside it against the burst peak
    peaks = load_peaks()
    roof = None
    kernel_share = None
    if rank == 0:
        fwd_fl, bwd_fl = attention_kernel_flops(cfg)
        kernel_share = {k.removeprefix("hx_"): {"launches": v["launches"] // args.steps,
                                                "ms_per_step": v["total_ms"] / args.steps,
                                                "share": v["total_ms"] / args.steps / ms}
                        for k, v in sorted(ktimes.items(), key=lambda kv: -kv[1]["total_ms"])}
        h, heads = cfg.h, cfg.num_heads
        qkv = torch.randn(T, 3 * h, device=dev).to(torch.bfloat16)
        o = torch.empty(T, h, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(cfg.b, heads, cfg.s, device=dev)
        K.attention_fwd(qkv, cfg.s, cfg.b, heads, o, lse)
        do = torch.randn(T, h, device=dev).to(torch.bfloat16)
        dqkv = torch.empty_like(qkv)
        delta = torch.empty(cfg.b * heads * cfg.s, device=dev)
        dq = torch.empty(T * h, device=dev)
        reps = 5
        for _ in range(2):
            K.attention_bwd(qkv, o, do, lse, cfg.s, cfg.b, heads, dqkv, delta, dq)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(reps):
            K.attention_bwd(qkv, o, do, lse, cfg.s, cfg.b, heads, dqkv, delta, dq)
        a1.record()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(reps):
            K.attention_fwd(qkv, cfg.s, cfg.b, heads, o, lse)
        f1.record()
        torch.cuda.synchronize()
        iso_bwd_ms = a0.elapsed_time(a1) / reps
        iso_fwd_ms = f0.elapsed_time(f1) / reps
        burst, sustained = float(peaks["bf16_tflops"]), float(peaks["bf16_tflops_sustained"])
        bwd_ms = ktimes["hx_attn_bwd"]["mean_ms"] if "hx_attn_bwd" in ktimes else iso_bwd_ms
        fwd_ms = ktimes["hx_attn_fwd"]["mean_ms"] if "hx_attn_fwd" in ktimes else iso_fwd_ms
        ach = bwd_fl / (bwd_ms / 1e3) / 1e12
        src = "fallback" if "fallback" in peaks else "MEASURED_PEAKS.json"
        roof = {"kernel": "attn_bwd_fused_kernel (hx_attn_bwd, incl. pre/convert)", "bound": "tensor",
                "achieved": ach, "peak": sustained, "unit": "TFLOP/s", "frac": ach / sustained,
                "traffic": profile_traffic("attn_bwd"),
                "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside the timed steps)",
                "timing": f"mean of {ktimes.get('hx_attn_bwd', {}).get('launches', 0)} launches inside "
                          "the timed steps, CUDA events on the launching stream",
                "attn_bwd_ms": bwd_ms,
                "attn_fwd": {"achieved": fwd_fl / (fwd_ms / 1e3) / 1e12, "ms": fwd_ms,
                             "frac": fwd_fl / (fwd_ms / 1e3) / 1e12 / sustained},
                "isolated": {"peak": burst, "peak_source": f"{src} bf16_tflops (burst)",
                             "attn_bwd_ms": iso_bwd_ms, "attn_bwd_frac": bwd_fl / (iso_bwd_ms / 1e3) / 1e12 / burst,
                             "attn_fwd_ms": iso_fwd_ms, "attn_fwd_frac": fwd_fl / (iso_fwd_ms / 1e3) / 1e12 / burst},
                "flops_convention": "causal: fwd 2*b*n*s^2*d, bwd 2.5x fwd"}
        del qkv, o, lse, do, dqkv, delta, dq

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, wall, desc = cpu_sample_tokens_per_s(wl, args.cpu_sample_s, 1)
        cpu = {"value": v, "unit": "tokens/s", "cores": 1, "kind": "port", "sample": desc}

    if rank == 0:
        fpt = b200_flops_per_token(cfg)
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (N(0,1) inputs, random-init weights)",
            "config": {"workload": args.workload, **wl, "p": p, "m": cfg.m, "method": args.method,
                       "mlp_chunk": args.mlp_chunk, "parallelism": f"pp{p} (one helix stage per GPU)",
                       "l2": "inputs/activations >> L2 (134 MB per tensor), no flush"},
            "mfu": value * fpt / (world * float(peaks["bf16_tflops"]) * 1e12),
            "model_flops_per_token": fpt,
            "bubble_fraction": bubble,
            "bubble_predicted_by_reference_model": predicted,
            "baseline_1f1b_same_kernels": base_1f1b,
            "losses": losses,
            "gpu_launches": launches,
            "e2e": e2e,
            "roofline": roof,
            "kernel_share": kernel_share,
            "cpu_baseline": cpu,
            "clocks": clk,
            "max_memory_gb": torch.cuda.max_memory_allocated(dev) / 2**30,
            "stash_offload": rt.offload_stats(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

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

``--gpus N`` without a torchrun environment re-launches this script under
``torch.distributed.run`` with N ranks (one helix stage per GPU).

Reference arm (``--impl reference``): the reference's own ``execute_schedule``
(``pipelab`` installed in baseline/_ref; the float64 oracle port if absent) on
BASELINE config 1's model, on every host core -- see :func:`run_reference`.
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
    ap.add_argument("--no-extrapolate", dest="extrapolate", action="store_false",
                    help="skip the labelled FLOP-scaled CPU extrapolation to the workload")
    ap.add_argument("--no-config1", dest="config1", action="store_false",
                    help="skip the B200 measurement at BASELINE config 1 (N=1 only)")
    ap.add_argument("--stash-budget-gb", type=float, default=None,
                    help="device budget for stashed activations; the rest is FILO-offloaded to pinned "
                         "host memory ('auto': free HBM after weights/grads minus a working-set margin; "
                         "default: auto for gpt7b_128k, off otherwise)")
    ap.add_argument("--trace-out", default=None,
                    help="write the measured per-task device timeline of one iteration as a Chrome "
                         "trace (<prefix>.trace.json) and CSV (<prefix>.csv), reference schema")
    ap.add_argument("--lm-vocab", type=int, default=None,
                    help="language-model mode (paper 4.6, runtime/lm.py): token inputs, word + position "
                         "embeddings and the tied head with the loss in backward, vocabulary V")
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
    """FLOP-scaled extrapolation (a labelled extra, not the CPU baseline): the
    float64 oracle on one layer of the workload's width at a bounded sequence
    length, converted to whole-workload tokens/s by the reference's own FLOP
    count (P/costs.py:62-71: 72h^2 + 12hs per token per layer)."""
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
    desc = (f"oracle (float64 numpy einsum) one layer h={h} heads={heads} s={sample_s} fwd+bwd x{threads} "
            f"threads in {wall:.2f}s = {rate / 1e9:.2f} GFLOP/s, scaled by the reference's FLOPs/token "
            f"(L*(72h^2+12hs)) to L={wl['L']} s={wl['s']}")
    return rate / full_per_token, wall, desc


# BASELINE config 1: the reference's CPU-runnable case (tiny GPT, 2 stages x 4 micro-batches)
CONFIG1 = dict(L=4, h=256, s=1024, b=1, num_heads=4, p=2, m=4)
CONFIG1_METHOD = "helix_twofold"
# the bounded per-step sample of config 1: one of its layers (same h, heads, s, b)
# through one helix stage with the smallest two-fold micro-batch count
CONFIG1_SLICE = dict(L=1, h=256, s=1024, b=1, num_heads=4, p=1, m=2)


def config1_dict() -> dict:
    return {"workload": "tiny (BASELINE configs[0])", **CONFIG1, "method": CONFIG1_METHOD,
            "durations": "DurationTable.from_units(1, 3, 2)", "params_seed": 0, "inputs_seed": 1}


def _ref_pipelab():
    """The unmodified reference package from baseline/_ref, or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "pipelab").is_dir():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import pipelab  # noqa: F401
        import pipelab.runtime.executor as ex
        ex._WAIT_TIMEOUT = 1e9      # P/runtime/executor.py:56 (threaded waits; SURVEY 8d caveat)
        return pipelab
    except ImportError:
        return None


def _ref_worker(job: tuple) -> tuple[float, str]:
    """One bounded sample in a worker process: the reference's own
    ``execute_schedule`` (P/runtime/executor.py:425-440) on ``cfg_kw``, or the
    oracle port's ``sequential_oracle`` when pipelab is not installed."""
    cfg_kw, threaded = job
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    pl = _ref_pipelab()
    if pl is not None:
        from pipelab import ModelConfig as RC, generate as rgen
        from pipelab.costs import DurationTable as RD
        from pipelab.runtime import execute_schedule as rexec, make_inputs as rin, make_model as rmod
        cfg = RC(**cfg_kw)
        sched = rgen(CONFIG1_METHOD, cfg, RD.from_units(1, 3, 2))
        P, X = rmod(cfg, 0), rin(cfg, 1)
        t0 = time.perf_counter()
        rexec(sched, P, X, threaded=threaded)
        return time.perf_counter() - t0, "reference"
    from oracle import helix_oracle as O
    c = cfg_kw
    P = O.make_model(c["L"], c["h"], 0)
    X = O.make_inputs(c["m"], c["s"], c["b"], c["h"], 1)
    t0 = time.perf_counter()
    O.sequential_oracle(P, X, c["num_heads"])
    return time.perf_counter() - t0, "port"


class ReferenceSampler:
    """Config-1 tokens/s of the reference's CPU implementation on this host.

    Each step runs ``R`` independent replicas (one per host core, separate
    processes: the reference's numerics are single-threaded einsum) of the
    config-1 slice; step time = the slowest replica.  tokens/s at config 1
    = R * m_slice * s * b / step_time * (L_slice / L_config1): per-layer work
    is identical, so the 4-layer config costs exactly L/L_slice slices.
    """

    def __init__(self, replicas: int):
        import multiprocessing as mp
        self.replicas = replicas
        self.pool = mp.get_context("spawn").Pool(replicas)   # no fork of a CUDA process
        self.kind = None

    def step(self, cfg_kw: dict, threaded: bool = False) -> float:
        res = self.pool.map(_ref_worker, [(cfg_kw, threaded)] * self.replicas, chunksize=1)
        self.kind = res[0][1]
        return max(t for t, _ in res)

    def tokens_per_s(self, wall: float) -> float:
        c = CONFIG1_SLICE
        return self.replicas * c["m"] * c["s"] * c["b"] / wall * (c["L"] / CONFIG1["L"])

    def describe(self) -> str:
        impl = ("the reference's own execute_schedule (pipelab from baseline/_ref, replay driver)"
                if self.kind == "reference" else "the float64 oracle port (sequential_oracle)")
        c = CONFIG1_SLICE
        return (f"{impl}; per step {self.replicas} concurrent replicas (1 per host core) of one config-1 "
                f"layer (h={c['h']} heads={c['num_heads']} s={c['s']} b={c['b']}) x {c['m']} micro-batches "
                f"fwd+bwd, helix_twofold p=1; tokens/s scaled by L_slice/L = {c['L']}/{CONFIG1['L']}")

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args, wl, rank: int, world: int) -> None:
    """--impl reference: the reference's CPU implementation of the path on this
    host's cores, at BASELINE config 1 (the only configuration a CPU runs; the
    B200 line reports its own number at the same config under ``config1``).
    Rank 0 alone runs under torchrun."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    smp = ReferenceSampler(cores)
    try:
        warm = dict(L=2, h=64, s=128, b=1, num_heads=2, p=2, m=4)     # SURVEY 8c fast CI shape
        for _ in range(args.warmup):
            smp.step(warm)
        walls = [smp.step(CONFIG1_SLICE) for _ in range(args.steps)]
    finally:
        smp.close()
    wall = sum(walls) / len(walls)
    value = smp.tokens_per_s(wall)
    ext, _w, ext_desc = cpu_sample_tokens_per_s(wl, 64, cores) if args.extrapolate else (None, 0, "")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference fixtures: make_model seed 0, make_inputs seed 1)",
        "config": config1_dict(),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": smp.kind,
                         "sample": smp.describe(), "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "warmup_sample": "fast CI shape L=2 h=64 s=128 p=2 m=4 per replica",
    }
    if ext is not None:
        line["extrapolated_to_workload"] = {"workload": args.workload, "value": ext, "unit": "tokens/s",
                                            "how": ext_desc}
    print(json.dumps(line), flush=True)


def _cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(args) -> int:
    """``python bench.py --gpus N`` outside torchrun: one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ GPU leg


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


def profile_traffic(kernel: str) -> float | None:
    """DRAM bytes per launch of ``kernel`` from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ncu_summary_r02.json"   # this round's capture of the current kernels
    if not p.exists():
        p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        data = json.loads(p.read_text())
        return data.get(kernel, {}).get("dram_bytes")
    except (ValueError, OSError):
        return None


def baseline_memory_plan() -> dict:
    """Worst-rank device memory of BASELINE configs 2-4 at their GPU counts
    (runtime/memplan.py; 180 GB B200) and the host memory the FILO offloader
    needs: the plan the stage probes check on the B200."""
    from paper_2507_00394_b200 import ModelConfig, generate
    from paper_2507_00394_b200.costs import DurationTable
    from paper_2507_00394_b200.runtime.memplan import GB, offload_needed, plan
    U = DurationTable.from_units(1, 3, 2)
    rows = {
        "gpt1.3b_32k p4": (ModelConfig(L=24, h=2048, s=32768, b=1, num_heads=16, p=4, m=8), None,
                           [("helix_twofold", {}), ("1f1b", {})]),
        "gpt3b_64k p8": (ModelConfig(L=16, h=4096, s=65536, b=1, num_heads=32, p=8, m=16), 8192,
                         [("helix_twofold_rc", {}), ("1f1b", {}), ("1f1b_rc", {})]),
        "gpt7b_128k p8": (ModelConfig(L=32, h=4096, s=131072, b=1, num_heads=32, p=8, m=16), 16384,
                          [("helix_twofold_rc", {"regen_pre_x": True, "stream_inputs": True}), ("1f1b_rc", {})]),
    }
    out = {}
    for name, (cfg, chunk, methods) in rows.items():
        for method, kw in methods:
            sched = generate(method, cfg, U)
            worst = max((plan(sched, r, chunk, durations=U, **kw) for r in range(cfg.p)), key=lambda x: x.total)
            key = f"{name} {method}" + "".join(f" +{k}" for k in kw)
            out[key] = {"worst_rank": worst.stage, "device_total_gb": round(worst.total / GB, 1),
                        "stash_gb": round(worst.stash_peak / GB, 1),
                        "host_offload_gb": round(offload_needed(worst, 180 * GB) / GB, 1)}
    return out


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
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world} (one rank per GPU)")
    # test-only: run the same multi-rank driver on CPU over gloo with the float64
    # test double (tests/cpu_math.py) at a toy shape -- never a bench number
    cpu_double = os.environ.get("HX_BENCH_CPU_DOUBLE") == "1"
    if world > 1 and not cpu_double:
        # NCCL init lines (nRanks per communicator) on stderr for the launch check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.workload == "gpt7b_128k" or args.stash_budget_gb is not None:
        # offloading churns GB-sized blocks: grow segments instead of fragmenting them
        os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    if cpu_double:
        return bench_cpu_double(args, world, rank)
    bench_gpu(args, wl, world, rank, local)


def bench_cpu_double(args, world: int, rank: int) -> None:
    """Test-only leg (HX_BENCH_CPU_DOUBLE=1): the launch and the multi-rank
    distributed driver exactly as on the GPU box, over gloo with float64 CPU
    math, at the toy shape L=4 h=8 s=8 with p = N and m = 2N."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2507_00394_b200 import ModelConfig, generate
    from paper_2507_00394_b200.costs import DurationTable
    from paper_2507_00394_b200.runtime.executor import DeviceModel, HelixRuntime, pair_groups, stage_fields
    from paper_2507_00394_b200.runtime.model import DeviceLayer, make_inputs, make_model
    from tests.cpu_math import CpuMath

    if world > 1:
        dist.init_process_group("gloo")
    p = world
    cfg = ModelConfig(L=4, h=8, s=8, b=1, num_heads=2, p=p, m=2 * p)
    sched = generate(args.method, cfg, DurationTable.from_units(1, 3, 2))
    stages = [rank] if world > 1 else list(range(p))
    layers = {}
    for l, prm in enumerate(make_model(cfg, 0)):
        need, own = set(), set()
        for st in stages:
            n_, o_ = stage_fields(sched, st, l)
            need |= set(n_)
            own |= set(o_)
        if need:
            layers[l] = DeviceLayer({k: torch.from_numpy(np.ascontiguousarray(getattr(prm, k))) for k in need},
                                    tuple(own), grad_dtype=torch.float64)
    rt = HelixRuntime(sched, DeviceModel(layers), None, "distributed" if world > 1 else "replay",
                      torch.device("cpu"), math=CpuMath(cfg, bool(int(sched.meta["qkv"]))),
                      rank=rank if world > 1 else None, groups=pair_groups(p) if world > 1 else None)
    inputs = [torch.from_numpy(x).reshape(cfg.s * cfg.b, cfg.h) for x in make_inputs(cfg, 1)]
    for _ in range(args.warmup):
        rt.run(inputs)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rt.run(inputs)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if world > 1:
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        sums = torch.tensor(rt.sumsq.tolist(), dtype=torch.float64)
        dist.all_reduce(sums)
    else:
        sums = rt.sumsq
    if rank == 0:
        tokens = cfg.m * cfg.s * cfg.b
        print(json.dumps({
            "metric": METRIC, "value": tokens / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "TEST DOUBLE (CPU, gloo)",
            "config": {"workload": "toy", "L": cfg.L, "h": cfg.h, "s": cfg.s, "b": cfg.b, "p": p, "m": cfg.m,
                       "method": args.method},
            "losses": [float(v) / (cfg.s * cfg.b * cfg.h) for v in sums.tolist()],
            "comm": rt.comm_stats}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def measure_config1(dev) -> dict:
    """The B200 at BASELINE config 1, like for like with the reference arm:
    ``execute_schedule`` with the reference's host fixtures (float64 numpy in,
    RunResult of numpy out; wall clock per call, all copies inside), and the
    same schedule through HelixRuntime device-timed.  Losses are checked
    against the reference's known config-1 values."""
    import torch
    from paper_2507_00394_b200 import ModelConfig, generate
    from paper_2507_00394_b200.costs import DurationTable
    from paper_2507_00394_b200.runtime import execute_schedule, make_inputs, make_model
    from paper_2507_00394_b200.runtime.executor import DeviceModel, HelixRuntime

    known = [3.327261203817688, 3.3800507339316543, 3.443091222231624, 3.4279542847160513]
    cfg = ModelConfig(**CONFIG1)
    sched = generate(CONFIG1_METHOD, cfg, DurationTable.from_units(1, 3, 2))
    P, X = make_model(cfg, 0), make_inputs(cfg, 1)
    tokens = cfg.m * cfg.s * cfg.b
    out = {"config": config1_dict()}
    for threaded in (False, True):
        for _ in range(3):
            res = execute_schedule(sched, P, X, threaded=threaded)
        reps = 10
        t0 = time.perf_counter()
        for _ in range(reps):
            res = execute_schedule(sched, P, X, threaded=threaded)
        wall = (time.perf_counter() - t0) / reps
        out["execute_schedule_threaded" if threaded else "execute_schedule_replay"] = {
            "tokens_per_s": tokens / wall, "ms_per_call": 1e3 * wall,
            "loss_max_rel_err_vs_reference": max(abs(a - b) / b for a, b in zip(res.losses, known))}
    model = DeviceModel.from_host(sched, P, range(cfg.p), dev)
    rt = HelixRuntime(sched, model, None, "multistream", dev)
    xs = [torch.from_numpy(x).to(dev, torch.bfloat16).reshape(cfg.s * cfg.b, cfg.h) for x in X]
    for _ in range(3):
        rt.run(xs)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        rt.run(xs)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    out["device"] = {"tokens_per_s": tokens / (ms / 1e3), "ms_per_step": ms,
                     "how": "HelixRuntime multistream (one CUDA stream per stage), CUDA events"}
    # the same iteration captured as one CUDA graph (config 1 is host-launch bound eagerly)
    try:
        g = rt.capture(xs)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(20):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        gms = a.elapsed_time(b) / 20
        out["device_cuda_graph"] = {"tokens_per_s": tokens / (gms / 1e3), "ms_per_step": gms,
                                    "how": "HelixRuntime.capture: the multistream iteration as one CUDA graph"}
    except Exception as e:  # noqa: BLE001 -- reported, not fatal for the bench line
        out["device_cuda_graph"] = {"error": f"{type(e).__name__}: {e}"[:200]}
    out["value"] = out["execute_schedule_threaded"]["tokens_per_s"]
    out["unit"] = "tokens/s"
    out["value_is"] = "execute_schedule(threaded=True) with host float64 fixtures, wall clock per call"
    return out


def bench_gpu(args, wl, world: int, rank: int, local: int) -> None:
    import torch
    import torch.distributed as dist
    from paper_2507_00394_b200 import ModelConfig, generate
    from paper_2507_00394_b200.analytic import bubble_fraction, bubble_time_from_table
    from paper_2507_00394_b200.costs import DurationTable, attention_kernel_flops, b200_flops_per_token
    from paper_2507_00394_b200.runtime import HelixRuntime
    from paper_2507_00394_b200.runtime import _lib, kernels as K
    from paper_2507_00394_b200.runtime.executor import DeviceModel, pair_groups, stage_fields
    from paper_2507_00394_b200.runtime.model import DeviceLayer, random_device_layer
    from paper_2507_00394_b200.simulate import (measured_durations, metrics_from_timeline, overlap_report,
                                                predict_pipeline, simulate)
    from paper_2507_00394_b200.engine import CommModel

    # test-only (HX_BENCH_SHARED_GPU=1): all ranks on cuda:0 over gloo (host-staged
    # payloads), so the N > 1 leg of this script runs end to end on a one-GPU box;
    # its numbers are time-shared and never a bench value
    shared_gpu = world > 1 and os.environ.get("HX_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import datetime
        if shared_gpu:
            dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=900))
        else:
            dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=900))
    p = world
    cfg = ModelConfig(L=wl["L"], h=wl["h"], s=wl["s"], b=wl["b"], num_heads=wl["num_heads"], p=p, m=2 * p)
    units = DurationTable.from_units(1, 3, 2)
    sched = generate(args.method, cfg, units)
    stages = [rank] if world > 1 else list(range(p))
    groups = pair_groups(p) if world > 1 else None

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
        lm_kw = {}
        if args.lm_vocab:
            from paper_2507_00394_b200.runtime.lm import LMSpec
            lm_kw = {"lm": LMSpec(args.lm_vocab)}
        return HelixRuntime(schedule, DeviceModel(layers), args.mlp_chunk,
                            "distributed" if world > 1 else "replay", dev,
                            rank=rank if world > 1 else None, groups=groups, stash_budget_bytes=budget, **lm_kw)

    rt = build_runtime(sched)
    T = cfg.s * cfg.b
    ig = torch.Generator(device=dev).manual_seed(1)
    if args.lm_vocab:   # token ids (N(0,1) activations otherwise)
        inputs = [torch.randint(0, args.lm_vocab, (cfg.s, cfg.b), generator=ig, device=dev) for _ in range(cfg.m)]
    else:
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
    ktimes, ktagged = _lib.stop_kernel_timers(with_tags=True)
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
            # analytic (closed form, zero comm) / simulated (zero comm and NVLink-modelled) /
            # measured bubble side by side for this p: the gaps attribute any shortfall
            nv = CommModel("bytes", latency=5000, bytes_per_element=2, bandwidth=int(770e9))
            sim_nv = simulate(sched, table, nv)
            try:
                analytic_ms = bubble_time_from_table(args.method, p, cfg.L, table) / 1e6
                analytic_frac = bubble_fraction(args.method, cfg, table)
            except Exception:   # noqa: BLE001 -- no formula for this method
                analytic_ms = analytic_frac = None
            predicted["bubble_table"] = {
                "analytic": {"fraction": analytic_frac, "per_stage_bubble_ms": analytic_ms},
                "simulated_zero_comm": {"fraction": sim.metrics.bubble_fraction,
                                        "makespan_ms": sim.metrics.makespan / 1e6},
                "simulated_nvlink": {"fraction": sim_nv.metrics.bubble_fraction,
                                     "makespan_ms": sim_nv.metrics.makespan / 1e6},
                "measured": {"fraction": measured.bubble_fraction, "makespan_ms": measured.makespan,
                             "per_stage_bubble_ms": list(measured.per_stage_bubble)}}
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
        # pinned host inputs straight into the runtime: its input streamer copies
        # each micro-batch to the device just before layer 0's forward and again
        # for its backward (side stream), so no stage keeps all inputs resident
        host = [x.cpu().pin_memory() for x in inputs]
        rt.run(host)                      # warm the streaming path
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e2e_ev0, e2e_ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h2d0 = 0
        e2e_ev0.record()
        for _ in range(args.steps):
            rt.run(host)
            h2d0 += rt.core.streamer.h2d_bytes if rt.core.streamer is not None else \
                sum(x.numel() * 4 for x in host)       # LM mode: int32 token ids
            got = rt.sumsq.cpu()  # D2H read of the step's losses (sync)
        h2d = h2d0 // args.steps
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
        del host

    # roofline of the dominant kernel (attention backward): its mean duration over
    # the launches inside the timed steps (CUDA events on the launching stream),
    # against the SUSTAINED bf16 peak since it runs inside a long power-capped step;
    # the same kernel timed alone afterwards is reported beside it against the burst peak
    peaks = load_peaks()
    roof = None
    kernel_share = None
    gemm_shapes = None
    if rank == 0:
        fwd_fl, bwd_fl = attention_kernel_flops(cfg)
        kernel_share = {k.removeprefix("hx_"): {"launches": v["launches"] // args.steps,
                                                "ms_per_step": v["total_ms"] / args.steps,
                                                "share": v["total_ms"] / args.steps / ms}
                        for k, v in sorted(ktimes.items(), key=lambda kv: -kv[1]["total_ms"])}
        # GEMMs by shape (layout A/B: N = K-major, T = MN-major; M x N x K; epilogue):
        # achieved TFLOP/s inside the timed steps, for the GEMM roofline per shape
        gemm_shapes = []
        for key, v in sorted(ktagged.items(), key=lambda kv: -kv[1]["total_ms"]):
            if not key.startswith("hx_gemm:"):
                continue
            lay, mnk, epi = key.split(":", 1)[1].split()
            M_, N_, K_ = (int(x) for x in mnk.split("x"))
            gemm_shapes.append({"layout": lay, "M": M_, "N": N_, "K": K_, "epilogue": epi,
                                "calls_per_step": v["launches"] // args.steps, "mean_ms": v["mean_ms"],
                                "tflops": 2 * M_ * N_ * K_ / (v["mean_ms"] / 1e3) / 1e12,
                                "ms_per_step": v["total_ms"] / args.steps})
        # each shape once more in isolation, next to cuBLAS (torch.matmul, bf16 out) on the
        # same operand layouts: the library yardstick for the tcgen05 GEMM
        def _iso(fn, reps=5):
            fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps

        for g_ in gemm_shapes:
            M_, N_, K_ = g_["M"], g_["N"], g_["K"]
            a_t, b_t = g_["layout"][0] == "T", g_["layout"][1] == "T"
            A_ = torch.randn(K_, M_, device=dev).to(torch.bfloat16) if a_t else \
                torch.randn(M_, K_, device=dev).to(torch.bfloat16)
            B_ = torch.randn(K_, N_, device=dev).to(torch.bfloat16) if b_t else \
                torch.randn(N_, K_, device=dev).to(torch.bfloat16)
            acc = g_["epilogue"] in (f"epi{_lib.EPI_ACC_F32}", f"epi{_lib.EPI_STORE_F32}")
            C_ = torch.zeros(M_, N_, device=dev, dtype=torch.float32 if acc else torch.bfloat16)
            epi_ = _lib.EPI_ACC_F32 if acc else _lib.EPI_STORE_BF16
            ours = _iso(lambda: K.gemm(A_, a_t, B_, b_t, C_, M_, N_, K_, epi_))
            At, Bt = (A_.t() if a_t else A_), (B_ if b_t else B_.t())   # logical [M,K], [K,N]
            cub = _iso(lambda: torch.matmul(At, Bt))
            fl = 2 * M_ * N_ * K_
            g_["isolated_tflops"] = fl / (ours / 1e3) / 1e12
            g_["cublas_tflops"] = fl / (cub / 1e3) / 1e12
            g_["vs_cublas"] = cub / ours
            del A_, B_, C_
        h, heads = cfg.h, cfg.num_heads
        qkv = torch.randn(T, 3 * h, device=dev).to(torch.bfloat16)
        o = torch.empty(T, h, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(cfg.b, heads, cfg.s, device=dev)
        K.attention_fwd(qkv, cfg.s, cfg.b, heads, o, lse)
        do = torch.randn(T, h, device=dev).to(torch.bfloat16)
        dqkv = torch.empty_like(qkv)
        delta = torch.empty(cfg.b * heads * cfg.s, device=dev)
        dq = K.attention_bwd_ws(cfg.s, cfg.b, heads, h // heads, dev)
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
        roof = {"kernel": "attn_bwd_fused_kernel (hx_attn_bwd incl. the dq convert; D from hx_attn_bwd_delta)", "bound": "tensor",
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
        # the sustained peak was measured at its own (power-capped) median clock;
        # rescaled to the clock this step ran at, the fraction is clock-neutral
        peak_mhz = (peaks.get("clocks_under_load") or {}).get("sm_mhz_median")
        if peak_mhz and clk.get("sm_mhz"):
            scaled_peak = sustained * float(clk["sm_mhz"]) / float(peak_mhz)
            roof["frac_at_step_clock"] = ach / scaled_peak
            roof["peak_at_step_clock"] = {"value": scaled_peak, "how": f"bf16_tflops_sustained x step "
                                          f"{clk['sm_mhz']:.0f} MHz / its {peak_mhz:.0f} MHz median"}
        del qkv, o, lse, do, dqkv, delta, dq

    # like-for-like pair at BASELINE config 1 (the reference arm's configuration)
    config1 = None
    if rank == 0 and world == 1 and args.config1:
        config1 = measure_config1(dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        smp = ReferenceSampler(cores)
        try:
            wall = smp.step(CONFIG1_SLICE)
        finally:
            smp.close()
        cpu = {"value": smp.tokens_per_s(wall), "unit": "tokens/s (BASELINE config 1)", "cores": cores,
               "kind": smp.kind, "sample": smp.describe() + "; 1 step", "cpu_model": _cpu_model(),
               "config": config1_dict()}
        if config1 is not None:
            cpu["b200_same_config"] = {"tokens_per_s": config1["value"], "ratio": config1["value"] / cpu["value"]}
        if args.extrapolate:
            v, _w, desc = cpu_sample_tokens_per_s(wl, 256, 1)
            cpu["extrapolated_to_workload"] = {"value": v, "unit": "tokens/s", "cores": 1, "how": desc}

    if rank == 0:
        fpt = b200_flops_per_token(cfg)
        if args.lm_vocab:   # tied head: logits, dz, dW_emb GEMMs (2hV FLOPs each per token)
            fpt += 6 * cfg.h * args.lm_vocab
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "TEST: ranks time-sharing one GPU over gloo -- not a bench value" if shared_gpu
            else "synthetic (N(0,1) inputs, random-init weights)",
            "config": {"workload": args.workload, **wl, "p": p, "m": cfg.m, "method": args.method,
                       "n_gpus": world,
                       "mlp_chunk": args.mlp_chunk, "parallelism": f"pp{p} (one helix stage per GPU)",
                       **({"lm_vocab": args.lm_vocab} if args.lm_vocab else {}),
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
            "gemm_shapes": gemm_shapes,
            "cpu_baseline": cpu,
            "config1": config1,
            "comm": rt.comm_stats,
            "clocks": clk,
            "max_memory_gb": torch.cuda.max_memory_allocated(dev) / 2**30,
            "stash_offload": rt.offload_stats(),
        }
        line["memory_plan"] = baseline_memory_plan()
        pred = ROOT / "profiles" / "r02_pipeline_predictions.json"
        if pred.exists():
            line["pipeline_prediction_from_stage_probes"] = {
                "source": "profiles/r02_pipeline_predictions.json (tools/predict_from_probes.py: rank-0 stage "
                          "probes measured on a B200 at the 8-stage per-rank shapes, replayed by the reference "
                          "list scheduler with NVLink 770 GB/s + 5 us); predictions, not measurements",
                **{wl: {k: {kk: vv for kk, vv in v.items() if kk in ("makespan_ms", "bubble_fraction",
                                                                        "tokens_per_s") or kk.startswith("speedup")}
                            for k, v in rows.items()}
                   for wl, rows in json.loads(pred.read_text()).items()}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

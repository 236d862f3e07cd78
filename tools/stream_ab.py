#!/usr/bin/env python
"""A/B of one bench iteration with device-resident vs host-streamed inputs
(executor._InputStreamer), CUDA-event timed, alternating, same runtime."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2507_00394_b200 import ModelConfig, generate  # noqa: E402
from paper_2507_00394_b200.costs import DurationTable  # noqa: E402
from paper_2507_00394_b200.runtime import HelixRuntime  # noqa: E402
from paper_2507_00394_b200.runtime.executor import DeviceModel  # noqa: E402
from paper_2507_00394_b200.runtime.model import DeviceLayer, random_device_layer  # noqa: E402

cfg = ModelConfig(L=int(sys.argv[1]) if len(sys.argv) > 1 else 24, h=2048, s=32768, b=1, num_heads=16, p=1, m=2)
dev = torch.device("cuda", 0)
sched = generate("helix_twofold", cfg, DurationTable.from_units(1, 3, 2))
gen = torch.Generator(device=dev).manual_seed(1)
layers = {}
for l in range(cfg.L):
    w = random_device_layer(cfg.h, gen, dev)
    layers[l] = DeviceLayer(w, tuple(w))
rt = HelixRuntime(sched, DeviceModel(layers), None, "replay", dev)
ig = torch.Generator(device=dev).manual_seed(2)
dev_in = [torch.randn(cfg.s, cfg.h, generator=ig, device=dev).to(torch.bfloat16) for _ in range(cfg.m)]
host = [x.cpu().pin_memory() for x in dev_in]


def timed(inp, reps=3):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(reps):
        rt.run(inp)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, (time.perf_counter() - t0) * 1e3 / reps


for inp in (dev_in, host):
    rt.run(inp)
for rnd in range(3):
    d = timed(dev_in)
    h = timed(host)
    print(f"round {rnd}: device inputs {d[0]:.1f} ms (wall {d[1]:.1f}), streamed {h[0]:.1f} ms (wall {h[1]:.1f})",
          flush=True)

#!/usr/bin/env python
"""Where the time of one execute_schedule call at BASELINE config 1 goes
(replay vs multistream), host-side cProfile + wall clock."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2507_00394_b200 import ModelConfig, generate  # noqa: E402
from paper_2507_00394_b200.costs import DurationTable  # noqa: E402
from paper_2507_00394_b200.runtime import execute_schedule, make_inputs, make_model  # noqa: E402

cfg = ModelConfig(L=4, h=256, s=1024, b=1, num_heads=4, p=2, m=4)
sched = generate("helix_twofold", cfg, DurationTable.from_units(1, 3, 2))
P, X = make_model(cfg, 0), make_inputs(cfg, 1)
for threaded in (False, True):
    for _ in range(3):
        execute_schedule(sched, P, X, threaded=threaded)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        execute_schedule(sched, P, X, threaded=threaded)
    print(f"threaded={threaded}: {(time.perf_counter() - t0) / 5 * 1e3:.1f} ms per call", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    execute_schedule(sched, P, X, threaded=threaded)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)

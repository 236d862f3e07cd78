"""bench.py launch contract on CPU.

* ``--gpus 2`` outside torchrun re-launches itself with 2 ranks (one helix
  stage per rank).  ``HX_BENCH_CPU_DOUBLE=1`` (test-only) swaps the B200 math
  for the float64 test double over gloo, so the launch, the multi-rank driver
  and the JSON line are exercised here exactly as on the GPU box.
* ``--impl reference`` times the reference's own ``execute_schedule`` at
  BASELINE config 1 and reports the config the B200 line's ``config1`` uses.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

from oracle import helix_oracle as O

ROOT = Path(__file__).resolve().parent.parent


def _json_line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_gpus_flag_launches_one_rank_per_stage():
    env = {**os.environ, "HX_BENCH_CPU_DOUBLE": "1"}
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _json_line(r.stdout)
    assert line["n_gpus"] == 2 and line["config"]["p"] == 2 and line["config"]["m"] == 4
    ref = O.sequential_oracle(O.make_model(4, 8, 0), O.make_inputs(4, 8, 1, 8, 1), 2)
    assert np.allclose(line["losses"], ref.losses, rtol=1e-10)


def test_reference_arm_reports_config1():
    sys.path.insert(0, str(ROOT))
    import bench
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--no-extrapolate"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _json_line(r.stdout)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"] == bench.config1_dict()
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["cores"] == (os.cpu_count() or 1)

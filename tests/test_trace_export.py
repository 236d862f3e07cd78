"""Timeline exports in the reference's schema (P/simulate.py:157-196), applied to
a timeline from the reference-equivalent simulator (no GPU needed)."""

import csv
import io
import json

from paper_2507_00394_b200 import ModelConfig, generate
from paper_2507_00394_b200.costs import DurationTable
from paper_2507_00394_b200.simulate import chrome_trace, simulate, timeline_csv, write_chrome_trace


def _sim():
    cfg = ModelConfig(L=4, h=64, s=128, b=1, num_heads=2, p=2, m=4)
    sched = generate("helix_twofold", cfg, DurationTable.from_units(1, 3, 2))
    return sched, simulate(sched, DurationTable.from_units(1, 3, 2))


def test_chrome_trace_schema(tmp_path):
    sched, res = _sim()
    ev = chrome_trace(sched, res.timeline, "units")
    assert len(ev) == len(res.timeline)
    lanes = {e["tid"] for e in ev}
    assert lanes <= {"compute", "in", "out"} and "compute" in lanes and "out" in lanes
    for e in ev:
        t = sched.tasks[e["name"]]
        assert e["ph"] == "X" and e["pid"] == t.stage and e["dur"] >= 0
        assert e["args"] == {"kind": t.kind, "comp": t.comp, "mb": t.mb, "layer": t.layer}
    # CUDA-event timelines are in ms -> microseconds in the trace
    ms = chrome_trace(sched, {k: (a / 1e3, b / 1e3) for k, (a, b) in res.timeline.items()}, "ms")
    assert [round(e["ts"], 6) for e in ms] == [round(e["ts"], 6) for e in ev]
    path = tmp_path / "t.trace.json"
    write_chrome_trace(path, sched, res.timeline, "units")
    assert len(json.loads(path.read_text())["traceEvents"]) == len(ev)


def test_timeline_csv_sorted_and_complete():
    sched, res = _sim()
    rows = list(csv.reader(io.StringIO(timeline_csv(sched, res.timeline))))
    assert rows[0] == ["task", "stage", "kind", "mb", "layer", "start", "end"]
    body = rows[1:]
    assert len(body) == len(res.timeline)
    keys = [(float(r[5]), float(r[6]), r[0]) for r in body]
    assert keys == sorted(keys)
    assert timeline_csv(sched, res.timeline) == timeline_csv(sched, dict(res.timeline))  # deterministic


def test_exports_equal_reference_when_importable():
    """Byte-for-byte against the reference's own exporters (this container only;
    the GPU box has no /root/reference)."""
    import os
    import sys
    import pytest
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not mounted")
    sys.path.insert(0, ref)
    try:
        from pipelab import ModelConfig as RC, generate as rgen
        from pipelab.costs import DurationTable as RDT
        from pipelab.simulate import chrome_trace as rct, simulate as rsim, timeline_csv as rcsv
    finally:
        sys.path.remove(ref)
    rr = rsim(rgen("helix_twofold", RC(L=4, h=64, s=128, b=1, num_heads=2, p=2, m=4), RDT.from_units(1, 3, 2)),
              RDT.from_units(1, 3, 2))
    sched, res = _sim()
    assert rct(rr) == chrome_trace(sched, res.timeline, res.metrics.time_unit)
    assert rcsv(rr) == timeline_csv(sched, res.timeline)

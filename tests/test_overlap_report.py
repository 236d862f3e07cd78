"""Communication-wait accounting (overlap_report, P/simulate.py:100-151) on
simulated timelines with a non-zero wire model, and on a measured-style
timeline (float ms).  Equality with the reference's own overlap_report is
checked when /root/reference is mounted (this container only)."""

import importlib
import os
import sys

import pytest

from paper_2507_00394_b200 import ModelConfig, generate
from paper_2507_00394_b200.costs import DurationTable
from paper_2507_00394_b200.engine import CommModel

sim = importlib.import_module("paper_2507_00394_b200.simulate")

UNITS = DurationTable.from_units(1, 3, 2)
CASES = [("helix_twofold", 2, 4, 1, 0), ("helix_twofold", 4, 8, 2, 1), ("helix_naive", 2, 4, 2, 0),
         ("1f1b", 4, 8, 1, 1), ("zb1p", 2, 4, 2, 0), ("helix_twofold_rc", 2, 8, 1, 1)]


def _run(method, p, m, cost, lat):
    cfg = ModelConfig(L=2 * p, h=64, s=128, b=1, num_heads=2, p=p, m=m)
    sched = generate(method, cfg, UNITS)
    return sched, sim.simulate(sched, UNITS, CommModel.uniform(cost, lat))


@pytest.mark.parametrize("method,p,m,cost,lat", CASES)
def test_overlap_report_invariants(method, p, m, cost, lat):
    sched, res = _run(method, p, m, cost, lat)
    rep = sim.overlap_report(res)
    assert rep == sim.overlap_report(sched, res.timeline)
    assert rep.total_wait == sum(rep.per_stage_wait) == sum(r.wait for r in rep.rows)
    assert 0 <= rep.steady_wait <= rep.total_wait
    assert all(r.wait > 0 for r in rep.rows)
    # with free, instant transfers nothing waits beyond its producers
    free = sim.simulate(sched, UNITS)
    assert sim.overlap_report(free).total_wait == 0
    # the same accounting on a float (ms) timeline scales linearly
    ms = {k: (a * 0.25, b * 0.25) for k, (a, b) in res.timeline.items()}
    rep_ms = sim.overlap_report(sched, ms)
    assert rep_ms.total_wait == pytest.approx(rep.total_wait * 0.25)


@pytest.mark.parametrize("method,p,m,cost,lat", CASES)
def test_overlap_report_equals_reference(method, p, m, cost, lat):
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not mounted")
    sys.path.insert(0, ref)
    try:
        from pipelab import ModelConfig as RC, generate as rgen
        from pipelab.costs import DurationTable as RDT
        from pipelab.engine import CommModel as RCM
        from pipelab.simulate import overlap_report as r_overlap, simulate as rsim
    finally:
        sys.path.remove(ref)
    _, res = _run(method, p, m, cost, lat)
    rcfg = RC(L=2 * p, h=64, s=128, b=1, num_heads=2, p=p, m=m)
    rsched = rgen(method, rcfg, RDT.from_units(1, 3, 2))
    rrep = r_overlap(rsim(rsched, RDT.from_units(1, 3, 2), RCM.uniform(cost, lat)))
    rep = sim.overlap_report(res)
    assert [(r.task_id, r.stage, r.mb, r.wait, r.hidden) for r in rep.rows] == \
        [(r.task_id, r.stage, r.mb, r.wait, r.hidden) for r in rrep.rows]
    assert rep.per_stage_wait == rrep.per_stage_wait
    assert (rep.total_wait, rep.steady_wait, rep.warmup_mbs) == \
        (rrep.total_wait, rrep.steady_wait, rrep.warmup_mbs)

"""Closed-form bubble / memory formulas (restating ``P/analytic.py``), pinned
to the reference's worked examples (``T/test_analytic.py:27-60``) and checked
against the list-scheduling simulator with tolerance 0 (the reference's own
``compare`` contract, ``P/analytic.py:128-158``)."""

import pytest

from paper_2507_00394_b200 import ModelConfig, generate, simulate
from paper_2507_00394_b200.analytic import (bubble_fraction, bubble_time, compare,
                                            peak_activation_elements, stage_memory_bytes)
from paper_2507_00394_b200.config import ConfigError
from paper_2507_00394_b200.costs import DurationTable


def _cfg(**kw):
    base = dict(L=4, h=8, s=8, b=1, num_heads=2, p=2, m=4)
    base.update(kw)
    return ModelConfig(**base)


def test_bubble_worked_examples():
    assert bubble_time("1f1b", 4, 8, 1, 3, 2) == 108
    assert bubble_time("zb1p", 4, 8, 1, 3, 2) == 72
    assert bubble_time("helix_naive", 4, 8, 1, 3, 2) == 27
    assert bubble_time("helix_twofold", 4, 8, 1, 3, 2) == 54
    assert bubble_time("helix_twofold_rc", 4, 8, 1, 3, 2) == 72
    assert bubble_time("helix_naive", 4, 9, 1, 3, 2) == 27
    for bad in (("1f1b", 4, 9), ("zb1p", 4, 9), ("whatever", 4, 8)):
        with pytest.raises(ConfigError):
            bubble_time(*bad, 1, 3, 2)


def test_memory_worked_examples():
    cfg = _cfg(L=8, p=4, m=8)
    bshL = cfg.b * cfg.s * cfg.h * cfg.L
    assert peak_activation_elements("1f1b", cfg, 0) == 16 * bshL
    assert peak_activation_elements("1f1b", _cfg(L=8, p=2, m=4), 0) == \
        peak_activation_elements("1f1b", _cfg(L=8, p=8, m=16), 0)
    assert {peak_activation_elements("helix_twofold_rc", cfg, i) for i in range(4)} == \
        {4 * cfg.b * cfg.s * cfg.h * cfg.m * cfg.L // cfg.p}
    with pytest.raises(ConfigError):
        peak_activation_elements("nope", cfg, 0)


@pytest.mark.parametrize("method", ["1f1b", "zb1p", "helix_naive", "helix_twofold", "helix_twofold_rc"])
@pytest.mark.parametrize("p,L,m", [(2, 4, 4), (4, 8, 8), (4, 4, 16)])
def test_formulas_match_simulator_exactly(method, p, L, m):
    cfg = _cfg(L=L, p=p, m=m)
    table = DurationTable.from_units(1, 3, 2)
    res = simulate(generate(method, cfg, table), table)
    rep = compare(method, cfg, table, res.metrics, tolerance=0.0)
    assert rep.ok, "\n".join(rep.lines())


def test_bubble_fraction_and_memory_model():
    table = DurationTable.from_units(1, 3, 2)
    cfg = _cfg(L=8, p=4, m=8)
    assert 0 < bubble_fraction("helix_twofold", cfg, table) < bubble_fraction("1f1b", cfg, table)
    assert bubble_fraction("helix_twofold", cfg.with_(p=1, m=2), table) == 0
    big = ModelConfig(L=32, h=4096, s=131072, b=1, num_heads=32, p=8, m=16)
    full = stage_memory_bytes("helix_twofold_rc", big, mlp_chunk=16384)
    dropped = stage_memory_bytes("helix_twofold_rc", big, drop_pre_x=True, mlp_chunk=16384)
    assert dropped["stash"] * 4 == full["stash"] * 3
    assert full["total"] == sum(v for k, v in full.items() if k != "total")


def test_task_class_simulation_reproduces_table_simulation():
    """simulate_classes with per-class durations recovered from a simulated
    timeline replays to the same makespan (the stage probe's prediction path)."""
    from paper_2507_00394_b200 import ModelConfig, generate
    from paper_2507_00394_b200.costs import DurationTable
    from paper_2507_00394_b200.simulate import simulate, simulate_classes, task_class_durations
    cfg = ModelConfig(L=8, h=64, s=128, b=1, num_heads=2, p=4, m=8)
    table = DurationTable.from_units(1, 3, 2)
    for method in ("helix_twofold", "helix_twofold_rc", "1f1b", "zb1p"):
        sched = generate(method, cfg, table)
        ref = simulate(sched, table)
        tl_ms = {k: (a / 1e6, b / 1e6) for k, (a, b) in ref.timeline.items()}
        classes = task_class_durations(sched, tl_ms)
        got = simulate_classes(sched, classes)
        assert got.metrics.makespan == ref.metrics.makespan, method

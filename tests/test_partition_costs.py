"""Placement rules (T/test_partition.py) and the cost-model identities the
executor relies on (payload volumes, stash elements)."""

import random

import pytest

from paper_2507_00394_b200.config import ConfigError, ModelConfig
from paper_2507_00394_b200.costs import (
    EDGE_ATTN_POST, EDGE_BOUNDARY, EDGE_PRE_ATTN, DurationTable, activation_elements,
    attention_kernel_flops, b200_flops_per_token, comm_volume, op_flops)
from paper_2507_00394_b200.partition import (
    attn_stage, audit_partition, check_helix_config, post_stage, pre_stage)
from paper_2507_00394_b200.simulate import simulate
from paper_2507_00394_b200 import generate


def _cfg(L, p, m=None):
    return ModelConfig(L=L, h=8, s=8, b=1, num_heads=2, p=p, m=m or p)


def test_placement_small_case_by_hand():
    cfg = _cfg(L=4, p=2)
    assert [pre_stage(l, cfg) for l in range(4)] == [0, 1, 0, 1]
    assert [post_stage(l, cfg) for l in range(4)] == [1, 0, 1, 0]
    assert [attn_stage(0, i, cfg) for i in range(4)] == [1, 0, 1, 0]
    assert [attn_stage(1, i, cfg) for i in range(4)] == [0, 1, 0, 1]


def test_fused_unit_shares_a_stage():
    rng = random.Random(21)
    for _ in range(100):
        p = rng.choice([2, 4, 8])
        cfg = _cfg(L=p * rng.randint(1, 4), p=p)
        assert post_stage(cfg.L - 1, cfg) == 0
        for l in range(1, cfg.L - 1):
            assert post_stage(l - 1, cfg) == pre_stage(l, cfg)


def test_attention_spread_covers_all_stages():
    rng = random.Random(5)
    for _ in range(100):
        p = rng.choice([2, 3, 4, 8])
        cfg = _cfg(L=p, p=p, m=2 * p)
        l, i0 = rng.randrange(cfg.L), rng.randrange(cfg.m)
        assert {attn_stage(l, i0 + k, cfg) for k in range(p)} == set(range(p))


def test_audit_balanced():
    for p, mult in ((2, 1), (2, 4), (4, 2), (8, 1)):
        rep = audit_partition(_cfg(L=p * mult, p=p))
        assert rep.balanced and rep.pre_counts == [mult] * p
        assert all(row == [mult] * p for row in rep.attn_counts_by_mb)
        assert len(set(rep.params_per_stage)) == 1


def test_check_helix_config_divisibility():
    check_helix_config(_cfg(L=4, p=2, m=2))
    for bad in (dict(L=3, p=2, m=2), dict(L=4, p=2, m=3)):
        with pytest.raises(ConfigError):
            check_helix_config(_cfg(**bad))
    check_helix_config(_cfg(L=4, p=2, m=4), fold=2)
    with pytest.raises(ConfigError):
        check_helix_config(_cfg(L=4, p=2, m=2), fold=2)


def test_config_validation():
    with pytest.raises(ConfigError):
        ModelConfig(L=1, h=6, s=4, b=1, num_heads=4, p=1, m=1)
    with pytest.raises(ConfigError):
        ModelConfig(L=0, h=8, s=4, b=1, num_heads=2, p=1, m=1)


def test_volumes_and_stash_split():
    cfg = ModelConfig(L=4, h=256, s=1024, b=1, num_heads=4, p=2, m=4)
    bsh = 1024 * 256
    assert comm_volume(cfg, EDGE_PRE_ATTN, True) == 2 * bsh + 3 * 256 * 256
    assert comm_volume(cfg, EDGE_PRE_ATTN, False) == 4 * bsh
    assert comm_volume(cfg, EDGE_ATTN_POST) == 2 * bsh
    assert comm_volume(cfg, EDGE_BOUNDARY) == bsh
    assert activation_elements(cfg, qkv_in_attention=True) == \
        {"pre": bsh, "attn": 4 * bsh, "post": 11 * bsh}
    assert activation_elements(cfg, recompute=True) == {"pre": 0, "attn": 2 * bsh, "post": 2 * bsh}
    with pytest.raises(ConfigError):
        comm_volume(cfg, "nope")


def test_flop_accounting():
    cfg = ModelConfig(L=24, h=2048, s=32768, b=1, num_heads=16, p=4, m=8)
    assert b200_flops_per_token(cfg) == 16_911_433_728  # 1.691e10
    ops = op_flops(cfg)
    assert ops["attn"].bwd_b == 2 * ops["attn"].fwd
    fwd, bwd = attention_kernel_flops(cfg)
    assert fwd == ops["attn"].fwd // 2 and bwd == fwd * 5 // 2


def test_simulated_1f1b_bubble_fraction():
    # (p-1)/(m+p-1) for 1F1B under unit tables (T/test_sim.py:134-142)
    for p, m in ((2, 4), (4, 8), (4, 4)):
        cfg = ModelConfig(L=p, h=8, s=8, b=1, num_heads=2, p=p, m=m)
        res = simulate(generate("1f1b", cfg, DurationTable.from_units(1, 3, 2)),
                       DurationTable.from_units(1, 3, 2))
        assert res.metrics.bubble_fraction == pytest.approx((p - 1) / (m + p - 1))


def test_1f1b_rc_extension_schedule():
    """B200 extension: 1F1B with recomputation-without-attention inside chunks.
    Same tasks and order as 1F1B, stash accounting at the recompute retention,
    and the chunk backward billed with the re-run pre / post forward."""
    from paper_2507_00394_b200 import ModelConfig, generate, validate_schedule
    from paper_2507_00394_b200.costs import DurationTable, layer_activation_elements
    from paper_2507_00394_b200.simulate import simulate

    cfg = ModelConfig(L=4, h=64, s=128, b=1, num_heads=2, p=2, m=4)
    units = DurationTable.from_units(1, 3, 2)
    base, rc = generate("1f1b", cfg, units), generate("1f1b_rc", cfg, units)
    validate_schedule(rc)
    assert rc.method == "1f1b_rc" and int(rc.meta["recompute"]) == 1
    assert sorted(base.tasks) == sorted(rc.tasks) and base.per_stage_order == rc.per_stage_order
    span = cfg.L // cfg.p
    f = rc.tasks["f.s0.m0"]
    assert f.mem_delta == layer_activation_elements(cfg, recompute=True) * span
    assert rc.tasks["b.s0.m0"].mem_delta == -f.mem_delta
    # the rc chunk backward costs span * (pre fwd + post fwd) more
    sb, sr = simulate(base, units), simulate(rc, units)
    db = sb.timeline["b.s0.m0"][1] - sb.timeline["b.s0.m0"][0]
    dr = sr.timeline["b.s0.m0"][1] - sr.timeline["b.s0.m0"][0]
    assert dr - db == span * (units.of("pre", "fwd") + units.of("post", "fwd"))
    assert sr.metrics.makespan > sb.metrics.makespan

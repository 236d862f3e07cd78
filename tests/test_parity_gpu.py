"""End-to-end parity on the B200: ``execute_schedule`` (libhx kernels, bf16 with
fp32 accumulation) against the float64 oracle on the same seeded inputs.

Stated tolerances (bf16 activations / weights, fp32 accumulation and grads):
  loss            |got - ref| / ref                     <= 2e-3
  each gradient   cosine(got, ref)                      >= 0.9995
                  max|got - ref| / max|ref|             <= 2e-2
The schedule itself is bit-exact (tests/test_schedule_parity.py).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import helix_oracle as O  # noqa: E402
from paper_2507_00394_b200 import METHODS, ModelConfig, generate  # noqa: E402
from paper_2507_00394_b200.costs import DurationTable  # noqa: E402
from paper_2507_00394_b200.runtime import (PayloadMismatch, StalledSchedule,  # noqa: E402
                                           execute_schedule, make_inputs, make_model)

UNIT = DurationTable.from_units(1, 3, 2)
LOSS_TOL, COS_TOL, MAX_TOL = 2e-3, 0.9995, 2e-2

SMALL = ModelConfig(L=2, h=128, s=256, b=1, num_heads=2, p=2, m=4)      # head_dim 64
WIDE = ModelConfig(L=2, h=256, s=384, b=2, num_heads=2, p=2, m=4)       # head_dim 128, b=2
TINY = ModelConfig(L=4, h=256, s=1024, b=1, num_heads=4, p=2, m=4)      # BASELINE config 1
TINY_LOSSES = [3.327261203817688, 3.3800507339316543, 3.443091222231624, 3.4279542847160513]

_ORACLE_CACHE = {}


def oracle_for(cfg, pseed=0, iseed=1, chunk=None):
    key = (cfg, pseed, iseed)
    if key not in _ORACLE_CACHE:
        params = O.make_model(cfg.L, cfg.h, pseed)
        inputs = O.make_inputs(cfg.m, cfg.s, cfg.b, cfg.h, iseed)
        _ORACLE_CACHE[key] = O.sequential_oracle(params, inputs, cfg.num_heads, chunk)
    return _ORACLE_CACHE[key]


def compare(res, ref, L, label=""):
    worst = {"loss": 0.0, "cos": 1.0, "max": 0.0}
    for got, want in zip(res.losses, ref.losses):
        worst["loss"] = max(worst["loss"], abs(got - want) / abs(want))
    for l in range(L):
        for k in O.FIELDS:
            g, r = res.param_grads[l][k].ravel(), ref.param_grads[l][k].ravel()
            cos = float(g @ r / (np.linalg.norm(g) * np.linalg.norm(r)))
            mx = float(np.abs(g - r).max() / np.abs(r).max())
            worst["cos"] = min(worst["cos"], cos)
            worst["max"] = max(worst["max"], mx)
    print(f"[parity] {label} worst loss rel {worst['loss']:.2e} cos {worst['cos']:.6f} max {worst['max']:.2e}")
    assert worst["loss"] <= LOSS_TOL, worst
    assert worst["cos"] >= COS_TOL, worst
    assert worst["max"] <= MAX_TOL, worst
    return worst


def run(cfg, method, pseed=0, iseed=1, **kw):
    sched = generate(method, cfg, UNIT)
    return execute_schedule(sched, make_model(cfg, pseed), make_inputs(cfg, iseed), **kw)


@pytest.mark.parametrize("method", METHODS)
def test_every_method_matches_oracle_small(method):
    res = run(SMALL, method)
    assert res.mode == "replay"
    compare(res, oracle_for(SMALL), SMALL.L, f"small {method}")


@pytest.mark.parametrize("method", ["helix_twofold", "helix_twofold_rc", "1f1b", "1f1b_rc"])
def test_head_dim_128_batch_2_matches_oracle(method):
    compare(run(WIDE, method), oracle_for(WIDE), WIDE.L, f"wide {method}")


def test_multistream_equals_replay_within_tolerance():
    a = run(SMALL, "helix_twofold")
    b = run(SMALL, "helix_twofold", threaded=True)
    assert b.mode == "threaded"
    compare(b, oracle_for(SMALL), SMALL.L, "small multistream")
    assert np.allclose(a.losses, b.losses, rtol=1e-3)


def test_chunk_and_recompute_invariance():
    ref = oracle_for(SMALL)
    for chunk in (64, 100, None):
        compare(run(SMALL, "helix_twofold_rc", mlp_chunk=chunk), ref, SMALL.L, f"rc chunk={chunk}")


def test_tiny_baseline_config_against_oracle():
    res = run(TINY, "helix_twofold")
    for got, want in zip(res.losses, TINY_LOSSES):
        assert abs(got - want) / want <= LOSS_TOL
    compare(res, oracle_for(TINY), TINY.L, "tiny helix_twofold")


def test_peak_stash_accounting_matches_reference_formula():
    cfg = SMALL
    bsh = cfg.b * cfg.s * cfg.h
    res = run(cfg, "helix_twofold")
    full = (16 * bsh + 3 * cfg.h * cfg.h) * cfg.m * cfg.L // cfg.p
    assert res.peak_stash_elements == [full] * cfg.p
    rc = run(cfg, "helix_twofold_rc")
    kept = (4 * bsh + 3 * cfg.h * cfg.h) * cfg.m * cfg.L // cfg.p
    assert all(kept <= pk <= kept + 16 * bsh for pk in rc.peak_stash_elements)


def test_rejects_wrong_volume():
    from dataclasses import replace
    sched = generate("helix_naive", SMALL, UNIT)
    sid = next(t.id for t in sched.tasks.values() if t.kind == "SEND")
    sched.tasks[sid] = replace(sched.tasks[sid], volume=sched.tasks[sid].volume + 1)
    with pytest.raises(PayloadMismatch):
        execute_schedule(sched, make_model(SMALL, 0), make_inputs(SMALL, 1))


def test_reports_stall():
    sched = generate("1f1b", SMALL, UNIT)
    sched.per_stage_order[0].reverse()
    with pytest.raises(StalledSchedule):
        execute_schedule(sched, make_model(SMALL, 0), make_inputs(SMALL, 1))


@pytest.mark.parametrize("qkv", [True, False])
def test_regen_pre_x_matches_oracle(qkv):
    """pre stashes drop x; rc.pre(l) rebuilds it from
    post(l-1)'s retention (two extra MLP GEMMs) -- same numbers, ragged slabs."""
    for cfg, chunk in ((SMALL, 100), (WIDE, None)):
        sched = generate("helix_twofold_rc", cfg, UNIT, qkv_in_attention=qkv)
        res = execute_schedule(sched, make_model(cfg, 0), make_inputs(cfg, 1), mlp_chunk=chunk,
                               regen_pre_x=True)
        compare(res, oracle_for(cfg), cfg.L, f"regen_pre_x qkv={qkv} chunk={chunk}")


def test_streamed_inputs_equal_resident_inputs():
    """The input streamer (host inputs copied per task on a side stream) gives
    the results of device-resident inputs."""
    for method in ("helix_twofold", "helix_twofold_rc", "1f1b"):
        a = run(SMALL, method, stream_inputs=False)
        b = run(SMALL, method, stream_inputs=True)
        assert np.allclose(a.losses, b.losses, rtol=1e-6), method
        for l in range(SMALL.L):
            for k in O.FIELDS:
                g, r = b.param_grads[l][k], a.param_grads[l][k]
                assert np.abs(g - r).max() <= 1e-3 * np.abs(r).max(), (method, l, k)


@pytest.mark.parametrize("method,chunk,regen,stream", [("helix_twofold", None, False, False),
                                                       ("helix_twofold_rc", 64, False, True),
                                                       ("helix_twofold_rc", 100, True, False),
                                                       ("1f1b_rc", 64, False, True),
                                                       ("zb1p", None, False, False)])
def test_device_stash_bytes_match_memplan(method, chunk, regen, stream):
    """runtime/memplan.stash_walk with the LayerMath tensor set (bf16, fp32 LSE,
    per-slab m1/g, no stashed O) equals the distinct device bytes the executor
    holds, at p = 1 (one stage per process: the same sharing as one rank)."""
    from paper_2507_00394_b200.runtime import HelixRuntime
    from paper_2507_00394_b200.runtime.executor import DeviceModel
    from paper_2507_00394_b200.runtime.memplan import stash_walk
    cfg = ModelConfig(L=4, h=128, s=256, b=1, num_heads=2, p=1, m=2)
    sched = generate(method, cfg, UNIT)
    dev = torch.device("cuda", 0)
    model = DeviceModel.from_host(sched, make_model(cfg, 0), [0], dev)
    rt = HelixRuntime(sched, model, chunk, "replay", dev, regen_pre_x=regen)
    inputs = [torch.from_numpy(x).to(torch.bfloat16).reshape(cfg.s * cfg.b, cfg.h) for x in make_inputs(cfg, 1)]
    inputs = [x.pin_memory() if stream else x.to(dev) for x in inputs]
    rt.run(inputs)
    torch.cuda.synchronize()
    want, at = stash_walk(sched, 0, regen_pre_x=regen, stream_inputs=stream)
    assert rt.stages[0].peak_bytes == want, (rt.stages[0].peak_bytes, rt.stages[0].peak_bytes_at, want, at)


@pytest.mark.parametrize("method", ["helix_twofold_rc", "1f1b"])
def test_stage_probe_memory_matches_plan(method):
    """HelixRuntime mode "probe" (one rank of a 4-stage pipeline, loopback
    receives) with the B200 kernels holds exactly the distinct device bytes
    runtime/memplan.py predicts for that rank, on every stage."""
    from paper_2507_00394_b200.partition import pre_stage
    from paper_2507_00394_b200.runtime import HelixRuntime
    from paper_2507_00394_b200.runtime.executor import DeviceModel
    from paper_2507_00394_b200.runtime.memplan import stash_walk
    cfg = ModelConfig(L=4, h=128, s=256, b=1, num_heads=2, p=4, m=8)
    sched = generate(method, cfg, UNIT)
    dev = torch.device("cuda", 0)
    chunked = method == "1f1b"
    for rank in range(cfg.p):
        model = DeviceModel.from_host(sched, make_model(cfg, 0), [rank], dev)
        rt = HelixRuntime(sched, model, 64, "probe", dev, rank=rank)
        first = 0 if chunked else pre_stage(0, cfg)
        xs = [torch.from_numpy(x).to(dev, torch.bfloat16).reshape(cfg.s * cfg.b, cfg.h) if rank == first else None
              for x in make_inputs(cfg, 1)]
        rt.run(xs)
        torch.cuda.synchronize()
        want, at = stash_walk(sched, rank)
        assert rt.stages[rank].peak_bytes == want, (method, rank, rt.stages[rank].peak_bytes_at, at)


@pytest.mark.parametrize("mode", ["replay", "multistream"])
def test_cuda_graph_iteration_matches_eager(mode):
    """HelixRuntime.capture: one iteration as a CUDA graph (BASELINE config 1,
    host-launch bound eagerly) replays to the eager results, and keeps doing so
    with new inputs copied into its static buffers."""
    import time
    from paper_2507_00394_b200.runtime import HelixRuntime
    from paper_2507_00394_b200.runtime.executor import DeviceModel
    cfg = TINY
    sched = generate("helix_twofold", cfg, UNIT)
    dev = torch.device("cuda", 0)
    model = DeviceModel.from_host(sched, make_model(cfg, 0), range(cfg.p), dev)
    rt = HelixRuntime(sched, model, None, mode, dev)
    xs = [torch.from_numpy(x).to(dev, torch.bfloat16).reshape(cfg.s * cfg.b, cfg.h) for x in make_inputs(cfg, 1)]
    rt.run(xs)
    eager_l = rt.losses()
    eager_g = {l: {k: g.clone() for k, g in dl.grad.items()} for l, dl in model.layers.items()}
    g = rt.capture(xs)
    g.replay()
    torch.cuda.synchronize()
    assert np.allclose(rt.losses(), eager_l, rtol=1e-5)
    for l, d in eager_g.items():
        for k, v in d.items():
            assert torch.allclose(model.layers[l].grad[k], v, rtol=1e-3, atol=1e-5), (l, k)
    assert np.allclose(rt.losses(), TINY_LOSSES, rtol=LOSS_TOL)
    xs2 = [x.flip(0).contiguous() for x in xs]       # new inputs through the static buffers
    rt2 = HelixRuntime(sched, DeviceModel.from_host(sched, make_model(cfg, 0), range(cfg.p), dev), None, mode, dev)
    rt2.run(xs2)
    g.replay(xs2)
    torch.cuda.synchronize()
    assert np.allclose(rt.losses(), rt2.losses(), rtol=1e-5)
    # timing (printed): eager vs graphed iteration, CUDA events
    def t(fn, n=10):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n
    te, tg = t(lambda: rt2.run(xs2)), t(lambda: g.replay())
    print(f"[graph] config 1 {mode}: eager {te:.2f} ms, graphed {tg:.2f} ms per iteration")


# Ragged shapes end to end: s not a multiple of the 128-row tiles, b = 3, three
# heads of 64 (h = 192: GEMM N / K not multiples of the 256-wide tiles), an MLP
# chunk that does not divide s*b, and a p = 3 helix (every stage pair exchanges).
RAGGED = ModelConfig(L=3, h=192, s=200, b=3, num_heads=3, p=3, m=6)


@pytest.mark.parametrize("method,chunk", [("helix_twofold", None), ("helix_twofold_rc", 250), ("1f1b", None),
                                          ("zb1p", 130)])
def test_ragged_shapes_match_oracle(method, chunk):
    compare(run(RAGGED, method, mlp_chunk=chunk), oracle_for(RAGGED), RAGGED.L, f"ragged {method} chunk={chunk}")

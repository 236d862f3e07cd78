"""The per-rank memory plan (runtime/memplan.py) against the executor's own
measurement: on every rank of a gloo world, the distinct tensors held by the
stash and the deferred W contexts (weights and inputs excluded) peak at
exactly the bytes ``stash_walk`` predicts, for every method, with and
without recomputation and ``regen_pre_x``.  The float64 test double keeps
m1 / g whole and has no LSE, which ``Dtypes`` states."""

import pytest

from paper_2507_00394_b200 import EXTENSION_METHODS, METHODS, ModelConfig, generate
from paper_2507_00394_b200.runtime.memplan import GB, Dtypes, offload_needed, plan, stash_walk
from tests.test_distributed_cpu import TOY2, TOY4, UNIT, run_world

F64 = Dtypes(act=8, wgrad=8, weight=8, lse=0, delta=0, slab_mlp=False)


def _check(world, toy, method, regen=False):
    env = {"HX_TEST_REGEN_PRE_X": "1"} if regen else None
    *_, allstats = run_world(world, toy, method, with_stats=True, env=env)
    sched = generate(method, ModelConfig(**toy), UNIT)
    for rank, per_iter in enumerate(allstats):
        want, at = stash_walk(sched, rank, F64, regen_pre_x=regen)
        for st in per_iter:
            assert st["stash_peak_bytes"] == want, (method, rank, st["stash_peak_bytes"], want,
                                                    st["stash_peak_at"], at)


@pytest.mark.parametrize("method", METHODS + EXTENSION_METHODS)
def test_stash_walk_matches_executor_two_ranks(method):
    _check(2, TOY2, method)


@pytest.mark.parametrize("method", ["helix_twofold", "helix_twofold_rc", "1f1b_rc"])
def test_stash_walk_matches_executor_four_ranks(method):
    _check(4, TOY4, method)


def test_stash_walk_with_regen_pre_x():
    _check(4, TOY4, "helix_twofold_rc", regen=True)


def test_config4_plan_fits_with_bounded_host_offload():
    """SURVEY H1 at BASELINE config 4 (7B, s=128k, p=8, m=16): the rc stash
    does not fit one B200 as recorded in round 1 (4bsh + O per layer-mb); with
    D shipped instead of O, x regenerated and the inputs streamed from host
    memory, every rank needs at most 64 GB of host offload (verdict r1 item 6)."""
    cfg = ModelConfig(L=32, h=4096, s=131072, b=1, num_heads=32, p=8, m=16)
    sched = generate("helix_twofold_rc", cfg, UNIT)
    hbm = 180 * GB
    plain = [plan(sched, r, 16384, durations=UNIT) for r in range(8)]
    regen = [plan(sched, r, 16384, regen_pre_x=True, durations=UNIT, stream_inputs=True) for r in range(8)]
    worst_plain = max(offload_needed(x, hbm) for x in plain)
    worst_regen = max(offload_needed(x, hbm) for x in regen)
    assert worst_plain > 64 * GB                # 4bsh retention alone overflows
    assert worst_regen <= 64 * GB, worst_regen / GB
    # regenerating x removes b*s*h per (layer, micro-batch) the rank holds at its peak
    assert max(x.stash_peak for x in plain) - max(x.stash_peak for x in regen) > 40 * GB


def test_plan_bounds_and_single_stage():
    cfg = ModelConfig(L=24, h=2048, s=32768, b=1, num_heads=16, p=1, m=2)
    sched = generate("helix_twofold", cfg, UNIT)
    pl = plan(sched, 0)
    # full stash at p=1: x (input for l=0), ln_out, qkv, lse / o, x2, ln2, m1, g per layer-mb
    act = cfg.s * cfg.h * 2
    per = 1 + 3 + 1 + 1 + 1 + 1 + 4 + 4
    lse = cfg.num_heads * cfg.s * 4
    # peak at the end of the forward; the inputs (l = 0's x) are resident, not
    # stash, and every micro-batch's output z waits for its loss (stage-local payload)
    assert pl.stash_peak == cfg.m * cfg.L * (per * act + lse) - cfg.m * act + cfg.m * act, pl
    assert pl.comm == 0 and pl.inputs == cfg.m * act
    # worst-case comm bound >= timeline estimate
    cfg4 = ModelConfig(L=8, h=1024, s=8192, b=1, num_heads=8, p=4, m=8)
    s4 = generate("helix_twofold_rc", cfg4, UNIT)
    for r in range(4):
        assert plan(s4, r).comm >= plan(s4, r, durations=UNIT).comm


@pytest.mark.parametrize("method", ["helix_twofold", "helix_twofold_rc", "1f1b", "zb1p"])
def test_stage_probe_matches_stash_walk(method):
    """HelixRuntime mode "probe" (one rank, loopback receives) holds exactly the
    per-rank stash the plan predicts, on every stage of a 4-stage pipeline."""
    import numpy as np
    import torch

    from paper_2507_00394_b200.partition import pre_stage
    from paper_2507_00394_b200.runtime.executor import DeviceModel, HelixRuntime, stage_fields
    from paper_2507_00394_b200.runtime.model import DeviceLayer, make_inputs, make_model
    from tests.cpu_math import CpuMath

    cfg = ModelConfig(**TOY4)
    sched = generate(method, cfg, UNIT)
    params = make_model(cfg, 0)
    chunked = method in ("1f1b", "zb1p")
    for rank in range(cfg.p):
        layers = {}
        for l, p in enumerate(params):
            need, own = stage_fields(sched, rank, l)
            if need:
                layers[l] = DeviceLayer({k: torch.from_numpy(np.ascontiguousarray(getattr(p, k))) for k in need},
                                        own, grad_dtype=torch.float64)
        rt = HelixRuntime(sched, DeviceModel(layers), None, "probe", torch.device("cpu"),
                          math=CpuMath(cfg, bool(int(sched.meta["qkv"]))), rank=rank)
        first = 0 if chunked else pre_stage(0, cfg)
        xs = [torch.from_numpy(x).reshape(cfg.s * cfg.b, cfg.h) if rank == first else None
              for x in make_inputs(cfg, 1)]
        rt.run(xs)
        want, at = stash_walk(sched, rank, F64)
        assert rt.stages[rank].peak_bytes == want, (method, rank, rt.stages[rank].peak_bytes_at, at)


@pytest.mark.parametrize("method", ["helix_twofold", "helix_twofold_rc", "1f1b_rc", "zb1p"])
def test_streamed_inputs_match_walk_and_results(method):
    """Host-resident inputs (executor _InputStreamer): same losses and grads as
    resident inputs, and the held bytes the walk predicts with stream_inputs."""
    import numpy as np
    import torch

    from paper_2507_00394_b200.runtime.executor import DeviceModel, HelixRuntime, stage_fields
    from paper_2507_00394_b200.runtime.model import DeviceLayer, make_inputs, make_model
    from tests.cpu_math import CpuMath

    cfg = ModelConfig(**TOY2)
    sched = generate(method, cfg, UNIT)
    params = make_model(cfg, 0)
    xs = [torch.from_numpy(x).reshape(cfg.s * cfg.b, cfg.h) for x in make_inputs(cfg, 1)]
    out = []
    for stream in (False, True):
        layers = {}
        for l, p in enumerate(params):
            t = {k: torch.from_numpy(np.ascontiguousarray(getattr(p, k))) for k in p.__dataclass_fields__}
            layers[l] = DeviceLayer(t, tuple(t), grad_dtype=torch.float64)
        # one stage of the pipeline at a time (probe) so sharing matches one rank
        rt = HelixRuntime(sched, DeviceModel(layers), None, "probe", torch.device("cpu"),
                          math=CpuMath(cfg, bool(int(sched.meta["qkv"]))), rank=0, stream_inputs=stream)
        rt.run(xs)
        want, _ = stash_walk(sched, 0, F64, stream_inputs=stream)
        assert rt.stages[0].peak_bytes == want, (stream, rt.stages[0].peak_bytes_at)
        out.append(rt.grads_numpy())
    for l in out[0]:
        for k in out[0][l]:
            assert np.array_equal(out[0][l][k], out[1][l][k]), (l, k)

"""Executor host logic on CPU (replay driver + the float64 test double
``tests/cpu_math.CpuMath``): stash accounting against the reference's frozen
peaks (``T/test_runtime.py:188-208``; ``tests/golden/runtime_meta.json``)."""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2507_00394_b200 import METHODS, ModelConfig, generate
from paper_2507_00394_b200.costs import DurationTable
from paper_2507_00394_b200.runtime.executor import DeviceModel, HelixRuntime, stage_fields
from paper_2507_00394_b200.runtime.model import DeviceLayer, make_inputs, make_model
from tests.cpu_math import CpuMath

META = json.loads((Path(__file__).parent / "golden" / "runtime_meta.json").read_text())
UNIT = DurationTable.from_units(1, 3, 2)


def run_replay(cfg, method, **kw):
    sched = generate(method, cfg, UNIT)
    params = make_model(cfg, 0)
    layers = {}
    for l, p in enumerate(params):
        need, own = set(), set()
        for st in range(cfg.p):
            n, o = stage_fields(sched, st, l)
            need |= set(n)
            own |= set(o)
        t = {k: torch.from_numpy(np.ascontiguousarray(getattr(p, k))) for k in need}
        layers[l] = DeviceLayer(t, tuple(own), grad_dtype=torch.float64)
    rt = HelixRuntime(sched, DeviceModel(layers), None, "replay", torch.device("cpu"),
                      math=CpuMath(cfg, bool(int(sched.meta["qkv"]))), **kw)
    rt.run([torch.from_numpy(x).reshape(cfg.s * cfg.b, cfg.h) for x in make_inputs(cfg, 1)])
    return rt


@pytest.mark.parametrize("method", METHODS)
def test_peak_stash_elements_match_reference(method):
    """Includes ZB1P, whose deferred W contexts the reference counts with the
    LayerNorm ``xhat``/``d_ln`` tensors (frozen value [9216, 10240])."""
    toy = META["toy"]
    cfg = ModelConfig(**toy["config"])
    rt = run_replay(cfg, method)
    peaks = [rt.stages[i].peak for i in range(cfg.p)]
    assert peaks == toy["peak_stash_elements"][method], (method, peaks)
    losses = rt.losses()
    assert np.allclose(losses, toy["losses"], rtol=1e-10)


@pytest.mark.parametrize("qkv", [True, False])
def test_regen_pre_x_replay_matches_plain_rc(qkv):
    """regen_pre_x rebuilds every pre stash's x (l > 0) from post(l-1): same
    losses and gradients as the plain rc run, same logical peaks."""
    toy = META["toy"]
    cfg = ModelConfig(**toy["config"])

    def run(**kw):
        sched = generate("helix_twofold_rc", cfg, UNIT, qkv_in_attention=qkv)
        params = make_model(cfg, 0)
        layers = {}
        for l, p in enumerate(params):
            t = {k: torch.from_numpy(np.ascontiguousarray(getattr(p, k))) for k in p.__dataclass_fields__}
            layers[l] = DeviceLayer(t, tuple(t), grad_dtype=torch.float64)
        rt = HelixRuntime(sched, DeviceModel(layers), None, "replay", torch.device("cpu"),
                          math=CpuMath(cfg, qkv), **kw)
        rt.run([torch.from_numpy(x).reshape(cfg.s * cfg.b, cfg.h) for x in make_inputs(cfg, 1)])
        return rt

    a, b = run(), run(regen_pre_x=True)
    assert np.allclose(a.losses(), b.losses(), rtol=1e-12)
    ga, gb = a.grads_numpy(), b.grads_numpy()
    for l in ga:
        for k in ga[l]:
            assert np.allclose(ga[l][k], gb[l][k], rtol=1e-10, atol=1e-13), (l, k)
    assert [a.stages[i].peak for i in range(cfg.p)] == [b.stages[i].peak for i in range(cfg.p)]


def test_regen_pre_x_rejects_schedules_without_rc():
    cfg = ModelConfig(**META["toy"]["config"])
    with pytest.raises(Exception, match="regen_pre_x"):
        run_replay(cfg, "helix_twofold", regen_pre_x=True)

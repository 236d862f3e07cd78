"""Multi-process executor on CPU: world_size 2 and 4 over gloo, one rank per
helix stage, running the SAME distributed driver (P2PPlan + per-directed-pair
groups + pre-posted receives) that uses NCCL on the B200 box.  The component
math is the float64 test double in tests/cpu_math.py, so results must match
the float64 oracle to ~1e-10 — which pins routing, send/recv ordering,
payload layouts and gradient ownership for every schedule method.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import helix_oracle as O
from paper_2507_00394_b200 import EXTENSION_METHODS, METHODS, ModelConfig, generate
from paper_2507_00394_b200.costs import DurationTable
from paper_2507_00394_b200.runtime.executor import (
    DeviceModel, HelixRuntime, P2PPlan, _gather_distributed, pair_groups, stage_fields)
from paper_2507_00394_b200.runtime.model import DeviceLayer, make_inputs, make_model

UNIT = DurationTable.from_units(1, 3, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg_kw, method, qkv, q, env=None):
    try:
        from tests.cpu_math import CpuMath
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **(env or {}))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = ModelConfig(**cfg_kw)
        sched = generate(method, cfg, UNIT, qkv_in_attention=qkv)
        params = make_model(cfg, 0)
        layers = {}
        for l, p in enumerate(params):
            need, own = stage_fields(sched, rank, l)
            if need:
                t = {k: torch.from_numpy(np.ascontiguousarray(getattr(p, k))) for k in need}
                layers[l] = DeviceLayer(t, own, grad_dtype=torch.float64)
        math = CpuMath(cfg, bool(int(sched.meta["qkv"])))
        rt = HelixRuntime(sched, DeviceModel(layers), None, "distributed", torch.device("cpu"),
                          math=math, rank=rank, groups=pair_groups(world),
                          regen_pre_x=os.environ.get("HX_TEST_REGEN_PRE_X") == "1")
        inputs = [torch.from_numpy(x).reshape(cfg.s * cfg.b, cfg.h) for x in make_inputs(cfg, 1)]
        rt.run(inputs)
        stats = [rt.comm_stats]
        rt.run(inputs)          # a second iteration reuses the cached groups and plan
        stats.append(rt.comm_stats)
        assert pair_groups(world) is rt.groups
        res = _gather_distributed(rt, params)
        allstats = [None] * world
        dist.all_gather_object(allstats, stats)
        if rank == 0:
            q.put(("ok", res.losses, res.param_grads, res.peak_stash_elements, allstats))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put(("err", f"rank {rank}: {type(e).__name__}: {e}", None, None, None))


def run_world(world, cfg_kw, method, qkv=True, with_stats=False, env=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_kw, method, qkv, q, env))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert out[0] == "ok", out[1]
    return out[1:] if with_stats else out[1:4]


def _oracle(cfg_kw):
    cfg = ModelConfig(**cfg_kw)
    return O.sequential_oracle(O.make_model(cfg.L, cfg.h, 0), O.make_inputs(cfg.m, cfg.s, cfg.b, cfg.h, 1),
                               cfg.num_heads)


TOY2 = dict(L=4, h=8, s=8, b=2, num_heads=2, p=2, m=4)
TOY4 = dict(L=4, h=8, s=8, b=1, num_heads=2, p=4, m=8)


@pytest.mark.parametrize("method", METHODS + EXTENSION_METHODS)
def test_two_ranks_every_method_matches_oracle(method):
    losses, grads, peaks = run_world(2, TOY2, method)
    ref = _oracle(TOY2)
    assert np.allclose(losses, ref.losses, rtol=1e-10, atol=0)
    for l in range(TOY2["L"]):
        for k in O.FIELDS:
            assert np.allclose(grads[l][k], ref.param_grads[l][k], rtol=1e-9, atol=1e-12), (method, l, k)
    assert len(peaks) == 2


def test_four_ranks_two_fold_and_recompute():
    ref = _oracle(TOY4)
    for method in ("helix_twofold", "helix_twofold_rc"):
        losses, grads, _ = run_world(4, TOY4, method)
        assert np.allclose(losses, ref.losses, rtol=1e-10)
        for l in range(TOY4["L"]):
            for k in O.FIELDS:
                assert np.allclose(grads[l][k], ref.param_grads[l][k], rtol=1e-9, atol=1e-12), (method, l, k)


def test_qkv_in_pre_layout_two_ranks():
    losses, grads, _ = run_world(2, TOY2, "helix_twofold", qkv=False)
    ref = _oracle(TOY2)
    assert np.allclose(losses, ref.losses, rtol=1e-10)


def test_p2p_plan_orders_are_consistent():
    # every directed pair: receiver's post order == sender's issue order, and
    # every SEND/RECV appears exactly once
    for method in METHODS:
        cfg = ModelConfig(**TOY4) if method.startswith("helix") else ModelConfig(**TOY4)
        sched = generate(method, cfg, UNIT)
        plan = P2PPlan(sched)
        sends = sorted(t.id for t in sched.tasks.values() if t.kind == "SEND")
        recvs = sorted(t.id for t in sched.tasks.values() if t.kind == "RECV")
        assert sorted(x for v in plan.send_seq.values() for x in v) == sends
        assert sorted(x for v in plan.recv_seq.values() for x in v) == recvs
        for (src, dst), seq in plan.send_seq.items():
            assert [sched.tasks[r].deps[0] for r in plan.recv_seq[(src, dst)]] == seq
            assert all(sched.tasks[s].stage == src and sched.tasks[s].peer == dst for s in seq)


@pytest.mark.parametrize("method", ["helix_twofold", "helix_twofold_rc", "1f1b"])
def test_sent_payloads_are_released(method):
    """A sender keeps a payload only until the receiver has taken it (the
    reference moves payload ownership to the consumer, ``executor.py:160-164``;
    round 1 kept every sent tensor until the iteration ended).  On NCCL
    completed sends are polled and dropped, and at most ``HX_SEND_CAP`` (4) per
    peer stay live; gloo's p2p work reports completion only from ``wait()``,
    so here the cap path itself is driven (cap 2, receives posted up front so
    the blocking wait cannot deadlock) and results must stay exact."""
    losses, grads, _peaks, allstats = run_world(
        4, TOY4, method, with_stats=True, env={"HX_RECV_AHEAD": "100000", "HX_SEND_CAP": "2"})
    for rank, per_iter in enumerate(allstats):
        for st in per_iter:
            live = st["max_live_sends_per_peer"]
            assert live and max(live.values()) <= 2, (rank, live)
    ref = _oracle(TOY4)
    assert np.allclose(losses, ref.losses, rtol=1e-10)
    for l in range(TOY4["L"]):
        for k in O.FIELDS:
            assert np.allclose(grads[l][k], ref.param_grads[l][k], rtol=1e-9, atol=1e-12), (method, l, k)


def test_default_lookahead_bounds_transit():
    """Default look-ahead: a payload waits on its sender until the receiver
    is ``recv_ahead`` tasks from consuming it; the per-peer count can never
    exceed the messages of that pair in one iteration and is 0 at the end."""
    cfg = ModelConfig(**TOY4)
    plan = P2PPlan(generate("helix_twofold", cfg, UNIT))
    *_, allstats = run_world(4, TOY4, "helix_twofold", with_stats=True)
    for rank, per_iter in enumerate(allstats):
        for st in per_iter:
            for peer, n in st["max_live_sends_per_peer"].items():
                assert 1 <= n <= len(plan.send_seq[(rank, peer)])


def test_regen_pre_x_two_and_four_ranks():
    """SURVEY H1 step 1 over the distributed driver: the pre stash drops x and
    rc.pre(l) rebuilds it from post(l-1)'s retention on the same rank."""
    for world, toy in ((2, TOY2), (4, TOY4)):
        losses, grads, peaks = run_world(world, toy, "helix_twofold_rc", env={"HX_TEST_REGEN_PRE_X": "1"})
        ref = _oracle(toy)
        assert np.allclose(losses, ref.losses, rtol=1e-10, atol=0)
        for l in range(toy["L"]):
            for k in O.FIELDS:
                assert np.allclose(grads[l][k], ref.param_grads[l][k], rtol=1e-9, atol=1e-12), (world, l, k)
        # the logical stash (reference keys) is unchanged
        _, _, base_peaks = run_world(world, toy, "helix_twofold_rc")
        assert peaks == base_peaks

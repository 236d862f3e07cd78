"""The one-rank-per-stage driver (executor._Distributed) with the real sm_100a
kernels: two processes share the one B200 of this environment (gloo carries
the CUDA payloads -- NCCL refuses two ranks on one device), each running its
helix stage on its own CUDA streams (compute, idle receive stream, input
streamer), exactly the code path torchrun uses on an 8-GPU box except the
collective library.  Results must match the float64 oracle within the parity
tolerances of test_parity_gpu.py, and the gradients must be owned by the right
stage."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, method, cfg_kw, mlp_chunk, q, extra=None):
    try:
        import torch.distributed as dist

        from paper_2507_00394_b200 import ModelConfig, generate
        from paper_2507_00394_b200.costs import DurationTable
        from paper_2507_00394_b200.runtime import execute_schedule, make_inputs, make_model
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), HX_SEND_CAP="0")
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = ModelConfig(**cfg_kw)
        sched = generate(method, cfg, DurationTable.from_units(1, 3, 2))
        res = execute_schedule(sched, make_model(cfg, 0), make_inputs(cfg, 1), mlp_chunk=mlp_chunk, threaded=True,
                               **(extra or {}))
        if rank == 0:
            q.put(("ok", res.losses, res.param_grads, res.mode))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put(("err", f"rank {rank}: {type(e).__name__}: {e}", None, None))


@pytest.mark.parametrize("method,chunk", [("helix_twofold", None), ("helix_twofold_rc", 100), ("1f1b", None)])
def test_two_ranks_on_one_gpu_match_oracle(method, chunk):
    from tests.test_parity_gpu import SMALL, compare, oracle_for
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    cfg_kw = dict(L=SMALL.L, h=SMALL.h, s=SMALL.s, b=SMALL.b, num_heads=SMALL.num_heads, p=2, m=4)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, method, cfg_kw, chunk, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert out[0] == "ok", out[1]
    _, losses, grads, mode = out
    assert mode == "threaded"

    class R:
        pass

    r = R()
    r.losses, r.param_grads = losses, grads
    compare(r, oracle_for(SMALL), SMALL.L, f"2 ranks on one GPU {method}")
    assert all(np.isfinite(losses))


@pytest.mark.parametrize("method,chunk,extra", [("helix_twofold_rc", 100, {"regen_pre_x": True}),
                                                 ("zb1p", None, {}), ("1f1b_rc", None, {})])
def test_four_ranks_on_one_gpu_match_oracle(method, chunk, extra):
    """p = 4: every stage pair exchanges payloads (two-fold pair edges across four
    stages), with x regenerated from post(l-1) on the rc schedule."""
    from paper_2507_00394_b200 import ModelConfig
    from tests.test_parity_gpu import compare, oracle_for
    cfg = ModelConfig(L=4, h=128, s=256, b=1, num_heads=2, p=4, m=8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    cfg_kw = dict(L=cfg.L, h=cfg.h, s=cfg.s, b=cfg.b, num_heads=cfg.num_heads, p=cfg.p, m=cfg.m)
    procs = [ctx.Process(target=_worker, args=(r, 4, port, method, cfg_kw, chunk, q, extra)) for r in range(4)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert out[0] == "ok", out[1]
    _, losses, grads, mode = out

    class R:
        pass

    r = R()
    r.losses, r.param_grads = losses, grads
    compare(r, oracle_for(cfg), cfg.L, f"4 ranks on one GPU {method}")


def _lm_worker(rank, world, port, method, chunk, regen, q):
    """LM mode (runtime/lm.py) under the one-rank-per-stage driver: the tied
    embedding and the loss-in-backward head live on stage 0 (helix places pre(0)
    and post(L-1) there), rank 1 only runs its layer components.  Every rank
    checks the gradients it owns against the fp32 autograd model of
    tests/test_lm_gpu.py."""
    try:
        import torch.distributed as dist

        from paper_2507_00394_b200 import ModelConfig, generate
        from paper_2507_00394_b200.costs import DurationTable
        from paper_2507_00394_b200.partition import post_stage, pre_stage
        from paper_2507_00394_b200.runtime import HelixRuntime
        from paper_2507_00394_b200.runtime.executor import DeviceModel, pair_groups
        from paper_2507_00394_b200.runtime.lm import LMParams, LMSpec, default_labels
        from paper_2507_00394_b200.runtime.model import (PARAM_FIELDS, POST_FIELDS, PRE_FIELDS, DeviceLayer,
                                                         random_device_layer)
        from tests.test_lm_gpu import _cos_max, _reference
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), HX_SEND_CAP="0")
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = ModelConfig(L=2, h=128, s=256, b=2, num_heads=2, p=world, m=2 * world)
        V = 1000
        sched = generate(method, cfg, DurationTable.from_units(1, 3, 2))
        gen = torch.Generator(device=dev).manual_seed(11)
        layers = [random_device_layer(cfg.h, gen, dev) for _ in range(cfg.L)]
        spec = LMSpec(V, head_chunk=192)
        params = LMParams(spec, cfg.h, cfg.s, dev, gen)
        model = DeviceModel({l: DeviceLayer(dict(w), PARAM_FIELDS) for l, w in enumerate(layers)})
        rt = HelixRuntime(sched, model, chunk, "distributed", dev, rank=rank, groups=pair_groups(world),
                          regen_pre_x=regen, lm=spec, lm_params=params)
        tg = torch.Generator(device=dev).manual_seed(12)
        tokens = [torch.randint(0, V, (cfg.s, cfg.b), generator=tg, device=dev) for _ in range(cfg.m)]
        rt.run(tokens)
        torch.cuda.synchronize()
        labels = [default_labels(t.reshape(-1).int(), cfg.s, cfg.b) for t in tokens]
        ref_l, ref_g, ref_e, ref_p = _reference(cfg, layers, params.w_emb[:V], params.w_pos,
                                                [t.reshape(-1) for t in tokens], labels)
        worst_cos, worst_max, owned = 1.0, 0.0, 0
        for l in range(cfg.L):
            fields = (PRE_FIELDS if pre_stage(l, cfg) == rank else ()) + \
                (POST_FIELDS if post_stage(l, cfg) == rank else ())
            for k in fields:
                c, m = _cos_max(model.layers[l].grad[k], ref_g[l][k])
                worst_cos, worst_max, owned = min(worst_cos, c), max(worst_max, m), owned + 1
        loss_err = None
        g = rt.lm_grads()
        if g is not None:
            for got, want in ((g["w_emb"][:V], ref_e), (g["w_pos"], ref_p)):
                c, m = _cos_max(got, want)
                worst_cos, worst_max = min(worst_cos, c), max(worst_max, m)
            loss_err = max(abs(a - b) / b for a, b in zip(rt.losses(), ref_l))
        q.put(("ok", rank, worst_cos, worst_max, owned, loss_err, g is not None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put(("err", rank, f"{type(e).__name__}: {e}\n{traceback.format_exc()[-1500:]}", None, None, None, None))


@pytest.mark.parametrize("method,chunk,regen", [("helix_twofold", None, False), ("helix_twofold_rc", 100, True)])
def test_two_ranks_on_one_gpu_lm_mode(method, chunk, regen):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lm_worker, args=(r, 2, port, method, chunk, regen, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for o in outs:
        assert o[0] == "ok", f"rank {o[1]}: {o[2]}"
    by_rank = {o[1]: o for o in outs}
    assert by_rank[0][6] and not by_rank[1][6], "the LM head must live on stage 0 only"
    assert by_rank[0][5] is not None and by_rank[0][5] <= 2e-3, by_rank[0][5]
    assert sum(o[4] for o in outs) == 2 * 8, "every layer field is owned by exactly one rank"
    for o in outs:
        print(f"[lm x2] {method} rank {o[1]}: cos {o[2]:.6f} max {o[3]:.2e}")
        assert o[2] >= 0.9995 and o[3] <= 2e-2, o


def test_bench_multirank_leg_on_one_gpu():
    """bench.py --gpus 4 end to end (self-launch through torch.distributed.run,
    max-over-ranks timing, bubble table, overlap report, 1F1B baseline, e2e) with
    the ranks time-sharing this one GPU over gloo (HX_BENCH_SHARED_GPU=1)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, HX_BENCH_SHARED_GPU="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "4", "--workload", "tiny", "--steps", "2",
                          "--warmup", "3", "--no-cpu-baseline"], cwd=root, env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 4 and d["config"]["p"] == 4 and d["config"]["m"] == 8
    assert d["data"].startswith("TEST")
    assert d["gpu_launches"] > 0 and d["value"] > 0
    table = d["bubble_predicted_by_reference_model"]["bubble_table"]
    assert set(table) >= {"analytic", "simulated_zero_comm", "simulated_nvlink", "measured"}
    assert d["comm"]["max_live_sends_per_peer"] and max(d["comm"]["max_live_sends_per_peer"].values()) <= \
        d["comm"]["send_cap"]

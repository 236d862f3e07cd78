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


def _worker(rank, world, port, method, cfg_kw, mlp_chunk, q):
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
        res = execute_schedule(sched, make_model(cfg, 0), make_inputs(cfg, 1), mlp_chunk=mlp_chunk, threaded=True)
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

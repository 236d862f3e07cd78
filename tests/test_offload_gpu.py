"""FILO host offload of stashed activations (runtime/offload.py) on the B200.

With a zero device budget every stashed activation is copied to pinned host
memory when it is stored and brought back (stream-ordered) before its backward
or recompute task; the result must still match the float64 oracle within the
parity tolerances of test_parity_gpu.py, every evicted byte must come back
exactly once per eviction, and no tracking state may leak.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from tests.test_parity_gpu import SMALL, WIDE, compare, oracle_for, run  # noqa: E402


@pytest.mark.parametrize("method", ["helix_twofold_rc", "helix_twofold", "1f1b", "zb1p"])
def test_zero_budget_offloads_everything_and_matches_oracle(method):
    res = run(SMALL, method, stash_budget_bytes=0, offload_min_bytes=0)
    st = res.offload
    assert st["evictions"] > 0 and st["d2h_bytes"] > 0
    assert st["h2d_bytes"] == st["d2h_bytes"]          # each tensor left and came back once
    assert st["live_entries"] == 0
    compare(res, oracle_for(SMALL), SMALL.L, f"offload {method}")


def test_partial_budget_head_dim_128():
    # half of one micro-batch's stash fits: a mix of resident and offloaded tensors
    budget = WIDE.L * 3 * WIDE.s * WIDE.b * WIDE.h * 2 // 2
    res = run(WIDE, "helix_twofold_rc", stash_budget_bytes=budget, offload_min_bytes=0)
    assert res.offload["evictions"] > 0
    assert res.offload["live_entries"] == 0
    compare(res, oracle_for(WIDE), WIDE.L, "offload partial wide")


def test_multistream_driver_with_offload():
    res = run(SMALL, "helix_twofold", threaded=True, stash_budget_bytes=0, offload_min_bytes=0)
    assert res.offload["evictions"] > 0
    compare(res, oracle_for(SMALL), SMALL.L, "offload multistream")


@pytest.mark.parametrize("qkv", [True, False])
def test_regen_pre_x_with_zero_budget(qkv):
    """regen_pre_x reads post(l-1)'s retention in rc.pre(l): the offloader
    prefetches it for that task too (consumed_keys), so with everything
    offloaded the results still match the oracle and nothing leaks."""
    from paper_2507_00394_b200 import generate
    from paper_2507_00394_b200.runtime import execute_schedule, make_inputs, make_model
    from tests.test_parity_gpu import UNIT
    sched = generate("helix_twofold_rc", SMALL, UNIT, qkv_in_attention=qkv)
    res = execute_schedule(sched, make_model(SMALL, 0), make_inputs(SMALL, 1), mlp_chunk=100,
                           regen_pre_x=True, stash_budget_bytes=0, offload_min_bytes=0)
    st = res.offload
    assert st["evictions"] > 0 and st["h2d_bytes"] == st["d2h_bytes"] and st["live_entries"] == 0
    compare(res, oracle_for(SMALL), SMALL.L, f"offload + regen_pre_x qkv={qkv}")

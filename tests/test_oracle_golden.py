"""The oracle (oracle/helix_oracle.py) is pinned against golden vectors made by
running the reference (tests/golden/make_golden.py): bit-for-bit, since the
restatement keeps the reference's einsum evaluation order."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import helix_oracle as O

GOLD = Path(__file__).parent / "golden"
META = json.loads((GOLD / "runtime_meta.json").read_text())


@pytest.mark.parametrize("case", ["toy", "ci"])
def test_oracle_bitwise_equals_reference(case):
    entry = META[case]
    kw = entry["config"]
    params = O.make_model(kw["L"], kw["h"], entry["param_seed"])
    inputs = O.make_inputs(kw["m"], kw["s"], kw["b"], kw["h"], entry["input_seed"])
    res = O.sequential_oracle(params, inputs, kw["num_heads"])
    gold = O.read_plt1(GOLD / f"numerics_{case}.plt")
    assert res.losses == list(gold["losses"])
    assert res.losses == entry["losses"]
    for l in range(kw["L"]):
        for k in O.FIELDS:
            assert np.array_equal(res.param_grads[l][k], gold[f"grad.l{l}.{k}"]), (l, k)


def test_reference_schedules_were_bitwise_on_reference():
    # sanity on the fixture itself: every method reproduced the oracle on the reference
    for entry in META.values():
        assert all(entry["bitwise_equal"].values())


def test_oracle_chunk_invariance():
    entry = META["toy"]
    kw = entry["config"]
    params = O.make_model(kw["L"], kw["h"], 5)
    inputs = O.make_inputs(kw["m"], kw["s"], kw["b"], kw["h"], 6)
    ref = O.sequential_oracle(params, inputs, kw["num_heads"])
    for chunk in (1, 3, 5):
        got = O.sequential_oracle(params, inputs, kw["num_heads"], chunk=chunk)
        assert got.losses == ref.losses


def test_tiny_config_known_loss_forward_only():
    # SURVEY §8c / BASELINE.md: tiny config (L4 h256 s1024 heads4), seeds 0/1, loss[0]
    params = O.make_model(4, 256, 0)
    x = O.make_inputs(1, 1024, 1, 256, 1)[0]
    for P in params:
        x, _ = O.layer_fwd(x, P, 4)
    assert O.loss_and_grad(x)[0] == 3.327261203817688


def test_plt1_round_trip(tmp_path):
    rng = np.random.default_rng(8)
    t = {"a": rng.standard_normal((3, 4)), "empty": np.zeros((0, 2)),
         "deep": rng.standard_normal((2, 3, 2, 2))}
    O.write_plt1(tmp_path / "t.plt", t)
    back = O.read_plt1(tmp_path / "t.plt")
    assert all(np.array_equal(back[k], t[k]) for k in t)
    (tmp_path / "bad.plt").write_bytes(b"NOPE" + (tmp_path / "t.plt").read_bytes()[4:])
    with pytest.raises(ValueError):
        O.read_plt1(tmp_path / "bad.plt")

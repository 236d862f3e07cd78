"""Parity at the benchmark's full per-layer size (GPT-1.3B: h=2048, 16 heads,
s=32768), where the float64 oracle cannot run (it materialises [b, n, s, s]).

* schedule invariance: every method (helix naive / two-fold / two-fold + rc,
  1F1B, ZB1P, and the 1F1B + recompute extension) computes the same losses
  and gradients from the same weights and inputs;
* an independent fp32 PyTorch model of the reference block (LayerNorm, QKV,
  causal softmax attention via SDPA, output projection, LayerNorm, erf-GeLU MLP,
  mean(z^2) loss; P/runtime/layers.py:94-137, model.py:61-64) on the same bf16
  weights and inputs, differentiated by autograd.
Tolerances (bf16 activations against fp32): loss rel <= 5e-3, gradient cosine
>= 0.999, max|diff| / max|ref| <= 5e-2.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2507_00394_b200 import ModelConfig, generate  # noqa: E402
from paper_2507_00394_b200.costs import DurationTable  # noqa: E402
from paper_2507_00394_b200.runtime import HelixRuntime  # noqa: E402
from paper_2507_00394_b200.runtime.executor import DeviceModel  # noqa: E402
from paper_2507_00394_b200.runtime.model import PARAM_FIELDS, DeviceLayer, random_device_layer  # noqa: E402

CFG = ModelConfig(L=2, h=2048, s=32768, b=1, num_heads=16, p=2, m=4)
UNIT = DurationTable.from_units(1, 3, 2)
DEV = torch.device("cuda", 0)
LOSS_TOL, COS_TOL, MAX_TOL = 5e-3, 0.999, 5e-2


@pytest.fixture(scope="module")
def weights_inputs():
    gen = torch.Generator(device=DEV).manual_seed(7)
    layers = [random_device_layer(CFG.h, gen, DEV) for _ in range(CFG.L)]
    ig = torch.Generator(device=DEV).manual_seed(8)
    inputs = [torch.randn(CFG.s * CFG.b, CFG.h, generator=ig, device=DEV).to(torch.bfloat16)
              for _ in range(CFG.m)]
    return layers, inputs


def run_method(method, layers, inputs):
    sched = generate(method, CFG, UNIT)
    model = DeviceModel({l: DeviceLayer(dict(w), PARAM_FIELDS) for l, w in enumerate(layers)})
    rt = HelixRuntime(sched, model, None, "replay", DEV)
    rt.run(inputs)
    torch.cuda.synchronize()
    grads = {l: {k: g.clone() for k, g in dl.grad.items()} for l, dl in model.layers.items()}
    return rt.losses(), grads


def compare(losses, grads, ref_losses, ref_grads, label):
    worst = {"loss": 0.0, "cos": 1.0, "max": 0.0}
    for a, b in zip(losses, ref_losses):
        worst["loss"] = max(worst["loss"], abs(a - b) / abs(b))
    for l in range(CFG.L):
        for k in PARAM_FIELDS:
            g, r = grads[l][k].double().flatten(), ref_grads[l][k].double().flatten()
            worst["cos"] = min(worst["cos"], float(g @ r / (g.norm() * r.norm())))
            worst["max"] = max(worst["max"], float((g - r).abs().max() / r.abs().max()))
    print(f"[full-size] {label}: worst loss rel {worst['loss']:.2e} cos {worst['cos']:.6f} max {worst['max']:.2e}")
    assert worst["loss"] <= LOSS_TOL, worst
    assert worst["cos"] >= COS_TOL, worst
    assert worst["max"] <= MAX_TOL, worst


def torch_reference(layers, inputs):
    """fp32 autograd model of the reference block, same weights (bf16 -> fp32)."""
    h, n, s, b = CFG.h, CFG.num_heads, CFG.s, CFG.b
    d = h // n
    params = [{k: v.detach().float().clone().requires_grad_(True) for k, v in w.items()} for w in layers]

    def ln(x, g, bb):
        mu = x.mean(-1, keepdim=True)
        var = ((x - mu) ** 2).mean(-1, keepdim=True)
        return (x - mu) / torch.sqrt(var + 1e-5) * g + bb

    losses = []
    for x0 in inputs:
        x = x0.float()
        for P in params:
            qkv = ln(x, P["ln1_gain"], P["ln1_bias"]) @ P["qkv_weight"]
            q, k, v = (t.view(s, b, n, d).permute(1, 2, 0, 3) for t in qkv.split(h, dim=-1))
            o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True,
                                                                 scale=1.0 / math.sqrt(d))
            o = o.permute(2, 0, 1, 3).reshape(s * b, h)
            x2 = x + o @ P["o_weight"]
            m1 = ln(x2, P["ln2_gain"], P["ln2_bias"]) @ P["mlp_w1"]
            x = x2 + torch.nn.functional.gelu(m1) @ P["mlp_w2"]
        loss = (x * x).mean()
        loss.backward()
        losses.append(float(loss))
        del x, loss
    return losses, {l: {k: P[k].grad for k in PARAM_FIELDS} for l, P in enumerate(params)}


def test_schedule_invariance_at_full_size(weights_inputs):
    layers, inputs = weights_inputs
    base_l, base_g = run_method("helix_twofold", layers, inputs)
    assert all(np.isfinite(base_l))
    for method in ("helix_naive", "helix_twofold_rc", "1f1b", "zb1p", "1f1b_rc"):
        l, g = run_method(method, layers, inputs)
        compare(l, g, base_l, base_g, f"{method} vs helix_twofold")


def test_full_size_against_torch_fp32(weights_inputs):
    layers, inputs = weights_inputs
    ref_l, ref_g = torch_reference(layers, inputs)
    l, g = run_method("helix_twofold", layers, inputs)
    compare(l, g, ref_l, ref_g, "helix_twofold vs torch fp32")


def test_stage_count_invariance_at_full_size():
    """The same model run as a 1-, 2- and 4-stage helix pipeline (all stages on
    this GPU, replay driver): the partition changes, the math does not."""
    cfg1 = ModelConfig(L=4, h=2048, s=32768, b=1, num_heads=16, p=1, m=8)
    gen = torch.Generator(device=DEV).manual_seed(11)
    layers = [random_device_layer(cfg1.h, gen, DEV) for _ in range(cfg1.L)]
    ig = torch.Generator(device=DEV).manual_seed(12)
    inputs = [torch.randn(cfg1.s, cfg1.h, generator=ig, device=DEV).to(torch.bfloat16) for _ in range(cfg1.m)]
    results = {}
    for p in (1, 2, 4):
        cfg = cfg1.with_(p=p)
        sched = generate("helix_twofold", cfg, UNIT)
        model = DeviceModel({l: DeviceLayer(dict(w), PARAM_FIELDS) for l, w in enumerate(layers)})
        rt = HelixRuntime(sched, model, None, "replay", DEV)
        rt.run(inputs)
        torch.cuda.synchronize()
        results[p] = (rt.losses(), {l: {k: g.clone() for k, g in dl.grad.items()} for l, dl in model.layers.items()})
        del rt, model
        torch.cuda.empty_cache()
    base_l, base_g = results[1]
    for p in (2, 4):
        l, g = results[p]
        worst_cos, worst_max = 1.0, 0.0
        for a, b in zip(l, base_l):
            assert abs(a - b) / abs(b) <= LOSS_TOL
        for li in range(cfg1.L):
            for k in PARAM_FIELDS:
                x, y = g[li][k].double().flatten(), base_g[li][k].double().flatten()
                worst_cos = min(worst_cos, float(x @ y / (x.norm() * y.norm())))
                worst_max = max(worst_max, float((x - y).abs().max() / y.abs().max()))
        print(f"[full-size] helix_twofold p={p} vs p=1: cos {worst_cos:.6f} max {worst_max:.2e}")
        assert worst_cos >= COS_TOL and worst_max <= MAX_TOL

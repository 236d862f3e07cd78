"""Parity at the shapes the 3B/64k and 7B/128k performance numbers use
(BASELINE configs 3 and 4: h=4096, 32 heads, head_dim 128, s=65536 / 131072,
recomputation-without-attention, chunked MLP, host offload), where the float64
oracle cannot run.

* against an independent fp32 PyTorch autograd model of the reference block
  (``P/runtime/layers.py:122-247``, ``mathops.py:44-157``; causal attention by
  SDPA's memory-efficient kernel, or per-head checkpointed math if that
  backend is unavailable) on the same bf16 weights and inputs;
* schedule invariance on the same weights: helix two-fold + rc == 1F1B + rc
  == helix two-fold + rc with the stash FILO-offloaded to host memory.

This exercises what only the large shapes reach: attention backward with
one-head CTA bands and an L2-resident fp32 dQ at s=128k, split-K weight
gradients over K=131072 rows, chunked-MLP row slabs of 8192 / 16384, and the
offload path under a budget smaller than one layer's stash.
Tolerances (bf16 activations vs fp32): loss rel <= 5e-3, gradient cosine
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

UNIT = DurationTable.from_units(1, 3, 2)
DEV = torch.device("cuda", 0)
LOSS_TOL, COS_TOL, MAX_TOL = 5e-3, 0.999, 5e-2

CFG_3B = ModelConfig(L=2, h=4096, s=65536, b=1, num_heads=32, p=2, m=4)
CFG_7B = ModelConfig(L=1, h=4096, s=131072, b=1, num_heads=32, p=1, m=2)


def make_weights(cfg, seed):
    gen = torch.Generator(device=DEV).manual_seed(seed)
    layers = [random_device_layer(cfg.h, gen, DEV) for _ in range(cfg.L)]
    ig = torch.Generator(device=DEV).manual_seed(seed + 1)
    inputs = [torch.randn(cfg.s * cfg.b, cfg.h, generator=ig, device=DEV).to(torch.bfloat16)
              for _ in range(cfg.m)]
    return layers, inputs


def run_method(cfg, method, layers, inputs, mlp_chunk, stash_budget_bytes=None):
    sched = generate(method, cfg, UNIT)
    model = DeviceModel({l: DeviceLayer(dict(w), PARAM_FIELDS) for l, w in enumerate(layers)})
    rt = HelixRuntime(sched, model, mlp_chunk, "replay", DEV, stash_budget_bytes=stash_budget_bytes,
                      offload_min_bytes=0 if stash_budget_bytes is not None else 32 << 20)
    rt.run(inputs)
    torch.cuda.synchronize()
    grads = {l: {k: g.clone() for k, g in dl.grad.items()} for l, dl in model.layers.items()}
    stats = rt.offload_stats()
    out = rt.losses(), grads, stats
    del rt, model
    torch.cuda.empty_cache()
    return out


def compare(cfg, losses, grads, ref_losses, ref_grads, label):
    worst = {"loss": 0.0, "cos": 1.0, "max": 0.0}
    for a, b in zip(losses, ref_losses):
        worst["loss"] = max(worst["loss"], abs(a - b) / abs(b))
    for l in range(cfg.L):
        for k in PARAM_FIELDS:
            g, r = grads[l][k].double().flatten(), ref_grads[l][k].double().flatten()
            worst["cos"] = min(worst["cos"], float(g @ r / (g.norm() * r.norm())))
            worst["max"] = max(worst["max"], float((g - r).abs().max() / r.abs().max()))
    print(f"[large] {label}: worst loss rel {worst['loss']:.2e} cos {worst['cos']:.6f} max {worst['max']:.2e}")
    assert worst["loss"] <= LOSS_TOL, (label, worst)
    assert worst["cos"] >= COS_TOL, (label, worst)
    assert worst["max"] <= MAX_TOL, (label, worst)


class _HeadAttention(torch.autograd.Function):
    """Causal attention of one head in fp32 with the probabilities recomputed
    in backward (the [s, s] matrix of every head would not fit), computed in
    query blocks; ``mathops.py:83-116`` restated."""

    @staticmethod
    def _probs(q, k, a, e, scale):
        sc = (q[a:e] @ k[:e].T) * scale
        idx = torch.arange(a, e, device=q.device)[:, None] < torch.arange(e, device=q.device)[None, :]
        sc.masked_fill_(idx, float("-inf"))
        return torch.softmax(sc, -1)

    @staticmethod
    def forward(ctx, q, k, v, block):
        scale = 1.0 / math.sqrt(q.shape[-1])
        out = torch.empty_like(q)
        for a in range(0, q.shape[0], block):
            e = min(a + block, q.shape[0])
            out[a:e] = _HeadAttention._probs(q, k, a, e, scale) @ v[:e]
        ctx.save_for_backward(q, k, v)
        ctx.block = block
        return out

    @staticmethod
    def backward(ctx, do):
        q, k, v = ctx.saved_tensors
        scale = 1.0 / math.sqrt(q.shape[-1])
        dq, dk, dv = torch.zeros_like(q), torch.zeros_like(k), torch.zeros_like(v)
        for a in range(0, q.shape[0], ctx.block):
            e = min(a + ctx.block, q.shape[0])
            p = _HeadAttention._probs(q, k, a, e, scale)
            dv[:e] += p.T @ do[a:e]
            dp = do[a:e] @ v[:e].T
            ds = p * (dp - (dp * p).sum(-1, keepdim=True))
            dq[a:e] = ds @ k[:e] * scale
            dk[:e] += ds.T @ q[a:e] * scale
        return dq, dk, dv, None


def causal_attention_fp32(q, k, v):
    """q, k, v: [b, n, s, d] fp32."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    try:
        with sdpa_kernel([SDPBackend.EFFICIENT_ATTENTION]):
            return torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True,
                                                                    scale=1.0 / math.sqrt(q.shape[-1]))
    except RuntimeError:
        b, n, s, d = q.shape
        heads = [_HeadAttention.apply(q[i, j], k[i, j], v[i, j], 8192) for i in range(b) for j in range(n)]
        return torch.stack(heads).view(b, n, s, d)


def torch_reference(cfg, layers, inputs):
    """fp32 autograd model of the reference block on the same (bf16) weights."""
    h, n, s, b = cfg.h, cfg.num_heads, cfg.s, cfg.b
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
            q, k, v = (t.reshape(s, b, n, d).permute(1, 2, 0, 3).contiguous() for t in qkv.split(h, dim=-1))
            del qkv
            o = causal_attention_fp32(q, k, v)
            del q, k, v
            o = o.permute(2, 0, 1, 3).reshape(s * b, h)
            x2 = x + o @ P["o_weight"]
            m1 = ln(x2, P["ln2_gain"], P["ln2_bias"]) @ P["mlp_w1"]
            x = x2 + torch.nn.functional.gelu(m1) @ P["mlp_w2"]
            del m1, x2, o
        loss = (x * x).mean()
        loss.backward()
        losses.append(float(loss))
        del x, loss
    grads = {l: {k: P[k].grad for k in PARAM_FIELDS} for l, P in enumerate(params)}
    torch.cuda.empty_cache()
    return losses, grads


@pytest.fixture(scope="module")
def gpt3b():
    layers, inputs = make_weights(CFG_3B, 21)
    base = run_method(CFG_3B, "helix_twofold_rc", layers, inputs, 8192)
    return layers, inputs, base


def test_3b_64k_rc_chunked_mlp_against_torch_fp32(gpt3b):
    layers, inputs, (l, g, _) = gpt3b
    ref_l, ref_g = torch_reference(CFG_3B, layers, inputs)
    compare(CFG_3B, l, g, ref_l, ref_g, "3B/64k helix_twofold_rc mlp_chunk=8192 vs torch fp32")


def test_3b_64k_schedule_invariance(gpt3b):
    """helix_rc == 1f1b_rc == helix_rc + offload on the same weights."""
    layers, inputs, (bl, bg, _) = gpt3b
    l, g, _ = run_method(CFG_3B, "1f1b_rc", layers, inputs, 8192)
    compare(CFG_3B, l, g, bl, bg, "3B/64k 1f1b_rc vs helix_twofold_rc")
    # budget below one layer-micro-batch's rc retention (4 bsh): every stage offloads
    budget = CFG_3B.s * CFG_3B.h * 2 * 3
    l, g, st = run_method(CFG_3B, "helix_twofold_rc", layers, inputs, 8192, stash_budget_bytes=budget)
    assert st["evictions"] > 0 and st["h2d_bytes"] == st["d2h_bytes"] and st["live_entries"] == 0, st
    compare(CFG_3B, l, g, bl, bg, "3B/64k helix_twofold_rc + offload vs resident")


def test_7b_128k_layer_rc_offload_against_torch_fp32():
    layers, inputs = make_weights(CFG_7B, 31)
    budget = CFG_7B.s * CFG_7B.h * 2 * 3          # < one micro-batch's retention: forces offload
    l, g, st = run_method(CFG_7B, "helix_twofold_rc", layers, inputs, 16384, stash_budget_bytes=budget)
    assert st["evictions"] > 0 and st["live_entries"] == 0, st
    assert all(np.isfinite(l))
    ref_l, ref_g = torch_reference(CFG_7B, layers, inputs)
    compare(CFG_7B, l, g, ref_l, ref_g, "7B/128k layer helix_twofold_rc mlp_chunk=16384 + offload vs torch fp32")
    rl, rg, _ = run_method(CFG_7B, "1f1b_rc", layers, inputs, 16384)
    compare(CFG_7B, rl, rg, l, g, "7B/128k layer 1f1b_rc vs helix_twofold_rc + offload")

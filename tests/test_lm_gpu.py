"""Paper §4.6 extras on the B200 (runtime/lm.py): word + position embeddings
and the tied next-token head with the loss computed in the backward.

The reference has no code for this path, so there is no oracle:
the check is an fp32 PyTorch autograd model of the same network on the same
(bf16-rounded) weights and tokens.  Tolerances as the other bf16 parity tests:
loss rel <= 2e-3, gradient cosine >= 0.9995, max|diff| / max|ref| <= 2e-2.
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
from paper_2507_00394_b200.runtime import kernels as K  # noqa: E402
from paper_2507_00394_b200.runtime import _lib  # noqa: E402
from paper_2507_00394_b200.runtime.executor import DeviceModel  # noqa: E402
from paper_2507_00394_b200.runtime.lm import LMParams, LMSpec, default_labels  # noqa: E402
from paper_2507_00394_b200.runtime.model import PARAM_FIELDS, DeviceLayer, random_device_layer  # noqa: E402

DEV = torch.device("cuda", 0)
UNIT = DurationTable.from_units(1, 3, 2)
LOSS_TOL, COS_TOL, MAX_TOL = 2e-3, 0.9995, 2e-2


def test_ce_loss_kernel_against_torch():
    rows, V, Vp = 300, 1000, 1024
    g = torch.Generator(device=DEV).manual_seed(3)
    logits = (torch.randn(rows, Vp, generator=g, device=DEV) * 3).to(torch.bfloat16)
    labels = torch.randint(0, V, (rows,), generator=g, device=DEV, dtype=torch.int32)
    labels[::7] = -1
    ref = logits.float()[:, :V]
    valid = labels >= 0
    want_loss = torch.nn.functional.cross_entropy(ref[valid], labels[valid].long(), reduction="sum")
    sm = torch.softmax(ref, -1)
    sm[valid, labels[valid].long()] -= 1
    sm[~valid] = 0
    scale = 1.0 / int(valid.sum())
    acc = torch.zeros(1, dtype=torch.float64, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int32, device=DEV)
    _lib.call("hx_ce_loss", logits.data_ptr(), Vp, labels.data_ptr(), rows, V, Vp, scale, acc.data_ptr(),
              cnt.data_ptr(), K._stream())
    torch.cuda.synchronize()
    assert int(cnt) == int(valid.sum())
    assert abs(float(acc) - float(want_loss)) / float(want_loss) < 1e-4
    got = logits.float()
    assert got[:, V:].abs().max() == 0
    assert ((got[:, :V] - sm * scale).abs().max() / (sm * scale).abs().max()) < 1e-2


def test_embedding_kernels_against_torch():
    s, b, h, V = 200, 3, 256, 500
    g = torch.Generator(device=DEV).manual_seed(4)
    params = LMParams(LMSpec(V), h, s, DEV, g)
    from paper_2507_00394_b200.runtime.lm import LMHead
    head = LMHead(LMSpec(V), params, s, b, h)
    tok = torch.randint(0, V, (s * b,), generator=g, device=DEV, dtype=torch.int32)
    x = torch.empty(s * b, h, dtype=torch.bfloat16, device=DEV)
    head.embed(tok, x)
    pos = torch.arange(s * b, device=DEV) // b
    want = params.w_emb.float()[tok.long()] + params.w_pos.float()[pos]
    dx = torch.randn(s * b, h, generator=g, device=DEV).to(torch.bfloat16)
    head.embed_backward(tok, dx)
    torch.cuda.synchronize()
    assert (x.float() - want).abs().max() <= 1e-2 * want.abs().max()
    d_emb = torch.zeros(params.w_emb.shape, device=DEV).index_add_(0, tok.long(), dx.float())
    d_pos = dx.float().view(s, b, h).sum(1)
    assert torch.allclose(params.d_emb, d_emb, rtol=1e-5, atol=1e-5)
    assert torch.allclose(params.d_pos, d_pos, rtol=1e-5, atol=1e-5)


def _reference(cfg, layers, w_emb, w_pos, tokens, labels):
    """fp32 autograd: embeddings, the reference block (P/runtime/layers.py), tied CE head."""
    h, n, s, b = cfg.h, cfg.num_heads, cfg.s, cfg.b
    d = h // n
    P = [{k: v.detach().float().clone().requires_grad_(True) for k, v in w.items()} for w in layers]
    E = w_emb.detach().float().clone().requires_grad_(True)
    Q = w_pos.detach().float().clone().requires_grad_(True)

    def ln(x, g, bb):
        mu = x.mean(-1, keepdim=True)
        var = ((x - mu) ** 2).mean(-1, keepdim=True)
        return (x - mu) / torch.sqrt(var + 1e-5) * g + bb

    losses = []
    pos = torch.arange(s * b, device=DEV) // b
    mask = torch.triu(torch.ones(s, s, dtype=torch.bool, device=DEV), 1)
    for tok, lab in zip(tokens, labels):
        x = E[tok.long()] + Q[pos]
        for W in P:
            qkv = ln(x, W["ln1_gain"], W["ln1_bias"]) @ W["qkv_weight"]
            q, k, v = (t.reshape(s, b, n, d).permute(1, 2, 0, 3) for t in qkv.split(h, -1))
            sc = (q @ k.transpose(-1, -2)) / math.sqrt(d)
            o = torch.softmax(sc.masked_fill(mask, float("-inf")), -1) @ v
            o = o.permute(2, 0, 1, 3).reshape(s * b, h)
            x2 = x + o @ W["o_weight"]
            x = x2 + torch.nn.functional.gelu(ln(x2, W["ln2_gain"], W["ln2_bias"]) @ W["mlp_w1"]) @ W["mlp_w2"]
        valid = lab >= 0
        loss = torch.nn.functional.cross_entropy((x @ E.T)[valid], lab[valid].long())
        loss.backward()
        losses.append(float(loss.detach()))
    return losses, [{k: W[k].grad for k in PARAM_FIELDS} for W in P], E.grad, Q.grad


def _cos_max(g, r):
    g, r = g.double().flatten(), r.double().flatten()
    return float(g @ r / (g.norm() * r.norm())), float((g - r).abs().max() / r.abs().max())


@pytest.mark.parametrize("method,chunk,regen", [("helix_twofold", None, False),
                                                ("helix_twofold_rc", 100, True), ("1f1b", None, False)])
def test_lm_runtime_against_torch_fp32(method, chunk, regen):
    cfg = ModelConfig(L=2, h=128, s=256, b=2, num_heads=2, p=2 if method != "1f1b" else 1, m=4)
    V = 1000
    sched = generate(method, cfg, UNIT)
    gen = torch.Generator(device=DEV).manual_seed(11)
    layers = [random_device_layer(cfg.h, gen, DEV) for _ in range(cfg.L)]
    spec = LMSpec(V, head_chunk=192)
    params = LMParams(spec, cfg.h, cfg.s, DEV, gen)
    model = DeviceModel({l: DeviceLayer(dict(w), PARAM_FIELDS) for l, w in enumerate(layers)})
    rt = HelixRuntime(sched, model, chunk, "replay", DEV, regen_pre_x=regen, lm=spec, lm_params=params)
    tg = torch.Generator(device=DEV).manual_seed(12)
    tokens = [torch.randint(0, V, (cfg.s, cfg.b), generator=tg, device=DEV) for _ in range(cfg.m)]
    rt.run(tokens)
    torch.cuda.synchronize()
    labels = [default_labels(t.reshape(-1).int(), cfg.s, cfg.b) for t in tokens]
    ref_l, ref_g, ref_e, ref_p = _reference(cfg, layers, params.w_emb[:V], params.w_pos,
                                            [t.reshape(-1) for t in tokens], labels)
    for got, want in zip(rt.losses(), ref_l):
        assert abs(got - want) / want <= LOSS_TOL, (got, want)
    worst_cos, worst_max = 1.0, 0.0
    for l in range(cfg.L):
        for k in PARAM_FIELDS:
            c, m = _cos_max(model.layers[l].grad[k], ref_g[l][k])
            worst_cos, worst_max = min(worst_cos, c), max(worst_max, m)
    g = rt.lm_grads()
    for got, want in ((g["w_emb"][:V], ref_e), (g["w_pos"], ref_p)):
        c, m = _cos_max(got, want)
        worst_cos, worst_max = min(worst_cos, c), max(worst_max, m)
    print(f"[lm] {method} chunk={chunk} regen={regen}: cos {worst_cos:.6f} max {worst_max:.2e}")
    assert worst_cos >= COS_TOL and worst_max <= MAX_TOL, (worst_cos, worst_max)
    assert np.all(np.isfinite(rt.losses()))

"""Test double for :class:`paper_2507_00394_b200.runtime.layers.LayerMath`:
the same component interface and payload / stash keys, computed in float64
torch on the CPU.  TEST INFRASTRUCTURE ONLY — it lets the multi-process
executor drivers (the exact code that moves payloads over NCCL on the GPU
box) run here over gloo and be checked against the float64 oracle.  The
product path never imports this file.
"""

from __future__ import annotations

import math

import torch

F64 = torch.float64


def _ln(x, g, b):
    mu = x.mean(-1, keepdim=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdim=True)
    return xc / torch.sqrt(var + 1e-5) * g + b


def _ln_bwd(dy, x, g):
    mu = x.mean(-1, keepdim=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdim=True)
    inv = 1.0 / torch.sqrt(var + 1e-5)
    xh = xc * inv
    dxh = dy * g
    dx = inv * (dxh - dxh.mean(-1, keepdim=True) - xh * (dxh * xh).mean(-1, keepdim=True))
    return dx, (dy * xh).sum(0), dy.sum(0)


def _gelu(x):
    return 0.5 * x * (1.0 + torch.erf(x / math.sqrt(2.0)))


def _gelu_grad(x):
    return 0.5 * (1.0 + torch.erf(x / math.sqrt(2.0))) + x * torch.exp(-0.5 * x * x) / math.sqrt(2 * math.pi)


class CpuMath:
    act_dtype = F64
    wgrad_dtype = F64

    def __init__(self, cfg, qkv_in_attention: bool, mlp_chunk=None):
        self.cfg, self.qkv, self.chunk = cfg, qkv_in_attention, mlp_chunk

    def zero_(self, t):
        return t.zero_()

    # attention on token-major [s*b, 3h]
    def _split(self, t):
        s, b, n = self.cfg.s, self.cfg.b, self.cfg.num_heads
        return t.view(s, b, n, -1).permute(1, 2, 0, 3)  # [b, n, s, d]

    def _merge(self, t):
        return t.permute(2, 0, 1, 3).reshape(self.cfg.s * self.cfg.b, -1)

    def _probs(self, q, k):
        s = q.shape[2]
        sc = q @ k.transpose(-1, -2) / math.sqrt(q.shape[-1])
        sc = sc.masked_fill(torch.triu(torch.ones(s, s, dtype=torch.bool), 1), float("-inf"))
        return torch.softmax(sc, -1)

    def _attn(self, qkv):
        h = self.cfg.h
        q, k, v = (self._split(qkv[:, i * h:(i + 1) * h]) for i in range(3))
        return self._merge(self._probs(q, k) @ v)

    def _attn_bwd(self, qkv, do):
        h = self.cfg.h
        q, k, v = (self._split(qkv[:, i * h:(i + 1) * h]) for i in range(3))
        d4 = self._split(do)
        p = self._probs(q, k)
        scale = 1.0 / math.sqrt(q.shape[-1])
        dv = p.transpose(-1, -2) @ d4
        dp = d4 @ v.transpose(-1, -2)
        ds = p * (dp - (dp * p).sum(-1, keepdim=True))
        dq = ds @ k * scale
        dk = ds.transpose(-1, -2) @ q * scale
        return torch.cat([self._merge(dq), self._merge(dk), self._merge(dv)], -1)

    def pre_forward(self, x, W):
        ln = _ln(x, W["ln1_gain"], W["ln1_bias"])
        if self.qkv:
            return {"ln_out": ln, "residual": x, "qkv_weight": W["qkv_weight"]}, {"x": x}
        return {"qkv": ln @ W["qkv_weight"], "residual": x}, {"x": x, "ln_out": ln}

    def attn_forward(self, payload):
        if self.qkv:
            qkv = payload["ln_out"] @ payload["qkv_weight"]
            stash = {"ln_out": payload["ln_out"], "qkv": qkv, "qkv_weight": payload["qkv_weight"]}
        else:
            qkv = payload["qkv"]
            stash = {"qkv": qkv}
        return {"attn_out": self._attn(qkv), "residual": payload["residual"]}, stash

    def _post_trunk(self, attn_out, residual, W):
        x2 = residual + attn_out @ W["o_weight"]
        ln2 = _ln(x2, W["ln2_gain"], W["ln2_bias"])
        m1 = ln2 @ W["mlp_w1"]
        return {"attn_out": attn_out, "x2": x2, "ln2_out": ln2, "m1": m1, "g": _gelu(m1)}

    def post_forward(self, payload, W):
        t = self._post_trunk(payload["attn_out"], payload["residual"], W)
        return t["x2"] + t["g"] @ W["mlp_w2"], t

    def loss(self, z, slot):
        slot += (z * z).sum()
        return z * (2.0 / z.numel())

    def post_backward_b(self, d_out, W, G, st, fuse_w=False):
        d_m1 = (d_out @ W["mlp_w2"].t()) * _gelu_grad(st["m1"])
        d_ln2 = d_m1 @ W["mlp_w1"].t()
        dx, dg, db = _ln_bwd(d_ln2, st["x2"], W["ln2_gain"])
        G["ln2_gain"] += dg
        G["ln2_bias"] += db
        d_x2 = d_out + dx
        wctx = {"attn_out": st["attn_out"], "d_o": d_x2, "ln2_out": st["ln2_out"], "d_m1": d_m1,
                "g": st["g"], "d_out": d_out}
        return {"d_attn_out": d_x2 @ W["o_weight"].t(), "d_residual": d_x2}, wctx

    def post_backward_w(self, w, G):
        G["o_weight"] += w["attn_out"].t() @ w["d_o"]
        G["mlp_w1"] += w["ln2_out"].t() @ w["d_m1"]
        G["mlp_w2"] += w["g"].t() @ w["d_out"]

    def post_backward(self, d_out, W, G, st):
        gap, w = self.post_backward_b(d_out, W, G, st)
        self.post_backward_w(w, G)
        return gap

    def attn_backward(self, payload, st):
        qkv = st.get("qkv")
        if qkv is None:
            qkv = st["ln_out"] @ st["qkv_weight"]
        d_qkv = self._attn_bwd(qkv, payload["d_attn_out"])
        if not self.qkv:
            return {"d_qkv": d_qkv, "d_residual": payload["d_residual"]}
        return {"d_ln_out": d_qkv @ st["qkv_weight"].t(), "d_residual": payload["d_residual"],
                "d_qkv_weight": st["ln_out"].t() @ d_qkv}

    def pre_backward_b(self, payload, W, G, st):
        if self.qkv:
            d_ln, w = payload["d_ln_out"], {"d_qkv_weight": payload["d_qkv_weight"]}
        else:
            d_ln = payload["d_qkv"] @ W["qkv_weight"].t()
            w = {"ln_out": st["ln_out"], "d_qkv": payload["d_qkv"]}
        dx, dg, db = _ln_bwd(d_ln, st["x"], W["ln1_gain"])
        G["ln1_gain"] += dg
        G["ln1_bias"] += db
        return dx + payload["d_residual"], w

    def pre_backward_w(self, w, G):
        G["qkv_weight"] += w["d_qkv_weight"] if "d_qkv_weight" in w else w["ln_out"].t() @ w["d_qkv"]

    def pre_backward(self, payload, W, G, st):
        d_x, w = self.pre_backward_b(payload, W, G, st)
        self.pre_backward_w(w, G)
        return d_x

    def reduce_stash(self, comp, stash, payload):
        if comp == "pre":
            return {"x": stash["x"]}
        if comp == "attn":
            return {"ln_out": stash["ln_out"], "qkv_weight": stash["qkv_weight"]} if self.qkv \
                else {"qkv": stash["qkv"]}
        return {"attn_out": payload["attn_out"], "residual": payload["residual"]}

    def regenerate_stash(self, comp, kept, W):
        if comp == "pre":
            if self.qkv:
                return {"x": kept["x"]}
            return {"x": kept["x"], "ln_out": _ln(kept["x"], W["ln1_gain"], W["ln1_bias"])}
        if "_x2" in kept:
            x2, ln2 = kept["_x2"], kept["_ln2_out"]
            m1 = ln2 @ W["mlp_w1"]
            return {"attn_out": kept["attn_out"], "x2": x2, "ln2_out": ln2, "m1": m1, "g": _gelu(m1)}
        return self._post_trunk(kept["attn_out"], kept["residual"], W)

    def post_output(self, kept, W):
        t = self._post_trunk(kept["attn_out"], kept["residual"], W)
        return t["x2"] + t["g"] @ W["mlp_w2"], {"_x2": t["x2"], "_ln2_out": t["ln2_out"]}

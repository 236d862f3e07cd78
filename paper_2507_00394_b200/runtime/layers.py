"""Transformer-layer components on the B200: pre / attention / post, forward and
fused backward, recompute-stash management.

Mirrors ``P/runtime/layers.py`` component by component (same payload and stash
dictionary keys, so the executor's payload-size contract with
``costs.comm_volume`` holds unchanged), but every op is a libhx kernel:

  pre   fwd  LN1                                   hx_ln_fwd
  attn  fwd  QKV GEMM, flash attention             hx_gemm, hx_attn_fwd
  post  fwd  O GEMM + residual, LN2, W1 GEMM + GeLU, W2 GEMM + residual
  post  bwd  W2^T GEMM * GeLU', W1^T GEMM, LN2 bwd + residual, Wo^T GEMM,
             three weight-gradient GEMMs accumulating into fp32
  attn  bwd  (recompute QKV), flash backward, Wqkv^T GEMM, dWqkv GEMM
  pre   bwd  LN1 bwd + residual, dWqkv accumulate

Layout: activations are bf16 ``[s*b, width]`` (token-major).  Besides the
reference's stash entries the attention stash keeps the row LSE of the
softmax (flash backward needs it instead of the full probability matrix).
The flash backward's other extra input, D = rowsum(dO * O) per head, is
computed by the post stage's backward, where O (``attn_out``) is stashed
anyway, and travels in the ``gap`` payload as ``delta`` (b*heads*s fp32, 1/d of
the payload's bytes; not part of the reference's payload, so not counted
against ``comm_volume``).  The attention stage therefore never stashes O
(SURVEY H10).

Chunked MLP (``mathops.py:122-157``): with recomputation the
forward keeps no ``m1``/``g`` at all, and the backward regenerates them one
row slab at a time next to that slab's ``d_m1``, accumulating the two MLP
weight gradients per slab, so the MLP's transient memory is ``3 * c * 4h``
instead of ``12 * s*b * h``.  The stash still *counts* the reference's
``m1``/``g`` (placeholders), so ``peak_stash_elements`` matches the reference.
"""

from __future__ import annotations

import torch

from . import kernels as K

BF16 = torch.bfloat16
Arrays = dict[str, torch.Tensor]


# Payload entries that are B200 additions, not the reference's payload keys
# (excluded from the comm_volume contract check).
LOCAL_PAYLOAD_KEYS = ("delta",)


def payload_elements(payload: Arrays) -> int:
    return sum(int(t.numel()) for k, t in payload.items() if k not in LOCAL_PAYLOAD_KEYS)


class Pending:
    """Stash placeholder for a tensor the reference keeps but this runtime
    regenerates per MLP row slab inside the backward (``m1``, ``g``): it only
    carries the element count for ``peak_stash_elements``."""

    __slots__ = ("n",)

    def __init__(self, n: int):
        self.n = n

    def numel(self) -> int:
        return self.n


class LayerMath:
    """Component kernels for one model shape (bf16 activations, fp32 grads)."""

    act_dtype = torch.bfloat16     # activations / payload tensors / qkv_weight copies
    wgrad_dtype = torch.float32    # shipped weight gradients (d_qkv_weight)

    ships_delta = True             # gap payload carries D = rowsum(dO * O)

    def __init__(self, cfg, qkv_in_attention: bool, mlp_chunk: int | None, device,
                 recompute: bool = False, defer_w: bool = False):
        self.cfg = cfg
        self.qkv = qkv_in_attention
        self.chunk = mlp_chunk
        self.device = device
        self.T = cfg.s * cfg.b
        self.h = cfg.h
        self.heads = cfg.num_heads
        # set by the executor from the schedule: recomputation-without-attention
        # (m1/g never kept) and a split backward (W half deferred to BWD_W)
        self.recompute = recompute
        self.defer_w = defer_w

    def zero_(self, t: torch.Tensor) -> torch.Tensor:
        return K.zero_(t)

    # -- helpers ------------------------------------------------------------------

    def _empty(self, width: int, dtype=BF16) -> torch.Tensor:
        return torch.empty(self.T, width, dtype=dtype, device=self.device)

    def _row_slabs(self):
        """Row ranges of the chunked MLP (``mathops.py:132-142``): chunks of c
        sequence positions = c*b token rows; None means one slab."""
        s, b = self.cfg.s, self.cfg.b
        c = s if self.chunk is None else min(self.chunk, s)
        return [(a * b, min(a + c, s) * b) for a in range(0, s, c)]

    # -- forward ----------------------------------------------------------------------

    def pre_forward(self, x: torch.Tensor, W) -> tuple[Arrays, Arrays]:
        ln_out = K.layernorm(x, W["ln1_gain"], W["ln1_bias"], self._empty(self.h))
        if self.qkv:
            return {"ln_out": ln_out, "residual": x, "qkv_weight": W["qkv_weight"]}, {"x": x}
        qkv = K.linear(ln_out, W["qkv_weight"], self._empty(3 * self.h))
        return {"qkv": qkv, "residual": x}, {"x": x, "ln_out": ln_out}

    def _attention(self, qkv: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        o = self._empty(self.h)
        lse = torch.empty(self.cfg.b, self.heads, self.cfg.s, dtype=torch.float32, device=self.device)
        K.attention_fwd(qkv, self.cfg.s, self.cfg.b, self.heads, o, lse)
        return o, lse

    def attn_forward(self, payload: Arrays) -> tuple[Arrays, Arrays]:
        if self.qkv:
            qkv = K.linear(payload["ln_out"], payload["qkv_weight"], self._empty(3 * self.h))
            stash = {"ln_out": payload["ln_out"], "qkv": qkv, "qkv_weight": payload["qkv_weight"]}
        else:
            qkv = payload["qkv"]
            stash = {"qkv": qkv}
        o, lse = self._attention(qkv)
        stash["lse"] = lse
        return {"attn_out": o, "residual": payload["residual"]}, stash

    def _slab_rows(self) -> int:
        a, e = self._row_slabs()[0]
        return e - a

    def _post_trunk(self, attn_out, residual, W, mlp: bool = True, x2=None, ln2=None) -> Arrays:
        """x2, LN2 and (``mlp``) the whole-tensor MLP activations m1, g;
        without ``mlp`` they are placeholders, regenerated per slab later.
        ``x2``/``ln2`` given: already regenerated (``post_output``), reused."""
        if x2 is None:
            x2 = K.linear_resid(attn_out, W["o_weight"], residual, self._empty(self.h))
            ln2 = K.layernorm(x2, W["ln2_gain"], W["ln2_bias"], self._empty(self.h))
        t = {"attn_out": attn_out, "x2": x2, "ln2_out": ln2}
        if not mlp:
            t["m1"], t["g"] = Pending(self.T * 4 * self.h), Pending(self.T * 4 * self.h)
            return t
        m1 = self._empty(4 * self.h)
        g = self._empty(4 * self.h)
        for a, e in self._row_slabs():
            K.linear_gelu(ln2[a:e], W["mlp_w1"], m1[a:e], g[a:e])
        t["m1"], t["g"] = m1, g
        return t

    def post_forward(self, payload: Arrays, W) -> tuple[torch.Tensor, Arrays]:
        # with recomputation only {attn_out, residual} is kept (layers.py:229-230):
        # m1 / g live one row slab at a time
        keep_mlp = not self.recompute
        t = self._post_trunk(payload["attn_out"], payload["residual"], W, mlp=keep_mlp)
        out = self._empty(self.h)
        if keep_mlp:
            for a, e in self._row_slabs():
                K.linear_resid(t["g"][a:e], W["mlp_w2"], t["x2"][a:e], out[a:e])
            return out, t
        self._mlp_slabs_forward(t, W, out)
        return out, t

    def _mlp_slabs_forward(self, t: Arrays, W, out: torch.Tensor) -> None:
        """out = x2 + GeLU(ln2 W1) W2 with m1 / g one row slab at a time."""
        c = self._slab_rows()
        m1, g = self._empty_rows(c, 4 * self.h), self._empty_rows(c, 4 * self.h)
        for a, e in self._row_slabs():
            n = e - a
            K.linear_gelu(t["ln2_out"][a:e], W["mlp_w1"], m1[:n], g[:n])
            K.linear_resid(g[:n], W["mlp_w2"], t["x2"][a:e], out[a:e])

    def post_output(self, kept: Arrays, W) -> tuple[torch.Tensor, Arrays]:
        """Rebuild ``post(l)``'s output -- the next layer's input x -- from its
        recompute retention {attn_out, residual} (the pre
        stash's x is not kept).  Returns x and the regenerated x2 / LN2 output
        under cache keys ``_x2`` / ``_ln2_out``, which ``regenerate_stash``
        reuses instead of recomputing them for ``rc.post(l)``."""
        t = self._post_trunk(kept["attn_out"], kept["residual"], W, mlp=False)
        out = self._empty(self.h)
        self._mlp_slabs_forward(t, W, out)
        return out, {"_x2": t["x2"], "_ln2_out": t["ln2_out"]}

    def _empty_rows(self, rows: int, width: int, dtype=BF16) -> torch.Tensor:
        return torch.empty(rows, width, dtype=dtype, device=self.device)

    # -- loss ---------------------------------------------------------------------------

    def loss(self, z: torch.Tensor, sumsq_slot: torch.Tensor) -> torch.Tensor:
        dz = torch.empty_like(z)
        K.mse_loss(z, dz, sumsq_slot)
        return dz

    # -- backward (fused B + W) ------------------------------------------------------------

    def _mlp_backward(self, d_out, W, stash: Arrays, G=None) -> tuple[torch.Tensor, Arrays]:
        """MLP backward over row slabs (``mathops.py:145-162``) -> d_ln2.

        m1 / g come from the stash, or (placeholders) are regenerated per slab.
        With ``G`` the two MLP weight gradients accumulate per slab and only
        slab-sized workspaces exist; without it (W half deferred) d_m1 and g are
        materialised whole and returned for the W half."""
        regen = not isinstance(stash["m1"], torch.Tensor)
        whole = G is None
        d_ln2 = self._empty(self.h)
        c = self._slab_rows()
        wctx: Arrays = {}
        if whole:
            d_m1 = self._empty(4 * self.h)
            g_all = self._empty(4 * self.h) if regen else stash["g"]
            wctx = {"d_m1": d_m1, "g": g_all}
        else:
            d_m1_w = self._empty_rows(c, 4 * self.h)
        if regen:
            m1_w = self._empty_rows(c, 4 * self.h)
            g_w = None if whole else self._empty_rows(c, 4 * self.h)
        for a, e in self._row_slabs():
            n = e - a
            if regen:
                m1 = m1_w[:n]
                g = g_all[a:e] if whole else g_w[:n]
                K.linear_gelu(stash["ln2_out"][a:e], W["mlp_w1"], m1, g)
            else:
                m1, g = stash["m1"][a:e], stash["g"][a:e]
            dm = d_m1[a:e] if whole else d_m1_w[:n]
            K.linear_dx_dgelu(d_out[a:e], W["mlp_w2"], m1, dm)
            K.linear_dx(dm, W["mlp_w1"], d_ln2[a:e])
            if not whole:
                K.linear_dw(g, d_out[a:e], G["mlp_w2"])
                K.linear_dw(stash["ln2_out"][a:e], dm, G["mlp_w1"])
        return d_ln2, wctx

    def post_backward_b(self, d_out: torch.Tensor, W, G, stash: Arrays,
                        fuse_w: bool = False) -> tuple[Arrays, Arrays]:
        """Input-gradient half (``layers.py:143-154``).  The LN2 gain/bias
        gradients are row reductions the LN-backward kernel produces anyway, so
        they accumulate here.  The three weight GEMMs go to the W half, except
        with ``fuse_w`` (fused backward), where the MLP ones run per row slab
        inside the MLP backward.  Also computes the flash backward's
        D = rowsum(d_attn_out * attn_out) for the ``gap`` payload."""
        d_ln2, wctx = self._mlp_backward(d_out, W, stash, G if fuse_w else None)
        d_x2 = self._empty(self.h)
        K.layernorm_bwd(d_ln2, stash["x2"], W["ln2_gain"], d_out, d_x2,
                        G["ln2_gain"], G["ln2_bias"])
        d_attn = K.linear_dx(d_x2, W["o_weight"], self._empty(self.h))
        delta = torch.empty(self.cfg.b * self.heads * self.cfg.s, dtype=torch.float32, device=self.device)
        K.attention_delta(stash["attn_out"], d_attn, self.cfg.s, self.cfg.b, self.heads, delta)
        wctx.update({"attn_out": stash["attn_out"], "d_o": d_x2})
        if not fuse_w:
            wctx.update({"ln2_out": stash["ln2_out"], "d_out": d_out})
        return {"d_attn_out": d_attn, "d_residual": d_x2, "delta": delta}, wctx

    def post_backward_w(self, wctx: Arrays, G) -> None:
        """Weight-gradient half (``layers.py:157-162``): fp32 accumulate over all
        rows (the MLP ones only if ``post_backward_b`` did not run them per slab)."""
        K.linear_dw(wctx["attn_out"], wctx["d_o"], G["o_weight"])
        if "d_m1" in wctx:
            K.linear_dw(wctx["ln2_out"], wctx["d_m1"], G["mlp_w1"])
            K.linear_dw(wctx["g"], wctx["d_out"], G["mlp_w2"])

    def post_backward(self, d_out: torch.Tensor, W, G, stash: Arrays) -> Arrays:
        """Fused backward of the post component (B then W immediately)."""
        gap, wctx = self.post_backward_b(d_out, W, G, stash, fuse_w=True)
        self.post_backward_w(wctx, G)
        return gap

    def attn_backward(self, payload: Arrays, stash: Arrays) -> Arrays:
        """``layers.attn_backward`` (``layers.py:165-184``)."""
        qkv = stash.get("qkv")
        if qkv is None:  # recompute retention: rebuild the projection, never the attention
            qkv = K.linear(stash["ln_out"], stash["qkv_weight"], self._empty(3 * self.h))
        d_qkv = self._empty(3 * self.h)
        # workspace from the stream-ordered caching allocator (stages on different
        # streams never share it)
        K.attention_bwd(qkv, None, payload["d_attn_out"], stash["lse"], self.cfg.s,
                        self.cfg.b, self.heads, d_qkv, payload["delta"])
        if not self.qkv:
            return {"d_qkv": d_qkv, "d_residual": payload["d_residual"]}
        d_ln = K.linear_dx(d_qkv, stash["qkv_weight"], self._empty(self.h))
        d_w = torch.empty(self.h, 3 * self.h, dtype=torch.float32, device=self.device)
        K.linear_dw(stash["ln_out"], d_qkv, d_w, accumulate=False)
        return {"d_ln_out": d_ln, "d_residual": payload["d_residual"], "d_qkv_weight": d_w}

    def pre_backward_b(self, payload: Arrays, W, G, stash: Arrays) -> tuple[torch.Tensor, Arrays]:
        """Input-gradient half (``layers.py:187-198``) + LN1 gain/bias grads."""
        if self.qkv:
            d_ln = payload["d_ln_out"]
            wctx = {"d_qkv_weight": payload["d_qkv_weight"]}
        else:
            d_ln = K.linear_dx(payload["d_qkv"], W["qkv_weight"], self._empty(self.h))
            wctx = {"ln_out": stash["ln_out"], "d_qkv": payload["d_qkv"]}
        d_x = self._empty(self.h)
        K.layernorm_bwd(d_ln, stash["x"], W["ln1_gain"], payload["d_residual"], d_x,
                        G["ln1_gain"], G["ln1_bias"])
        return d_x, wctx

    def pre_backward_w(self, wctx: Arrays, G) -> None:
        """Weight-gradient half (``layers.py:201-207``)."""
        if "d_qkv_weight" in wctx:
            K.axpy(G["qkv_weight"], wctx["d_qkv_weight"])
        else:
            K.linear_dw(wctx["ln_out"], wctx["d_qkv"], G["qkv_weight"])

    def pre_backward(self, payload: Arrays, W, G, stash: Arrays) -> torch.Tensor:
        d_x, wctx = self.pre_backward_b(payload, W, G, stash)
        self.pre_backward_w(wctx, G)
        return d_x

    # -- recompute (layers.py:213-247) -------------------------------------------------------

    def reduce_stash(self, comp: str, stash: Arrays, payload: Arrays) -> Arrays:
        if comp == "pre":
            return {"x": stash["x"]}
        if comp == "attn":
            keep = {"ln_out": stash["ln_out"], "qkv_weight": stash["qkv_weight"]} if self.qkv \
                else {"qkv": stash["qkv"]}
            keep["lse"] = stash["lse"]
            return keep
        if comp == "post":
            return {"attn_out": payload["attn_out"], "residual": payload["residual"]}
        raise ValueError(f"no recompute retention for component {comp!r}")

    def regenerate_stash(self, comp: str, kept: Arrays, W) -> Arrays:
        if comp == "pre":
            if self.qkv:
                return {"x": kept["x"]}
            return {"x": kept["x"],
                    "ln_out": K.layernorm(kept["x"], W["ln1_gain"], W["ln1_bias"], self._empty(self.h))}
        if comp == "post":
            # m1 / g are regenerated per row slab inside the backward unless the
            # W half is deferred (ZB1P), which needs them whole
            return self._post_trunk(kept["attn_out"], kept["residual"], W, mlp=self.defer_w,
                                    x2=kept.get("_x2"), ln2=kept.get("_ln2_out"))
        raise ValueError(f"component {comp!r} is never recomputed")

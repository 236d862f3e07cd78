"""Word / position embeddings and the tied next-token head with the loss in
backward -- the paper's §4.6 extras.

The reference package has no code for these (SPEC.md:467 puts "embeddings,
vocabulary projection, and loss-in-backward (§4.6)" out of its scope; its loss
is the mean square of the last layer's output, ``P/runtime/model.py:61-64``).
This module is therefore a B200 extension behind the same runtime: with an
``LMSpec`` the micro-batch inputs are token ids and

* ``f.pre.l0`` embeds them (``hx_embed_fwd``: x = W_emb[tok] + W_pos[pos]);
* the loss task (``b.post.l{L-1}``, or the last 1F1B chunk's backward) runs
  the head *in the backward*, one row slab at a time: logits = z W_emb^T
  (tcgen05 GEMM), cross-entropy and dlogits in place (``hx_ce_loss``),
  dz += dlogits W_emb, dW_emb += dlogits^T z -- the [s, b, V] logits are never
  stashed, only the layer output z waits for its backward, as the paper
  prescribes;
* ``b.pre.l0`` scatters d_x into the embedding gradients (``hx_embed_bwd``).

The word embedding is tied to the head, so its two uses must be on one stage:
helix places pre(0) and post(L-1) on stage 0 (``P/partition.py:25-36``); a
layer-wise 1F1B has them on the first and last stage, which this module does
not support for p > 1.  The vocabulary is padded to a multiple of 128
columns (zero rows of W_emb, masked out of the softmax), as Megatron-LM does.
Labels default to the next token of the same sequence; the last position of
each sequence is ignored.  Parity: ``tests/test_lm_gpu.py`` against an fp32
PyTorch autograd model (there is no reference oracle for this path).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from . import kernels as K

BF16 = torch.bfloat16


@dataclass(frozen=True)
class LMSpec:
    vocab: int
    head_chunk: int = 4096     # logits rows per slab in the backward head

    @property
    def vpad(self) -> int:
        return (self.vocab + 127) // 128 * 128


class LMParams:
    """Embedding weights (bf16) and fp32 gradients on the stage that owns them."""

    def __init__(self, spec: LMSpec, h: int, s: int, device, gen: torch.Generator | None = None,
                 w_emb: torch.Tensor | None = None, w_pos: torch.Tensor | None = None):
        self.spec = spec
        if w_emb is None:
            w_emb = torch.randn(spec.vocab, h, generator=gen, device=device) * 0.02
        if w_pos is None:
            w_pos = torch.randn(s, h, generator=gen, device=device) * 0.01
        pad = torch.zeros(spec.vpad, h, dtype=BF16, device=device)
        pad[:spec.vocab] = w_emb.to(device=device, dtype=BF16)
        self.w_emb = pad
        self.w_pos = w_pos.to(device=device, dtype=BF16).contiguous()
        self.d_emb = torch.zeros(spec.vpad, h, dtype=torch.float32, device=device)
        self.d_pos = torch.zeros_like(self.w_pos, dtype=torch.float32)

    def zero_grads(self, zero_fn) -> None:
        zero_fn(self.d_emb)
        zero_fn(self.d_pos)


def default_labels(tokens: torch.Tensor, s: int, b: int) -> torch.Tensor:
    """Next token of the same sequence; -1 (ignored) at the last position."""
    t = tokens.reshape(s, b)
    lab = torch.full_like(t, -1)
    lab[:-1] = t[1:]
    return lab.reshape(-1)


class LMHead:
    """The three LM-path operations on one stage."""

    def __init__(self, spec: LMSpec, params: LMParams, s: int, b: int, h: int):
        self.spec, self.p, self.s, self.b, self.h = spec, params, s, b, h

    def embed(self, tokens: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        _lib.call("hx_embed_fwd", tokens.data_ptr(), self.p.w_emb.data_ptr(), self.p.w_pos.data_ptr(),
                  out.data_ptr(), self.s, self.b, self.h, K._stream())
        return out

    def embed_backward(self, tokens: torch.Tensor, dx: torch.Tensor) -> None:
        _lib.call("hx_embed_bwd", tokens.data_ptr(), dx.data_ptr(), self.p.d_emb.data_ptr(),
                  self.p.d_pos.data_ptr(), self.s, self.b, self.h, K._stream())

    def loss_backward(self, z: torch.Tensor, labels: torch.Tensor, n_valid: int,
                      loss_acc: torch.Tensor, count_acc: torch.Tensor) -> torch.Tensor:
        """Head forward + cross-entropy + head backward over row slabs;
        returns dz.  loss_acc (f64) / count_acc (i32) accumulate the summed
        token loss and the token count."""
        T, V, Vp = z.shape[0], self.spec.vocab, self.spec.vpad
        c = min(self.spec.head_chunk, T)
        logits = torch.empty(c, Vp, dtype=BF16, device=z.device)
        dz = torch.empty_like(z)
        scale = 1.0 / max(1, n_valid)
        for a in range(0, T, c):
            e = min(a + c, T)
            lg = logits[:e - a]
            K.linear_dx(z[a:e], self.p.w_emb, lg)                 # z W_emb^T
            _lib.call("hx_ce_loss", lg.data_ptr(), Vp, labels[a:e].data_ptr(), e - a, V, Vp, scale,
                      loss_acc.data_ptr(), count_acc.data_ptr(), K._stream())
            K.linear(lg, self.p.w_emb, dz[a:e])                    # dlogits W_emb
            K.linear_dw(lg, z[a:e], self.p.d_emb)                  # dW_emb += dlogits^T z
        return dz

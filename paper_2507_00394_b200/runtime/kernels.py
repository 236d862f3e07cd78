"""Tensor-level wrappers over libhx (torch tensors in, stream-ordered launches).

torch is used only as device memory + stream plumbing: every arithmetic op on
the stage-execution path below is one of this library's sm_100a kernels.
Shapes use the reference's token-major layout: an ``[s, b, w]`` activation is
a row-major ``[s*b, w]`` matrix (``P/runtime/mathops.py:22``).
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import (EPI_ACC_F32, EPI_DGELU, EPI_GELU, EPI_RESID_BF16, EPI_STORE_BF16,
                   EPI_STORE_F32)

BF16 = torch.bfloat16
F32 = torch.float32


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype, name: str) -> None:
    if not t.is_cuda:
        raise _lib.KernelLibraryError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if t.dim() == 2 and t.stride(1) != 1:
        raise ValueError(f"{name}: last dim must be contiguous")


def _rows(t: torch.Tensor) -> torch.Tensor:
    return t.reshape(-1, t.shape[-1]) if t.dim() != 2 else t


# --- GEMM family (mathops.linear / linear_backward_x / linear_backward_w) ---------


def gemm(a: torch.Tensor, a_mn: bool, b: torch.Tensor, b_mn: bool, out: torch.Tensor,
         M: int, N: int, K: int, epi: int, aux: torch.Tensor | None = None,
         out2: torch.Tensor | None = None) -> torch.Tensor:
    _lib.call("hx_gemm", a.data_ptr(), a.stride(0), int(a_mn), b.data_ptr(), b.stride(0), int(b_mn),
              out.data_ptr(), out.stride(0), M, N, K, epi, _ptr(aux),
              aux.stride(0) if aux is not None else 0, _ptr(out2),
              out2.stride(0) if out2 is not None else 0, _stream(),
              tag=f"{'T' if a_mn else 'N'}{'T' if b_mn else 'N'} {M}x{N}x{K} epi{epi}")
    return out


def linear(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[T, o] = x[T, i] @ w[i, o]  (``mathops.py:21-23``)."""
    x = _rows(x)
    _need(x, BF16, "x"); _need(w, BF16, "w")
    T, K = x.shape
    N = w.shape[1]
    out = torch.empty(T, N, dtype=BF16, device=x.device) if out is None else out
    return gemm(x, False, w, True, out, T, N, K, EPI_STORE_BF16)


def linear_resid(x, w, resid, out=None):
    """out = resid + x @ w (O projection + residual, ``layers.py:124-125``)."""
    x = _rows(x)
    T, K = x.shape
    N = w.shape[1]
    out = torch.empty(T, N, dtype=BF16, device=x.device) if out is None else out
    return gemm(x, False, w, True, out, T, N, K, EPI_RESID_BF16, aux=_rows(resid))


def linear_gelu(x, w, m1_out, g_out):
    """m1 = x @ w1, g = gelu_erf(m1) (``mathops.py:139-140``)."""
    x = _rows(x)
    T, K = x.shape
    N = w.shape[1]
    gemm(x, False, w, True, m1_out, T, N, K, EPI_GELU, out2=g_out)
    return m1_out, g_out


def linear_dx(dy, w, out=None):
    """out[T, i] = dy[T, o] @ w[i, o]^T  (``mathops.py:26-27``)."""
    dy = _rows(dy)
    T, K = dy.shape
    N = w.shape[0]
    out = torch.empty(T, N, dtype=BF16, device=dy.device) if out is None else out
    return gemm(dy, False, w, False, out, T, N, K, EPI_STORE_BF16)


def linear_dx_dgelu(dy, w, m1, out):
    """d_m1 = (dy @ w2^T) * gelu'(m1)  (``mathops.py:155``)."""
    dy = _rows(dy)
    T, K = dy.shape
    N = w.shape[0]
    return gemm(dy, False, w, False, out, T, N, K, EPI_DGELU, aux=_rows(m1))


def linear_dw(x, dy, acc: torch.Tensor, accumulate: bool = True):
    """acc[i, o] (+)= x[T, i]^T @ dy[T, o] over all rows (``mathops.py:30-32``)."""
    x, dy = _rows(x), _rows(dy)
    _need(acc, F32, "acc")
    T, M = x.shape
    N = dy.shape[1]
    return gemm(x, True, dy, True, acc, M, N, T, EPI_ACC_F32 if accumulate else EPI_STORE_F32)


# --- LayerNorm (mathops.py:44-72) ----------------------------------------------------


def layernorm(x, gain, bias, out=None):
    x = _rows(x)
    _need(x, BF16, "x"); _need(gain, F32, "gain"); _need(bias, F32, "bias")
    out = torch.empty_like(x) if out is None else out
    _lib.call("hx_ln_fwd", x.data_ptr(), gain.data_ptr(), bias.data_ptr(), out.data_ptr(),
              x.shape[0], x.shape[1], _stream())
    return out


def layernorm_bwd(dy, x, gain, dres, dx, dgain_acc, dbias_acc):
    dy, x = _rows(dy), _rows(x)
    stats = torch.empty(2 * x.shape[0], dtype=F32, device=x.device)
    _lib.call("hx_ln_bwd", dy.data_ptr(), x.data_ptr(), gain.data_ptr(),
              _ptr(None if dres is None else _rows(dres)), dx.data_ptr(), dgain_acc.data_ptr(),
              dbias_acc.data_ptr(), stats.data_ptr(), x.shape[0], x.shape[1], _stream())
    return dx


# --- attention (mathops.py:83-116) ---------------------------------------------------


def attention_fwd(qkv, s: int, b: int, heads: int, o: torch.Tensor, lse: torch.Tensor):
    qkv = _rows(qkv)
    h = qkv.shape[1] // 3
    _lib.call("hx_attn_fwd", qkv.data_ptr(), qkv.stride(0), o.data_ptr(), _rows(o).stride(0),
              lse.data_ptr(), s, b, heads, h // heads, _stream())
    return o, lse


def attention_delta(o, d_o, s: int, b: int, heads: int, delta: torch.Tensor):
    """delta [b, heads, s] f32 = rowsum(d_o * o) per head (flash backward's D)."""
    o, d_o = _rows(o), _rows(d_o)
    if o.stride(0) != d_o.stride(0):
        raise ValueError("o and d_o must share a row stride")
    _need(delta, torch.float32, "delta")
    _lib.call("hx_attn_bwd_delta", o.data_ptr(), d_o.data_ptr(), o.stride(0), delta.data_ptr(),
              s, b, heads, o.shape[1] // heads, _stream())
    return delta


def attention_bwd_ws_bytes(s: int, b: int, heads: int, d: int) -> int:
    """Bytes of the backward's workspace (fp32 dQ accumulator + per-tile counters)."""
    return int(_lib.load().hx_attn_bwd_ws_bytes(s, b, heads, d))


def attention_bwd_ws(s: int, b: int, heads: int, d: int, device) -> torch.Tensor:
    n = attention_bwd_ws_bytes(s, b, heads, d)
    return torch.empty((n + 3) // 4, dtype=F32, device=device)


def attention_bwd(qkv, o, d_o, lse, s: int, b: int, heads: int, dqkv: torch.Tensor,
                  delta_ws: torch.Tensor, dq_ws: torch.Tensor | None = None):
    """``o=None``: ``delta_ws`` already holds D (``attention_delta``).
    ``dq_ws``: at least ``attention_bwd_ws_bytes`` (allocated here if None)."""
    qkv = _rows(qkv)
    h = qkv.shape[1] // 3
    need = attention_bwd_ws_bytes(s, b, heads, h // heads)
    if dq_ws is None:
        dq_ws = attention_bwd_ws(s, b, heads, h // heads, qkv.device)
    elif dq_ws.numel() * dq_ws.element_size() < need:
        raise ValueError(f"dq_ws holds {dq_ws.numel() * dq_ws.element_size()} bytes, need {need}")
    ld_o = _rows(d_o).stride(0) if o is None else _rows(o).stride(0)
    _lib.call("hx_attn_bwd", qkv.data_ptr(), qkv.stride(0), None if o is None else o.data_ptr(),
              d_o.data_ptr(), ld_o, lse.data_ptr(), delta_ws.data_ptr(), dq_ws.data_ptr(),
              dqkv.data_ptr(), _rows(dqkv).stride(0), s, b, heads, h // heads, _stream())
    return dqkv


# --- misc ------------------------------------------------------------------------------


def mse_loss(z, dz, sumsq_slot):
    """sumsq_slot (f64, 1 elt) += sum(z^2); dz = 2 z / numel (``model.py:61-64``)."""
    _lib.call("hx_mse_loss", z.data_ptr(), z.numel(), dz.data_ptr(), sumsq_slot.data_ptr(), _stream())
    return dz


def axpy(y: torch.Tensor, x: torch.Tensor):
    _lib.call("hx_axpy_f32", y.data_ptr(), x.data_ptr(), y.numel(), _stream())
    return y


def zero_(t: torch.Tensor):
    _lib.call("hx_zero", t.data_ptr(), t.numel() * t.element_size(), _stream())
    return t

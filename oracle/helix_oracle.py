"""CPU oracle for the HelixPipe stage-execution path — TEST INFRASTRUCTURE ONLY.

This module is a float64 NumPy restatement of the reference's numeric model
(``pipelab.runtime``; paths below are under ``/root/reference/pkg/src/pipelab``).
It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and the CPU
baseline leg of ``bench.py`` may import it.  The product path (the package
``paper_2507_00394_b200``) never imports or executes anything under
``oracle/`` and fails loudly when its CUDA library is missing.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by importing the reference itself
(``tests/golden/make_golden.py``); the restatement uses the same
``np.einsum`` contractions in the same evaluation order, so it reproduces the
reference bit-for-bit (losses and every gradient), not just to tolerance.

The arithmetic of the reference lives in two third-party libraries that are
not vendored under /root/reference: NumPy's non-optimising ``einsum``
(c_einsum; reference pins ``numpy>=1.24``, measured 2.3.5) and
``scipy.special.erf`` (``scipy>=1.10``, measured 1.18.1); ``pkg/pyproject.toml:10-17``.

Model (runtime/layers.py:1-8, runtime/mathops.py):
    pre   : ln_out = LN1(x)                                    layers.py:94-105
    attn  : qkv = ln_out @ Wqkv ; o = causal_softmax(qk^T/sqrt d) v   layers.py:108-119
    post  : x2 = x + o @ Wo ; out = x2 + gelu(LN2(x2) @ W1) @ W2      layers.py:122-137
    loss  : mean(z^2), dz = 2 z / numel                        model.py:61-64
Grads are summed over micro-batches in ascending order (model.py:72-76, 105-122).
"""

from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np
from scipy.special import erf

EPS = 1e-5                               # mathops.py:15
_R2 = np.sqrt(2.0)
_INV_SQRT_2PI = 1.0 / np.sqrt(2.0 * np.pi)

FIELDS = ("ln1_gain", "ln1_bias", "qkv_weight", "o_weight",
          "ln2_gain", "ln2_bias", "mlp_w1", "mlp_w2")   # layers.py:62-69


@dataclass
class Params:
    """One layer's weights, ``[in, out]`` layout (layers.py:54-78)."""

    ln1_gain: np.ndarray
    ln1_bias: np.ndarray
    qkv_weight: np.ndarray
    o_weight: np.ndarray
    ln2_gain: np.ndarray
    ln2_bias: np.ndarray
    mlp_w1: np.ndarray
    mlp_w2: np.ndarray

    def field_names(self) -> tuple[str, ...]:
        return tuple(f.name for f in fields(self))


# --- fixtures (model.py:31-58) ------------------------------------------------


def make_layer_params(rng: np.random.Generator, h: int) -> Params:
    """Draw order is the contract: gain, bias, Wqkv, Wo, gain, bias, W1, W2."""
    draws = {}
    for name in FIELDS:
        if name.endswith("_gain"):
            draws[name] = 1.0 + 0.1 * rng.standard_normal(h)
        elif name.endswith("_bias"):
            draws[name] = 0.1 * rng.standard_normal(h)
        else:
            n_in, n_out = {"qkv_weight": (h, 3 * h), "o_weight": (h, h),
                           "mlp_w1": (h, 4 * h), "mlp_w2": (4 * h, h)}[name]
            draws[name] = rng.standard_normal((n_in, n_out)) / np.sqrt(n_in)
    return Params(**draws)


def make_model(L: int, h: int, seed: int) -> list[Params]:
    rng = np.random.default_rng(seed)
    return [make_layer_params(rng, h) for _ in range(L)]


def make_inputs(m: int, s: int, b: int, h: int, seed: int) -> list[np.ndarray]:
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((s, b, h)) for _ in range(m)]


# --- primitives (mathops.py) --------------------------------------------------


def mm(x, w):                       # mathops.py:21-23
    return np.einsum("sbi,io->sbo", x, w)


def mm_dx(dy, w):                   # mathops.py:26-27
    return np.einsum("sbo,io->sbi", dy, w)


def mm_dw(x, dy):                   # mathops.py:30-32 (all rows at once)
    return np.einsum("sbi,sbo->io", x, dy)


def gelu(x):                        # mathops.py:35-37
    return 0.5 * x * (1.0 + erf(x / _R2))


def gelu_grad(x):                   # mathops.py:40-41
    return 0.5 * (1.0 + erf(x / _R2)) + x * np.exp(-0.5 * x * x) * _INV_SQRT_2PI


def _ln_stats(x):
    mu = np.mean(x, axis=-1, keepdims=True)
    xc = x - mu
    var = np.mean(xc * xc, axis=-1, keepdims=True)
    return xc, var


def layernorm(x, g, b):             # mathops.py:44-49
    xc, var = _ln_stats(x)
    return xc / np.sqrt(var + EPS) * g + b


def layernorm_bwd(dy, x, g):        # mathops.py:52-72 -> (dx, dgain, dbias)
    xc, var = _ln_stats(x)
    inv = 1.0 / np.sqrt(var + EPS)
    xhat = xc * inv
    dxh = dy * g
    dx = inv * (dxh - np.mean(dxh, axis=-1, keepdims=True)
                - xhat * np.mean(dxh * xhat, axis=-1, keepdims=True))
    return dx, np.einsum("sbh,sbh->h", dy, xhat), np.einsum("sbh->h", dy)


def _heads(t, n):
    s, b, h = t.shape
    return t.reshape(s, b, n, h // n)


def causal_probs(q4, k4):           # mathops.py:83-92
    s = q4.shape[0]
    sc = np.einsum("sbnd,tbnd->bnst", q4, k4) * (1.0 / np.sqrt(q4.shape[-1]))
    sc = sc + np.triu(np.full((s, s), -np.inf), k=1)
    e = np.exp(sc - np.max(sc, axis=-1, keepdims=True))
    return e / np.sum(e, axis=-1, keepdims=True)


def attention(q, k, v, n):          # mathops.py:95-100
    p = causal_probs(_heads(q, n), _heads(k, n))
    return np.einsum("bnst,tbnd->sbnd", p, _heads(v, n)).reshape(q.shape)


def attention_lse(q, k, n):
    """Natural-log row log-sum-exp of the scaled, masked scores: [b, n, s].
    Not in the reference (its backward recomputes P whole); used to check the
    flash kernels' LSE output."""
    q4, k4 = _heads(q, n), _heads(k, n)
    s = q4.shape[0]
    sc = np.einsum("sbnd,tbnd->bnst", q4, k4) * (1.0 / np.sqrt(q4.shape[-1]))
    sc = sc + np.triu(np.full((s, s), -np.inf), k=1)
    mx = np.max(sc, axis=-1, keepdims=True)
    return (mx + np.log(np.sum(np.exp(sc - mx), axis=-1, keepdims=True)))[..., 0]


def attention_bwd(q, k, v, do, n):  # mathops.py:103-116
    q4, k4, v4, d4 = (_heads(t, n) for t in (q, k, v, do))
    p = causal_probs(q4, k4)
    scale = 1.0 / np.sqrt(q4.shape[-1])
    dv = np.einsum("bnst,sbnd->tbnd", p, d4)
    dp = np.einsum("sbnd,tbnd->bnst", d4, v4)
    ds = p * (dp - np.sum(dp * p, axis=-1, keepdims=True))
    dq = np.einsum("bnst,tbnd->sbnd", ds, k4) * scale
    dk = np.einsum("bnst,sbnd->tbnd", ds, q4) * scale
    return dq.reshape(q.shape), dk.reshape(q.shape), dv.reshape(q.shape)


def _row_slabs(s, chunk):
    c = s if chunk is None else min(chunk, s)
    return [slice(a, min(a + c, s)) for a in range(0, s, c)]


def mlp_fwd(x, w1, w2, chunk=None):     # mathops.py:122-142 -> (out, m1, g)
    m1 = np.empty(x.shape[:2] + (w1.shape[1],))
    g = np.empty_like(m1)
    out = np.empty(x.shape[:2] + (w2.shape[1],))
    for sl in _row_slabs(x.shape[0], chunk):
        m1[sl] = mm(x[sl], w1)
        g[sl] = gelu(m1[sl])
        out[sl] = mm(g[sl], w2)
    return out, m1, g


def mlp_bwd(d_out, w1, w2, m1, chunk=None):   # mathops.py:145-157 -> (dx, d_m1)
    d_m1 = np.empty_like(m1)
    dx = np.empty(d_out.shape[:2] + (w1.shape[0],))
    for sl in _row_slabs(d_out.shape[0], chunk):
        d_m1[sl] = mm_dx(d_out[sl], w2) * gelu_grad(m1[sl])
        dx[sl] = mm_dx(d_m1[sl], w1)
    return dx, d_m1


def loss_and_grad(z):                # model.py:61-64
    return float(np.mean(z * z)), z * (2.0 / z.size)


# --- one layer, forward and fused backward ---------------------------------------


def layer_fwd(x, P: Params, n_heads: int, chunk=None):
    """Returns (out, cache) with every intermediate the components produce."""
    ln1 = layernorm(x, P.ln1_gain, P.ln1_bias)                       # layers.py:97
    qkv = mm(ln1, P.qkv_weight)                                      # layers.py:102/111
    h = qkv.shape[-1] // 3
    o = attention(qkv[..., :h], qkv[..., h:2 * h], qkv[..., 2 * h:], n_heads)  # :118
    x2 = x + mm(o, P.o_weight)                                       # layers.py:124-125
    ln2 = layernorm(x2, P.ln2_gain, P.ln2_bias)                      # layers.py:126
    m2, m1, g = mlp_fwd(ln2, P.mlp_w1, P.mlp_w2, chunk)              # layers.py:127
    out = x2 + m2                                                    # layers.py:136
    return out, dict(x=x, ln1=ln1, qkv=qkv, o=o, x2=x2, ln2=ln2, m1=m1, g=g)


def layer_bwd(d_out, P: Params, c: dict, n_heads: int, chunk=None):
    """Fused backward; returns (d_x, grads, inter) where ``inter`` holds the
    component payloads (d_attn_out, d_x2, d_qkv, d_ln1) for kernel-level checks."""
    d_ln2, d_m1 = mlp_bwd(d_out, P.mlp_w1, P.mlp_w2, c["m1"], chunk)   # layers.py:146-147
    d_x2_ln, dg2, db2 = layernorm_bwd(d_ln2, c["x2"], P.ln2_gain)      # :148, :159
    d_x2 = d_out + d_x2_ln                                            # :149
    d_o = mm_dx(d_x2, P.o_weight)                                     # :150
    qkv = c["qkv"]
    h = qkv.shape[-1] // 3
    dq, dk, dv = attention_bwd(qkv[..., :h], qkv[..., h:2 * h], qkv[..., 2 * h:], d_o, n_heads)
    d_qkv = np.concatenate([dq, dk, dv], axis=-1)                     # :178
    d_ln1 = mm_dx(d_qkv, P.qkv_weight)                                # :181 / :194
    d_x_ln, dg1, db1 = layernorm_bwd(d_ln1, c["x"], P.ln1_gain)       # :196, :202
    grads = {
        "ln1_gain": dg1, "ln1_bias": db1, "qkv_weight": mm_dw(c["ln1"], d_qkv),
        "o_weight": mm_dw(c["o"], d_x2), "ln2_gain": dg2, "ln2_bias": db2,
        "mlp_w1": mm_dw(c["ln2"], d_m1), "mlp_w2": mm_dw(c["g"], d_out),
    }
    inter = dict(d_m1=d_m1, d_ln2=d_ln2, d_x2=d_x2, d_o=d_o, d_qkv=d_qkv, d_ln1=d_ln1)
    return d_x_ln + d_x2, grads, inter


@dataclass
class OracleResult:
    losses: list[float]
    param_grads: list[dict[str, np.ndarray]]


def sequential_oracle(params: list[Params], inputs: list[np.ndarray], n_heads: int,
                      chunk=None) -> OracleResult:
    """Sequential reference run (model.py:105-122): one micro-batch at a time,
    forward through all layers, loss, backward, ascending-mb accumulation."""
    total = [{k: np.zeros_like(getattr(P, k)) for k in FIELDS} for P in params]
    losses = []
    for x in inputs:
        caches = []
        for P in params:
            x, cache = layer_fwd(x, P, n_heads, chunk)
            caches.append(cache)
        loss, d = loss_and_grad(x)
        losses.append(loss)
        per_mb = [None] * len(params)
        for li in reversed(range(len(params))):
            d, per_mb[li], _ = layer_bwd(d, params[li], caches[li], n_heads, chunk)
        for acc, g in zip(total, per_mb):
            for k in FIELDS:
                acc[k] += g[k]
    return OracleResult(losses, total)


# --- PLT1 golden container (runtime/tensorio.py:1-61) -----------------------------


def write_plt1(path, tensors: dict[str, np.ndarray]) -> None:
    import struct
    out = bytearray(b"PLT1" + struct.pack("<I", len(tensors)))
    for name, arr in tensors.items():
        a = np.ascontiguousarray(arr, dtype="<f8")
        enc = name.encode()
        out += struct.pack("<H", len(enc)) + enc + struct.pack("<B", a.ndim)
        out += struct.pack(f"<{a.ndim}Q", *a.shape) + a.tobytes()
    with open(path, "wb") as f:
        f.write(bytes(out))


def read_plt1(path) -> dict[str, np.ndarray]:
    import struct
    data = open(path, "rb").read()
    if data[:4] != b"PLT1":
        raise ValueError(f"{path}: bad magic")
    (count,), off = struct.unpack_from("<I", data, 4), 8
    out = {}
    for _ in range(count):
        (nlen,) = struct.unpack_from("<H", data, off)
        name = data[off + 2: off + 2 + nlen].decode()
        off += 2 + nlen
        (rank,) = struct.unpack_from("<B", data, off)
        shape = struct.unpack_from(f"<{rank}Q", data, off + 1)
        off += 1 + 8 * rank
        n = int(np.prod(shape)) if rank else 1
        out[name] = np.frombuffer(data, "<f8", n, off).reshape(shape).copy()
        off += 8 * n
    if off != len(data):
        raise ValueError(f"{path}: trailing bytes")
    return out

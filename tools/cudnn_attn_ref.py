#!/usr/bin/env python
"""Library yardstick for the attention kernels: PyTorch SDPA on the cuDNN
backend (bf16, causal, head_dim 128) at the bench shape, forward and backward,
CUDA-event timed, next to hx_attn_fwd / hx_attn_bwd on the same box.  Off the
product path (like tools/flashinfer_fmha_ref.py)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

from paper_2507_00394_b200.runtime import kernels as K  # noqa: E402

s, heads, d = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 16, 128)))
dev = "cuda"
fl_f = 2 * heads * s * s * d          # causal: 2 matmuls over the lower triangle
fl_b = 2.5 * fl_f


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = {"s": s, "heads": heads, "d": d}
q, k, v = (torch.randn(1, heads, s, d, device=dev, dtype=torch.bfloat16, requires_grad=True) for _ in range(3))
try:
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
        go = torch.randn_like(o)
        f_ms = timed(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True))
        fb_ms = timed(lambda: torch.autograd.grad(
            torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True), (q, k, v), go))
    out["cudnn"] = {"fwd_ms": f_ms, "fwd_tflops": fl_f / f_ms / 1e9, "bwd_ms": fb_ms - f_ms,
                    "bwd_tflops": fl_b / (fb_ms - f_ms) / 1e9}
except Exception as e:  # noqa: BLE001
    out["cudnn"] = {"error": str(e)[:200]}
h = heads * d
qkv = torch.randn(s, 3 * h, device=dev).to(torch.bfloat16)
o2 = torch.empty(s, h, dtype=torch.bfloat16, device=dev)
lse = torch.empty(1, heads, s, device=dev)
do = torch.randn(s, h, device=dev).to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
delta = torch.empty(heads * s, device=dev)
ws = K.attention_bwd_ws(s, 1, heads, d, dev)
fm = timed(lambda: K.attention_fwd(qkv, s, 1, heads, o2, lse))
bm = timed(lambda: K.attention_bwd(qkv, o2, do, lse, s, 1, heads, dqkv, delta, ws))
out["hx"] = {"fwd_ms": fm, "fwd_tflops": fl_f / fm / 1e9, "bwd_ms": bm, "bwd_tflops": fl_b / bm / 1e9}
print(json.dumps(out))

#!/usr/bin/env python
"""Runs the two heavy-epilogue GEMMs of the MLP once each at the GPT-1.3B/32k
shape (W1 + GeLU writing m1 and g; W2^T + GeLU' reading m1) -- a target for
`ncu -k regex:gemm_2sm -c 2` source-counter captures.  ``--ln`` adds one
LayerNorm backward (+ residual gradient) at T=32k, h=2048."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2507_00394_b200.runtime import kernels as K  # noqa: E402

T, h = 32768, 2048
dev, bf = torch.device("cuda", 0), torch.bfloat16
a = torch.randn(T, h, device=dev).to(bf)
w1 = (torch.randn(h, 4 * h, device=dev) / h ** 0.5).to(bf)
w2 = (torch.randn(4 * h, h, device=dev) / (4 * h) ** 0.5).to(bf)
m1 = torch.empty(T, 4 * h, dtype=bf, device=dev)
g = torch.empty_like(m1)
K.linear_gelu(a, w1, m1, g)
dy = torch.randn(T, h, device=dev).to(bf)
dm1 = torch.empty(T, 4 * h, dtype=bf, device=dev)
K.linear_dx_dgelu(dy, w2, m1, dm1)
if "--ln" in sys.argv:
    x = torch.randn(T, h, device=dev).to(bf)
    gain = torch.ones(h, device=dev)
    dx = torch.empty_like(x)
    dg, db = torch.zeros(h, device=dev), torch.zeros(h, device=dev)
    K.layernorm_bwd(dy, x, gain, dy, dx, dg, db)
torch.cuda.synchronize()
print("ok")

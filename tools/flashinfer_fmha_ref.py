"""Library yardstick for the attention forward: flashinfer's prebuilt trtllm-gen
sm100a context FMHA (bf16, head_dim 128, causal) at the bench's shape
(s=32768, 16 heads, batch 1), timed with CUDA events like tools/kernel_bench.py.
Not part of the product: it only calibrates how far hx_attn_fwd is from a
vendor kernel on the same box (attention forward).

    python tools/flashinfer_fmha_ref.py [--seq 32768] [--heads 16] [--reps 20]
"""

import argparse
import json
import sys
from pathlib import Path

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--page", type=int, default=64)   # cubins ship P16/P32/P64
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    from flashinfer.prefill import trtllm_batch_context_with_kv_cache

    dev = torch.device("cuda", 0)
    s, n, d, pg = a.seq, a.heads, a.dim, a.page
    torch.manual_seed(0)
    q = torch.randn(s, n, d, device=dev, dtype=torch.bfloat16)
    pages = s // pg
    kv = torch.randn(pages, 2, n, pg, d, device=dev, dtype=torch.bfloat16)   # HND
    block_tables = torch.arange(pages, device=dev, dtype=torch.int32).view(1, pages)
    seq_lens = torch.tensor([s], device=dev, dtype=torch.int32)
    cum = torch.tensor([0, s], device=dev, dtype=torch.int32)
    ws = torch.zeros(256 << 20, device=dev, dtype=torch.uint8)
    out = torch.empty_like(q)

    def run():
        trtllm_batch_context_with_kv_cache(q, kv, ws, block_tables, seq_lens, s, s,
                                           d ** -0.5, 1.0, 1, cum, cum, out=out,
                                           kv_layout="HND", causal=True)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    flops = 2 * 2 * s * s * d * n / 2          # QK^T + PV, causal half

    def report(name, ms):
        ms = sorted(ms)
        med = ms[len(ms) // 2]
        print(json.dumps({"kernel": name, "ms": round(med, 4), "s": s, "heads": n, "d": d,
                          "tflops": round(flops / med / 1e9, 1)}))

    report("flashinfer_trtllm_gen_fmha_fwd", ms)
    # hx_attn_fwd on the same box, same shape, timed the same way
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_2507_00394_b200.runtime import kernels as K
    qkv = torch.randn(s, 3 * n * d, device=dev).to(torch.bfloat16)
    o = torch.empty(s, n * d, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(1, n, s, device=dev)
    ours = []
    for i in range(a.reps + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        K.attention_fwd(qkv, s, 1, n, o, lse)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ours.append(e0.elapsed_time(e1))
    report("hx_attn_fwd", ours)


if __name__ == "__main__":
    main()

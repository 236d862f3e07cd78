#!/usr/bin/env python
"""Per-kernel throughput at the benchmark workload's shapes (CUDA-event timed).

    python tools/kernel_bench.py [--workload gpt1.3b_32k] [--only attn|gemm|ln] [--reps N]

Prints one JSON object per kernel: shape, ms, achieved TFLOP/s (GEMM/attention,
causal FLOP convention) or GB/s (LayerNorm), fraction of MEASURED_PEAKS.json.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2507_00394_b200.runtime import kernels as K  # noqa: E402

WL = {"gpt1.3b_32k": (2048, 16, 32768), "gpt3b_64k": (4096, 32, 65536), "gpt7b_128k": (4096, 32, 131072),
      "tiny": (256, 4, 1024)}


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt1.3b_32k")
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cublas", action="store_true", help="also time torch.matmul (cuBLAS) on each GEMM shape")
    args = ap.parse_args()
    h, heads, s = WL[args.workload]
    T = s
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
        else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}
    dev = "cuda"
    bf = torch.bfloat16

    def out(name, ms, flops=None, bytes_=None, **kw):
        rec = {"kernel": name, "ms": round(ms, 4), **kw}
        if flops:
            rec["tflops"] = flops / ms / 1e9
            rec["frac_of_peak"] = rec["tflops"] / peaks["bf16_tflops"]
        if bytes_:
            rec["gbs"] = bytes_ / ms / 1e6
            rec["frac_of_hbm"] = rec["gbs"] / peaks["hbm_gbs"]
        print(json.dumps(rec), flush=True)

    if args.only in ("", "gemm"):
        x = torch.randn(T, 4 * h, device=dev).to(bf)
        for (name, kin, nout) in (("qkv", h, 3 * h), ("o_proj", h, h), ("mlp_w1", h, 4 * h), ("mlp_w2", 4 * h, h)):
            w = (torch.randn(kin, nout, device=dev) / kin ** 0.5).to(bf)
            a = x[:, :kin].contiguous()
            y = torch.empty(T, nout, dtype=bf, device=dev)
            fl = 2 * T * kin * nout
            out(f"fwd_{name}", timed(lambda: K.linear(a, w, y), args.reps), fl, M=T, N=nout, K=kin)
            if args.cublas:
                out(f"cublas_fwd_{name}", timed(lambda: torch.matmul(a, w, out=y), args.reps), fl, M=T, N=nout, K=kin)
            dy = torch.randn(T, nout, device=dev).to(bf)
            dx = torch.empty(T, kin, dtype=bf, device=dev)
            out(f"dx_{name}", timed(lambda: K.linear_dx(dy, w, dx), args.reps), fl, M=T, N=kin, K=nout)
            acc = torch.zeros(kin, nout, device=dev)
            out(f"dw_{name}", timed(lambda: K.linear_dw(a, dy, acc), args.reps), fl, M=kin, N=nout, K=T)
            if args.cublas:
                wt = torch.empty(kin, nout, dtype=bf, device=dev)
                out(f"cublas_dw_{name}", timed(lambda: torch.matmul(a.t(), dy, out=wt), args.reps), fl,
                    M=kin, N=nout, K=T)
            if name == "mlp_w1":   # fused GeLU epilogue: writes m1 and g
                g = torch.empty_like(y)
                out("fwd_mlp_w1_gelu", timed(lambda: K.linear_gelu(a, w, y, g), args.reps), fl, M=T, N=nout, K=kin)
                del g
            if name == "mlp_w2":   # fused GeLU' epilogue: reads the pre-activation m1
                m1 = torch.randn(T, kin, device=dev).to(bf)
                out("dx_mlp_w2_dgelu", timed(lambda: K.linear_dx_dgelu(dy, w, m1, dx), args.reps), fl,
                    M=T, N=kin, K=nout)
                del m1
            del w, a, y, dy, dx, acc
        del x
        torch.cuda.empty_cache()

    if args.only in ("", "attn"):
        qkv = torch.randn(T, 3 * h, device=dev).to(bf)
        o = torch.empty(T, h, dtype=bf, device=dev)
        lse = torch.empty(1, heads, s, device=dev)
        fwd_fl = 2 * heads * s * s * (h // heads)
        out("attn_fwd", timed(lambda: K.attention_fwd(qkv, s, 1, heads, o, lse), args.reps), fwd_fl,
            s=s, heads=heads, d=h // heads)
        do = torch.randn(T, h, device=dev).to(bf)
        dqkv = torch.empty_like(qkv)
        delta = torch.empty(heads * s, device=dev)
        dq = K.attention_bwd_ws(s, 1, heads, h // heads, dev)
        out("attn_bwd", timed(lambda: K.attention_bwd(qkv, o, do, lse, s, 1, heads, dqkv, delta, dq),
                              args.reps), fwd_fl * 5 // 2, s=s, heads=heads, d=h // heads)
        del qkv, o, lse, do, dqkv, delta, dq

    if args.only in ("", "ln"):
        x = torch.randn(T, h, device=dev).to(bf)
        g = torch.ones(h, device=dev)
        b_ = torch.zeros(h, device=dev)
        y = torch.empty_like(x)
        out("ln_fwd", timed(lambda: K.layernorm(x, g, b_, y), args.reps), bytes_=2 * T * h * 2, T=T, h=h)
        dy = torch.randn(T, h, device=dev).to(bf)
        dx = torch.empty_like(x)
        dg = torch.zeros(h, device=dev)
        db = torch.zeros(h, device=dev)
        out("ln_bwd", timed(lambda: K.layernorm_bwd(dy, x, g, dy, dx, dg, db), args.reps),
            bytes_=4 * T * h * 2, T=T, h=h)
        z = torch.randn(T, h, device=dev).to(bf)
        dz = torch.empty_like(z)
        slot = torch.zeros(1, dtype=torch.float64, device=dev)
        out("mse_loss", timed(lambda: K.mse_loss(z, dz, slot), args.reps), bytes_=2 * T * h * 2, T=T, h=h)


if __name__ == "__main__":
    main()

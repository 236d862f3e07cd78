#!/usr/bin/env python
"""Interleaved A/B timing of the attention kernels from two builds of libhx.so
in ONE process (both loaded with ctypes), so box-to-box and power-cap drift
cancel: A B A B ... for --rounds rounds, median per build.

    python tools/ab_attn.py NEW.so OLD.so [--seq 32768] [--heads 16] [--rounds 15] [--only fwd|bwd]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import statistics

import torch

P, I = ctypes.c_void_p, ctypes.c_int


def load(path):
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
    lib.hx_attn_fwd.argtypes = [P, I, P, I, P, I, I, I, I, P]
    lib.hx_attn_bwd.argtypes = [P, I, P, P, I, P, P, P, P, I, I, I, I, I, P]
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--rounds", type=int, default=15)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    libs = [load(p) for p in a.libs]
    s, n, d = a.seq, a.heads, a.dim
    h = n * d
    dev, bf = "cuda", torch.bfloat16
    torch.manual_seed(0)
    qkv = torch.randn(s, 3 * h, device=dev).to(bf)
    o = torch.empty(s, h, dtype=bf, device=dev)
    lse = torch.empty(n, s, device=dev)
    do = torch.randn(s, h, device=dev).to(bf)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(n * s, device=dev)
    dq = torch.empty(s * h, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def fwd(lib):
        assert lib.hx_attn_fwd(qkv.data_ptr(), 3 * h, o.data_ptr(), h, lse.data_ptr(), s, 1, n, d, st) == 0

    def bwd(lib):
        assert lib.hx_attn_bwd(qkv.data_ptr(), 3 * h, o.data_ptr(), do.data_ptr(), h, lse.data_ptr(),
                               delta.data_ptr(), dq.data_ptr(), dqkv.data_ptr(), 3 * h, s, 1, n, d, st) == 0

    fl = 2 * n * s * s * d
    kinds = [k for k in ("fwd", "bwd") if a.only in ("", k)]
    for kind in kinds:
        fn, flops = (fwd, fl) if kind == "fwd" else (bwd, fl * 5 // 2)
        fwd(libs[0])
        times = [[], []]
        for r in range(a.rounds):
            for i in (0, 1) if r % 2 == 0 else (1, 0):
                fn(libs[i])
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn(libs[i])
                fn(libs[i])
                e1.record()
                torch.cuda.synchronize()
                times[i].append(e0.elapsed_time(e1) / 2)
        med = [statistics.median(t) for t in times]
        print(json.dumps({"kernel": f"attn_{kind}", "A": a.libs[0], "A_ms": round(med[0], 4),
                          "B": a.libs[1], "B_ms": round(med[1], 4), "A_over_B": round(med[1] / med[0], 4),
                          "A_tflops": round(flops / med[0] / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Pipeline trace of the attention forward kernel (debug build).

Builds libhx with -DHX_FWD_TRACE into build/trace/, runs one forward at the
GPT-1.3B/32k shape and prints, for CTA (0,0) (the heaviest query-tile pair),
the per-step clock64 intervals:
  sm_wait   softmax group waiting for S (s_full)
  sm_work   softmax group from S ready to P handed to the MMA warp
  mma_gap   P ready -> MMA thread issued PV (wake-up latency)
  s_lat     S issued -> softmax saw it (tensor-pipe queue + execution)

    python tools/fwd_trace.py [--s 32768] [--heads 16]
"""

from __future__ import annotations

import argparse
import ctypes
import glob
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def build() -> Path:
    out = ROOT / "build" / "trace"
    out.mkdir(parents=True, exist_ok=True)
    lib = out / "libhx.so"
    srcs = sorted(glob.glob(str(ROOT / "paper_2507_00394_b200" / "csrc" / "*.cu")))
    cmd = ["nvcc", "-O3", "-std=c++17", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", "-DHX_FWD_TRACE",
           "-DHX_POLY_EVERY=" + os.environ.get("HX_POLY_EVERY", "0"), "-shared", "-o", str(lib), *srcs]
    subprocess.run(cmd, check=True)
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--no-build", action="store_true")
    args = ap.parse_args()
    lib = ROOT / "build" / "trace" / "libhx.so" if args.no_build else build()
    os.environ["HX_LIB"] = str(lib)
    sys.path.insert(0, str(ROOT))
    import torch
    from paper_2507_00394_b200.runtime import kernels as K

    d = 128
    h = args.heads * d
    qkv = torch.randn(args.s, 3 * h, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(args.s, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(args.heads, args.s, device="cuda", dtype=torch.float32)
    for _ in range(2):
        K.attention_fwd(qkv, s=args.s, b=1, heads=args.heads, o=o, lse=lse)
    torch.cuda.synchronize()
    cl = ctypes.CDLL(str(lib))
    buf = (ctypes.c_longlong * 8192)()
    assert cl.hx_debug_fwd_trace(buf) == 0
    tr = [list(buf[i * 1024:(i + 1) * 1024]) for i in range(8)]
    nq = (args.s + 127) // 128
    nkv = nq  # CTA 0 holds the last pair
    t0 = min(tr[0][0], tr[1][0])
    rows = []
    for j in range(1, nkv - 1):
        for g in range(2):
            ready, done = tr[g][2 * j], tr[g][2 * j + 1]
            prev_done = tr[g][2 * j - 1]
            pv_issue = tr[2][2 * j + g] if 2 * j + g < 1024 else 0
            s_issue = tr[3][2 * j + g]
            ld, mx = tr[4 + g][j], tr[6 + g][j]
            rows.append((j, g, ready - prev_done, done - ready, pv_issue - done, ready - s_issue,
                         ld - ready, mx - ld, done - mx))
    print("step g  sm_wait  sm_work  mma_gap  s_lat  ld  max  exp")
    for r in rows[:6] + rows[len(rows) // 2:len(rows) // 2 + 6]:
        print("%4d %d %8d %8d %8d %8d %6d %6d %6d" % r)
    mid = rows[len(rows) // 4: 3 * len(rows) // 4]
    import statistics as st
    print({k: st.median(x[i] for x in mid) for i, k in
           [(2, "sm_wait"), (3, "sm_work"), (4, "mma_gap"), (5, "s_lat"), (6, "ld"), (7, "max"), (8, "exp")]})
    step = (tr[0][2 * (nkv - 2)] - tr[0][2 * 10]) / (nkv - 12)
    print({"cycles_per_step": step, "total_cycles": tr[0][2 * nkv - 1] - t0,
           "tensor_cycles_per_step_ideal": 2048})


if __name__ == "__main__":
    main()

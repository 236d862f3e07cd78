#!/usr/bin/env python
"""Pipeline trace of the fused attention backward kernel (debug build).

Builds libhx with -DHX_BWD_TRACE into build/trace_bwd/, runs one backward at the
GPT-1.3B/32k shape and prints, for CTA (0, 0) (key tile 0: every query tile),
median clock64 intervals per iteration of the MMA / compute / reduce roles.

    python tools/bwd_trace.py [--s 32768] [--heads 16]
"""

from __future__ import annotations

import argparse
import ctypes
import glob
import os
import statistics as st
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
EVENTS = ["mma_dV", "mma_dP", "mma_S_next", "mma_dK", "mma_dQ", "c_s_seen", "c_p_done", "c_dp_seen",
          "c_ds_done", "r_dq_seen", "r_dq_free", "r_stage_done", "c_bar_passed", "c7_ds_done", "c7_s_seen", "unused",
          "done_dP", "done_dV", "done_S_next", "done_dK", "done_dQ", "u21", "u22", "u23"]


def build() -> Path:
    out = ROOT / "build" / "trace_bwd"
    out.mkdir(parents=True, exist_ok=True)
    lib = out / "libhx.so"
    srcs = sorted(glob.glob(str(ROOT / "paper_2507_00394_b200" / "csrc" / "*.cu")))
    cmd = ["nvcc", "-O3", "-std=c++17", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", "-DHX_BWD_TRACE",
           "-DHX_POLY_EVERY=0", *os.environ.get("HX_TRACE_FLAGS", "").split(), "-shared", "-o", str(lib), *srcs]
    subprocess.run(cmd, check=True)
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--heads", type=int, default=16)
    args = ap.parse_args()
    lib = build()
    os.environ["HX_LIB"] = str(lib)
    sys.path.insert(0, str(ROOT))
    import torch
    from paper_2507_00394_b200.runtime import kernels as K

    d, s, heads = 128, args.s, args.heads
    h = heads * d
    qkv = torch.randn(s, 3 * h, device="cuda").to(torch.bfloat16)
    o = torch.empty(s, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(heads, s, device="cuda")
    K.attention_fwd(qkv, s, 1, heads, o, lse)
    do = torch.randn(s, h, device="cuda").to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(heads * s, device="cuda")
    dq = K.attention_bwd_ws(s, 1, heads, h // heads, "cuda")
    for _ in range(2):
        K.attention_bwd(qkv, o, do, lse, s, 1, heads, dqkv, delta, dq)
    torch.cuda.synchronize()
    cl = ctypes.CDLL(str(lib))
    buf = (ctypes.c_longlong * (24 * 512))()
    assert cl.hx_debug_bwd_trace(buf) == 0
    tr = {e: list(buf[i * 512:(i + 1) * 512]) for i, e in enumerate(EVENTS)}
    n = min(512, (s + 127) // 128)
    lo, hi = n // 4, 3 * n // 4

    def med(f):
        return st.median(f(i) for i in range(lo, hi))

    period = med(lambda i: tr["mma_dV"][i + 1] - tr["mma_dV"][i])
    out = {
        "period_cycles": period,
        "ideal_mma_cycles": 5 * 512,
        "dV->dP issue (dq_empty wait)": med(lambda i: tr["mma_dP"][i] - tr["mma_dV"][i]),
        "dP->dK issue (ds_full wait)": med(lambda i: tr["mma_dK"][i] - tr["mma_dP"][i]),
        "dK->dV(next) (p_full wait)": med(lambda i: tr["mma_dV"][i + 1] - tr["mma_dK"][i]),
        "compute: S seen -> P done": med(lambda i: tr["c_p_done"][i] - tr["c_s_seen"][i]),
        "compute: P done -> dP seen": med(lambda i: tr["c_dp_seen"][i] - tr["c_p_done"][i]),
        "compute: dP seen -> dS done": med(lambda i: tr["c_ds_done"][i] - tr["c_dp_seen"][i]),
        "compute: dS done -> S(next) seen": med(lambda i: tr["c_s_seen"][i + 1] - tr["c_ds_done"][i]),
        "dP issue -> compute sees dP": med(lambda i: tr["c_dp_seen"][i] - tr["mma_dP"][i]),
        "S(i+1) issue -> compute sees S": med(lambda i: tr["c_s_seen"][i + 1] - tr["mma_S_next"][i]),
        "dQ issue -> reduce sees dQ": med(lambda i: tr["r_dq_seen"][i] - tr["mma_dQ"][i]),
        "reduce: dQ seen -> TMEM freed": med(lambda i: tr["r_dq_free"][i] - tr["r_dq_seen"][i]),
        "reduce: TMEM freed -> staged": med(lambda i: tr["r_stage_done"][i] - tr["r_dq_free"][i]),
        "reduce: staged -> next dQ seen": med(lambda i: tr["r_dq_seen"][i + 1] - tr["r_stage_done"][i]),
        "dq freed -> dP(next) issue": med(lambda i: tr["mma_dP"][i + 1] - tr["r_dq_free"][i]),
    }
    out.update({
        "compute: dS done -> barrier passed": med(lambda i: tr["c_bar_passed"][i + 1] - tr["c_ds_done"][i]),
        "compute: barrier -> s_full wait start": med(lambda i: tr["u21"][i + 1] - tr["c_bar_passed"][i + 1]),
        "compute: s_full wait": med(lambda i: tr["c_s_seen"][i + 1] - tr["u21"][i + 1]),
        "S(i+1) done (observer) -> compute sees": med(lambda i: tr["c_s_seen"][i + 1] - tr["done_S_next"][i]),
        "pipe: dP done -> dV done": med(lambda i: tr["done_dV"][i] - tr["done_dP"][i]),
        "pipe: dV done -> S(i+1) done": med(lambda i: tr["done_S_next"][i] - tr["done_dV"][i]),
        "pipe: S(i+1) done -> dK done": med(lambda i: tr["done_dK"][i] - tr["done_S_next"][i]),
        "pipe: dK done -> dQ done": med(lambda i: tr["done_dQ"][i] - tr["done_dK"][i]),
        "pipe: dQ done -> dP(i+1) done": med(lambda i: tr["done_dP"][i + 1] - tr["done_dQ"][i]),
    })
    for k, v in out.items():
        print(f"{k:36s} {v:10.0f}")
    # raw event times of three mid iterations, relative to dV issue of the first
    base = tr["mma_dV"][n // 2]
    evs = sorted((tr[e][i] - base, e, i) for e in EVENTS[:15] + EVENTS[16:21]
                 for i in range(n // 2, n // 2 + 3))
    for t, e, i in evs:
        print(f"{t:8d}  {e:14s} it={i}")


if __name__ == "__main__":
    main()

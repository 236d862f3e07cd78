#!/usr/bin/env python
"""GEMM DRAM traffic against algorithmic bytes, per shape, from the per-launch
ncu CSV of `ncu --set full ... python tools/kernel_bench.py --reps 1` (every
kernel_bench case launches twice: warm-up + 1 rep; the order below is
kernel_bench's).  Algorithmic bytes = A + B read once, C written once
(+ the aux operand read for the fused GeLU' epilogue, + the second output of the
GeLU epilogue; fp32 C read and written for the weight-gradient accumulation).

    python tools/gemm_traffic.py profiles/ncu_launches_r02_kernel_bench.csv [h T]
"""
import csv
import json
import sys

h = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
T = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
cases = []
for name, kin, nout in (("qkv", h, 3 * h), ("o_proj", h, h), ("mlp_w1", h, 4 * h), ("mlp_w2", 4 * h, h)):
    cases += [(f"fwd_{name}", T, nout, kin, "store"), (f"dx_{name}", T, kin, nout, "store"),
              (f"dw_{name}", kin, nout, T, "acc_f32")]
    if name == "mlp_w1":
        cases.append(("fwd_mlp_w1_gelu", T, nout, kin, "gelu"))
    if name == "mlp_w2":
        cases.append(("dx_mlp_w2_dgelu", T, kin, nout, "dgelu"))

rows = list(csv.reader(open(sys.argv[1])))
idx = {k: i for i, k in enumerate(rows[0])}
launches = [r for r in rows[2:] if "gemm" in r[idx["Kernel Name"]]]
out = []
for k, (name, M, N, K, epi) in enumerate(cases):
    r = launches[2 * k + 1]  # the timed launch (second of the pair)
    rd = float(r[idx["dram__bytes_read.sum"]]) * 1e9
    wr = float(r[idx["dram__bytes_write.sum"]]) * 1e9
    alg = 2 * (M * K + K * N)
    alg += {"store": 2 * M * N, "gelu": 4 * M * N, "dgelu": 4 * M * N, "acc_f32": 8 * M * N}[epi]
    ms = float(r[idx["gpu__time_duration.sum"]])
    out.append({"case": name, "kernel": r[idx["Kernel Name"]].split("(")[0].replace("void ", ""),
                "M": M, "N": N, "K": K, "epilogue": epi, "ms_ncu": ms,
                "tflops_ncu": 2 * M * N * K / ms / 1e9, "dram_read_gb": rd / 1e9, "dram_write_gb": wr / 1e9,
                "algorithmic_gb": alg / 1e9, "traffic_over_algorithmic": (rd + wr) / alg})
print(json.dumps(out, indent=1))

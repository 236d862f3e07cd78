"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (needs the read-only reference mount):

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Outputs (all committed; nothing at test time reads /root/reference):
  schedules/<name>.txt        full ``dumps()`` text of reference schedules
  schedule_sha256.json        sha256 of ``dumps()`` over a config grid and the
                              BASELINE shapes (FLOPs-derived duration tables)
  numerics_<name>.plt         PLT1 (f64) losses + every parameter gradient of
                              the reference ``sequential_oracle`` and of its
                              ``execute_schedule`` for every method
  runtime_meta.json           reference peak_stash_elements / loss values
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

# Config grid for schedule hashes: (p, L-multiple, m-multiple) x tables x qkv.
GRID_P = (1, 2, 4, 8)
GRID_LMUL = (1, 2)
GRID_MMUL = (2, 4)
TABLES = ((1, 3, 2), (1, 30, 2), (2, 3, 2), (1, 1, 1), (3, 1, 2))

BASELINE = {
    "tiny": dict(L=4, h=256, s=1024, b=1, num_heads=4, p=2, m=4),
    "gpt1.3b_32k": dict(L=24, h=2048, s=32768, b=1, num_heads=16, p=4, m=8),
    "gpt3b_64k": dict(L=16, h=4096, s=65536, b=1, num_heads=32, p=8, m=16),
    "gpt7b_128k": dict(L=32, h=4096, s=131072, b=1, num_heads=32, p=8, m=16),
    "gpt1.3b_32k_p1": dict(L=24, h=2048, s=32768, b=1, num_heads=16, p=1, m=2),
}

NUMERIC_CASES = {
    # reference test shape (T/test_runtime.py:32) and the survey's fast CI shape
    "toy": (dict(L=4, h=8, s=8, b=2, num_heads=2, p=2, m=4), 0, 1),
    "ci": (dict(L=2, h=64, s=128, b=1, num_heads=2, p=2, m=4), 0, 1),
}


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import pipelab
    from pipelab.config import ModelConfig, device_preset
    from pipelab.costs import DurationTable
    from pipelab.runtime import execute_schedule, make_inputs, make_model, sequential_oracle
    from pipelab.runtime.tensorio import write_tensors
    from pipelab.schedule import dumps

    (HERE / "schedules").mkdir(exist_ok=True)
    unit = DurationTable.from_units(1, 3, 2)

    # Full texts: the tiny BASELINE config (all methods) and the reference test shape.
    for name, kw in (("tiny", BASELINE["tiny"]),
                     ("toy", NUMERIC_CASES["toy"][0])):
        cfg = ModelConfig(**kw)
        for method in pipelab.METHODS:
            (HERE / "schedules" / f"{name}_{method}.txt").write_text(
                dumps(pipelab.generate(method, cfg, unit)))

    hashes: dict[str, str] = {}
    for p in GRID_P:
        for lm in GRID_LMUL:
            for mm in GRID_MMUL:
                for tab in TABLES:
                    for qkv in (True, False):
                        kw = dict(L=p * lm, h=8, s=8, b=2, num_heads=2, p=p, m=mm * p)
                        cfg = ModelConfig(**kw)
                        for method in pipelab.METHODS:
                            key = (f"{method}|L{kw['L']}|p{p}|m{kw['m']}|"
                                   f"t{tab[0]}-{tab[1]}-{tab[2]}|qkv{int(qkv)}")
                            text = dumps(pipelab.generate(method, cfg, DurationTable.from_units(*tab),
                                                          qkv_in_attention=qkv))
                            hashes[key] = sha(text)
    for name, kw in BASELINE.items():
        cfg = ModelConfig(**kw)
        for dev in ("h20_like", "a800_like"):
            tab = DurationTable.from_flops(cfg, device_preset(dev), True)
            for method in pipelab.METHODS:
                try:
                    text = dumps(pipelab.generate(method, cfg, tab))
                except Exception as e:  # e.g. ConfigError for a shape a method rejects
                    text = f"error:{type(e).__name__}"
                hashes[f"{method}|{name}|flops-{dev}"] = sha(text)
    (HERE / "schedule_sha256.json").write_text(json.dumps(hashes, indent=1, sort_keys=True) + "\n")

    meta: dict[str, dict] = {}
    for name, (kw, pseed, iseed) in NUMERIC_CASES.items():
        cfg = ModelConfig(**kw)
        params, inputs = make_model(cfg, pseed), make_inputs(cfg, iseed)
        ref = sequential_oracle(params, inputs, cfg.num_heads)
        tensors = {"losses": np.array(ref.losses)}
        for l, g in enumerate(ref.param_grads):
            for k, v in g.items():
                tensors[f"grad.l{l}.{k}"] = v
        write_tensors(HERE / f"numerics_{name}.plt", tensors)
        entry = {"config": kw, "param_seed": pseed, "input_seed": iseed,
                 "losses": ref.losses, "peak_stash_elements": {}, "bitwise_equal": {}}
        for method in pipelab.METHODS:
            res = execute_schedule(pipelab.generate(method, cfg, unit), params, inputs)
            entry["peak_stash_elements"][method] = res.peak_stash_elements
            entry["bitwise_equal"][method] = bool(
                res.losses == ref.losses and all(
                    np.array_equal(res.param_grads[l][k], ref.param_grads[l][k])
                    for l in range(cfg.L) for k in ref.param_grads[l]))
        meta[name] = entry
    (HERE / "runtime_meta.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(f"wrote {len(hashes)} schedule hashes, {len(NUMERIC_CASES)} numeric cases")


if __name__ == "__main__":
    main()

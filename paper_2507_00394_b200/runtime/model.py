"""Model parameters on host and device, seeded fixtures, the synthetic loss.

Drop-in for ``pipelab.runtime.model`` fixtures (``P/runtime/model.py:31-64``):
``make_model`` / ``make_inputs`` draw from NumPy's PCG64 in the reference's
field order, so the same seeds give the same float64 weights and inputs, and
GPU results are directly comparable with the reference oracle.

Device side: :class:`DeviceLayer` holds one layer's weights as bf16 matrices
(``[in, out]`` layout, exactly the reference's) plus fp32 LayerNorm vectors,
and the fp32 gradient accumulators for whatever components a stage owns.
For performance runs at 1.3B-7B scale :func:`random_device_model` draws the
same distributions directly on the GPU (NumPy float64 would need 50+ GB).
"""

from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np
import torch

PARAM_FIELDS = ("ln1_gain", "ln1_bias", "qkv_weight", "o_weight",
                "ln2_gain", "ln2_bias", "mlp_w1", "mlp_w2")
MATRIX_FIELDS = ("qkv_weight", "o_weight", "mlp_w1", "mlp_w2")
PRE_FIELDS = ("ln1_gain", "ln1_bias", "qkv_weight")                     # layers.py:83
POST_FIELDS = ("o_weight", "ln2_gain", "ln2_bias", "mlp_w1", "mlp_w2")  # layers.py:84

Grads = dict[str, np.ndarray]


@dataclass
class LayerParams:
    """One layer's float64 weights (``P/runtime/layers.py:54-78``)."""

    ln1_gain: np.ndarray
    ln1_bias: np.ndarray
    qkv_weight: np.ndarray   # [h, 3h]
    o_weight: np.ndarray     # [h, h]
    ln2_gain: np.ndarray
    ln2_bias: np.ndarray
    mlp_w1: np.ndarray       # [h, 4h]
    mlp_w2: np.ndarray       # [4h, h]

    def field_names(self) -> tuple[str, ...]:
        return tuple(f.name for f in fields(self))

    def element_count(self) -> int:
        return sum(getattr(self, n).size for n in self.field_names())

    def as_dict(self) -> dict[str, np.ndarray]:
        return {n: getattr(self, n) for n in self.field_names()}


def _shape(name: str, h: int):
    return {"qkv_weight": (h, 3 * h), "o_weight": (h, h),
            "mlp_w1": (h, 4 * h), "mlp_w2": (4 * h, h)}.get(name, (h,))


def make_layer_params(rng: np.random.Generator, h: int) -> LayerParams:
    vals = {}
    for name in PARAM_FIELDS:
        shape = _shape(name, h)
        z = rng.standard_normal(shape)
        if name.endswith("gain"):
            vals[name] = 1.0 + 0.1 * z
        elif name.endswith("bias"):
            vals[name] = 0.1 * z
        else:
            vals[name] = z / np.sqrt(shape[0])
    return LayerParams(**vals)


def make_model(cfg, seed: int) -> list[LayerParams]:
    rng = np.random.default_rng(seed)
    return [make_layer_params(rng, cfg.h) for _ in range(cfg.L)]


def make_inputs(cfg, seed: int) -> list[np.ndarray]:
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((cfg.s, cfg.b, cfg.h)) for _ in range(cfg.m)]


def loss_and_grad(z: np.ndarray) -> tuple[float, np.ndarray]:
    """Host form of the synthetic head: mean(z^2), dz = 2z/numel (``model.py:61-64``)."""
    return float(np.mean(z * z)), z * (2.0 / z.size)


def zero_grads(params: list[LayerParams]) -> list[Grads]:
    return [{n: np.zeros_like(getattr(p, n)) for n in p.field_names()} for p in params]


# --- device side -----------------------------------------------------------------


class DeviceLayer:
    """One layer on a device: bf16 weight matrices, fp32 LN vectors, fp32 grads.

    Only the fields in ``owned`` get gradient buffers (a helix stage owns the
    pre fields of layers ``l % p == st`` and the post fields of layers whose
    post lands on it, ``P/partition.py:25-36``).
    """

    def __init__(self, tensors: dict[str, torch.Tensor], owned: tuple[str, ...],
                 grad_dtype: torch.dtype = torch.float32):
        self.w = tensors
        self.grad: dict[str, torch.Tensor] = {
            n: torch.zeros(tensors[n].shape, dtype=grad_dtype, device=tensors[n].device)
            for n in owned}

    def __getitem__(self, name: str) -> torch.Tensor:
        return self.w[name]

    def zero_grads(self, zero_fn) -> None:
        for g in self.grad.values():
            zero_fn(g)


def layer_to_device(p: LayerParams, device, fields_: tuple[str, ...] = PARAM_FIELDS) -> dict:
    out = {}
    for n in fields_:
        arr = torch.from_numpy(np.ascontiguousarray(getattr(p, n)))
        dt = torch.bfloat16 if n in MATRIX_FIELDS else torch.float32
        out[n] = arr.to(device=device, dtype=dt)
    return out


def random_device_layer(h: int, gen: torch.Generator, device) -> dict[str, torch.Tensor]:
    """Same distributions as :func:`make_layer_params`, drawn on the GPU."""
    out = {}
    for name in PARAM_FIELDS:
        shape = _shape(name, h)
        z = torch.randn(shape, generator=gen, device=device, dtype=torch.float32)
        if name.endswith("gain"):
            out[name] = 1.0 + 0.1 * z
        elif name.endswith("bias"):
            out[name] = 0.1 * z
        else:
            out[name] = (z / float(np.sqrt(shape[0]))).to(torch.bfloat16)
        del z
    return out

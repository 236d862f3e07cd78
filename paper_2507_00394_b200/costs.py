"""Integer cost model of one transformer layer split into pre / attn / post.

Drop-in for ``pipelab.costs`` (reference ``P/costs.py``).  Three things in here
are load-bearing for the B200 runtime, the rest is kept for API parity:

* ``comm_volume`` (``P/costs.py:139-156``) is the payload-size contract: the
  executor hard-fails a SEND whose element count differs from it.
* ``activation_elements`` (``P/costs.py:113-131``) sets every task's
  ``mem_delta`` and therefore the bit-exact schedule text.
* ``DurationTable`` (``P/costs.py:164-218``) is an input of the helix
  list-scheduling pass; the naive helix order depends on it.

``b200_flops_per_token`` is this framework's own accounting for MFU /
roofline: causal attention does half the reference's full-s^2 Table-1 count
(SURVEY.md H8), so the model-FLOPs numerator is ``L*(72h^2 + 6hs)`` per token.
"""

from __future__ import annotations

from dataclasses import dataclass

from .config import ConfigError, DeviceSpec, ModelConfig

COMPONENTS = ("pre", "attn", "post")
PASSES = ("fwd", "bwd_b", "bwd_w")

EDGE_PRE_ATTN = "pre_attn"
EDGE_ATTN_POST = "attn_post"
EDGE_BOUNDARY = "boundary"


@dataclass(frozen=True)
class PassFlops:
    fwd: int
    bwd_b: int
    bwd_w: int

    def __add__(self, other: "PassFlops") -> "PassFlops":
        return PassFlops(self.fwd + other.fwd, self.bwd_b + other.bwd_b,
                         self.bwd_w + other.bwd_w)


_ZERO = PassFlops(0, 0, 0)


@dataclass(frozen=True)
class ComponentCosts:
    pre: PassFlops
    attn: PassFlops
    post: PassFlops
    qkv_in_attention: bool

    def of(self, comp: str) -> PassFlops:
        return getattr(self, comp)


def op_flops(cfg: ModelConfig) -> dict[str, PassFlops]:
    """Dense-matmul FLOPs per op for one (layer, micro-batch): the paper's Table 1."""
    tok_h2 = cfg.b * cfg.s * cfg.h * cfg.h
    s2h = cfg.b * cfg.h * cfg.s * cfg.s
    uniform = lambda k: PassFlops(k * tok_h2, k * tok_h2, k * tok_h2)  # noqa: E731
    return {"qkv": uniform(6), "attn": PassFlops(4 * s2h, 8 * s2h, 0),
            "o": uniform(2), "mlp": uniform(16)}


def component_flops(cfg: ModelConfig, qkv_in_attention: bool = False) -> ComponentCosts:
    ops = op_flops(cfg)
    if qkv_in_attention:
        pre, attn = _ZERO, ops["qkv"] + ops["attn"]
    else:
        pre, attn = ops["qkv"], ops["attn"]
    return ComponentCosts(pre=pre, attn=attn, post=ops["o"] + ops["mlp"],
                          qkv_in_attention=qkv_in_attention)


def layer_flops(cfg: ModelConfig) -> PassFlops:
    c = component_flops(cfg)
    return c.pre + c.attn + c.post


def attention_flops_share(cfg: ModelConfig) -> float:
    return cfg.s / (6 * cfg.h + cfg.s)


def params_per_layer(h: int) -> int:
    return 12 * h * h + 4 * h


def activation_elements(cfg: ModelConfig, recompute: bool = False,
                        qkv_in_attention: bool = False) -> dict[str, int]:
    """Stashed elements per (component, layer, micro-batch); ``P/costs.py:113-131``.

    Full mode: 16 bsh per layer split 2/3/11 (1/4/11 with the projection in the
    attention component).  Recompute mode: the 4 bsh boundary inputs, attributed
    0/2/2.
    """
    bsh = cfg.tokens * cfg.h
    if recompute:
        split = (0, 2, 2)
    elif qkv_in_attention:
        split = (1, 4, 11)
    else:
        split = (2, 3, 11)
    return {comp: k * bsh for comp, k in zip(COMPONENTS, split)}


def layer_activation_elements(cfg: ModelConfig, recompute: bool = False) -> int:
    return sum(activation_elements(cfg, recompute=recompute).values())


def comm_volume(cfg: ModelConfig, edge: str, qkv_in_attention: bool = False) -> int:
    """Elements of one micro-batch payload crossing ``edge`` (either direction)."""
    bsh = cfg.tokens * cfg.h
    if edge == EDGE_PRE_ATTN:
        return 2 * bsh + 3 * cfg.h * cfg.h if qkv_in_attention else 4 * bsh
    if edge == EDGE_ATTN_POST:
        return 2 * bsh
    if edge == EDGE_BOUNDARY:
        return bsh
    raise ConfigError(f"unknown edge kind {edge!r}")


def qkv_transfer_saves(cfg: ModelConfig) -> bool:
    return 3 * cfg.h * cfg.h < 2 * cfg.tokens * cfg.h


@dataclass(frozen=True)
class DurationTable:
    """Integer duration per (component, pass); ``time_unit`` is "unit" or "ns"."""

    entries: dict[tuple[str, str], int]
    time_unit: str

    def of(self, comp: str, pass_: str) -> int:
        return self.entries[(comp, pass_)]

    def comp_totals(self, pass_: str) -> int:
        return sum(self.entries[(comp, pass_)] for comp in COMPONENTS)

    @staticmethod
    def _build(rows: dict[str, tuple[int, int, int]], unit: str) -> "DurationTable":
        entries = {(comp, pass_): val for comp, trip in rows.items()
                   for pass_, val in zip(PASSES, trip)}
        return DurationTable(entries=entries, time_unit=unit)

    @staticmethod
    def from_units(t_pre: int, t_attn: int, t_post: int) -> "DurationTable":
        """Abstract table with the FLOPs ratios: attention B = 2F, W = 0."""
        for t in (t_pre, t_attn, t_post):
            if not isinstance(t, int) or t < 0:
                raise ConfigError("unit durations must be non-negative ints")
        return DurationTable._build({"pre": (t_pre, t_pre, t_pre),
                                     "attn": (t_attn, 2 * t_attn, 0),
                                     "post": (t_post, t_post, t_post)}, "unit")

    @staticmethod
    def from_flops(cfg: ModelConfig, device: DeviceSpec,
                   qkv_in_attention: bool = False) -> "DurationTable":
        """Nanoseconds: each op's forward floored first, then the ratio rules."""
        rate = device.compute_rate * cfg.sp_size
        ns = {name: (pf.fwd * 1_000_000_000) // rate for name, pf in op_flops(cfg).items()}
        post = ns["o"] + ns["mlp"]
        if qkv_in_attention:
            pre = (0, 0, 0)
            attn = (ns["qkv"] + ns["attn"], ns["qkv"] + 2 * ns["attn"], ns["qkv"])
        else:
            pre = (ns["qkv"],) * 3
            attn = (ns["attn"], 2 * ns["attn"], 0)
        return DurationTable._build({"pre": pre, "attn": attn, "post": (post,) * 3}, "ns")

    @staticmethod
    def from_measured(pre_ns: tuple[int, int, int], attn_ns: tuple[int, int, int],
                      post_ns: tuple[int, int, int]) -> "DurationTable":
        """Table from device-measured (fwd, bwd_b, bwd_w) per component."""
        return DurationTable._build({"pre": tuple(pre_ns), "attn": tuple(attn_ns),
                                     "post": tuple(post_ns)}, "ns")


def transfer_ns(volume_elements: int, device: DeviceSpec) -> int:
    return (volume_elements * device.bytes_per_element * 1_000_000_000) // device.link_bandwidth


# --- B200 accounting (not in the reference) ---------------------------------


def b200_flops_per_token(cfg: ModelConfig, causal: bool = True) -> int:
    """Model FLOPs per token for fwd+bwd over all layers.

    Causal: ``L*(72h^2 + 6hs)``; the reference's full-square convention
    (``P/costs.py:62-71``) is ``L*(72h^2 + 12hs)``.
    """
    attn = 6 if causal else 12
    return cfg.L * (72 * cfg.h * cfg.h + attn * cfg.h * cfg.s)


def attention_kernel_flops(cfg: ModelConfig) -> tuple[int, int]:
    """(forward, backward) FLOPs of one causal attention call for one micro-batch.

    fwd = 2*b*n*s^2*d (two matmuls over the causal half), bwd = 2.5x fwd.
    """
    fwd = 2 * cfg.b * cfg.num_heads * cfg.s * cfg.s * cfg.head_dim
    return fwd, (5 * fwd) // 2

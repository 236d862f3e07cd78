"""Closed-form pipeline bubble and activation-memory predictions.

Restates ``P/analytic.py`` (the paper's §3 formulas): per-stage bubble for
zero-cost communication and the canonical duration ratios (attention backward
B = 2F, W = 0), and per-stage peak stashed-activation elements.  The bench
puts these beside the simulated and the device-measured bubble,
so a gap between the three points at the cause: formula assumptions, the list
scheduler, or the hardware (transfers, launch gaps).

Per-stage bubble (``P/analytic.py:46-58``; worked examples ``T/test_analytic.py:27-32``):

  1f1b              3 (p-1) (t_pre + t_attn + t_post) L/p
  zb1p                (p-1) (t_pre + 3 t_attn + t_post) L/p
  helix_naive       3 (p-1) (t_pre + t_post)
  helix_twofold     6 (p-1) (t_pre + t_post)
  helix_twofold_rc  8 (p-1) (t_pre + t_post)

Peak stashed activations (``P/analytic.py:65-77``), bsh = tokens per
micro-batch times hidden:

  1f1b stage i   16 bsh (p-i) L/p      helix          16 bsh m L/p
  zb1p           16 bsh L (a cap)      helix + rc      4 bsh m L/p

B200 extension: :func:`stage_memory_bytes` turns the element model into a
per-rank byte budget (bf16 stash + the flash-attention extras + weights and
fp32 gradients + transfer buffers) for DESIGN.md's per-config table.
"""

from __future__ import annotations

from dataclasses import dataclass

from .config import ConfigError, ModelConfig
from .costs import DurationTable

# helix rows: bubble = factor * (p - 1) * (t_pre + t_post), independent of L and m
_HELIX_BUBBLE = {"helix_naive": 3, "helix_twofold": 6, "helix_twofold_rc": 8}


def bubble_time(method: str, p: int, L: int, t_pre: int, t_attn: int, t_post: int) -> int:
    """Predicted per-stage bubble, in the unit of the durations (integer)."""
    if method in _HELIX_BUBBLE:
        return _HELIX_BUBBLE[method] * (p - 1) * (t_pre + t_post)
    if method in ("1f1b", "zb1p"):
        if L % p:
            raise ConfigError(f"{method} formula needs L % p == 0")
        per_layer = t_pre + t_attn + t_post
        if method == "1f1b":
            return 3 * (p - 1) * per_layer * L // p
        return (p - 1) * (per_layer + 2 * t_attn) * L // p
    raise ConfigError(f"no bubble formula for method {method!r}")


def bubble_time_from_table(method: str, p: int, L: int, table: DurationTable) -> int:
    """:func:`bubble_time` with the forward durations of a table."""
    fwd = {comp: table.of(comp, "fwd") for comp in ("pre", "attn", "post")}
    return bubble_time(method, p, L, fwd["pre"], fwd["attn"], fwd["post"])


def peak_activation_elements(method: str, cfg: ModelConfig, stage: int) -> int:
    """Peak stashed activation elements of ``stage`` (``P/analytic.py:65-77``)."""
    bsh = cfg.tokens * cfg.h
    if method == "1f1b":
        return 16 * bsh * (cfg.p - stage) * cfg.L // cfg.p
    if method == "zb1p":
        return 16 * bsh * cfg.L
    if method in ("helix_naive", "helix_twofold"):
        return 16 * bsh * cfg.m * cfg.L // cfg.p
    if method == "helix_twofold_rc":
        return 4 * bsh * cfg.m * cfg.L // cfg.p
    raise ConfigError(f"no memory formula for method {method!r}")


def memory_is_bound(method: str) -> bool:
    """True where the memory figure is a cap (ZB1P) rather than exact."""
    return method == "zb1p"


def activation_bytes_per_gpu(method: str, cfg: ModelConfig, stage: int, bytes_per_element: int = 2) -> int:
    """Stashed-activation bytes on one GPU of ``stage`` (sp shards evenly)."""
    return peak_activation_elements(method, cfg, stage) * bytes_per_element // cfg.sp_size


def activation_bytes_by_stage(method: str, cfg: ModelConfig, bytes_per_element: int = 2) -> list[int]:
    return [activation_bytes_per_gpu(method, cfg, st, bytes_per_element) for st in range(cfg.p)]


# --- comparison against a simulated / measured run ----------------------------------------


@dataclass
class CheckRow:
    quantity: str
    stage: int
    predicted: int
    observed: float
    rel_diff: float
    ok: bool


@dataclass
class ComparisonReport:
    method: str
    rows: list[CheckRow]
    tolerance: float

    @property
    def ok(self) -> bool:
        return all(r.ok for r in self.rows)

    def lines(self) -> list[str]:
        return [f"{'ok  ' if r.ok else 'FAIL'} {r.quantity:<10} stage {r.stage}: predicted {r.predicted} "
                f"observed {r.observed} rel_diff {r.rel_diff:.3e}" for r in self.rows]


def compare(method: str, cfg: ModelConfig, table: DurationTable, metrics, tolerance: float = 0.0) -> ComparisonReport:
    """Formula vs a run's per-stage bubble and peak activation (``P/analytic.py:128-158``)."""
    rel = lambda pred, obs: (obs - pred) / max(1, abs(pred))  # noqa: E731
    pred_b = bubble_time_from_table(method, cfg.p, cfg.L, table)
    rows = [CheckRow("bubble", st, pred_b, obs, rel(pred_b, obs), abs(rel(pred_b, obs)) <= tolerance)
            for st, obs in enumerate(metrics.per_stage_bubble)]
    capped = memory_is_bound(method)
    attained = False
    for st, obs in enumerate(metrics.per_stage_peak_activation):
        pred = peak_activation_elements(method, cfg, st)
        ok = obs <= pred if capped else abs(rel(pred, obs)) <= tolerance
        attained = attained or obs == pred
        rows.append(CheckRow("memory", st, pred, obs, rel(pred, obs), ok))
    if capped:
        rows.append(CheckRow("memory_cap_attained", -1, 1, int(attained), 0.0 if attained else -1.0, attained))
    return ComparisonReport(method, rows, tolerance)


def bubble_fraction(method: str, cfg: ModelConfig, table: DurationTable) -> float:
    """Formula bubble as a fraction of a stage's window: B / (B + busy), with
    busy = every task's duration summed over the iteration / p (all stages
    carry equal work under the helix and 1F1B partitions)."""
    B = bubble_time_from_table(method, cfg.p, cfg.L, table)
    per_layer_mb = sum(table.of(c, ps) for c in ("pre", "attn", "post") for ps in ("fwd", "bwd_b", "bwd_w"))
    if method.endswith("_rc"):
        per_layer_mb += table.of("pre", "fwd") + table.of("post", "fwd")
    busy = per_layer_mb * cfg.L * cfg.m / cfg.p
    return B / (B + busy) if B + busy else 0.0


# --- per-rank HBM model (B200 extension) ----------------------------------------------------


def stage_memory_bytes(method: str, cfg: ModelConfig, stage: int = 0, *, drop_pre_x: bool = False,
                       mlp_chunk: int | None = None, send_cap: int = 4) -> dict[str, int]:
    """Per-rank peak HBM estimate of one stage (bytes) at bf16 activations.

    stash      the analytic peak (elements x 2 B); with ``drop_pre_x`` the rc
               retention drops the pre stash's x (4 -> 3 bsh per layer-mb)
    extras     flash backward's O and row LSE per attention stash (bf16 O is
               the post stash's attn_out when co-located, so only the LSE counts)
    params     bf16 weights + fp32 gradients of the layers this stage owns
               (12 h^2 per layer, split pre 3h^2 / post 9h^2 over stages)
    transient  the largest backward working set: regenerated post stash of one
               layer (11 bsh, or 3 bsh + 8 c*b*h with a chunked MLP) + MLP and
               attention gradients (~8 bsh) + fp32 dQ accumulator (2 bsh)
    transfer   in-flight send payloads (``send_cap`` per peer, 3 bsh + 3h^2 each,
               worst case) -- bounded by the driver, not by the schedule
    """
    bsh = cfg.tokens * cfg.h
    stash_el = peak_activation_elements(method, cfg, stage)
    if drop_pre_x and method == "helix_twofold_rc":
        stash_el = 3 * bsh * cfg.m * cfg.L // cfg.p
    layers_here = cfg.L // cfg.p
    lse = 4 * cfg.tokens * cfg.num_heads * (cfg.m * layers_here)
    params = layers_here * 12 * cfg.h * cfg.h * (2 + 4)
    c = cfg.s if mlp_chunk is None else min(mlp_chunk, cfg.s)
    regen = (3 * bsh + 8 * c * cfg.b * cfg.h) if mlp_chunk else 11 * bsh
    transient = 2 * (regen + 8 * bsh) + 4 * bsh
    peers = max(0, cfg.p - 1)
    transfer = 2 * send_cap * peers * (3 * bsh + 3 * cfg.h * cfg.h) if peers else 0
    out = {"stash": 2 * stash_el, "extras": lse, "params": params, "transient": transient,
           "transfer_worst": transfer}
    out["total"] = sum(out.values())
    return out

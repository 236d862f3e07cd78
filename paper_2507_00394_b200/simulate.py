"""Bubble / makespan metrics over a timeline (simulated or device-measured).

The metric definitions are the reference's (``P/simulate.py:54-97``):

* makespan   = latest task end;
* busy[st]   = sum of compute-task durations on stage ``st``;
* bubble[st] = makespan - busy[st];
* bubble fraction = sum(bubble) / (n_stages * makespan);
* peak activation = max prefix sum of ``mem_delta`` applied at task end,
  frees ordered before allocations at equal times.

:func:`simulate` replays a schedule through the integer engine (the
reference's prediction); :func:`metrics_from_timeline` applies the same
definitions to CUDA-event timelines recorded by the B200 executor, so
predicted and measured bubble are directly comparable.
"""

from __future__ import annotations

from dataclasses import dataclass

from .costs import DurationTable
from .engine import CommModel, make_duration_fn, replay
from .generators import comm_hidden, warmup_mbs
from .schedule import RECV, SEND, Schedule


@dataclass
class Metrics:
    makespan: float
    per_stage_busy: list[float]
    per_stage_bubble: list[float]
    bubble_fraction: float
    per_stage_peak_activation: list[int]
    total_send_elements: int
    time_unit: str


@dataclass
class SimResult:
    sched: Schedule
    timeline: dict[str, tuple[float, float]]
    metrics: Metrics


def memory_profile(sched: Schedule, timeline) -> list[list[tuple[float, int]]]:
    profiles = []
    for order in sched.per_stage_order:
        events = sorted((timeline[tid][1], sched.tasks[tid].mem_delta > 0, tid,
                         sched.tasks[tid].mem_delta)
                        for tid in order if sched.tasks[tid].mem_delta)
        level, prof = 0, []
        for when, _alloc, _tid, delta in events:
            level += delta
            prof.append((when, level))
        profiles.append(prof)
    return profiles


def metrics_from_timeline(sched: Schedule, timeline, time_unit: str = "ms") -> Metrics:
    """Reference metric definitions applied to an arbitrary (start, end) timeline.

    ``timeline`` must cover every compute task; comm tasks are optional (a
    device timeline records them on the comm stream).
    """
    n = sched.n_stages
    makespan = max((end for _s, end in timeline.values()), default=0)
    t0 = min((start for start, _e in timeline.values()), default=0)
    makespan -= t0
    busy = [0.0] * n
    for tid, (start, end) in timeline.items():
        task = sched.tasks[tid]
        if task.is_compute:
            busy[task.stage] += end - start
    bubble = [makespan - b for b in busy]
    peaks = [max((lvl for _t, lvl in prof), default=0)
             for prof in memory_profile(sched, timeline)]
    sends = sum(t.volume for t in sched.tasks.values() if t.kind == SEND)
    frac = sum(bubble) / (n * makespan) if makespan else 0.0
    return Metrics(makespan, busy, bubble, frac, peaks, sends, time_unit)


def measured_durations(sched: Schedule, timeline) -> DurationTable:
    """Average device time per (component, pass) from a CUDA-event timeline, as a
    ``DurationTable`` in integer nanoseconds.  Fused backward
    tasks bill B and W together, so the W column is set to 0 and B carries both."""
    sums: dict[tuple[str, str], list[float]] = {}
    kinds = {"FWD": "fwd", "BWD_B": "bwd_b", "BWD_W": "bwd_w"}
    for tid, (start, end) in timeline.items():
        t = sched.tasks.get(tid)
        if t is None or t.kind not in kinds or t.comp == "chunk":
            continue
        sums.setdefault((t.comp, kinds[t.kind]), []).append(end - start)
    avg = {k: int(round(1e6 * sum(v) / len(v))) for k, v in sums.items()}  # ms -> ns
    row = lambda comp: (avg.get((comp, "fwd"), 0), avg.get((comp, "bwd_b"), 0),  # noqa: E731
                        avg.get((comp, "bwd_w"), 0))
    return DurationTable.from_measured(row("pre"), row("attn"), row("post"))


def task_class_durations(sched: Schedule, timeline) -> dict[str, int]:
    """Average device ns per task class ``KIND.comp`` (FWD.pre, RECOMPUTE.post,
    BWD_B.chunk, ...) from a CUDA-event timeline -- finer than a
    ``DurationTable``: recompute tasks keep their own (measured) cost, and chunk
    tasks (1F1B) are covered."""
    sums: dict[str, list[float]] = {}
    for tid, (start, end) in timeline.items():
        t = sched.tasks.get(tid)
        if t is None or not t.is_compute:
            continue
        key = f"{t.kind}.{t.comp}" + (f".x{t.span}" if t.comp == "chunk" else "")
        sums.setdefault(key, []).append(end - start)
    return {k: int(round(1e6 * sum(v) / len(v))) for k, v in sums.items()}


def simulate_classes(sched: Schedule, classes: dict[str, int], comm: CommModel | None = None) -> SimResult:
    """The reference's list scheduler (``P/engine.py``) replaying ``sched`` with
    per-task-class durations (``task_class_durations``, e.g. measured on one
    rank by the stage probe); SEND/RECV cost per ``comm``."""

    def dur(task) -> int:
        key = f"{task.kind}.{task.comp}" + (f".x{task.span}" if task.comp == "chunk" else "")
        return classes[key]

    res = replay(sched, dur, comm or CommModel.zero())
    return SimResult(sched, res.timeline, metrics_from_timeline(sched, res.timeline, "ns"))


def _analytic_fraction(method: str, cfg, durations: DurationTable) -> float | None:
    from .analytic import bubble_fraction
    from .config import ConfigError
    try:
        return bubble_fraction(method, cfg, durations)
    except ConfigError:     # no formula (e.g. 1f1b_rc, a B200 extension)
        return None


def predict_pipeline(cfg, durations: DurationTable, stages=(2, 4, 8), link_gbs: float = 770.0,
                     latency_us: float = 5.0,
                     methods=("helix_twofold", "helix_twofold_rc", "1f1b", "1f1b_rc")) -> dict:
    """Predicted throughput of each method at p stages (m = 2p, weak scaling),
    from measured per-component durations (ns) and an NVLink transfer model
    (bytes over ``link_gbs`` per direction + latency) in the reference's own
    list-scheduling simulator (``P/simulate.py:54-75``).  A prediction, not a
    measurement: it shows where the measured kernels put the helix-vs-1F1B ratio."""
    from .engine import CommModel
    from .generators import generate

    comm = CommModel("bytes", latency=int(latency_us * 1000), bytes_per_element=2,
                     bandwidth=int(link_gbs * 1e9))
    out = {}
    for p in stages:
        if cfg.L % p:
            continue
        c = cfg.with_(p=p, m=2 * p)
        row = {}
        for method in methods:
            res = simulate(generate(method, c, durations), durations, comm)
            tokens = c.m * c.s * c.b
            ov = overlap_report(res)
            row[method] = {"tokens_per_s": tokens / (res.metrics.makespan * 1e-9),
                           "bubble_fraction": res.metrics.bubble_fraction,
                           # closed form (P/analytic.py:46-58), zero comm, forward durations only
                           "analytic_bubble_fraction": _analytic_fraction(method, c, durations),
                           "makespan_ms": res.metrics.makespan / 1e6,
                           # transfer waits: all, and those the schedule meant to hide
                           "comm_wait_ms": ov.total_wait / 1e6, "steady_comm_wait_ms": ov.steady_wait / 1e6}
        if "1f1b" in row:
            for method in methods:
                if method != "1f1b":
                    row[method]["speedup_vs_1f1b"] = (row["1f1b"]["makespan_ms"] / row[method]["makespan_ms"])
        if "1f1b_rc" in row and "helix_twofold_rc" in row:
            # like for like when the full stash does not fit: both with recomputation
            row["helix_twofold_rc"]["speedup_vs_1f1b_rc"] = (row["1f1b_rc"]["makespan_ms"] /
                                                            row["helix_twofold_rc"]["makespan_ms"])
        out[f"p{p}"] = row
    return out


def simulate(sched: Schedule, durations: DurationTable, comm: CommModel | None = None) -> SimResult:
    fused = sched.meta.get("backward") == "fused"
    chunk_rc = bool(int(sched.meta.get("recompute", 0))) and any(
        t.comp == "chunk" for t in sched.tasks.values() if t.is_compute)
    res = replay(sched, make_duration_fn(durations, fused, chunk_rc), comm or CommModel.zero())
    return SimResult(sched, res.timeline,
                     metrics_from_timeline(sched, res.timeline, durations.time_unit))


# --- communication-wait accounting (``P/simulate.py:100-151``) ----------------------------


@dataclass
class OverlapRow:
    task_id: str
    stage: int
    mb: int
    wait: float
    hidden: bool          # the schedule expects this task's inbound transfer to be hidden


@dataclass
class OverlapReport:
    rows: list[OverlapRow]
    per_stage_wait: list[float]
    total_wait: float
    steady_wait: float    # waits on tasks whose transfers should have been hidden
    warmup_mbs: set[int]


def overlap_report(sched_or_result, timeline=None) -> OverlapReport:
    """How long each compute task started after it could have (its stage free
    and every producer finished), on a simulated or device-measured timeline.

    A task's floor is the end of the previous task on its stage and of each
    dependency; a RECV dependency is charged at its payload's producer finish,
    so the wait beyond the floor is wire / queueing time.  Two-fold schedules
    expect the second member of each micro-batch pair to hide its transfer
    (``comm_hidden``); other schedules expect every micro-batch after the
    warm-up to.  ``steady_wait`` sums the waits of those tasks: the part of the
    communication the schedule failed to hide.  Accepts ``overlap_report(result)``
    (a :class:`SimResult`, as the reference) or ``overlap_report(sched, timeline)``.
    """
    if timeline is None:
        sched, tl = sched_or_result.sched, sched_or_result.timeline
    else:
        sched, tl = sched_or_result, timeline
    p = int(sched.meta["p"])
    twofold = int(sched.meta.get("fold", 1)) == 2
    warm = warmup_mbs(sched)
    rows: list[OverlapRow] = []
    per_stage = [0] * sched.n_stages
    for st, order in enumerate(sched.per_stage_order):
        stage_free = 0
        for tid in order:
            task = sched.tasks[tid]
            ready = stage_free
            for dep in task.deps:
                d = sched.tasks[dep]
                # RECV -> its SEND -> the compute task that produced the payload
                src = sched.tasks[d.deps[0]].deps[0] if d.kind == RECV else dep
                ready = max(ready, tl[src][1])
            start, end = tl[tid]
            if start > ready:
                hidden = comm_hidden(task.kind, task.mb, p) if twofold else task.mb not in warm
                rows.append(OverlapRow(tid, st, task.mb, start - ready, hidden))
                per_stage[st] += start - ready
            stage_free = end
    return OverlapReport(rows, per_stage, sum(per_stage),
                         sum(r.wait for r in rows if r.hidden), warm)


# --- exports (reference schema, ``P/simulate.py:157-196``) -------------------------------


def chrome_trace(sched: Schedule, timeline, time_unit: str = "ms") -> list[dict]:
    """Chrome trace-event list of a (simulated or device-measured) timeline:
    pid = stage, tid = lane ("compute", "in" for RECV, "out" for SEND), ts / dur
    in microseconds, args = (kind, comp, mb, layer), the reference's schema.
    ``time_unit``: "ms" (CUDA-event timelines), "ns", or "units" (1:1)."""
    from .schedule import RECV
    scale = {"ms": 1e3, "ns": 1e-3}.get(time_unit, 1.0)
    events = []
    for tid in sorted(timeline):
        t = sched.tasks[tid]
        start, end = timeline[tid]
        lane = {SEND: "out", RECV: "in"}.get(t.kind, "compute")
        events.append({
            "name": tid, "ph": "X", "pid": t.stage, "tid": lane,
            "ts": start * scale, "dur": (end - start) * scale, "cat": t.kind,
            "args": {"kind": t.kind, "comp": t.comp, "mb": t.mb, "layer": t.layer},
        })
    return events


def write_chrome_trace(path, sched: Schedule, timeline, time_unit: str = "ms") -> None:
    import json
    from pathlib import Path
    Path(path).write_text(json.dumps({"traceEvents": chrome_trace(sched, timeline, time_unit)}, indent=1))


def timeline_csv(sched: Schedule, timeline) -> str:
    """Task intervals as CSV (task, stage, kind, mb, layer, start, end), sorted by
    (start, end, task) like the reference's export."""
    import csv
    import io
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["task", "stage", "kind", "mb", "layer", "start", "end"])
    for tid, (start, end) in sorted(timeline.items(), key=lambda kv: (kv[1][0], kv[1][1], kv[0])):
        t = sched.tasks[tid]
        w.writerow([tid, t.stage, t.kind, t.mb, t.layer, start, end])
    return buf.getvalue()

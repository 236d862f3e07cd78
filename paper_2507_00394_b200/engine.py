"""Integer-time list scheduler: the core the helix / ZB1P generators run.

Semantics follow ``P/engine.py:160-262`` exactly, because the helix forward
order *is* the order this pass realises (``P/generators.py:374-375``) and the
schedule must be bit-exact:

* every stage owns one compute executor, one outbound and one inbound channel;
* the event queue is a heap of ``(time, tag, key)`` with tags
  FINISH(0) < ARRIVAL(1) < WAKE(2); WAKE keys are zero-padded stage strings,
  so ties resolve by (time, tag, id) and runs are reproducible;
* a SEND is placed when its last producer finishes, occupies the outbound
  channel for the wire time and lands ``latency`` later as an ARRIVAL that
  queues on the receiver's inbound channel;
* a stage only picks a task (through the selector) when it is free.

On the B200 runtime the same pass is reused, fed with device-measured
component times, to predict bubble and makespan next to the measured ones
(SURVEY.md §8f-1).
"""

from __future__ import annotations

import heapq
from bisect import bisect_right
from dataclasses import dataclass, field

from .config import DeviceSpec
from .schedule import BWD_B, BWD_W, FWD, RECOMPUTE, RECV, SEND, Schedule, Task

FINISH, ARRIVAL, WAKE = 0, 1, 2


@dataclass(frozen=True)
class CommModel:
    """Wire time per payload plus a fixed latency (``P/engine.py:32-75``)."""

    mode: str = "zero"
    latency: int = 0
    uniform_cost: int = 0
    ref_volume: int = 0
    bytes_per_element: int = 2
    bandwidth: int = 0
    slowdown: float = 1.0

    def wire_time(self, volume: int) -> int:
        if self.mode == "zero":
            return 0
        if self.mode == "uniform":
            return (volume * self.uniform_cost) // self.ref_volume if self.ref_volume \
                else self.uniform_cost
        return (volume * self.bytes_per_element * 1_000_000_000) // self.bandwidth

    @staticmethod
    def zero() -> "CommModel":
        return CommModel()

    @staticmethod
    def uniform(cost: int, latency: int = 0, slowdown: float = 1.0,
                ref_volume: int = 0) -> "CommModel":
        return CommModel("uniform", latency, cost, ref_volume, slowdown=slowdown)

    @staticmethod
    def from_device(device: DeviceSpec, slowdown: float = 1.0) -> "CommModel":
        return CommModel("bytes", device.latency_ns, bytes_per_element=device.bytes_per_element,
                         bandwidth=device.link_bandwidth, slowdown=slowdown)


_PASS_OF = {FWD: "fwd", RECOMPUTE: "fwd", BWD_B: "bwd_b", BWD_W: "bwd_w"}


def make_duration_fn(table, fused_backward: bool = False, chunk_recompute: bool = False):
    """Task -> integer duration; a fused BWD_B also bills the weight pass.
    ``chunk_recompute`` (B200 extension, ``1f1b_rc``): a chunk's backward also
    re-runs the pre and post forward of each of its layers."""

    def duration(task: Task) -> int:
        pass_ = _PASS_OF[task.kind]
        if task.comp == "chunk":
            total = task.span * table.comp_totals(pass_)
            extra = task.span * table.comp_totals("bwd_w")
            if chunk_recompute and task.kind == BWD_B:
                total += task.span * (table.of("pre", "fwd") + table.of("post", "fwd"))
        else:
            total = table.of(task.comp, pass_)
            extra = table.of(task.comp, "bwd_w")
        return total + extra if fused_backward and task.kind == BWD_B else total

    return duration


class DeadlockError(RuntimeError):
    def __init__(self, missing: list[str], detail: str):
        super().__init__(f"schedule deadlocked; {len(missing)} tasks never ran. {detail}")
        self.missing = missing


class ReplaySelector:
    """Follow a recorded per-stage order strictly, stalling in place."""

    def __init__(self, per_stage_order: list[list[str]]):
        self.orders = per_stage_order
        self.ptr = [0] * len(per_stage_order)

    def pick(self, stage: int, pool: dict[str, int], now: int) -> str | None:
        i = self.ptr[stage]
        order = self.orders[stage]
        if i < len(order) and order[i] in pool:
            self.ptr[stage] = i + 1
            return order[i]
        return None


class PrioritySelector:
    """Pick the ready task with the smallest precomputed key."""

    def __init__(self, key: dict[str, tuple]):
        self.key = key

    def pick(self, stage: int, pool: dict[str, int], now: int) -> str | None:
        return min(pool, key=self.key.__getitem__) if pool else None


@dataclass
class _Intervals:
    """Placed, non-overlapping busy intervals of one channel."""

    starts: list[int] = field(default_factory=list)
    ends: list[int] = field(default_factory=list)

    def add(self, start: int, end: int) -> None:
        self.starts.append(start)
        self.ends.append(end)

    def covers(self, t: int) -> bool:
        i = bisect_right(self.starts, t) - 1
        return i >= 0 and t < self.ends[i]


@dataclass
class EngineResult:
    timeline: dict[str, tuple[int, int]]
    stage_sequence: list[list[str]]


class _Sim:
    """One run of the event loop; state lives on the instance."""

    def __init__(self, tasks: dict[str, Task], n_stages: int, dur_of, comm: CommModel, selector):
        self.tasks, self.dur_of, self.comm, self.selector = tasks, dur_of, comm, selector
        self.waiting: dict[str, int] = {}          # compute/RECV task -> unmet deps
        self.send_waiting: dict[str, int] = {}
        self.consumers: dict[str, list[str]] = {tid: [] for tid in tasks}
        self.sends: dict[str, list[str]] = {tid: [] for tid in tasks}
        self.recv_for: dict[str, str] = {}
        for t in tasks.values():
            if t.kind == SEND:
                self.send_waiting[t.id] = len(t.deps)
                for d in t.deps:
                    self.sends[d].append(t.id)
            elif t.kind == RECV:
                self.recv_for[t.deps[0]] = t.id
            else:
                self.waiting[t.id] = len(t.deps)
                for d in t.deps:
                    self.consumers[d].append(t.id)
        for lst in self.sends.values():
            lst.sort()
        self.timeline: dict[str, tuple[int, int]] = {}
        self.sequence: list[list[str]] = [[] for _ in range(n_stages)]
        self.stage_free = [0] * n_stages
        self.out_free = [0] * n_stages
        self.in_free = [0] * n_stages
        self.out_busy = [_Intervals() for _ in range(n_stages)]
        self.in_busy = [_Intervals() for _ in range(n_stages)]
        self.ready: list[dict[str, int]] = [{} for _ in range(n_stages)]
        self.heap: list[tuple[int, int, str]] = []

    def _push(self, t: int, tag: int, key: str) -> None:
        heapq.heappush(self.heap, (t, tag, key))

    def _wake(self, t: int, stage: int) -> None:
        self._push(t, WAKE, f"{stage:06d}")

    def _on_finish(self, tid: str, t: int) -> None:
        for sid in self.sends[tid]:
            self.send_waiting[sid] -= 1
            if self.send_waiting[sid]:
                continue
            st = self.tasks[sid].stage
            start = max(self.out_free[st], t)
            end = start + self.comm.wire_time(self.tasks[sid].volume)
            self.out_free[st] = end
            self.out_busy[st].add(start, end)
            self.timeline[sid] = (start, end)
            self._push(start + self.comm.latency, ARRIVAL, self.recv_for[sid])
        for nid in self.consumers[tid]:
            self.waiting[nid] -= 1
            if not self.waiting[nid]:
                st = self.tasks[nid].stage
                self.ready[st][nid] = t
                self._wake(t, st)
        task = self.tasks[tid]
        if task.is_compute:
            self._wake(t, task.stage)

    def _on_arrival(self, rid: str, t: int) -> None:
        st = self.tasks[rid].stage
        start = max(self.in_free[st], t)
        end = start + self.comm.wire_time(self.tasks[rid].volume)
        self.in_free[st] = end
        self.in_busy[st].add(start, end)
        self.timeline[rid] = (start, end)
        self._push(end, FINISH, rid)

    def _on_wake(self, st: int, t: int) -> None:
        if self.stage_free[st] > t:
            return
        tid = self.selector.pick(st, self.ready[st], t)
        if tid is None:
            return
        d = self.dur_of(self.tasks[tid])
        if self.comm.slowdown != 1.0 and d > 0 and (
                self.out_busy[st].covers(t) or self.in_busy[st].covers(t)):
            d = int(round(d * self.comm.slowdown))
        self.timeline[tid] = (t, t + d)
        self.stage_free[st] = t + d
        self.sequence[st].append(tid)
        del self.ready[st][tid]
        self._push(t + d, FINISH, tid)

    def run(self) -> EngineResult:
        for tid, n in self.waiting.items():
            if n == 0:
                st = self.tasks[tid].stage
                self.ready[st][tid] = 0
                self._wake(0, st)
        while self.heap:
            t, tag, key = heapq.heappop(self.heap)
            if tag == FINISH:
                self._on_finish(key, t)
            elif tag == ARRIVAL:
                self._on_arrival(key, t)
            else:
                self._on_wake(int(key), t)
        if len(self.timeline) != len(self.tasks):
            missing = sorted(set(self.tasks) - set(self.timeline))
            detail = "; ".join(
                f"{tid} waiting on {[d for d in self.tasks[tid].deps if d not in self.timeline] or 'selector'}"
                for tid in missing[:6])
            raise DeadlockError(missing, detail)
        return EngineResult(self.timeline, self.sequence)


def execute(tasks: dict[str, Task], n_stages: int, dur_of, comm: CommModel,
            selector) -> EngineResult:
    return _Sim(tasks, n_stages, dur_of, comm, selector).run()


def replay(sched: Schedule, dur_of, comm: CommModel) -> EngineResult:
    return execute(sched.tasks, sched.n_stages, dur_of, comm,
                   ReplaySelector(sched.per_stage_order))

"""Executes a helix / 1F1B / ZB1P schedule on B200s.

Drop-in for ``pipelab.runtime.executor`` (``P/runtime/executor.py``):
``execute_schedule(sched, params, inputs, mlp_chunk=None, threaded=False)``
returns a :class:`RunResult` with the same fields, raising the same exception
classes (``ExecutionError`` / ``PayloadMismatch`` / ``StalledSchedule``).

Task semantics are the reference's (``executor.py:177-293``): FWD / BWD_B /
BWD_W / RECOMPUTE_FWD run component math (here :class:`LayerMath`, i.e.
libhx kernels); SEND moves the producer's payload after checking its element
count against both the task volume and ``costs.comm_volume`` (hard error);
RECV hands the payload to the consumer.  Gradients accumulate in fp32 device
buffers; losses accumulate as sum(z^2) in fp64 device slots.

Drivers
  replay        one process, one CUDA stream, every stage time-multiplexed on
                the current GPU, global dependency order exactly as the
                reference's replay loop (``executor.py:297-332``).
  multi-stream  ``threaded=True`` on one process: one CUDA stream per stage;
                SEND records an event on the producer stream, the consumer
                stream waits on it (the analogue of the reference's keyed
                channels, ``executor.py:334-382``).
  distributed   ``threaded=True`` under ``torch.distributed`` with world size
                == n_stages: rank r runs stage r on its own GPU; every SEND /
                RECV becomes a NCCL send / recv on a dedicated 2-rank
                communicator per *directed* stage pair, receives posted in the
                sender's issue order (no cross-direction FIFO deadlock, SURVEY
                H5).  Pure ordering edges between stages (two-fold pair edges)
                are not synchronised, as in the reference's threaded driver.
"""

from __future__ import annotations

import os
from collections import deque
from contextlib import nullcontext
from dataclasses import dataclass

import numpy as np
import torch

from ..costs import comm_volume
from ..generators import meta_config
from ..partition import post_stage, pre_stage
from ..schedule import BWD_B, BWD_W, FWD, RECOMPUTE, RECV, SEND, Schedule, Task
from .layers import LayerMath, Pending, payload_elements
from .model import (MATRIX_FIELDS, PARAM_FIELDS, POST_FIELDS, PRE_FIELDS, DeviceLayer,
                    LayerParams, layer_to_device)


class ExecutionError(Exception):
    pass


class PayloadMismatch(ExecutionError):
    """A transferred payload disagrees with the declared communication volume."""


class StalledSchedule(ExecutionError):
    """No stage can make progress (missing payload or unsatisfiable edge)."""


@dataclass
class RunResult:
    losses: list[float]
    param_grads: list[dict[str, np.ndarray]]
    peak_stash_elements: list[int]
    mode: str
    timeline: dict[str, tuple[float, float]] | None = None   # device ms, if recorded
    offload: dict | None = None    # host-offload statistics, when a stash budget was set


# Stash entries that exist only for the flash backward (never part of the
# reference's stash accounting, never sent between stages).
_LOCAL_EXTRAS = ("lse",)


def _logical_elements(entry: dict) -> int:
    # tensors, offloaded / pending placeholders; "_"-prefixed keys are regeneration
    # caches (layers.post_output), not stash entries of the reference
    return sum(int(t.numel()) for k, t in entry.items() if k not in _LOCAL_EXTRAS and k[0] != "_")


class _Stage:
    """Per-stage state.  ``ln_wctx_elements`` is T*h: each of the reference's
    deferred W contexts also holds two such tensors, the LayerNorm's normalised input and output
    gradient (``xhat2``/``d_ln2`` post, ``xhat1``/``d_ln1`` pre,
    ``P/runtime/layers.py:150-152``, ``:197``).  Here the LN gain/bias
    gradients are reduced in the B pass, so those tensors never exist, but
    ``peak_stash_elements`` counts them so the number matches the reference."""

    def __init__(self, idx: int, device, stream, ln_wctx_elements: int = 0):
        self.idx = idx
        self.device = device
        self.stream = stream
        self.values: dict[str, dict] = {}
        self.stash: dict[tuple[int, int, str], dict] = {}
        self.wctx: dict[int, list] = {}
        self.peak = 0
        self.ln_wctx_elements = ln_wctx_elements
        # device bytes of the distinct tensors held by stash, W contexts and
        # stage-local payloads (weights and inputs excluded), after each task:
        # checked against runtime/memplan.py
        self.peak_bytes = 0
        self.peak_bytes_at = ""
        self.resident_ptrs: set[int] = set()

    def held_bytes(self) -> int:
        seen: dict[int, int] = {}

        def visit(d):
            for v in d.values():
                if isinstance(v, torch.Tensor):
                    st = v.untyped_storage()
                    ptr = st.data_ptr()
                    if ptr not in self.resident_ptrs:
                        seen[ptr] = st.nbytes()

        for e in self.stash.values():
            visit(e)
        for e in self.values.values():
            visit(e)
        for lst in self.wctx.values():
            for _l, w_post, w_pre in lst:
                visit(w_post)
                visit(w_pre)
        return sum(seen.values())

    def bump(self, tid: str = "") -> None:
        n = sum(_logical_elements(e) for e in self.stash.values())
        for lst in self.wctx.values():
            for _l, w_post, w_pre in lst:
                n += _logical_elements(w_post) + _logical_elements(w_pre) + 4 * self.ln_wctx_elements
        self.peak = max(self.peak, n)
        nb = self.held_bytes()
        if nb > self.peak_bytes:
            self.peak_bytes, self.peak_bytes_at = nb, tid


def stage_fields(sched: Schedule, stage: int, layer: int) -> tuple[tuple[str, ...], tuple[str, ...]]:
    """(weights needed, gradient buffers owned) by ``stage`` for ``layer``."""
    cfg = meta_config(sched)
    chunked = any(t.comp == "chunk" for t in sched.tasks.values() if t.is_compute)
    if chunked:
        span = cfg.L // cfg.p
        mine = layer // span == stage
        return (PARAM_FIELDS, PARAM_FIELDS) if mine else ((), ())
    need: tuple[str, ...] = ()
    own: tuple[str, ...] = ()
    if pre_stage(layer, cfg) == stage:
        need += PRE_FIELDS
        own += PRE_FIELDS
    if post_stage(layer, cfg) == stage:
        need += POST_FIELDS
        own += POST_FIELDS
    return need, own


class DeviceModel:
    """Per-layer device weights + fp32 gradient buffers for a set of local stages."""

    def __init__(self, layers: dict[int, DeviceLayer]):
        self.layers = layers

    @staticmethod
    def from_host(sched: Schedule, params: list[LayerParams], stages, device) -> "DeviceModel":
        layers = {}
        for l, p in enumerate(params):
            need, own = set(), set()
            for st in stages:
                n, o = stage_fields(sched, st, l)
                need.update(n)
                own.update(o)
            if need:
                fields_ = tuple(f for f in PARAM_FIELDS if f in need)
                layers[l] = DeviceLayer(layer_to_device(p, device, fields_),
                                        tuple(f for f in PARAM_FIELDS if f in own))
        return DeviceModel(layers)

    def zero_grads(self, zero_fn) -> None:
        for dl in self.layers.values():
            dl.zero_grads(zero_fn)


_SIDE_STREAMS: dict[tuple, torch.cuda.Stream] = {}


def side_stream(device, role: str) -> torch.cuda.Stream:
    """One persistent CUDA stream per (device, role): per-stage compute streams,
    the receive stream, the input streamer's and the offloader's copy streams.
    The caching allocator keeps freed blocks per stream, so a fresh stream per
    call / iteration would miss its cache and cudaMalloc anew every time."""
    key = (str(torch.device(device)), role)
    st = _SIDE_STREAMS.get(key)
    if st is None:
        st = _SIDE_STREAMS[key] = torch.cuda.Stream(device=device)
    return st


class HostInput:
    """Stash placeholder for a micro-batch input (layer 0's x) that stays in
    host memory while the input streamer is active; counted like the tensor
    (``numel``) and copied back to the device by the task that reads it."""

    __slots__ = ("mb", "n")

    def __init__(self, mb: int, n: int):
        self.mb = mb
        self.n = n

    def numel(self) -> int:
        return self.n


class _InputStreamer:
    """Micro-batch inputs kept in (pinned) host memory and copied to the device
    just before the tasks that read them: layer 0's forward, and its recompute
    / backward (LayerNorm-1 backward needs x), on a side stream a few tasks
    ahead (``lookahead``) so the copy overlaps compute.  The device copy lives
    only as long as those tasks' payloads and stashes hold it, so a stage never
    keeps all m inputs resident (16 GB on stage 0 at 7B/128k)."""

    def __init__(self, sched: Schedule, stages: dict, host: list, device, lookahead: int = 3):
        self.host = host
        self.device = device
        self.cuda = device.type == "cuda"
        self.stream = side_stream(device, "inputs") if self.cuda else None
        self.lookahead = lookahead
        self.ready: dict[str, tuple] = {}
        self.uses: dict[int, list[tuple[int, str, int]]] = {}
        self.pos: dict[str, int] = {}
        for si in stages:
            seen_bwd: set[int] = set()
            lst = []
            for pos, tid in enumerate(sched.per_stage_order[si]):
                t = sched.tasks[tid]
                self.pos[tid] = pos
                if t.layer != 0 or t.kind not in (FWD, RECOMPUTE, BWD_B) or t.comp not in ("pre", "chunk"):
                    continue
                if t.kind == FWD:
                    lst.append((pos, tid, t.mb))
                elif t.mb not in seen_bwd:      # the first of rc.pre.l0 / b.pre.l0 (or the chunk bwd)
                    seen_bwd.add(t.mb)
                    lst.append((pos, tid, t.mb))
            self.uses[si] = lst
        self.h2d_bytes = 0

    def _issue(self, tid: str, mb: int) -> None:
        if tid in self.ready:
            return
        src = self.host[mb]
        if not self.cuda:
            self.ready[tid] = (src.clone(), None)
            return
        # allocated and filled on the side stream (its own allocator pool, so no
        # ordering against the compute stream is needed); the consumer waits on
        # the copy's event and takes the buffer over with record_stream
        with torch.cuda.stream(self.stream):
            dev = torch.empty(src.shape, dtype=src.dtype, device=self.device)
            dev.copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
        self.ready[tid] = (dev, ev)
        self.h2d_bytes += src.numel() * src.element_size()

    def before_task(self, si: int, tid: str) -> None:
        pos = self.pos.get(tid)
        if pos is None:
            return
        for p, use, mb in self.uses.get(si, ()):
            if pos <= p < pos + self.lookahead:
                self._issue(use, mb)

    def get(self, tid: str, mb: int) -> torch.Tensor:
        self._issue(tid, mb)
        dev, ev = self.ready.pop(tid)
        if ev is not None:
            cur = torch.cuda.current_stream(self.device)
            cur.wait_event(ev)
            dev.record_stream(cur)
        return dev


class _Core:
    """Task interpreter shared by the drivers (``executor.py:136-293``)."""

    def __init__(self, sched: Schedule, model: DeviceModel, math, stages: dict[int, _Stage],
                 sumsq: torch.Tensor | None):
        self.sched = sched
        self.tasks = sched.tasks
        self.cfg = meta_config(sched)
        self.qkv = bool(int(sched.meta.get("qkv", 0)))
        self.rc = bool(int(sched.meta.get("recompute", 0)))
        self.split = sched.meta.get("backward") == "split"
        self.model = model
        self.math = math
        self.stages = stages
        self.sumsq = sumsq
        self.offload = None   # StashOffloader (FILO host offload) or None
        # the pre stash drops x (l > 0); rc.pre(l) rebuilds it
        # from post(l-1)'s retention on the same stage (HelixRuntime.regen_pre_x)
        self.regen_pre_x = False
        self.inputs: list[torch.Tensor] = []
        self.streamer: _InputStreamer | None = None    # host-resident inputs (HelixRuntime.run)
        # LM mode (runtime/lm.py, paper §4.6): token inputs, embedding, loss-in-backward head
        self.lm = None
        self.tokens: list[torch.Tensor] = []
        self.labels: list[torch.Tensor] = []
        self.n_valid: list[int] = []
        self.loss_count: torch.Tensor | None = None
        self.recv_of_send = {t.deps[0]: t.id for t in self.tasks.values() if t.kind == RECV}
        self.sends_by_producer: dict[str, list[Task]] = {}
        for t in self.tasks.values():
            if t.kind == SEND:
                self.sends_by_producer.setdefault(t.deps[0], []).append(t)
        for lst in self.sends_by_producer.values():
            lst.sort(key=lambda t: t.id)

    # -- routing -------------------------------------------------------------------

    def input_id(self, t: Task) -> str | None:
        i, l = t.mb, t.layer
        if t.kind == FWD:
            if t.comp == "chunk":
                c = f"rv.fb.s{t.stage}.m{i}"
                return c if c in t.deps else None
            if t.comp == "pre":
                return f"f.post.l{l - 1}.m{i}" if l > 0 else None
            tag, comp = {"attn": ("pa", "pre"), "post": ("ap", "attn")}[t.comp]
            c = f"rv.{tag}.l{l}.m{i}"
            return c if c in t.deps else f"f.{comp}.l{l}.m{i}"
        if t.kind == BWD_B:
            if t.comp == "chunk":
                c = f"rv.gb.s{t.stage}.m{i}"
                return c if c in t.deps else None
            if t.comp == "post":
                return f"b.pre.l{l + 1}.m{i}" if l < self.cfg.L - 1 else None
            tag, comp = {"attn": ("gap", "post"), "pre": ("gpa", "attn")}[t.comp]
            c = f"rv.{tag}.l{l}.m{i}"
            return c if c in t.deps else f"b.{comp}.l{l}.m{i}"
        return None

    def take(self, st: _Stage, tid: str) -> dict:
        try:
            return st.values.pop(tid)
        except KeyError:
            raise StalledSchedule(f"stage {st.idx}: payload of {tid} not present") from None

    def store_stash(self, st: _Stage, l: int, mb: int, comp: str, full: dict, payload: dict) -> None:
        kept = self.math.reduce_stash(comp, full, payload) if self.rc else full
        if self.regen_pre_x and comp == "pre" and l > 0:
            kept = dict(kept)
            kept["x"] = Pending(int(kept["x"].numel()))
        st.stash[(l, mb, comp)] = kept
        if self.offload is not None:
            self.offload.after_store(st, (l, mb, comp))

    def W(self, l: int):
        return self.model.layers[l].w

    def G(self, l: int):
        return self.model.layers[l].grad

    # -- compute tasks ------------------------------------------------------------------

    def input_x(self, t: Task) -> torch.Tensor:
        """Layer 0's input for ``t``'s micro-batch (device tensor)."""
        if self.lm is not None:
            cfg = self.cfg
            x = torch.empty(cfg.s * cfg.b, cfg.h, dtype=torch.bfloat16, device=self.stages[t.stage].device)
            return self.lm.embed(self.tokens[t.mb], x)
        if self.streamer is not None:
            return self.streamer.get(t.id, t.mb)
        return self.inputs[t.mb]

    def _keep_x(self, stash: dict, mb: int) -> dict:
        """With streamed inputs the layer-0 pre stash keeps a host placeholder."""
        if self.streamer is not None and isinstance(stash.get("x"), torch.Tensor):
            stash = dict(stash)
            stash["x"] = HostInput(mb, int(stash["x"].numel()))
        return stash

    def _fetch_x(self, stash: dict | None, t: Task) -> None:
        if stash is not None and isinstance(stash.get("x"), HostInput):
            stash["x"] = self.streamer.get(t.id, t.mb)

    def run_compute(self, t: Task) -> None:
        st = self.stages[t.stage]
        if self.streamer is not None:
            self.streamer.before_task(t.stage, t.id)
        if self.offload is not None:
            self.offload.before_task(st, t)
        self._run_compute(st, t)
        if self.offload is not None:
            self.offload.after_task(st, t)
        st.bump(t.id)

    def _run_compute(self, st: _Stage, t: Task) -> None:
        if t.kind == FWD:
            (self._fwd_chunk if t.comp == "chunk" else self._fwd_component)(st, t)
        elif t.kind == BWD_B:
            (self._bwd_chunk if t.comp == "chunk" else self._bwd_component)(st, t)
        elif t.kind == BWD_W:
            for l, w_post, w_pre in st.wctx.pop(t.mb):
                self.math.post_backward_w(w_post, self.G(l))
                self.math.pre_backward_w(w_pre, self.G(l))
        elif t.kind == RECOMPUTE:
            key = (t.layer, t.mb, t.comp)
            if t.comp == "pre" and t.layer == 0:
                self._fetch_x(st.stash.get(key), t)
            if self.regen_pre_x and t.comp == "pre" and t.layer > 0:
                # post(l-1) runs on this stage (pre_stage(l) == post_stage(l-1),
                # P/partition.py:25-36) and its rc.post comes after this task
                # (P/generators.py:397-444), so its retention is still here
                kept_post = st.stash[(t.layer - 1, t.mb, "post")]
                x, cache = self.math.post_output(kept_post, self.W(t.layer - 1))
                kept_post.update(cache)
                st.stash[key]["x"] = x
            st.stash[key] = self.math.regenerate_stash(t.comp, st.stash[key],
                                                       self.W(t.layer) if t.layer in self.model.layers else None)
        else:
            raise ExecutionError(f"{t.id}: kind {t.kind} is not a compute task")

    def _loss(self, z: torch.Tensor, mb: int) -> torch.Tensor:
        if self.lm is not None:   # the head runs here, in the backward
            return self.lm.loss_backward(z, self.labels[mb], self.n_valid[mb], self.sumsq[mb:mb + 1],
                                         self.loss_count[mb:mb + 1])
        return self.math.loss(z, self.sumsq[mb:mb + 1])

    def _fwd_component(self, st: _Stage, t: Task) -> None:
        src = self.input_id(t)
        if t.comp == "pre":
            x = self.input_x(t) if src is None else self.take(st, src)["x"]
            payload, full = self.math.pre_forward(x, self.W(t.layer))
            if t.layer == 0:
                full = self._keep_x(full, t.mb)
            self.store_stash(st, t.layer, t.mb, "pre", full, {})
            st.values[t.id] = payload
        elif t.comp == "attn":
            payload = self.take(st, src)
            out, full = self.math.attn_forward(payload)
            self.store_stash(st, t.layer, t.mb, "attn", full, payload)
            st.values[t.id] = out
        else:
            payload = self.take(st, src)
            out, full = self.math.post_forward(payload, self.W(t.layer))
            self.store_stash(st, t.layer, t.mb, "post", full, payload)
            st.values[t.id] = {"x": out}

    def _bwd_component(self, st: _Stage, t: Task) -> None:
        src = self.input_id(t)
        l = t.layer
        if t.comp == "post":
            if src is None:
                z = self.take(st, f"f.post.l{l}.m{t.mb}")["x"]
                d_out = self._loss(z, t.mb)
            else:
                d_out = self.take(st, src)["d_x"]
            stash = st.stash.pop((l, t.mb, "post"))
            st.values[t.id] = self.math.post_backward(d_out, self.W(l), self.G(l), stash)
        elif t.comp == "attn":
            payload = self.take(st, src)
            stash = st.stash.pop((l, t.mb, "attn"))
            st.values[t.id] = self.math.attn_backward(payload, stash)
        else:
            payload = self.take(st, src)
            stash = st.stash.pop((l, t.mb, "pre"))
            self._fetch_x(stash, t)
            d_x = self.math.pre_backward(payload, self.W(l), self.G(l), stash)
            if l > 0:
                st.values[t.id] = {"d_x": d_x}
            elif self.lm is not None:
                self.lm.embed_backward(self.tokens[t.mb], d_x)

    def _fwd_chunk(self, st: _Stage, t: Task) -> None:
        src = self.input_id(t)
        x = self.input_x(t) if src is None else self.take(st, src)["x"]
        for l in range(t.layer, t.layer + t.span):
            pa, s_pre = self.math.pre_forward(x, self.W(l))
            if l == 0:
                s_pre = self._keep_x(s_pre, t.mb)
            self.store_stash(st, l, t.mb, "pre", s_pre, {})
            ap, s_attn = self.math.attn_forward(pa)
            self.store_stash(st, l, t.mb, "attn", s_attn, pa)
            x, s_post = self.math.post_forward(ap, self.W(l))
            self.store_stash(st, l, t.mb, "post", s_post, ap)
        st.values[t.id] = {"x": x}

    def _bwd_chunk(self, st: _Stage, t: Task) -> None:
        src = self.input_id(t)
        if src is None:
            d = self._loss(self.take(st, f"f.s{t.stage}.m{t.mb}")["x"], t.mb)
        else:
            d = self.take(st, src)["d_x"]
        deferred = []
        for l in range(t.layer + t.span - 1, t.layer - 1, -1):
            W, G = self.W(l), self.G(l)
            s_post = st.stash.pop((l, t.mb, "post"))
            s_attn = st.stash.pop((l, t.mb, "attn"))
            s_pre = st.stash.pop((l, t.mb, "pre"))
            if l == 0:
                self._fetch_x(s_pre, t)
            if self.rc:  # 1f1b_rc: regenerate this layer's non-attention stash in place
                s_post = self.math.regenerate_stash("post", s_post, W)
                s_pre = self.math.regenerate_stash("pre", s_pre, W)
            gap, w_post = self.math.post_backward_b(d, W, G, s_post, fuse_w=not self.split)
            gpa = self.math.attn_backward(gap, s_attn)
            d, w_pre = self.math.pre_backward_b(gpa, W, G, s_pre)
            if self.split:
                deferred.append((l, w_post, w_pre))
            else:
                self.math.post_backward_w(w_post, G)
                self.math.pre_backward_w(w_pre, G)
        if self.split:
            st.wctx[t.mb] = deferred
        if t.stage > 0:
            st.values[t.id] = {"d_x": d}
        elif self.lm is not None and t.layer == 0:
            self.lm.embed_backward(self.tokens[t.mb], d)

    # -- comm ---------------------------------------------------------------------

    def checked_payload(self, t: Task) -> dict:
        payload = self.take(self.stages[t.stage], t.deps[0])
        n = payload_elements(payload)
        declared = comm_volume(self.cfg, t.edge, self.qkv)
        if n != t.volume or n != declared:
            raise PayloadMismatch(
                f"{t.id}: payload carries {n} elements, task declares {t.volume}, "
                f"cost model expects {declared} for edge {t.edge!r}")
        return payload


# ======================================================================================
# drivers
# ======================================================================================


class _Timer:
    """Per-task CUDA-event timeline on each stage's stream."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        self.ev: dict[str, tuple[torch.cuda.Event, torch.cuda.Event]] = {}
        self.t0: torch.cuda.Event | None = None

    def start(self):
        if self.enabled:
            self.t0 = torch.cuda.Event(enable_timing=True)
            self.t0.record()

    def around(self, tid: str):
        timer = self

        class _Ctx:
            def __enter__(self_):
                if timer.enabled:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    timer.ev[tid] = (a, b)

            def __exit__(self_, *exc):
                if timer.enabled and exc[0] is None:
                    timer.ev[tid][1].record()

        return _Ctx()

    def collect(self) -> dict[str, tuple[float, float]] | None:
        if not self.enabled:
            return None
        torch.cuda.synchronize()
        return {tid: (self.t0.elapsed_time(a), self.t0.elapsed_time(b)) for tid, (a, b) in self.ev.items()}


def _replay(core: _Core, timer: _Timer) -> None:
    """Single-threaded global-order driver (``executor.py:297-332``)."""
    tasks, order = core.tasks, core.sched.per_stage_order
    done: set[str] = set()
    ptr = [0] * len(order)
    comm = sorted(tid for tid, t in tasks.items() if not t.is_compute)
    transit: dict[str, dict] = {}
    while len(done) < len(tasks):
        progressed = False
        for tid in comm:
            t = tasks[tid]
            if tid in done or not all(d in done for d in t.deps):
                continue
            if t.kind == SEND:
                transit[core.recv_of_send[tid]] = core.checked_payload(t)
            else:
                core.stages[t.stage].values[tid] = transit.pop(tid)
            done.add(tid)
            progressed = True
        for si, seq in enumerate(order):
            while ptr[si] < len(seq):
                t = tasks[seq[ptr[si]]]
                if not all(d in done for d in t.deps):
                    break
                with timer.around(t.id):
                    core.run_compute(t)
                done.add(t.id)
                ptr[si] += 1
                progressed = True
        if not progressed:
            blocked = {seq[ptr[si]]: [d for d in tasks[seq[ptr[si]]].deps if d not in done]
                       for si, seq in enumerate(order) if ptr[si] < len(seq)}
            raise StalledSchedule(f"schedule cannot progress; blocked on {blocked}")
    if transit:
        raise ExecutionError(f"undelivered payloads: {sorted(transit)}")




def _multistream(core: _Core, timer: _Timer) -> None:
    """One CUDA stream per stage on one GPU; host issues in replay order, the
    device overlaps stages.  Cross-stage payloads are ordered by events."""
    tasks, order = core.tasks, core.sched.per_stage_order
    main = torch.cuda.current_stream()
    streams = {si: side_stream(main.device, f"stage{si}") for si in core.stages}
    start = torch.cuda.Event()
    start.record(main)
    for s in streams.values():
        s.wait_event(start)
    done: set[str] = set()
    ptr = [0] * len(order)
    events: dict[str, torch.cuda.Event] = {}
    transit: dict[str, dict] = {}
    comm = sorted(tid for tid, t in tasks.items() if not t.is_compute)
    while len(done) < len(tasks):
        progressed = False
        for tid in comm:
            t = tasks[tid]
            if tid in done or not all(d in done for d in t.deps):
                continue
            if t.kind == SEND:
                with torch.cuda.stream(streams[t.stage]):
                    payload = core.checked_payload(t)
                    ev = torch.cuda.Event()
                    ev.record()
                rid = core.recv_of_send[tid]
                events[rid] = ev
                transit[rid] = payload
            else:
                dst = streams[t.stage]
                dst.wait_event(events.pop(tid))
                payload = transit.pop(tid)
                for tensor in payload.values():
                    tensor.record_stream(dst)
                core.stages[t.stage].values[tid] = payload
            done.add(tid)
            progressed = True
        for si, seq in enumerate(order):
            while ptr[si] < len(seq):
                t = tasks[seq[ptr[si]]]
                if not all(d in done for d in t.deps):
                    break
                with torch.cuda.stream(streams[si]), timer.around(t.id):
                    core.run_compute(t)
                done.add(t.id)
                ptr[si] += 1
                progressed = True
        if not progressed:
            raise StalledSchedule("schedule cannot progress (multi-stream)")
    for s in streams.values():
        end = torch.cuda.Event()
        end.record(s)
        main.wait_event(end)


# --- distributed -----------------------------------------------------------------------


def _payload_layout(cfg, edge_tag: str, qkv: bool, math=None) -> list[tuple[str, tuple, torch.dtype]]:
    """Tensor names/shapes/dtypes of each edge's payload (``layers.py`` dict keys)."""
    T, h = cfg.s * cfg.b, cfg.h
    bf = getattr(math, "act_dtype", torch.bfloat16)
    f32 = getattr(math, "wgrad_dtype", torch.float32)
    act = lambda n, w=h: (n, (T, w), bf)  # noqa: E731
    if edge_tag == "pa":
        return [act("ln_out"), act("residual"), ("qkv_weight", (h, 3 * h), bf)] if qkv \
            else [act("qkv", 3 * h), act("residual")]
    if edge_tag == "ap":
        return [act("attn_out"), act("residual")]
    if edge_tag == "gap":
        lay = [act("d_attn_out"), act("d_residual")]
        if getattr(math, "ships_delta", False):   # flash backward's D (layers.py docstring)
            lay.append(("delta", (cfg.b * cfg.num_heads * cfg.s,), torch.float32))
        return lay
    if edge_tag == "gpa":
        return [act("d_ln_out"), act("d_residual"), ("d_qkv_weight", (h, 3 * h), f32)] if qkv \
            else [act("d_qkv", 3 * h), act("d_residual")]
    if edge_tag == "fb":
        return [act("x")]
    if edge_tag == "gb":
        return [act("d_x")]
    raise ExecutionError(f"unknown edge tag {edge_tag!r}")


def _edge_tag(task_id: str) -> str:
    return task_id.split(".")[1]


class P2PPlan:
    """Send / receive issue order per directed stage pair.

    Rank r sends to q in the order its compute tasks run (per_stage_order[r],
    then each producer's SENDs sorted by id, ``executor.py:127-132``).  The
    receiver posts its RECVs from q in exactly that order, so FIFO matching on
    the (q -> r) communicator pairs every message with the right buffer.
    """

    def __init__(self, sched: Schedule):
        self.sched = sched
        sends_by_producer: dict[str, list[Task]] = {}
        recv_of_send = {}
        for t in sched.tasks.values():
            if t.kind == SEND:
                sends_by_producer.setdefault(t.deps[0], []).append(t)
            elif t.kind == RECV:
                recv_of_send[t.deps[0]] = t.id
        for lst in sends_by_producer.values():
            lst.sort(key=lambda t: t.id)
        n = sched.n_stages
        self.send_seq: dict[tuple[int, int], list[str]] = {}
        self.recv_seq: dict[tuple[int, int], list[str]] = {}
        for src in range(n):
            for tid in sched.per_stage_order[src]:
                for snd in sends_by_producer.get(tid, ()):
                    self.send_seq.setdefault((src, snd.peer), []).append(snd.id)
                    self.recv_seq.setdefault((src, snd.peer), []).append(recv_of_send[snd.id])
        self.pairs = sorted(self.send_seq)


class _SendQueue:
    """Outstanding sends to one peer, oldest first.

    A send's tensors are dropped as soon as its work reports completion
    (polled before every task), so a payload lives on the sender only until
    the receiver has taken it -- the reference's ownership rule, where a SEND
    moves the payload to the consumer (``executor.py:160-164``, ``:286``).
    ``cap`` bounds the number kept per peer: past it the oldest is waited on,
    which for NCCL only orders the launching stream after that send (the host
    never blocks); blocking backends (gloo) pass ``cap=None``.
    """

    def __init__(self, cap: int | None):
        self.cap = cap
        self.q: deque = deque()
        self.max_live = 0

    def push(self, works: list, tensors: list) -> None:
        self.q.append((works, tensors))
        if self.cap is not None:
            while len(self.q) > self.cap:
                for w in self.q.popleft()[0]:
                    w.wait()
        self.max_live = max(self.max_live, len(self.q))

    def prune(self) -> None:
        while self.q and all(w.is_completed() for w in self.q[0][0]):
            self.q.popleft()

    def drain(self) -> None:
        while self.q:
            for w in self.q.popleft()[0]:
                w.wait()

    def __len__(self) -> int:
        return len(self.q)


class _WqkvDedupe:
    """Receiver-side dedupe of the W_qkv copies in ``pa`` payloads.

    Every pre -> attention payload carries the layer's qkv weight
    (``P/costs.py:139-150``; 3h^2 bf16, 100 MB at h=4096), and the attention
    stash keeps it for the backward.  The weights do not change within an
    iteration, so all copies of one layer that a stage receives are equal: the
    first is kept (weakly referenced) and later payloads of that layer reuse
    it, freeing their buffers.  The wire contract (``comm_volume``) is
    unchanged; at 7B/128k p=8 a rank holds 32 instead of 64 copies (3.2 GB)."""

    def __init__(self):
        import weakref
        self.cache: "weakref.WeakValueDictionary[int, torch.Tensor]" = weakref.WeakValueDictionary()

    def dedupe(self, rid: str, payload: dict) -> dict:
        w = payload.get("qkv_weight")
        if w is None or _edge_tag(rid) != "pa":
            return payload
        layer = int(rid.split(".")[2][1:])
        prev = self.cache.get(layer)
        if prev is None:
            self.cache[layer] = w
        else:
            payload["qkv_weight"] = prev
        return payload


class _Distributed:
    """Rank r executes stage r; payloads move over NCCL (or gloo on CPU tests).

    Receives are posted ``recv_ahead`` compute tasks before their consumer, in
    the sender's issue order (``P2PPlan``).  On CUDA they are issued from a
    dedicated idle stream with buffers allocated on it: ProcessGroupNCCL
    orders a p2p op after the work already queued on the *issuing* stream, so
    a receive issued from the compute stream could not start before the
    compute queued ahead of it -- the transfer the two-fold order is meant to
    hide would serialise behind it.  The consumer's stream waits on the
    receive (``Work.wait``) and takes ownership (``record_stream``).  Sends
    are issued from the compute stream (they must follow their producer).
    """

    def __init__(self, core: _Core, rank: int, groups: dict, recv_ahead: int | None = None,
                 send_cap: int | None = -1, plan: "P2PPlan | None" = None):
        self.core = core
        self.rank = rank
        self.plan = plan if plan is not None else P2PPlan(core.sched)
        self.groups = groups
        st = core.stages[rank]
        self.cuda = st.device.type == "cuda"
        if recv_ahead is None:
            recv_ahead = int(os.environ.get("HX_RECV_AHEAD", "4"))
        self.recv_ahead = max(0, recv_ahead)
        if send_cap == -1:
            # default: bounded where waiting is non-blocking for the host (NCCL only
            # orders the stream); a blocking backend (gloo) bounds only when asked to
            env = os.environ.get("HX_SEND_CAP")
            send_cap = int(env) if env else (4 if self.cuda else None)
            if send_cap is not None and send_cap <= 0:
                send_cap = None
        self.sends: dict[int, _SendQueue] = {}
        self.send_cap = send_cap
        self.comm_stream = side_stream(st.device, "recv") if self.cuda else None
        self.wqkv = _WqkvDedupe()
        # gloo cannot move device memory: CUDA payloads are staged through host
        # buffers (lets several ranks share one GPU for testing; NCCL is direct)
        # (asked of a pair group this rank belongs to: from p = 3 on, the first
        # group in the dict may not include it, and get_backend rejects that)
        mine = [g for (a, b), g in (groups or {}).items() if rank in (a, b)]
        self.host_staging = self.cuda and torch.distributed.get_backend(mine[0] if mine else None) == "gloo"
        self.posted: dict[str, tuple[list, dict]] = {}    # rid -> (works, payload)
        self.next_recv: dict[int, int] = {}               # src -> index into recv_seq
        self.recv_index = {rid: (src, k) for (src, dst), seq in self.plan.recv_seq.items()
                           if dst == rank for k, rid in enumerate(seq)}
        order = core.sched.per_stage_order[rank]
        # per compute task, the RECVs (on this stage) that must have landed before it
        # runs; a RECV shared by a recompute task and its BWD_B lands once, for the first
        self.needs: list[list[str]] = []
        seen: set[str] = set()
        for tid in order:
            t = core.tasks[tid]
            need = [d for d in t.deps if d not in seen and (dt := core.tasks.get(d)) is not None
                    and dt.kind == RECV and dt.stage == rank]
            seen.update(need)
            self.needs.append(need)

    def _post_upto(self, src: int, want: int) -> None:
        """Post the receives from ``src`` up to index ``want`` of its sequence."""
        seq = self.plan.recv_seq[(src, self.rank)]
        core, cfg = self.core, self.core.cfg
        st = core.stages[self.rank]
        ctx = torch.cuda.stream(self.comm_stream) if self.cuda else nullcontext()
        with ctx:
            while self.next_recv.get(src, 0) <= want:
                k = self.next_recv.get(src, 0)
                r_id = seq[k]
                payload, works = {}, []
                for name, shape, dtype in _payload_layout(cfg, _edge_tag(r_id), core.qkv, core.math):
                    buf = torch.empty(shape, dtype=dtype, device="cpu" if self.host_staging else st.device)
                    payload[name] = buf
                    works.append(torch.distributed.irecv(buf, src=src, group=self.groups[(src, self.rank)]))
                self.posted[r_id] = (works, payload)
                self.next_recv[src] = k + 1

    def _post(self, rid: str) -> None:
        src, k = self.recv_index[rid]
        if k >= self.next_recv.get(src, 0):
            self._post_upto(src, k)

    def _receive(self, rid: str) -> dict:
        self._post(rid)
        works, payload = self.posted.pop(rid)
        for w in works:
            w.wait()        # NCCL: the current (compute) stream waits; gloo: blocks
        if self.host_staging:
            dev = self.core.stages[self.rank].device
            payload = {k: v.to(dev) for k, v in payload.items()}
        if self.cuda:
            cur = torch.cuda.current_stream()
            for t in payload.values():
                t.record_stream(cur)
        return self.wqkv.dedupe(rid, payload)

    def live_sends(self) -> int:
        return sum(len(q) for q in self.sends.values())

    def run(self, timer: _Timer) -> None:
        core, r = self.core, self.rank
        st = core.stages[r]
        order = core.sched.per_stage_order[r]
        for k, tid in enumerate(order):
            for j in range(k, min(len(order), k + 1 + self.recv_ahead)):
                for rid in self.needs[j]:
                    self._post(rid)
            for q in self.sends.values():
                q.prune()
            for d in self.needs[k]:
                st.values[d] = self._receive(d)
            t = core.tasks[tid]
            with timer.around(tid):
                core.run_compute(t)
            for snd in core.sends_by_producer.get(tid, ()):
                payload = core.checked_payload(snd)
                layout = _payload_layout(core.cfg, _edge_tag(snd.id), core.qkv, core.math)
                grp = self.groups[(r, snd.peer)]
                works, tensors = [], []
                for name, _shape, dtype in layout:
                    tensor = payload[name].contiguous()
                    if tensor.dtype != dtype:
                        raise PayloadMismatch(f"{snd.id}: {name} has dtype {tensor.dtype}, want {dtype}")
                    if self.host_staging:
                        tensor = tensor.cpu()
                    works.append(torch.distributed.isend(tensor, dst=snd.peer, group=grp))
                    tensors.append(tensor)
                q = self.sends.get(snd.peer)
                if q is None:
                    q = self.sends[snd.peer] = _SendQueue(self.send_cap)
                q.push(works, tensors)
                del payload, tensors
        for q in self.sends.values():
            q.drain()
        if self.posted:
            raise ExecutionError(f"undelivered payloads: {sorted(self.posted)}")

    @property
    def max_live_sends(self) -> dict[int, int]:
        return {peer: q.max_live for peer, q in self.sends.items()}


class _Loopback:
    """Stage probe: rank ``rank``'s tasks of a p-stage schedule alone on this
    GPU, with no peers.  Each RECV is satisfied just before its consumer by a
    freshly allocated payload of the wire layout (``_payload_layout``: the
    same buffers a real receive allocates), filled with synthetic values
    (N(0, 1) activations, N(0, 1e-3) gradients, N(0, 1/h) weights); each
    SEND's payload is checked against ``comm_volume`` and dropped (``send_cap``
    > 0 keeps that many per peer, the distributed driver's bound; how long a
    real send stays outstanding depends on its receiver, which the memory plan
    models on a timeline instead).  Compute runs the product kernels at the real per-stage shapes, so
    one B200 measures a rank's device memory and busy time for a p = 2..8
    pipeline it cannot otherwise host (memory plan validation)."""

    def __init__(self, core: _Core, rank: int, send_cap: int = 0, seed: int = 7):
        self.core = core
        self.rank = rank
        self.send_cap = send_cap
        st = core.stages[rank]
        self.gen = torch.Generator(device=st.device).manual_seed(seed)
        self.wqkv = _WqkvDedupe()
        order = core.sched.per_stage_order[rank]
        self.needs: list[list[str]] = []
        seen: set[str] = set()
        for tid in order:
            t = core.tasks[tid]
            need = [d for d in t.deps if d not in seen and (dt := core.tasks.get(d)) is not None
                    and dt.kind == RECV and dt.stage == rank]
            seen.update(need)
            self.needs.append(need)

    def _fake(self, rid: str) -> dict:
        core, cfg = self.core, self.core.cfg
        dev = core.stages[self.rank].device
        out = {}
        for name, shape, dtype in _payload_layout(cfg, _edge_tag(rid), core.qkv, core.math):
            buf = torch.empty(shape, dtype=dtype, device=dev)
            scale = (cfg.h ** -0.5) if name == "qkv_weight" else \
                (1e-3 if name.startswith("d_") or name == "delta" else 1.0)
            buf.normal_(0.0, scale, generator=self.gen)
            out[name] = buf
        return self.wqkv.dedupe(rid, out)

    def run(self, timer: _Timer) -> None:
        core, r = self.core, self.rank
        st = core.stages[r]
        inflight: dict[int, deque] = {}
        for k, tid in enumerate(core.sched.per_stage_order[r]):
            for d in self.needs[k]:
                st.values[d] = self._fake(d)
            with timer.around(tid):
                core.run_compute(core.tasks[tid])
            for snd in core.sends_by_producer.get(tid, ()):
                q = inflight.setdefault(snd.peer, deque())
                q.append(core.checked_payload(snd))
                while len(q) > self.send_cap:
                    q.popleft()


def make_pair_groups(n_stages: int, warm: bool = True, device=None) -> dict[tuple[int, int], object]:
    """One 2-rank group per directed stage pair; every rank must call this in
    the same order (``torch.distributed.new_group`` is collective).

    With ``warm`` each group's point-to-point communicator is created right
    away by one tiny send/recv, walking the groups in the same global order on
    every rank.  NCCL creates p2p communicators lazily and the creation blocks
    the host until the peer joins, so first touching pairs in rank-dependent
    order inside the schedule could deadlock two hosts; a single total order
    over all groups cannot."""
    groups = {}
    for a in range(n_stages):
        for b in range(n_stages):
            if a != b:
                groups[(a, b)] = torch.distributed.new_group([a, b])
    if warm:
        rank = torch.distributed.get_rank()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) \
                if torch.distributed.get_backend() == "nccl" else torch.device("cpu")
        token = torch.zeros(1, device=device)
        for (a, b), grp in groups.items():
            if rank == a:
                torch.distributed.send(token, dst=b, group=grp)
            elif rank == b:
                torch.distributed.recv(token, src=a, group=grp)
    return groups


_PAIR_GROUP_CACHE: list = []   # [(world process group, n_stages, groups)]


def pair_groups(n_stages: int) -> dict[tuple[int, int], object]:
    """``make_pair_groups`` once per (world process group, n_stages).

    ``execute_schedule`` is called once per iteration (``P/runtime/executor.py:425``);
    creating n(n-1) communicators on every call would leak NCCL communicators
    and pay their setup each step.  A re-initialised world (new default group
    object) gets fresh groups."""
    world = torch.distributed.group.WORLD
    for w, n, groups in _PAIR_GROUP_CACHE:
        if w is world and n == n_stages:
            return groups
    groups = make_pair_groups(n_stages)
    _PAIR_GROUP_CACHE[:] = [e for e in _PAIR_GROUP_CACHE if e[0] is world]
    _PAIR_GROUP_CACHE.append((world, n_stages, groups))
    return groups


# ======================================================================================
# public API
# ======================================================================================


class HelixRuntime:
    """Device-resident state for repeatedly executing one schedule.

    ``run(inputs)`` enqueues one full iteration (all micro-batches, forward and
    backward, gradient accumulation) without synchronising the host; the
    benchmark times it with CUDA events.  ``result()`` synchronises and
    returns a :class:`RunResult`.
    """

    def __init__(self, sched: Schedule, model: DeviceModel, mlp_chunk: int | None = None,
                 mode: str = "replay", device=None, math=None, rank: int | None = None,
                 groups: dict | None = None, record_timeline: bool = False,
                 stash_budget_bytes: int | None = None, offload_min_bytes: int = 32 << 20,
                 regen_pre_x: bool = False, stream_inputs: bool = False, lm=None, lm_params=None):
        self.sched = sched
        self.stream_inputs = stream_inputs
        self.cfg = meta_config(sched)
        self.mode = mode
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        qkv = bool(int(sched.meta.get("qkv", 0)))
        self.math = math if math is not None else LayerMath(
            self.cfg, qkv, mlp_chunk, self.device, recompute=bool(int(sched.meta.get("recompute", 0))),
            defer_w=sched.meta.get("backward") == "split")
        self.model = model
        self.rank = rank
        local = [rank] if mode in ("distributed", "probe") else list(range(sched.n_stages))
        ln_ctx = self.cfg.s * self.cfg.b * self.cfg.h
        self.stages = {si: _Stage(si, self.device, None, ln_ctx) for si in local}
        self.sumsq = torch.zeros(self.cfg.m, dtype=torch.float64, device=self.device)
        self.timeline = None
        self.core = _Core(sched, model, self.math, self.stages, self.sumsq)
        self.lm_spec = lm
        if lm is not None:
            self._setup_lm(lm, lm_params)
        if regen_pre_x:
            chunked = any(t.comp == "chunk" for t in sched.tasks.values() if t.is_compute)
            if not self.core.rc or chunked:
                raise ExecutionError("regen_pre_x needs a layer-wise schedule with recomputation "
                                     "(rc.pre tasks rebuild x)")
            self.core.regen_pre_x = True
        self.groups = groups
        self.record_timeline = record_timeline
        self.timeline = None
        self._plan = None
        self.comm_stats = None
        if mode == "distributed" and self.device.type == "cuda":
            # persistent GEMMs size their grids to the SMs left after this reserve, so
            # the NCCL p2p kernels that run next to them always find a free SM
            from . import _lib
            _lib.set_sm_reserve(int(os.environ.get("HX_SM_RESERVE", "8")))
        if stash_budget_bytes is not None:
            from .offload import StashOffloader
            weights = [w for dl in model.layers.values() for w in dl.w.values()]
            self.core.offload = StashOffloader(sched, self.stages, weights, stash_budget_bytes,
                                               min_bytes=offload_min_bytes, regen_pre_x=regen_pre_x)

    def _setup_lm(self, spec, params) -> None:
        """LM mode (runtime/lm.py): the tied word embedding is read by layer 0's
        pre (embedding) and by the loss task (head) -- both must run here."""
        from .lm import LMHead, LMParams
        cfg = self.cfg
        chunked = any(t.comp == "chunk" for t in self.sched.tasks.values() if t.is_compute)
        first = 0 if chunked else pre_stage(0, cfg)
        last = (self.sched.n_stages - 1) if chunked else post_stage(cfg.L - 1, cfg)
        if first != last:
            raise ExecutionError("LM head: the tied embedding's two uses are on stages "
                                 f"{first} and {last}; only schedules placing them together are supported")
        if first not in self.stages:
            return                           # this rank holds neither end
        if params is None:
            gen = torch.Generator(device=self.device).manual_seed(4321)
            params = LMParams(spec, cfg.h, cfg.s, self.device, gen)
        self.lm_params = params
        self.core.lm = LMHead(spec, params, cfg.s, cfg.b, cfg.h)
        self.core.loss_count = torch.zeros(cfg.m, dtype=torch.int32, device=self.device)

    def lm_grads(self) -> dict[str, torch.Tensor] | None:
        """fp32 gradients of the word (padded rows included) and position embeddings."""
        if self.core.lm is None:
            return None
        return {"w_emb": self.lm_params.d_emb, "w_pos": self.lm_params.d_pos}

    def run(self, inputs: list[torch.Tensor], labels: list[torch.Tensor] | None = None) -> None:
        """One iteration.  LM mode: ``inputs`` are token ids ``[s, b]`` per
        micro-batch and ``labels`` (default: the next token, last position
        ignored = -1) the targets."""
        cfg = self.cfg
        if len(inputs) != cfg.m:
            raise ExecutionError(f"need {cfg.m} input microbatches, got {len(inputs)}")
        if self.core.lm is not None:
            from .lm import default_labels
            T = cfg.s * cfg.b
            toks = [x.to(device=self.device, dtype=torch.int32).reshape(T).contiguous() for x in inputs]
            for x in toks:
                if int(x.min()) < 0 or int(x.max()) >= self.core.lm.spec.vocab:
                    raise ExecutionError("token id outside the vocabulary")
            labs = [default_labels(x, cfg.s, cfg.b) if labels is None else
                    labels[i].to(device=self.device, dtype=torch.int32).reshape(T).contiguous()
                    for i, x in enumerate(toks)]
            self.core.tokens, self.core.labels = toks, labs
            self.core.n_valid = [int((lb >= 0).sum()) for lb in labs]
            self.core.lm.p.zero_grads(self.math.zero_)
            self.math.zero_(self.core.loss_count)
            inputs = [None] * cfg.m
        elif self.lm_spec is not None:      # LM mode on a rank that holds neither end
            inputs = [None] * cfg.m
        # (a stage probe of a rank that never reads the inputs may pass None)
        self.core.inputs = [None if x is None else x.reshape(cfg.s * cfg.b, cfg.h) for x in inputs]
        # host inputs on a CUDA runtime (or stream_inputs): copied in per task, never all resident
        host = any(x is not None and x.device.type == "cpu" for x in self.core.inputs) and \
            self.device.type == "cuda"
        self.core.streamer = _InputStreamer(self.sched, self.stages, self.core.inputs, self.device) \
            if (host or self.stream_inputs) and self.core.lm is None else None
        if self.core.offload is not None and self.core.streamer is None:
            self.core.offload.exclude([x for x in self.core.inputs if x is not None])
        resident = {w.untyped_storage().data_ptr() for dl in self.model.layers.values() for w in dl.w.values()}
        if self.core.lm is not None:
            resident |= {self.lm_params.w_emb.untyped_storage().data_ptr(),
                         self.lm_params.w_pos.untyped_storage().data_ptr()}
        if self.core.streamer is None:
            resident |= {x.untyped_storage().data_ptr() for x in self.core.inputs if x is not None}
        for st in self.stages.values():
            st.peak = 0
            st.peak_bytes, st.peak_bytes_at = 0, ""
            st.resident_ptrs = resident
        self.model.zero_grads(self.math.zero_)
        self.math.zero_(self.sumsq)
        timer = _Timer(self.record_timeline)
        timer.start()
        if self.mode == "replay":
            _replay(self.core, timer)
        elif self.mode == "multistream":
            _multistream(self.core, timer)
        elif self.mode == "distributed":
            if self._plan is None:
                self._plan = P2PPlan(self.sched)
            drv = _Distributed(self.core, self.rank, self.groups, plan=self._plan)
            drv.run(timer)
            st = self.stages[self.rank]
            self.comm_stats = {"max_live_sends_per_peer": drv.max_live_sends,
                               "recv_ahead": drv.recv_ahead, "send_cap": drv.send_cap,
                               "stash_peak_bytes": st.peak_bytes, "stash_peak_at": st.peak_bytes_at}
        elif self.mode == "probe":
            _Loopback(self.core, self.rank).run(timer)
        else:
            raise ExecutionError(f"unknown mode {self.mode!r}")
        self.timeline = timer.collect()
        self._check_drained()

    def capture(self, inputs: list[torch.Tensor]) -> "GraphedIteration":
        """Capture one whole iteration (every launch of ``run``) into a CUDA
        graph, for launch-bound small shapes (BASELINE config 1: hundreds of
        tiny kernels per iteration, host-issue bound).  ``inputs`` must be
        device tensors; they become the graph's static input buffers.  Host
        offload, input streaming, LM mode and the distributed / probe drivers
        are not capturable (host-synchronising or data-dependent)."""
        if self.mode not in ("replay", "multistream") or self.core.offload is not None or \
                self.core.lm is not None or self.record_timeline:
            raise ExecutionError("capture needs replay / multistream mode without offload, LM mode or timeline")
        if any(x.device.type != "cuda" for x in inputs):
            raise ExecutionError("capture needs device-resident inputs")
        static = [x.reshape(self.cfg.s * self.cfg.b, self.cfg.h).clone() for x in inputs]
        self.run(static)                       # warm-up: lazy kernel attributes, allocator pools
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                self.run(static)
        torch.cuda.current_stream().wait_stream(side)
        return GraphedIteration(self, graph, static)

    def _check_drained(self) -> None:
        leftovers = sorted(tid for st in self.stages.values() for tid in st.values)
        if leftovers:
            raise ExecutionError(f"unconsumed payloads: {leftovers[:6]}")
        dirty = [st.idx for st in self.stages.values() if st.stash or st.wctx]
        if dirty:
            raise ExecutionError(f"stash not drained on stages {dirty}")

    def offload_stats(self) -> dict | None:
        off = self.core.offload
        if off is None:
            return None
        live = sum(len(e) for e in off.entries.values())
        return {**off.stats, "budget_bytes": off.budget, "live_entries": live}

    def loss_stage(self, mb: int) -> int:
        chunked = any(t.comp == "chunk" for t in self.sched.tasks.values() if t.is_compute)
        return 0 if chunked else post_stage(self.cfg.L - 1, self.cfg)

    def losses(self) -> list[float]:
        if self.core.lm is not None:   # mean next-token cross-entropy per micro-batch
            cnt = self.core.loss_count.cpu().tolist()
            return [float(v) / max(1, c) for v, c in zip(self.sumsq.cpu().tolist(), cnt)]
        n = self.cfg.s * self.cfg.b * self.cfg.h
        return [float(v) / n for v in self.sumsq.cpu().tolist()]

    def grads_numpy(self) -> dict[int, dict[str, np.ndarray]]:
        return {l: {k: g.double().cpu().numpy() for k, g in dl.grad.items()}
                for l, dl in self.model.layers.items()}


class GraphedIteration:
    """One captured ``HelixRuntime.run``: ``replay(inputs)`` copies new inputs
    into the static buffers and launches the whole iteration as one graph."""

    def __init__(self, rt: HelixRuntime, graph, static: list[torch.Tensor]):
        self.rt, self.graph, self.static = rt, graph, static

    def replay(self, inputs: list[torch.Tensor] | None = None) -> None:
        if inputs is not None:
            for dst, src in zip(self.static, inputs):
                dst.copy_(src.reshape(dst.shape), non_blocking=True)
        self.graph.replay()


def _to_device_inputs(inputs, cfg, device, stream: bool = False) -> list[torch.Tensor]:
    """bf16 ``[s*b, h]`` inputs: on ``device``, or (``stream``) in pinned host
    memory for the runtime's input streamer.  Input tensors already on the
    device stay there."""
    out = []
    for i, x in enumerate(inputs):
        shape = tuple(x.shape)
        if shape != (cfg.s, cfg.b, cfg.h):
            raise ExecutionError(f"input {i} has shape {shape}, want {(cfg.s, cfg.b, cfg.h)}")
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
        if stream and t.device.type == "cpu":
            out.append(t.to(dtype=torch.bfloat16).reshape(cfg.s * cfg.b, cfg.h).contiguous().pin_memory())
        else:
            out.append(t.to(device=device, dtype=torch.bfloat16).reshape(cfg.s * cfg.b, cfg.h).contiguous())
    return out


def execute_schedule(sched: Schedule, params: list[LayerParams], inputs: list,
                     mlp_chunk: int | None = None, threaded: bool = False,
                     record_timeline: bool = False, *, stash_budget_bytes: int | None = None,
                     offload_min_bytes: int = 32 << 20, regen_pre_x: bool = False,
                     stream_inputs: bool = True) -> RunResult:
    """Run ``sched`` numerically on the B200(s); same contract as the reference.

    ``threaded=False``: replay on the current GPU.  ``threaded=True``: one rank
    per stage when ``torch.distributed`` is initialised with world size ==
    n_stages (every rank calls this and gets the same, all-gathered result),
    otherwise one CUDA stream per stage on the current GPU.

    ``stash_budget_bytes`` (B200 extension): keep at most this many bytes of
    stashed activations per process on the device, FILO-offloading the rest to
    pinned host memory (``runtime/offload.py``); tensors smaller than
    ``offload_min_bytes`` always stay.

    ``regen_pre_x`` (B200 extension, rc schedules): the pre stash drops its
    ``x``; ``rc.pre(l)`` rebuilds it from ``post(l-1)``'s retention on the same
    stage, trading two MLP GEMMs per (layer, micro-batch)
    for ``b*s*h`` of stash.

    ``stream_inputs`` (default): host inputs (NumPy, as the reference passes
    them) stay in pinned host memory and are copied to the device per
    micro-batch right before layer 0's forward and backward; False copies all
    of them to the device up front.
    """
    cfg = meta_config(sched)
    if len(params) != cfg.L:
        raise ExecutionError(f"need {cfg.L} layer params, got {len(params)}")
    if len(inputs) != cfg.m:
        raise ExecutionError(f"need {cfg.m} input microbatches, got {len(inputs)}")
    if not torch.cuda.is_available():
        raise ExecutionError("execute_schedule needs a CUDA device (no CPU fallback)")
    device = torch.device("cuda", torch.cuda.current_device())
    dist = threaded and torch.distributed.is_available() and torch.distributed.is_initialized() \
        and torch.distributed.get_world_size() == sched.n_stages
    if dist:
        rank = torch.distributed.get_rank()
        model = DeviceModel.from_host(sched, params, [rank], device)
        rt = HelixRuntime(sched, model, mlp_chunk, "distributed", device, rank=rank,
                          groups=pair_groups(sched.n_stages), record_timeline=record_timeline,
                          stash_budget_bytes=stash_budget_bytes, offload_min_bytes=offload_min_bytes,
                          regen_pre_x=regen_pre_x)
    else:
        model = DeviceModel.from_host(sched, params, range(sched.n_stages), device)
        rt = HelixRuntime(sched, model, mlp_chunk, "multistream" if threaded else "replay", device,
                          record_timeline=record_timeline, stash_budget_bytes=stash_budget_bytes,
                          offload_min_bytes=offload_min_bytes, regen_pre_x=regen_pre_x)
    rt.run(_to_device_inputs(inputs, cfg, device, stream=stream_inputs))
    torch.cuda.synchronize()
    if dist:
        return _gather_distributed(rt, params)
    grads = rt.grads_numpy()
    losses = rt.losses()
    peaks = [rt.stages[i].peak for i in range(sched.n_stages)]
    return RunResult(losses, [grads[l] for l in range(cfg.L)], peaks, "threaded" if threaded else "replay",
                     rt.timeline, rt.offload_stats())


def _gather_distributed(rt: HelixRuntime, params) -> RunResult:
    """All ranks contribute their owned gradients, loss slots and peaks."""
    import torch.distributed as dist
    local = {"grads": rt.grads_numpy(), "sumsq": rt.sumsq.cpu().tolist(),
             "peak": rt.stages[rt.rank].peak, "rank": rt.rank, "timeline": rt.timeline,
             "offload": rt.offload_stats()}
    allv = [None] * dist.get_world_size()
    dist.all_gather_object(allv, local)
    cfg = rt.cfg
    n = cfg.s * cfg.b * cfg.h
    sumsq = np.zeros(cfg.m)
    grads: list[dict[str, np.ndarray]] = [{} for _ in range(cfg.L)]
    for part in allv:
        sumsq += np.array(part["sumsq"])
        for l, g in part["grads"].items():
            for k, v in g.items():
                if k in grads[l]:
                    raise ExecutionError(f"gradient site ({l}, {k}) recorded on two stages")
                grads[l][k] = v
    for l in range(cfg.L):
        missing = [k for k in PARAM_FIELDS if k not in grads[l]]
        if missing:
            raise ExecutionError(f"gradient sites missing: {[(l, k) for k in missing][:6]}")
    peaks = [p["peak"] for p in sorted(allv, key=lambda p: p["rank"])]
    tl = {}
    for part in allv:
        tl.update(part["timeline"] or {})
    offload = None
    if any(part["offload"] for part in allv):
        # per-rank statistics plus the byte totals across ranks
        per_rank = {part["rank"]: part["offload"] for part in allv}
        totals = {}
        for st in per_rank.values():
            for k, v in (st or {}).items():
                if isinstance(v, (int, float)) and not isinstance(v, bool):
                    totals[k] = totals.get(k, 0) + v
        offload = {"total": totals, "per_rank": per_rank}
    return RunResult(list(sumsq / n), grads, peaks, "threaded", tl or None, offload)

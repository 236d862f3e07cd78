"""FILO host offload of stashed activations.

Helix / 1F1B schedules keep a stash per (layer, micro-batch, component) from
its forward task until its backward (or recompute) task.  At long sequence
lengths the stash outgrows HBM (GPT-7B at s=128k keeps 3*b*s*h bf16 per layer
and micro-batch even with recomputation-without-attention: 206 GB for one
GPU's 64 layer-micro-batches).  This offloader keeps the device-resident stash
under a byte budget:

* eviction (at stash time): while resident bytes exceed the budget, the
  resident tensor whose next use is furthest away in this stage's task order
  (Belady; for FILO schedules the oldest stash) is copied device->host on a
  D2H stream into a pinned buffer and its device memory is released;
* prefetch (before every task): upcoming offloaded tensors, in consumption
  order, are copied back host->device on an H2D stream while they fit in the
  budget, so the copies overlap the compute of the tasks in between;
* use: a task that reads a stash waits (stream-ordered, no host sync) for its
  tensors' H2D events.

The unit is a tensor storage, not a stash entry: stash dictionaries share
tensors (the post stash's ``residual`` is the pre stash's ``x``, its
``attn_out`` is the attention stash's ``o``), and a shared tensor moves once.
Weights (e.g. the attention stash's ``qkv_weight`` reference) and small
tensors are never moved.  All copies are stream-ordered; PCIe traffic overlaps
compute in both directions (measured here: 55 GB/s each way, 83 GB/s both).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from ..schedule import BWD_B, RECOMPUTE


class _Offloaded:
    """Placeholder left in a stash dictionary while its tensor is on the host."""

    __slots__ = ("entry",)

    def __init__(self, entry):
        self.entry = entry

    def numel(self) -> int:  # stash accounting (peak_stash_elements) counts it as present
        return self.entry.numel


@dataclass
class _Entry:
    tensor: torch.Tensor | None          # device tensor while resident
    nbytes: int
    numel: int
    shape: tuple
    dtype: torch.dtype
    refs: set = field(default_factory=set)   # {(key, name)} stash slots holding it
    host: torch.Tensor | None = None     # pinned copy while offloaded
    d2h_done: torch.cuda.Event | None = None
    h2d_done: torch.cuda.Event | None = None
    incoming: torch.Tensor | None = None  # device tensor being prefetched


class StashOffloader:
    """Budgeted stash residency for the stages one process executes."""

    def __init__(self, sched, stages: dict, weights: list[torch.Tensor], budget_bytes: int,
                 min_bytes: int = 32 << 20, regen_pre_x: bool = False):
        self.regen_pre_x = regen_pre_x
        self.budget = int(budget_bytes)
        self.min_bytes = min_bytes
        self.weight_ptrs = {w.untyped_storage().data_ptr() for w in weights}
        from .executor import side_stream
        dev = torch.cuda.current_device()
        self.d2h = side_stream(dev, "offload_d2h")
        self.h2d = side_stream(dev, "offload_h2d")
        self.pool: dict[tuple, list[tuple[torch.Tensor, torch.cuda.Event | None]]] = {}
        # stage -> serial -> entry; resident tensors are found by object identity
        # (id(tensor) -> serial, validated with `is`): device addresses and ids are
        # reused after a tensor is freed, serials never are
        self.entries: dict[int, dict[int, _Entry]] = {si: {} for si in stages}
        self.by_obj: dict[int, int] = {}
        self.serial = 0
        self.excluded: set[int] = set()
        self.resident: dict[int, int] = {si: 0 for si in stages}
        self.cursor: dict[int, int] = {si: 0 for si in stages}
        self.stats = {"d2h_bytes": 0, "h2d_bytes": 0, "evictions": 0, "prefetches": 0}
        # consumption positions of every stash key in each stage's task order
        self.order: dict[int, list] = {}
        self.key_uses: dict[int, dict[tuple, list[int]]] = {}
        self.pos_of: dict[str, int] = {}
        for si in stages:
            seq = sched.per_stage_order[si]
            uses: dict[tuple, list[int]] = {}
            keys_at = []
            for pos, tid in enumerate(seq):
                t = sched.tasks[tid]
                ks = self.consumed_keys(t)
                keys_at.append(ks)
                for k in ks:
                    uses.setdefault(k, []).append(pos)
                self.pos_of[tid] = pos
            self.order[si] = keys_at
            self.key_uses[si] = uses

    # -- schedule knowledge ---------------------------------------------------------------

    def consumed_keys(self, t) -> list[tuple]:
        if t.kind == RECOMPUTE:
            if self.regen_pre_x and t.comp == "pre" and t.layer > 0:
                # rc.pre(l) rebuilds x from post(l-1)'s retention (executor regen_pre_x)
                return [(t.layer, t.mb, "pre"), (t.layer - 1, t.mb, "post")]
            return [(t.layer, t.mb, t.comp)]
        if t.kind == BWD_B:
            if t.comp == "chunk":
                return [(l, t.mb, c) for l in range(t.layer + t.span - 1, t.layer - 1, -1)
                        for c in ("post", "attn", "pre")]
            return [(t.layer, t.mb, t.comp)]
        return []

    def _next_use(self, si: int, e: _Entry) -> int:
        cur = self.cursor[si]
        best = 1 << 60
        for key, _name in e.refs:
            for p in self.key_uses[si].get(key, ()):
                if p >= cur:
                    best = min(best, p)
                    break
        return best

    # -- hooks called by the executor ------------------------------------------------------

    def exclude(self, tensors) -> None:
        """Storages owned by the caller (e.g. the iteration's inputs): never moved."""
        self.excluded = {t.untyped_storage().data_ptr() for t in tensors}

    def after_store(self, st, key: tuple) -> None:
        """A forward task stashed ``st.stash[key]``: track its tensors, evict over budget."""
        ents = self.entries[st.idx]
        for name, t in st.stash[key].items():
            if not isinstance(t, torch.Tensor) or not t.is_cuda:
                continue
            nbytes = t.numel() * t.element_size()
            ptr = t.untyped_storage().data_ptr()
            if nbytes < self.min_bytes or ptr in self.weight_ptrs or ptr in self.excluded:
                continue
            sn = self.by_obj.get(id(t))
            e = ents.get(sn) if sn is not None else None
            if e is None or e.tensor is not t:
                self.serial += 1
                sn = self.serial
                e = _Entry(t, nbytes, t.numel(), tuple(t.shape), t.dtype)
                ents[sn] = e
                self.by_obj[id(t)] = sn
                self.resident[st.idx] += nbytes
            e.refs.add((key, name))
        self._evict(st)

    def before_task(self, st, t) -> None:
        """Make the stash tensors ``t`` reads resident (stream waits), then prefetch."""
        si = st.idx
        self.cursor[si] = self.pos_of.get(t.id, self.cursor[si])
        cur = torch.cuda.current_stream()
        for key in self.consumed_keys(t):
            entry = st.stash.get(key)
            if entry is None:
                continue
            for name, v in list(entry.items()):
                if isinstance(v, _Offloaded):
                    self._fetch(st, v.entry, cur)
                    self._land(st, v.entry, cur)
        self._prefetch(st, cur)

    def after_task(self, st, t) -> None:
        """Forget stash slots the task consumed (popped or regenerated)."""
        si = st.idx
        keys = self.consumed_keys(t)
        if not keys:
            return
        ents = self.entries[si]
        for sid, e in list(ents.items()):
            drop = {(k, n) for (k, n) in e.refs if k in keys and
                    (k not in st.stash or not self._holds(st.stash[k].get(n), e))}
            if drop:
                e.refs -= drop
            if not e.refs:
                if e.tensor is not None or e.incoming is not None:
                    self.resident[si] -= e.nbytes
                if e.tensor is not None and self.by_obj.get(id(e.tensor)) == sid:
                    del self.by_obj[id(e.tensor)]
                self._release_host(e)
                del ents[sid]

    # -- mechanics ----------------------------------------------------------------------------

    @staticmethod
    def _holds(v, e: _Entry) -> bool:
        if isinstance(v, _Offloaded):
            return v.entry is e
        return isinstance(v, torch.Tensor) and e.tensor is not None and v is e.tensor

    def _host_buffer(self, e: _Entry) -> torch.Tensor:
        k = (e.shape, e.dtype)
        lst = self.pool.get(k)
        if lst:
            buf, ev = lst.pop()
            if ev is not None:
                self.d2h.wait_event(ev)
            return buf
        return torch.empty(e.shape, dtype=e.dtype, pin_memory=True)

    def _release_host(self, e: _Entry) -> None:
        if e.host is not None:
            self.pool.setdefault((e.shape, e.dtype), []).append((e.host, e.h2d_done))
            e.host = None

    def _evict(self, st) -> None:
        si = st.idx
        if self.resident[si] <= self.budget:
            return
        cur = torch.cuda.current_stream()
        ready = None
        cands = sorted((e for e in self.entries[si].values() if e.tensor is not None and e.incoming is None),
                       key=lambda e: -self._next_use(si, e))
        for e in cands:
            if self.resident[si] <= self.budget:
                break
            if ready is None:
                ready = torch.cuda.Event()
                ready.record(cur)
                self.d2h.wait_event(ready)
            if e.host is None:
                e.host = self._host_buffer(e)
                with torch.cuda.stream(self.d2h):
                    e.host.copy_(e.tensor, non_blocking=True)
                e.d2h_done = torch.cuda.Event()
                e.d2h_done.record(self.d2h)
                self.stats["d2h_bytes"] += e.nbytes
            e.tensor.record_stream(self.d2h)
            self.by_obj.pop(id(e.tensor), None)
            ph = _Offloaded(e)
            for key, name in e.refs:
                st.stash[key][name] = ph
            e.tensor = None
            self.resident[si] -= e.nbytes
            self.stats["evictions"] += 1

    def _fetch(self, st, e: _Entry, cur) -> None:
        """Start the H2D copy of an offloaded tensor (no-op if already under way)."""
        if e.tensor is not None or e.incoming is not None:
            return
        dev = torch.empty(e.shape, dtype=e.dtype, device=cur.device)
        alloc = torch.cuda.Event()
        alloc.record(cur)
        self.h2d.wait_event(alloc)
        if e.d2h_done is not None:
            self.h2d.wait_event(e.d2h_done)
        with torch.cuda.stream(self.h2d):
            dev.copy_(e.host, non_blocking=True)
        dev.record_stream(self.h2d)
        e.h2d_done = torch.cuda.Event()
        e.h2d_done.record(self.h2d)
        e.incoming = dev
        self.resident[st.idx] += e.nbytes
        self.stats["h2d_bytes"] += e.nbytes
        self.stats["prefetches"] += 1

    def _land(self, st, e: _Entry, cur) -> None:
        """The compute stream waits for the prefetch; the tensor returns to its stash slots."""
        if e.incoming is None:
            return
        cur.wait_event(e.h2d_done)
        e.tensor, e.incoming = e.incoming, None
        self.by_obj[id(e.tensor)] = next(sn for sn, x in self.entries[st.idx].items() if x is e)
        for key, name in e.refs:
            st.stash[key][name] = e.tensor
        # the host copy stays valid (the tensor is read-only from here on): a later
        # eviction of the same tensor needs no second D2H copy

    def _prefetch(self, st, cur, lookahead: int = 256) -> None:
        si = st.idx
        seq = self.order[si]
        seen = set()
        for pos in range(self.cursor[si], min(len(seq), self.cursor[si] + lookahead)):
            for key in seq[pos]:
                entry = st.stash.get(key)
                if entry is None:
                    continue
                for v in entry.values():
                    if isinstance(v, _Offloaded) and id(v.entry) not in seen:
                        e = v.entry
                        seen.add(id(e))
                        if self.resident[si] + e.nbytes > self.budget:
                            return
                        self._fetch(st, e, cur)
            if len(seen) > 64:
                return

    def resident_bytes(self) -> int:
        return sum(self.resident.values())

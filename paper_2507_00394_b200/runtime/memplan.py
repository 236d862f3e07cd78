"""Per-rank device-memory plan of one schedule iteration (B200 sizing; no
reference counterpart -- the reference only counts logical stash elements,
``P/runtime/executor.py:146-151`` / ``peak_stash_elements``).

One rank runs one stage.  Its HBM holds

* weights (bf16 matrices, fp32 LayerNorm vectors) of the components it owns
  and the fp32 gradient accumulators (``stage_fields``);
* the **stash**: walked task by task over ``per_stage_order`` with the
  runtime's actual tensors (``runtime/layers.py``), counting each distinct
  tensor once -- e.g. at p = 1 the post stash's ``residual`` *is* the pre
  stash's ``x``; a ``qkv_weight`` received from another stage is a copy, the
  local one is the weight itself;
* the largest per-task **workspace** (transients of one component call);
* **communication buffers**: receives posted ``recv_ahead`` tasks early and
  up to ``send_cap`` in-flight sends per peer (``executor._Distributed``).

``stash_walk`` is exact for the tensors it models and is checked against the
executor's own distinct-storage measurement (``_Stage.peak_bytes``) in
``tests/test_memplan_cpu.py``; workspace and comm terms are upper estimates.
``plan`` combines them and, for a device budget, says how much the FILO
offloader must move to host memory.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass

from ..config import ModelConfig
from ..partition import attn_stage, post_stage, pre_stage
from ..schedule import BWD_B, BWD_W, FWD, RECOMPUTE, RECV, Schedule
from .model import PARAM_FIELDS

GB = 1 << 30


@dataclass(frozen=True)
class Dtypes:
    act: int = 2        # activation / payload element (bf16)
    wgrad: int = 4      # fp32 gradient accumulators and the shipped d_qkv_weight
    weight: int = 2     # bf16 weight matrices
    lse: int = 4        # per-row softmax statistics kept by the attention stash (0: none)
    delta: int = 4      # flash D shipped in the gap payload (0: not shipped)
    slab_mlp: bool = True   # m1 / g regenerated per row slab (LayerMath); False: whole


@dataclass
class StagePlan:
    stage: int
    weights: int
    grads: int
    stash_peak: int
    stash_peak_at: str
    workspace: int
    comm: int
    inputs: int

    @property
    def total(self) -> int:
        return self.weights + self.grads + self.stash_peak + self.workspace + self.comm + self.inputs

    def as_gb(self) -> dict:
        d = {k: round(v / GB, 3) if isinstance(v, int) else v for k, v in asdict(self).items()}
        d["total"] = round(self.total / GB, 3)
        return d


def _cfg(sched: Schedule) -> ModelConfig:
    m = sched.meta
    return ModelConfig(L=int(m["L"]), h=int(m["h"]), s=int(m["s"]), b=int(m["b"]),
                       num_heads=int(m["heads"]), p=int(m["p"]), m=int(m["m"]))


def _is_chunked(sched: Schedule) -> bool:
    return any(t.comp == "chunk" for t in sched.tasks.values() if t.is_compute)


def stash_walk(sched: Schedule, stage: int, dt: Dtypes = Dtypes(), regen_pre_x: bool = False,
               with_trace: bool = False, stream_inputs: bool = False):
    """(peak bytes, task id at the peak[, per-task trace]) of the distinct
    tensors held on ``stage`` after each task: stash, deferred W contexts and
    stage-local payloads (produced, not yet consumed or sent).  With
    ``stream_inputs`` layer 0's x is a device copy of a host input (counted)
    that its pre stash does not keep (executor ``_InputStreamer``)."""
    cfg = _cfg(sched)
    qkv = bool(int(sched.meta.get("qkv", 0)))
    rc = bool(int(sched.meta.get("recompute", 0)))
    split = sched.meta.get("backward") == "split"
    chunked = _is_chunked(sched)
    T, h, A = cfg.s * cfg.b, cfg.h, dt.act
    act = T * h * A
    lse = cfg.b * cfg.num_heads * cfg.s * dt.lse

    sizes: dict[str, int] = {}
    refs: dict[str, int] = {}
    held: dict[tuple, list[str]] = {}

    def hold(key, idents):
        lst = held.setdefault(key, [])
        for ident, nbytes in idents:
            if nbytes <= 0:
                continue
            sizes[ident] = nbytes
            refs[ident] = refs.get(ident, 0) + 1
            lst.append(ident)

    def release(key):
        for ident in held.pop(key, ()):
            refs[ident] -= 1
            if refs[ident] == 0:
                del refs[ident], sizes[ident]

    def x_of(l, i):          # a layer input: the micro-batch input for l = 0 (resident, unless streamed)
        return (f"x:{l}.{i}", 0 if (l == 0 and not stream_inputs) else act)

    def stage_of(comp, l, i):
        if chunked:
            return stage
        return {"pre": pre_stage, "post": post_stage}[comp](l, cfg) if comp != "attn" else attn_stage(l, i, cfg)

    def local(ident, comp_from, l, i):
        """A tensor produced by another component: shared if it ran on this
        stage (same object), else the received copy (one per message)."""
        return ident if stage_of(comp_from, l, i) == stage else f"{ident}@rx"

    def fwd(comp, l, i):
        if comp == "pre":
            x = [] if ((rc and regen_pre_x and l > 0) or (stream_inputs and l == 0)) else [x_of(l, i)]
            if not qkv and not rc:
                x.append((f"ln:{l}.{i}", act))
            hold((l, i, "pre"), x)
        elif comp == "attn":
            t = []
            if qkv:
                t.append((local(f"ln:{l}.{i}", "pre", l, i), act))
                if not rc:
                    t.append((f"qkv:{l}.{i}", 3 * act))
                if stage_of("pre", l, i) != stage:   # received copy, one per layer (executor _WqkvDedupe)
                    t.append((f"wqkv:{l}@rx", 3 * h * h * A))
            else:
                t.append((local(f"qkv:{l}.{i}", "pre", l, i), 3 * act))
            t.append((f"lse:{l}.{i}", lse))
            hold((l, i, "attn"), t)
        else:
            o = (local(f"o:{l}.{i}", "attn", l, i), act)
            if rc:
                xid = x_of(l, i)[0]
                res = (xid if stage_of("pre", l, i) == stage else f"{xid}@rx", x_of(l, i)[1])
                if l == 0 and stage_of("pre", l, i) != stage:
                    res = (res[0], act)          # a received copy of the input
                hold((l, i, "post"), [o])
                hold((l, i, "post_res"), [res])   # dropped by rc.post (the trunk omits it)
            else:
                hold((l, i, "post"), [o, (f"x2:{l}.{i}", act), (f"ln2:{l}.{i}", act),
                                      (f"m1:{l}.{i}", 4 * act), (f"g:{l}.{i}", 4 * act)])

    def regen(comp, l, i):
        if comp == "pre":
            if stream_inputs and l == 0:
                hold((l, i, "pre"), [x_of(l, i)])
            if regen_pre_x and l > 0:
                hold((l, i, "pre"), [(f"x:{l}.{i}", act)])
                hold((l - 1, i, "post"), [(f"x2:{l - 1}.{i}", act), (f"ln2:{l - 1}.{i}", act)])
            if not qkv:
                hold((l, i, "pre"), [(f"ln:{l}.{i}", act)])
        else:
            release((l, i, "post_res"))
            hold((l, i, "post"), [(f"x2:{l}.{i}", act), (f"ln2:{l}.{i}", act)])
            if split or not dt.slab_mlp:
                hold((l, i, "post"), [(f"m1:{l}.{i}", 4 * act), (f"g:{l}.{i}", 4 * act)])

    def wctx(l, i):
        """Deferred W contexts of a split backward (zb1p): post {attn_out,
        d_o, ln2_out, d_m1, g, d_out}, pre {d_qkv_weight} or {ln_out, d_qkv}."""
        post = [(f"o:{l}.{i}", act), (f"dx2:{l}.{i}", act), (f"ln2:{l}.{i}", act),
                (f"dm1:{l}.{i}", 4 * act), (f"g:{l}.{i}", 4 * act), (f"dout:{l}.{i}", act)]
        pre = [(f"dwqkv:{l}.{i}", 3 * h * h * dt.wgrad)] if qkv else \
            [(f"ln:{l}.{i}", act), (f"dqkv:{l}.{i}", 3 * act)]
        return post + pre

    # --- stage-local payloads (the executor's ``values``): a task's output is
    # held from its end until its same-stage consumer runs, or -- if it is
    # sent -- only at its own end (the drivers pop it right after the task)
    L = cfg.L
    dlt = cfg.b * cfg.num_heads * cfg.s * dt.delta
    sent = {t.deps[0] for t in sched.tasks.values() if t.kind == "SEND"}
    deps_of = {tid: set(sched.tasks[tid].deps) for tid in sched.per_stage_order[stage]}

    def producer_of(t):
        """Mirror of executor._Core.input_id for a local producer (None: an
        input, a received payload, or nothing)."""
        l, i, d = t.layer, t.mb, deps_of[t.id]
        if t.comp == "chunk":
            if t.kind == BWD_B and f"rv.gb.s{t.stage}.m{i}" not in d:
                return f"f.s{t.stage}.m{i}"
            return None
        if t.kind == FWD:
            if t.comp == "pre":
                return f"f.post.l{l - 1}.m{i}" if l > 0 else None
            tag, comp = {"attn": ("pa", "pre"), "post": ("ap", "attn")}[t.comp]
            return None if f"rv.{tag}.l{l}.m{i}" in d else f"f.{comp}.l{l}.m{i}"
        if t.kind == BWD_B:
            if t.comp == "post":
                return f"b.pre.l{l + 1}.m{i}" if l < L - 1 else f"f.post.l{l}.m{i}"
            tag, comp = {"attn": ("gap", "post"), "pre": ("gpa", "attn")}[t.comp]
            return None if f"rv.{tag}.l{l}.m{i}" in d else f"b.{comp}.l{l}.m{i}"
        return None

    def output_of(t):
        l, i = t.layer, t.mb
        if t.comp == "chunk":
            if t.kind == FWD:
                e = l + t.span
                return [(f"x:{e}.{i}", act) if e < L else (f"z:{i}", act)]
            return [(f"dx:{l}.{i}", act)] if t.kind == BWD_B and t.stage > 0 else []
        if t.kind == FWD:
            if t.comp == "pre":
                first = (f"ln:{l}.{i}", act) if qkv else (f"qkv:{l}.{i}", 3 * act)
                return [first, x_of(l, i)]
            if t.comp == "attn":
                xid, xb = x_of(l, i)
                res = (xid, xb) if stage_of("pre", l, i) == stage else (f"{xid}@rx", act)
                return [(local(f"o:{l}.{i}", "attn", l, i), act), res]
            return [(f"x:{l + 1}.{i}", act) if l < L - 1 else (f"z:{i}", act)]
        if t.kind == BWD_B:
            if t.comp == "post":
                return [(f"dao:{l}.{i}", act), (f"dx2:{l}.{i}", act), (f"dlt:{l}.{i}", dlt)]
            if t.comp == "attn":
                res = (local(f"dx2:{l}.{i}", "post", l, i), act)
                if qkv:
                    return [(f"dln:{l}.{i}", act), res, (f"dwqkv:{l}.{i}", 3 * h * h * dt.wgrad)]
                return [(f"dqkv:{l}.{i}", 3 * act), res]
            return [(f"dx:{l}.{i}", act)] if l > 0 else []
        return []

    peak, at, trace = 0, "", []
    for tid in sched.per_stage_order[stage]:
        t = sched.tasks[tid]
        l, i = t.layer, t.mb
        if t.is_compute and t.kind in (FWD, BWD_B):
            src = producer_of(t)
            if src is not None:
                release(("v", src))
        if t.kind == FWD:
            if t.comp == "chunk":
                for ll in range(l, l + t.span):
                    for c in ("pre", "attn", "post"):
                        fwd(c, ll, i)
            else:
                fwd(t.comp, l, i)
        elif t.kind == RECOMPUTE:
            regen(t.comp, l, i)
        elif t.kind == BWD_B:
            if t.comp == "chunk":
                # (a chunk backward regenerates and frees layer by layer inside the
                # task: that transient is workspace, not stash)
                for ll in range(l + t.span - 1, l - 1, -1):
                    for c in ("post", "post_res", "attn", "pre"):
                        release((ll, i, c))
                    if split:
                        hold(("w", ll, i), wctx(ll, i))
            else:
                release((l, i, t.comp))
                if t.comp == "post":
                    release((l, i, "post_res"))
        elif t.kind == BWD_W:
            for key in [k for k in held if k[0] == "w" and k[2] == i]:
                release(key)
        hold(("v", tid), output_of(t))
        cur = sum(sizes.values())
        if with_trace:
            trace.append((tid, cur))
        if cur > peak:
            peak, at = cur, tid
        if tid in sent:
            release(("v", tid))
    return (peak, at, trace) if with_trace else (peak, at)


def _weight_bytes(sched: Schedule, stage: int, dt: Dtypes) -> tuple[int, int]:
    from .executor import stage_fields
    cfg = _cfg(sched)
    h = cfg.h
    shape = {"qkv_weight": 3 * h * h, "o_weight": h * h, "mlp_w1": 4 * h * h, "mlp_w2": 4 * h * h}
    w = g = 0
    for l in range(cfg.L):
        need, own = stage_fields(sched, stage, l)
        for f in need:
            w += shape[f] * dt.weight if f in shape else h * 4
        for f in own:
            g += shape.get(f, h) * dt.wgrad
    return w, g


def _workspace(sched: Schedule, mlp_chunk: int | None, dt: Dtypes) -> int:
    """Largest transient of one component call (layers.py), beyond the stash."""
    cfg = _cfg(sched)
    T, h, A = cfg.s * cfg.b, cfg.h, dt.act
    act = T * h * A
    qkv = bool(int(sched.meta.get("qkv", 0)))
    rc = bool(int(sched.meta.get("recompute", 0)))
    c = min(mlp_chunk or cfg.s, cfg.s) * cfg.b
    slab = c * 4 * h * A
    d_heads = cfg.b * cfg.num_heads * cfg.s * 4
    attn_fwd = (3 * act if qkv else 0) + act + d_heads
    attn_bwd = (3 * act if rc or not qkv else 0) + 3 * act + T * h * 4 + act + \
        (3 * h * h * dt.wgrad if qkv else 0) + d_heads
    post_fwd = 3 * act + (2 * slab if rc else 8 * act)
    post_bwd = 3 * act + d_heads + (3 * slab if rc else (slab + 4 * act))
    return max(attn_fwd, attn_bwd, post_fwd, post_bwd)


def _comm(sched: Schedule, stage: int, dt: Dtypes, recv_ahead: int, send_cap: int) -> int:
    from .executor import _edge_tag
    cfg = _cfg(sched)
    T, h, A = cfg.s * cfg.b, cfg.h, dt.act
    qkv = bool(int(sched.meta.get("qkv", 0)))

    def payload(tag):
        if tag == "pa":
            return 2 * T * h * A + 3 * h * h * A if qkv else 4 * T * h * A
        if tag == "gpa":
            return 2 * T * h * A + 3 * h * h * dt.wgrad if qkv else 4 * T * h * A
        if tag in ("ap", "gap"):
            return 2 * T * h * A
        return T * h * A

    order = sched.per_stage_order[stage]
    inbound = []
    for tid in order:
        t = sched.tasks[tid]
        inbound.append(sum(payload(_edge_tag(d)) for d in t.deps
                           if (dt_ := sched.tasks.get(d)) is not None and dt_.kind == RECV and dt_.stage == stage))
    recv = max((sum(inbound[k:k + 1 + recv_ahead]) for k in range(len(order))), default=0)
    out_sizes = [payload(_edge_tag(t.id)) for t in sched.tasks.values()
                 if t.kind == "SEND" and t.stage == stage]
    peers = {t.peer for t in sched.tasks.values() if t.kind == "SEND" and t.stage == stage}
    send = send_cap * len(peers) * max(out_sizes, default=0)
    return recv + min(send, sum(out_sizes))


def _payload_bytes(sched: Schedule, tid: str, dt: Dtypes) -> int:
    from .executor import _edge_tag
    cfg = _cfg(sched)
    T, h, A = cfg.s * cfg.b, cfg.h, dt.act
    qkv = bool(int(sched.meta.get("qkv", 0)))
    tag = _edge_tag(tid)
    if tag == "pa":
        return 2 * T * h * A + 3 * h * h * A if qkv else 4 * T * h * A
    if tag == "gpa":
        return 2 * T * h * A + 3 * h * h * dt.wgrad if qkv else 4 * T * h * A
    if tag == "gap":     # + the flash backward's D (layers.py)
        return 2 * T * h * A + cfg.b * cfg.num_heads * cfg.s * 4
    if tag == "ap":
        return 2 * T * h * A
    return T * h * A


def timeline_peak(sched: Schedule, stage: int, timeline: dict, dt: Dtypes = Dtypes(),
                  regen_pre_x: bool = False, recv_ahead: int = 4,
                  stream_inputs: bool = False) -> tuple[int, int, float]:
    """(stash + in-flight payload peak, its payload part, time) on a task
    timeline (simulated or measured).  The stash steps at each task's end
    (``stash_walk``).  A payload occupies its sender from the producer's end
    until the receiver posts the receive (``recv_ahead`` tasks before the
    consumer, ``executor._Distributed``) and its receiver from then until the
    consumer ends (after which the stash walk owns what is kept)."""
    _, _, trace = stash_walk(sched, stage, dt, regen_pre_x, with_trace=True, stream_inputs=stream_inputs)
    events: list[tuple[float, int, int]] = []    # (time, stash delta, payload delta)
    prev = 0
    for tid, level in trace:
        events.append((timeline[tid][1], level - prev, 0))
        prev = level
    pos = {tid: k for k, tid in enumerate(sched.per_stage_order[stage])}
    consumer = {}
    for t in sched.tasks.values():
        if t.is_compute:
            for d in t.deps:
                dt_ = sched.tasks.get(d)
                if dt_ is not None and dt_.kind == RECV:
                    c = consumer.get(d)
                    if c is None or timeline[t.id][0] < timeline[c][0]:
                        consumer[d] = t.id
    orders = sched.per_stage_order
    for r in sched.tasks.values():
        if r.kind != RECV or r.id not in consumer:
            continue
        snd = sched.tasks[r.deps[0]]
        src, dst = snd.stage, r.stage
        if stage not in (src, dst):
            continue
        produced = timeline[snd.deps[0]][1]
        cons = consumer[r.id]
        k = {tid: j for j, tid in enumerate(orders[dst])}[cons] if dst != stage else pos[cons]
        posted = max(produced, timeline[orders[dst][max(0, k - recv_ahead)]][0])
        nbytes = _payload_bytes(sched, snd.id, dt)
        if stage == src and posted > produced:
            events += [(produced, 0, nbytes), (posted, 0, -nbytes)]
        if stage == dst:
            events += [(posted, 0, nbytes), (timeline[cons][1], 0, -nbytes)]
    # frees before allocations at equal times
    events.sort(key=lambda e: (e[0], e[1] + e[2] > 0))
    st = pl = 0
    best = (0, 0, 0.0)
    for when, ds, dp in events:
        st += ds
        pl += dp
        if st + pl > best[0]:
            best = (st + pl, pl, when)
    return best


def plan(sched: Schedule, stage: int, mlp_chunk: int | None = None, dt: Dtypes = Dtypes(),
         regen_pre_x: bool = False, recv_ahead: int = 4, send_cap: int = 4,
         durations=None, stream_inputs: bool = False) -> StagePlan:
    """Per-rank plan.  With ``durations`` (a ``DurationTable``) the stash and
    the in-flight payloads are combined on the simulated timeline
    (``timeline_peak``); without, the comm term is the worst-case bound of
    ``recv_ahead`` posted receives plus ``send_cap`` sends per peer."""
    cfg = _cfg(sched)
    peak, at = stash_walk(sched, stage, dt, regen_pre_x, stream_inputs=stream_inputs)
    w, g = _weight_bytes(sched, stage, dt)
    if sched.n_stages == 1:
        comm = 0
    elif durations is not None:
        from ..simulate import simulate
        tl = simulate(sched, durations).timeline
        both, comm, when = timeline_peak(sched, stage, tl, dt, regen_pre_x, recv_ahead, stream_inputs)
        peak, at = both - comm, f"t={when:g}"
    else:
        comm = _comm(sched, stage, dt, recv_ahead, send_cap)
    # the micro-batch inputs are held by the stage that runs layer 0's pre
    first = 0 if _is_chunked(sched) else pre_stage(0, cfg)
    inputs = cfg.m * cfg.s * cfg.b * cfg.h * dt.act if (stage == first and not stream_inputs) else 0
    return StagePlan(stage, w, g, peak, at, _workspace(sched, mlp_chunk, dt), comm, inputs)


def offload_needed(p: StagePlan, hbm_bytes: int, reserve_bytes: int = 6 * GB) -> int:
    """Bytes of stash the FILO offloader must keep on the host at the peak so
    the rank fits ``hbm_bytes`` (minus a reserve for the CUDA context, NCCL
    and allocator fragmentation)."""
    return max(0, p.total - (hbm_bytes - reserve_bytes))

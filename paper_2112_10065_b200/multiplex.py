"""GPU multiplexing: a single-GPU background job packed under the
burst-parallel foreground on every GPU (BP+Col).

The reference models this with a discrete-event device
(`/root/reference/pkg/src/burstplan/simulator.py:451-819`); here the same
knobs drive real CUDA mechanisms, in one process per GPU so that stream
priorities arbitrate inside one CUDA context:

* priorities   -- the foreground runs on the highest-priority CUDA stream,
  the background on the lowest (``priority_scheduling_enabled``, :712-714);
* graph split  -- the background iteration is captured as CUDA graphs of at
  most ``graph_split_size`` ops each (the reference's launch groups,
  compile_timeline :280-294);
* pacing       -- at most ``launch_pace_limit`` background graphs are
  outstanding on the device at any time (0 = 64), tracked with CUDA events
  (try_submit :592-617); the foreground host runs at most one iteration
  ahead (:605-608);
* feedback     -- foreground ops whose collocated duration exceeds
  ``slowdown_ban_threshold`` x their isolated duration are flagged
  (feedback_update :896-911); a flagged op is captured as its own graph,
  waits for in-flight background graphs to drain and holds background
  submission until it finishes (eligible :685-700, refresh_sensitive
  :619-629).

Per-op durations come from CUDA events captured inside the foreground
graphs; iteration ends and background completions are event timestamps, so
``SimTrace`` / ``SimMetrics`` carry measured, not simulated, numbers.
"""

from __future__ import annotations

import time
from collections import deque
from dataclasses import replace
from typing import Iterable, Optional

import torch

from .comm import LocalComm
from .graph import CompGraph
from .network import net_for_graph, synthetic_batch
from .planner import TrainingPlan
from .timeline import FG_TASK, SimConfig, SimTrace, us_to_ticks


def op_name(step, key) -> str:
    """Stable name of a program op for traces and feedback flags:
    'compute:<layer>', 'transfer:<layer>', 'allreduce:g<g>', 'loss', 'sgd'."""
    kind, idx, _ = key
    if kind in ("compute", "transfer"):
        return f"{kind}:{step.layers[idx].spec.name}"
    if kind == "allreduce":
        return f"allreduce:g{idx}"
    return kind


def single_gpu_plan(graph: CompGraph, batch: int) -> tuple[TrainingPlan, CompGraph]:
    g = replace(graph, global_batch=batch)
    ids = [l.id for l in g.layers]
    plan = TrainingPlan(g.name, 1, float("inf"), batch, tuple((i, 1) for i in ids),
                        0.0, (), ())
    return plan, g


class BgJob:
    """The background job on one GPU: a full single-GPU training step of the
    network behind ``bg_graph`` at ``config.bg_batch_size``, captured as
    chunk graphs of <= ``graph_split_size`` program ops."""

    def __init__(self, bg_graph: CompGraph, config: SimConfig, seed: int = 1,
                 lr: float = 1e-3, sm_budget: Optional[int] = None):
        import os
        from . import ops
        from .executor import BurstStep
        plan, g = single_gpu_plan(bg_graph, config.bg_batch_size)
        self.batch = config.bg_batch_size
        self.step = BurstStep(plan, g, comm=LocalComm(), seed=seed, lr=lr)
        x, y = synthetic_batch(self.step.net, self.batch, seed)
        self.step.load(x, y)
        prog = self.step.program()
        cut = set(range(0, len(prog), config.graph_split_size))
        self.pool = torch.cuda.graph_pool_handle()
        # SM budget (B200 addition to the reference's knobs): the chunks are
        # captured with persistent grids and split-K sized to <= sm_budget
        # SMs, so the background's long-lived CTAs never occupy the whole
        # GPU and foreground kernels always find free SMs (the device
        # scheduler does not preempt running CTAs)
        if sm_budget is None:
            sm_budget = int(os.environ.get("BPX_BG_SM_BUDGET", "0"))
        self.sm_budget = sm_budget
        with ops.sm_budget(sm_budget):
            self.chunks = [gr for _, _, gr in self.step.capture_segments(cut, pool=self.pool)]
        self.n_ops = len(prog)


class Multiplexer:
    """Host loop of one GPU: foreground segments on the high-priority
    stream, background chunks on the low-priority stream."""

    def __init__(self, fg_step, bg: Optional[BgJob], config: SimConfig,
                 sensitive: Iterable[str] = (), measure_ops: bool = False,
                 fg_sm_budget: int = 0):
        self.fg = fg_step
        self.bg = bg
        self.cfg = config
        lo, hi = torch.cuda.Stream.priority_range()
        prio = config.priority_scheduling_enabled
        self.fg_stream = torch.cuda.Stream(priority=hi if prio else 0)
        self.bg_stream = torch.cuda.Stream(priority=lo if prio else 0)
        self.pace = config.launch_pace_limit or 64
        self.sensitive = frozenset(sensitive)
        self.measure = measure_ops
        prog = fg_step.program()
        names = [op_name(fg_step, k) for k, _ in prog]
        cut = set()
        for i, n in enumerate(names):
            if n in self.sensitive:
                cut |= {i, i + 1}
        fg_step.op_events = [] if measure_ops else None
        from . import ops
        with torch.cuda.stream(self.fg_stream), ops.sm_budget(fg_sm_budget):
            self.segments = fg_step.capture_segments(cut)
        self.events = fg_step.op_events or []
        fg_step.op_events = None
        self.flagged = [any(names[i] in self.sensitive for i in range(a, a + len(keys)))
                        for a, keys, _ in self.segments]

    def run(self, iterations: int, inputs=None, trace: Optional[SimTrace] = None,
            rank: int = 0, comm=None):
        """Run ``iterations`` foreground steps with the background packed
        underneath; returns the filled trace (ticks relative to the start)."""
        tr = trace or SimTrace()
        fg, bg = self.fg, self.bg
        ev0 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if comm is not None:
            comm.barrier()
        ev0.record(self.fg_stream)
        outstanding: deque = deque()         # (event, closes_iteration)
        bg_next = 0
        bg_iter = 0
        hold: Optional[torch.cuda.Event] = None      # flagged fg segment in flight
        fg_pending: deque = deque()          # (event, iteration, is_last_segment)
        seg_queue = [(it, j) for it in range(iterations) for j in range(len(self.segments))]
        qi = 0
        ends = []
        op_acc: dict[str, list] = {}
        # busy intervals of this GPU (measure_ops only: per-op CUDA events of
        # the foreground replays, start/end events of the background chunks);
        # the reference's utilisation is the union of per-op busy intervals
        busy: list = []
        bg_spans: list = []
        # Inputs arrive end to end every iteration, pipelined: the H2D copy of
        # iteration it+1 runs on a copy stream into a staging buffer while
        # iteration it computes; the step then takes it with one D2D copy.
        # Each iteration's loss is read back to pinned host memory.
        pairs = fg.input_pairs(*inputs) if inputs is not None else []
        staging = [torch.empty_like(d) for d, _ in pairs]
        copy_stream = torch.cuda.Stream()
        h2d_done: dict[int, torch.cuda.Event] = {}
        d2d_done: dict[int, torch.cuda.Event] = {}
        loss_host = torch.empty(2, dtype=torch.float32).pin_memory()

        def prefetch(it):
            if not pairs or it >= iterations:
                return
            with torch.cuda.stream(copy_stream):
                if it - 1 in d2d_done:
                    copy_stream.wait_event(d2d_done[it - 1])
                for buf, (_, src) in zip(staging, pairs):
                    buf.copy_(src, non_blocking=True)
                e = torch.cuda.Event()
                e.record(copy_stream)
                h2d_done[it] = e

        prefetch(0)

        def retire_bg():
            nonlocal bg_iter
            while outstanding and outstanding[0][0].query():
                e, closes = outstanding.popleft()
                if closes:
                    tr.bg_completions.append((_tick(ev0, e), rank))

        def submit_bg():
            nonlocal bg_next
            if bg is None:
                return
            while len(outstanding) < self.pace:
                if hold is not None and not hold.query():
                    return
                with torch.cuda.stream(self.bg_stream):
                    if hold is not None:
                        self.bg_stream.wait_event(hold)
                    s0 = None
                    if self.measure:
                        s0 = torch.cuda.Event(enable_timing=True)
                        s0.record(self.bg_stream)
                    bg.chunks[bg_next].replay()
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(self.bg_stream)
                closes = bg_next == len(bg.chunks) - 1
                outstanding.append((e, closes))
                if s0 is not None:
                    bg_spans.append((s0, e))
                bg_next = 0 if closes else bg_next + 1

        while qi < len(seg_queue) or fg_pending:
            # foreground: keep at most one iteration queued ahead
            while qi < len(seg_queue):
                it, j = seg_queue[qi]
                if fg_pending and fg_pending[0][1] < it - (0 if self.measure else 1):
                    break
                if pairs and j == 0:
                    with torch.cuda.stream(self.fg_stream):
                        self.fg_stream.wait_event(h2d_done[it])
                        for (dst, _), buf in zip(pairs, staging):
                            dst.copy_(buf, non_blocking=True)
                        e = torch.cuda.Event()
                        e.record(self.fg_stream)
                        d2d_done[it] = e
                    prefetch(it + 1)
                with torch.cuda.stream(self.fg_stream):
                    if self.flagged[j]:
                        for e, _ in outstanding:         # let queued bg drain first
                            self.fg_stream.wait_event(e)
                    self.segments[j][2].replay()
                    if j == len(self.segments) - 1:     # the step's result to the host
                        loss_host[it % 2].copy_(fg.loss_buf[0], non_blocking=True)
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(self.fg_stream)
                if self.flagged[j]:
                    hold = e
                fg_pending.append((e, it, j == len(self.segments) - 1))
                qi += 1
            retire_bg()
            submit_bg()
            while fg_pending and fg_pending[0][0].query():
                e, it, last = fg_pending.popleft()
                if last:
                    ends.append(e)
                    if self.measure:
                        _collect(fg, self.events, op_acc, ev0, busy)
            if hold is not None and hold.query():
                hold = None
            time.sleep(0)
        torch.cuda.synchronize()
        retire_bg()
        prev = 0
        for it, e in enumerate(ends):
            t = _tick(ev0, e)
            if comm is not None:
                t = int(comm.max_scalar(float(t), fg.device))
            tr.iteration_ticks.append(t)
            tr.events.append((t, rank, FG_TASK, f"iteration#{it}", "end"))
            prev = t
        tr.stop_tick = prev
        if self.measure:
            busy.extend((_tick(ev0, a), _tick(ev0, b)) for a, b in bg_spans)
            if comm is not None:
                for r, spans in enumerate(comm.allgather_object(busy)):
                    tr.busy.setdefault(r, []).extend(spans)
            else:
                tr.busy.setdefault(rank, []).extend(busy)
        for name, vals in op_acc.items():
            tr.op_durations.setdefault(name, []).extend(vals)
        tr.loss = float(fg.loss_buf[0].item())
        return tr


def _tick(ev0, e) -> int:
    return us_to_ticks(ev0.elapsed_time(e) * 1000.0)


def _collect(step, events, acc, ev0=None, busy=None) -> None:
    """Per-op durations (ms -> us) of the last completed foreground replay,
    fwd and bwd halves of an op summed (the reference's op granularity);
    with ``busy`` also the ops' (start, end) ticks relative to ``ev0``."""
    starts = {}
    per = {}
    for (key, what), ev in events:
        if what == "start":
            starts[key] = ev
        elif key in starts:
            name = op_name(step, key)
            per[name] = per.get(name, 0.0) + starts[key].elapsed_time(ev) * 1000.0
            if busy is not None:
                busy.append((_tick(ev0, starts[key]), _tick(ev0, ev)))
    for name, us in per.items():
        acc.setdefault(name, []).append(us)

"""Per-iteration op program, executor knobs, trace and metrics types.

Mirror of the executor-model types of
`/root/reference/pkg/src/burstplan/simulator.py` (SimConfig :72-91,
OpRecord :175-196, Timeline :199-208, compile_timeline :211-298,
SimTrace :305-323, SimMetrics :326-351, _metrics_from_trace :841-889,
feedback_update :896-911, forced_plan :918-942).  In the reference these feed
a discrete-event *model*; here ``compile_timeline``'s op program is what the
B200 executor (`executor.py`) runs for real, and ``SimTrace``/``SimMetrics``
are filled from CUDA-event timestamps instead of simulated ticks.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

from .costs import CostModel, LayerCost, make_context
from .errors import GraphFormatError
from .graph import CompGraph, ceil_div, comp_at_batch
from .planner import TrainingPlan

TICKS_PER_US = 10
FG_TASK = "fg"
HIGH = "high"
LOW = "low"


def us_to_ticks(us: float) -> int:
    return max(0, math.ceil(us * TICKS_PER_US))


def ticks_to_us(ticks: int) -> float:
    return ticks / TICKS_PER_US


@dataclass(frozen=True)
class SimConfig:
    """Executor knobs; field names and defaults follow the reference.

    On hardware: ``launch_pace_limit`` bounds outstanding background graph
    launches, ``graph_split_size`` is the number of background layers per
    captured CUDA graph, ``priority_scheduling_enabled`` selects
    high/low CUDA stream priorities, ``slowdown_ban_threshold`` drives the
    feedback loop.  ``contexts``/``stream_depth``/``launch_overhead_us`` only
    matter to the simulator and are kept for API compatibility.
    """

    launch_pace_limit: int = 2
    graph_split_size: int = 32
    bg_batch_size: int = 8
    slowdown_ban_threshold: float = 1.5
    priority_scheduling_enabled: bool = True
    rng_seed: int = 0
    contexts: int = 2
    stream_depth: int = 2
    launch_overhead_us: float = 5.0
    warmup_iterations: int = 1

    def __post_init__(self):
        if self.slowdown_ban_threshold <= 1:
            raise GraphFormatError("slowdown_ban_threshold must be > 1")
        if self.graph_split_size < 1:
            raise GraphFormatError("graph_split_size must be >= 1")
        if self.launch_pace_limit < 0 or self.contexts < 1 or self.stream_depth < 1:
            raise GraphFormatError("invalid simulator configuration")


def latency_bucket(duration_us: float) -> str:
    return "short" if duration_us < 100.0 else (
        "medium" if duration_us < 1000.0 else "long")


def op_class(kind: str, duration_us: float) -> str:
    return f"{'math' if kind == 'compute' else 'mem'}.{latency_bucket(duration_us)}"


@dataclass(frozen=True)
class OpRecord:
    op_id: str
    task_id: str
    kind: str                       # compute | allreduce | transfer
    isolated_duration_us: float
    stream_priority: str
    group_id: int
    participants: tuple[int, ...]
    barrier: bool
    payload_bytes: int = 0
    sensitive: bool = False

    @property
    def dur_ticks(self) -> int:
        return us_to_ticks(self.isolated_duration_us)

    @property
    def clazz(self) -> str:
        return op_class(self.kind, self.isolated_duration_us)


@dataclass(frozen=True)
class Timeline:
    n_gpus: int
    global_batch: int
    fg_ops: tuple[OpRecord, ...]
    bg_ops: tuple[OpRecord, ...]
    bg_batch: int
    predicted_fg_iteration_us: float


def compile_timeline(plan: TrainingPlan, graph: CompGraph, n_gpus: int,
                     bg_graph: Optional[CompGraph] = None,
                     config: Optional[SimConfig] = None) -> Timeline:
    """Plan -> op program: compute on [0, g); a transfer barrier over
    [0, max(g_prev, g)) at every scale change; one allreduce per
    parameterised layer with g > 1, in reverse layer order after compute;
    background template ops grouped by ``graph_split_size``."""
    config = config or SimConfig()
    peak = plan.max_gpus_used()
    if peak > n_gpus:
        raise GraphFormatError(
            f"plan uses {peak} GPUs but only {n_gpus} are simulated")
    cm = CostModel(make_context(graph, max(peak, 1),
                                candidates=sorted({g for _, g in plan.assignments} | {1})))
    ops: list[OpRecord] = []
    gid = 0
    seq = 0
    predicted = 0.0
    prev = None
    for lid, g in plan.assignments:
        layer = graph.layer(lid)
        if layer.is_virtual:
            continue
        if prev is not None:
            tr = cm.transfer(prev[0], lid, prev[1], g)
            if tr > 0:
                gid += 1
                ops.append(OpRecord(f"fg{seq:03d}.transfer.{layer.name}", FG_TASK,
                                    "transfer", tr, HIGH, gid,
                                    tuple(range(max(prev[1], g))), True, 0))
                seq += 1
            predicted += tr
        comp = cm.comp(lid, g)
        if comp > 0:
            ops.append(OpRecord(f"fg{seq:03d}.compute.{layer.name}", FG_TASK,
                                "compute", comp, HIGH, gid, tuple(range(g)),
                                False))
            seq += 1
        predicted += comp
        prev = (lid, g)
    for lid, g in reversed(plan.assignments):
        layer = graph.layer(lid)
        if layer.is_virtual or layer.params_bytes == 0:
            continue
        sync = cm.sync(lid, g)
        if sync > 0:
            gid += 1
            ops.append(OpRecord(f"fg{seq:03d}.allreduce.{layer.name}", FG_TASK,
                                "allreduce", sync, HIGH, gid, tuple(range(g)),
                                True, layer.params_bytes))
            seq += 1
        predicted += sync

    bg: list[OpRecord] = []
    if bg_graph is not None:
        for i, layer in enumerate(bg_graph.layers):
            if layer.is_virtual:
                continue
            dur = comp_at_batch(bg_graph, layer.id, config.bg_batch_size)
            if dur <= 0:
                continue
            bg.append(OpRecord(f"bg{i:03d}.compute.{layer.name}", "bg",
                               "compute", dur, LOW,
                               i // config.graph_split_size, (), False))
    return Timeline(n_gpus, graph.global_batch, tuple(ops), tuple(bg),
                    config.bg_batch_size, predicted)


# ---------------------------------------------------------------------------
# Trace / metrics


@dataclass
class SimTrace:
    """Event log in the reference schema: (tick, gpu, task, op, event) with
    ticks of 0.1 us.  The executor fills it from CUDA-event times."""

    events: list = field(default_factory=list)
    op_durations: dict = field(default_factory=dict)
    op_isolated: dict = field(default_factory=dict)
    iteration_ticks: list = field(default_factory=list)
    bg_completions: list = field(default_factory=list)
    busy: dict = field(default_factory=dict)
    stop_tick: int = 0

    def lines(self) -> list[str]:
        return ["tick\tgpu\ttask\top\tevent"] + [
            f"{t}\t{g}\t{task}\t{op}\t{kind}" for t, g, task, op, kind in self.events]

    def save(self, path: str) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("\n".join(self.lines()) + "\n")


@dataclass(frozen=True)
class SimMetrics:
    fg_iteration_time_us_mean: float
    fg_iteration_time_us_p99: float
    fg_throughput_samples_per_s: float
    bg_throughput_samples_per_s: float
    cluster_total_throughput_samples_per_s: float
    per_gpu_utilization: Optional[tuple[float, ...]]   # None: not measured
    qos_degradation: float

    def to_dict(self) -> dict:
        return {
            "fg_iteration_time_us_mean": self.fg_iteration_time_us_mean,
            "fg_iteration_time_us_p99": self.fg_iteration_time_us_p99,
            "fg_throughput_samples_per_s": self.fg_throughput_samples_per_s,
            "bg_throughput_samples_per_s": self.bg_throughput_samples_per_s,
            "cluster_total_throughput_samples_per_s":
                self.cluster_total_throughput_samples_per_s,
            "per_gpu_utilization": (None if self.per_gpu_utilization is None
                                    else list(self.per_gpu_utilization)),
            "qos_degradation": self.qos_degradation,
        }

    def save(self, path: str) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(self.to_dict(), fh, indent=1)
            fh.write("\n")


def percentile(sorted_vals: Sequence[float], q: float) -> float:
    """Ceil-rank percentile (reference :834-838)."""
    if not sorted_vals:
        return 0.0
    k = min(len(sorted_vals) - 1, max(0, math.ceil(q * len(sorted_vals)) - 1))
    return sorted_vals[k]


def metrics_from_trace(trace: SimTrace, n_gpus: int, global_batch: int,
                       bg_batch: int, config: SimConfig, iterations: int,
                       baseline_us: float) -> SimMetrics:
    """Same definitions as the reference (:841-889): warmup iterations are
    excluded; fg samples/s = B * iterations / window; bg samples/s counts
    background iterations completed inside the window; utilisation is the
    union of busy intervals."""
    warm = min(config.warmup_iterations, iterations - 1)
    bounds = [0] + list(trace.iteration_ticks)
    times = [ticks_to_us(b - a) for a, b in zip(bounds, bounds[1:])]
    meas = times[warm:]
    w0, w1 = bounds[warm], bounds[-1]
    wt = max(1, w1 - w0)
    ws = ticks_to_us(wt) / 1e6
    mean = sum(meas) / len(meas)
    fg = global_batch * len(meas) / ws
    bg_done = sum(1 for t, _ in trace.bg_completions if w0 < t <= w1)
    bg = bg_done * bg_batch / ws
    if not trace.busy:
        # no per-op intervals were recorded (run() without measure_ops):
        # utilisation is unknown rather than a fabricated number
        return SimMetrics(mean, percentile(sorted(meas), 0.99), fg, bg, fg + bg,
                          None, mean / baseline_us if baseline_us > 0 else 1.0)
    utils = []
    for gpu in range(n_gpus):
        covered, cur = 0, None
        for s, e in sorted(trace.busy.get(gpu, [])):
            s, e = max(s, w0), min(e, w1)
            if e <= s:
                continue
            if cur is None:
                cur = [s, e]
            elif s <= cur[1]:
                cur[1] = max(cur[1], e)
            else:
                covered += cur[1] - cur[0]
                cur = [s, e]
        if cur is not None:
            covered += cur[1] - cur[0]
        utils.append(covered / wt)
    return SimMetrics(mean, percentile(sorted(meas), 0.99), fg, bg, fg + bg,
                      tuple(utils), mean / baseline_us if baseline_us > 0 else 1.0)


def feedback_update(trace: SimTrace, config: SimConfig,
                    current: Iterable[str] = ()) -> frozenset:
    """Flag ops whose mean measured/isolated duration exceeds the ban
    threshold (isolated < 1 us ignored); union with ``current``."""
    flags = set(current)
    for key, meas in trace.op_durations.items():
        if not meas:
            continue
        iso = trace.op_isolated.get(key, 0.0)
        if iso < 1.0:
            continue
        if (sum(meas) / len(meas)) / iso > config.slowdown_ban_threshold:
            flags.add(key)
    return frozenset(flags)


def forced_plan(graph: CompGraph, g: int, total_gpus: int) -> TrainingPlan:
    """Uniform data parallelism: every real layer on g GPUs."""
    cm = CostModel(make_context(graph, max(g, 1), candidates=sorted({1, g})))
    assign, rows = [], []
    total = 0.0
    prev = None
    for lid in graph.topo_order():
        gi = 1 if graph.layer(lid).is_virtual else g
        tr = cm.transfer(prev, lid, g, gi) if prev is not None else 0.0
        cost = (tr + cm.comp(lid, gi)) + cm.sync(lid, gi)
        total += cost
        assign.append((lid, gi))
        rows.append(LayerCost(lid, gi, cm.comp(lid, gi), cm.sync(lid, gi),
                              cm.amp_of(lid, gi, cost)))
        prev = lid
    return TrainingPlan(graph.name, total_gpus, math.inf, graph.global_batch,
                        tuple(assign), total, tuple(rows), ())


def isolated_bg_iteration_us(bg_graph: CompGraph, config: SimConfig) -> float:
    total, n = 0.0, 0
    for layer in bg_graph.layers:
        if layer.is_virtual:
            continue
        total += comp_at_batch(bg_graph, layer.id, config.bg_batch_size)
        n += 1
    return max(total, ceil_div(n, config.graph_split_size) * config.launch_overhead_us)

"""Measured Pareto sweep: burst-parallel collocation operating points against
static cluster-partition baselines, on the GPUs instead of the simulator.

Mirrors the reference's ``pareto_sweep`` (simulator.py:984-1044): same
arguments, same plot-ready row schema (``PARETO_HEADER``), rows sorted by
label.  Every number is measured here:

* ``bp+col`` rows: for each amp limit, ``plan(graph, total_gpus, amp)``; for
  each config, ``run_two_phase`` (isolated pass, collocated pass with the
  background job, slowdown feedback, re-run) -- executor.py;
* ``partition k`` rows: the uniform plan ``forced_plan(graph, k, total)``
  runs the foreground alone on ranks [0, k) (simulator.py:1025-1029); the
  other ``total - k`` GPUs each train the background job alone, so their
  throughput is ``(total - k) * bg_batch / bg_iteration`` with the bg
  iteration measured in isolation on this GPU (the reference prices it with
  ``isolated_bg_iteration_us``, simulator.py:1033-1035);
* ``fg_speedup`` is relative to the measured one-GPU iteration of the same
  graph (the reference's ``iteration_time(graph, 1, B)``, :1007).

``interference`` is accepted for signature compatibility and ignored: on
hardware the interference is whatever the collocated kernels really do.
Launch one process per GPU (torchrun) for ``total_gpus > 1``; every rank
returns the same rows.
"""

from __future__ import annotations

from typing import Optional, Sequence

import torch

from .graph import CompGraph
from .timeline import SimConfig, forced_plan

PARETO_HEADER = ("label", "scenario", "amp_limit", "fg_speedup",
                 "fg_iteration_us", "cluster_throughput", "bg_throughput")


def measure_bg_iteration_us(bg_graph: CompGraph, config: SimConfig, reps: int = 10,
                            seed: int = 1) -> float:
    """Mean device time of one background training iteration alone on this
    GPU (all of its captured chunk graphs, back to back, CUDA events)."""
    from .multiplex import BgJob
    bg = BgJob(bg_graph, config, seed=seed)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for g in bg.chunks:            # warm-up iteration
            g.replay()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            for g in bg.chunks:
                g.replay()
        e1.record(s)
    s.synchronize()
    return 1000.0 * e0.elapsed_time(e1) / reps


def pareto_sweep(graph: CompGraph, total_gpus: int,
                 amp_limits: Sequence[float], configs: Sequence[SimConfig],
                 bg_graph: Optional[CompGraph] = None,
                 interference=None, iterations: int = 4,
                 partition_sizes: Sequence[int] = (1, 2, 4, 8),
                 feedback_rounds: int = 1) -> list[dict]:
    """Rows of PARETO_HEADER, sorted by label (simulator.py:1000-1044)."""
    from .executor import run, run_two_phase
    from .planner import plan as plan_fn

    del interference                   # real collocation, not a table
    bg_graph = bg_graph or graph
    one = forced_plan(graph, 1, total_gpus)
    _, m1 = run(one, graph, total_gpus, None, configs[0] if configs else SimConfig(),
                iterations)
    one_gpu_us = m1.fg_iteration_time_us_mean
    rows: list[dict] = []

    for amp_limit in amp_limits:
        p = plan_fn(graph, total_gpus, amp_limit)
        for cfg in configs:
            _, metrics, _ = run_two_phase(p, graph, total_gpus, bg_graph, cfg, iterations,
                                          feedback_rounds=feedback_rounds,
                                          baseline_fg_iteration_us=p.predicted_iteration_us)
            rows.append({
                "label": f"bp+col amp={amp_limit:g} pace={cfg.launch_pace_limit}"
                         f" bg={cfg.bg_batch_size}",
                "scenario": "bp+col",
                "amp_limit": amp_limit,
                "fg_speedup": one_gpu_us / metrics.fg_iteration_time_us_mean,
                "fg_iteration_us": metrics.fg_iteration_time_us_mean,
                "cluster_throughput": metrics.cluster_total_throughput_samples_per_s,
                "bg_throughput": metrics.bg_throughput_samples_per_s,
            })

    base_cfg = configs[0] if configs else SimConfig()
    bg_iter_us = None
    for k in partition_sizes:
        if k > total_gpus:
            continue
        p = forced_plan(graph, k, total_gpus)
        _, metrics = run(p, graph, total_gpus, None, base_cfg, iterations,
                         baseline_fg_iteration_us=p.predicted_iteration_us)
        fg_thr = metrics.fg_throughput_samples_per_s
        bg_thr = 0.0
        if bg_graph is not None and k < total_gpus:
            if bg_iter_us is None:
                bg_iter_us = measure_bg_iteration_us(bg_graph, base_cfg)
            bg_thr = (total_gpus - k) * base_cfg.bg_batch_size / (bg_iter_us / 1e6)
        rows.append({
            "label": f"partition k={k}",
            "scenario": "partition",
            "amp_limit": float("nan"),
            "fg_speedup": one_gpu_us / metrics.fg_iteration_time_us_mean,
            "fg_iteration_us": metrics.fg_iteration_time_us_mean,
            "cluster_throughput": fg_thr + bg_thr,
            "bg_throughput": bg_thr,
        })

    rows.sort(key=lambda r: r["label"])
    return rows


def pareto_to_table(rows: Sequence[dict]) -> str:
    """Tab-separated table in PARETO_HEADER order with the reference's
    number formats (simulator.py:1047-1055)."""
    out = ["\t".join(PARETO_HEADER)]
    for r in rows:
        out.append("\t".join((r["label"], r["scenario"], f"{r['amp_limit']:g}",
                              f"{r['fg_speedup']:.4f}", f"{r['fg_iteration_us']:.3f}",
                              f"{r['cluster_throughput']:.3f}",
                              f"{r['bg_throughput']:.3f}")))
    return "\n".join(out) + "\n"

"""B200 layer profiler: measured per-layer costs in the reference's profile
schema, so ``plan()`` plans against this GPU instead of the synthetic
A100-class knees (the paper's "performance monitor ->
planner" loop).

The reference's cost model reads ``comp(i, g)`` from a ``LayerProfile`` of
``{per_device_batch: (fwd_us, bwd_us)}`` entries (graph.py:49-57,
comp_at_batch graph.py:352-385; synth.py:29-30 profiles batches 2^0..2^17).
``profile_graph`` times every executable layer of ``net_for_graph(graph)``
through libbpx at the requested per-device batches -- fwd = the forward
op, bwd = weight gradient + data gradient (+ pool backward) -- and returns
the same ``CompGraph`` with measured profiles and a B200 ``NetworkProfile``.
Batches outside the measured range are clamped by the reference's own
lookup, exactly as for synthetic profiles.
"""

from __future__ import annotations

from typing import Callable, Iterable, Optional, Sequence

import torch

from .graph import CompGraph, LayerProfile, NetworkProfile, build_graph
from .network import LayerSpec, net_for_graph

# NVLink 5 peer copy measured on this pool's B200s (B200_PROFILING.md:
# "a peer copy of 770 GB/s per direction"); the launch + signal latency of a
# P2P reshard/allreduce step on NVSwitch is a few microseconds.
B200_NETWORK = NetworkProfile(per_gpu_bandwidth_bytes_per_sec=770e9,
                              propagation_delay_us=5.0)

DEFAULT_BATCHES = (1, 2, 4, 8, 16, 32)


def _layer_ops(spec: LayerSpec, b: int, first: bool, kernels, dev, ws):
    """(fwd_fn, bwd_fn) closures over freshly allocated buffers."""
    k = kernels
    g = torch.Generator(device="cpu").manual_seed(b)
    x = torch.relu(torch.randn(spec.in_shape(b), generator=g)).to(dev)
    y = torch.empty(spec.out_shape(b), device=dev)
    dy = torch.randn(spec.out_shape(b), generator=g).to(dev)
    dx = torch.empty_like(x)
    if spec.kind == "pool":
        return (lambda: k.maxpool2x2_fwd(x, y)), (lambda: k.maxpool2x2_bwd(x, dy, dx))
    wshape, bshape = spec.param_shapes()
    w = (torch.randn(wshape, generator=g) * 0.02).to(dev)
    bias = torch.zeros(bshape, device=dev)
    dw = torch.empty_like(w)
    db = torch.empty_like(bias)
    mask = x if spec.in_relu else None
    if spec.kind == "conv":
        def fwd():
            k.conv3x3_fwd(x, w, bias, y, relu=spec.relu, ws=ws)

        def bwd():
            k.conv3x3_wgrad(x, dy, dw, db, ws=ws)
            if not first:
                k.conv3x3_dgrad(dy, w, mask, dx, ws=ws)
        return fwd, bwd
    x2 = x.view(b, spec.cin)

    def fwd():
        k.linear_fwd(x2, w, bias, y, spec.relu, ws=ws)

    def bwd():
        k.linear_wgrad(x2, dy, dw, db, ws=ws)
        if not first:
            k.linear_dgrad(dy, w, None if mask is None else x2, dx.view(b, spec.cin), ws=ws)
    return fwd, bwd


def time_us(fn: Callable[[], None], reps: int = 5) -> float:
    """Mean device time of ``fn`` over ``reps`` back-to-back launches on the
    current stream (CUDA events, one warm-up call)."""
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 1000.0 * e0.elapsed_time(e1) / reps


def measure_layers(graph: CompGraph, batches: Sequence[int] = DEFAULT_BATCHES,
                   reps: int = 5, kernels=None,
                   timer: Callable[[Callable[[], None], int], float] = time_us
                   ) -> dict[str, dict[int, tuple[float, float]]]:
    """{layer name: {batch: (fwd_us, bwd_us)}} for every executable layer."""
    from . import ops
    k = kernels or ops
    net = net_for_graph(graph)
    dev = torch.device("cuda")
    ws = k.Workspace(dev)
    need = 0
    for spec in net.layers:
        for b in batches:
            if spec.kind == "conv":
                need = max(need, k.conv_workspace_bytes(b, spec.hw, spec.hw, spec.cin, spec.cout))
            elif spec.kind == "dense":
                need = max(need, k.linear_workspace_bytes(b, spec.cin, spec.cout))
    ws.reserve(need)
    out: dict[str, dict[int, tuple[float, float]]] = {}
    for i, spec in enumerate(net.layers):
        rows = {}
        for b in batches:
            fwd, bwd = _layer_ops(spec, b, i == 0, k, dev, ws)
            rows[b] = (timer(fwd, reps), timer(bwd, reps))
        out[spec.name] = rows
    return out


def graph_with_profiles(graph: CompGraph, measured: dict[str, dict[int, tuple[float, float]]],
                        network: Optional[NetworkProfile] = None,
                        name: Optional[str] = None) -> CompGraph:
    """The same graph (layers, ids, bytes) with measured profiles; virtual
    layers keep no profile, as in the reference (graph.py:200-214)."""
    profiles = {}
    for l in graph.layers:
        if l.is_virtual:
            continue
        rows = measured[l.name]
        profiles[l.id] = LayerProfile(l.id, {int(b): (float(f), float(w))
                                              for b, (f, w) in sorted(rows.items())})
    real = [l for l in graph.layers if not l.is_virtual]
    return build_graph(name or f"{graph.name}_b200", graph.global_batch, real, profiles,
                       network or B200_NETWORK, graph.input_shape)


def profile_graph(graph: CompGraph, batches: Iterable[int] = DEFAULT_BATCHES, reps: int = 5,
                  network: Optional[NetworkProfile] = None) -> CompGraph:
    """Measure ``graph``'s executable layers on the current B200 and return
    it with reference-schema profiles (save with ``graph.save_graph``)."""
    return graph_with_profiles(graph, measure_layers(graph, tuple(batches), reps), network)

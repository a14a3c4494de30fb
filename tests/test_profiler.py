"""B200 profiler -> reference profile schema -> planner.

CPU: measured rows (synthetic here) build a graph that round-trips through
the reference JSON schema and plans; the measured B200 network profile is
carried.  GPU: real measurement of VGG-16 at small batches."""

import json
import os

import pytest

from paper_2112_10065_b200 import synth
from paper_2112_10065_b200.graph import graph_from_dict, graph_to_dict
from paper_2112_10065_b200.planner import plan
from paper_2112_10065_b200.profiler import B200_NETWORK, graph_with_profiles
from paper_2112_10065_b200.timeline import forced_plan


def _fake_rows(g, batches=(1, 2, 4, 8, 16, 32)):
    rows = {}
    for l in g.layers:
        if l.is_virtual:
            continue
        base = 1.0 + (l.params_bytes + l.activation_bytes_per_sample) * 1e-6
        rows[l.name] = {b: (base * max(b, 4) / 4, 2 * base * max(b, 4) / 4) for b in batches}
    return rows


def test_profiled_graph_roundtrips_and_plans():
    g0 = synth.vgg_like(seed=0, global_batch=32)
    g = graph_with_profiles(g0, _fake_rows(g0))
    assert g.network == B200_NETWORK
    assert [l.name for l in g.layers] == [l.name for l in g0.layers]
    doc = json.loads(json.dumps(graph_to_dict(g)))
    g2 = graph_from_dict(doc)
    assert graph_to_dict(g2) == graph_to_dict(g)
    for G in (1, 2, 4, 8):
        p = plan(g2, G, 2.0)
        assert len(p.assignments) == len(g2.layers)
        dp = forced_plan(g2, G, G)
        assert p.predicted_iteration_us <= dp.predicted_iteration_us * (1 + 1e-12) or \
            p.fallback_layers


def test_profiled_graph_loads_in_the_reference():
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    import sys
    sys.path.insert(0, ref)
    try:
        import burstplan
        g0 = synth.vgg_like(seed=0, global_batch=32)
        g = graph_with_profiles(g0, _fake_rows(g0))
        gr = burstplan.graph.graph_from_dict(json.loads(json.dumps(graph_to_dict(g))))
        pr = burstplan.plan(gr, 8, 2.0)
        pm = plan(g, 8, 2.0)
        assert [n for _, n in pr.assignments] == [n for _, n in pm.assignments]
        assert pr.predicted_iteration_us == pm.predicted_iteration_us
    finally:
        sys.path.remove(ref)


@pytest.mark.gpu
def test_measure_vgg_layers_on_b200():
    from paper_2112_10065_b200.profiler import profile_graph
    g0 = synth.vgg_like(seed=0, global_batch=8)
    g = profile_graph(g0, batches=(1, 2), reps=2)
    for l in g.layers:
        e = g.profiles[l.id].entries
        assert set(e) == {1, 2}
        assert all(f > 0 and w > 0 for f, w in e.values())
    assert plan(g, 2, 2.0).predicted_iteration_us > 0

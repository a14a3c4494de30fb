"""Planner / cost-model / op-program parity against the reference.

Every expectation here was produced by the reference ``burstplan`` itself
(`oracle/gen_golden_plans.py`), and is compared with exact equality
(plan JSON byte-for-byte, floats bit-for-bit)."""

import hashlib
import json
import os

import pytest

from paper_2112_10065_b200 import synth
from paper_2112_10065_b200.costs import moved_samples, reshard_segments
from paper_2112_10065_b200.graph import graph_from_dict, graph_to_dict
from paper_2112_10065_b200.planner import plan, plan_to_json
from paper_2112_10065_b200.timeline import (SimConfig, compile_timeline,
                                            forced_plan)

from conftest import GOLDEN


def _load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


FAM = _load("families.json")


def _family(name, kwargs):
    return getattr(synth, name)(**kwargs)


def _sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


@pytest.mark.parametrize("name", sorted(FAM["families"]))
def test_family_profiles_byte_identical(name):
    meta = FAM["families"][name]
    g = _family(name, meta["kwargs"])
    text = json.dumps(graph_to_dict(g), indent=1) + "\n"
    assert _sha(text) == meta["graph_sha256"]


def test_vgg_golden_plan_sha_f2():
    g = synth.vgg_like(seed=0)
    p = plan(g, 8, 2.0)
    assert [gi for _, gi in p.assignments] == [8] * 10 + [4] * 4 + [1] * 7
    assert p.predicted_iteration_us == 6793.239412883865
    assert _sha(plan_to_json(p, g)) == FAM["families"]["vgg_like"]["plan_g8_amp2_sha256"]


@pytest.mark.parametrize("case", FAM["plans"],
                         ids=lambda c: f"{c['family']}-G{c['G']}-B{c['B']}-amp{c['amp']}")
def test_family_plans_exact(case):
    g = _family(case["family"], case["kwargs"])
    if case.get("forced"):
        p = forced_plan(g, case["G"], case["G"])
    else:
        p = plan(g, case["G"], case["amp"], global_batch=case["B"])
        if case["B"] != g.global_batch:
            from dataclasses import replace
            g = replace(g, global_batch=case["B"])
    assert plan_to_json(p, g) == case["plan_json"]


RND = _load("random_plans.json")["instances"]


@pytest.mark.parametrize("idx", range(len(RND)))
def test_random_instances_exact(idx):
    case = RND[idx]
    g = graph_from_dict(case["graph"])
    p = plan(g, case["G"], case["amp"], candidates=case["candidates"])
    assert plan_to_json(p) == case["plan_json"]


def test_moved_samples_table():
    for B, g, h, want in _load("moved_samples.json")["rows"]:
        assert moved_samples(B, g, h) == want, (B, g, h)


def test_reshard_segments_cover_batch_exactly():
    for B in range(1, 70):
        for g in range(1, 9):
            for h in range(1, 9):
                segs = reshard_segments(B, g, h)
                assert sum(n for *_, n in segs) == B
                pos = 0
                for p, q, s, n in segs:
                    assert s == pos and n > 0 and p < g and q < h
                    pos += n


def test_timeline_c1_matches_reference():
    want = _load("timeline_c1.json")
    g = synth.vgg_like(seed=0)
    tl = compile_timeline(plan(g, 8, 2.0), g, 8, synth.small_bg_model(),
                          SimConfig())
    got = lambda seq: [[o.op_id, o.kind, o.isolated_duration_us, o.group_id,
                        list(o.participants), o.barrier, o.payload_bytes,
                        o.stream_priority] for o in seq]
    assert got(tl.fg_ops) == want["fg"]
    assert got(tl.bg_ops) == want["bg"]
    assert tl.predicted_fg_iteration_us == want["predicted"]


BF = _load("brute_force_plans.json")["instances"]


@pytest.mark.parametrize("k", range(len(BF)))
def test_brute_force_plan_matches_reference_oracle(k):
    """brute_force_plan (the reference's exhaustive oracle, planner.py:592-682)
    reproduces the reference's own brute-force plan JSON on every small
    random instance, and agrees with the DP planner's optimum."""
    from paper_2112_10065_b200 import brute_force_plan
    case = BF[k]
    inst = RND[case["index"]]
    g = graph_from_dict(inst["graph"])
    bf = brute_force_plan(g, 4, inst["amp"], candidates=(1, 2, 4))
    assert plan_to_json(bf) == case["plan_json"]
    dp = plan(g, 4, inst["amp"], candidates=(1, 2, 4))
    if not dp.fallback_layers:
        assert bf.predicted_iteration_us == pytest.approx(dp.predicted_iteration_us, rel=1e-12)


def test_brute_force_plan_guards_large_instances():
    from paper_2112_10065_b200 import brute_force_plan
    from paper_2112_10065_b200.errors import InfeasiblePlanError
    with pytest.raises(InfeasiblePlanError):
        brute_force_plan(synth.vgg_like(seed=0), 8, 2.0)

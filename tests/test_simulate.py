"""Restated cluster simulation (paper_2112_10065_b200/simulate.py) against
the reference's own ``simulate`` / ``run_two_phase`` (simulator.py:451-977):
the same op programs give the same trace, bit for bit (event log digest,
iteration ticks, per-op durations) and the same metrics.  Fixtures from
oracle/gen_golden_sim.py; the op programs are rebuilt here with this
package's planner and compile_timeline (themselves pinned in
tests/test_planner_parity.py)."""

import hashlib
import json
import os

import pytest

from conftest import GOLDEN
from paper_2112_10065_b200 import synth
from paper_2112_10065_b200.planner import plan
from paper_2112_10065_b200.simulate import simulate, simulate_two_phase
from paper_2112_10065_b200.timeline import SimConfig, compile_timeline, forced_plan

with open(os.path.join(GOLDEN, "sim_cases.json")) as fh:
    CASES = json.load(fh)


def _digest(trace):
    lines = "\n".join(f"{t}\t{g}\t{task}\t{op}\t{k}" for t, g, task, op, k in trace.events)
    return hashlib.sha256(lines.encode()).hexdigest()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_simulation_matches_reference(case):
    g = getattr(synth, case["family"])(seed=0, **case["kwargs"])
    kind, arg = case["plan"]
    G = case["gpus"]
    p = plan(g, G, arg) if kind == "plan" else forced_plan(g, arg, G)
    bg = {"small": synth.small_bg_model(), "vgg": synth.vgg_like(seed=0, global_batch=8),
          None: None}[case["bg"]]
    cfg = SimConfig(**case["config"])
    tl = compile_timeline(p, g, G, bg, cfg)
    if case["two_phase"]:
        trace, m, flags = simulate_two_phase(tl, cfg, iterations=case["iterations"])
        assert sorted(flags) == case["flags"]
    else:
        trace, m = simulate(tl, cfg, iterations=case["iterations"],
                            sensitive=case["sensitive"])
    assert len(trace.events) == case["n_events"]
    assert list(trace.iteration_ticks) == case["iteration_ticks"]
    assert trace.stop_tick == case["stop_tick"]
    assert len(trace.bg_completions) == case["bg_completions"]
    assert _digest(trace) == case["trace_sha256"]
    assert hashlib.sha256(json.dumps(dict(sorted(trace.op_durations.items()))).encode()
                          ).hexdigest() == case["op_durations_sha256"]
    got = {k: (list(v) if isinstance(v, tuple) else v) for k, v in m.__dict__.items()}
    assert got == case["metrics"]

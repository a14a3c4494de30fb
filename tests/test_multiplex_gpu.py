"""GPU multiplexing (BP+Col) on one B200: foreground VGG-16 step on the
high-priority stream with the reference's default background job packed
underneath; the feedback loop measures per-op slowdowns."""

import pytest
import torch

from paper_2112_10065_b200 import synth
from paper_2112_10065_b200.executor import BurstStep, run, run_two_phase
from paper_2112_10065_b200.network import synthetic_batch
from paper_2112_10065_b200.planner import plan
from paper_2112_10065_b200.timeline import SimConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fg():
    g = synth.vgg_like(seed=0, global_batch=8)
    p = plan(g, 1, 2.0)
    st = BurstStep(p, g, seed=0, lr=0.0)
    x, y = synthetic_batch(st.net, 8, 0)
    return p, g, st, (x.pin_memory(), y.pin_memory())


@pytest.mark.timeout(600)
def test_collocated_run_keeps_fg_results_and_runs_bg(fg):
    p, g, st, inputs = fg
    cfg = SimConfig(warmup_iterations=1)
    tr0, m0 = run(p, g, 1, None, cfg, 4, inputs=inputs, step=st)
    loss_alone = tr0.loss
    tr1, m1 = run(p, g, 1, synth.small_bg_model(), cfg, 4, inputs=inputs, step=st)
    assert tr1.loss == loss_alone                   # lr=0: bg must not touch fg state
    assert len(tr1.bg_completions) > 0
    assert m1.bg_throughput_samples_per_s > 0
    assert m1.cluster_total_throughput_samples_per_s > m1.fg_throughput_samples_per_s
    assert len(tr1.iteration_ticks) == 4


@pytest.mark.timeout(600)
def test_two_phase_feedback_and_gated_rerun(fg):
    p, g, st, inputs = fg
    cfg = SimConfig(warmup_iterations=1, slowdown_ban_threshold=1.05)
    tr, m, flags = run_two_phase(p, g, 1, synth.small_bg_model(), cfg, iterations=3,
                                 inputs=inputs, step=st)
    assert isinstance(flags, frozenset)
    assert tr.op_isolated and all(v > 0 for v in tr.op_isolated.values())
    assert all(f.split(":")[0] in ("compute", "transfer", "allreduce", "loss", "sgd")
               for f in flags)
    assert m.fg_throughput_samples_per_s > 0 and len(tr.iteration_ticks) == 3

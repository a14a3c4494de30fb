"""Golden-fixture generator for the restated cluster simulation
(paper_2112_10065_b200/simulate.py).

TEST INFRASTRUCTURE ONLY (oracle/): imports the *reference* ``burstplan``
from /root/reference (read-only, present only in the build container), runs
its ``simulate`` (simulator.py:451-819) on a set of op programs and records
the outputs under tests/golden/sim_cases.json.  The product never imports
this module or the reference.  Re-run with

    python oracle/gen_golden_sim.py
"""

import hashlib
import json
import os
import sys

REF = "/root/reference/pkg"
sys.path[:0] = [f"{REF}/src"]
sys.dont_write_bytecode = True

from burstplan import synth                                          # noqa: E402
from burstplan.planner import plan                                  # noqa: E402
from burstplan.simulator import (SimConfig, compile_timeline, forced_plan,  # noqa: E402
                                 run_two_phase, simulate)

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden", "sim_cases.json")

# (name, family, kwargs, G, plan spec, bg, config kwargs, iterations, sensitive, two_phase)
CASES = [
    ("c1_bp_col", "vgg_like", {"global_batch": 32}, 8, ("plan", 2.0), "small", {}, 4, (), False),
    ("c1_bp_only", "vgg_like", {"global_batch": 32}, 8, ("plan", 2.0), None, {}, 4, (), False),
    ("c1_dp8", "vgg_like", {"global_batch": 32}, 8, ("forced", 8), None, {}, 3, (), False),
    ("c1_pace1_noprio", "vgg_like", {"global_batch": 32}, 4, ("plan", 2.0), "small",
     {"launch_pace_limit": 1, "priority_scheduling_enabled": False}, 3, (), False),
    ("c1_pace0_depth1", "vgg_like", {"global_batch": 64}, 2, ("plan", 2.0), "small",
     {"launch_pace_limit": 0, "stream_depth": 1, "contexts": 1}, 3, (), False),
    ("c1_sensitive", "vgg_like", {"global_batch": 32}, 8, ("plan", 2.0), "small", {}, 3,
     ("fg013.allreduce.conv3_3", "fg020.compute.conv5_1"), False),
    ("c1_two_phase", "vgg_like", {"global_batch": 32}, 8, ("plan", 2.0), "small", {}, 4, (),
     True),
    ("wrn_amp2", "wideresnet_like", {"global_batch": 32}, 8, ("plan", 2.0), "small", {}, 2, (),
     False),
    ("inception_g1", "inception_like", {"global_batch": 32}, 1, ("plan", 2.0), "vgg", {}, 3, (),
     False),
]


def digest(trace):
    lines = "\n".join(f"{t}\t{g}\t{task}\t{op}\t{k}" for t, g, task, op, k in trace.events)
    return hashlib.sha256(lines.encode()).hexdigest()


def main():
    out = []
    for name, fam, kw, G, spec, bg, ckw, iters, sens, two in CASES:
        g = getattr(synth, fam)(seed=0, **kw)
        p = plan(g, G, spec[1]) if spec[0] == "plan" else forced_plan(g, spec[1], G)
        bgg = {"small": synth.small_bg_model(), "vgg": synth.vgg_like(seed=0, global_batch=8),
               None: None}[bg]
        cfg = SimConfig(**ckw)
        tl = compile_timeline(p, g, G, bgg, cfg)
        if two:
            trace, m, flags = run_two_phase(tl, cfg, iterations=iters)
            flags = sorted(flags)
        else:
            trace, m = simulate(tl, cfg, iterations=iters, sensitive=sens)
            flags = None
        out.append({
            "name": name, "family": fam, "kwargs": kw, "gpus": G, "plan": list(spec),
            "bg": bg, "config": ckw, "iterations": iters, "sensitive": list(sens),
            "two_phase": two, "flags": flags,
            "metrics": {k: (list(v) if isinstance(v, tuple) else v)
                        for k, v in m.__dict__.items()},
            "n_events": len(trace.events), "trace_sha256": digest(trace),
            "iteration_ticks": list(trace.iteration_ticks),
            "bg_completions": len(trace.bg_completions), "stop_tick": trace.stop_tick,
            "op_durations_sha256": hashlib.sha256(json.dumps(
                {k: v for k, v in sorted(trace.op_durations.items())}).encode()).hexdigest(),
        })
        print(name, len(trace.events), m.fg_iteration_time_us_mean, flush=True)
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=1)
        fh.write("\n")


if __name__ == "__main__":
    main()

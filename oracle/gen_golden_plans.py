"""Golden-fixture generator for planner / cost-model / timeline parity.

TEST INFRASTRUCTURE ONLY (oracle/): imports the *reference* ``burstplan``
package from /root/reference (read-only, present only in the build
container) and records its outputs under tests/golden/.  The product never
imports this module or the reference.  Re-run with

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python oracle/gen_golden_plans.py

Generators reused from the reference test-suite:
`/root/reference/pkg/tests/conftest.py:46-142` (random_chain_graph,
random_sp_graph); acceptance seeds 1001/2002
(`/root/reference/pkg/tests/test_acceptance.py:33-69`).
"""

import hashlib
import json
import os
import random
import sys

REF = "/root/reference/pkg"
sys.path[:0] = [f"{REF}/src", f"{REF}/tests"]
sys.dont_write_bytecode = True

from burstplan import synth                                   # noqa: E402
from burstplan.costs import moved_samples                     # noqa: E402
from burstplan.graph import graph_to_dict                     # noqa: E402
from burstplan.planner import brute_force_plan, plan, plan_to_json  # noqa: E402
from burstplan.simulator import compile_timeline, forced_plan, SimConfig  # noqa: E402
from conftest import random_chain_graph, random_sp_graph      # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")
AMP_CHOICES = (1.0, 1.1, 1.3, 1.5, 2.0, 4.0, 16.0, 1e9)


def sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as fh:
        json.dump(obj, fh, indent=0, sort_keys=True)
        fh.write("\n")


def main():
    os.makedirs(OUT, exist_ok=True)
    # --- synthetic families: profile bytes + plans --------------------------
    fam = {}
    for name, kw in (("vgg_like", {}), ("wideresnet_like", {"global_batch": 32}),
                     ("inception_like", {}), ("small_bg_model", {})):
        g = getattr(synth, name)(**kw) if name != "small_bg_model" else synth.small_bg_model()
        text = json.dumps(graph_to_dict(g), indent=1) + "\n"
        fam[name] = {"kwargs": kw, "graph_sha256": sha(text)}
    plans = []
    vgg = synth.vgg_like(seed=0)
    for G in (1, 2, 4, 8):
        for B in (8, 16, 32, 64, 128, 256):
            p = plan(vgg, G, 2.0, global_batch=B)
            plans.append({"family": "vgg_like", "kwargs": {}, "G": G, "amp": 2.0,
                          "B": B, "plan_json": plan_to_json(p, vgg)})
        d = forced_plan(vgg, G, G)
        plans.append({"family": "vgg_like", "kwargs": {}, "G": G, "amp": None,
                      "B": 32, "forced": True, "plan_json": plan_to_json(d, vgg)})
    for fname, kw, amps in (("wideresnet_like", {"global_batch": 32}, (2.0, 4.0)),
                            ("inception_like", {}, (2.0, 8.0))):
        g = getattr(synth, fname)(**kw)
        for amp in amps:
            p = plan(g, 8, amp)
            plans.append({"family": fname, "kwargs": kw, "G": 8, "amp": amp,
                          "B": g.global_batch, "plan_json": plan_to_json(p, g)})
        d = forced_plan(g, 8, 8)
        plans.append({"family": fname, "kwargs": kw, "G": 8, "amp": None,
                      "B": g.global_batch, "forced": True,
                      "plan_json": plan_to_json(d, g)})
    # the F2 golden file hash: `burstplan plan --gpus 8 --amp-limit 2`
    p8 = plan(vgg, 8, 2.0)
    fam["vgg_like"]["plan_g8_amp2_sha256"] = sha(plan_to_json(p8, vgg))
    dump("families.json", {"families": fam, "plans": plans})

    # --- random instances (acceptance criteria 1-2 generators) -------------
    rnd = []
    rng = random.Random(1001)
    for _ in range(100):
        g = random_chain_graph(rng, max_layers=6)
        amp = rng.choice(AMP_CHOICES)
        p = plan(g, 4, amp, candidates=(1, 2, 4))
        rnd.append({"graph": graph_to_dict(g), "G": 4, "amp": amp,
                    "candidates": [1, 2, 4], "plan_json": plan_to_json(p)})
    rng = random.Random(2002)
    for i in range(50):
        g = random_sp_graph(rng, max_layers=6, nested=(i % 2 == 0))
        amp = rng.choice(AMP_CHOICES)
        p = plan(g, 4, amp, candidates=(1, 2, 4))
        rnd.append({"graph": graph_to_dict(g), "G": 4, "amp": amp,
                    "candidates": [1, 2, 4], "plan_json": plan_to_json(p)})
    rng = random.Random(4004)
    for i in range(60):   # bigger SP graphs at G=8 (incl. concurrency paths)
        g = random_sp_graph(rng, max_layers=14, nested=(i % 2 == 0),
                            global_batch=rng.choice([8, 12, 32]))
        amp = rng.choice(AMP_CHOICES)
        p = plan(g, 8, amp)
        rnd.append({"graph": graph_to_dict(g), "G": 8, "amp": amp,
                    "candidates": None, "plan_json": plan_to_json(p)})
    dump("random_plans.json", {"instances": rnd})

    # --- the exhaustive oracle on the small instances (G=4, <= 6 layers):
    # reference brute_force_plan (planner.py:592-682) per random_plans index
    bf = []
    for k, inst in enumerate(rnd[:150]):
        from burstplan.graph import graph_from_dict
        g = graph_from_dict(inst["graph"])
        try:
            p = brute_force_plan(g, 4, inst["amp"], candidates=(1, 2, 4))
            bf.append({"index": k, "plan_json": plan_to_json(p)})
        except Exception as exc:                   # guard / infeasible: record the type
            bf.append({"index": k, "error": type(exc).__name__})
    dump("brute_force_plans.json", {"instances": bf})

    # --- sample layout ------------------------------------------------------
    ms = []
    for B in list(range(1, 41)) + [64, 100, 128, 256]:
        for g in (1, 2, 3, 4, 5, 6, 7, 8):
            for h in (1, 2, 3, 4, 5, 6, 7, 8):
                ms.append([B, g, h, moved_samples(B, g, h)])
    dump("moved_samples.json", {"rows": ms})

    # --- op program for C1 ---------------------------------------------------
    tl = compile_timeline(p8, vgg, 8, synth.small_bg_model(), SimConfig())
    ops = lambda seq: [[o.op_id, o.kind, o.isolated_duration_us, o.group_id,
                        list(o.participants), o.barrier, o.payload_bytes,
                        o.stream_priority] for o in seq]
    dump("timeline_c1.json", {"fg": ops(tl.fg_ops), "bg": ops(tl.bg_ops),
                              "predicted": tl.predicted_fg_iteration_us})


if __name__ == "__main__":
    main()

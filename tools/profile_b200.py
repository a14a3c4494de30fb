"""Profile VGG-16 on this B200 into the reference's profile schema and plan
against it.

  python tools/profile_b200.py [--batches 1 2 4 8 16 32 64 128 256] [--out profiles/b200_vgg16]

Writes <out>_graph.json (graph.save_graph: reference JSON schema, loadable
by burstplan.load_graph) and <out>_plans.json: for G in 1, 2, 4, 8 and each
amp limit, the burst plan's GPUs per layer and predicted iteration time
next to uniform data parallelism (forced_plan) on the same measured costs.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_10065_b200 import synth                          # noqa: E402
from paper_2112_10065_b200.graph import save_graph               # noqa: E402
from paper_2112_10065_b200.planner import plan                   # noqa: E402
from paper_2112_10065_b200.profiler import profile_graph         # noqa: E402
from paper_2112_10065_b200.timeline import forced_plan           # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, nargs="+", default=[1, 2, 4, 8, 16, 32])
    ap.add_argument("--global-batch", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="profiles/b200_vgg16")
    a = ap.parse_args()
    g0 = synth.vgg_like(seed=0, global_batch=a.global_batch)
    g = profile_graph(g0, a.batches, a.reps)
    save_graph(g, a.out + "_graph.json")
    rows = []
    for G in (1, 2, 4, 8):
        dp = forced_plan(g, G, G)
        for amp in (1.5, 2.0, 4.0, 8.0):
            p = plan(g, G, amp)
            rows.append({"gpus": G, "amp_limit": amp,
                         "gpus_per_layer": [n for _, n in p.assignments],
                         "bp_iteration_us": p.predicted_iteration_us,
                         "dp_iteration_us": dp.predicted_iteration_us,
                         "bp_over_dp_speedup": dp.predicted_iteration_us / p.predicted_iteration_us})
    with open(a.out + "_plans.json", "w") as fh:
        json.dump({"global_batch": a.global_batch, "batches_profiled": a.batches,
                   "network": {"bandwidth_bytes_per_sec": g.network.per_gpu_bandwidth_bytes_per_sec,
                               "delay_us": g.network.propagation_delay_us},
                   "plans": rows}, fh, indent=1)
    for r in rows:
        print(f"G={r['gpus']} amp={r['amp_limit']}: BP {r['bp_iteration_us']:9.1f} us  "
              f"DP {r['dp_iteration_us']:9.1f} us  x{r['bp_over_dp_speedup']:.3f}  "
              f"{r['gpus_per_layer']}")


if __name__ == "__main__":
    main()

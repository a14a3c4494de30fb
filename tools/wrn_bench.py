"""One-B200 timing of the branch/join nets through the executor: the
residual net behind wideresnet_like (C3 shape: B=32, 34 diamonds at
100/50/25) or the four-tower net behind inception_like (C4 foreground: B=32,
14 modules at 35/17/8), SURVEY.md §8d.  Captured step, CUDA events,
samples/s and TFLOP/s of the algorithmic work.
usage: python tools/wrn_bench.py [--family wideresnet_like|inception_like]
       [--batch 32] [--steps 5] [--warmup 3]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_10065_b200 import synth                              # noqa: E402
from paper_2112_10065_b200.executor import BurstStep                 # noqa: E402
from paper_2112_10065_b200.network import synthetic_batch            # noqa: E402
from paper_2112_10065_b200.planner import plan                       # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--family", default="wideresnet_like",
                    choices=("wideresnet_like", "inception_like"))
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    g = getattr(synth, a.family)(seed=0, global_batch=a.batch)
    p = plan(g, 1, 2.0)
    st = BurstStep(p, g, seed=0, lr=1e-3)
    x, y = synthetic_batch(st.net, a.batch, seed=0)
    st.load(x.pin_memory(), y.pin_memory())
    st.capture(warmup=1)
    for _ in range(a.warmup):
        st.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        st.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    flops = st.net.train_flops_per_sample() * a.batch
    print(json.dumps({"workload": f"{a.family} B={a.batch} ({st.net.name} net, "
                                  f"{len(st.net.layers)} layers) on 1 GPU",
                      "samples_per_s": a.batch / (ms / 1e3), "ms_per_step": ms,
                      "tflops": flops / (ms / 1e3) / 1e12, "loss": st.loss()}))


if __name__ == "__main__":
    main()

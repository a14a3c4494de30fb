"""One eager VGG-16 training step at global batch B on one GPU (for ncu
captures of the non-GEMM kernels: pools, loss, SGD, split-K finishes, the
weight lo split).  usage: python tools/step_once.py [--batch 32] [--steps 1]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_10065_b200 import synth                              # noqa: E402
from paper_2112_10065_b200.executor import BurstStep                 # noqa: E402
from paper_2112_10065_b200.network import synthetic_batch            # noqa: E402
from paper_2112_10065_b200.planner import plan                       # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
g = synth.vgg_like(seed=0, global_batch=a.batch)
st = BurstStep(plan(g, 1, 2.0), g, seed=0, lr=1e-3)
x, y = synthetic_batch(st.net, a.batch, 0)
st.load(x, y)
for _ in range(a.steps):
    st.step()
torch.cuda.synchronize()
print("loss", st.loss())

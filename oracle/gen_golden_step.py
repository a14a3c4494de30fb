"""Golden fp64 losses of the VGG-16 training step (TEST INFRASTRUCTURE).

Writes tests/golden/vgg16_step_fp64.json: for global batches 4, 8 and 32
(the per-GPU batches of the C1 plan [8]*10+[4]*4+[1]*7 at B=32, and the
whole B=32 step bench.py times) the mean cross-entropy of the first step at
the seed-0 init and seed-0 synthetic batch, computed by the CPU fp64 oracle
(oracle/vgg_ref.py), plus per-parameter gradient norms.  bench.py checks its
first step's loss against the B=32 entry (|dL|/L <= 1e-4);
tests/test_step_gpu.py recomputes the full fp64 step on the GPU box.

    python oracle/gen_golden_step.py
"""

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import vgg_ref  # noqa: E402
from paper_2112_10065_b200.network import init_params, synthetic_batch, vgg16  # noqa: E402


def main():
    torch.set_num_threads(os.cpu_count() or 1)
    net = vgg16()
    params = init_params(net, 0)
    out = {"model": "vgg16", "seed": 0, "dtype": "float64",
           "torch": torch.__version__, "batches": {}}
    for B in (4, 8, 32):
        x, y = synthetic_batch(net, B, 0)
        t0 = time.time()
        loss, grads = vgg_ref.forward_backward(net, params, x, y, torch.float64)
        out["batches"][str(B)] = {
            "loss": float(loss),
            "x_sum": float(x.double().sum()), "labels": [int(v) for v in y[:8]],
            "grad_norms": {k: [float(dw.double().norm()), float(db.double().norm())]
                           for k, (dw, db) in grads.items()},
            "cpu_seconds": time.time() - t0}
        print(B, loss, f"{time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "vgg16_step_fp64.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()

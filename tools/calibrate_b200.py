"""Simulator calibration on the B200: run a plan with
per-op device timing, then compare the reference cost model's prediction and
the measurement-priced simulation with the measured iteration.
usage: [torchrun ...] python tools/calibrate_b200.py out.json [--family vgg_like]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_10065_b200 import synth                           # noqa: E402
from paper_2112_10065_b200.planner import plan                   # noqa: E402
from paper_2112_10065_b200.simulate import calibration_report    # noqa: E402
from paper_2112_10065_b200.timeline import SimConfig             # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?")
    ap.add_argument("--family", default="vgg_like")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--iterations", type=int, default=8)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
        dist.init_process_group("nccl")
    g = getattr(synth, a.family)(seed=0, global_batch=a.batch)
    p = plan(g, world, 2.0)
    rep = calibration_report(p, g, world, SimConfig(warmup_iterations=2), a.iterations)
    rep.update(family=a.family, batch=a.batch, gpus=world)
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({k: v for k, v in rep.items() if k != "ops"}))
        if a.out:
            with open(a.out, "w") as fh:
                json.dump(rep, fh, indent=1)


if __name__ == "__main__":
    main()

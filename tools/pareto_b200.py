"""Measured Pareto sweep of VGG-16 BP+Col operating points vs static
partitions (sweep.pareto_sweep) -> TSV in the reference CLI's `sweep`
format.  usage: [torchrun ...] python tools/pareto_b200.py out.tsv"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_10065_b200 import synth                                    # noqa: E402
from paper_2112_10065_b200.sweep import pareto_sweep, pareto_to_table      # noqa: E402
from paper_2112_10065_b200.timeline import SimConfig                       # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
        dist.init_process_group("nccl")
    g = synth.vgg_like(seed=0, global_batch=32)
    cfgs = [SimConfig(warmup_iterations=2, launch_pace_limit=p, bg_batch_size=8)
            for p in (1, 2, 4)]
    rows = pareto_sweep(g, world, [2.0, 4.0], cfgs, bg_graph=synth.small_bg_model(),
                        iterations=12)
    tab = pareto_to_table(rows)
    if int(os.environ.get("RANK", "0")) == 0:
        print(tab, end="")
        if len(sys.argv) > 1:
            with open(sys.argv[1], "w") as fh:
                fh.write(tab)


if __name__ == "__main__":
    main()

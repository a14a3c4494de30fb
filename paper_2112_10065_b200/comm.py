"""Cross-rank plumbing of the burst-parallel step (one process per GPU).

Two exchange steps exist:

* **reshard** -- at every change of GPU count between consecutive layers,
  samples move between the g-way and h-way contiguous ceil layouts
  (`costs.reshard_segments`, the index map behind the reference's
  ``moved_samples``, /root/reference/pkg/src/burstplan/costs.py:85-104).
  Forward moves activations, backward moves their gradients.
* **subset allreduce** -- weight gradients of a layer on g GPUs are summed
  over ranks [0, g) (`costs.py:130-140`, `simulator.py:264-278`).

``TorchComm`` implements both with torch.distributed point-to-point and
prefix sub-groups (NCCL over NVLink on B200; gloo in the CPU tests, where
the same code path and index map are exercised with world_size 2).
The libbpx P2P kernels (``bpx_reshard_pull`` / ``bpx_allreduce_sum_prefix``)
are the peer-memory alternative (PeerComm).
"""

from __future__ import annotations

from typing import Optional

import torch

from .costs import reshard_segments, shard_range
from .graph import ceil_div


def reshard_moves(B: int, g: int, h: int, rank: int, bytes_per_sample: int):
    """This rank's part of a g->h reshard as byte ranges.

    Returns (local, sends, recvs): local = [(src_off, dst_off, nbytes)],
    sends = [(peer, src_off, nbytes)], recvs = [(peer, dst_off, nbytes)];
    offsets are into this rank's local g-layout source / h-layout
    destination buffers, in sample order (so every pair of ranks agrees on
    message order)."""
    cg, ch = ceil_div(B, g), ceil_div(B, h)
    local, sends, recvs = [], [], []
    for p, q, s, n in reshard_segments(B, g, h):
        if p != rank and q != rank:
            continue
        so = (s - p * cg) * bytes_per_sample
        do = (s - q * ch) * bytes_per_sample
        nb = n * bytes_per_sample
        if p == rank and q == rank:
            local.append((so, do, nb))
        elif p == rank:
            sends.append((q, so, nb))
        else:
            recvs.append((p, do, nb))
    return local, sends, recvs


def _bytes(t: torch.Tensor) -> torch.Tensor:
    return t.view(-1).view(torch.uint8)


class TorchComm:
    """torch.distributed backend (NCCL on GPUs, gloo on CPU tests)."""

    def __init__(self, rank: int, world: int, group_sizes=()):
        import torch.distributed as dist
        self.dist = dist
        self.rank = rank
        self.world = world
        self.groups = {}
        # new_group is collective over the WORLD: every rank creates every
        # prefix group, in the same (sorted) order.
        for g in sorted(set(group_sizes)):
            if g <= 1:
                continue
            self.groups[g] = (dist.group.WORLD if g == world
                              else dist.new_group(ranks=list(range(g))))

    def reshard(self, src: Optional[torch.Tensor], g: int, dst: Optional[torch.Tensor],
                h: int, B: int, bytes_per_sample: int) -> None:
        local, sends, recvs = reshard_moves(B, g, h, self.rank, bytes_per_sample)
        sb = _bytes(src) if sends or local else None
        db = _bytes(dst) if recvs or local else None
        for so, do, nb in local:
            db[do:do + nb].copy_(sb[so:so + nb])
        ops = []
        for peer, so, nb in sends:
            ops.append(self.dist.P2POp(self.dist.isend, sb[so:so + nb], peer))
        tmp = []
        for peer, do, nb in recvs:
            view = db[do:do + nb]
            ops.append(self.dist.P2POp(self.dist.irecv, view, peer))
            tmp.append(view)
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def allreduce(self, flat: torch.Tensor, g: int) -> None:
        if g <= 1 or self.rank >= g:
            return
        self.dist.all_reduce(flat, op=self.dist.ReduceOp.SUM, group=self.groups[g])

    def max_scalar(self, value: float, device) -> float:
        t = torch.tensor([value], dtype=torch.float64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_scalar(self, value: float, device) -> float:
        t = torch.tensor([value], dtype=torch.float64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def barrier(self):
        self.dist.barrier()


class LocalComm:
    """world_size 1: every layer has g == 1, nothing crosses a GPU."""

    rank = 0
    world = 1

    def reshard(self, src, g, dst, h, B, bytes_per_sample):
        if g != 1 or h != 1:
            raise ValueError("single-GPU executor got a multi-GPU layout")
        if src is not None and dst is not None and src.data_ptr() != dst.data_ptr():
            dst.copy_(src)

    def allreduce(self, flat, g):
        if g > 1:
            raise ValueError("single-GPU executor got a multi-GPU allreduce")

    def max_scalar(self, value, device):
        return value

    def sum_scalar(self, value, device):
        return value

    def barrier(self):
        pass

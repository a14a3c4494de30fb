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


class PeerComm:
    """P2P backend of the step's communication (north_star (2)-(3)): peer
    memory instead of NCCL for the data path, every op graph-capturable.

    Each rank owns one device arena -- signal pads, per-group-size epoch
    counters and a staging area -- whose CUDA IPC handle is exchanged once
    through torch.distributed (any backend: only handles and scalars go
    through it).  Peers map each other's arenas (NVLink peer addresses on a
    multi-GPU box; the same device for two processes sharing one GPU).

    * reshard (the `transfer` op, simulator.py:242-253): each source rank
      stages its shard, a device barrier over the participants, then every
      destination rank pulls its contiguous runs (costs.reshard_segments)
      from the sources' staging areas with ``bpx_reshard_pull``, and a second
      barrier before the staging areas may be reused;
    * allreduce over ranks [0, g) (`allreduce`, :264-278): stage, barrier,
      one-shot pull-sum in rank order (``bpx_allreduce_sum_prefix``: the
      same bits on every rank), barrier.
    Barriers are ``bpx_signal_barrier_dev`` (device-resident epochs), so a
    captured step replays correctly.  Call ``prepare`` (collective) before
    use: BurstStep does, with its largest shard and gradient bucket.

    Processes must load their kernels eagerly (``CUDA_MODULE_LOADING=EAGER``
    before CUDA initialises): with lazy loading, a kernel's first launch can
    wait on the device while a peer's barrier kernel spins waiting on this
    process -- a deadlock."""

    def __init__(self, rank: int, world: int, group_sizes=(), device=None):
        import os
        import warnings
        if os.environ.get("CUDA_MODULE_LOADING", "").upper() != "EAGER":
            warnings.warn("PeerComm: set CUDA_MODULE_LOADING=EAGER before CUDA starts; "
                          "lazy kernel loading can deadlock with device barriers")
        self.rank, self.world = rank, world
        self.host = TorchComm(rank, world, ())   # handle exchange, scalars, host barrier
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        self.arena = None

    def prepare(self, stage_bytes: int) -> None:
        from . import ops
        W = self.world
        pad_bytes = 4 * W * (W + 1)               # pads for group sizes 1..W, W slots each
        cnt_bytes = 4 * (W + 1)                   # one epoch counter per group size
        head = (pad_bytes + cnt_bytes + 255) // 256 * 256
        size = head + max(16, (stage_bytes + 255) // 256 * 256)
        if self.arena is not None and self.arena.numel() >= size:
            return
        self.arena = torch.zeros(size, dtype=torch.uint8, device=self.device)
        self.head = head
        self.pad_bytes = pad_bytes
        handle = self.arena.untyped_storage()._share_cuda_()
        handles = [None] * W
        self.host.dist.all_gather_object(handles, handle)
        self.peer_storages = []
        self.peer_base = []
        for r in range(W):
            if r == self.rank:
                self.peer_base.append(self.arena.data_ptr())
                self.peer_storages.append(None)
            else:
                st = torch.UntypedStorage._new_shared_cuda(*handles[r])
                self.peer_storages.append(st)     # keeps the mapping alive
                # the handle covers the caching allocator's block; the arena
                # starts at the storage's offset inside it (handle[3])
                self.peer_base.append(st.data_ptr())
        self.host.dist.barrier()
        self._ops = ops

    # layout helpers (the same offsets in every rank's arena)
    def _pads(self, g: int) -> list:
        return [b + 4 * self.world * g for b in self.peer_base[:g]]

    def _counter(self, g: int) -> int:
        return self.arena.data_ptr() + self.pad_bytes + 4 * g

    def _stage(self, r: int) -> int:
        return self.peer_base[r] + self.head

    def _barrier(self, g: int) -> None:
        if g > 1 and self.rank < g:
            self._ops.signal_barrier_dev(self._pads(g), self._counter(g), self.rank)

    def _stage_view(self, nbytes: int) -> torch.Tensor:
        return self.arena[self.head:self.head + nbytes]

    def reshard(self, src: Optional[torch.Tensor], g: int, dst: Optional[torch.Tensor],
                h: int, B: int, bytes_per_sample: int) -> None:
        P = max(g, h)
        if self.rank >= P:
            return
        if src is not None and self.rank < g:
            sb = _bytes(src)
            self._stage_view(sb.numel()).copy_(sb)
        self._barrier(P)
        if dst is not None and self.rank < h:
            cg, ch = ceil_div(B, g), ceil_div(B, h)
            srcs, soff, doff, nb = [], [], [], []
            for p, q, s0, n in reshard_segments(B, g, h):
                if q != self.rank:
                    continue
                srcs.append(self._stage(p))
                soff.append((s0 - p * cg) * bytes_per_sample)
                doff.append((s0 - q * ch) * bytes_per_sample)
                nb.append(n * bytes_per_sample)
            for k in range(0, len(nb), 64):
                self._ops.reshard_pull(srcs[k:k + 64], soff[k:k + 64], dst, doff[k:k + 64],
                                       nb[k:k + 64])
        self._barrier(P)

    def allreduce(self, flat: torch.Tensor, g: int) -> None:
        if g <= 1 or self.rank >= g:
            return
        self._stage_view(flat.numel() * 4).copy_(_bytes(flat))
        self._barrier(g)
        self._ops.allreduce_sum_prefix([self._stage(r) for r in range(g)], flat, flat.numel())
        self._barrier(g)

    def max_scalar(self, value: float, device) -> float:
        return self.host.max_scalar(value, device)

    def sum_scalar(self, value: float, device) -> float:
        return self.host.sum_scalar(value, device)

    def barrier(self):
        self.host.barrier()


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

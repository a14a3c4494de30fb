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

    def _scalar_device(self, device):
        # gloo reduces host tensors; NCCL needs device tensors
        return "cpu" if self.dist.get_backend() == "gloo" else device

    def max_scalar(self, value: float, device) -> float:
        t = torch.tensor([value], dtype=torch.float64, device=self._scalar_device(device))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_scalar(self, value: float, device) -> float:
        t = torch.tensor([value], dtype=torch.float64, device=self._scalar_device(device))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def barrier(self):
        self.dist.barrier()

    def allgather_object(self, obj) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def check(self) -> None:
        pass


class PeerComm:
    """P2P backend of the step's communication (north_star (2)-(3)): peer
    memory instead of NCCL for the data path, every op graph-capturable.

    * Control arena (one per rank, mapped by every peer through CUDA IPC
      once, at construction): signal pads and an epoch counter per group
      size, an abort word and a status word.  Barriers are
      ``bpx_peer_barrier``: device-resident epochs (a captured step replays
      correctly), bounded by ``BPX_BARRIER_TIMEOUT_S`` (default 60 s) and
      by the abort words -- a dead or late peer fails the step with
      ``CommError`` (``check``) instead of hanging it.
    * Symmetric heaps (``make_heap``, collective): every buffer that a peer
      reads -- the producer side of each reshard (layer outputs, data
      gradients, shortcut gradients) and the gradient buckets -- lives in a
      per-rank arena whose handle and per-key offsets are exchanged once,
      so kernels pull straight out of the producer's buffer: no staging
      copy (SymHeap.reshard / SymHeap.allreduce).
    torch.distributed (any backend) carries only handles and scalars.  On a
    multi-GPU box peers are NVLink addresses; in tests several processes
    share one GPU.  Processes must load their kernels eagerly
    (``CUDA_MODULE_LOADING=EAGER`` before CUDA initialises): with lazy
    loading a kernel's first launch can wait on the device while a peer's
    barrier kernel spins waiting on this process."""

    def __init__(self, rank: int, world: int, group_sizes=(), device=None,
                 timeout_s: Optional[float] = None):
        import os
        import warnings
        if os.environ.get("CUDA_MODULE_LOADING", "").upper() != "EAGER":
            warnings.warn("PeerComm: set CUDA_MODULE_LOADING=EAGER before CUDA starts; "
                          "lazy kernel loading can deadlock with device barriers")
        from . import ops
        self._ops = ops
        self.rank, self.world = rank, world
        self.host = TorchComm(rank, world, ())   # handle exchange, scalars, host barrier
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        if timeout_s is None:
            timeout_s = float(os.environ.get("BPX_BARRIER_TIMEOUT_S", "60"))
        self.timeout_ns = int(timeout_s * 1e9)
        W = world
        # uint32 words: pads [g][r] for g = 0..W, counters [g], abort, status
        self._pad0, self._cnt0 = 0, W * (W + 1)
        self._abort = self._cnt0 + W + 1
        self._status = self._abort + 1
        words = (self._status + 1 + 63) // 64 * 64
        self.ctl = torch.zeros(words, dtype=torch.int32, device=self.device)
        self.peer_ctl, self._ctl_maps = self._exchange(self.ctl)
        self._heaps = []          # every heap stays mapped while this comm lives

    def _exchange(self, t: torch.Tensor, meta=None):
        """All ranks: share ``t``'s CUDA IPC handle (+ metadata), map every
        peer's; returns (base addresses per rank, [storages | metadata])."""
        handle = t.untyped_storage()._share_cuda_()
        got = self.host.allgather_object((handle, meta))
        bases, keep, metas = [], [], []
        for r, (h, m) in enumerate(got):
            metas.append(m)
            if r == self.rank:
                bases.append(t.data_ptr())
                keep.append(None)
            else:
                st = torch.UntypedStorage._new_shared_cuda(*h)
                keep.append(st)                  # keeps the mapping alive
                bases.append(st.data_ptr())
        self.host.barrier()
        return bases, (keep if meta is None else (keep, metas))

    # ---- control arena
    def _word(self, r: int, w: int) -> int:
        return self.peer_ctl[r] + 4 * w

    def barrier_dev(self, g: int) -> None:
        """Bounded device barrier over ranks [0, g) (stream-ordered)."""
        if g <= 1 or self.rank >= g:
            return
        W = self.world
        self._ops.peer_barrier([self._word(r, self._pad0 + g * W) for r in range(g)],
                               [self._word(r, self._abort) for r in range(g)],
                               self._word(self.rank, self._cnt0 + g),
                               self._word(self.rank, self._status), self.rank, self.timeout_ns)

    def status(self) -> int:
        return int(self.ctl[self._status].item())

    def check(self) -> None:
        """Raise CommError if a device barrier of this rank timed out or was
        aborted (synchronises with the device)."""
        from .errors import CommError
        st = self.status()
        if st:
            why = {1: "timed out waiting for a peer", 2: "was aborted by a peer"}.get(st, "failed")
            raise CommError(f"rank {self.rank}: a P2P barrier {why} "
                            f"(BPX_BARRIER_TIMEOUT_S={self.timeout_ns / 1e9:g})", st)

    def abort(self) -> None:
        """Raise every rank's abort word: their pending and future barriers
        fail fast (call on a host-side error before exiting)."""
        s = torch.cuda.Stream(device=self.device)
        with torch.cuda.stream(s):
            for r in range(self.world):
                st = self._ctl_maps[r] if r != self.rank else self.ctl.untyped_storage()
                t = torch.empty(0, dtype=torch.int32, device=self.device)
                t.set_(st, 0, (self.ctl.numel(),), (1,))
                t[self._abort].fill_(1)
        s.synchronize()

    # ---- symmetric heaps
    def make_heap(self, sizes: dict) -> "SymHeap":
        """Collective: allocate this rank's buffers ``sizes`` = {key: nbytes}
        (keys may differ across ranks) in one IPC-shared arena and learn
        every peer's offsets.  Returns the heap; its views are the tensors
        the step computes into."""
        keys = sorted(sizes, key=repr)
        layout, off = {}, 0
        for k in keys:
            nb = int(sizes[k])
            layout[k] = (off, nb)
            off += (nb + 255) // 256 * 256
        arena = torch.zeros(max(off, 256), dtype=torch.uint8, device=self.device)
        bases, (keep, layouts) = self._exchange(arena, layout)
        heap = SymHeap(self, arena, bases, layouts, keep)
        self._heaps.append(heap)
        return heap

    def max_scalar(self, value: float, device) -> float:
        return self.host.max_scalar(value, device)

    def sum_scalar(self, value: float, device) -> float:
        return self.host.sum_scalar(value, device)

    def barrier(self):
        self.host.barrier()

    def allgather_object(self, obj) -> list:
        return self.host.allgather_object(obj)


class SymHeap:
    """One BurstStep's peer-visible buffers on every rank (PeerComm.make_heap).

    * ``reshard`` (the `transfer` op, simulator.py:242-253): barrier over
      [0, max(g, h)) -- every producer has written its shard -- then each
      consumer pulls its contiguous runs (costs.reshard_segments) straight
      out of the producers' buffers with ``bpx_reshard_pull``, and a second
      barrier before any producer may overwrite them;
    * ``allreduce`` over ranks [0, g) (`allreduce`, :264-278), in place on
      the gradient bucket: two-shot -- reduce-scatter (rank r sums chunk r
      of all g buckets in rank order 0..g-1 into its own bucket), barrier,
      all-gather (rank r pulls every other chunk from its owner) -- so each
      rank reads 2(g-1)/g of the bucket over NVLink, the ring volume the
      reference prices (costs.py:130-140); buckets below 64 floats per rank
      take one shot (sum of all g buckets into private scratch, barrier,
      copy back).  Every rank adds in the same order: bitwise identical
      results on every rank, run to run."""

    SMALL = 64

    def __init__(self, comm: PeerComm, arena, bases, layouts, keep):
        self.comm, self.arena, self.bases, self.layouts, self._keep = \
            comm, arena, bases, layouts, keep
        self.rank = comm.rank
        self._scratch = {}

    def view(self, key, shape, dtype=torch.float32) -> torch.Tensor:
        off, nb = self.layouts[self.rank][key]
        n = 1
        for d in shape:
            n *= int(d)
        esz = torch.tensor([], dtype=dtype).element_size()
        if n * esz > nb:
            raise ValueError(f"heap buffer {key} holds {nb} bytes, {n * esz} requested")
        return self.arena[off:off + n * esz].view(dtype).view(*shape)

    def addr(self, r: int, key) -> int:
        from .errors import CommError
        ent = self.layouts[r].get(key)
        if ent is None:
            raise CommError(f"rank {r} has no heap buffer {key!r} (layouts disagree)")
        return self.bases[r] + ent[0]

    def reshard(self, src_key, g: int, dst: Optional[torch.Tensor], h: int, B: int,
                bytes_per_sample: int) -> None:
        P = max(g, h)
        if self.rank >= P:
            return
        self.comm.barrier_dev(P)
        if dst is not None and self.rank < h:
            cg, ch = ceil_div(B, g), ceil_div(B, h)
            srcs, soff, doff, nb = [], [], [], []
            for p, q, s0, n in reshard_segments(B, g, h):
                if q != self.rank:
                    continue
                srcs.append(self.addr(p, src_key))
                soff.append((s0 - p * cg) * bytes_per_sample)
                doff.append((s0 - q * ch) * bytes_per_sample)
                nb.append(n * bytes_per_sample)
            for k in range(0, len(nb), 64):
                self.comm._ops.reshard_pull(srcs[k:k + 64], soff[k:k + 64], dst,
                                            doff[k:k + 64], nb[k:k + 64])
        self.comm.barrier_dev(P)

    def allreduce(self, key, flat: torch.Tensor, g: int) -> None:
        if g <= 1 or self.rank >= g:
            return
        ops, r = self.comm._ops, self.rank
        n = flat.numel()
        peers = [self.addr(p, key) for p in range(g)]
        if n < self.SMALL * g:
            buf = self._scratch.get(key)
            if buf is None or buf.numel() < n:
                buf = self._scratch[key] = torch.empty(n, dtype=torch.float32,
                                                       device=flat.device)
            self.comm.barrier_dev(g)
            ops.allreduce_sum_prefix(peers, buf, n)
            self.comm.barrier_dev(g)
            flat.copy_(buf[:n])
            return
        c = ceil_div(ceil_div(n, g), 4) * 4            # 16-byte aligned chunks
        lo, hi = min(n, r * c), min(n, (r + 1) * c)
        self.comm.barrier_dev(g)
        if hi > lo:
            ops.allreduce_sum_prefix([a + 4 * lo for a in peers], flat[lo:hi], hi - lo)
        self.comm.barrier_dev(g)
        srcs, soff, doff, nb = [], [], [], []
        for p in range(g):
            a, b = min(n, p * c), min(n, (p + 1) * c)
            if p != r and b > a:
                srcs.append(peers[p])
                soff.append(4 * a)
                doff.append(4 * a)
                nb.append(4 * (b - a))
        if nb:
            ops.reshard_pull(srcs, soff, flat, doff, nb)
        self.comm.barrier_dev(g)


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

    def allgather_object(self, obj) -> list:
        return [obj]

    def check(self) -> None:
        pass

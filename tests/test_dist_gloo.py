"""Multi-rank data movement of the burst-parallel step, world_size 2 over
gloo on CPU: the same TorchComm code and reshard index map the NCCL path
uses on B200s.  Activations / gradients must land exactly on the ranks the
h-way ceil layout assigns them to; prefix allreduce sums over [0, g)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2112_10065_b200.comm import TorchComm, reshard_moves
from paper_2112_10065_b200.costs import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comm = TorchComm(rank, world, group_sizes=(1, 2))
        feat = 6
        for B in (1, 2, 3, 5, 8, 32):
            full = torch.arange(B * feat, dtype=torch.float32).view(B, feat)
            for g in (1, 2):
                for h in (1, 2):
                    if g == h:
                        continue
                    a, b = shard_range(B, g, rank)
                    src = full[a:b].clone() if rank < g else None
                    c, d = shard_range(B, h, rank)
                    dst = torch.full((d - c, feat), -1.0) if rank < h else None
                    comm.reshard(src, g, dst, h, B, feat * 4)
                    if dst is not None:
                        assert torch.equal(dst, full[c:d]), (B, g, h, rank)
        flat = torch.full((10,), float(rank + 1))
        comm.allreduce(flat, 2)
        assert torch.equal(flat, torch.full((10,), 3.0))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as exc:                      # surface in the parent
        q.put((rank, repr(exc)))


def test_reshard_and_prefix_allreduce_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}


def test_reshard_moves_partition_every_sample():
    for B in range(1, 40):
        for g in range(1, 9):
            for h in range(1, 9):
                got = {}
                for r in range(max(g, h)):
                    local, sends, recvs = reshard_moves(B, g, h, r, 1)
                    for so, do, n in local:
                        for k in range(n):
                            got[r * 0 + do + k + shard_range(B, h, r)[0]] = r
                    for peer, do, n in recvs:
                        for k in range(n):
                            got[do + k + shard_range(B, h, r)[0]] = r
                for s in range(B):
                    q = s // -(-B // h)
                    assert got[s] == q
                # sends and recvs pair up
                sends = sorted((r, peer, n) for r in range(g)
                               for peer, _, n in reshard_moves(B, g, h, r, 1)[1])
                recvs = sorted((peer, r, n) for r in range(h)
                               for peer, _, n in reshard_moves(B, g, h, r, 1)[2])
                assert sends == recvs

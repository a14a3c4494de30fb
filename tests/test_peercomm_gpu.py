"""P2P communication backend (comm.PeerComm) with two processes sharing one
B200: each process maps the other's arena through CUDA IPC, so resharding
(bpx_reshard_pull), the pull allreduce and the device-epoch signal barriers
run across real process boundaries; torch.distributed (gloo) only carries
the IPC handles.  On a multi-GPU box the same code pulls over NVLink."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def gpu_tiny_vgg():
    """tests/test_executor_dist.tiny_vgg with GPU-engine widths (channels
    x4, dense 32/32/16): same 21 layers, so the same plan GS applies."""
    from paper_2112_10065_b200.network import LayerSpec, NetSpec
    layers, hw, cin, first = [], 32, 3, True
    for stage, (cout, n) in enumerate(((16, 2), (32, 2), (32, 3), (64, 3), (64, 3)), start=1):
        for j in range(1, n + 1):
            layers.append(LayerSpec(f"conv{stage}_{j}", "conv", cin, cout, hw, True, not first))
            first, cin = False, cout
        layers.append(LayerSpec(f"pool{stage}", "pool", cout, cout, hw, False, True))
        hw //= 2
    feats = hw * hw * cin
    for k, (fout, relu) in enumerate(((32, True), (32, True), (16, False)), start=1):
        layers.append(LayerSpec(f"fc{k}", "dense", feats, fout, 0, relu, True))
        feats = fout
    return NetSpec("gpu_tiny_vgg", 32, 3, 16, tuple(layers))


def _worker(rank, port, q, case):
    if os.environ.get("BPX_PC_DEBUG"):
        import faulthandler
        import sys
        faulthandler.dump_traceback_later(int(os.environ["BPX_PC_DEBUG"]), exit=True,
                                          file=sys.stderr)
    try:
        # spin-waiting barrier kernels + lazy module loading can deadlock (a
        # first launch may wait on the device while the peer spins on us):
        # load every kernel at CUDA init, before the first barrier
        os.environ["CUDA_MODULE_LOADING"] = "EAGER"
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        from paper_2112_10065_b200.comm import PeerComm
        comm = PeerComm(rank, 2, device="cuda:0")
        res = {}
        if case == "ops":
            comm.prepare(1 << 20)
            B, bps = 7, 64
            # 2 -> 1 reshard: rank 0 gathers every sample
            src = torch.arange(B * bps, dtype=torch.uint8, device="cuda").view(B, bps)
            mine = src[0:4] if rank == 0 else src[4:7]
            dst = torch.zeros(B, bps, dtype=torch.uint8, device="cuda") if rank == 0 else None
            comm.reshard(mine.contiguous(), 2, dst, 1, B, bps)
            torch.cuda.synchronize()
            if rank == 0:
                res["gather_ok"] = bool(torch.equal(dst, src))
            # 1 -> 2 reshard: rank 0 scatters
            out = torch.zeros(4 if rank == 0 else 3, bps, dtype=torch.uint8, device="cuda")
            comm.reshard(src if rank == 0 else None, 1, out, 2, B, bps)
            torch.cuda.synchronize()
            res["scatter_ok"] = bool(torch.equal(out, src[0:4] if rank == 0 else src[4:7]))
            # allreduce, 3 rounds (epochs advance)
            for k in range(3):
                x = torch.full((1000,), float(rank + 1 + k), device="cuda")
                comm.allreduce(x, 2)
                torch.cuda.synchronize()
                res[f"ar{k}"] = float(x[0].item())
        else:
            from oracle import vgg_ref
            from paper_2112_10065_b200 import synth
            from paper_2112_10065_b200.executor import BurstStep
            from paper_2112_10065_b200.network import init_params, synthetic_batch
            from paper_2112_10065_b200.planner import TrainingPlan
            from paper_2112_10065_b200.network import LayerSpec, NetSpec
            from test_executor_dist import GS
            B = 5
            net = gpu_tiny_vgg()
            params = init_params(net, seed=3)
            graph = synth.vgg_like(seed=0, global_batch=B)
            ids = [l.id for l in graph.layers if not l.is_virtual]
            p = TrainingPlan("vgg_like", 2, 2.0, B, tuple(zip(ids, GS)), 0.0, (), ())
            x, y = synthetic_batch(net, B, seed=4)
            st = BurstStep(p, graph, comm=comm, params=params, net=net, lr=0.0)
            st.load(x, y)
            st.forward_backward()
            st.sync_and_update()
            torch.cuda.synchronize()
            res["loss"] = st.loss()
            g0 = {n: (a.cpu().clone(), b.cpu().clone()) for n, (a, b) in st.grads().items()}
            st.capture(warmup=1)                  # captured step: barriers must replay
            for _ in range(2):
                st.step()
            torch.cuda.synchronize()
            res["replay_same"] = all(torch.equal(a.cpu(), g0[n][0]) and torch.equal(b.cpu(), g0[n][1])
                                     for n, (a, b) in st.grads().items())
            if rank == 0:
                ref_loss, ref = vgg_ref.forward_backward(net, params, x, y, torch.float64)
                ref32, r32 = vgg_ref.forward_backward(net, params, x, y, torch.float32)
                res["ref_loss"] = ref_loss
                worst = 0.0
                for n, (dw, db) in g0.items():
                    for got, rf, rf32 in ((dw, ref[n][0], r32[n][0]), (db, ref[n][1], r32[n][1])):
                        gate = max(1e-3, 2 * vgg_ref.normwise_rel(rf32, rf))
                        worst = max(worst, vgg_ref.normwise_rel(got, rf) / gate)
                res["worst"] = worst
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


def _run(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, port, q, case)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in (0, 1):
        assert "error" not in out[r], out[r].get("error")
    return out


@pytest.mark.timeout(300)
def test_peer_reshard_and_allreduce_across_processes():
    out = _run("ops")
    assert out[0]["gather_ok"]
    assert out[0]["scatter_ok"] and out[1]["scatter_ok"]
    for k in range(3):
        assert out[0][f"ar{k}"] == out[1][f"ar{k}"] == float(1 + k + 2 + k)


@pytest.mark.timeout(300)
def test_peer_backend_burst_step_matches_oracle_and_replays():
    out = _run("step")
    r0 = out[0]
    assert abs(r0["loss"] - r0["ref_loss"]) <= 1e-4 * abs(r0["ref_loss"])
    assert r0["worst"] <= 1.0
    assert r0["replay_same"] and out[1]["replay_same"]

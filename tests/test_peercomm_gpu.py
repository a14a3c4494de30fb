"""P2P communication backend (comm.PeerComm) with 2 and 4 processes sharing
one B200: each process maps the others' control arenas and symmetric heaps
through CUDA IPC, so resharding (bpx_reshard_pull straight out of the
producer's buffer), the two-shot / one-shot allreduce and the bounded
device-epoch barriers run across real process boundaries; torch.distributed
(gloo) only carries the IPC handles.  On a multi-GPU box the same code pulls
over NVLink."""

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


# g per layer for 4 ranks: every transition 4->2->1->4->1, ragged B=7
GS4 = [4] * 5 + [2] * 4 + [1] * 3 + [4] * 4 + [1] * 5


def _step_case(comm, rank, world, gs, B, res):
    from oracle import vgg_ref
    from paper_2112_10065_b200 import synth
    from paper_2112_10065_b200.executor import BurstStep
    from paper_2112_10065_b200.network import init_params, synthetic_batch
    from paper_2112_10065_b200.planner import TrainingPlan
    net = gpu_tiny_vgg()
    params = init_params(net, seed=3)
    graph = synth.vgg_like(seed=0, global_batch=B)
    ids = [l.id for l in graph.layers if not l.is_virtual]
    p = TrainingPlan("vgg_like", world, 2.0, B, tuple(zip(ids, gs)), 0.0, (), ())
    x, y = synthetic_batch(net, B, seed=4)
    st = BurstStep(p, graph, comm=comm, params=params, net=net, lr=0.0)
    st.load(x, y)
    st.forward_backward()
    st.sync_and_update()
    torch.cuda.synchronize()
    res["loss"] = st.loss()
    res["last_g"] = gs[-1]
    g0 = {n: (a.cpu().clone(), b.cpu().clone()) for n, (a, b) in st.grads().items()}
    st.capture(warmup=1)                  # captured step: barriers must replay
    for _ in range(2):
        st.step()
    torch.cuda.synchronize()
    comm.check()
    res["replay_same"] = all(torch.equal(a.cpu(), g0[n][0]) and torch.equal(b.cpu(), g0[n][1])
                             for n, (a, b) in st.grads().items())
    # every rank of a layer's group holds the same (allreduced) gradient
    res["grads"] = _digest(g0)
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


def _digest(grads) -> dict:
    import hashlib
    return {n: hashlib.sha1(dw.cpu().numpy().tobytes() + db.cpu().numpy().tobytes()).hexdigest()
            for n, (dw, db) in grads.items()}


def _vgg16_b32_case(comm, rank, world, case, res):
    """Real VGG-16 at the benchmarked global batch 32 under the C1 plan
    plan(vgg_like, 8, 2.0) = [8]*10+[4]*4+[1]*7 (per-GPU batches 4, 8, 32)
    or uniform DP over 8 ranks.  Rank 0 is active in every layer, so its
    gradients are checked against fp64; every other rank's replicas must be
    bitwise identical to rank 0's (same-order allreduce)."""
    from oracle import vgg_ref
    from paper_2112_10065_b200 import synth
    from paper_2112_10065_b200.executor import BurstStep
    from paper_2112_10065_b200.network import init_params, synthetic_batch, vgg16
    from paper_2112_10065_b200.planner import plan
    from paper_2112_10065_b200.timeline import forced_plan
    B = 32
    graph = synth.vgg_like(seed=0, global_batch=B)
    p = plan(graph, world, 2.0) if case == "c1" else forced_plan(graph, world, world)
    res["gs"] = [g for _, g in p.assignments]
    net = vgg16()
    params = init_params(net, seed=0)
    x, y = synthetic_batch(net, B, seed=0)
    st = BurstStep(p, graph, comm=comm, params=params, lr=0.0)
    st.load(x, y)
    st.forward_backward()
    st.sync_and_update()
    torch.cuda.synchronize()
    res["loss"] = st.loss()
    d0 = _digest(st.grads())
    st.capture(warmup=1)
    for _ in range(2):
        st.step()
    torch.cuda.synchronize()
    comm.check()
    res["replay_same"] = _digest(st.grads()) == d0
    all_d = comm.allgather_object(d0)
    res["replicas_same"] = all(all_d[0][n] == h for d in all_d for n, h in d.items())
    if rank == 0:
        g0 = {n: (a.cpu(), b.cpu()) for n, (a, b) in st.grads().items()}
        del st
        torch.cuda.empty_cache()
        ref_loss, ref = vgg_ref.forward_backward(net, params, x, y, torch.float64)
        _, r32 = vgg_ref.forward_backward(net, params, x, y, torch.float32)
        res["ref_loss"] = float(ref_loss)
        worst = 0.0
        for n, (dw, db) in g0.items():
            for got, rf, rf32 in ((dw, ref[n][0], r32[n][0]), (db, ref[n][1], r32[n][1])):
                gate = max(1e-3, 2 * vgg_ref.normwise_rel(rf32, rf))
                worst = max(worst, vgg_ref.normwise_rel(got, rf) / gate)
        res["worst"] = worst
        res["layers"] = len(g0)


def _wrn_case(comm, rank, world, res):
    """Residual net with SyncBN on 2 ranks, g changing inside diamonds
    (test_wrn_executor.GS, ragged B=5): the BN sums travel through the
    symmetric heap's small allreduce, shortcuts through reshards."""
    from oracle import vgg_ref
    from paper_2112_10065_b200.executor import BurstStep
    from paper_2112_10065_b200.network import net_for_graph
    from paper_2112_10065_b200.planner import TrainingPlan
    from test_wrn_executor import GS, tiny_wrn_graph
    from test_wrn_gpu import margin_seed
    B = 5
    graph = tiny_wrn_graph(B, stem_c=32, stages=((32, 2, 8), (64, 2, 4)), classes=16)
    net = net_for_graph(graph)
    params, x, y = margin_seed(net, B)
    ids = [l.id for l in graph.layers if not l.is_virtual]
    p = TrainingPlan(graph.name, world, 2.0, B, tuple(zip(ids, GS)), 0.0, (), ())
    st = BurstStep(p, graph, comm=comm, params=params, lr=0.0)
    st.load(x, y)
    st.forward_backward()
    st.sync_and_update()
    torch.cuda.synchronize()
    res["loss"] = st.loss()
    res["last_g"] = GS[-1]
    g0 = {n: (a.cpu().clone(), b.cpu().clone()) for n, (a, b) in st.grads().items()}
    st.capture(warmup=1)
    st.step()
    torch.cuda.synchronize()
    comm.check()
    res["replay_same"] = _digest(st.grads()) == _digest(g0)
    res["grads"] = _digest(g0)
    if rank == 0:
        ref_loss, ref = vgg_ref.forward_backward(net, params, x, y, torch.float64)
        _, r32 = vgg_ref.forward_backward(net, params, x, y, torch.float32)
        res["ref_loss"] = ref_loss
        worst = 0.0
        errs = {}
        for n, (dw, db) in g0.items():
            for k, (got, rf, rf32) in enumerate(((dw, ref[n][0], r32[n][0]),
                                                 (db, ref[n][1], r32[n][1]))):
                gate = max(1e-3, 2 * vgg_ref.normwise_rel(rf32, rf))
                errs[(n, k)] = vgg_ref.normwise_rel(got, rf) / gate
                worst = max(worst, errs[(n, k)])
        res["worst"] = worst
        res["errs"] = errs


def _incep_case(comm, rank, world, res):
    """Four-tower net on 2 ranks with every kind of edge crossing 1 <-> 2
    GPUs (test_inception_executor.MIXED): fan-outs, concat parts and tower
    chains reshard through the symmetric heap."""
    from oracle import vgg_ref
    from paper_2112_10065_b200.executor import BurstStep
    from paper_2112_10065_b200.network import net_for_graph
    from paper_2112_10065_b200.planner import TrainingPlan
    from test_inception_executor import _gs, tiny_inception_graph
    from test_wrn_gpu import margin_seed
    B = 5
    graph = tiny_inception_graph(B, modules=2, classes=16)   # dense ops: out % 4 == 0
    net = net_for_graph(graph)
    params, x, y = margin_seed(net, B)
    gs = _gs(net, "mixed")
    ids = [l.id for l in graph.layers if not l.is_virtual]
    p = TrainingPlan(graph.name, world, 2.0, B, tuple(zip(ids, gs)), 0.0, (), ())
    st = BurstStep(p, graph, comm=comm, params=params, lr=0.0)
    st.load(x, y)
    st.forward_backward()
    st.sync_and_update()
    torch.cuda.synchronize()
    res["loss"] = st.loss()
    res["last_g"] = gs[-1]
    g0 = {n: (a.cpu().clone(), b.cpu().clone()) for n, (a, b) in st.grads().items()}
    st.capture(warmup=1)
    st.step()
    torch.cuda.synchronize()
    comm.check()
    res["replay_same"] = _digest(st.grads()) == _digest(g0)
    res["grads"] = _digest(g0)
    if rank == 0:
        ref_loss, ref = vgg_ref.forward_backward(net, params, x, y, torch.float64)
        _, r32 = vgg_ref.forward_backward(net, params, x, y, torch.float32)
        res["ref_loss"] = ref_loss
        worst, errs = 0.0, {}
        for n, (dw, db) in g0.items():
            for k, (got, rf, rf32) in enumerate(((dw, ref[n][0], r32[n][0]),
                                                 (db, ref[n][1], r32[n][1]))):
                gate = max(1e-3, 2 * vgg_ref.normwise_rel(rf32, rf))
                errs[(n, k)] = vgg_ref.normwise_rel(got, rf) / gate
                worst = max(worst, errs[(n, k)])
        res["worst"], res["errs"] = worst, errs


def _worker(rank, world, port, q, case):
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
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2112_10065_b200.comm import PeerComm
        from paper_2112_10065_b200.errors import CommError
        comm = PeerComm(rank, world, device="cuda:0",
                        timeout_s=3.0 if case == "timeout" else None)
        res = {}
        if case == "ops":
            B, bps = 7, 64
            src = torch.arange(B * bps, dtype=torch.uint8, device="cuda").view(B, bps)
            a, b = (0, 4) if rank == 0 else (4, 7)
            heap = comm.make_heap({"shard": (b - a) * bps, "full": B * bps,
                                   "big": 4 * 1000, "small": 4 * 10})
            mine = heap.view("shard", (b - a, bps), torch.uint8)
            mine.copy_(src[a:b])
            # 2 -> 1 reshard: rank 0 gathers every sample from the producers' buffers
            dst = torch.zeros(B, bps, dtype=torch.uint8, device="cuda") if rank == 0 else None
            heap.reshard("shard", 2, dst, 1, B, bps)
            torch.cuda.synchronize()
            if rank == 0:
                res["gather_ok"] = bool(torch.equal(dst, src))
            # 1 -> 2 reshard: rank 0 scatters out of its "full" buffer
            if rank == 0:
                heap.view("full", (B, bps), torch.uint8).copy_(src)
            out = torch.zeros(b - a, bps, dtype=torch.uint8, device="cuda")
            heap.reshard("full", 1, out, 2, B, bps)
            torch.cuda.synchronize()
            res["scatter_ok"] = bool(torch.equal(out, src[a:b]))
            # allreduce, two-shot (1000 floats) and one-shot (10), 3 rounds
            big, small = heap.view("big", (1000,)), heap.view("small", (10,))
            for k in range(3):
                big.copy_(torch.arange(1000, device="cuda", dtype=torch.float32) * (rank + 1) + k)
                small.fill_(float(rank + 1 + k))
                heap.allreduce("big", big, 2)
                heap.allreduce("small", small, 2)
                torch.cuda.synchronize()
                res[f"big{k}"] = big.cpu().tolist()   # plain data: workers exit first
                res[f"small{k}"] = float(small[0].item())
            # captured allreduce replays against fresh epochs
            gr = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                with torch.cuda.graph(gr):
                    heap.allreduce("big", big, 2)
            for _ in range(3):
                big.fill_(1.0)
                gr.replay()
            torch.cuda.synchronize()
            res["graph_big"] = float(big[999].item())
            comm.check()
        elif case == "timeout":
            # rank 1 never arrives: rank 0's barrier gives up after 3 s,
            # reports a timeout and aborts rank 1, whose next barrier fails fast
            if rank == 0:
                comm.barrier_dev(2)
                torch.cuda.synchronize()
                try:
                    comm.check()
                    res["raised"] = None
                except CommError as e:
                    res["raised"] = e.status
            dist.barrier()
            if rank == 1:
                comm.barrier_dev(2)
                torch.cuda.synchronize()
                res["status"] = comm.status()
        elif case in ("c1", "dp8"):
            _vgg16_b32_case(comm, rank, world, case, res)
        elif case == "wrn":
            _wrn_case(comm, rank, world, res)
        elif case == "incep":
            _incep_case(comm, rank, world, res)
        elif case == "step":
            from test_executor_dist import GS
            _step_case(comm, rank, world, GS, 5, res)
        else:
            _step_case(comm, rank, world, GS4, 7, res)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=850) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in out[r], out[r].get("error")
    return out


@pytest.mark.timeout(300)
def test_peer_reshard_and_allreduce_across_processes():
    out = _run("ops")
    assert out[0]["gather_ok"]
    assert out[0]["scatter_ok"] and out[1]["scatter_ok"]
    ar = torch.arange(1000, dtype=torch.float32)
    for k in range(3):
        ref = (ar * 1 + k) + (ar * 2 + k)
        assert out[0][f"big{k}"] == ref.tolist() and out[1][f"big{k}"] == ref.tolist()
        assert out[0][f"small{k}"] == out[1][f"small{k}"] == float(1 + k + 2 + k)
    assert out[0]["graph_big"] == out[1]["graph_big"] == 2.0


@pytest.mark.timeout(300)
def test_peer_barrier_times_out_and_aborts_instead_of_hanging():
    out = _run("timeout")
    assert out[0]["raised"] == 1          # timeout
    assert out[1]["status"] == 2          # aborted by rank 0


def _check_step(out, world):
    r0 = out[0]
    assert abs(r0["loss"] - r0["ref_loss"]) <= 1e-4 * abs(r0["ref_loss"])
    assert r0["worst"] <= 1.0, r0.get("errs")
    for r in range(world):
        assert out[r]["replay_same"]
        if r < out[0]["last_g"]:                  # ranks holding the loss layer
            assert out[r]["loss"] == r0["loss"]
        for n, h in out[r]["grads"].items():      # bitwise identical replicas
            assert h == r0["grads"][n], (r, n)


@pytest.mark.timeout(300)
def test_peer_backend_burst_step_matches_oracle_and_replays():
    _check_step(_run("step"), 2)


@pytest.mark.timeout(400)
def test_peer_backend_four_ranks_every_transition():
    _check_step(_run("step4", 4), 4)


def _check_vgg16(out, world):
    r0 = out[0]
    assert r0["layers"] == 16
    assert abs(r0["loss"] - r0["ref_loss"]) <= 1e-4 * abs(r0["ref_loss"])
    assert r0["worst"] <= 1.0, r0["worst"]
    for r in range(world):
        assert out[r]["replay_same"] and out[r]["replicas_same"]
        if r < r0["gs"][-1]:
            assert out[r]["loss"] == r0["loss"]


@pytest.mark.timeout(900)
def test_peer_backend_c1_plan_vgg16_b32_eight_ranks():
    out = _run("c1", 8)
    assert out[0]["gs"] == [8] * 10 + [4] * 4 + [1] * 7
    _check_vgg16(out, 8)


@pytest.mark.timeout(900)
def test_peer_backend_uniform_dp8_vgg16_b32():
    out = _run("dp8", 8)
    assert set(out[0]["gs"]) == {8}
    _check_vgg16(out, 8)


@pytest.mark.timeout(400)
def test_peer_backend_residual_net_syncbn_two_ranks():
    _check_step(_run("wrn", 2), 2)


@pytest.mark.timeout(400)
def test_peer_backend_branch_edges_across_gpu_counts():
    _check_step(_run("incep", 2), 2)

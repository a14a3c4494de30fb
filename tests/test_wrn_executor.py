"""Branch/join executor for the residual net behind the
reference's ``wideresnet_like`` family (synth.py:126-169), on CPU.

Drives the real ``BurstStep`` wiring -- shortcut fan-out and gradient
fan-in, stride-2 stage transitions with option-A shortcuts, global average
pool -- with the test-only torch op set (tests/cpu_kernels.py) and checks
loss and every weight gradient against the fp64 oracle (oracle/vgg_ref.py)."""

import math

import pytest
import torch

from paper_2112_10065_b200 import synth
from paper_2112_10065_b200.network import init_params, net_for_graph, synthetic_batch
from paper_2112_10065_b200.planner import TrainingPlan


def tiny_wrn_graph(batch, stem_c=8, stages=((16, 2, 8), (32, 2, 4)), classes=10):
    """A reduced wideresnet_like graph built like synth.wideresnet_like:
    stem, diamonds (conv1, conv2, add), pool, fc; (cout, blocks, hw) per stage."""
    net = synth._Net(0, synth.PROFILE_BATCHES_SMALL)
    hw0 = stages[0][2]
    head = net.layer("stem", "conv", 9 * 3 * stem_c, stem_c * hw0 * hw0 * 4, 1.0, 1, [])
    cin, k = stem_c, 0
    for cout, reps, hw in stages:
        for _ in range(reps):
            k += 1
            c1 = net.layer(f"res{k}_conv1", "conv", 9 * cin * cout, cout * hw * hw * 4, 1.0, 1,
                           [head])
            c2 = net.layer(f"res{k}_conv2", "conv", 9 * cout * cout, cout * hw * hw * 4, 1.0,
                           1, [c1])
            head = net.layer(f"res{k}_add", "add", 0, cout * hw * hw * 4, 0.01, 1, [c2, head])
            cin = cout
    pool = net.layer("pool", "pool", 0, cin * 4, 0.01, 1, [head])
    net.layer("fc", "dense", cin * classes, classes * 4, 1.0, 1, [pool])
    return net.finish("wideresnet_like", batch, synth.DEFAULT_BANDWIDTH,
                      synth.DEFAULT_DELAY_US, (3, hw0, hw0))


def one_gpu_plan(graph, g=1):
    ids = [l.id for l in graph.layers if not l.is_virtual]
    return TrainingPlan(graph.name, g, 2.0, graph.global_batch, tuple((i, g) for i in ids),
                        0.0, (), ())


def test_wideresnet_like_net_structure():
    net = net_for_graph(synth.wideresnet_like(seed=0, global_batch=32))
    assert len(net.layers) == 105 and net.input_hw == 100
    by = net.by_name()
    assert [l.name for l in net.layers if l.down] == ["res12_conv1", "res23_conv1"]
    assert [l.name for l in net.layers if l.skip_down] == ["res12_add", "res23_add"]
    assert by["res1_add"].skip == "stem" and by["res1_add"].skip_c == 64
    assert by["res12_add"].skip_c == 128 and by["res12_add"].cin == 256
    assert not by["res5_conv2"].relu and by["res5_conv1"].relu and by["res5_add"].relu
    assert by["pool"].kind == "gap" and by["fc"].cin == 512 and by["fc"].cout == 1000
    # conv FLOPs of the graph's own pricing (2*9*cin*cout*hw^2 per conv)
    g = synth.wideresnet_like(seed=0, global_batch=32)
    convs = [l for l in net.layers if l.kind == "conv"]
    assert sum(math.prod(c.param_shapes()[0]) for c in convs) == sum(
        l.params_bytes // 4 for l in g.layers if l.kind == "conv")


def test_tiny_wrn_step_matches_fp64_oracle():
    import cpu_kernels
    from oracle import vgg_ref
    from paper_2112_10065_b200.executor import BurstStep
    B = 3
    graph = tiny_wrn_graph(B)
    net = net_for_graph(graph)
    params = init_params(net, seed=5)
    x, y = synthetic_batch(net, B, seed=6)
    st = BurstStep(one_gpu_plan(graph), graph, params=params, kernels=cpu_kernels, lr=0.0)
    st.load(x, y)
    st.forward_backward()
    ref_loss, ref = vgg_ref.forward_backward(net, params, x, y, torch.float64)
    assert abs(st.loss() - ref_loss) <= 1e-6 * abs(ref_loss)
    grads = st.grads()
    assert len(grads) == 1 + 2 * 4 + 1
    for name, (dw, db) in grads.items():
        assert vgg_ref.normwise_rel(dw, ref[name][0]) < 1e-6, name
        assert vgg_ref.normwise_rel(db, ref[name][1]) < 1e-6, name


# world 2, ragged B=5, g changing inside diamonds: res1/res2 joins take the
# shortcut through a reshard, res3 (a stride-2 transition) has its conv1 on
# another g than its source (un-fused upsample + transfer, then a direct
# accumulate), res4 the same without the transition
GS = [2, 1, 2, 1, 1, 1, 2, 1, 2, 2, 1, 1, 2, 1, 1]
B2 = 5


def _worker(rank, port, q):
    try:
        import os
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.set_num_threads(1)
        import cpu_kernels
        from oracle import vgg_ref
        from paper_2112_10065_b200.comm import TorchComm
        from paper_2112_10065_b200.executor import BurstStep
        graph = tiny_wrn_graph(B2)
        net = net_for_graph(graph)
        params = init_params(net, seed=7)
        x, y = synthetic_batch(net, B2, seed=8)
        ids = [l.id for l in graph.layers if not l.is_virtual]
        p = TrainingPlan(graph.name, 2, 2.0, B2, tuple(zip(ids, GS)), 0.0, (), ())
        st = BurstStep(p, graph, comm=TorchComm(rank, 2, set(GS)), params=params,
                       kernels=cpu_kernels, lr=0.0)
        joins = {L.spec.name: L.join for L in st.layers if L.spec.kind == "add"}
        st.load(x, y)
        st.forward_backward()
        st.sync_and_update()
        res = {"loss": st.loss(), "joins": joins}
        if rank == 0:
            ref_loss, ref = vgg_ref.forward_backward(net, params, x, y, torch.float64)
            res["ref_loss"] = ref_loss
            res["errs"] = {n: max(vgg_ref.normwise_rel(dw, ref[n][0]),
                                  vgg_ref.normwise_rel(db, ref[n][1]))
                           for n, (dw, db) in st.grads().items()}
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


def test_world2_diamonds_across_gpu_counts_match_oracle():
    import socket
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in (0, 1):
        assert "error" not in out[r], out[r].get("error")
    r0 = out[0]
    assert r0["joins"] == {"res1_add": "reshard", "res2_add": "reshard",
                           "res3_add": "direct", "res4_add": "direct"}
    assert abs(r0["loss"] - r0["ref_loss"]) <= 1e-6 * abs(r0["ref_loss"])
    # rank 0 holds every layer's (allreduced) gradient: it is in every group
    assert len(r0["errs"]) == 10
    for name, e in r0["errs"].items():
        assert e < 1e-6, (name, e)


def tiny_resnet_graph(batch, hw=8, stages=((8, 2), (16, 1)), classes=10):
    """A reduced resnet50_like graph (bottleneck blocks) built like
    synth.resnet50_like."""
    net = synth._Net(2, synth.PROFILE_BATCHES_SMALL)

    def conv(name, cin, cout, k, h, preds):
        return net.layer(name, "conv", k * k * cin * cout, cout * h * h * 4, 1.0, 1, preds)

    head = conv("stem", 3, 8, 3, hw, [])
    cin, blk = 8, 0
    for s_, (w, reps) in enumerate(stages):
        for r in range(reps):
            blk += 1
            h_out = hw // 2 if (s_ > 0 and r == 0) else hw
            c1 = conv(f"res{blk}_c1_1x1", cin, w, 1, hw, [head])
            c2 = conv(f"res{blk}_c2", w, w, 3, h_out, [c1])
            c3 = conv(f"res{blk}_c3_1x1", w, 4 * w, 1, h_out, [c2])
            head = net.layer(f"res{blk}_add", "add", 0, 4 * w * h_out * h_out * 4, 0.01, 1,
                             [c3, head])
            cin, hw = 4 * w, h_out
    pool = net.layer("pool", "pool", 0, cin * 4, 0.01, 1, [head])
    net.layer("fc", "dense", cin * classes, classes * 4, 1.0, 1, [pool])
    return net.finish("resnet50_like", batch, synth.DEFAULT_BANDWIDTH,
                      synth.DEFAULT_DELAY_US, (3, 8, 8))


def test_resnet50_like_net_structure():
    net = net_for_graph(synth.resnet50_like())
    assert len(net.layers) == 1 + 16 * 4 + 2 and net.input_hw == 56
    by = net.by_name()
    assert by["res1_c1_1x1"].kind == "conv1x1" and by["res1_c2"].kind == "conv"
    assert [l.name for l in net.layers if l.down] == ["res4_c2", "res8_c2", "res14_c2"]
    assert by["res4_add"].skip_down and by["res4_add"].skip_c == 256
    assert by["fc"].cin == 2048 and not by["res1_c3_1x1"].relu


def test_tiny_bottleneck_step_matches_fp64_oracle():
    import cpu_kernels
    from oracle import vgg_ref
    from paper_2112_10065_b200.executor import BurstStep
    B = 3
    graph = tiny_resnet_graph(B)
    net = net_for_graph(graph)
    params = init_params(net, seed=9)
    x, y = synthetic_batch(net, B, seed=10)
    st = BurstStep(one_gpu_plan(graph), graph, params=params, kernels=cpu_kernels, lr=0.0)
    assert {L.spec.name: L.join for L in st.layers if L.spec.kind == "add"} == \
        {"res1_add": "direct", "res2_add": "direct", "res3_add": "direct"}
    st.load(x, y)
    st.forward_backward()
    ref_loss, ref = vgg_ref.forward_backward(net, params, x, y, torch.float64)
    assert abs(st.loss() - ref_loss) <= 1e-6 * abs(ref_loss)
    for name, (dw, db) in st.grads().items():
        assert vgg_ref.normwise_rel(dw, ref[name][0]) < 1e-6, name
        assert vgg_ref.normwise_rel(db, ref[name][1]) < 1e-6, name

"""Four-tower branch/join executor (SURVEY.md §8f-3, config C4 foreground)
for the net behind the reference's ``inception_like`` family
(synth.py:172-226), on CPU: 4-way fan-out of each module input (1x1 towers
and the pool tower), 4-way concat join, gradient fan-in by accumulation,
odd-pixel stride-2 transitions.  Test-only torch op set
(tests/cpu_kernels.py) against the fp64 oracle (oracle/vgg_ref.py)."""

import torch

from paper_2112_10065_b200 import synth
from paper_2112_10065_b200.network import init_params, net_for_graph, synthetic_batch
from paper_2112_10065_b200.planner import TrainingPlan


def tiny_inception_graph(batch, hw=9, modules=3, down_after=(1,), classes=10):
    """A reduced inception_like graph built like synth.inception_like: stem
    (2 convs, 3x3 pool, conv), `modules` four-tower modules, fc."""
    net = synth._Net(0, synth.PROFILE_BATCHES_SMALL)
    ch, half = 64, 32

    def conv(name, cout, preds, h):
        return net.layer(name, "conv", 9 * cout, cout * h * h * 4, 1.0, 1, preds)

    prev = [conv("stem_conv1", ch, [], hw)]
    prev = [conv("stem_conv2", ch, prev, hw)]
    prev = [net.layer("stem_pool", "pool", 0, ch * hw * hw * 4, 0.01, 1, prev)]
    prev = [conv("stem_conv5", ch, prev, hw)]
    for m in range(1, modules + 1):
        head = prev[0]
        t1 = conv(f"m{m}_t1_1x1", half, [head], hw)
        t2a = conv(f"m{m}_t2_1x1", half, [head], hw)
        t2b = conv(f"m{m}_t2_3x3", half, [t2a], hw)
        t3a = conv(f"m{m}_t3_1x1", half, [head], hw)
        t3b = conv(f"m{m}_t3_3x3", half, [t3a], hw)
        t3c = conv(f"m{m}_t3_3x3b", half, [t3b], hw)
        t4 = net.layer(f"m{m}_pool_proj", "pool", 0, half * hw * hw * 4, 0.01, 1, [head])
        prev = [net.layer(f"m{m}_concat", "concat", 0, 4 * half * hw * hw * 4, 0.01, 1,
                          [t1, t2b, t3c, t4])]
        if m in down_after:
            hw = (hw - 1) // 2
    net.layer("fc", "dense", 1000, classes * 4, 1.0, 1, prev)
    return net.finish("inception_like", batch, synth.DEFAULT_BANDWIDTH,
                      synth.DEFAULT_DELAY_US, (3, 9, 9))


def one_gpu_plan(graph, g=1):
    ids = [l.id for l in graph.layers if not l.is_virtual]
    return TrainingPlan(graph.name, g, 2.0, graph.global_batch, tuple((i, g) for i in ids),
                        0.0, (), ())


def test_inception_like_net_structure():
    net = net_for_graph(synth.inception_like(seed=0, global_batch=32))
    assert len(net.layers) == 119 and net.input_hw == 35
    by = net.by_name()
    assert by["m1_concat"].srcs == ("m1_t1_1x1", "m1_t2_3x3", "m1_t3_3x3b", "m1_pool_proj")
    assert by["m1_t2_1x1"].src == "stem_conv5" and by["m1_t2_1x1"].kind == "conv1x1"
    assert by["m1_pool_proj"].kind == "pool3" and by["m1_pool_proj"].cin == 64
    assert by["m2_pool_proj"].cin == 128 and by["m2_pool_proj"].cout == 32
    downs = [l.name for l in net.layers if l.down]
    assert downs == [f"m{m}_{t}" for m in (6, 11)
                     for t in ("t1_1x1", "t2_1x1", "t3_1x1", "pool_proj")]
    assert by["m6_t1_1x1"].in_hw == 35 and by["m6_t1_1x1"].sub_off == 1
    assert by["m11_t1_1x1"].in_hw == 17 and by["m11_t1_1x1"].hw == 8
    assert by["fc"].cin == 8 * 8 * 128 and by["fc"].cout == 1000


def test_tiny_inception_step_matches_fp64_oracle():
    import cpu_kernels
    from oracle import vgg_ref
    from paper_2112_10065_b200.executor import BurstStep
    B = 2
    graph = tiny_inception_graph(B)
    net = net_for_graph(graph)
    params = init_params(net, seed=3)
    x, y = synthetic_batch(net, B, seed=4)
    st = BurstStep(one_gpu_plan(graph), graph, params=params, kernels=cpu_kernels, lr=0.0)
    st.load(x, y)
    st.forward_backward()
    ref_loss, ref = vgg_ref.forward_backward(net, params, x, y, torch.float64)
    assert abs(st.loss() - ref_loss) <= 1e-6 * abs(ref_loss)
    grads = st.grads()
    assert len(grads) == 3 + 3 * 6 + 1
    for name, (dw, db) in grads.items():
        assert vgg_ref.normwise_rel(dw, ref[name][0]) < 1e-6, name
        assert vgg_ref.normwise_rel(db, ref[name][1]) < 1e-6, name


def test_reference_plans_of_branch_join_families_are_executable():
    """The reference planner's plans for C3 (wideresnet_like) and C4
    (inception_like) at G=8 keep branch edges and fan-outs on one GPU
    count, so the executor takes them as they are."""
    from paper_2112_10065_b200.executor import branch_topology
    from paper_2112_10065_b200.planner import plan
    for fam, amps in (("inception_like", (2.0, 4.0, 8.0)), ("wideresnet_like", (2.0, 4.0))):
        g = getattr(synth, fam)(seed=0, global_batch=32)
        net = net_for_graph(g)
        for amp in amps:
            p = plan(g, 8, amp)
            gs = [gg for lid, gg in p.assignments if not g.layer(lid).is_virtual]
            branch_topology(net.layers, gs)          # raises if not executable


# world 2, ragged B=5: the amp-2 plan's shape (stem on 2 GPUs, modules on 1)
# plus the classifier back on 2 -- chain transfers into and out of the
# branch/join section
# mixed: every kind of edge crossing g -- the module input fans out to
# towers on 1 and 2 GPUs, towers change g inside, concat parts arrive from
# both GPU counts and the concat itself alternates
MIXED = {"m1_t1_1x1": 2, "m1_t2_1x1": 1, "m1_t2_3x3": 2, "m1_t3_1x1": 2, "m1_t3_3x3": 1,
         "m1_t3_3x3b": 2, "m1_pool_proj": 1, "m1_concat": 2, "m2_t1_1x1": 1,
         "m2_t2_1x1": 2, "m2_t2_3x3": 2, "m2_t3_1x1": 1, "m2_t3_3x3": 1, "m2_t3_3x3b": 2,
         "m2_pool_proj": 2, "m2_concat": 1, "stem_conv5": 1}


def _gs(net, mode):
    if mode == "mixed":
        return [MIXED.get(l.name, 2) for l in net.layers]
    return [2 if (l.name.startswith("stem") and l.name != "stem_conv5") or l.name == "fc"
            else 1 for l in net.layers]


def _worker(rank, port, q, mode="amp2"):
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
        B = 5
        graph = tiny_inception_graph(B, modules=2)
        net = net_for_graph(graph)
        ids = [l.id for l in graph.layers if not l.is_virtual]
        gs = _gs(net, mode)
        params = init_params(net, seed=5)
        x, y = synthetic_batch(net, B, seed=6)
        p = TrainingPlan(graph.name, 2, 2.0, B, tuple(zip(ids, gs)), 0.0, (), ())
        st = BurstStep(p, graph, comm=TorchComm(rank, 2, set(gs)), params=params,
                       kernels=cpu_kernels, lr=0.0)
        st.load(x, y)
        st.forward_backward()
        st.sync_and_update()
        res = {"loss": st.loss()}
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


def _run_world2(mode):
    import socket
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ps = [ctx.Process(target=_worker, args=(r, port, q, mode)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in (0, 1):
        assert "error" not in out[r], out[r].get("error")
    r0 = out[0]
    assert abs(r0["loss"] - r0["ref_loss"]) <= 1e-6 * abs(r0["ref_loss"])
    assert len(r0["errs"]) == 3 + 2 * 6 + 1
    for name, e in r0["errs"].items():
        assert e < 1e-6, (name, e)


def test_world2_four_tower_net_matches_oracle():
    _run_world2("amp2")


def test_world2_branch_edges_across_gpu_counts_match_oracle():
    """Fan-outs, concat parts and tower chains crossing 1 <-> 2 GPUs."""
    from paper_2112_10065_b200.executor import BurstStep  # noqa: F401
    _run_world2("mixed")

"""Diagnostic: run the 2-rank tiny-VGG burst step (PeerComm, one GPU) and
check every conv layer's fp16x3 scale words against the tensors."""
import os
import sys
import torch
import torch.multiprocessing as mp
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def worker(rank, world, port, q):
    os.environ["CUDA_MODULE_LOADING"] = "EAGER"
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2112_10065_b200.comm import PeerComm
    from paper_2112_10065_b200 import synth
    from paper_2112_10065_b200.executor import BurstStep
    from paper_2112_10065_b200.network import init_params, synthetic_batch
    from paper_2112_10065_b200.planner import TrainingPlan
    from test_peercomm_gpu import gpu_tiny_vgg
    from test_executor_dist import GS
    comm = PeerComm(rank, world, device="cuda:0")
    net = gpu_tiny_vgg()
    B = 5
    graph = synth.vgg_like(seed=0, global_batch=B)
    ids = [l.id for l in graph.layers if not l.is_virtual]
    p = TrainingPlan("vgg_like", world, 2.0, B, tuple(zip(ids, GS)), 0.0, (), ())
    x, y = synthetic_batch(net, B, seed=4)
    st = BurstStep(p, graph, comm=comm, params=init_params(net, seed=3), net=net, lr=0.0)
    st.load(x, y)
    st.forward_backward()
    torch.cuda.synchronize()
    out = []
    for i, L in enumerate(st.layers):
        if L.amax is None or not L.active:
            continue
        w = lambda t: int(t.abs().max().view(torch.int32).item()) if t.numel() else 0  # noqa
        xa, da = int(L.amax[0]), int(L.amax[4])
        out.append((i, L.spec.name, L.g, L.x_fused, xa, w(L.x), L.dz_fused, da, w(L.dy)))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import socket
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in ps:
        pr.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for r in sorted(res):
        for row in res[r]:
            bad = (row[4] != row[5]) or (row[7] != row[8])
            print(r, row, "BAD" if bad else "")
    for pr in ps:
        pr.join()

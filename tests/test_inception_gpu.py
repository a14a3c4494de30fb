"""Four-tower net (inception_like, SURVEY.md §8f-3 / C4 foreground) on one
B200: the pool-tower / concat / offset-subsample kernels against the
test-only CPU op set, and a reduced-net training step through the executor
against the fp64 oracle with the §8c gate (tests/test_step_gpu.py)."""

import pytest
import torch

import cpu_kernels
from oracle import vgg_ref
from paper_2112_10065_b200 import ops
from paper_2112_10065_b200.executor import BurstStep
from paper_2112_10065_b200.network import init_params, net_for_graph, synthetic_batch
from test_inception_executor import one_gpu_plan, tiny_inception_graph

pytestmark = pytest.mark.gpu


def _rnd(*shape, seed=0):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(shape, generator=g)


def _same(got, ref):
    assert torch.allclose(got.cpu(), ref, rtol=1e-6, atol=1e-6), \
        (got.cpu() - ref).abs().max().item()


@pytest.mark.parametrize("n,h,c,cs", [(2, 9, 64, 64), (2, 35, 128, 32), (1, 8, 128, 32),
                                      (3, 1, 8, 4), (0, 5, 8, 8)])
def test_maxpool3x3(n, h, c, cs):
    x = _rnd(n, h, h, c, seed=1)
    y_ref, i_ref = torch.empty(n, h, h, cs), torch.empty(n, h, h, cs, dtype=torch.uint8)
    cpu_kernels.maxpool3x3_fwd_idx(x, y_ref, i_ref)
    y = torch.empty(n, h, h, cs, device="cuda")
    idx = torch.empty(n, h, h, cs, dtype=torch.uint8, device="cuda")
    ops.maxpool3x3_fwd_idx(x.cuda(), y, idx)
    _same(y, y_ref)
    assert torch.equal(idx.cpu(), i_ref)
    dy = _rnd(n, h, h, cs, seed=2)
    ref = cpu_kernels.maxpool3x3_bwd_idx(i_ref, dy, torch.empty(n, h, h, c))
    got = ops.maxpool3x3_bwd_idx(idx, dy.cuda(), torch.empty(n, h, h, c, device="cuda"))
    _same(got, ref)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_concat(k):
    parts = [_rnd(2, 5, 5, 4 * (j + 1), seed=j) for j in range(k)]
    C = sum(p.shape[-1] for p in parts)
    y = ops.concat_fwd([p.cuda() for p in parts], torch.empty(2, 5, 5, C, device="cuda"))
    _same(y, torch.cat(parts, dim=-1))
    dy = _rnd(2, 5, 5, C, seed=9)
    outs = [torch.empty_like(p).cuda() for p in parts]
    ops.concat_bwd(dy.cuda(), outs)
    ref = cpu_kernels.concat_bwd(dy, [torch.empty_like(p) for p in parts])
    for a, b in zip(outs, ref):
        _same(a, b)


@pytest.mark.parametrize("hin,h,off", [(35, 17, 1), (17, 8, 1), (16, 8, 0), (9, 4, 1)])
def test_subsample_offset(hin, h, off):
    x = _rnd(2, hin, hin, 8, seed=3)
    y = ops.subsample_fwd(x.cuda(), torch.empty(2, h, h, 8, device="cuda"), off)
    _same(y, x[:, off:off + 2 * h:2, off:off + 2 * h:2, :])
    dy = _rnd(2, h, h, 8, seed=4)
    got = ops.subsample_bwd(dy.cuda(), torch.empty(2, hin, hin, 8, device="cuda"), off)
    _same(got, cpu_kernels.subsample_bwd(dy, torch.empty(2, hin, hin, 8), off))


@pytest.mark.timeout(600)
def test_four_tower_net_step_matches_fp64():
    B = 2
    graph = tiny_inception_graph(B, hw=17, modules=3, down_after=(1,), classes=16)
    net = net_for_graph(graph)
    params = init_params(net, seed=0)
    x, y = synthetic_batch(net, B, seed=0)
    loss64, g64 = vgg_ref.forward_backward(net, params, x, y, torch.float64)
    loss32, g32 = vgg_ref.forward_backward(net, params, x, y, torch.float32)
    st = BurstStep(one_gpu_plan(graph), graph, params=params, lr=0.0)
    st.load(x, y)
    st.forward_backward()
    torch.cuda.synchronize()
    loss = st.loss()
    assert abs(loss - loss64) / abs(loss64) <= 1e-4, (loss, loss64)
    for name, (dw, db) in st.grads().items():
        for got, ref, ref32 in ((dw, g64[name][0], g32[name][0]),
                                (db, g64[name][1], g32[name][1])):
            e = vgg_ref.normwise_rel(got, ref)
            gate = max(1e-3, 2 * vgg_ref.normwise_rel(ref32, ref))
            assert e <= gate, (name, e, gate)
    g0 = {k: (a.clone(), b.clone()) for k, (a, b) in st.grads().items()}
    st.capture(warmup=1)
    st.step()
    torch.cuda.synchronize()
    for k, (a, b) in st.grads().items():
        assert torch.equal(a, g0[k][0]) and torch.equal(b, g0[k][1]), k


@pytest.mark.parametrize("b,fin,fout", [(4000, 128, 32), (2452, 64, 32), (39200, 128, 32),
                                        (578, 64, 32), (1000, 128, 32), (98, 2048, 512),
                                        (50, 64, 32)])
def test_pixel_batched_dense(b, fin, fout):
    """The 1x1 convs run as dense ops with batch = pixels (tensor-core engine
    for the forward); parity with fp64 like the other dense shapes."""
    x = torch.relu(_rnd(b, fin, seed=5))
    w = _rnd(fout, fin, seed=6) * 0.1
    bias = _rnd(fout, seed=7)
    y = ops.linear_fwd(x.cuda(), w.cuda(), bias.cuda(), torch.empty(b, fout, device="cuda"),
                       True)
    ref = torch.relu(x.double() @ w.double().T + bias.double())
    e = vgg_ref.normwise_rel(y, ref)
    e32 = vgg_ref.normwise_rel(torch.relu(x @ w.T + bias), ref)
    assert e <= max(2e-6, 2 * e32), (e, e32)
    dy = _rnd(b, fout, seed=8)
    dx = ops.linear_dgrad(dy.cuda(), w.cuda(), x.cuda(), torch.empty(b, fin, device="cuda"))
    ref = (dy.double() @ w.double()) * (x > 0)
    e = vgg_ref.normwise_rel(dx, ref)
    e32 = vgg_ref.normwise_rel((dy @ w) * (x > 0), ref)
    assert e <= max(2e-6, 2 * e32), (e, e32)
    dw = torch.empty(fout, fin, device="cuda")
    db = torch.empty(fout, device="cuda")
    ops.linear_wgrad(x.cuda(), dy.cuda(), dw, db)
    for got, ref, r32 in ((dw, dy.double().T @ x.double(), dy.T @ x),
                          (db, dy.double().sum(0), dy.sum(0))):
        e, e32 = vgg_ref.normwise_rel(got, ref), vgg_ref.normwise_rel(r32, ref)
        assert e <= max(2e-6, 2 * e32), (e, e32)

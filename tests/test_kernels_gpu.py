"""Per-kernel parity of libbpx against the CPU fp64 oracle (oracle/vgg_ref.py).

Gate: normwise relative error against fp64 <= max(2e-6, 4 x the error of
the same op computed in fp32 on the CPU).  fp32-accurate kernels (FFMA or
the 3xTF32 tensor-core split) pass; plain TF32 (~1e-3) fails by ~100x."""

import math

import pytest
import torch

from paper_2112_10065_b200 import ops
from paper_2112_10065_b200.network import LayerSpec
from oracle import vgg_ref

pytestmark = pytest.mark.gpu
DEV = "cuda"


def close(got, ref64, ref32):
    e = vgg_ref.normwise_rel(got, ref64)
    gate = max(2e-6, 4 * vgg_ref.normwise_rel(ref32, ref64))
    assert e <= gate, (e, gate)


def rnd(*shape, seed=0, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(shape, generator=g, dtype=torch.float32) * scale


def relu_input(*shape, seed=0):
    return torch.relu(rnd(*shape, seed=seed))


# (n, h, cin, cout): every VGG-16 conv channel pair at small spatial sizes,
# plus ragged pixel counts (M not a multiple of the 128-row tile) and n=1.
CONV_SHAPES = [
    (2, 16, 3, 64), (2, 16, 64, 64), (2, 12, 64, 128), (1, 10, 128, 128),
    (2, 8, 128, 256), (3, 7, 256, 256), (2, 6, 256, 512), (2, 4, 512, 512),
    (1, 14, 512, 512), (5, 9, 64, 64),
    # full-size images: 2-D output tiles with 4-D TMA halos (32x4 at 224,
    # 16x8 at 112) and the 64-channel stages of 64-wide N tiles
    (1, 224, 64, 64), (1, 112, 64, 128),
    # the four-tower net's 32 -> 32 tower convs (35 / 17 / 8 px; thin FFMA wgrad)
    (4, 35, 32, 32), (3, 17, 32, 32), (5, 8, 32, 32),
    # the residual net's 100 x 100 stage: 25 x 5 tiles (125 of 128 rows)
    (1, 100, 128, 128), (2, 100, 64, 128),
]


@pytest.mark.parametrize("shape", CONV_SHAPES, ids=str)
def test_conv_fwd(shape):
    n, h, cin, cout = shape
    x = rnd(n, h, h, cin, seed=1)
    w = rnd(cout, 3, 3, cin, seed=2, scale=math.sqrt(2 / (9 * cin)))
    b = rnd(cout, seed=3, scale=0.1)
    spec = LayerSpec("c", "conv", cin, cout, h, True, False)
    ref = vgg_ref.layer_fwd(spec, x, w, b)
    ref32 = vgg_ref.layer_fwd(spec, x, w, b, dtype=torch.float32)
    y = torch.empty(n, h, h, cout, device=DEV)
    ops.conv3x3_fwd(x.to(DEV), w.to(DEV), b.to(DEV), y, relu=True)
    if cin % 64 == 0 and cout % 64 == 0:
        assert ops.last_engine() == "fdt"
    torch.cuda.synchronize()
    close(y, ref, ref32)


@pytest.mark.parametrize("shape", [s for s in CONV_SHAPES if s[2] % 4 == 0], ids=str)
def test_conv_dgrad_masked(shape):
    n, h, cin, cout = shape
    x = relu_input(n, h, h, cin, seed=4)            # layer input = a ReLU output
    w = rnd(cout, 3, 3, cin, seed=5, scale=math.sqrt(2 / (9 * cin)))
    dz = rnd(n, h, h, cout, seed=6)
    dx_ref, _, _ = vgg_ref.conv_grads(x, w, dz)
    dx_ref = dx_ref * (x > 0)
    dx32 = vgg_ref.conv_grads(x, w, dz, torch.float32)[0] * (x > 0)
    dx = torch.empty(n, h, h, cin, device=DEV)
    ops.conv3x3_dgrad(dz.to(DEV), w.to(DEV), x.to(DEV), dx)
    if cin % 64 == 0 and cout % 64 == 0:
        assert ops.last_engine() == "fdt"
    torch.cuda.synchronize()
    close(dx, dx_ref, dx32)


@pytest.mark.parametrize("shape", CONV_SHAPES, ids=str)
def test_conv_wgrad(shape):
    n, h, cin, cout = shape
    x = relu_input(n, h, h, cin, seed=7)
    w = rnd(cout, 3, 3, cin, seed=8)
    dz = rnd(n, h, h, cout, seed=9)
    _, dw_ref, db_ref = vgg_ref.conv_grads(x, w, dz)
    _, dw32, db32 = vgg_ref.conv_grads(x, w, dz, torch.float32)
    dw = torch.empty(cout, 3, 3, cin, device=DEV)
    db = torch.empty(cout, device=DEV)
    ops.conv3x3_wgrad(x.to(DEV), dz.to(DEV), dw, db)
    if cin == cout == 32:
        assert ops.last_engine() == "thin"
    torch.cuda.synchronize()
    close(dw, dw_ref, dw32)
    close(db, db_ref, db32)


def test_conv_wgrad_large_k_split():
    # conv1_2-like reduction depth (split-K path), deterministic run to run
    n, h, cin, cout = 4, 56, 64, 64
    x = relu_input(n, h, h, cin, seed=10).to(DEV)
    dz = rnd(n, h, h, cout, seed=11).to(DEV)
    outs = []
    for _ in range(2):
        dw = torch.empty(cout, 3, 3, cin, device=DEV)
        db = torch.empty(cout, device=DEV)
        ops.conv3x3_wgrad(x, dz, dw, db)
        outs.append((dw.clone(), db.clone()))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    _, dw_ref, db_ref = vgg_ref.conv_grads(x.cpu(), torch.zeros(cout, 3, 3, cin), dz.cpu())
    _, dw32, _ = vgg_ref.conv_grads(x.cpu(), torch.zeros(cout, 3, 3, cin), dz.cpu(),
                                    torch.float32)
    close(outs[0][0], dw_ref, dw32)


def test_conv_matches_ffma_engine():
    # tensor-core engine vs the independent FFMA engine at a full VGG shape
    n, h, cin, cout = 2, 56, 256, 256
    x = relu_input(n, h, h, cin, seed=12).to(DEV)
    w = rnd(cout, 3, 3, cin, seed=13, scale=0.03).to(DEV)
    b = rnd(cout, seed=14).to(DEV)
    y1 = torch.empty(n, h, h, cout, device=DEV)
    y2 = torch.empty_like(y1)
    ops.conv3x3_fwd(x, w, b, y1, relu=True)
    ops.simt_conv3x3_fwd(x, w, b, y2, relu=True)
    torch.cuda.synchronize()
    spec = LayerSpec("c", "conv", cin, cout, h, True, False)
    ref = vgg_ref.layer_fwd(spec, x.cpu(), w.cpu(), b.cpu())
    ref32 = vgg_ref.layer_fwd(spec, x.cpu(), w.cpu(), b.cpu(), dtype=torch.float32)
    close(y1, ref, ref32)
    close(y2, ref, ref32)


@pytest.mark.parametrize("b,fin,fout,relu", [(4, 25088, 4096, True), (32, 4096, 4096, True),
                                             (32, 4096, 1000, False), (3, 64, 40, True),
                                             (1, 128, 1000, False), (17, 256, 384, True),
                                             (2, 512, 128, False), (12, 100, 36, True),
                                             (32, 25088, 4096, True),
                                             # pixel-batched 1x1 convs (thin FFMA engine)
                                             (1000, 128, 32, True), (2050, 64, 32, False),
                                             (39200, 128, 32, True)], ids=str)
def test_linear_fwd_bwd(b, fin, fout, relu):
    x = relu_input(b, fin, seed=15)
    w = rnd(fout, fin, seed=16, scale=0.01)
    bias = rnd(fout, seed=17, scale=0.1)
    dy = rnd(b, fout, seed=18)
    spec = LayerSpec("f", "dense", fin, fout, 0, relu, True)
    y_ref = vgg_ref.layer_fwd(spec, x, w, bias)
    xd, wd = x.double(), w.double()
    dx_ref = (dy.double() @ wd) * (x > 0)
    dw_ref = dy.double().t() @ xd
    db_ref = dy.double().sum(0)
    X, W = x.to(DEV), w.to(DEV)
    y = torch.empty(b, fout, device=DEV)
    ops.linear_fwd(X, W, bias.to(DEV), y, relu)
    dx = torch.empty(b, fin, device=DEV)
    ops.linear_dgrad(dy.to(DEV), W, X, dx)
    dw = torch.empty(fout, fin, device=DEV)
    db = torch.empty(fout, device=DEV)
    ops.linear_wgrad(X, dy.to(DEV), dw, db)
    if b > 256 and fout == 32:
        assert ops.last_engine() == "thin"
    torch.cuda.synchronize()
    y32 = vgg_ref.layer_fwd(spec, x, w, bias, dtype=torch.float32)
    dx32 = (dy @ w) * (x > 0)
    close(y, y_ref, y32)
    close(dx, dx_ref, dx32)
    close(dw, dw_ref, dy.t() @ x)
    close(db, db_ref, dy.sum(0))


@pytest.mark.parametrize("n,h,c", [(2, 8, 64), (3, 14, 512), (1, 224, 64), (2, 2, 4)])
def test_maxpool_fwd_bwd_exact(n, h, c):
    x = relu_input(n, h, h, c, seed=19)
    x[0, 0, 0, :] = 0.0                       # all-zero windows (ReLU ties)
    dy = rnd(n, h // 2, h // 2, c, seed=20)
    xr = x.double().permute(0, 3, 1, 2).requires_grad_(True)
    yr = torch.nn.functional.max_pool2d(xr, 2, 2)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    y = torch.empty(n, h // 2, h // 2, c, device=DEV)
    dx = torch.empty(n, h, h, c, device=DEV)
    ops.maxpool2x2_fwd(x.to(DEV), y)
    ops.maxpool2x2_bwd(x.to(DEV), dy.to(DEV), dx)
    # index variants: first-max positions recorded by the forward
    y2 = torch.empty_like(y)
    dx2 = torch.empty_like(dx)
    idx = torch.empty(y.shape, dtype=torch.uint8, device=DEV)
    ops.maxpool2x2_fwd_idx(x.to(DEV), y2, idx)
    ops.maxpool2x2_bwd_idx(idx, dy.to(DEV), dx2)
    torch.cuda.synchronize()
    assert torch.equal(y.cpu(), yr.detach().permute(0, 2, 3, 1).float())
    assert torch.equal(dx.cpu(), xr.grad.permute(0, 2, 3, 1).float())
    assert torch.equal(y2, y) and torch.equal(dx2, dx)


@pytest.mark.parametrize("b,bg", [(32, 32), (4, 32), (1, 8)])
def test_softmax_xent(b, bg):
    z = rnd(b, 1000, seed=21, scale=3.0)
    lab = torch.randint(0, 1000, (b,), generator=torch.Generator().manual_seed(3)).int()
    zr = z.double().requires_grad_(True)
    l = torch.nn.functional.cross_entropy(zr, lab.long(), reduction="sum") / bg
    l.backward()
    loss = torch.empty(b + 1, device=DEV)
    dz = torch.empty(b, 1000, device=DEV)
    ops.softmax_xent(z.to(DEV), lab.to(DEV), bg, loss, dz)
    torch.cuda.synchronize()
    assert abs(loss[0].item() - l.item()) / abs(l.item()) < 1e-6
    assert vgg_ref.normwise_rel(dz, zr.grad) < 1e-6


def test_sgd_update():
    w = rnd(1003, seed=22)
    g = rnd(1003, seed=23)
    W = w.to(DEV)
    ops.sgd_update(W, g.to(DEV), 0.1)
    torch.cuda.synchronize()
    # the GPU fuses w - lr*g into one FMA (single rounding)
    ref = (w.double() - 0.1 * g.double()).float()
    assert torch.allclose(W.cpu(), ref, atol=1e-7, rtol=1e-6)


def test_reshard_pull_with_local_peers():
    # 4 "peers" simulated as 4 buffers on one device: a g=4 -> h=1 gather of
    # B=10 samples (ceil layout 3,3,3,1) into rank 0, then 1 -> 4 scatter.
    from paper_2112_10065_b200.comm import reshard_moves
    from paper_2112_10065_b200.costs import reshard_segments, shard_range
    B, bps_f = 10, 48
    full = rnd(B, bps_f, seed=24)
    src = []
    for r in range(4):
        a, b = shard_range(B, 4, r)
        src.append(full[a:b].clone().to(DEV))
    dst = torch.empty(B, bps_f, device=DEV)
    segs = [(p, q, s, n) for p, q, s, n in reshard_segments(B, 4, 1)]
    ops.reshard_pull([src[p].data_ptr() for p, *_ in segs],
                     [(s - p * 3) * bps_f * 4 for p, q, s, n in segs], dst,
                     [s * bps_f * 4 for p, q, s, n in segs],
                     [n * bps_f * 4 for *_, n in segs])
    torch.cuda.synchronize()
    assert torch.equal(dst.cpu(), full)
    # scatter back with the moves this rank-r view computes
    for r in range(4):
        a, b = shard_range(B, 4, r)
        out = torch.empty(b - a, bps_f, device=DEV)
        segs = [sg for sg in reshard_segments(B, 1, 4) if sg[1] == r]
        ops.reshard_pull([dst.data_ptr()] * len(segs), [s * bps_f * 4 for _, _, s, _ in segs],
                         out, [(s - r * 3) * bps_f * 4 for _, _, s, _ in segs],
                         [n * bps_f * 4 for *_, n in segs])
        torch.cuda.synchronize()
        assert torch.equal(out.cpu(), full[a:b])


def test_allreduce_prefix_with_local_peers():
    n = 1 << 20
    bufs = [rnd(n, seed=30 + r).to(DEV) for r in range(4)]
    for g in (2, 4):
        out = torch.empty(n, device=DEV)
        ops.allreduce_sum_prefix([b.data_ptr() for b in bufs[:g]], out, n)
        torch.cuda.synchronize()
        ref = bufs[0].clone()
        for r in range(1, g):
            ref += bufs[r]
        assert torch.equal(out, ref)        # same fixed rank order


def test_signal_barrier_single_rank():
    pad = torch.zeros(1, dtype=torch.int32, device=DEV)
    ops.signal_barrier([pad.data_ptr()], 0, 7)
    torch.cuda.synchronize()
    assert pad.item() == 7


# ---- engine dispatch at the benchmarked per-GPU batches ----------------------
# Every VGG-16 conv / dense op at b = 32 (bench, N=1), 8 and 4 (the C1 plan's
# 4- and 8-GPU segments) must be served by a TMA tensor-core engine (or, for
# the <= 8-row dense weight gradient and the 1000-output classifier, the
# dense FFMA kernels chosen for them by measurement) -- never by a legacy
# engine (simt / ts / tc / wg / small).
ALLOWED = {
    "conv": {"fwd": {"fdt", "c1"}, "dgrad": {"fdt"}, "wgrad": {"wgh", "wgc", "wg1"}},
    "dense": {"fwd": {"dtc", "dns"}, "dgrad": {"dtc", "dns"}, "wgrad": {"dwt", "dns"}},
}


@pytest.mark.parametrize("b", [4, 8, 32])
def test_vgg16_ops_take_tensor_core_engines(b):
    from paper_2112_10065_b200.network import vgg16
    net = vgg16()
    ws = ops.Workspace(torch.device(DEV))
    seen = []
    for i, sp in enumerate(net.layers):
        if sp.kind not in ("conv", "dense"):
            continue
        x = torch.zeros(sp.in_shape(b), device=DEV)
        dy = torch.zeros(sp.out_shape(b), device=DEV)
        y = torch.empty_like(dy)
        dx = torch.empty_like(x)
        shapes = sp.param_shapes()
        w = torch.zeros(shapes[0], device=DEV)
        bias = torch.zeros(shapes[1], device=DEV)
        dw, db = torch.empty_like(w), torch.empty_like(bias)
        calls = []
        if sp.kind == "conv":
            ws.reserve(ops.conv_workspace_bytes(b, sp.hw, sp.hw, sp.cin, sp.cout))
            calls.append(("fwd", lambda: ops.conv3x3_fwd(x, w, bias, y, relu=True, ws=ws)))
            calls.append(("wgrad", lambda: ops.conv3x3_wgrad(x, dy, dw, db, ws=ws)))
            if i > 0:
                calls.append(("dgrad", lambda: ops.conv3x3_dgrad(dy, w, x, dx, ws=ws)))
        else:
            ws.reserve(ops.linear_workspace_bytes(b, sp.cin, sp.cout))
            x2, dx2 = x.view(b, sp.cin), dx.view(b, sp.cin)
            calls.append(("fwd", lambda: ops.linear_fwd(x2, w, bias, y, sp.relu, ws=ws)))
            calls.append(("wgrad", lambda: ops.linear_wgrad(x2, dy, dw, db, ws=ws)))
            calls.append(("dgrad", lambda: ops.linear_dgrad(dy, w, x2, dx2, ws=ws)))
        for op, fn in calls:
            fn()
            eng = ops.last_engine()
            seen.append((sp.name, op, eng))
            assert eng in ALLOWED[sp.kind][op], (b, sp.name, op, eng)
        torch.cuda.synchronize()
    assert len(seen) == 3 * 16 - 1


# ---- synchronised batch norm (bn_*): one rank holding the whole batch, so
# the local sums are the global ones; against torch's fp64 batch_norm
@pytest.mark.parametrize("n,h,c", [(4, 13, 64), (2, 7, 128), (3, 5, 2048), (1, 35, 32)])
def test_batchnorm_fwd_bwd(n, h, c):
    z = rnd(n, h, h, c, seed=40, scale=2.0) + 0.5
    g = rnd(n, h, h, c, seed=41)
    gb = torch.cat([rnd(c, seed=42, scale=0.1), 1.0 + rnd(c, seed=43, scale=0.1)])
    zz = z.double().permute(0, 3, 1, 2).requires_grad_(True)
    beta = gb[:c].double().requires_grad_(True)
    gamma = gb[c:].double().requires_grad_(True)
    yr = torch.nn.functional.batch_norm(zz, None, None, gamma, beta, True, 0.0, 1e-5)
    yr.backward(g.double().permute(0, 3, 1, 2))
    Z, G, GB = z.to(DEV), g.to(DEV), gb.to(DEV)
    st = torch.empty(2 * c, device=DEV)
    y = torch.empty_like(Z)
    ops.bn_stats(Z, st)
    ops.bn_apply(Z, st, GB, n * h * h, y, relu=False)
    sums = torch.empty(2 * c, device=DEV)
    ops.bn_bwd_sums(G, Z, st, n * h * h, sums)
    dz = torch.empty_like(Z)
    ops.bn_bwd_apply(G, Z, st, sums, GB, n * h * h, dz)
    torch.cuda.synchronize()
    assert vgg_ref.normwise_rel(y, yr.detach().permute(0, 2, 3, 1)) < 1e-6
    assert vgg_ref.normwise_rel(dz, zz.grad.permute(0, 2, 3, 1)) < 1e-5
    assert vgg_ref.normwise_rel(sums[:c], beta.grad) < 1e-6
    assert vgg_ref.normwise_rel(sums[c:], gamma.grad) < 1e-5
    # relu variant and bitwise reproducibility
    y2 = torch.empty_like(Z)
    ops.bn_apply(Z, st, GB, n * h * h, y2, relu=True)
    st2 = torch.empty_like(st)
    ops.bn_stats(Z, st2)
    torch.cuda.synchronize()
    assert torch.equal(y2, torch.relu(y)) and torch.equal(st, st2)


@pytest.mark.parametrize("scale", [1e-30, 1e-7, 1e5, 1e30], ids=str)
def test_conv_fp16x3_scaling(scale):
    # fp16x3 operands carry a power-of-two scale from each tensor's max |v|:
    # the result is scale-invariant far outside fp16's own range, and
    # elements ~2^-20 below the max keep their share of the norm
    n, h, cin, cout = 2, 12, 64, 128
    x = rnd(n, h, h, cin, seed=21) * scale
    x[0, :3] *= 2.0 ** -20
    w = rnd(cout, 3, 3, cin, seed=22, scale=0.05 / scale ** 0.5)
    w[:7] *= 2.0 ** -18
    b = torch.zeros(cout)
    spec = LayerSpec("c", "conv", cin, cout, h, False, False)
    ref = vgg_ref.layer_fwd(spec, x, w, b)
    ref32 = vgg_ref.layer_fwd(spec, x, w, b, dtype=torch.float32)
    y = torch.empty(n, h, h, cout, device=DEV)
    ops.conv3x3_fwd(x.to(DEV), w.to(DEV), b.to(DEV), y, relu=False)
    dz = rnd(n, h, h, cout, seed=23) * scale
    dx_ref = vgg_ref.conv_grads(x, w, dz)[0]
    dx32 = vgg_ref.conv_grads(x, w, dz, torch.float32)[0]
    dx = torch.empty(n, h, h, cin, device=DEV)
    ops.conv3x3_dgrad(dz.to(DEV), w.to(DEV), None, dx)
    torch.cuda.synchronize()
    close(y, ref, ref32)
    close(dx, dx_ref, dx32)
    # the rescaled rows too (normwise over them alone)
    close(y[0, :3], ref[0, :3], ref32[0, :3])


def test_f16_split_roundtrip():
    # hi + lo reproduces w to 2^-22 relative (RN halves), scale from max |w|
    w = rnd(4096, seed=24) * 3.0
    w[:16] *= 2.0 ** -30
    sp = ops.F16Split(w.to(DEV)).refresh(w.to(DEV))
    torch.cuda.synchronize()
    back = sp.dequant().cpu()
    amax = int(sp.amax[0].item()) & 0xFFFFFFFF
    assert amax == int(w.abs().max().view(torch.int32).item())
    err = (back - w.double()).abs()
    rel = (err[16:] / w.double()[16:].abs()).max().item()
    assert rel < 2.0 ** -21, rel
    # below fp16's normal range the split is exact to 2^-25 in scaled units
    s = ops.f16_scale_exp(amax)
    assert err[:16].max().item() <= 2.0 ** (-24 - s), err[:16].max().item()


def test_f16_split_batch_matches_single():
    ws = [rnd(64, 3, 3, 64, seed=30).to(DEV), rnd(8, seed=31).to(DEV) * 1e-9,
          rnd(128, 3, 3, 64, seed=32).to(DEV) * 7.0]
    b = ops.F16SplitBatch(ws).refresh()
    for w, sp in zip(ws, b.splits):
        one = ops.F16Split(w).refresh(w)
        torch.cuda.synchronize()
        assert torch.equal(sp.hi, one.hi) and torch.equal(sp.lo, one.lo)
        assert int(sp.amax[0]) == int(one.amax[0])


def test_producers_reduce_amax():
    # fused max |v| words: conv fwd (fdt, c1), conv dgrad, maxpool fwd / bwd
    def word(t):
        return int(t.abs().max().view(torch.int32).item())

    z = lambda: torch.zeros(4, dtype=torch.int32, device=DEV)      # noqa: E731
    for (n, h, cin, cout) in [(2, 16, 64, 128), (1, 14, 512, 512), (2, 16, 3, 64)]:
        x = rnd(n, h, h, cin, seed=33).to(DEV)
        w = rnd(cout, 3, 3, cin, seed=34, scale=0.05).to(DEV)
        b = rnd(cout, seed=35).to(DEV)
        y = torch.empty(n, h, h, cout, device=DEV)
        ya = z()
        ops.conv3x3_fwd(x, w, b, y, relu=True, y_amax=ya)
        torch.cuda.synchronize()
        assert int(ya[0]) == word(y), (n, h, cin, cout)
        if cin % 64 == 0:
            dz = rnd(n, h, h, cout, seed=36).to(DEV)
            dx = torch.empty_like(x)
            da = z()
            ops.conv3x3_dgrad(dz, w, torch.relu(x), dx, dx_amax=da)
            torch.cuda.synchronize()
            assert int(da[0]) == word(dx)
    x = rnd(2, 8, 8, 64, seed=37).to(DEV)
    y = torch.empty(2, 4, 4, 64, device=DEV)
    idx = torch.empty(2, 4, 4, 64, dtype=torch.uint8, device=DEV)
    ya = z()
    ops.maxpool2x2_fwd_idx(x, y, idx, y_amax=ya)
    dy = rnd(2, 4, 4, 64, seed=38).to(DEV)
    dx = torch.empty_like(x)
    da = z()
    ops.maxpool2x2_bwd_idx(idx, dy, dx, dx_amax=da)
    torch.cuda.synchronize()
    assert int(ya[0]) == word(y) and int(da[0]) == word(dx)
    # the residual nets' producers: BN normalise / BN backward, residual join
    # (same-shape flat path and the stride-2 transition), first conv's x
    c = 128
    zt = rnd(2, 10, 10, c, seed=39, scale=2.0).to(DEV)
    gt = rnd(2, 10, 10, c, seed=40).to(DEV)
    gb = torch.cat([torch.zeros(c), torch.ones(c)]).to(DEV)
    st = torch.empty(2 * c, device=DEV)
    ops.bn_stats(zt, st)
    yb, ya = torch.empty_like(zt), z()
    ops.bn_apply(zt, st, gb, 200, yb, relu=True, y_amax=ya)
    sums, dzb, da = torch.empty(2 * c, device=DEV), torch.empty_like(zt), z()
    ops.bn_bwd_sums(gt, zt, st, 200, sums)
    ops.bn_bwd_apply(gt, zt, st, sums, gb, 200, dzb, dz_amax=da)
    torch.cuda.synchronize()
    assert int(ya[0]) == word(yb) and int(da[0]) == word(dzb)
    for s_shape in ((2, 10, 10, c), (2, 20, 20, 64)):
        sk = rnd(*s_shape, seed=41).to(DEV)
        yr, ra = torch.empty_like(zt), z()
        ops.residual_add_fwd(zt, sk, yr, relu=True, y_amax=ra)
        torch.cuda.synchronize()
        assert int(ra[0]) == word(yr), s_shape
    xi = rnd(2, 16, 16, 3, seed=42).to(DEV)
    wi = rnd(64, 3, 3, 3, seed=43, scale=0.1).to(DEV)
    yi, xa = torch.empty(2, 16, 16, 64, device=DEV), z()
    ops.conv3x3_fwd(xi, wi, torch.zeros(64, device=DEV), yi, relu=True, x_amax=xa)
    torch.cuda.synchronize()
    assert ops.last_engine() == "c1" and int(xa[0]) == word(xi)


@pytest.mark.parametrize("shape", [(2, 80, 64, 64), (1, 224, 64, 64)], ids=str)
def test_conv_wgrad_resident_tiles(shape):
    # the Cin = Cout = 64 engine (all five M tiles resident, x halo per 16x4
    # block, promotion into per-CTA slabs): fp64 parity and run-to-run equality
    n, h, cin, cout = shape
    x = relu_input(n, h, h, cin, seed=40)
    dz = rnd(n, h, h, cout, seed=41)
    _, dw_ref, db_ref = vgg_ref.conv_grads(x, torch.zeros(cout, 3, 3, cin), dz)
    _, dw32, db32 = vgg_ref.conv_grads(x, torch.zeros(cout, 3, 3, cin), dz, torch.float32)
    outs = []
    for _ in range(2):
        dw = torch.empty(cout, 3, 3, cin, device=DEV)
        db = torch.empty(cout, device=DEV)
        ops.conv3x3_wgrad(x.to(DEV), dz.to(DEV), dw, db)
        assert ops.last_engine() == "wgc"
        outs.append((dw, db))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    close(outs[0][0], dw_ref, dw32)
    close(outs[0][1], db_ref, db32)


@pytest.mark.parametrize("shape", [(2, 224, 3, 64), (3, 32, 3, 64)], ids=str)
def test_conv_wgrad_first_layer(shape):
    # Cin = 3: im2col rows in every TMEM lane quadrant, x halo by TMA
    n, h, cin, cout = shape
    x = rnd(n, h, h, cin, seed=42)
    dz = rnd(n, h, h, cout, seed=43)
    _, dw_ref, db_ref = vgg_ref.conv_grads(x, torch.zeros(cout, 3, 3, cin), dz)
    _, dw32, db32 = vgg_ref.conv_grads(x, torch.zeros(cout, 3, 3, cin), dz, torch.float32)
    dw = torch.empty(cout, 3, 3, cin, device=DEV)
    db = torch.empty(cout, device=DEV)
    ops.conv3x3_wgrad(x.to(DEV), dz.to(DEV), dw, db)
    assert ops.last_engine() == "wg1"
    torch.cuda.synchronize()
    close(dw, dw_ref, dw32)
    close(db, db_ref, db32)


def test_split_k_paths_deterministic():
    """Split-K paths (fixed-order finishes): conv5 fwd / dgrad at B = 32
    (fdt split-K), a wgrad with K splits (wgh, weight + bias partials
    reduced in one launch), fc fwd / dgrad (dtc with the activations' lo
    split made in-kernel, dns): two runs are bitwise equal and match
    fp64."""
    n, h, c = 32, 14, 512
    x = relu_input(n, h, h, c, seed=41)
    w = rnd(c, 3, 3, c, seed=42, scale=math.sqrt(2 / (9 * c)))
    b = rnd(c, seed=43, scale=0.1)
    dz = rnd(n, h, h, c, seed=44)
    X, Wd, B, DZ = x.to(DEV), w.to(DEV), b.to(DEV), dz.to(DEV)
    outs = []
    for _ in range(2):
        y = torch.empty(n, h, h, c, device=DEV)
        ops.conv3x3_fwd(X, Wd, B, y, relu=True)
        dx = torch.empty(n, h, h, c, device=DEV)
        ops.conv3x3_dgrad(DZ, Wd, X, dx)
        dw = torch.empty(c, 3, 3, c, device=DEV)
        db = torch.empty(c, device=DEV)
        ops.conv3x3_wgrad(X, DZ, dw, db)
        outs.append((y, dx, dw, db))
    torch.cuda.synchronize()
    for a, b2 in zip(*outs):
        assert torch.equal(a, b2)
    spec = LayerSpec("c", "conv", c, c, h, True, False)
    close(outs[0][0], vgg_ref.layer_fwd(spec, x, w, b),
          vgg_ref.layer_fwd(spec, x, w, b, dtype=torch.float32))
    dx_ref, dw_ref, db_ref = vgg_ref.conv_grads(x, w, dz)
    dx32, dw32, db32 = vgg_ref.conv_grads(x, w, dz, torch.float32)
    close(outs[0][1], dx_ref * (x > 0), dx32 * (x > 0))
    close(outs[0][2], dw_ref, dw32)
    close(outs[0][3], db_ref, db32)
    for fin, fout in ((25088, 4096), (4096, 1000)):
        xa = relu_input(32, fin, seed=45).to(DEV)
        wa = rnd(fout, fin, seed=46, scale=0.01).to(DEV)
        ba = rnd(fout, seed=47, scale=0.1).to(DEV)
        dya = rnd(32, fout, seed=48).to(DEV)
        res = []
        for _ in range(2):
            ya = torch.empty(32, fout, device=DEV)
            ops.linear_fwd(xa, wa, ba, ya, True)
            dxa = torch.empty(32, fin, device=DEV)
            ops.linear_dgrad(dya, wa, xa, dxa)
            res.append((ya, dxa))
        torch.cuda.synchronize()
        for a, b2 in zip(*res):
            assert torch.equal(a, b2)
        y64 = torch.relu(xa.double() @ wa.double().t() + ba.double())
        assert vgg_ref.normwise_rel(res[0][0].cpu(), y64.cpu()) < 2e-6

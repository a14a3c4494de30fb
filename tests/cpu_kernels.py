"""TEST-ONLY op set with the libbpx call signatures, implemented with torch
on CPU (fp64 inside, results written into the executor's fp32 buffers).

Lets tests drive ``BurstStep``'s multi-rank orchestration (shard ranges,
reshards in both directions, prefix allreduce, loss partials) over gloo
without a GPU.  Never imported by the product."""

import torch
import torch.nn.functional as F


class Workspace:
    def __init__(self, device):
        pass

    def reserve(self, n):
        pass


def conv_workspace_bytes(*a):
    return 0


def linear_workspace_bytes(*a):
    return 0


def _nchw(t):
    return t.double().permute(0, 3, 1, 2)


def _nhwc(t):
    return t.permute(0, 2, 3, 1)


def conv3x3_fwd(x, w, bias, y, relu=True, ws=None):
    if x.shape[0] == 0:
        return y
    o = F.conv2d(_nchw(x), w.double().permute(0, 3, 1, 2),
                 None if bias is None else bias.double(), padding=1)
    y.copy_(_nhwc(F.relu(o) if relu else o))
    return y


def conv3x3_dgrad(dz, w, mask, dx, ws=None):
    if dz.shape[0] == 0:
        return dx
    cin = w.shape[3]
    shape = (dz.shape[0], cin, dz.shape[1], dz.shape[2])
    g = torch.nn.grad.conv2d_input(shape, w.double().permute(0, 3, 1, 2), _nchw(dz), padding=1)
    g = _nhwc(g)
    if mask is not None:
        g = g * (mask > 0)
    dx.copy_(g)
    return dx


def conv3x3_wgrad(x, dz, dw, dbias, ws=None):
    if x.shape[0] == 0:
        dw.zero_()
        if dbias is not None:
            dbias.zero_()
        return dw
    g = torch.nn.grad.conv2d_weight(_nchw(x), (dw.shape[0], dw.shape[3], 3, 3), _nchw(dz),
                                    padding=1)
    dw.copy_(g.permute(0, 2, 3, 1))
    if dbias is not None:
        dbias.copy_(dz.double().sum(dim=(0, 1, 2)))
    return dw


def linear_fwd(x, w, bias, y, relu, ws=None):
    o = x.double() @ w.double().t()
    if bias is not None:
        o = o + bias.double()
    y.copy_(F.relu(o) if relu else o)
    return y


def linear_dgrad(dy, w, mask, dx, ws=None):
    g = dy.double() @ w.double()
    if mask is not None:
        g = g * (mask > 0)
    dx.copy_(g)
    return dx


def linear_wgrad(x, dy, dw, dbias, ws=None):
    dw.copy_(dy.double().t() @ x.double())
    if dbias is not None:
        dbias.copy_(dy.double().sum(0))
    return dw


# synchronised BN (libbpx bn_*: local sums, the executor allreduces them)
def bn_workspace_bytes(*a):
    return 0


def _pc(t):
    return t.double().reshape(-1, t.shape[-1])


def _coef(stats, ntot, eps):
    c = stats.numel() // 2
    m = stats[:c].double() / ntot
    v = (stats[c:].double() / ntot - m * m).clamp_min(0)
    return m, 1.0 / torch.sqrt(v + eps)


def bn_stats(z, stats, ws=None):
    zz = _pc(z)
    stats.copy_(torch.cat([zz.sum(0), (zz * zz).sum(0)]))


def bn_apply(z, stats, gb, ntot, y, relu, eps=1e-5):
    c = z.shape[-1]
    m, r = _coef(stats, ntot, eps)
    o = (_pc(z) - m) * r * gb[c:].double() + gb[:c].double()
    y.copy_((F.relu(o) if relu else o).reshape(y.shape))


def bn_bwd_sums(g, z, stats, ntot, sums, ws=None, eps=1e-5):
    m, r = _coef(stats, ntot, eps)
    gg, xh = _pc(g), (_pc(z) - m) * r
    sums.copy_(torch.cat([gg.sum(0), (gg * xh).sum(0)]))


def bn_bwd_apply(g, z, stats, sums, gb, ntot, dz, eps=1e-5):
    c = z.shape[-1]
    m, r = _coef(stats, ntot, eps)
    xh = (_pc(z) - m) * r
    t0, t1 = sums[:c].double() / ntot, sums[c:].double() / ntot
    d = gb[c:].double() * r * (_pc(g) - t0 - xh * t1)
    dz.copy_(d.reshape(dz.shape))


def maxpool2x2_fwd(x, y):
    if x.shape[0]:
        y.copy_(_nhwc(F.max_pool2d(_nchw(x), 2, 2)))
    return y


def maxpool2x2_bwd(x, dy, dx):
    if x.shape[0] == 0:
        return dx
    xx = _nchw(x).detach().requires_grad_(True)
    F.max_pool2d(xx, 2, 2).backward(_nchw(dy))
    dx.copy_(_nhwc(xx.grad))
    return dx


def softmax_xent(logits, labels, b_global, loss_out, dlogits):
    b = logits.shape[0]
    if b == 0:
        loss_out.zero_()
        return loss_out
    z = logits.double().detach().requires_grad_(True)
    l = F.cross_entropy(z, labels.long(), reduction="sum") / b_global
    l.backward()
    loss_out[0] = l.item()
    dlogits.copy_(z.grad)
    return loss_out


def sgd_update(w, g, lr):
    w.sub_(lr * g)


# ---- residual-net elements (include/bpx.h: bpx_residual_*, subsample2,
# global_avgpool), same semantics as the CUDA kernels
def _shortcut(s, h, c):
    """P(s): stride-2 subsample when s is 2h x 2h, zero channels up to c."""
    if s.shape[1] == 2 * h:
        s = s[:, ::2, ::2, :]
    if s.shape[3] < c:
        s = F.pad(s, (0, c - s.shape[3]))
    return s


def residual_add_fwd(a, s, y, relu=True):
    o = a.double() + _shortcut(s.double(), a.shape[1], a.shape[3])
    y.copy_(F.relu(o) if relu else o)
    return y


def residual_skip_bwd(dz, mask, dh, dmain=None, accumulate=True):
    f = 2 if dh.shape[1] == 2 * dz.shape[1] else 1
    cs = dh.shape[3]
    g = torch.zeros(dh.shape, dtype=torch.float64)
    low = dz.double()[..., :cs] * (mask.double()[:, ::f, ::f, :] > 0)
    if dmain is not None:
        low = low + dmain.double()
    g[:, ::f, ::f, :] = low
    if accumulate:
        g = g + dh.double()
    dh.copy_(g)
    return dh


def subsample2_fwd(x, y):
    y.copy_(x[:, ::2, ::2, :])
    return y


def global_avgpool_fwd(x, y):
    y.copy_(x.double().mean(dim=(1, 2)))
    return y


def global_avgpool_bwd(dy, mask, dx):
    hw = dx.shape[1] * dx.shape[2]
    g = (dy.double() / hw)[:, None, None, :].expand(dx.shape)
    if mask is not None:
        g = g * (mask > 0)
    dx.copy_(g)
    return dx


def subsample2_bwd(dy, dx):
    dx.zero_()
    dx[:, ::2, ::2, :] = dy
    return dx


def accumulate(dst, src):
    dst.copy_(dst.double() + src.double().reshape(dst.shape))
    return dst


# ---- four-tower (inception_like) elements: bpx_maxpool3x3_*, bpx_concat_*,
# bpx_subsample_*
def maxpool3x3_fwd_idx(x, y, idx):
    cs = y.shape[3]
    xs = _nchw(x[..., :cs])
    o, ind = F.max_pool2d(xs, 3, 1, 1, return_indices=True)
    y.copy_(_nhwc(o))
    # flat index in the (h, w) plane -> window position (dy+1)*3 + (dx+1)
    h, w = x.shape[1], x.shape[2]
    oh = torch.arange(h).view(1, 1, h, 1)
    ow = torch.arange(w).view(1, 1, 1, w)
    ih, iw = ind // w, ind % w
    idx.copy_(_nhwc((ih - oh + 1) * 3 + (iw - ow + 1)).to(torch.uint8))
    return y


def maxpool3x3_bwd_idx(idx, dy, dx):
    n, h, w, c = dx.shape
    cs = dy.shape[3]
    g = torch.zeros((n, h, w, c), dtype=torch.float64)
    k = idx.long()
    for t in range(9):
        ddy, ddx = t // 3 - 1, t % 3 - 1
        sel = (k == t).double() * dy.double()        # outputs whose max sits at tap t
        for oh in range(h):
            ih = oh + ddy
            if not 0 <= ih < h:
                continue
            lo, hi = max(0, -ddx), min(w, w - ddx)
            g[:, ih, lo + ddx:hi + ddx, :cs] += sel[:, oh, lo:hi, :]
    dx.copy_(g)
    return dx


def concat_fwd(parts, y):
    y.copy_(torch.cat([p.double() for p in parts], dim=-1))
    return y


def concat_bwd(dy, parts):
    o = 0
    for p in parts:
        c = p.shape[-1]
        p.copy_(dy[..., o:o + c])
        o += c
    return parts


def subsample_fwd(x, y, off):
    h, w = y.shape[1], y.shape[2]
    y.copy_(x[:, off:off + 2 * h:2, off:off + 2 * w:2, :])
    return y


def subsample_bwd(dy, dx, off):
    h, w = dy.shape[1], dy.shape[2]
    dx.zero_()
    dx[:, off:off + 2 * h:2, off:off + 2 * w:2, :] = dy
    return dx

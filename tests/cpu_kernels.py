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
    o = F.conv2d(_nchw(x), w.double().permute(0, 3, 1, 2), bias.double(), padding=1)
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
        dbias.zero_()
        return dw
    g = torch.nn.grad.conv2d_weight(_nchw(x), (dw.shape[0], dw.shape[3], 3, 3), _nchw(dz),
                                    padding=1)
    dw.copy_(g.permute(0, 2, 3, 1))
    dbias.copy_(dz.double().sum(dim=(0, 1, 2)))
    return dw


def linear_fwd(x, w, bias, y, relu, ws=None):
    o = x.double() @ w.double().t() + bias.double()
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
    dbias.copy_(dy.double().sum(0))
    return dw


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

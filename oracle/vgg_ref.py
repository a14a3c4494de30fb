"""CPU numerics oracle for one burst-parallel training step.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product.

The reference toolkit has no forward/backward at all (it prices a
`compute` op per layer: /root/reference/pkg/src/burstplan/simulator.py:254-261,
synth.py:86-123), so this is a restatement of the *paper's* step
 for the networks of `paper_2112_10065_b200.network`
(VGG-16; the residual net behind `wideresnet_like`: conv with an optional
stride-2 input subsample, residual `add` with a ResNet option-A shortcut,
global average pool; the four-tower net behind `inception_like`: 1x1 convs,
3x3/s1 max pool over a channel subset, channel concat, branch inputs):
forward layer by layer (the residual nets' convs followed by BatchNorm
over the whole global batch: the executor's SyncBN over [0, g) is plan-
independent), mean softmax cross-entropy over the global batch,
backward, per-layer weight gradients.  Numerics parity is therefore
"unpinned" against the reference (no golden vectors exist there); it is
pinned against this oracle in fp64, with the tolerance stated in
tests/test_step_gpu.py (SURVEY.md §8c gate).

Layouts follow the product: NHWC activations, OHWI conv weights, dense
weights [out][in], fc1 input in NHWC-flatten order.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F


def _relu(h, margins):
    if margins is not None:
        margins.append(float(h.detach().abs().min()))
    return F.relu(h)


def forward_backward(net, params, x_nhwc, labels, dtype=torch.float64,
                     threads=None, margins=None):
    """Return (loss, grads) with grads[name] = (dW, db) in product layouts.

    ``params``: dict name -> (w, b) CPU tensors; ``labels`` int tensor.
    The loss is the mean over the batch given (= the global batch).
    ``margins`` (a list, optional) receives min |pre-activation| of every
    ReLU: a value inside the fp32 error band can flip the ReLU mask between
    two fp32-accurate implementations, and one flipped element moves every
    upstream gradient by ~1/sqrt(elements) (tests pick inputs with a margin).
    """
    if threads:
        torch.set_num_threads(threads)
    leaves = {}
    for name, (w, b) in params.items():
        leaves[name] = (w.detach().to(dtype).clone().requires_grad_(True),
                        b.detach().to(dtype).clone().requires_grad_(True))
    h = x_nhwc.to(dtype).permute(0, 3, 1, 2).contiguous()       # NCHW
    flat = False
    outs = {}
    for l in net.layers:
        src = getattr(l, "src", None)
        if src is not None:                  # branch edge: input from a named layer
            h = outs[src]
            flat = h.dim() == 2
        if getattr(l, "down", False):        # stride-2 subsample (offset 0 or 1)
            off = l.sub_off
            h = h[:, :, off:off + 2 * l.hw:2, off:off + 2 * l.hw:2]
        if l.kind == "conv":
            w, b = leaves[l.name]
            if getattr(l, "bn", False):      # conv -> BatchNorm (full batch) -> ReLU
                h = F.conv2d(h, w.permute(0, 3, 1, 2), None, padding=1)
                h = F.batch_norm(h, None, None, b[l.cout:], b[:l.cout], True, 0.0, 1e-5)
            else:
                h = F.conv2d(h, w.permute(0, 3, 1, 2), b, padding=1)
            if l.relu:
                h = _relu(h, margins)
        elif l.kind == "conv1x1":
            w, b = leaves[l.name]
            if getattr(l, "bn", False):
                h = F.conv2d(h, w.permute(0, 3, 1, 2), None)
                h = F.batch_norm(h, None, None, b[l.cout:], b[:l.cout], True, 0.0, 1e-5)
            else:
                h = F.conv2d(h, w.permute(0, 3, 1, 2), b)
            if l.relu:
                h = _relu(h, margins)
        elif l.kind == "pool3":              # 3x3/s1/p1 max over the first cout channels
            h = F.max_pool2d(h[:, :l.cout], 3, 1, 1)
        elif l.kind == "concat":
            h = torch.cat([outs[n] for n in l.srcs], dim=1)
        elif l.kind == "pool":
            h = F.max_pool2d(h, 2, 2)
        elif l.kind == "add":            # residual join, ResNet option-A shortcut
            s = outs[l.skip]
            if l.skip_down:
                s = s[:, :, ::2, ::2]
            if s.shape[1] < h.shape[1]:
                s = F.pad(s, (0, 0, 0, 0, 0, h.shape[1] - s.shape[1]))
            h = h + s
            if l.relu:
                h = _relu(h, margins)
        elif l.kind == "gap":
            h = h.mean(dim=(2, 3))
            flat = True
        else:
            if not flat:
                h = h.permute(0, 2, 3, 1).reshape(h.shape[0], -1)   # NHWC flatten
                flat = True
            w, b = leaves[l.name]
            h = F.linear(h, w, b)
            if l.relu:
                h = _relu(h, margins)
        outs[l.name] = h
    loss = F.cross_entropy(h, labels.to(torch.int64))
    loss.backward()
    grads = {n: (w.grad.detach(), b.grad.detach()) for n, (w, b) in leaves.items()}
    return float(loss.detach()), grads


def layer_fwd(l, x, w=None, b=None, dtype=torch.float64):
    """One layer forward on CPU (NHWC in/out) for kernel unit tests."""
    x = x.to(dtype)
    if l.kind == "conv":
        y = F.conv2d(x.permute(0, 3, 1, 2), w.to(dtype).permute(0, 3, 1, 2),
                     None if b is None else b.to(dtype), padding=1)
        if l.relu:
            y = F.relu(y)
        return y.permute(0, 2, 3, 1).contiguous()
    if l.kind == "pool":
        return F.max_pool2d(x.permute(0, 3, 1, 2), 2, 2).permute(0, 2, 3, 1).contiguous()
    y = F.linear(x, w.to(dtype), None if b is None else b.to(dtype))
    return F.relu(y) if l.relu else y


def conv_grads(x, w, dz, dtype=torch.float64):
    """dx (unmasked), dw, db of a 3x3/pad-1 conv given dz (NHWC)."""
    xx = x.to(dtype).permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    ww = w.to(dtype).permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    y = F.conv2d(xx, ww, None, padding=1)
    y.backward(dz.to(dtype).permute(0, 3, 1, 2))
    return (xx.grad.permute(0, 2, 3, 1).contiguous(),
            ww.grad.permute(0, 2, 3, 1).contiguous(),
            dz.to(dtype).sum(dim=(0, 1, 2)))


def normwise_rel(a, ref):
    """||a - ref|| / ||ref|| in fp64 (0 when both are 0)."""
    a = a.detach().to(torch.float64).cpu()
    ref = ref.detach().to(torch.float64).cpu()
    den = torch.linalg.vector_norm(ref)
    num = torch.linalg.vector_norm(a - ref)
    if den == 0:
        return float(num)
    return float(num / den)

"""Per-layer kernel timing at the VGG-16 B=32 shapes (CUDA events, warm,
averaged) -> TFLOP/s per op.  Used for optimisation work and under ncu
(--op / --layer pick a single launch pattern)."""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_10065_b200 import ops                       # noqa: E402
from paper_2112_10065_b200.network import vgg16            # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--layer", default=None)
    ap.add_argument("--op", default=None, choices=(None, "fwd", "dgrad", "wgrad"))
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--engine", default="auto", choices=("auto", "simt"))
    ap.add_argument("--inline-prep", action="store_true",
                    help="conv fwd/dgrad prepare their fp16x3 operands per call "
                         "(default: weights split and amax words made once, as the executor)")
    a = ap.parse_args()
    net = vgg16()
    dev = "cuda"
    ws = ops.Workspace(dev)
    rows = []
    for l in net.layers:
        if l.kind not in ("conv", "dense") or (a.layer and l.name != a.layer):
            continue
        b = a.batch
        x = torch.relu(torch.randn(l.in_shape(b), device=dev))
        w = torch.randn(l.param_shapes()[0], device=dev) * 0.02
        bias = torch.zeros(l.cout, device=dev)
        y = torch.empty(l.out_shape(b), device=dev)
        dy = torch.randn(l.out_shape(b), device=dev)
        dx = torch.empty_like(x)
        dw = torch.empty_like(w)
        db = torch.empty_like(bias)
        flops = l.fwd_flops() * b
        if l.kind == "conv":
            sp = xa = dya = None
            if not a.inline_prep and hasattr(ops, "F16Split"):
                sp = ops.F16Split(w).refresh(w)
                xa = ops.absmax(x, torch.zeros(4, dtype=torch.int32, device=dev))
                dya = ops.absmax(dy, torch.zeros(4, dtype=torch.int32, device=dev))
            fns = {"fwd": lambda: ops.conv3x3_fwd(x, w, bias, y, True, ws, wsplit=sp, x_amax=xa),
                   "dgrad": lambda: ops.conv3x3_dgrad(dy, w, x, dx, ws, wsplit=sp, dz_amax=dya),
                   "wgrad": lambda: ops.conv3x3_wgrad(x, dy, dw, db, ws, x_amax=xa, dz_amax=dya)}
            if a.engine == "simt":
                fns = {"fwd": lambda: ops.simt_conv3x3_fwd(x, w, bias, y, True),
                       "dgrad": lambda: ops.simt_conv3x3_dgrad(dy, w, x, dx),
                       "wgrad": lambda: ops.simt_conv3x3_wgrad(x, dy, dw, db, ws)}
            if l.name == "conv1_1":
                fns.pop("dgrad")
        else:
            x2 = x.view(b, -1)
            fns = {"fwd": lambda: ops.linear_fwd(x2, w, bias, y, True, ws),
                   "dgrad": lambda: ops.linear_dgrad(dy, w, x2, dx.view(b, -1), ws),
                   "wgrad": lambda: ops.linear_wgrad(x2, dy, dw, db, ws)}
        for op, fn in fns.items():
            if a.op and op != a.op:
                continue
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            rows.append({"layer": l.name, "op": op, "ms": ms,
                         "tflops": flops / ms / 1e9})
    tot = sum(r["ms"] for r in rows)
    for r in rows:
        print(f"{r['layer']:8s} {r['op']:6s} {r['ms']:8.3f} ms {r['tflops']:7.1f} TF/s "
              f"{100 * r['ms'] / tot:5.1f}%")
    print(f"total {tot:.3f} ms")
    print(json.dumps(rows))


if __name__ == "__main__":
    main()

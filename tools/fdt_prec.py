"""fp64 error of the fwd / dgrad engine per promotion-chunk length: run with
BPX_LIB pointing at builds made with BPX_NVCC_EXTRA=-DFDT_PCHK=<K>; prints
normwise relative error against fp64 and the test gate (max(2e-6, 4 x fp32))."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import vgg_ref                                  # noqa: E402
from paper_2112_10065_b200 import ops                       # noqa: E402
from paper_2112_10065_b200.network import LayerSpec         # noqa: E402


def rnd(*shape, seed=0, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(shape, generator=g, dtype=torch.float32) * scale


for (n, h, cin, cout) in [(2, 56, 256, 256), (1, 112, 128, 128), (2, 28, 512, 512),
                          (1, 224, 64, 64)]:
    x = torch.relu(rnd(n, h, h, cin, seed=1))
    w = rnd(cout, 3, 3, cin, seed=2, scale=math.sqrt(2 / (9 * cin)))
    b = rnd(cout, seed=3, scale=0.1)
    spec = LayerSpec("c", "conv", cin, cout, h, True, False)
    ref = vgg_ref.layer_fwd(spec, x, w, b)
    ref32 = vgg_ref.layer_fwd(spec, x, w, b, dtype=torch.float32)
    y = torch.empty(n, h, h, cout, device="cuda")
    ops.conv3x3_fwd(x.cuda(), w.cuda(), b.cuda(), y, relu=True)
    dz = rnd(n, h, h, cout, seed=6)
    dx_ref = vgg_ref.conv_grads(x, w, dz)[0] * (x > 0)
    dx32 = vgg_ref.conv_grads(x, w, dz, torch.float32)[0] * (x > 0)
    dx = torch.empty(n, h, h, cin, device="cuda")
    ops.conv3x3_dgrad(dz.cuda(), w.cuda(), x.cuda(), dx)
    torch.cuda.synchronize()
    ef = vgg_ref.normwise_rel(y, ref)
    ed = vgg_ref.normwise_rel(dx, dx_ref)
    gf = max(2e-6, 4 * vgg_ref.normwise_rel(ref32, ref))
    gd = max(2e-6, 4 * vgg_ref.normwise_rel(dx32, dx_ref))
    print(f"{(n, h, cin, cout)}  fwd {ef:.2e} (gate {gf:.2e})  dgrad {ed:.2e} (gate {gd:.2e})")

# weight gradient (wgh: K = pixels, promotion every WGH_PCHK)
for (n, h, cin, cout) in [(8, 56, 256, 256), (8, 28, 512, 512), (8, 112, 128, 128)]:
    x = torch.relu(rnd(n, h, h, cin, seed=7))
    w = rnd(cout, 3, 3, cin, seed=8)
    dz = rnd(n, h, h, cout, seed=9)
    _, dw_ref, _ = vgg_ref.conv_grads(x, w, dz)
    _, dw32, _ = vgg_ref.conv_grads(x, w, dz, torch.float32)
    dw = torch.empty(cout, 3, 3, cin, device="cuda")
    db = torch.empty(cout, device="cuda")
    ops.conv3x3_wgrad(x.cuda(), dz.cuda(), dw, db)
    torch.cuda.synchronize()
    e = vgg_ref.normwise_rel(dw, dw_ref)
    gt = max(2e-6, 4 * vgg_ref.normwise_rel(dw32, dw_ref))
    print(f"{(n, h, cin, cout)}  wgrad {e:.2e} (gate {gt:.2e})  engine {ops.last_engine()}")

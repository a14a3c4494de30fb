"""fp64 error of the Cin = Cout = 64 weight gradient at conv1_2 sizes
(promotion-chunk length experiments): python tools/wgc_prec.py"""
import sys, torch
sys.path.insert(0, ".")
from paper_2112_10065_b200 import ops
from oracle import vgg_ref


def rnd(*shape, seed=0, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(shape, generator=g, dtype=torch.float32) * scale


def relu_input(*shape, seed=0):
    return torch.relu(rnd(*shape, seed=seed))
for shape in [(1, 224, 64, 64), (4, 224, 64, 64), (16, 224, 64, 64)]:
    n, h, cin, cout = shape
    x = relu_input(n, h, h, cin, seed=40); dz = rnd(n, h, h, cout, seed=41)
    _, dw_ref, db_ref = vgg_ref.conv_grads(x, torch.zeros(cout, 3, 3, cin), dz)
    _, dw32, _ = vgg_ref.conv_grads(x, torch.zeros(cout, 3, 3, cin), dz, torch.float32)
    dw = torch.empty(cout, 3, 3, cin, device="cuda"); db = torch.empty(cout, device="cuda")
    ops.conv3x3_wgrad(x.cuda(), dz.cuda(), dw, db); torch.cuda.synchronize()
    e = vgg_ref.normwise_rel(dw, dw_ref); e32 = vgg_ref.normwise_rel(dw32, dw_ref)
    print(shape, ops.last_engine(), f"err {e:.3e} fp32cpu {e32:.3e} gate {max(2e-6, 4*e32):.3e}")

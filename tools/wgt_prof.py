"""MMA-issuer cycle breakdown of the wgrad engine (needs a library built with
BPX_NVCC_EXTRA=-DWGT_PROF, path in BPX_LIB or ./ab_wprof.so)."""
import ctypes, os, sys, torch
sys.path.insert(0, os.getcwd())
os.environ.setdefault("BPX_LIB", os.path.abspath("ab_wprof.so"))
from paper_2112_10065_b200 import ops
from paper_2112_10065_b200.network import vgg16
lib = ops.load_library()
f = lib.bpx_wgt_prof
net = vgg16()
ws = ops.Workspace("cuda")
for name in ("conv1_2", "conv2_2", "conv3_2", "conv4_2", "conv5_1"):
    l = [x for x in net.layers if x.name == name][0]
    b = 32
    x = torch.relu(torch.randn(l.in_shape(b), device="cuda"))
    dy = torch.randn(l.out_shape(b), device="cuda")
    dw = torch.empty(l.param_shapes()[0], device="cuda")
    db = torch.empty(l.cout, device="cuda")
    ws.reserve(ops.conv_workspace_bytes(b, l.hw, l.hw, l.cin, l.cout))
    out = (ctypes.c_ulonglong * 6)()
    f(out, 1)
    ops.conv3x3_wgrad(x, dy, dw, db, ws)
    torch.cuda.synchronize()
    f(out, 0)
    tot, acc, a, bb, iss, n = list(out)
    print(f"{name}: stages {n}  per stage cycles: total {tot/n:.0f}  wait_hfree {acc/n:.0f}  "
          f"wait_A {a/n:.0f}  wait_B {bb/n:.0f}  issue {iss/n:.0f}")

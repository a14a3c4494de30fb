"""MMA-issuer cycle breakdown of the fwd/dgrad engine (needs a library built with
BPX_NVCC_EXTRA=-DFDT_PROF, path in BPX_LIB or ./ab_prof.so)."""
import ctypes, os, sys, torch
sys.path.insert(0, os.getcwd())
os.environ.setdefault("BPX_LIB", os.path.abspath("ab_prof.so"))  # a -DFDT_PROF build
from paper_2112_10065_b200 import ops
from paper_2112_10065_b200.network import vgg16
lib = ops.load_library()
f = lib.bpx_fdt_prof
net = vgg16()
ws = ops.Workspace("cuda")
for name in ("conv1_2", "conv2_2", "conv3_2", "conv4_2", "conv5_1"):
    l = [x for x in net.layers if x.name == name][0]
    b = 32
    x = torch.relu(torch.randn(l.in_shape(b), device="cuda"))
    w = torch.randn(l.param_shapes()[0], device="cuda") * 0.02
    bias = torch.zeros(l.cout, device="cuda")
    y = torch.empty(l.out_shape(b), device="cuda")
    for op in ("fwd", "dgrad"):
        if op == "fwd":
            ops.conv3x3_fwd(x, w, bias, y, True, ws)
        else:
            dy = torch.randn(l.out_shape(b), device="cuda")
            ops.conv3x3_dgrad(dy, w, x, torch.empty_like(x), ws)
        torch.cuda.synchronize()
        out = (ctypes.c_ulonglong * 6)()
        f(out)
        tot, acc, a, bb, iss, n = list(out)
        print(f"{name} {op}: stages/CTA-thread {n/148:.0f}  per stage cycles: total {tot/n:.0f}  wait_acc {acc/n:.0f}  wait_A {a/n:.0f}  wait_B {bb/n:.0f}  issue {iss/n:.0f}")

"""Role cycle breakdown of the fwd/dgrad engine (needs a library built with
BPX_NVCC_EXTRA=-DFDT_PROF, path in BPX_LIB or ./ab_prof.so).  Counters are
warp 0 of each role summed over CTAs, printed per stage (MMA issuer) or per
CTA-share of the launch."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
os.environ.setdefault("BPX_LIB", os.path.abspath("ab_prof.so"))
from paper_2112_10065_b200 import ops                     # noqa: E402
from paper_2112_10065_b200.network import vgg16          # noqa: E402

NAMES = {0: "mma_total", 1: "mma_wait_accfree", 2: "mma_wait_aready", 4: "stages",
         6: "conv_wait_hfull", 7: "conv_split", 8: "conv_wait_tmem", 9: "conv_wait_bfull",
         10: "conv_wait_st",
         11: "tma_wait_hempty", 12: "tma_wait_empty", 14: "drain_wait_accfull",
         15: "drain_epilogue"}

lib = ops.load_library()
f = lib.bpx_fdt_prof
net = vgg16()
ws = ops.Workspace("cuda")
layers = sys.argv[1:] or ["conv1_2", "conv2_2", "conv3_2", "conv4_2", "conv5_1"]
for name in layers:
    l = [x for x in net.layers if x.name == name][0]
    b = 32
    x = torch.relu(torch.randn(l.in_shape(b), device="cuda"))
    w = torch.randn(l.param_shapes()[0], device="cuda") * 0.02
    bias = torch.zeros(l.cout, device="cuda")
    y = torch.empty(l.out_shape(b), device="cuda")
    dy = torch.randn(l.out_shape(b), device="cuda")
    sp = ops.F16Split(w).refresh(w)
    xa = ops.absmax(x, torch.zeros(4, dtype=torch.int32, device="cuda"))
    da = ops.absmax(dy, torch.zeros(4, dtype=torch.int32, device="cuda"))
    for op in ("fwd", "dgrad"):
        run = (lambda: ops.conv3x3_fwd(x, w, bias, y, True, ws, wsplit=sp, x_amax=xa)) \
            if op == "fwd" else \
            (lambda: ops.conv3x3_dgrad(dy, w, x, torch.empty_like(x), ws, wsplit=sp, dz_amax=da))
        run()
        torch.cuda.synchronize()
        out = (ctypes.c_ulonglong * 16)()
        f(out)                       # reset after the warm-up
        run()
        f(out)
        v = list(out)
        n = max(v[4], 1)
        tot = max(v[0], 1)
        parts = "  ".join(f"{NAMES[k]} {100 * v[k] / tot:5.1f}%" for k in (1, 2, 6, 7, 8, 9, 10,
                                                                         11, 12, 14, 15))
        print(f"{name} {op}: MMA-issuer cycles/stage {tot / n:6.0f} | {parts}")

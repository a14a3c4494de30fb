import sys, torch
sys.path.insert(0, ".")
from paper_2112_10065_b200 import ops
for n, h in [(2, 224), (3, 32)]:
    x = torch.randn(n, h, h, 3, device="cuda"); dz = torch.randn(n, h, h, 64, device="cuda")
    dw = torch.empty(64, 3, 3, 3, device="cuda"); db = torch.empty(64, device="cuda")
    try:
        ops.conv3x3_wgrad(x, dz, dw, db); torch.cuda.synchronize(); print(n, h, "ok", ops.last_engine())
    except Exception as e:
        print(n, h, "ERR", e)

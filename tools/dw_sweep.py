"""Dense weight-gradient timing sweep (fc1/fc2/fc3 shapes, b = 1..32) through
ops.linear_wgrad -- the per-call numbers include the prep and column-sum
launches; the small shapes are host-bound."""
import os, sys, torch, json
sys.path.insert(0, os.getcwd())
from paper_2112_10065_b200 import ops
ws = ops.Workspace("cuda")
res = {}
for (fin, fout) in [(25088, 4096), (4096, 4096), (4096, 1000)]:
    for b in (1, 4, 8, 16, 32):
        x = torch.randn(b, fin, device="cuda"); dy = torch.randn(b, fout, device="cuda")
        dw = torch.empty(fout, fin, device="cuda"); db = torch.empty(fout, device="cuda")
        for _ in range(3): ops.linear_wgrad(x, dy, dw, db, ws)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(20): ops.linear_wgrad(x, dy, dw, db, ws)
        e1.record(); torch.cuda.synchronize()
        res[f"{fin}x{fout} b{b}"] = round(e0.elapsed_time(e1) / 20 * 1000, 1)
print(json.dumps(res))

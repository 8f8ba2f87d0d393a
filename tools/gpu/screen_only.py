"""Screen kernel time alone (dist.Plan: create once, run all tiles, reset;
no finalize), C3 operands -- for the ADG_SCREEN_DEBUG ablations, whose
results are deliberately wrong (profiling aid)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds, dist
D, R = int(os.environ.get("D", "784")), int(os.environ.get("R", "50"))
X = torch.from_numpy(ds.c3_mnist_like()).cuda()[:, :D].contiguous()
W = torch.randn(D, R, device="cuda", dtype=torch.float64) / 28
Y = (X.double() @ W).float().contiguous()
pl = dist.Plan(X, Y, hist_bins=50)
flush = torch.empty(64 << 20, device="cuda")
ts = []
for k in range(12):
    flush.zero_()
    pl.reset()
    pl.run(0, pl.num_tiles)
    torch.cuda.synchronize()
    if k >= 2:
        ts.append(adg.api.last_screen_kernel_ms(0))
print(json.dumps({"debug": os.environ.get("ADG_SCREEN_DEBUG", "0"), "d": D, "r": R, "median_ms": statistics.median(ts),
                  "min_ms": min(ts)}), flush=True)

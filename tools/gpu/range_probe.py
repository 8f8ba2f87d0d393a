"""Screen time for sub-ranges of the C3 tile list (a rank's share at W = 8 and
others): per-tile cost vs the full launch (profiling aid)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds, dist
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(m, X).data
pl = dist.Plan(X, Y, hist_bins=50)
T = pl.num_tiles
flush = torch.empty(64 << 20, device="cuda")
warm = torch.randn(4096, 4096, device="cuda")
WARM = int(os.environ.get("WARM", "0"))  # busy matmuls right before the launch (GPU clocks up)
def t(a, b, reps=7):
    ts = []
    for _ in range(reps):
        flush.zero_(); pl.reset()
        for _ in range(WARM):
            warm @ warm
        pl.run(a, b); torch.cuda.synchronize()
        ts.append(adg.api.last_screen_kernel_ms(0))
    return statistics.median(ts[1:])
full = t(0, T)
print(json.dumps({"range": "full", "tiles": T, "ms": full, "us_per_tile": 1e3 * full / T}), flush=True)
if os.environ.get("WARM_SWEEP"):
    a, b = dist.shard_range(T, 8, 0)
    for w in (0, 1, 2, 5, 10, 20):
        WARM = w
        ms = t(a, b)
        print(json.dumps({"warm_matmuls": w, "range": "W8 rank 0", "ms": ms, "vs_full": (ms / (b - a)) / (full / T)}), flush=True)
    sys.exit(0)
for W in (8, 4):
    for r in (0, W // 2, W - 1):
        a, b = dist.shard_range(T, W, r)
        ms = t(a, b)
        print(json.dumps({"range": f"W{W} rank {r}", "tiles": b - a, "ms": ms, "us_per_tile": 1e3 * ms / (b - a),
                          "vs_full": (ms / (b - a)) / (full / T)}), flush=True)

"""Screen kernel time of each rank's tile range at world size W (one GPU,
one range at a time, L2 flushed before each): how even is the partition,
and what does a 1/W range cost against 1/W of the whole?  Profiling aid."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds, dist

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
X = torch.from_numpy(ds.c3_mnist_like()).to(dev)
model = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(model, X).data.clone()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
plan = dist.Plan(X, Y, 50, 1.0)
T = plan.num_tiles
for W in [int(a) for a in sys.argv[1:]] or [1, 8]:
    res = []
    for r in range(W):
        ts = []
        for _ in range(5):
            plan.reset()
            flush.zero_()
            plan.run(*dist.shard_range(T, W, r))
            torch.cuda.synchronize()
            ts.append(adg.api.last_screen_kernel_ms(0))
        res.append(statistics.median(ts))
    print(f"W={W} tiles={T}: per-rank screen ms " + " ".join(f"{v:.3f}" for v in res)
          + f" | max {max(res):.3f} sum {sum(res):.3f}", flush=True)
plan.close()

# fixed cost of a launch: tiny ranges
plan = dist.Plan(X, Y, 50, 1.0)
for cnt in [1, 74, 148, 740, 1480, 5528]:
    ts = []
    for _ in range(5):
        plan.reset()
        flush.zero_()
        plan.run(0, cnt)
        torch.cuda.synchronize()
        ts.append(adg.api.last_screen_kernel_ms(0))
    print(f"range of {cnt} tiles: screen {statistics.median(ts):.4f} ms", flush=True)
plan.close()

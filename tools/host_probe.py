"""Host enqueue time of the step's API calls with the GPU idle (right after a
synchronize) and busy (a queued memset ahead), profiling aid."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds, dist

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
X = torch.from_numpy(ds.c3_mnist_like()).to(dev)
model = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(model, X).data.clone()
busy = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
Xl = X[:7500]


def hostt(fn, idle, reps=20):
    ts = []
    for _ in range(reps):
        if not idle:
            busy.zero_()
        else:
            torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t) * 1e3)
        torch.cuda.synchronize()
    return statistics.median(ts)


plans = []
for idle in (True, False):
    tag = "idle" if idle else "busy"
    print(f"[{tag}] transform_all(7500 rows) host ms {hostt(lambda: adg.transform_all(model, Xl), idle):.4f}")
    print(f"[{tag}] torch.empty host ms {hostt(lambda: torch.empty(10, device=dev), idle):.4f}")
    print(f"[{tag}] small kernel (zero_) host ms {hostt(lambda: Y[:1].zero_(), idle):.4f}")
    print(f"[{tag}] Plan create host ms {hostt(lambda: plans.append(dist.Plan(X, Y, 50, 1.0)), idle):.4f}")
    while plans:
        plans.pop().close()

"""Timeline of one bench step (CUPTI via torch.profiler): kernels, copies, gaps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
def step():
    Y = adg.transform_all(m, X).data
    return adg.evaluate(X, Y, hist_bins=50, engine="screen")
for _ in range(3): step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step(); torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev = t0
for e in evs:
    s, en = e.time_range.start, e.time_range.end
    print(f"{(s - t0)/1000:8.3f} ms  +gap {(s - prev)/1000:6.3f}  dur {(en - s)/1000:7.3f}  {e.name[:70]}")
    prev = en
print(f"total {(prev - t0)/1000:.3f} ms")

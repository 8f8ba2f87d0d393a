"""Host vs device timeline of one bench step: CUDA runtime API calls (host
side) and kernels/copies (device side) from CUPTI via torch.profiler, merged
in time order, so host-induced device idle time is visible."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def step():
    Y = adg.transform_all(m, X).data
    return adg.evaluate(X, Y, hist_bins=50, engine="screen")


for _ in range(3):
    step()
torch.cuda.synchronize()
flush.zero_()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
evs = []
for e in prof.events():
    dev = e.device_type == torch.autograd.DeviceType.CUDA
    if not dev and not e.name.startswith("cuda"):
        continue
    evs.append((e.time_range.start, e.time_range.end, "GPU" if dev else "cpu", e.name))
evs.sort()
t0 = evs[0][0]
for s, en, kind, name in evs:
    if kind == "cpu" and (en - s) < 5 and not name.startswith(("cudaStreamSynchronize", "cudaMemcpy")):
        continue  # hide tiny API calls
    print(f"{(s - t0)/1000:8.3f} ms  {kind}  dur {(en - s)/1000:7.3f}  {name[:80]}")
print(f"host wall for the step: {wall*1e3:.3f} ms")

"""transform_all on the C3 workload: host enqueue time per call (no sync),
device time per call with X cold (L2 flushed before each call) and warm, and
cuBLAS sgemm of the same shape for scale."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
torch.backends.cuda.matmul.allow_tf32 = False
W = torch.randn(784, 50, device="cuda")

for _ in range(3):
    adg.transform_all(m, X)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    adg.transform_all(m, X)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue per call: {(t1 - t0) / 50 * 1e3:.4f} ms; wall incl. drain per call {(t2 - t0) / 50 * 1e3:.4f} ms")


def timed(fn, reps=20, cold=True):
    for _ in range(3):
        fn()
    tot = 0.0
    for _ in range(reps):
        if cold:
            flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


for cold in (False, True):
    tag = "cold" if cold else "warm"
    print(f"[{tag}] cublas sgemm 60000x784x50 ms: {timed(lambda: X @ W, cold=cold):.4f}")
    print(f"[{tag}] adg transform_all ms:          {timed(lambda: adg.transform_all(m, X), cold=cold):.4f}")
print("bytes X:", X.numel() * 4, " -> HBM floor ms at 7.7 TB/s:", X.numel() * 4 / 7.7e9)

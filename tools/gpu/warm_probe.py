"""Bench-style C3 steps (transform_all + evaluate, L2 flushed between steps)
with and without a busy matmul queued right before each step (profiling aid:
does an idle host gap before a step cost device time?)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
warm = torch.randn(4096, 4096, device="cuda")
def step():
    Y = adg.transform_all(m, X).data
    return adg.evaluate(X, Y, hist_bins=50, engine="screen")
for _ in range(3):
    step()
for rnd in range(3):
    for w in (0, 1):
        ts, ks = [], []
        for _ in range(6):
            flush.zero_()
            if w:
                warm @ warm
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); step(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1)); ks.append(adg.api.last_screen_kernel_ms(0))
        print(f"warm={w}: step ms median {statistics.median(ts):.4f}  screen ms median {statistics.median(ks):.4f}", flush=True)

"""Does a concurrent host->device copy slow the screen?  C3 evaluate on
device-resident data, screen kernel time alone and with 188 MB pinned H2D
copies running on another stream (profiling aid)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
Xh = ds.c3_mnist_like()
X = torch.from_numpy(Xh).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(m, X).data
Xp = torch.from_numpy(Xh).pin_memory()
dst = torch.empty_like(X)
cs = torch.cuda.Stream()
def run(copy):
    ks = []
    for _ in range(6):
        torch.cuda.synchronize()
        if copy:
            with torch.cuda.stream(cs):
                for _ in range(3):
                    dst.copy_(Xp, non_blocking=True)
        adg.evaluate(X, Y, hist_bins=50, engine="screen")
        torch.cuda.synchronize()
        ks.append(adg.api.last_screen_kernel_ms(0))
    return statistics.median(ks[1:])
for k in range(2):
    print("alone %.3f ms   with h2d %.3f ms" % (run(False), run(True)), flush=True)

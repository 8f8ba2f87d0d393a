"""One C3 evaluate (after a warm-up one) for ncu captures of the screen kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(m, X).data
eng = os.environ.get("ENGINE", "screen")
for _ in range(2):
    r = adg.evaluate(X, Y, hist_bins=50, engine=eng)
torch.cuda.synchronize()
print(r.max_distortion, r.edge_pairs)

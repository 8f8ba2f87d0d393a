"""One pipelined adg_distort_model call on C3 from pinned host memory (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
Xh = ds.c3_mnist_like()
X = torch.from_numpy(Xh).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
mh = adg.AdagioModel(m.mean.cpu().numpy(), adg.OrthonormalBasis(m.basis.rows.cpu().numpy()),
                     adg.JlMatrix(m.sketch.entries.cpu().numpy()), 0)
Xp = torch.from_numpy(Xh).pin_memory().numpy()
adg.distort_model(mh, Xp, hist_bins=50, engine="screen")
torch.cuda.synchronize()
print("ok")

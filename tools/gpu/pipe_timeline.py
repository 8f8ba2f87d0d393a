"""Event timeline of the pipelined run_distort flow (adg_distort_model from a
pinned host X, C3): ADG_PIPE_PROFILE=1 prints per-phase device times to
stderr (profiling aid).  Usage: ADG_PIPE_CHUNKS=K ADG_PIPE_POWER=p python ..."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
Xh = ds.c3_mnist_like()
X = torch.from_numpy(Xh).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
mh = adg.AdagioModel(m.mean.cpu().numpy(), adg.OrthonormalBasis(m.basis.rows.cpu().numpy()),
                     adg.JlMatrix(m.sketch.entries.cpu().numpy()), 0)
Xp = torch.from_numpy(Xh).pin_memory().numpy()
ts = []
for k in range(int(os.environ.get('REPS', '4'))):
    t = time.perf_counter()
    r = adg.distort_model(mh, Xp, hist_bins=50, engine="screen")
    ts.append(time.perf_counter() - t)
ts = ts[1:]
print("e2e ms min %.3f median %.3f" % (1e3 * min(ts), 1e3 * sorted(ts)[len(ts) // 2]), r.max_distortion, flush=True)

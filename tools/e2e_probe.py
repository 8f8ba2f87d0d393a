"""e2e of the run_distort --model flow (adg_distort_model) from pinned host
memory on C3: median of 9 repetitions per setting; arguments are
CHUNKS[:POWER] (ADG_PIPE_CHUNKS, ADG_PIPE_POWER)."""
import os, sys, time, statistics, json
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
out = {}
for k in sys.argv[1:]:
    ch, _, pw = k.partition(":")
    os.environ["ADG_PIPE_CHUNKS"] = ch
    os.environ["ADG_PIPE_POWER"] = pw or "1.0"
    for _ in range(2):
        adg.distort_model(mh, Xp, hist_bins=50, engine="screen")
    ts = []
    for _ in range(9):
        t = time.perf_counter()
        adg.distort_model(mh, Xp, hist_bins=50, engine="screen")
        ts.append(time.perf_counter() - t)
    out[k] = round(statistics.median(ts) * 1e3, 3)
print(json.dumps({"e2e_ms_median_by_chunks": out}))

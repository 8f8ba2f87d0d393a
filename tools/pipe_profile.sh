python - <<'PY'
import os, sys, time
sys.path.insert(0, '.')
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
Xh = ds.c3_mnist_like()
X = torch.from_numpy(Xh).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
mh = adg.AdagioModel(m.mean.cpu().numpy(), adg.OrthonormalBasis(m.basis.rows.cpu().numpy()),
                     adg.JlMatrix(m.sketch.entries.cpu().numpy()), 0)
Xp = torch.from_numpy(Xh).pin_memory().numpy()
for _ in range(3):
    adg.distort_model(mh, Xp, hist_bins=50, engine="screen")
os.environ["ADG_PIPE_PROFILE"] = "1"
for _ in range(2):
    t = time.perf_counter(); adg.distort_model(mh, Xp, hist_bins=50, engine="screen"); print("wall", time.perf_counter() - t, file=sys.stderr, flush=True)
PY

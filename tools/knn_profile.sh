python - <<'PY'
import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
Y = adg.transform_all(adg.fit(X, 50, adg.SpectralBackend.exact, 0), X).data
adg.build_knn_graph(X[:5000], 30)
os.environ["ADG_KNN_PROFILE"] = "1"
for name, c in (("raw", X), ("emb", Y)):
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        adg.build_knn_graph(c, 30)
        print(name, "total", time.perf_counter() - t0, file=sys.stderr, flush=True)
PY

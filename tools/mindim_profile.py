import os, sys, time
sys.path.insert(0, '.')
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import Method, datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
adg.min_dim_for_distortion(X[:5000], Method.pca, 0.5, 0, 1, 20)
os.environ["ADG_FIT_PROFILE"] = "1"
t = time.perf_counter(); r = adg.min_dim_for_distortion(X, Method.pca, 0.5, 0, 1, 200); print("pca", time.perf_counter() - t, r, file=sys.stderr)
t = time.perf_counter(); rows = adg.tradeoff(X, [10, 200], [Method.pca], [0]); print("tradeoff", time.perf_counter() - t, [(x.target_dim, x.fit_seconds, x.eval_seconds) for x in rows], file=sys.stderr)

"""Fit stage profile (ADG_FIT_PROFILE=1): finite check, fp64 Gram, top
eigenvectors (subspace iteration count) for C3 exact and randomized."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

X = torch.from_numpy(ds.c3_mnist_like()).cuda()
adg.fit(X[:5000], 50, adg.SpectralBackend.exact, 0)
os.environ["ADG_FIT_PROFILE"] = "1"
for be in (adg.SpectralBackend.exact, adg.SpectralBackend.randomized):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        adg.fit(X, 50, be, 0)
        print(be, "fit total", time.perf_counter() - t0, file=sys.stderr, flush=True)

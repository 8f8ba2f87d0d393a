"""Profiling aid: screen-kernel time with parts of the pipeline disabled
(ADG_SCREEN_DEBUG): 1 = no pair math, 2 = no MMAs, 3 = TMA only, 4 = MMA only."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(m, X).data
names = {"0": "full", "1": "no_pair_math", "2": "no_mma", "3": "tma_only", "4": "mma_only"}
out = {}
for mode in sys.argv[1:] or list(names):
    os.environ["ADG_SCREEN_DEBUG"] = mode
    ts = []
    for _ in range(4):
        adg.evaluate(X, Y, engine="screen")
        ts.append(adg.api.last_screen_kernel_ms())
    out[names[mode]] = round(min(ts[1:]), 3)
os.environ["ADG_SCREEN_DEBUG"] = "0"
print(json.dumps(out))

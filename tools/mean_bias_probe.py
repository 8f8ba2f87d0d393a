"""Diagnostic: screen-engine mean vs exact-engine mean on C3 subsets."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
X = ds.c3_mnist_like(n=4096, seed=3)
for dcut in [784, 392, 196, 98]:
    Xs = np.ascontiguousarray(X[:, :dcut]) if dcut < 784 else X
    m = adg.fit(Xs, 50, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(m, Xs).data
    for name, xx in [("orig", Xs), ("shift+10", Xs + 10.0)]:
        s = adg.evaluate(xx, Y, engine="screen")
        e = adg.evaluate(xx, Y, engine="exact")
        print(f"d={dcut:4d} {name:9s} mean_exact={e.mean_distortion:.9f} rel_bias={(s.mean_distortion-e.mean_distortion)/e.mean_distortion:+.3e} max_eq={s.max_distortion==e.max_distortion}", flush=True)
rng = np.random.default_rng(1)
G = rng.standard_normal((4096, 784)).astype(np.float32)
m = adg.fit(G, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(m, G).data
s = adg.evaluate(G, Y, engine="screen"); e = adg.evaluate(G, Y, engine="exact")
print(f"gaussian d=784 rel_bias={(s.mean_distortion-e.mean_distortion)/e.mean_distortion:+.3e} mean={e.mean_distortion:.5f}")

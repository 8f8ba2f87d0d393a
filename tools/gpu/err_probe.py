"""Screen error scale, measured through the product path: screen vs exact
engine histograms at fine bin widths over [0, hist_max] on subsampled
C3 / C4 / C5-like clouds.  sum|dhist|/2 is a lower bound on the pairs whose
screened value crossed an edge of that width."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

def run(name, X, r):
    Xd = torch.as_tensor(X).cuda() if not torch.is_tensor(X) else X.cuda()
    m = adg.fit(Xd, r, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(m, Xd).data
    e0 = adg.evaluate(Xd, Y, hist_bins=50, engine="exact")
    s0 = adg.evaluate(Xd, Y, hist_bins=50, engine="screen")
    vmax = e0.max_distortion
    out = {"name": name, "n": Xd.shape[0], "d": Xd.shape[1], "r": r, "mean_exact": e0.mean_distortion,
           "mean_screen": s0.mean_distortion,
           "mean_rel_bias": (s0.mean_distortion - e0.mean_distortion) / e0.mean_distortion,
           "max_eq": s0.max_distortion == e0.max_distortion, "hist50_moved_lb": int(np.abs(np.asarray(s0.histogram, np.int64) - np.asarray(e0.histogram, np.int64)).sum() // 2),
           "eps": s0.screen_error_bound if hasattr(s0, "screen_error_bound") else None, "widths": {}}
    hm = float(min(1.0, vmax * 1.01))
    for bins, hmx in [(100, hm), (1000, hm), (10000, hm), (10000, hm / 10), (10000, hm / 100)]:
        e = adg.evaluate(Xd, Y, hist_bins=bins, hist_max=hmx, engine="exact")
        s = adg.evaluate(Xd, Y, hist_bins=bins, hist_max=hmx, engine="screen")
        dh = np.abs(np.asarray(s.histogram, np.int64) - np.asarray(e.histogram, np.int64))
        out["widths"][f"{hmx / bins:.2e}"] = [int(dh[:-1].sum() // 2), int(np.asarray(e.histogram)[:-1].sum())]
    print(json.dumps(out), flush=True)

rng = np.random.default_rng(0)
X3 = ds.c3_mnist_like(n=60000, seed=3)
run("c3_sub8192", np.ascontiguousarray(X3[np.sort(rng.choice(60000, 8192, replace=False))]), 50)
X4 = ds.c4_power_law(n=8192, seed=4)
run("c4_8192", X4, 64)
X5 = ds.c5_mixture(n=8192, seed=5)
run("c5_8192", X5, 128)

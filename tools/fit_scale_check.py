"""Fit at full scale (C4, C5; C3 for reference): timing of the exact fit and
its basis against numpy eigh of the same fp64 Gram (adg_gram), largest
per-row difference after the reference's sign rule and the subspace gap
sin(max principal angle).  Usage: fit_scale_check.py [c3 c4 c5]"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds, dist
from oracle import oracle as o

for name in (sys.argv[1:] or ["c3", "c4", "c5"]):
    n, d, r, bins, _ = ds.CONFIGS[name]
    X = ds.make(name)
    times = []
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        m = adg.fit(X, r, adg.SpectralBackend.exact, 0)
        torch.cuda.synchronize(); times.append(time.perf_counter() - t0)
    P = torch.as_tensor(m.basis.rows).double().cpu().numpy()
    s = P.shape[0]
    x = adg.api._matrix(X)
    ctx, dev = adg.api._ctx_for(x)
    mean = torch.as_tensor(m.mean).double().to(dev)
    G = dist._gram_dev(x, ctx, dev, mean.double(), adg.SpectralBackend.exact).cpu().numpy()
    t0 = time.perf_counter(); w, v = np.linalg.eigh(G); te = time.perf_counter() - t0
    ref = o._normalize_row_signs(v[:, ::-1][:, :s].T.copy())
    sv = np.linalg.svd(ref @ P.T, compute_uv=False)
    gap = float(np.sqrt(max(0.0, 1.0 - sv.min() ** 2)))
    print(json.dumps({"config": name, "n": n, "d": d, "s": s, "fit_s": times,
                      "max_row_diff": float(np.abs(P - ref).max()), "subspace_sin": gap,
                      "eig_gap_s_s1": float(w[::-1][s - 1] / w[::-1][s]), "numpy_eigh_s": te}), flush=True)
    del X, m, G
    torch.cuda.empty_cache()

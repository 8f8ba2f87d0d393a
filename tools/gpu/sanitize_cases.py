"""Small invocations of every libadg kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck; tools/gpu/sanitize.sh).  Each case checks
its result loosely so a silent failure also shows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1609_05388_b200 as adg
from oracle import oracle

which = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(0)


def cloud(n, d, seed):
    return torch.from_numpy(oracle.gaussian_cloud(n, d, seed).astype(np.float32)).cuda()


if which in ("all", "screen"):
    X = cloud(3000, 96, 1)
    m = adg.fit(X, 24, adg.SpectralBackend.exact, 0)          # whole-Gram Jacobi (d <= 384)
    Y = adg.transform_all(m, X).data                           # transform_tc_kernel
    for bins, eng in ((50, "screen"), (50, "screen_exact_hist"), (1000, "screen"), (20000, "screen")):
        r = adg.evaluate(X, Y, hist_bins=bins, engine=eng)     # HMODE 1 / edges / 3 / 0 (global)
        assert r.n_pairs_evaluated == 3000 * 2999 // 2
    assert adg.max_distortion(X, Y) > 0                        # HMODE 2
    print("screen ok", flush=True)
if which in ("all", "exact"):
    X = cloud(4200, 32, 2)
    Y = X[:, :8].contiguous()
    r = adg.evaluate(X, Y, hist_bins=50, engine="exact")      # tiled exact
    s = adg.evaluate(X, Y, adg.PairSampling.sample(20000, 5), hist_bins=50)  # block exact
    print("exact ok", r.max_distortion, flush=True)
if which in ("all", "fit"):
    for d, s in ((512, 30), (1024, 60)):                       # subspace iteration; grid CholQR / Jacobi
        X = cloud(2000, d, 3)
        m = adg.fit_with_split(X, s, 8, adg.SpectralBackend.exact, 0)
        assert np.allclose(m.basis.rows.cpu().numpy() @ m.basis.rows.cpu().numpy().T, np.eye(s), atol=1e-8)
    m = adg.fit(cloud(2000, 200, 4), 40, adg.SpectralBackend.randomized, 3)
    print("fit ok", flush=True)
if which in ("all", "knn"):
    X = cloud(4500, 40, 5)
    g = adg.build_knn_graph(X, 8)                              # tensor-core candidate path
    q = adg.knn_query_batch(X, X[:70], 5)                       # SIMT tiles
    print("knn ok", len(g.edges), flush=True)

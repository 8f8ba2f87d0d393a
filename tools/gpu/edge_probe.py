"""Edge band calibration (profiling aid): for each ADG_EDGE_BAND value, the
SCREEN histogram against (a) the committed C3 full-oracle fixture and (b) the
EXACT engine on 8192-row C3 / C4 / C5-like clouds; prints pairs moved
(sum |dhist| / 2), pairs sent to exact binning, and the evaluate time."""
import json, os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

def child():
    import numpy as np, torch
    import paper_1609_05388_b200 as adg
    from paper_1609_05388_b200 import datasets as ds
    from oracle import oracle
    out = {"band": os.environ.get("ADG_EDGE_BAND")}
    fx = json.load(open(os.path.join(ROOT, "tests/golden/c3_fixture.json")))
    X = ds.c3_mnist_like()
    z = np.load(os.path.join(ROOT, "tests/golden/c3_fixture.npz"))
    S = oracle.sample_jl(25, 784, oracle.derive_seed(0, "jl"))
    Y = oracle.transform_all(z["mean"], z["P"], S, X.astype(np.float64)).astype(np.float32)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    rep = adg.evaluate(Xd, Yd, hist_bins=50, engine=os.environ.get("PROBE_ENGINE", "screen_exact_hist"))
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t = time.perf_counter()
        rep = adg.evaluate(Xd, Yd, hist_bins=50, engine=os.environ.get("PROBE_ENGINE", "screen_exact_hist"))
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    dh = np.asarray(rep.histogram, np.int64) - np.asarray(fx["histogram"], np.int64)
    out["c3_full"] = {"moved": int(np.abs(dh).sum() // 2), "edge_pairs": rep.edge_pairs,
                      "ms": 1e3 * min(ts), "dh_nonzero": {int(i): int(v) for i, v in enumerate(dh) if v},
                      "mean_rel": (rep.mean_distortion - fx["mean_distortion"]) / fx["mean_distortion"],
                      "max_err": rep.max_distortion - fx["max_distortion"]}
    rng = np.random.default_rng(0)
    clouds = [("c3_8192", torch.from_numpy(np.ascontiguousarray(X[np.sort(rng.choice(60000, 8192, replace=False))])).cuda(), 50),
              ("c4_8192", ds.c4_power_law(n=8192, seed=4), 64),
              ("c5_8192", ds.c5_mixture(n=8192, seed=5), 128)]
    for name, C, r in clouds:
        m = adg.fit(C, r, adg.SpectralBackend.exact, 0)
        Yc = adg.transform_all(m, C).data
        res = {}
        for bins in (50, 1000):
            e = adg.evaluate(C, Yc, hist_bins=bins, engine="exact")
            s = adg.evaluate(C, Yc, hist_bins=bins, engine=os.environ.get("PROBE_ENGINE", "screen_exact_hist"))
            d = np.asarray(s.histogram, np.int64) - np.asarray(e.histogram, np.int64)
            res[bins] = {"moved": int(np.abs(d).sum() // 2), "edge_pairs": s.edge_pairs,
                         "max_diff": s.max_distortion - e.max_distortion}
        out[name] = res
    print(json.dumps(out), flush=True)

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
    else:
        for band in sys.argv[1:] or ["0", "0.125", "0.25", "0.5"]:
            env = dict(os.environ, ADG_EDGE_BAND=band)
            subprocess.run([sys.executable, __file__, "child"], env=env, check=False)

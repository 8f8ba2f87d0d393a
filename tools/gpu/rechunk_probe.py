import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
def child():
    import numpy as np, torch
    import paper_1609_05388_b200 as adg
    from paper_1609_05388_b200 import datasets as ds
    X = ds.c3_mnist_like()
    rng = np.random.default_rng(0)
    C = torch.from_numpy(np.ascontiguousarray(X[np.sort(rng.choice(60000, 8192, replace=False))])).cuda()
    m = adg.fit(C, 50, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(m, C).data
    e = adg.evaluate(C, Y, hist_bins=1000, engine="exact")
    s = adg.evaluate(C, Y, hist_bins=1000, engine="screen")
    d = np.asarray(s.histogram, np.int64) - np.asarray(e.histogram, np.int64)
    print(json.dumps({"band": os.environ.get("ADG_EDGE_BAND"), "cap": os.environ.get("ADG_EDGE_CAP"),
                      "moved": int(np.abs(d).sum() // 2), "sum_dh": int(d.sum()), "edges": s.edge_pairs,
                      "tot_s": int(np.asarray(s.histogram).sum()), "tot_e": int(np.asarray(e.histogram).sum())}), flush=True)
if __name__ == "__main__":
    if sys.argv[1:] == ["child"]:
        child()
    else:
        for band, cap in [("1", ""), ("1", "20000000"), ("0.25", ""), ("0.25", "400000"), ("0.25", "200000"), ("0.125", "100000")]:
            env = dict(os.environ, ADG_EDGE_BAND=band)
            if cap: env["ADG_EDGE_CAP"] = cap
            subprocess.run([sys.executable, __file__, "child"], env=env)

"""Reports of two builds of libadg.so on the same inputs, bit for bit
(profiling / refactoring aid): python report_identity.py A.so B.so"""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def child():
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    import paper_1609_05388_b200 as adg
    from paper_1609_05388_b200 import datasets as ds
    out = {}
    Xh = ds.c3_mnist_like()
    X = torch.from_numpy(Xh).cuda()
    m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(m, X).data
    for eng in ("screen", "screen_exact_hist"):
        r = adg.evaluate(X, Y, hist_bins=50, engine=eng)
        out["c3_" + eng] = [r.max_distortion.hex(), r.mean_distortion.hex(), list(r.argmax), [int(h) for h in r.histogram]]
    g = torch.Generator().manual_seed(5)
    for (n, d, rr, dt) in ((9000, 388, 40, torch.float32), (7000, 256, 24, torch.bfloat16), (5000, 1000, 70, torch.float32)):
        Xr = torch.randn(n, d, generator=g).to(dt).cuda()
        Yr = (Xr.float() @ (torch.randn(d, rr, generator=g).cuda() / d ** 0.5)).contiguous()
        r = adg.evaluate(Xr, Yr, hist_bins=40, engine="screen")
        out[f"rand_{n}_{d}_{rr}_{dt}"] = [r.max_distortion.hex(), r.mean_distortion.hex(), list(r.argmax), [int(h) for h in r.histogram]]
    mh = adg.AdagioModel(m.mean.cpu().numpy(), adg.OrthonormalBasis(m.basis.rows.cpu().numpy()),
                         adg.JlMatrix(m.sketch.entries.cpu().numpy()), 0)
    Xp = torch.from_numpy(Xh).pin_memory().numpy()
    r = adg.distort_model(mh, Xp, hist_bins=50, engine="screen")
    out["c3_distort_model"] = [r.max_distortion.hex(), r.mean_distortion.hex(), list(r.argmax), [int(h) for h in r.histogram]]
    print(json.dumps(out))

if __name__ == "__main__":
    if sys.argv[1] == "child":
        child()
    else:
        res = []
        for lib in sys.argv[1:3]:
            p = subprocess.run([sys.executable, __file__, "child"], env={**os.environ, "ADG_LIB": lib},
                               capture_output=True, text=True)
            line = [l for l in p.stdout.splitlines() if l.startswith("{")]
            if not line:
                print(lib, "FAILED", p.stderr[-2000:])
                sys.exit(1)
            res.append(json.loads(line[0]))
        a, b = res
        for k in a:
            print(("SAME " if a[k] == b.get(k) else "DIFF ") + k, a[k][:3], "" if a[k] == b.get(k) else b.get(k)[:3])

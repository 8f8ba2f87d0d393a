"""fit() outputs of two builds bit for bit, and the steady-state fit time
(profiling / refactoring aid): python fit_identity.py A.so B.so"""
import os, sys, json, subprocess, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import numpy as np, torch, hashlib
    import paper_1609_05388_b200 as adg
    from paper_1609_05388_b200 import datasets as ds
    out = {}
    g = torch.Generator().manual_seed(3)
    cases = [("c3", torch.from_numpy(ds.c3_mnist_like()).cuda(), 50, adg.SpectralBackend.exact),
             ("c3_rand", torch.from_numpy(ds.c3_mnist_like()).cuda(), 50, adg.SpectralBackend.randomized),
             ("g2000", torch.randn(2000, 256, generator=g).cuda(), 30, adg.SpectralBackend.exact),
             ("g5000_600", torch.randn(5000, 600, generator=g).cuda(), 80, adg.SpectralBackend.exact)]
    for name, X, r, be in cases:
        m = adg.fit(X, r, be, 0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            m = adg.fit(X, r, be, 0)
        torch.cuda.synchronize()
        h = hashlib.sha256(m.basis.rows.cpu().numpy().tobytes() + m.mean.cpu().numpy().tobytes()).hexdigest()[:16]
        out[name] = [h, round((time.perf_counter() - t) / 3 * 1e3, 2)]
    print(json.dumps(out))
else:
    res = []
    for lib in sys.argv[1:3]:
        p = subprocess.run([sys.executable, __file__, "child"], env={**os.environ, "ADG_LIB": lib}, capture_output=True, text=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("{")]
        if not line:
            print(lib, "FAILED", p.stderr[-1500:]); sys.exit(1)
        res.append(json.loads(line[0]))
    for k in res[0]:
        print(("SAME " if res[0][k][0] == res[1][k][0] else "DIFF ") + k, "fit ms", res[0][k][1], "->", res[1][k][1])

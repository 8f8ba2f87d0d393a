"""4-CTA multicast screen (ADG_SCREEN_MC=1) against the 2-CTA kernel: reports
bit for bit on C3 and random shapes, and the screen time (profiling aid)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

def rep_key(r):
    return [r.max_distortion.hex(), r.mean_distortion.hex(), list(r.argmax), [int(h) for h in r.histogram],
            r.n_pairs_evaluated, r.n_zero_distance_pairs]

def both(X, Y, bins=50, engine="screen"):
    out = {}
    for mc in ("0", "1"):
        os.environ["ADG_SCREEN_MC"] = mc
        r = adg.evaluate(X, Y, hist_bins=bins, engine=engine)
        torch.cuda.synchronize()
        out[mc] = rep_key(r)
    return out["0"] == out["1"], out

g = torch.Generator().manual_seed(7)
for (n, d, rr, dt) in ((5000, 64, 16, torch.float32), (9001, 388, 40, torch.float32), (7000, 256, 24, torch.bfloat16),
                       (12345, 784, 50, torch.float32)):
    X = torch.randn(n, d, generator=g).to(dt).cuda()
    Y = (X.float() @ (torch.randn(d, rr, generator=g).cuda() / d ** 0.5)).contiguous()
    ok, o = both(X, Y, 40)
    print(f"n={n} d={d} r={rr} {dt}: identical={ok}", "" if ok else o, flush=True)
    ok, o = both(X, Y, 40, "screen_exact_hist")
    print(f"  exact_hist identical={ok}", flush=True)
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(m, X).data
ok, o = both(X, Y)
print("C3 identical", ok, o["1"][:3], flush=True)
flush = torch.empty(64 << 20, device="cuda")
for rnd in range(3):
    for mc in ("0", "1"):
        os.environ["ADG_SCREEN_MC"] = mc
        ks = []
        for _ in range(6):
            flush.zero_()
            adg.evaluate(X, Y, hist_bins=50, engine="screen")
            torch.cuda.synchronize()
            ks.append(adg.api.last_screen_kernel_ms(0))
        print(f"MC={mc}: screen ms median {statistics.median(ks[1:]):.4f} min {min(ks[1:]):.4f}", flush=True)

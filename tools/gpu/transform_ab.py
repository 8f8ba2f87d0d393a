"""TMEM-fed transform (transform_tm_kernel) against the TMA-box kernel
(ADG_TRANSFORM_TC=1): bit-identical Y on several shapes, and cold-L2 device
time on C3 (profiling / parity aid)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

def both(m, X):
    os.environ.pop("ADG_TRANSFORM_TC", None)
    a = adg.transform_all(m, X).data.clone()
    os.environ["ADG_TRANSFORM_TC"] = "1"
    b = adg.transform_all(m, X).data.clone()
    os.environ.pop("ADG_TRANSFORM_TC", None)
    return a, b

g = torch.Generator().manual_seed(1)
for (n, d, r) in ((1000, 256, 20), (5000, 388, 40), (777, 96, 17), (20000, 1024, 128), (3000, 512, 250)):
    X = torch.randn(n, d, generator=g).cuda()
    m = adg.fit(X, r, adg.SpectralBackend.exact, 0)
    a, b = both(m, X)
    print(f"n={n} d={d} r={r}: identical={torch.equal(a, b)} maxdiff={(a - b).abs().max().item():.3e}", flush=True)
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
a, b = both(m, X)
print(f"C3: identical={torch.equal(a, b)} maxdiff={(a - b).abs().max().item():.3e}", flush=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for tc in (None, "1", None, "1"):
    if tc:
        os.environ["ADG_TRANSFORM_TC"] = tc
    else:
        os.environ.pop("ADG_TRANSFORM_TC", None)
    ts = []
    for _ in range(12):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); adg.transform_all(m, X); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(("tma-box" if tc else "tmem-fed"), "transform_all ms median %.4f min %.4f" % (statistics.median(ts[2:]), min(ts[2:])), flush=True)
if os.environ.get("TM_DEBUG_SWEEP"):
    os.environ.pop("ADG_TRANSFORM_TC", None)
    for dbg in ("1", "0"):
        os.environ["ADG_TM_DEBUG"] = dbg
        ts = []
        for _ in range(12):
            flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); adg.transform_all(m, X); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print("ADG_TM_DEBUG", dbg, "ms median %.4f" % statistics.median(ts[2:]), flush=True)

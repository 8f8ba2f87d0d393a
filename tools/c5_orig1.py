"""C5 screen with the one-pass original side (bf16 planes exact) against the
forced three-pass kernel (ADG_SCREEN_ORIG3), full size, one GPU."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
X = ds.c5_mixture(n=n)
m = adg.fit(X, 128, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(m, X).data
out = {}
for tag in ["orig1", "orig3", "orig1"]:
    if tag == "orig3":
        os.environ["ADG_SCREEN_ORIG3"] = "1"
    else:
        os.environ.pop("ADG_SCREEN_ORIG3", None)
    adg.evaluate(X, Y, hist_bins=50, engine="screen")
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = adg.evaluate(X, Y, hist_bins=50, engine="screen")
    torch.cuda.synchronize()
    out[tag] = {"wall_s": time.perf_counter() - t, "screen_ms": adg.api.last_screen_kernel_ms(0),
                "max": rep.max_distortion, "argmax": rep.argmax, "mean": rep.mean_distortion}
P = n * (n - 1) / 2
for k, v in out.items():
    v["alg_tflops"] = 2 * (X.shape[1] + 128) * P / (v["screen_ms"] / 1e3) / 1e12
print(json.dumps({"n": n, "d": X.shape[1], **out}))

"""The pipelined run_distort flow (adg_distort_model from pinned host X) on
C4 / C5 at full size: report bit-identical to transform_all + evaluate on the
device, and the end-to-end time (robustness / profiling aid).
  python e2e_big.py c4|c5"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
cfg = sys.argv[1]
n, d, r, bins, _ = ds.CONFIGS[cfg]
X = ds.make(cfg)
m = adg.fit(X, r, adg.SpectralBackend.exact, 0)
torch.cuda.synchronize()
t = time.perf_counter()
Y = adg.transform_all(m, X).data
ref = adg.evaluate(X, Y, hist_bins=bins, engine="screen")
torch.cuda.synchronize()
dev_s = time.perf_counter() - t
mh = adg.AdagioModel(m.mean.cpu().numpy(), adg.OrthonormalBasis(m.basis.rows.cpu().numpy()),
                     adg.JlMatrix(m.sketch.entries.cpu().numpy()), 0)
Xp = X.cpu().pin_memory()
del X, Y
torch.cuda.empty_cache()
ts = []
for k in range(2):
    t = time.perf_counter()
    got = adg.distort_model(mh, Xp if Xp.dtype != torch.bfloat16 else Xp, hist_bins=bins, engine="screen")
    ts.append(time.perf_counter() - t)
same = (got.max_distortion == ref.max_distortion and got.argmax == ref.argmax and
        got.mean_distortion == ref.mean_distortion and list(got.histogram) == list(ref.histogram))
print(json.dumps({"config": cfg, "identical": same, "device_job_s": dev_s, "e2e_s": ts,
                  "pairs": n * (n - 1) // 2, "max": got.max_distortion, "argmax": got.argmax}), flush=True)

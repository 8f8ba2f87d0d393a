"""Generate tests/golden/c3_fixture.{npz,json} (TEST INFRASTRUCTURE).

BASELINE config C3 (n=60000, d=784, r=50) through the CPU oracle:
  * the oracle fit (numpy/LAPACK stand-in for BDCSVD; see oracle/oracle.py) is
    stored (mean, P) so the GPU box rebuilds the identical fp64 embedding with
    the oracle's deterministic C transform instead of re-running LAPACK;
  * the full all-pairs evaluate of (X, fp32(Y)) with the reference algorithm
    (1,799,970,000 pairs, fp64 direct differences, block-ordered Neumaier),
    plus per-edge counts of pairs within EDGE_BAND of a histogram edge.
X is regenerated from its seed on the GPU box; its sha256 is recorded and
checked first.  Run:  python tests/golden/make_c3_fixture.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_1609_05388_b200 import datasets as ds  # noqa: E402

EDGE_BAND = 1e-4


def main():
    t0 = time.time()
    X = ds.c3_mnist_like()
    n, d, r, bins, _ = ds.CONFIGS["c3"]
    X64 = X.astype(np.float64)
    mean, P, S = oracle.fit(X64, r, "exact", 0)
    Y = oracle.transform_all(mean, P, S, X64)
    Y32 = Y.astype(np.float32)
    t1 = time.time()
    rep = oracle.evaluate(X64, Y32.astype(np.float64), hist_bins=bins, edge_band=EDGE_BAND)
    t2 = time.time()
    out = os.path.join(ROOT, "tests", "golden")
    np.savez_compressed(os.path.join(out, "c3_fixture.npz"), mean=mean, P=P)
    doc = {
        "config": "c3", "n": n, "d": d, "r": r, "hist_bins": bins, "edge_band": EDGE_BAND,
        "x_sha256": hashlib.sha256(X.tobytes()).hexdigest(),
        "y32_sha256": hashlib.sha256(Y32.tobytes()).hexdigest(),
        "max_distortion": rep.max_distortion, "mean_distortion": rep.mean_distortion,
        "argmax": list(rep.argmax), "n_pairs_evaluated": rep.n_pairs_evaluated,
        "n_zero_distance_pairs": rep.n_zero_distance_pairs,
        "histogram": [int(v) for v in rep.histogram],
        "edge_near": [int(v) for v in rep.edge_near],
        "edge_near10": [int(v) for v in rep.edge_near10],
        "seconds": {"fit_transform": t1 - t0, "evaluate": t2 - t1},
        "threads": os.cpu_count(),
        "_provenance": "oracle/adagio_oracle.c evaluate (restatement of proj/src/distortion.cpp)",
    }
    with open(os.path.join(out, "c3_fixture.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({k: v for k, v in doc.items() if k not in ("histogram", "edge_near")}))


if __name__ == "__main__":
    main()

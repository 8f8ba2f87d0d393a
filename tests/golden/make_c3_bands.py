"""Add the SCREEN error-band edge counts to tests/golden/c3_fixture.json
(TEST INFRASTRUCTURE).  For the fixture's C3 job (X from its seed, Y from the
committed oracle model), oracle.edge_band_counts gives, per bin edge, the
pairs whose exact value lies within the GPU screen's rigorous per-pair error
bound of that edge ("band_rigorous") and within 1/4 of it ("band_quarter",
the exact-histogram mode's band).  Run:  python tests/golden/make_c3_bands.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_1609_05388_b200 import datasets as ds  # noqa: E402


def main():
    path = os.path.join(ROOT, "tests", "golden", "c3_fixture.json")
    doc = json.load(open(path))
    X = ds.c3_mnist_like()
    z = np.load(os.path.join(ROOT, "tests", "golden", "c3_fixture.npz"))
    S = oracle.sample_jl(25, 784, oracle.derive_seed(0, "jl"))
    Y = oracle.transform_all(z["mean"], z["P"], S, X.astype(np.float64)).astype(np.float32)
    t0 = time.time()
    rig, quarter = oracle.edge_band_counts(X, Y, hist_bins=doc["hist_bins"], frac=0.25)
    doc["band_rigorous"] = [int(v) for v in rig]
    doc["band_quarter"] = [int(v) for v in quarter]
    doc["band_rel_eps"] = oracle.screen_rel_eps(784, 50)
    doc.setdefault("seconds", {})["band_counts"] = time.time() - t0
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({"rigorous_total": int(rig.sum()), "quarter_total": int(quarter.sum()),
                      "seconds": time.time() - t0}))


if __name__ == "__main__":
    main()

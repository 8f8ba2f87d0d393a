"""Sweep benchmark on BASELINE config C3 (n=60000, d=784, MNIST-shaped
synthetic): proj/src/sweep.cpp's tradeoff over dims x methods and a
min_dim_for_distortion search, every cell scored on all 1.8e9 pairs.

Prints one JSON line: per-cell GPU seconds (fit / eval as the reference
splits them), the min_dim result and probe count, and the CPU port's cost
per cell from its measured all-pairs rate on a bounded row sample (the
reference itself cannot be built here).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import Method
from paper_1609_05388_b200 import datasets as ds

X = torch.from_numpy(ds.c3_mnist_like()).cuda()
n, d = X.shape
dims = [10, 25, 50, 100]
methods = [Method.adagio_exact, Method.pca, Method.jl]
adg.tradeoff(X[:5000], [2, 10], [Method.pca, Method.jl], [0])  # warm-up (lazy module load, pools)
torch.cuda.synchronize()
t0 = time.perf_counter()
rows = adg.tradeoff(X, dims, methods, [0])
t_sweep = time.perf_counter() - t0
t0 = time.perf_counter()
md = adg.min_dim_for_distortion(X, Method.adagio_exact, 0.5, 0, 1, 200)
t_min = time.perf_counter() - t0
t0 = time.perf_counter()
mp = adg.min_dim_for_distortion(X, Method.pca, 0.5, 0, 1, 200)
t_minp = time.perf_counter() - t0

# CPU port: all-pairs evaluate rate on a bounded sample (rows [0, R) of one cell)
from oracle import oracle as orc
orc.lib()
Y = adg.transform_all(adg.fit(X, 50, adg.SpectralBackend.exact, 0), X).data.cpu().numpy()
Xh = X.cpu().numpy()
rows_s = 1500
t0 = time.perf_counter()
rep = orc.evaluate_f32(Xh, Y, hist_bins=50, threads=0, row_range=(0, rows_s))
cpu_dt = time.perf_counter() - t0
cpu_rate = (rep.n_pairs_evaluated + rep.n_zero_distance_pairs) / cpu_dt
P = n * (n - 1) // 2
print(json.dumps({
    "workload": "c3 sweep: tradeoff dims %s x methods %s x seed 0; min_dim adagio_exact delta 0.5 in [1, 200]"
                % (dims, [m.name for m in methods]),
    "pairs_per_cell": P,
    "tradeoff_seconds": t_sweep, "cells": len(rows),
    "cells_detail": [{"method": r.method.name, "r": r.target_dim, "max": r.max_distortion,
                      "fit_s": round(r.fit_seconds, 4), "eval_s": round(r.eval_seconds, 4)} for r in rows],
    "gpu_pairs_per_s_per_cell": P / (t_sweep / len(rows)),
    "min_dim": {"target_dim": md.target_dim, "achieved": md.achieved,
                "achieved_distortion": md.achieved_distortion, "monotone": md.monotone,
                "probes": md.probes, "probes_refined": md.probes_refined, "seconds": t_min},
    "min_dim_pca": {"target_dim": mp.target_dim, "achieved": mp.achieved,
                    "achieved_distortion": mp.achieved_distortion, "monotone": mp.monotone,
                    "probes": mp.probes, "probes_refined": mp.probes_refined, "seconds": t_minp},
    "cpu_port": {"pairs_per_s": cpu_rate, "threads": os.cpu_count(),
                 "sample": f"rows [0,{rows_s}) of one C3 cell", "seconds_per_cell": P / cpu_rate},
}), flush=True)

"""BASELINE configs C4 (n=1e6, d=960, 5e11 pairs) and C5 (n=2e5, d=4096,
bf16) at full size on one GPU, pinned to the reference's arithmetic:

* EXACT engine (adg_exact_tiled.cu: the reference's per-pair fp64 direct
  differences over every pair, ~3 min for C4, ~30 s for C5) is the golden
  report; its per-pair arithmetic is the block engine's, itself pinned to the
  oracle (tests/test_gpu_parity.py, test_exact_tiled_matches_block_and_oracle);
* SCREEN_EXACT_HIST gives the golden histogram bin for bin, and the golden
  counts, max and argmax;
* SCREEN (default) gives the golden counts, max and argmax; its histogram may
  move pairs across an edge within the screened error, and its mean carries
  the tensor-core accumulation bias: both are measured and bounded
  (moved <= 2e-5 of the pairs, mean within 1e-4 relative) and written to
  $ADG_REPORT_DIR/full_scale_<config>.json when that is set;
* the reference CLI's default mode above n = 5000 (sampled, m = 2e6,
  derive_seed(0, "sampling"); proj/tools/adagio_main.cpp:215-219) on the GPU
  equals the CPU oracle's on the same host copies: histogram identical, max /
  mean within 1e-13, same argmax;
* determinism: a second SCREEN evaluation is bit-identical.
"""
import json
import os
import time

import numpy as np
import pytest

import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _timed(fn):
    import torch
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t


def _check(name, oracle):
    import torch
    n, d, r, bins, _ = ds.CONFIGS[name]
    X = ds.make(name)
    m = adg.fit(X, r, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(m, X).data
    P = n * (n - 1) // 2
    ex, t_ex = _timed(lambda: adg.evaluate(X, Y, hist_bins=bins, engine="exact"))
    sc, t_sc = _timed(lambda: adg.evaluate(X, Y, hist_bins=bins, engine="screen"))
    eh, t_eh = _timed(lambda: adg.evaluate(X, Y, hist_bins=bins, engine="screen_exact_hist"))
    assert ex.engine == "exact" and ex.n_pairs_evaluated + ex.n_zero_distance_pairs == P
    for rep in (sc, eh):
        assert rep.n_pairs_evaluated == ex.n_pairs_evaluated
        assert rep.n_zero_distance_pairs == ex.n_zero_distance_pairs
        assert abs(rep.max_distortion - ex.max_distortion) <= 1e-13
        assert rep.argmax == ex.argmax
        assert int(np.asarray(rep.histogram).sum()) == rep.n_pairs_evaluated
    h_ex = np.asarray(ex.histogram, np.int64)
    assert np.array_equal(np.asarray(eh.histogram, np.int64), h_ex)
    dh = np.asarray(sc.histogram, np.int64) - h_ex
    moved = int(np.abs(dh).sum() // 2)
    bias = (sc.mean_distortion - ex.mean_distortion) / ex.mean_distortion
    assert moved <= 2e-5 * P
    assert abs(bias) <= 1e-4
    # the reference CLI's default mode at this size, GPU vs CPU oracle
    seed = adg.derive_seed(0, "sampling")
    smp = adg.evaluate(X, Y, adg.PairSampling.sample(2000000, seed), hist_bins=bins)
    Xh = X.float().cpu().numpy()
    Yh = Y.float().cpu().numpy()
    ref = oracle.evaluate_f32_sampled(Xh, Yh, 2000000, seed, hist_bins=bins)
    assert smp.n_pairs_evaluated == ref.n_pairs_evaluated
    assert smp.n_zero_distance_pairs == ref.n_zero_distance_pairs
    assert np.array_equal(np.asarray(smp.histogram, np.int64), np.asarray(ref.histogram, np.int64))
    assert abs(smp.max_distortion - ref.max_distortion) <= 1e-13 and smp.argmax == ref.argmax
    assert abs(smp.mean_distortion - ref.mean_distortion) <= 1e-13
    assert ex.max_distortion >= smp.max_distortion
    again = adg.evaluate(X, Y, hist_bins=bins, engine="screen")
    assert again.max_distortion == sc.max_distortion and again.argmax == sc.argmax
    assert again.mean_distortion == sc.mean_distortion
    assert np.array_equal(again.histogram, sc.histogram)
    out = {"config": name, "n": n, "d": d, "r": r, "pairs": P,
           "exact": {"max": ex.max_distortion, "argmax": ex.argmax, "mean": ex.mean_distortion,
                     "zero": ex.n_zero_distance_pairs, "seconds": t_ex},
           "screen": {"moved_pairs_net": moved, "mean_rel_bias": bias, "seconds": t_sc,
                      "dh_nonzero": {int(i): int(v) for i, v in enumerate(dh) if v}},
           "screen_exact_hist": {"edge_pairs": eh.edge_pairs, "seconds": t_eh, "hist_equal": True},
           "sampled_2e6": {"max": smp.max_distortion, "mean": smp.mean_distortion,
                           "equal_to_oracle": True}}
    print(json.dumps(out))
    rd = os.environ.get("ADG_REPORT_DIR")
    if rd:
        os.makedirs(rd, exist_ok=True)
        with open(os.path.join(rd, f"full_scale_{name}.json"), "w") as f:
            json.dump(out, f, indent=1)
    del X, Y
    torch.cuda.empty_cache()


def test_c5_full_scale(oracle):
    _check("c5", oracle)


def test_c4_full_scale(oracle):
    _check("c4", oracle)

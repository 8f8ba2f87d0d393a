"""BASELINE configs C4 (n=1e6, d=960, 5e11 pairs) and C5 (n=2e5, d=4096,
bf16) at full size on one GPU.  The CPU oracle cannot evaluate them (~1 day /
~4 h), so parity is checked through size-independent properties:

* counts: evaluated + zero pairs = n(n-1)/2; histogram sums to the evaluated count;
* the reported maximum is an exact fp64 value: it equals the reference formula
  (oracle.pair_distortion, fp64 direct differences) at the reported argmax pair;
* it dominates an exact evaluation of 2e6 sampled pairs (the reference CLI's
  default mode above n = 5000, adagio_main.cpp:215-219, same Floyd indices);
* the mean agrees with the sampled mean to sampling accuracy;
* determinism: a second evaluation is bit-identical.
"""
import numpy as np
import pytest

import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _check(name, oracle):
    import torch
    n, d, r, bins, _ = ds.CONFIGS[name]
    X = ds.make(name)
    m = adg.fit(X, r, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(m, X).data
    rep = adg.evaluate(X, Y, hist_bins=bins, engine="screen")
    P = n * (n - 1) // 2
    assert rep.n_pairs_evaluated + rep.n_zero_distance_pairs == P
    assert int(rep.histogram.sum()) == rep.n_pairs_evaluated
    i, j = rep.argmax
    xi, xj = X[i].double().cpu().numpy(), X[j].double().cpu().numpy()
    fi, fj = Y[i].double().cpu().numpy(), Y[j].double().cpu().numpy()
    assert abs(oracle.pair_distortion(xi, xj, fi, fj) - rep.max_distortion) <= 1e-12
    smp = adg.evaluate(X, Y, adg.PairSampling.sample(2000000, adg.derive_seed(0, "sampling")),
                       hist_bins=bins)
    assert smp.n_pairs_evaluated == 2000000
    assert rep.max_distortion >= smp.max_distortion
    assert abs(rep.mean_distortion - smp.mean_distortion) <= 5e-3 * rep.mean_distortion
    again = adg.evaluate(X, Y, hist_bins=bins, engine="screen")
    assert again.max_distortion == rep.max_distortion and again.argmax == rep.argmax
    assert again.mean_distortion == rep.mean_distortion
    assert np.array_equal(again.histogram, rep.histogram)
    del X, Y
    torch.cuda.empty_cache()


def test_c4_full_scale(oracle):
    _check("c4", oracle)


def test_c5_full_scale(oracle):
    _check("c5", oracle)

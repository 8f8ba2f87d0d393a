"""Sweeps on the GPU (proj/src/sweep.cpp through adg_tradeoff /
adg_min_dim_for_distortion): the reference's own tests
(proj/tests/test_sweep.cpp) restated, plus parity of every cell with the
oracle's sweep restatement (oracle/oracle.py tradeoff / min_dim_for_distortion)
on the same clouds, including n > 4096 where cells are scored by the max-only
SCREEN evaluator.
"""
import numpy as np
import pytest

import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import Method

pytestmark = pytest.mark.gpu

NAMES = {Method.adagio_exact: "adagio_exact", Method.adagio_randomized: "adagio_randomized",
         Method.pca: "pca", Method.jl: "jl", Method.external: "external"}


def median(v):
    v = sorted(v)
    return v[len(v) // 2]


# ------------------------------------------------ proj/tests/test_sweep.cpp
def test_method_names_round_trip():
    for m in Method:
        assert adg.method_from_name(adg.method_name(m)) == m
    with pytest.raises(ValueError, match="unknown method 'numax'"):
        adg.method_from_name("numax")


def test_pca_at_cloud_rank_is_isometry(oracle):
    rows = adg.tradeoff(oracle.low_rank_cloud(50, 20, 5, 1), [5], [Method.pca], [0])
    assert len(rows) == 1 and rows[0].max_distortion <= 1e-9 and rows[0].target_dim == 5


def test_pca_rows_seed_independent(oracle):
    rows = adg.tradeoff(oracle.gaussian_cloud(40, 15, 2), [6], [Method.pca], [0, 1, 2])
    assert len(rows) == 3
    assert rows[0].max_distortion == rows[1].max_distortion == rows[2].max_distortion


def test_median_distortion_decreases(oracle):
    cloud = oracle.split_energy_cloud(120, 40, 6, 0.9, 3)
    dims = [4, 10, 20, 36]
    for method in (Method.adagio_exact, Method.pca, Method.jl):
        rows = adg.tradeoff(cloud, dims, [method], [0, 1, 2, 3, 4])
        by = {}
        for r in rows:
            by.setdefault(r.target_dim, []).append(r.max_distortion)
        prev = 1e9
        for r in dims:
            m = median(by[r])
            assert m <= prev + 0.02
            prev = m


def test_tradeoff_reproducible(oracle):
    cloud = oracle.gaussian_cloud(35, 12, 4)
    a = adg.tradeoff(cloud, [3, 8], [Method.adagio_exact, Method.jl], [7, 8])
    b = adg.tradeoff(cloud, [3, 8], [Method.adagio_exact, Method.jl], [7, 8])
    assert [(r.method, r.target_dim, r.seed, r.max_distortion) for r in a] == \
           [(r.method, r.target_dim, r.seed, r.max_distortion) for r in b]


def test_tradeoff_validation(oracle):
    cloud = oracle.gaussian_cloud(20, 10, 5)
    with pytest.raises(ValueError, match="dims must be non-empty"):
        adg.tradeoff(cloud, [], [Method.pca], [0])
    with pytest.raises(ValueError, match=r"dim 11 outside \[1, 10\]"):
        adg.tradeoff(cloud, [11], [Method.pca], [0])
    with pytest.raises(ValueError, match="external needs an embedding matrix"):
        adg.tradeoff(cloud, [5], [Method.external], [0])
    with pytest.raises(ValueError, match="external matrix has 9 columns, cloud has 10"):
        adg.tradeoff(cloud, [5], [Method.external], [0], external_map=np.zeros((3, 9)))


def test_external_orthonormal_map_zero(oracle):
    rows = adg.tradeoff(oracle.gaussian_cloud(25, 8, 6), [1], [Method.external], [0],
                        external_map=np.eye(8))
    assert len(rows) == 1 and rows[0].target_dim == 8 and rows[0].max_distortion <= 1e-12


def test_min_dim_low_rank(oracle):
    res = adg.min_dim_for_distortion(oracle.low_rank_cloud(60, 25, 5, 7), Method.pca, 1e-6, 0, 1, 25)
    assert res.achieved and res.target_dim == 5 and res.achieved_distortion <= 1e-6


def test_min_dim_meets_delta_and_predecessor_misses(oracle):
    cloud = oracle.split_energy_cloud(100, 30, 5, 0.85, 8)
    res = adg.min_dim_for_distortion(cloud, Method.adagio_exact, 0.2, 3, 1, 30)
    assert res.achieved

    def at(r):
        return adg.tradeoff(cloud, [r], [Method.adagio_exact], [3])[0].max_distortion

    assert at(res.target_dim) <= 0.2
    if res.target_dim > 1:
        assert at(res.target_dim - 1) > 0.2


def test_min_dim_unreachable(oracle):
    res = adg.min_dim_for_distortion(oracle.gaussian_cloud(80, 40, 9), Method.jl, 0.01, 0, 1, 5)
    assert not res.achieved and res.target_dim == 5 and res.achieved_distortion > 0.01


def test_min_dim_validation(oracle):
    c = oracle.gaussian_cloud(20, 6, 1)
    with pytest.raises(ValueError, match="delta must lie in"):
        adg.min_dim_for_distortion(c, Method.pca, 1.5, 0, 1, 6)
    with pytest.raises(ValueError, match="need 1 <= r_min <= r_max <= d"):
        adg.min_dim_for_distortion(c, Method.pca, 0.5, 0, 3, 2)
    with pytest.raises(ValueError, match="external maps have a fixed dimension"):
        adg.min_dim_for_distortion(c, Method.external, 0.5, 0, 1, 6)


def test_sweep_csv_header(oracle):
    rows = adg.tradeoff(oracle.gaussian_cloud(20, 6, 10), [3], [Method.pca], [0])
    csv = adg.sweep_csv(rows)
    assert csv.startswith("method,target_dim,seed,max_distortion,fit_seconds,eval_seconds\n")
    assert "pca,3,0," in csv


# ------------------------------------------------------ parity with the oracle
@pytest.mark.parametrize("n,d", [(200, 24), (5000, 32)])
def test_tradeoff_matches_oracle(oracle, n, d):
    """Every cell's max distortion vs the oracle (reference formula in fp64,
    LAPACK stand-in basis).  n = 5000 runs the max-only SCREEN evaluator."""
    cloud = oracle.split_energy_cloud(n, d, 4, 0.8, 21)
    dims, seeds = [2, 7, 16], [0, 5]
    methods = [Method.adagio_exact, Method.adagio_randomized, Method.pca, Method.jl]
    rows = adg.tradeoff(cloud, dims, methods, seeds)
    ref = oracle.tradeoff(cloud, dims, [NAMES[m] for m in methods], seeds)
    assert len(rows) == len(ref)
    for r, (m, dim, seed, mx) in zip(rows, ref):
        assert (NAMES[r.method], r.target_dim, r.seed) == (m, dim, seed)
        assert abs(r.max_distortion - mx) <= 1e-7 * max(1.0, mx), (m, dim, seed, r.max_distortion, mx)
    ext = np.linalg.qr(np.random.default_rng(1).standard_normal((d, 5)))[0].T
    r = adg.tradeoff(cloud, [1], [Method.external], [0], external_map=ext)[0]
    mx = oracle.tradeoff(cloud, [1], ["external"], [0], external_map=ext)[0][3]
    assert r.target_dim == 5 and abs(r.max_distortion - mx) <= 1e-9 * max(1.0, mx)


def test_tradeoff_sampled_mode_matches_oracle(oracle):
    cloud = oracle.gaussian_cloud(300, 20, 3)
    seed = adg.derive_seed(0, "sampling")
    rows = adg.tradeoff(cloud, [6], [Method.jl], [1], adg.PairSampling.sample(5000, seed))
    ref = oracle.tradeoff(cloud, [6], ["jl"], [1], all_pairs=False, m=5000, sample_seed=seed)
    assert abs(rows[0].max_distortion - ref[0][3]) <= 1e-12


@pytest.mark.parametrize("method,delta", [(Method.adagio_exact, 0.25), (Method.pca, 0.3),
                                          (Method.jl, 0.6)])
def test_min_dim_matches_oracle(oracle, method, delta):
    cloud = oracle.split_energy_cloud(150, 40, 6, 0.8, 12)
    res = adg.min_dim_for_distortion(cloud, method, delta, 4, 1, 40)
    t, a, ok, mono, probed = oracle.min_dim_for_distortion(cloud, NAMES[method], delta, 4, 1, 40)
    # decisions agree unless a probed value sits within rounding of delta
    if all(abs(v - delta) > 1e-9 for v in probed.values()):
        assert (res.target_dim, res.achieved, res.monotone) == (t, ok, mono)
        assert abs(res.achieved_distortion - a) <= 1e-9 * max(1.0, a)


def test_max_distortion_max_only_screen(oracle):
    """adg_max_distortion above the exact engine's range (max-only SCREEN) is
    the full evaluator's maximum, bit for bit."""
    c = oracle.gaussian_cloud(5000, 40, 13).astype(np.float32)
    m = adg.fit(c, 10, adg.SpectralBackend.exact, 1)
    y = adg.transform_all(m, c).data
    full = adg.evaluate(c, y, engine="screen")
    assert adg.max_distortion(c, y) == full.max_distortion


def test_collapsing_map_many_candidate_rows(oracle):
    """A 2-D projection nearly collapses many pairs: the screen's bounds are
    loose there, so many rows go to the exact refine (batched kernel).  The
    max and its lowest-(i, j) argmax must still be the reference's."""
    c = oracle.gaussian_cloud(5000, 40, 17)
    P = oracle.exact_top_svd(c - c.mean(0), 2)[0]
    y = ((c - c.mean(0)) @ P.T).astype(np.float32)
    x = c.astype(np.float32)
    rep = adg.evaluate(x, y, engine="screen")
    ref = oracle.evaluate(x.astype(np.float64), y.astype(np.float64))
    assert rep.candidate_rows > 16
    assert rep.argmax == ref.argmax and abs(rep.max_distortion - ref.max_distortion) <= 1e-12
    assert rep.n_pairs_evaluated == ref.n_pairs_evaluated


def _search(values, delta, r_min, r_max):
    """proj/src/sweep.cpp:214-264 on known exact maxima (dict r -> max)."""
    probed = {}

    def probe(r):
        probed[r] = values[r]
        return values[r]

    at_min = probe(r_min)
    if at_min <= delta:
        res = (r_min, at_min, True)
    else:
        lo = hi = r_min
        at_hi = at_min
        while at_hi > delta and hi < r_max:
            lo = hi
            hi = min(r_max, max(hi * 2, hi + 1))
            at_hi = probe(hi)
        if at_hi > delta:
            res = (r_max, at_hi, False)
        else:
            while hi - lo > 1:
                mid = lo + (hi - lo) // 2
                if probe(mid) <= delta:
                    hi = mid
                else:
                    lo = mid
            res = (hi, probed[hi], True)
    prev, mono = None, True
    for r in sorted(probed):
        if prev is not None and probed[r] > prev + 1e-12:
            mono = False
        prev = probed[r]
    return res + (mono, len(probed))


@pytest.mark.parametrize("method,delta", [(Method.adagio_exact, 0.5), (Method.pca, 0.35), (Method.jl, 0.6)])
def test_min_dim_brackets_equal_exact_search(method, delta):
    """n = 6000 (screen engine): probes decided by their [L, U] bracket give
    the same answer as the search on exact maxima (tradeoff over every dim)."""
    from paper_1609_05388_b200 import datasets as ds
    X = ds.c3_mnist_like()[:6000]
    r_max = 48
    res = adg.min_dim_for_distortion(X, method, delta, 0, 1, r_max)
    rows = adg.tradeoff(X, list(range(1, r_max + 1)), [method], [0])
    values = {row.target_dim: row.max_distortion for row in rows}
    t, a, ok, mono, nprobes = _search(values, delta, 1, r_max)
    assert (res.target_dim, res.achieved, res.monotone) == (t, ok, mono)
    assert res.achieved_distortion == a  # exact, bit for bit
    assert res.probes == nprobes and 0 <= res.probes_refined <= res.probes

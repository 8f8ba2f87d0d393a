"""Pin the CPU oracle (test infrastructure) before trusting it.

* RNG: bit-exact against tests/golden/rng_golden.json, printed by the
  reference's own proj/include/adagio/rng.hpp compiled from /root/reference.
* Everything else: the reference's own known-answer / property tests,
  restated (proj/tests/test_distortion.cpp, test_jl.cpp, test_embed.cpp,
  test_spectral.cpp, test_dataset.cpp, acceptance.cpp #1/#2/#7).
"""
import json
import os

import numpy as np
import pytest

from tests.rng_emul import Stream

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rng_golden.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLDEN) as f:
        return json.load(f)


# ------------------------------------------------------------------- rng.hpp
def test_mix64_fnv_derive_golden(oracle, gold):
    for s, v in gold["mix64"]:
        assert oracle.mix64(int(s)) == int(v)
    for p, v in gold["fnv1a64"]:
        assert oracle.fnv1a64(p) == int(v)
    for s, p, v in gold["derive_seed"]:
        assert oracle.derive_seed(int(s), p) == int(v)


def test_hash_position_golden(oracle, gold):
    for s, i, j, h, sign in gold["hash_position"]:
        assert oracle.hash_position(int(s), i, j) == int(h)
        assert oracle.rademacher_sign(int(s), i, j) == sign


def test_seeded_rng_stream_golden(oracle, gold):
    for st in gold["stream"]:
        seed = int(st["seed"])
        s = Stream(seed)
        assert [s.next_u64() for _ in range(8)] == [int(v) for v in st["u64"]]
        assert [s.below(1000) for _ in range(8)] == st["below_1000"]
        got = [s.normal() for _ in range(9)]
        assert np.allclose(got, st["normal"], rtol=0, atol=1e-15)
        # the C oracle's raw stream agrees with the emulation
        assert list(map(int, oracle.rng_u64(seed, 8))) == [int(v) for v in st["u64"]]


def test_oracle_normals_match_stream(oracle):
    s = Stream(77)
    ref = [s.normal() for _ in range(101)]
    assert np.array_equal(oracle.rng_normal(77, 101), np.array(ref))


# ------------------------------------------------------------ distortion.cpp
def test_pair_distortion_arithmetic(oracle):
    # test_distortion.cpp:24-44
    x, y = [0, 0], [2, 0]
    assert oracle.pair_distortion(x, y, [0], [2]) == 0.0
    assert abs(oracle.pair_distortion(x, y, [0], [1]) - 0.5) <= 1e-15
    assert abs(oracle.pair_distortion(x, [1, 0], [0], [1.3]) - 0.3) <= 1e-12 * 0.3
    with pytest.raises(ValueError):
        oracle.pair_distortion(x, x, [0], [1])


def test_identity_reports_zero(oracle):
    # test_distortion.cpp:46-56
    c = oracle.gaussian_cloud(25, 6, 1)
    r = oracle.evaluate(c, c)
    assert r.max_distortion == 0.0 and r.mean_distortion == 0.0
    assert r.n_pairs_evaluated == 300 and r.n_zero_distance_pairs == 0
    assert not r.sampled and int(r.histogram.sum()) == 300


def test_four_point_hand_max(oracle):
    # test_distortion.cpp:58-80
    X = np.array([[1, 0, 0], [0, 2, 0], [0, 0, 3], [1, 1, 1]], float)
    E = X[:, :1].copy()
    vals = [abs(abs(X[i, 0] - X[j, 0]) / np.linalg.norm(X[i] - X[j]) - 1)
            for i in range(4) for j in range(i + 1, 4)]
    r = oracle.evaluate(X, E)
    assert r.n_pairs_evaluated == 6
    assert abs(r.max_distortion - max(vals)) <= 1e-15 * max(vals)
    assert abs(r.mean_distortion - sum(vals) / 6) <= 1e-14


def test_uniform_scaling(oracle):
    c = oracle.gaussian_cloud(15, 4, 2)
    r = oracle.evaluate(c, 2.0 * c)
    assert abs(r.max_distortion - 1) <= 1e-12 and abs(r.mean_distortion - 1) <= 1e-12


def test_blocked_matches_naive(oracle):
    # test_distortion.cpp:91-107 (the reference's own generator sequence)
    st = Stream(404)
    for _ in range(10):
        n = 10 + st.below(190)
        d = 2 + st.below(30)
        cloud = oracle.gaussian_cloud(n, d, st.next_u64())
        emb = cloud @ oracle.sample_jl(5, d, st.next_u64()).T
        mx, mean, ev, _ = oracle.naive_distortion(cloud, emb)
        r = oracle.evaluate(cloud, emb)
        assert abs(r.max_distortion - mx) <= 1e-12
        assert abs(r.mean_distortion - mean) <= 1e-12
        assert r.n_pairs_evaluated == ev


def test_thread_and_block_invariance(oracle):
    # test_distortion.cpp:109-134
    c = oracle.gaussian_cloud(120, 10, 3)
    emb = c @ oracle.sample_jl(4, 10, 9).T
    one = oracle.evaluate(c, emb, threads=1)
    two = oracle.evaluate(c, emb, threads=2)
    many = oracle.evaluate(c, emb, threads=0)
    tiny = oracle.evaluate(c, emb, pairs_per_block=7)
    for o in (two, many):
        assert o.max_distortion == one.max_distortion
        assert np.array_equal(o.histogram, one.histogram)
        assert o.mean_distortion == one.mean_distortion
    assert tiny.max_distortion == one.max_distortion
    assert np.array_equal(tiny.histogram, one.histogram)
    assert abs(tiny.mean_distortion - one.mean_distortion) <= 1e-12
    assert one.argmax == two.argmax == tiny.argmax


def test_scale_invariance(oracle):
    c = oracle.gaussian_cloud(60, 8, 5)
    emb = c @ oracle.sample_jl(3, 8, 2).T
    a = oracle.evaluate(c, emb)
    b = oracle.evaluate(3.5 * c, 3.5 * emb)
    assert abs(a.max_distortion - b.max_distortion) <= 1e-12
    assert abs(a.mean_distortion - b.mean_distortion) <= 1e-12


def test_sampling(oracle):
    # test_distortion.cpp:152-183
    c = oracle.gaussian_cloud(40, 6, 6)
    emb = c @ oracle.sample_jl(3, 6, 4).T
    a = oracle.evaluate(c, emb)
    s = oracle.evaluate(c, emb, all_pairs=False, m=780, sample_seed=123)
    assert s.sampled and s.sample_seed == 123
    assert s.max_distortion == a.max_distortion and s.mean_distortion == a.mean_distortion
    assert np.array_equal(s.histogram, a.histogram)
    c2 = oracle.gaussian_cloud(50, 5, 7)
    e2 = c2 @ oracle.sample_jl(2, 5, 1).T
    x = oracle.evaluate(c2, e2, all_pairs=False, m=200, sample_seed=9)
    y = oracle.evaluate(c2, e2, all_pairs=False, m=200, sample_seed=9)
    assert x.max_distortion == y.max_distortion and np.array_equal(x.histogram, y.histogram)
    assert x.n_pairs_evaluated == 200
    idx = oracle.sample_pair_indices(1225, 200, 9)
    assert len(set(idx.tolist())) == 200 and np.all(np.diff(idx.astype(np.int64)) > 0)


def test_duplicates_and_edges(oracle):
    # test_distortion.cpp:185-212
    c = oracle.gaussian_cloud(10, 3, 8)
    c[4] = c[2]
    c[7] = c[2]
    r = oracle.evaluate(c, c[:, :2].copy())
    assert r.n_zero_distance_pairs == 3 and r.n_pairs_evaluated == 42
    r = oracle.evaluate(np.array([[0.0], [1.0], [10.0]]), np.array([[0.0], [2.0], [8.5]]),
                        hist_bins=10, hist_max=1.0)
    assert r.histogram[-1] == 1 and r.histogram[1] == 1 and r.histogram[2] == 1


def test_validation(oracle):
    a = oracle.gaussian_cloud(10, 3, 1)
    b = oracle.gaussian_cloud(11, 3, 1)
    for kw in [dict(orig=a, emb=b), dict(orig=a, emb=a, all_pairs=False, m=46),
               dict(orig=a, emb=a, all_pairs=False, m=0), dict(orig=a, emb=a, hist_bins=0),
               dict(orig=a, emb=a, hist_max=0.0)]:
        with pytest.raises(ValueError):
            oracle.evaluate(**kw)


def test_decode_pair(oracle):
    n = 37
    p = 0
    for i in range(n):
        for j in range(i + 1, n):
            assert oracle.decode_pair(p, n) == (i, j)
            p += 1


def test_acceptance_7_engine_equals_naive(oracle):
    # proj/tests/acceptance.cpp:297-345 (first 20 of the 50 instances)
    st = Stream(777)
    for _ in range(20):
        n = 10 + st.below(190)
        d = 2 + st.below(39)
        cloud = oracle.gaussian_cloud(n, d, st.next_u64())
        k = 1 + st.below(8)
        emb = cloud @ oracle.sample_jl(k, d, st.next_u64()).T
        mx, mean, _, _ = oracle.naive_distortion(cloud, emb)
        hists = []
        for threads in (1, 2, 0):
            r = oracle.evaluate(cloud, emb, threads=threads)
            assert abs(r.max_distortion - mx) <= 1e-12
            assert abs(r.mean_distortion - mean) <= 1e-12
            hists.append(r.histogram)
        assert all(np.array_equal(h, hists[0]) for h in hists)


# -------------------------------------------------------------------- jl.cpp
def test_jl(oracle):
    # proj/tests/test_jl.cpp:15-74
    m = oracle.sample_jl(4, 10, 123)
    v = 1 / np.sqrt(4.0)
    assert np.all((m == v) | (m == -v))
    assert 0 < int((m == v).sum()) < 40
    assert np.array_equal(oracle.sample_jl(8, 33, 7), oracle.sample_jl(8, 33, 7))
    assert not np.array_equal(oracle.sample_jl(8, 33, 7), oracle.sample_jl(8, 33, 8))
    col = oracle.sample_jl(10000, 1, 2024)
    assert 0.47 <= (col > 0).mean() <= 0.53
    m = oracle.sample_jl(6, 300, 11)
    ref = sum((1 / np.sqrt(6.0)) ** 2 for _ in range(300))
    for row in m:
        acc = 0.0
        for e in row:
            acc += e * e
        assert acc == ref
    assert oracle.jl_dimension(800, 0.2, 0.01) == 4148
    assert oracle.jl_dimension(400, 0.5, 0.01) == 797
    assert oracle.jl_dimension(100, 0.3, 0.05) == 1357
    for args in [(1, 0.3, 0.01), (10, 0.0, 0.01), (10, 1.0, 0.01), (10, 0.3, 0.0), (10, 0.3, 1.0)]:
        with pytest.raises(ValueError):
            oracle.jl_dimension(*args)


# --------------------------------------------------------------- dataset.cpp
def test_center(oracle):
    # proj/tests/test_dataset.cpp:185-213
    cen, mean = oracle.center(np.array([[0.0, 0.0], [2.0, 2.0]]))
    assert cen[0, 0] == -1.0 and cen[1, 1] == 1.0 and mean[0] == 1.0 and mean[1] == 1.0
    c = oracle.gaussian_cloud(50, 6, 3)
    once, _ = oracle.center(c)
    twice, m2 = oracle.center(once)
    assert np.max(np.abs(twice - once)) < 1e-12 and np.max(np.abs(m2)) < 1e-12
    cen, mean = oracle.center(np.array([[5.0]]))
    assert cen[0, 0] == 0.0 and mean[0] == 5.0


# ----------------------------------------------------------------- embed.cpp
def test_transform_hand_example(oracle):
    # proj/tests/test_embed.cpp:70-84
    out = oracle.transform_all(np.zeros(3), np.array([[1.0, 0, 0]]), np.array([[1.0, 1, 1]]),
                               np.array([[1.0, 2, 3]]))
    assert abs(out[0, 0] - 1.0) <= 1e-15 and abs(out[0, 1] - 5.0) <= 1e-15


def test_fit_split_and_pythagoras(oracle):
    # test_embed.cpp:38-48, :118-138 and acceptance #2
    c = oracle.gaussian_cloud(30, 25, 1)
    mean, P, S = oracle.fit(c, 20, "exact", 0)
    assert P.shape == (10, 25) and S.shape == (10, 25)
    mean, P, S = oracle.fit(c, 5, "exact", 0)
    assert P.shape[0] == 2 and S.shape[0] == 3
    c = oracle.gaussian_cloud(30, 20, 8)
    mean, P, S = oracle.fit(c, 10, "exact", 3)
    emb = oracle.transform_all(mean, P, S, c)
    for i in range(c.shape[0]):
        for j in range(i + 1, c.shape[0]):
            diff = c[i] - c[j]
            pr = P @ diff
            res = diff - P.T @ pr
            lhs = np.sum((emb[i] - emb[j]) ** 2)
            rhs = np.sum(pr ** 2) + np.sum((S @ res) ** 2)
            assert abs(lhs - rhs) <= 1e-9


def test_complement_isometry(oracle):
    # test_embed.cpp:140-147 / acceptance #1
    c = oracle.gaussian_cloud(50, 30, 9)
    mean, P, S = oracle.fit(c, 10, "exact", 4)
    _, _, vt = np.linalg.svd(P, full_matrices=True)
    comp = vt[P.shape[0]:]
    emb = oracle.transform_all(mean, P, comp, c)
    assert oracle.evaluate(c, emb).max_distortion <= 1e-9


# -------------------------------------------------------------- spectral.cpp
def test_spectral_stand_in(oracle):
    # proj/tests/test_spectral.cpp:32-131
    b, sig = oracle.exact_top_svd(np.diag([3.0, 2.0, 1.0]), 1)
    assert np.allclose(sig, [3, 2, 1], atol=1e-12) and abs(b[0, 0] - 1) < 1e-12
    cen, _ = oracle.center(oracle.low_rank_cloud(40, 12, 2, 5))
    b, sig = oracle.exact_top_svd(cen, 2)
    assert np.all(sig[2:] <= 1e-9)
    assert np.max(np.abs(cen @ b.T @ b - cen)) < 1e-9
    cen, _ = oracle.center(oracle.gaussian_cloud(50, 30, 12))
    a = oracle.randomized_top_svd(cen, 5, 10, 2, 99)
    bb = oracle.randomized_top_svd(cen, 5, 10, 2, 99)
    assert np.array_equal(a[0], bb[0])
    cen, _ = oracle.center(oracle.low_rank_cloud(80, 25, 4, 21))
    e = oracle.exact_top_svd(cen, 4)[0]
    r = oracle.randomized_top_svd(cen, 4, 10, 2, 3)[0]
    assert np.max(np.abs(e.T @ e - r.T @ r)) <= 1e-6


# ------------------------------------------------------------ sweep.cpp
def test_oracle_sweep_reference_cases(oracle):
    """proj/tests/test_sweep.cpp restated on the oracle's sweep restatement."""
    rows = oracle.tradeoff(oracle.low_rank_cloud(50, 20, 5, 1), [5], ["pca"], [0])
    assert len(rows) == 1 and rows[0][3] <= 1e-9 and rows[0][1] == 5
    rows = oracle.tradeoff(oracle.gaussian_cloud(40, 15, 2), [6], ["pca"], [0, 1, 2])
    assert rows[0][3] == rows[1][3] == rows[2][3]
    c = oracle.gaussian_cloud(25, 8, 6)
    rows = oracle.tradeoff(c, [1], ["external"], [0], external_map=np.eye(8))
    assert rows[0][1] == 8 and rows[0][3] <= 1e-12
    t, a, ok, mono, _ = oracle.min_dim_for_distortion(oracle.low_rank_cloud(60, 25, 5, 7), "pca",
                                                      1e-6, 0, 1, 25)
    assert ok and t == 5 and a <= 1e-6
    t, a, ok, _, _ = oracle.min_dim_for_distortion(oracle.gaussian_cloud(80, 40, 9), "jl", 0.01, 0, 1, 5)
    assert not ok and t == 5 and a > 0.01
    with pytest.raises(ValueError, match="dims must be non-empty"):
        oracle.tradeoff(oracle.gaussian_cloud(20, 10, 5), [], ["pca"], [0])
    with pytest.raises(ValueError, match="outside"):
        oracle.tradeoff(oracle.gaussian_cloud(20, 10, 5), [11], ["pca"], [0])

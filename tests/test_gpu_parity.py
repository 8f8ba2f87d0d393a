"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): integer/bit work bit-exact; max distortion
within 1e-5 absolute with the identical argmax pair; histogram counts exact
away from bin edges (per-bin |diff| <= oracle pairs within EDGE_BAND of an
edge); pair / zero-pair counts exact; embeddings within 1e-4 relative
Frobenius of the reference's.
"""
import json
import os

import numpy as np
import pytest

import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds

pytestmark = pytest.mark.gpu

MAX_TOL = 1e-5
EDGE_BAND = 1e-4        # screen |v_screen - v_exact| stays far below this
EMBED_TOL = 1e-4        # relative Frobenius
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel_fro(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def check_report(rep, ref, edge_near=None, exact_hist=False, mean_tol=1e-6):
    assert rep.n_pairs_evaluated == ref.n_pairs_evaluated
    assert rep.n_zero_distance_pairs == ref.n_zero_distance_pairs
    assert abs(rep.max_distortion - ref.max_distortion) <= MAX_TOL
    assert rep.argmax == ref.argmax
    assert abs(rep.mean_distortion - ref.mean_distortion) <= mean_tol * max(1.0, ref.mean_distortion)
    h = np.asarray(rep.histogram, np.int64)
    hr = np.asarray(ref.histogram, np.int64)
    assert h.sum() == hr.sum() == ref.n_pairs_evaluated
    if exact_hist:
        assert np.array_equal(h, hr)
    elif edge_near is not None:
        # a bin can only differ by pairs sitting within EDGE_BAND of its edges
        en = np.asarray(edge_near, np.int64)
        slack = np.zeros_like(hr)
        slack[:-1] += en                 # upper edge of bin b is edge b+1 (index b)
        slack[1:] += en                  # lower edge of bin b+1
        assert np.all(np.abs(h - hr) <= slack), (h - hr, slack)


# ----------------------------------------------------------------- RNG / JL
def test_sample_jl_bit_exact(oracle):
    for k, d, seed in [(4, 10, 123), (8, 33, 7), (25, 784, oracle.derive_seed(0, "jl")),
                       (64, 4096, 99)]:
        g = adg.sample_jl(k, d, seed).entries
        assert np.array_equal(g, oracle.sample_jl(k, d, seed))


def test_sample_jl_golden():
    g = json.load(open(os.path.join(GOLDEN, "rng_golden.json")))
    for s, i, j, _h, sign in g["hash_position"]:
        if i < 5 and j < 7:
            m = adg.sample_jl(5, 7, int(s)).entries
            assert m[i, j] == sign / np.sqrt(5.0)


# ------------------------------------------------- evaluate: known answers
ENGINES = ["exact", "screen"]


@pytest.mark.parametrize("engine", ENGINES)
def test_identity_embedding_zero(engine, oracle):
    # proj/tests/test_distortion.cpp:46-56
    c = oracle.gaussian_cloud(25, 6, 1)
    r = adg.evaluate(c, c, engine=engine)
    assert r.max_distortion <= (0.0 if engine == "exact" else 1e-6)
    assert r.n_pairs_evaluated == 25 * 24 // 2
    assert r.n_zero_distance_pairs == 0
    assert int(np.sum(r.histogram)) == r.n_pairs_evaluated


@pytest.mark.parametrize("engine", ENGINES)
def test_four_point_hand_max(engine):
    # proj/tests/test_distortion.cpp:58-80
    X = np.array([[1, 0, 0], [0, 2, 0], [0, 0, 3], [1, 1, 1]], np.float64)
    E = X[:, :1]
    mx, s = 0.0, 0.0
    for i in range(4):
        for j in range(i + 1, 4):
            v = abs(abs(X[i, 0] - X[j, 0]) / np.linalg.norm(X[i] - X[j]) - 1.0)
            mx, s = max(mx, v), s + v
    r = adg.evaluate(X, E, engine=engine)
    assert r.n_pairs_evaluated == 6
    assert abs(r.max_distortion - mx) <= 1e-15 * max(1, mx) + 1e-15
    assert abs(r.mean_distortion - s / 6) <= (1e-14 if engine == "exact" else 1e-6)


@pytest.mark.parametrize("engine", ENGINES)
def test_uniform_scaling(engine, oracle):
    # proj/tests/test_distortion.cpp:82-89
    c = oracle.gaussian_cloud(15, 4, 2)
    r = adg.evaluate(c, 2.0 * c, engine=engine)
    assert abs(r.max_distortion - 1.0) <= 1e-12
    assert abs(r.mean_distortion - 1.0) <= (1e-12 if engine == "exact" else 1e-6)


@pytest.mark.parametrize("engine", ENGINES)
def test_blocked_matches_naive(engine, oracle):
    # proj/tests/test_distortion.cpp:91-107 (same generator sequence)
    u = oracle.rng_u64(404, 64)
    rng_i = 0
    draws = list(u)
    # emulate SeededRng(404): below / next_u64 from the raw stream
    from tests.rng_emul import Stream
    st = Stream(404)
    for _ in range(10):
        n = 10 + st.below(190)
        d = 2 + st.below(30)
        cloud = oracle.gaussian_cloud(n, d, st.next_u64())
        S = oracle.sample_jl(5, d, st.next_u64())
        emb = cloud @ S.T
        mx, mean, ev, zp = oracle.naive_distortion(cloud, emb)
        r = adg.evaluate(cloud, emb, engine=engine)
        assert r.n_pairs_evaluated == ev
        if engine == "exact":
            assert abs(r.max_distortion - mx) <= 1e-12
            assert abs(r.mean_distortion - mean) <= 1e-12
        else:
            assert abs(r.max_distortion - mx) <= 1e-12  # refined exactly
            assert abs(r.mean_distortion - mean) <= 1e-6
    del rng_i, draws


@pytest.mark.parametrize("engine", ENGINES)
def test_duplicates_skipped(engine, oracle):
    # proj/tests/test_distortion.cpp:185-195
    c = oracle.gaussian_cloud(10, 3, 8)
    c[4] = c[2]
    c[7] = c[2]
    r = adg.evaluate(c, c[:, :2].copy(), engine=engine)
    assert r.n_zero_distance_pairs == 3
    assert r.n_pairs_evaluated == 45 - 3
    ref = oracle.evaluate(c, c[:, :2].copy())
    assert abs(r.max_distortion - ref.max_distortion) <= 1e-12
    assert r.argmax == ref.argmax


def test_histogram_edges_exact_engine():
    # proj/tests/test_distortion.cpp:197-212
    o = np.array([[0.0], [1.0], [10.0]])
    e = np.array([[0.0], [2.0], [8.5]])
    r = adg.evaluate(o, e, hist_bins=10, hist_max=1.0, engine="exact")
    assert r.histogram[-1] == 1 and r.histogram[1] == 1 and r.histogram[2] == 1


def test_evaluate_validation(oracle):
    # proj/tests/test_distortion.cpp:214-222
    a = oracle.gaussian_cloud(10, 3, 1)
    b = oracle.gaussian_cloud(11, 3, 1)
    with pytest.raises(ValueError, match="cloud sizes differ"):
        adg.evaluate(a, b)
    with pytest.raises(ValueError):
        adg.evaluate(a, a, adg.PairSampling.sample(46, 0))
    with pytest.raises(ValueError):
        adg.evaluate(a, a, adg.PairSampling.sample(0, 0))
    with pytest.raises(ValueError):
        adg.evaluate(a, a, hist_bins=0)
    with pytest.raises(ValueError):
        adg.evaluate(a, a, hist_bins=10, hist_max=0.0)


def test_sampling_all_equals_all(oracle):
    # proj/tests/test_distortion.cpp:152-169
    c = oracle.gaussian_cloud(40, 6, 6)
    emb = c @ oracle.sample_jl(3, 6, 4).T
    a = adg.evaluate(c, emb)
    s = adg.evaluate(c, emb, adg.PairSampling.sample(40 * 39 // 2, 123))
    assert s.sampled and s.sample_seed == 123
    assert s.max_distortion == a.max_distortion
    assert np.array_equal(s.histogram, a.histogram)
    assert s.n_pairs_evaluated == a.n_pairs_evaluated
    assert abs(s.mean_distortion - a.mean_distortion) <= 1e-15


def test_sampled_matches_oracle(oracle):
    c = oracle.gaussian_cloud(50, 5, 7)
    emb = c @ oracle.sample_jl(2, 5, 1).T
    r = adg.evaluate(c, emb, adg.PairSampling.sample(200, 9))
    ref = oracle.evaluate(c, emb, all_pairs=False, m=200, sample_seed=9)
    assert r.n_pairs_evaluated == 200
    assert abs(r.max_distortion - ref.max_distortion) <= 1e-13
    assert abs(r.mean_distortion - ref.mean_distortion) <= 1e-13
    assert np.array_equal(r.histogram, ref.histogram)
    assert r.argmax == ref.argmax


# -------------------------------------------- screen engine vs the oracle
@pytest.mark.parametrize("n,d,k,seed", [(300, 20, 5, 11), (129, 7, 3, 12), (1000, 64, 9, 13),
                                        (2, 3, 1, 14), (257, 130, 70, 15)])
def test_screen_random_shapes(n, d, k, seed, oracle):
    c = oracle.gaussian_cloud(n, d, seed)
    emb = c @ oracle.sample_jl(k, d, seed + 1).T
    ref = oracle.evaluate(c, emb, hist_bins=50, edge_band=EDGE_BAND)
    r = adg.evaluate(c, emb, engine="screen")
    assert r.engine == "screen"
    check_report(r, ref, ref.edge_near)


def _minimum_slice(name, oracle, hist_bins):
    """the oracle's own fp64 embedding rounded to fp32, with the
    fp32 original -- isolates evaluator parity from embedding parity."""
    X = ds.make(name)
    n, d, r, _, _ = ds.CONFIGS[name]
    mean, P, S = oracle.fit(X.astype(np.float64), r, "exact", 0)
    Y = oracle.transform_all(mean, P, S, X.astype(np.float64)).astype(np.float32)
    ref = oracle.evaluate(X.astype(np.float64), Y.astype(np.float64), hist_bins=hist_bins,
                          edge_band=EDGE_BAND)
    return X, Y, ref


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_screen_minimum_slice(name, oracle):
    bins = ds.CONFIGS[name][3]
    X, Y, ref = _minimum_slice(name, oracle, bins)
    r = adg.evaluate(X, Y, hist_bins=bins, engine="screen")
    check_report(r, ref, ref.edge_near)
    r2 = adg.evaluate(X, Y, hist_bins=bins, engine="exact")
    check_report(r2, ref, exact_hist=True, mean_tol=1e-12)


# ------------------------------------------------------ fit / transform
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_fit_transform_parity(name, oracle):
    X = ds.make(name)
    n, d, r, _, _ = ds.CONFIGS[name]
    mean, P, S = oracle.fit(X.astype(np.float64), r, "exact", 0)
    Yref = oracle.transform_all(mean, P, S, X.astype(np.float64))
    model = adg.fit(X, r, adg.SpectralBackend.exact, 0)
    assert np.array_equal(model.sketch.entries, S)
    assert np.max(np.abs(model.mean - mean)) <= 1e-12 * max(1.0, np.max(np.abs(mean)))
    Y = adg.transform_all(model, X).data
    assert rel_fro(Y, Yref) <= EMBED_TOL


def test_exact_tiled_matches_block_and_oracle(oracle, monkeypatch):
    """EXACT above n = 4096 runs the tiled kernel (adg_exact_tiled.cu): the
    block engine's per-pair arithmetic, so the counts, histogram, max and argmax
    are the block engine's bit for bit and the oracle's; the mean is summed in
    tile order (within 1e-14 relative)."""
    import torch
    c = oracle.gaussian_cloud(5003, 40, 17).astype(np.float32)
    c[4000] = c[7]  # a zero pair across tiles
    c[12] = c[7]
    e = (c.astype(np.float64) @ oracle.sample_jl(9, 40, 3).T).astype(np.float32)
    X, Y = torch.from_numpy(c).cuda(), torch.from_numpy(e).cuda()
    tiled = adg.evaluate(X, Y, hist_bins=60, hist_max=0.9, engine="exact")
    monkeypatch.setenv("ADG_EXACT_BLOCK", "1")
    block = adg.evaluate(X, Y, hist_bins=60, hist_max=0.9, engine="exact")
    ref = oracle.evaluate(c.astype(np.float64), e.astype(np.float64), hist_bins=60, hist_max=0.9)
    for r in (tiled, block):
        assert r.n_pairs_evaluated == ref.n_pairs_evaluated
        assert r.n_zero_distance_pairs == ref.n_zero_distance_pairs == 3
        assert np.array_equal(np.asarray(r.histogram, np.int64), np.asarray(ref.histogram, np.int64))
        assert r.argmax == ref.argmax and abs(r.max_distortion - ref.max_distortion) <= 1e-15
        assert abs(r.mean_distortion - ref.mean_distortion) <= 1e-14 * ref.mean_distortion
    assert tiled.max_distortion == block.max_distortion and tiled.argmax == block.argmax
    assert np.array_equal(tiled.histogram, block.histogram)


@pytest.mark.gpu
def test_screen_multicast_variant_bit_identical(monkeypatch):
    """ADG_SCREEN_MC=1 (4-CTA clusters sharing A by multicast, an experiment
    kept off by default) gives the 2-CTA kernel's report bit for bit."""
    import torch
    g = torch.Generator().manual_seed(11)
    for n, d, r, dt in ((6001, 200, 24, torch.float32), (5000, 128, 16, torch.bfloat16)):
        X = torch.randn(n, d, generator=g).to(dt).cuda()
        Y = (X.float() @ (torch.randn(d, r, generator=g).cuda() / d ** 0.5)).contiguous()
        reps = []
        for mc in ("0", "1"):
            monkeypatch.setenv("ADG_SCREEN_MC", mc)
            rep = adg.evaluate(X, Y, hist_bins=40, engine="screen")
            reps.append((rep.max_distortion, rep.mean_distortion, rep.argmax, tuple(int(h) for h in rep.histogram),
                         rep.n_pairs_evaluated, rep.n_zero_distance_pairs))
        assert reps[0] == reps[1]


@pytest.mark.parametrize("bins", [300, 3000, 70000])
def test_screen_histogram_modes_many_bins(bins):
    """Bin counts past the per-thread u8 counters select the other histogram
    modes of the screen (per-warp match counters, shared atomics, per-CTA
    global scratch): SCREEN_EXACT_HIST equals the EXACT engine's histogram
    bin for bin, and SCREEN's counts, max and argmax equal it
    (distortion.cpp:77-88, :113-192)."""
    import torch
    g = torch.Generator().manual_seed(bins)
    n, d, r = 5000, 48, 12
    X = torch.randn(n, d, generator=g, dtype=torch.float64)
    Y = X @ (torch.randn(d, r, generator=g, dtype=torch.float64) / d ** 0.5)
    X, Y = X.float().cuda(), Y.float().cuda()
    ex = adg.evaluate(X, Y, hist_bins=bins, hist_max=1.5, engine="exact")
    eh = adg.evaluate(X, Y, hist_bins=bins, hist_max=1.5, engine="screen_exact_hist")
    sc = adg.evaluate(X, Y, hist_bins=bins, hist_max=1.5, engine="screen")
    assert np.array_equal(np.asarray(eh.histogram), np.asarray(ex.histogram))
    for rep in (eh, sc):
        assert abs(rep.max_distortion - ex.max_distortion) <= 1e-13 and rep.argmax == ex.argmax
        assert (rep.n_pairs_evaluated, rep.n_zero_distance_pairs) == (ex.n_pairs_evaluated, ex.n_zero_distance_pairs)
        assert int(np.asarray(rep.histogram).sum()) == int(np.asarray(ex.histogram).sum())
        assert abs(rep.mean_distortion - ex.mean_distortion) <= 1e-4 * abs(ex.mean_distortion)


@pytest.mark.parametrize("n,d,r", [(4097, 128, 64), (5120, 64, 16), (5376, 200, 65), (6401, 784, 50)])
def test_screen_tile_boundaries_match_exact(n, d, r):
    """n on and just past the 256-row / 160-column tile grid, d a multiple of
    the 64-wide K chunk (no tail) or not, r filling one embedding chunk or
    spilling into a second: SCREEN_EXACT_HIST equals the EXACT engine bin for
    bin, and both screen modes reproduce its counts, max and argmax."""
    import torch
    g = torch.Generator().manual_seed(n)
    X = torch.rand(n, d, generator=g, dtype=torch.float64)
    Y = X @ (torch.randn(d, r, generator=g, dtype=torch.float64) / d ** 0.5)
    X, Y = X.float().cuda(), Y.float().cuda()
    ex = adg.evaluate(X, Y, hist_bins=50, engine="exact")
    for eng in ("screen_exact_hist", "screen"):
        rep = adg.evaluate(X, Y, hist_bins=50, engine=eng)
        # both maxima are fp64 direct differences, summed in different orders
        assert abs(rep.max_distortion - ex.max_distortion) <= 1e-13 and rep.argmax == ex.argmax
        assert (rep.n_pairs_evaluated, rep.n_zero_distance_pairs) == (ex.n_pairs_evaluated, ex.n_zero_distance_pairs)
        if eng == "screen_exact_hist":
            assert np.array_equal(np.asarray(rep.histogram), np.asarray(ex.histogram))
        assert abs(rep.mean_distortion - ex.mean_distortion) <= 1e-4 * abs(ex.mean_distortion)

"""GPU parity at BASELINE scale, the sharded (multi-GPU) protocol emulated on
one GPU, and size-independent properties for the configs too large for the
CPU oracle."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
from paper_1609_05388_b200 import dist

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SCREEN_MEAN_RTOL = 1e-4


def check_edges(h, hr, edge_near):
    h, hr, en = (np.asarray(a, np.int64) for a in (h, hr, edge_near))
    slack = np.zeros_like(hr)
    slack[:-1] += en
    slack[1:] += en
    assert np.all(np.abs(h - hr) <= slack), (h - hr, slack)


@pytest.fixture(scope="module")
def c3():
    fx = json.load(open(os.path.join(GOLDEN, "c3_fixture.json")))
    X = ds.c3_mnist_like()
    assert hashlib.sha256(X.tobytes()).hexdigest() == fx["x_sha256"], "C3 generator drifted"
    return X, fx


@pytest.fixture(scope="module")
def c3_xy(c3, oracle):
    """The oracle's C3 embedding (from the committed oracle model), fp32, on the GPU."""
    import torch
    X, fx = c3
    z = np.load(os.path.join(GOLDEN, "c3_fixture.npz"))
    S = oracle.sample_jl(25, 784, oracle.derive_seed(0, "jl"))
    Y = oracle.transform_all(z["mean"], z["P"], S, X.astype(np.float64)).astype(np.float32)
    assert hashlib.sha256(Y.tobytes()).hexdigest() == fx["y32_sha256"]
    return torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), fx


def _c3_common(rep, fx):
    assert rep.n_pairs_evaluated == fx["n_pairs_evaluated"]
    assert rep.n_zero_distance_pairs == fx["n_zero_distance_pairs"]
    assert abs(rep.max_distortion - fx["max_distortion"]) <= 1e-12
    assert list(rep.argmax) == fx["argmax"]
    # the mean is the screen's (tensor-core fp32 accumulation leaves a ~3.5e-5
    # relative bias at d=784); max/argmax/counts above are exact
    assert abs(rep.mean_distortion - fx["mean_distortion"]) <= SCREEN_MEAN_RTOL * fx["mean_distortion"]


def test_c3_evaluator_parity(c3_xy):
    """SURVEY 7.2 minimum slice at full C3 scale, SCREEN engine: a pair can
    only leave its exact bin across an edge its exact value lies within the
    screen's rigorous per-pair error bound of, so every bin differs from the
    reference's by at most the pairs in those bands (fixture band_rigorous,
    from oracle.edge_band_counts).  The net number of pairs moved is printed
    (profiles/r02_edge_band.md: 4449 of 1.8e9)."""
    X, Y, fx = c3_xy
    rep = adg.evaluate(X, Y, hist_bins=50, engine="screen")
    _c3_common(rep, fx)
    assert rep.edge_pairs == 0
    check_edges(rep.histogram, fx["histogram"], fx["band_rigorous"])
    dh = np.asarray(rep.histogram, np.int64) - np.asarray(fx["histogram"], np.int64)
    assert dh.sum() == 0
    print(f"C3 SCREEN histogram: {np.abs(dh).sum() // 2} pairs moved net "
          f"(rigorous band holds {sum(fx['band_rigorous'])})")
    assert np.abs(dh).sum() // 2 <= 2e-5 * fx["n_pairs_evaluated"]


def test_c3_exact_histogram(c3_xy):
    """SCREEN_EXACT_HIST: the pairs whose screened value lies within 1/4 of
    the rigorous bound of an edge are binned by their exact fp64 value -- the
    C3 histogram is the reference's bin for bin."""
    X, Y, fx = c3_xy
    rep = adg.evaluate(X, Y, hist_bins=50, engine="screen_exact_hist")
    _c3_common(rep, fx)
    assert rep.engine == "screen_exact_hist"
    assert rep.edge_pairs >= sum(fx["band_quarter"]) // 2  # every edge pair of the band, at least
    assert np.array_equal(np.asarray(rep.histogram, np.int64), np.asarray(fx["histogram"], np.int64))


def test_c3_fit_embedding_parity(c3, oracle):
    import torch
    X, _ = c3
    z = np.load(os.path.join(GOLDEN, "c3_fixture.npz"))
    S = oracle.sample_jl(25, 784, oracle.derive_seed(0, "jl"))
    Yref = oracle.transform_all(z["mean"], z["P"], S, X.astype(np.float64))
    m = adg.fit(torch.from_numpy(X).cuda(), 50, adg.SpectralBackend.exact, 0)
    assert np.array_equal(m.sketch.entries.cpu().numpy(), S)
    Y = adg.transform_all(m, torch.from_numpy(X).cuda()).data.double().cpu().numpy()
    err = np.linalg.norm(Y - Yref) / np.linalg.norm(Yref)
    assert err <= 1e-4, err


def _emulated_ranks(X, Y, world, bins=50, engine="screen"):
    """The sharded protocol with `world` ranks on one GPU (tests/local_comm.py:
    one thread, context and plan per rank; the library's own exchange over
    in-process collectives); every rank's report is identical -> rank 0's."""
    from tests.local_comm import assert_same_report, sharded_reports
    reps = sharded_reports(X, Y, world, bins, engine=engine)
    for r in reps[1:]:
        assert_same_report(r, reps[0])
    return reps[0]


def test_near_list_exchange_overflow_redo_bit_identical(oracle):
    """Near-coincident lists over the plan's capacity (ADG_NEAR_CAP, a testing
    aid) on a rank: every rank's finalize redoes the histogram and the near
    list in tile chunks; the report is bit-identical to the one without
    overflow (and the reference's max / zero count)."""
    import torch
    c = oracle.gaussian_cloud(1500, 24, 8).astype(np.float32)
    c[10], c[700], c[1400] = c[3], c[3], c[3]  # 6 coincident pairs over several tiles
    e = (c.astype(np.float64) @ oracle.sample_jl(6, 24, 1).T).astype(np.float32)
    X, Y = torch.from_numpy(c).cuda(), torch.from_numpy(e).cuda()
    ok = _emulated_ranks(X, Y, 2)
    os.environ["ADG_NEAR_CAP"] = "4"
    try:
        over = _emulated_ranks(X, Y, 2)
        over1 = adg.evaluate(X, Y, hist_bins=50, engine="screen")
    finally:
        del os.environ["ADG_NEAR_CAP"]
    from tests.local_comm import assert_same_report
    assert_same_report(over1, ok)
    ref = oracle.evaluate(c.astype(np.float64), e.astype(np.float64), hist_bins=50)
    assert ok.engine == "screen" and over.engine == "screen"
    for r in (ok, over):
        assert r.n_zero_distance_pairs == ref.n_zero_distance_pairs == 6
        assert abs(r.max_distortion - ref.max_distortion) <= 1e-12 and r.argmax == ref.argmax
    assert np.array_equal(over.histogram, ok.histogram)
    assert over.mean_distortion == ok.mean_distortion and over.max_distortion == ok.max_distortion


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_protocol_bit_identical(world, oracle):
    import torch
    c = oracle.gaussian_cloud(3000, 96, 31).astype(np.float32)
    c[2999] = c[5]       # a duplicate pair across distant tiles
    c[1500] = c[1]
    S = oracle.sample_jl(12, 96, 2)
    e = (c.astype(np.float64) @ S.T).astype(np.float32)
    X, Y = torch.from_numpy(c).cuda(), torch.from_numpy(e).cuda()
    one = adg.evaluate(X, Y, hist_bins=50, engine="screen")
    many = _emulated_ranks(X, Y, world)
    assert many.max_distortion == one.max_distortion and many.argmax == one.argmax
    assert many.mean_distortion == one.mean_distortion            # bitwise
    assert np.array_equal(many.histogram, one.histogram)
    assert many.n_zero_distance_pairs == one.n_zero_distance_pairs == 2
    ref = oracle.evaluate(c.astype(np.float64), e.astype(np.float64), hist_bins=50)
    assert one.n_zero_distance_pairs == ref.n_zero_distance_pairs
    assert abs(one.max_distortion - ref.max_distortion) <= 1e-12 and one.argmax == ref.argmax


def test_screen_vs_exact_engine_midsize(oracle):
    """n = 6000 (18M pairs): SCREEN against the GPU EXACT engine (itself pinned to
    the oracle), with an embedding of mixed quality so values spread over bins."""
    import torch
    rng = np.random.default_rng(5)
    c = (rng.standard_normal((6000, 200)) * np.linspace(2, 0.1, 200)).astype(np.float32)
    m = adg.fit(c, 30, adg.SpectralBackend.exact, 3)
    Y = adg.transform_all(m, c).data
    X = torch.from_numpy(c).cuda()
    Yd = torch.from_numpy(Y).cuda()
    s = adg.evaluate(X, Yd, hist_bins=40, engine="screen")
    e = adg.evaluate(X, Yd, hist_bins=40, engine="exact")
    assert s.n_pairs_evaluated == e.n_pairs_evaluated
    assert abs(s.max_distortion - e.max_distortion) <= 1e-13 and s.argmax == e.argmax
    assert abs(s.mean_distortion - e.mean_distortion) <= 1e-6 * e.mean_distortion
    diff = np.abs(s.histogram.astype(np.int64) - e.histogram.astype(np.int64))
    assert diff.sum() <= 2e-5 * e.n_pairs_evaluated


def test_bf16_input_c5_like(oracle):
    """C5 dtype path (bf16-stored data, fp32-accumulated): 4000 points of the
    C5 mixture generator, screen vs the oracle on the exact bf16 values."""
    import torch
    X = ds.c5_mixture(n=4000, d=1024, comps=64, sub=64)
    m = adg.fit(X, 64, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(m, X).data
    r = adg.evaluate(X, Y, hist_bins=50, engine="screen")
    Xh = X.float().cpu().numpy().astype(np.float64)
    Yh = Y.double().cpu().numpy()
    ref = oracle.evaluate(Xh, Yh, hist_bins=50, edge_band=1e-4)
    assert r.n_pairs_evaluated == ref.n_pairs_evaluated
    assert abs(r.max_distortion - ref.max_distortion) <= 1e-5 and r.argmax == ref.argmax
    check_edges(r.histogram, ref.histogram, ref.edge_near)
    # fit on bf16 data vs the fp64 LAPACK stand-in on the same (exactly widened) values
    mean, P, S = oracle.fit(Xh, 64, "exact", 0)
    Yref = oracle.transform_all(mean, P, S, Xh)
    assert np.linalg.norm(Yh - Yref) / np.linalg.norm(Yref) <= 1e-4


def test_sampled_mode_large_n(oracle):
    """CLI default above n = 5000 is sample:2000000 (adagio_main.cpp:215-219):
    identical Floyd indices and exact values vs the oracle."""
    X = ds.c3_mnist_like(n=20000, seed=9)
    m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(m, X).data
    seed = adg.derive_seed(0, "sampling")
    r = adg.evaluate(X, Y, adg.PairSampling.sample(200000, seed), hist_bins=50)
    ref = oracle.evaluate(X.astype(np.float64), Y.astype(np.float64), all_pairs=False, m=200000,
                          sample_seed=seed, hist_bins=50)
    assert r.sampled and r.sample_seed == seed
    assert np.array_equal(r.histogram, ref.histogram)
    assert abs(r.max_distortion - ref.max_distortion) <= 1e-13 and r.argmax == ref.argmax
    assert abs(r.mean_distortion - ref.mean_distortion) <= 1e-13


def test_repeat_determinism(oracle):
    import torch
    X = torch.from_numpy(ds.c1_low_rank()).cuda()
    m1 = adg.fit(X, 30, adg.SpectralBackend.exact, 0)
    m2 = adg.fit(X, 30, adg.SpectralBackend.exact, 0)
    assert torch.equal(m1.basis.rows, m2.basis.rows) and torch.equal(m1.mean, m2.mean)
    Y = adg.transform_all(m1, X).data
    a = adg.evaluate(X, Y, hist_bins=100, engine="screen")
    b = adg.evaluate(X, Y, hist_bins=100, engine="screen")
    assert a.mean_distortion == b.mean_distortion and np.array_equal(a.histogram, b.histogram)
    assert a.max_distortion == b.max_distortion and a.argmax == b.argmax


def _emulated_sharded_fit(Xd, world, target_dim, backend, seed):
    """dist.fit_sharded's exchange on one GPU: per-shard column sums and Grams
    through the C ABI, summed in rank order (what an all-reduce delivers),
    then the solve on the total."""
    import torch
    n = Xd.shape[0]
    s, k = target_dim // 2, target_dim - target_dim // 2
    sums, grams = [], []
    shards = [Xd[slice(*dist.shard_rows(n, world, r))] for r in range(world)]
    for Xl in shards:
        x = adg.api._matrix(Xl)
        ctx, dev = adg.api._ctx_for(x)
        sums.append(dist._colsum_dev(x, ctx, dev))
    total = sums[0].clone()
    for t in sums[1:]:
        total += t
    mean = total / torch.full_like(total, float(n))
    for Xl in shards:
        x = adg.api._matrix(Xl)
        ctx, dev = adg.api._ctx_for(x)
        grams.append(dist._gram_dev(x, ctx, dev, mean, backend))
    G = grams[0].clone()
    for g in grams[1:]:
        G += g
    x = adg.api._matrix(Xd)
    ctx, dev = adg.api._ctx_for(x)
    basis, sketch = dist._solve_dev(G, n, s, k, backend, seed, ctx, dev)
    return mean, basis, sketch


@pytest.mark.parametrize("backend", [adg.SpectralBackend.exact, adg.SpectralBackend.randomized])
def test_sharded_fit_matches_fit(backend, oracle):
    """row-sharded column sums + Gram all-reduce + replicated
    solve.  One shard is adg_fit bit for bit; more shards only reorder the
    fp64 sums, so the model agrees to rounding; both match the oracle."""
    import torch
    X = oracle.low_rank_cloud(5000, 300, 12, 4).astype(np.float32) + 0.5
    Xd = torch.from_numpy(X).cuda()
    ref = adg.fit(Xd, 20, backend, 9)
    m1, b1, s1 = _emulated_sharded_fit(Xd, 1, 20, backend, 9)
    assert torch.equal(m1, ref.mean) and torch.equal(b1, ref.basis.rows)
    assert torch.equal(s1, ref.sketch.entries)
    # the public wrapper at world size 1 (no process group) is the same call chain
    mw = dist.fit_sharded(Xd, Xd.shape[0], 20, backend, 9)
    assert torch.equal(mw.basis.rows, ref.basis.rows) and torch.equal(mw.mean, ref.mean)
    mean_o, P_o, S_o = oracle.fit(X.astype(np.float64), 20, backend.name, 9)
    for world in (2, 3, 8):
        m, b, s = _emulated_sharded_fit(Xd, world, 20, backend, 9)
        np.testing.assert_allclose(m.cpu().numpy(), ref.mean.cpu().numpy(), rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(b.cpu().numpy(), ref.basis.rows.cpu().numpy(), atol=1e-9)
        np.testing.assert_allclose(b.cpu().numpy(), P_o, atol=1e-8)
        assert np.array_equal(s.cpu().numpy(), S_o)


def test_sharded_fit_errors_and_empty_shard(oracle):
    import torch
    L = adg._lib.load()
    X = oracle.gaussian_cloud(64, 16, 2).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    # an empty shard contributes zeros
    x = adg.api._matrix(Xd[:0])
    ctx, dev = adg.api._ctx_for(adg.api._matrix(Xd))
    z = torch.ones(16, dtype=torch.float64, device="cuda")
    adg._lib.check(L.adg_column_sums(ctx, Xd.data_ptr(), x.code, 0, 16, z.data_ptr()))
    assert torch.count_nonzero(z) == 0
    # a non-finite shard: the backend's NumericError text (spectral.cpp:29-33)
    Xb = Xd.clone()
    Xb[5, 3] = float("nan")
    mean = torch.zeros(16, dtype=torch.float64, device="cuda")
    with pytest.raises(adg._lib.NumericError, match="exact_top_svd: input contains non-finite"):
        dist._gram_dev(adg.api._matrix(Xb), ctx, dev, mean, adg.SpectralBackend.exact)
    with pytest.raises(adg._lib.NumericError, match="randomized_top_svd: input contains non-finite"):
        dist._gram_dev(adg.api._matrix(Xb), ctx, dev, mean, adg.SpectralBackend.randomized)
    G = torch.eye(16, dtype=torch.float64, device="cuda")
    with pytest.raises(adg._lib.InvalidArgument, match="need at least 2 points"):
        dist._solve_dev(G, 1, 4, 4, adg.SpectralBackend.exact, 0, ctx, dev)
    with pytest.raises(adg._lib.InvalidArgument, match="k must be >= 1"):
        dist._solve_dev(G, 64, 4, 0, adg.SpectralBackend.exact, 0, ctx, dev)
    with pytest.raises(adg._lib.InvalidArgument, match="fit: target_dim"):
        dist.fit_sharded(Xd, 64, 17)


@pytest.mark.parametrize("kind", ["bf16_centred", "bf16_offset", "f32"])
def test_exact_fp16_planes_one_pass(kind, oracle, monkeypatch):
    """Nearly centred bf16 rows are left uncentred, so every original value is
    exactly its fp16 hi plane and the screen runs the original K chunks in one
    MMA pass (hi.lo and lo.hi are exact zeros); offset bf16 data keeps the
    centring (three passes), as does fp32.  Every report must equal the
    forced three-pass kernel's (ADG_SCREEN_ORIG3) and the oracle's."""
    import torch
    X = ds.c5_mixture(n=3000, d=512, comps=32, sub=32)
    if kind == "bf16_offset":
        X = (X.float() + 12.0).to(torch.bfloat16)
    elif kind == "f32":
        X = X.float()
    m = adg.fit(X, 24, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(m, X).data
    one = adg.evaluate(X, Y, hist_bins=50, engine="screen")
    assert adg.api.last_screen_orig_passes(0) == (1 if kind == "bf16_centred" else 3)
    monkeypatch.setenv("ADG_SCREEN_ORIG3", "1")
    three = adg.evaluate(X, Y, hist_bins=50, engine="screen")
    assert adg.api.last_screen_orig_passes(0) == 3
    monkeypatch.delenv("ADG_SCREEN_ORIG3")
    assert one.max_distortion == three.max_distortion and one.argmax == three.argmax
    assert np.array_equal(one.histogram, three.histogram)
    assert one.mean_distortion == three.mean_distortion
    Xh = X.float().cpu().numpy().astype(np.float64)
    ref = oracle.evaluate(Xh, Y.double().cpu().numpy(), hist_bins=50, edge_band=1e-4)
    assert one.n_pairs_evaluated == ref.n_pairs_evaluated
    assert abs(one.max_distortion - ref.max_distortion) <= 1e-12 and one.argmax == ref.argmax
    check_edges(one.histogram, ref.histogram, ref.edge_near)


def test_plan_reuse_refreshes_contents(oracle, monkeypatch):
    """Repeated evaluations over the same device buffers reuse the context's
    plan (and the sharded evaluator's) but re-read the data: a rewrite in
    place must give exactly the report of a fresh plan."""
    import torch
    c = oracle.gaussian_cloud(6000, 40, 3).astype(np.float32)
    S = oracle.sample_jl(8, 40, 1)
    X = torch.from_numpy(c).cuda()
    Y = torch.from_numpy((c.astype(np.float64) @ S.T).astype(np.float32)).cuda()
    ev = dist.ShardedEvaluator()
    a = adg.evaluate(X, Y, hist_bins=30, engine="screen")
    b = adg.evaluate(X, Y, hist_bins=30, engine="screen")
    sa = ev.evaluate(X, Y, hist_bins=30)
    for r in (b, sa):
        assert r.max_distortion == a.max_distortion and r.argmax == a.argmax
        assert r.mean_distortion == a.mean_distortion and np.array_equal(r.histogram, a.histogram)
    # rewrite both clouds in place (new contents, same addresses and shapes)
    c2 = oracle.gaussian_cloud(6000, 40, 4).astype(np.float32)
    X.copy_(torch.from_numpy(c2))
    Y.copy_(torch.from_numpy((c2.astype(np.float64) @ S.T).astype(np.float32)))
    got = adg.evaluate(X, Y, hist_bins=30, engine="screen")
    sgot = ev.evaluate(X, Y, hist_bins=30)
    monkeypatch.setenv("ADG_NO_PLAN_CACHE", "1")
    fresh = adg.evaluate(X.clone(), Y.clone(), hist_bins=30, engine="screen")
    for r in (got, sgot):
        assert r.max_distortion == fresh.max_distortion and r.argmax == fresh.argmax
        assert r.mean_distortion == fresh.mean_distortion
        assert np.array_equal(r.histogram, fresh.histogram)
    assert got.max_distortion != a.max_distortion
    ref = oracle.evaluate(c2.astype(np.float64), Y.double().cpu().numpy(), hist_bins=30)
    assert abs(got.max_distortion - ref.max_distortion) <= 1e-12 and got.argmax == ref.argmax
    ev.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,dtype", [(1000, 130, torch.float32), (77, 257, torch.float64),
                                       (3001, 300, torch.bfloat16), (5, 128, torch.float32)])
def test_centred_gram_fp64_tensor_cores(n, d, dtype):
    """adg_gram (DMMA tiles, split rows, ragged d and n) against the fp64
    centred Gram Xc^T Xc of the same (widened) values."""
    g = torch.Generator().manual_seed(n + d)
    Xh = (torch.rand((n, d), generator=g, dtype=torch.float64) * 2 - 1).to(dtype)
    Xd = Xh.cuda()
    x = adg.api._matrix(Xd)
    ctx, dev = adg.api._ctx_for(x)
    Xw = Xh.double()
    mean = Xw.mean(dim=0)
    G = dist._gram_dev(x, ctx, dev, mean.to(dev), adg.SpectralBackend.exact).cpu()
    c = Xw - mean
    ref = c.T @ c
    err = (G - ref).abs().max().item() / ref.abs().max().item()
    assert err <= 1e-13, err
    assert torch.equal(G, G.T)

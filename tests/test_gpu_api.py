"""The reference's own unit tests, restated against the CUDA path (C ABI).

proj/tests/test_embed.cpp, test_spectral.cpp, test_jl.cpp, test_dataset.cpp
(center) and acceptance.cpp #1 / #2 / #9, with the reference's tolerances.
Clouds come from the reference's SeededRng generators (oracle.gaussian_cloud
/ low_rank_cloud), so the inputs are the reference tests' own inputs.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_1609_05388_b200 as adg
from tests.rng_emul import Stream

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXACT = adg.SpectralBackend.exact
RAND = adg.SpectralBackend.randomized


def complement_rows(P):
    _, _, vt = np.linalg.svd(P, full_matrices=True)
    return vt[P.shape[0]:]


# ----------------------------------------------------------------- embed
def test_fit_split(oracle):
    c = oracle.gaussian_cloud(30, 25, 1)
    m = adg.fit(c, 20, EXACT, 0)
    assert (m.s(), m.k(), m.target_dim()) == (10, 10, 20)
    m = adg.fit(c, 5, EXACT, 0)
    assert (m.s(), m.k()) == (2, 3)


def test_fit_validation(oracle):
    c = oracle.gaussian_cloud(10, 6, 2)
    with pytest.raises(ValueError, match="target_dim"):
        adg.fit(c, 1, EXACT, 0)
    with pytest.raises(ValueError):
        adg.fit(c, 7, EXACT, 0)
    with pytest.raises(ValueError, match="k must be >= 1"):
        adg.fit_with_split(c, 2, 0, EXACT, 0)


def test_mean_to_zero_and_in_span(oracle):
    c = oracle.gaussian_cloud(40, 12, 3)
    m = adg.fit(c, 8, EXACT, 5)
    assert np.max(np.abs(adg.transform(m, m.mean))) <= 1e-12
    img = adg.transform(m, m.mean + 2.5 * m.basis.rows[1])
    assert np.max(np.abs(img[m.s():])) <= 1e-9


def test_transform_hand_example():
    m = adg.AdagioModel(np.zeros(3), adg.OrthonormalBasis(np.array([[1.0, 0, 0]])),
                        adg.JlMatrix(np.array([[1.0, 1, 1]])))
    img = adg.transform(m, np.array([1.0, 2, 3]))
    assert img.shape == (2,) and abs(img[0] - 1) <= 1e-15 and abs(img[1] - 5) <= 1e-15


def test_linearity(oracle):
    c = oracle.gaussian_cloud(25, 10, 4)
    m = adg.fit(c, 6, EXACT, 1)
    s = Stream(11)
    u = np.zeros(10)
    v = np.zeros(10)
    for i in range(10):
        u[i] = s.normal()
        v[i] = s.normal()
    g = lambda x: adg.transform(m, m.mean + x)  # noqa: E731
    assert np.max(np.abs(g(2 * u - 3 * v) - (2 * g(u) - 3 * g(v)))) <= 1e-9


def test_transform_all_matches_transform(oracle):
    c = oracle.gaussian_cloud(37, 14, 6)
    m = adg.fit(c, 9, EXACT, 2)
    e = adg.transform_all(m, c).data
    assert e.shape == (37, 9)
    for i in range(37):
        assert np.array_equal(e[i], adg.transform(m, c[i]))
    with pytest.raises(ValueError):
        adg.transform_all(m, oracle.gaussian_cloud(5, 13, 0))


def test_pythagoras(oracle):
    c = oracle.gaussian_cloud(30, 20, 8)
    m = adg.fit(c, 10, EXACT, 3)
    e = adg.transform_all(m, c).data
    P, S = m.basis.rows, m.sketch.entries
    for i in range(30):
        for j in range(i + 1, 30):
            diff = c[i] - c[j]
            pr = P @ diff
            res = diff - P.T @ pr
            lhs = np.sum((e[i] - e[j]) ** 2)
            assert abs(lhs - (pr @ pr + np.sum((S @ res) ** 2))) <= 1e-9
            assert np.sqrt(lhs) >= np.linalg.norm(pr) - 1e-12


def test_complement_isometry_and_full_basis(oracle):
    c = oracle.gaussian_cloud(50, 30, 9)
    m = adg.fit(c, 10, EXACT, 4)
    m.sketch.entries = complement_rows(m.basis.rows)
    e = adg.transform_all(m, c).data
    assert adg.max_distortion(c, e) <= 1e-9
    c = oracle.gaussian_cloud(30, 10, 10)
    m = adg.fit_with_split(c, 10, 4, EXACT, 0)
    assert adg.max_distortion(c, adg.transform_all(m, c).data) <= 1e-9


def test_pure_jl(oracle):
    c = oracle.gaussian_cloud(20, 15, 11)
    m = adg.fit_with_split(c, 0, 40, EXACT, 7)
    assert m.s() == 0
    cen, _ = oracle.center(c)
    exp = cen @ m.sketch.entries.T
    assert np.max(np.abs(adg.transform_all(m, c).data - exp)) <= 1e-12


def test_randomized_backend_usable(oracle):
    cen, _ = oracle.center(oracle.low_rank_cloud(60, 30, 3, 13))
    m = adg.fit(cen, 8, RAND, 21)
    assert m.backend == RAND
    e = adg.transform_all(m, cen).data
    assert e.shape[1] == 8 and adg.max_distortion(cen, e) <= 1e-6


def test_model_roundtrip_and_determinism(oracle, tmp_path):
    c = oracle.gaussian_cloud(20, 9, 14)
    m = adg.fit(c, 6, RAND, 17)
    p = str(tmp_path / "model.adg")
    adg.save_model(m, p)
    l = adg.load_model(p)
    assert l.seed == m.seed and l.backend == m.backend
    assert np.array_equal(l.mean, m.mean) and np.array_equal(l.basis.rows, m.basis.rows)
    assert np.array_equal(l.sketch.entries, m.sketch.entries)
    c = oracle.gaussian_cloud(25, 11, 15)
    adg.save_model(adg.fit(c, 7, EXACT, 9), str(tmp_path / "a.adg"))
    adg.save_model(adg.fit(c, 7, EXACT, 9), str(tmp_path / "b.adg"))
    assert open(tmp_path / "a.adg", "rb").read() == open(tmp_path / "b.adg", "rb").read()
    blob = open(p, "rb").read()
    (tmp_path / "short.adg").write_bytes(blob[:-5])
    with pytest.raises(adg.IoError, match="truncated"):
        adg.load_model(str(tmp_path / "short.adg"))
    (tmp_path / "magic.adg").write_bytes(b"X" + blob[1:])
    with pytest.raises(adg.IoError, match="magic"):
        adg.load_model(str(tmp_path / "magic.adg"))
    (tmp_path / "ver.adg").write_bytes(blob[:4] + b"\x09" + blob[5:])
    with pytest.raises(adg.IoError, match="version"):
        adg.load_model(str(tmp_path / "ver.adg"))


def test_padding_shrinks_distortion(oracle):
    # proj/tests/test_embed.cpp:273-289
    c = oracle.gaussian_cloud(400, 100, 20)
    scale = np.where(np.arange(100) < 10, np.sqrt(0.95 / 10), np.sqrt(0.05 / 90))
    c = c * scale
    cen, _ = oracle.center(c)
    b, _ = adg.exact_top_svd(cen, 10)
    pdist = adg.max_distortion(cen, cen @ b.rows.T)
    assert pdist > 0.05
    k = adg.jl_dimension(400, 0.5, 0.01)
    m = adg.fit_with_split(c, 10, k, EXACT, 1)
    assert adg.max_distortion(c, adg.transform_all(m, c).data) <= pdist * 0.5 + 0.02


# -------------------------------------------------------------- spectral
def test_exact_svd_diagonal():
    b, s = adg.exact_top_svd(np.diag([3.0, 2.0, 1.0]), 1)
    assert np.allclose(s.singular_values, [3, 2, 1], rtol=1e-12)
    assert not s.approximate
    assert abs(b.rows[0, 0] - 1) <= 1e-12 and abs(b.rows[0, 1]) < 1e-12 and abs(b.rows[0, 2]) < 1e-12


def test_exact_low_rank(oracle):
    cen, _ = oracle.center(oracle.low_rank_cloud(40, 12, 2, 5))
    b, s = adg.exact_top_svd(cen, 2)
    assert np.all(s.singular_values[2:] <= 1e-9)
    assert np.max(np.abs(cen @ b.rows.T @ b.rows - cen)) < 1e-9


def test_full_rank_isometry(oracle):
    cen, _ = oracle.center(oracle.gaussian_cloud(30, 8, 6))
    b, _ = adg.exact_top_svd(cen, 8)
    assert adg.max_distortion(cen, cen @ b.rows.T) <= 1e-9


def test_orthonormal_contractive(oracle):
    for seed in range(5):
        cen, _ = oracle.center(oracle.gaussian_cloud(50, 15, seed))
        s = 1 + seed % 7
        b, _ = adg.exact_top_svd(cen, s)
        assert np.max(np.abs(b.rows @ b.rows.T - np.eye(s))) <= 1e-8
        diffs = cen[:, None, :] - cen[None, :, :]
        assert np.all(np.linalg.norm(diffs @ b.rows.T, axis=-1)
                      <= np.linalg.norm(diffs, axis=-1) + 1e-9)


def test_exact_matches_lapack_stand_in(oracle):
    for seed in range(3):
        cen, _ = oracle.center(oracle.gaussian_cloud(40, 12, 100 + seed))
        b, s = adg.exact_top_svd(cen, 4)
        rb, rs = oracle.exact_top_svd(cen, 4)
        assert np.allclose(s.singular_values, rs, rtol=1e-10, atol=1e-12)
        assert np.max(np.abs(b.rows - rb)) <= 1e-8  # sign-normalised rows agree


def test_randomized(oracle):
    cen, _ = oracle.center(oracle.low_rank_cloud(60, 20, 2, 9))
    b, s = adg.randomized_top_svd(cen, 2, 10, 2, 4)
    assert s.approximate and len(s.singular_values) == 2
    assert np.max(np.abs(b.rows @ b.rows.T - np.eye(2))) <= 1e-8
    res = cen - cen @ b.rows.T @ b.rows
    assert np.sum(res ** 2) / np.sum(cen ** 2) <= 1e-6
    cen, _ = oracle.center(oracle.gaussian_cloud(50, 30, 12))
    a, sa = adg.randomized_top_svd(cen, 5, 10, 2, 99)
    a2, sa2 = adg.randomized_top_svd(cen, 5, 10, 2, 99)
    assert np.array_equal(a.rows, a2.rows) and np.array_equal(sa.singular_values, sa2.singular_values)
    # agrees with the reference's Halko restatement (same Gaussian test matrix)
    rb, rs = oracle.randomized_top_svd(cen, 5, 10, 2, 99)
    assert np.allclose(sa.singular_values, rs, rtol=1e-8)
    assert np.max(np.abs(a.rows.T @ a.rows - rb.T @ rb)) <= 1e-6


def test_exact_vs_randomized_projectors(oracle):
    cen, _ = oracle.center(oracle.low_rank_cloud(80, 25, 4, 21))
    e, _ = adg.exact_top_svd(cen, 4)
    r, _ = adg.randomized_top_svd(cen, 4, 10, 2, 3)
    assert np.max(np.abs(e.rows.T @ e.rows - r.rows.T @ r.rows)) <= 1e-6


def test_randomized_decaying(oracle):
    c = oracle.gaussian_cloud(150, 100, 33) * np.arange(1, 101) ** -1.2
    cen, _ = oracle.center(c)
    e, _ = adg.exact_top_svd(cen, 8)
    aligned = 0
    for seed in range(10):
        r, _ = adg.randomized_top_svd(cen, 8, 10, 2, seed)
        aligned += np.linalg.svd(e.rows @ r.rows.T, compute_uv=False).min() >= 0.99
    assert aligned >= 9
    c = oracle.gaussian_cloud(400, 300, 44) * np.arange(1, 301) ** -0.7
    cen, _ = oracle.center(c)
    _, ex = adg.exact_top_svd(cen, 40)
    _, rx = adg.randomized_top_svd(cen, 40, 10, 2, 7)
    assert abs(np.sum(rx.singular_values ** 2) / np.sum(ex.singular_values[:40] ** 2) - 1) <= 0.01


def test_spectral_validation(oracle):
    c = oracle.gaussian_cloud(10, 5, 0)
    with pytest.raises(ValueError):
        adg.exact_top_svd(c, 0)
    with pytest.raises(ValueError):
        adg.exact_top_svd(c, 6)
    with pytest.raises(ValueError):
        adg.randomized_top_svd(c, 3, 10, 2, 0)
    bad = c.copy()
    bad[0, 0] = np.nan
    with pytest.raises(adg.NumericError, match="non-finite"):
        adg.exact_top_svd(bad, 2)


def test_pca_bound_acceptance_9(oracle):
    # proj/tests/acceptance.cpp:421-446 (first 8 trials)
    st = Stream(909)
    worst = -1.0
    for _ in range(8):
        n = 20 + st.below(60)
        d = 5 + st.below(25)
        cen, _ = oracle.center(oracle.gaussian_cloud(n, d, st.next_u64()))
        s = 1 + st.below(min(n, d) - 1)
        b, sm = adg.exact_top_svd(cen, s)
        sig = sm.singular_values
        nxt = sig[s] if s < len(sig) else 0.0
        diffs = cen[:, None, :] - cen[None, :, :]
        iu = np.triu_indices(n, 1)
        dist = np.linalg.norm(diffs, axis=-1)[iu]
        meas = np.abs(np.linalg.norm(diffs @ b.rows.T, axis=-1)[iu] / dist - 1)
        worst = max(worst, float(np.max(meas - np.minimum(2 * nxt / dist, 1.0))))
    assert worst <= 1e-9


# -------------------------------------------------------------- jl / center
def test_jl_properties():
    m = adg.sample_jl(4, 10, 123).entries
    v = 0.5
    assert np.all((m == v) | (m == -v)) and 0 < (m == v).sum() < 40
    col = adg.sample_jl(10000, 1, 2024).entries
    assert 0.47 <= (col > 0).mean() <= 0.53
    with pytest.raises(ValueError):
        adg.sample_jl(0, 3, 0)


def test_center_gpu(oracle):
    cen, info = adg.center(np.array([[0.0, 0.0], [2.0, 2.0]]))
    assert cen.data[0, 0] == -1.0 and cen.data[1, 1] == 1.0 and np.all(info.mean == 1.0)
    c = oracle.gaussian_cloud(50, 6, 3)
    once, _ = adg.center(c)
    twice, m2 = adg.center(once.data)
    assert np.max(np.abs(twice.data - once.data)) < 1e-12 and np.max(np.abs(m2.mean)) < 1e-12
    rc, rm = oracle.center(c)
    assert np.max(np.abs(once.data - rc)) <= 1e-15


def test_torch_device_roundtrip(oracle):
    import torch
    c = oracle.gaussian_cloud(300, 24, 5).astype(np.float32)
    t = torch.from_numpy(c).cuda()
    m = adg.fit(t, 10, EXACT, 3)
    assert m.mean.is_cuda and m.basis.rows.is_cuda
    y = adg.transform_all(m, t).data
    assert y.is_cuda and y.dtype == torch.float32
    mh = adg.fit(c, 10, EXACT, 3)
    assert np.max(np.abs(m.basis.rows.cpu().numpy() - mh.basis.rows)) <= 1e-12
    r1 = adg.evaluate(t, y, engine="screen")
    r2 = adg.evaluate(c, y.cpu().numpy(), engine="screen")
    assert r1.max_distortion == r2.max_distortion and r1.argmax == r2.argmax


# ----------------------------------------------------- C++ facade / CLI flows
def test_cpp_facade_cli_flows(tmp_path):
    exe = str(tmp_path / "cli_flows")
    libdir = os.path.join(ROOT, "paper_1609_05388_b200")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "cli_flows.cpp"), "-L", libdir, "-ladg",
                           f"-Wl,-rpath,{libdir}", "-o", exe])
    import json
    docs = {}
    # ADAGIO_ENGINE (facade extension): the same flows through each engine
    for eng in (None, "exact", "screen", "screen_exact_hist"):
        env = dict(os.environ)
        env.pop("ADAGIO_ENGINE", None)
        if eng:
            env["ADAGIO_ENGINE"] = eng
        out = subprocess.run([exe, str(tmp_path / "m.adg")], capture_output=True, text=True,
                             timeout=120, env=env)
        assert out.returncode == 0, out.stderr
        doc = json.loads(out.stdout.strip().splitlines()[-1])
        assert doc["n_pairs_evaluated"] == 600 * 599 // 2 and doc["sampled"] is False
        docs[eng] = doc
    # n = 600: AUTO is the exact engine; the screen engines refine the max exactly
    assert docs[None]["histogram"] == docs["exact"]["histogram"] == docs["screen_exact_hist"]["histogram"]
    for eng in ("exact", "screen", "screen_exact_hist"):
        assert docs[eng]["max_distortion"] == docs[None]["max_distortion"]
    env = dict(os.environ, ADAGIO_ENGINE="fastest")
    bad = subprocess.run([exe, str(tmp_path / "m.adg")], capture_output=True, text=True, timeout=120, env=env)
    assert bad.returncode != 0 and "ADAGIO_ENGINE" in (bad.stderr + bad.stdout)
    m = adg.load_model(str(tmp_path / "m.adg"))
    assert m.target_dim() == 12 and m.seed == 7


# --------------------------------------------- run_distort --model flow
@pytest.mark.parametrize("n,engine", [(600, "exact"), (5000, "screen")])
def test_distort_model_matches_transform_then_evaluate(oracle, n, engine):
    """adg_distort_model (adagio_main.cpp:192-224) == transform_all + evaluate,
    bit for bit, for host and device inputs, with and without the embedding."""
    import torch
    c = oracle.gaussian_cloud(n, 48, 11).astype(np.float32)
    m = adg.fit(c, 12, EXACT, 2)
    y = adg.transform_all(m, c).data
    ref = adg.evaluate(c, y, hist_bins=40, engine=engine)
    got = adg.distort_model(m, c, hist_bins=40, engine=engine)
    rep_d, emb = adg.distort_model(m, torch.from_numpy(c).cuda(), hist_bins=40, engine=engine,
                                   return_embedded=True)
    assert np.array_equal(emb.data.cpu().numpy(), y)
    for r in (got, rep_d):
        assert r.max_distortion == ref.max_distortion and r.argmax == ref.argmax
        assert r.mean_distortion == ref.mean_distortion
        assert np.array_equal(r.histogram, ref.histogram)
        assert r.n_pairs_evaluated == ref.n_pairs_evaluated
    smp = adg.PairSampling.sample(1000, adg.derive_seed(0, "sampling"))
    a = adg.distort_model(m, c, smp, hist_bins=40)
    b = adg.evaluate(c, y, smp, hist_bins=40)
    assert a.sampled and a.max_distortion == b.max_distortion and np.array_equal(a.histogram, b.histogram)


def test_distort_model_validation(oracle):
    c = oracle.gaussian_cloud(50, 8, 1)
    m = adg.fit(c, 4, EXACT, 0)
    with pytest.raises(ValueError, match="sample size"):
        adg.distort_model(m, c, adg.PairSampling.sample(10**6, 1))
    with pytest.raises(ValueError, match="dimension"):
        adg.distort_model(m, c[:, :7])


@pytest.mark.parametrize("n,d,bins,knobs", [
    (5000, 48, 40, {}), (20000, 100, 50, {}),
    # one phase per chunk, and 3 chunks grouped by the flow model
    (20000, 100, 50, {"ADG_PIPE_GROUP": "0"}), (20000, 100, 50, {"ADG_PIPE_CHUNKS": "3"})])
def test_distort_model_pipelined_pinned_bit_exact(oracle, monkeypatch, n, d, bins, knobs):
    """Pinned host X takes the pipelined run_distort path (chunked H2D,
    embed/prep per group of chunks, phased screen): same report, bit for bit,
    as transform_all + evaluate on the device, for any chunking / grouping."""
    import torch
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    c = oracle.gaussian_cloud(n, d, 23).astype(np.float32)
    c[7] = c[4000]  # an exact duplicate pair (zero rule)
    m = adg.fit(c, 12, EXACT, 2)
    tc = torch.from_numpy(c).cuda()
    y = adg.transform_all(m, tc).data
    ref = adg.evaluate(tc, y, hist_bins=bins, engine="screen")
    pinned = torch.from_numpy(c).pin_memory()
    got, emb = adg.distort_model(m, pinned.numpy(), hist_bins=bins, engine="screen",
                                 return_embedded=True)
    assert np.array_equal(emb.data, y.cpu().numpy())
    assert got.max_distortion == ref.max_distortion and got.argmax == ref.argmax
    assert got.mean_distortion == ref.mean_distortion
    assert np.array_equal(got.histogram, ref.histogram)
    assert (got.n_pairs_evaluated, got.n_zero_distance_pairs) == (ref.n_pairs_evaluated, ref.n_zero_distance_pairs)


def _top_eig_sum(cen, s):
    w = np.linalg.eigvalsh(cen.T @ cen)
    return float(np.sort(w)[::-1][:s].sum())


@pytest.mark.parametrize("case", ["grid_jacobi_rank_deficient", "grid_cholesky_block"])
def test_exact_svd_large_blocks(case):
    """Large ranks: a 432-column block on the centred C3 rows (rank ~399 < 432)
    goes to one grid-wide Jacobi of the whole Gram; a 122-column block
    (d = 600) runs subspace iteration with the grid CholeskyQR.  Orthonormal,
    finite, and capturing the top-s variance of the fp64 eigen-solution."""
    import torch
    if case == "grid_jacobi_rank_deficient":
        from paper_1609_05388_b200 import datasets as ds
        X = ds.c3_mnist_like()[:8000].astype(np.float64)
        s = 200
    else:
        rng = np.random.default_rng(12)
        X = (rng.standard_normal((3000, 60)) * np.linspace(6.0, 2.0, 60)) @ rng.standard_normal((60, 600))
        X += 0.05 * rng.standard_normal(X.shape)
        s = 45
    cen = X - X.mean(0)
    b, _ = adg.exact_top_svd(torch.from_numpy(cen).cuda(), s, n_sigma=0)
    B = b.rows.cpu().numpy()
    assert np.isfinite(B).all()
    assert np.abs(B @ B.T - np.eye(s)).max() < 1e-10
    captured = float(np.square(cen @ B.T).sum())
    assert abs(captured - _top_eig_sum(cen, s)) <= 1e-9 * _top_eig_sum(cen, s)


@pytest.mark.parametrize("tail", ["flat", "slow"])
def test_exact_flat_spectrum_large_d(oracle, tail):
    """Subspace iteration (d > 384) on a spectrum that is flat around the
    wanted index: 10 strong directions, then lambda_i = 1 - 2e-4 i (flat) or a
    slow geometric tail.  Convergence is slow; the basis must still be the
    exact top-s subspace (the reference's BDCSVD is exact, spectral.cpp:52):
    the whole-Gram Jacobi takes over when the iteration would not converge."""
    rng = np.random.default_rng(7)
    n, d, s = 1200, 784, 25
    lam = np.ones(d)
    lam[:10] = 50.0 + 5.0 * np.arange(10)[::-1]
    idx = np.arange(d - 10)
    lam[10:] = 1.0 - 2e-4 * idx if tail == "flat" else 0.999 ** idx
    U = rng.standard_normal((n, d))
    U -= U.mean(axis=0)  # centred columns: the fit's centring leaves X as is
    U, _ = np.linalg.qr(U)
    V, _ = np.linalg.qr(rng.standard_normal((d, d)))
    X = (U * np.sqrt(lam * n)) @ V.T
    b, sv = adg.exact_top_svd(X - X.mean(axis=0), s)
    rb, rs = oracle.exact_top_svd(X - X.mean(axis=0), s)
    proj = b.rows.T @ b.rows - rb.T @ rb
    assert np.max(np.abs(proj)) <= 1e-8
    assert np.allclose(sv.singular_values[:s], rs[:s], rtol=1e-9)

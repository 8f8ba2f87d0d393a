"""Brute-force k-NN and the k-NN graph on the GPU (proj/src/downstream.cpp:24-137):
the reference's own tests (proj/tests/test_downstream.cpp:88-224) restated,
plus parity with the oracle's restatement (oracle/oracle.py nearest_rows /
knn_query / majority_classify / build_knn_graph) at sizes that span many
database tiles and query blocks, fp32 and bf16 storage, and k beyond the
shared-memory list capacity (global scratch lists).

Distances are fp64 norms of row differences in both; the per-dimension
summation order differs (Eigen's vectorised reduction, numpy's pairwise sum,
the kernel's sequential fma), so distances agree to ~1e-15 relative and the
neighbour order is compared exactly wherever two distances differ by more
than that -- exact ties (duplicate rows) must follow the index rule.
"""
import numpy as np
import pytest

import paper_1609_05388_b200 as adg

pytestmark = pytest.mark.gpu


def same_lists(got, ref, rtol=1e-13):
    assert len(got) == len(ref)
    for (gi, gd), (ri, rd) in zip(got, ref):
        assert abs(gd - rd) <= rtol * max(1.0, rd), (gi, gd, ri, rd)
    # index order must match except across near-equal (non-exact) distances
    gi = [i for i, _ in got]
    ri = [i for i, _ in ref]
    if gi != ri:
        for t in range(len(gi)):
            if gi[t] != ri[t]:
                assert abs(got[t][1] - ref[t][1]) <= rtol * max(1.0, ref[t][1])
                assert abs(got[t][1] - got[min(t + 1, len(got) - 1)][1]) <= 1e-12 or \
                    abs(got[t][1] - got[max(t - 1, 0)][1]) <= 1e-12


# ------------------------------------------- proj/tests/test_downstream.cpp
def test_knn_exact_match_and_tie_rule(oracle):
    db = oracle.gaussian_cloud(12, 4, 1)
    ex = adg.knn_query(db, db[7], 1)
    assert ex == [(7, 0.0)]
    line = np.arange(5, dtype=np.float64).reshape(5, 1)
    near = adg.knn_query(line, np.zeros(1), 3)
    assert [i for i, _ in near] == [0, 1, 2] and abs(near[2][1] - 2.0) < 1e-15
    pair = np.array([[1.0], [-1.0], [5.0]])
    tied = adg.knn_query(pair, np.zeros(1), 2)
    assert [i for i, _ in tied] == [0, 1]
    with pytest.raises(ValueError, match=r"knn_query: k = 4 outside \[1, 3\]"):
        adg.knn_query(pair, np.zeros(1), 4)
    with pytest.raises(ValueError, match="query dimension mismatch"):
        adg.knn_query(pair, np.zeros(2), 1)


def test_knn_matches_naive_sort_with_ties(oracle):
    db = oracle.gaussian_cloud(300, 6, 2)
    db[100] = db[10]
    db[200] = db[10]
    picks = oracle.rng_below(7, 300, 40)
    for t in range(20):
        q = db[int(picks[2 * t])]
        k = 1 + int(picks[2 * t + 1]) % 20
        got = adg.knn_query(db, q, k)
        ref = oracle.knn_query(db, q, k)
        same_lists(got, ref)
    # the duplicated rows tie exactly: lower index first
    got = adg.knn_query(db, db[10], 3)
    assert [i for i, _ in got] == [10, 100, 200] and all(dd == 0.0 for _, dd in got)


def test_majority_classify_pools_labels():
    db = adg.PointCloud(np.arange(10, dtype=np.float64).reshape(10, 1), [3 if i < 7 else 1 for i in range(10)])
    q = np.array([[3.2]])
    assert adg.majority_classify(q, db, 5, 0) == 3
    assert adg.majority_classify(q, db, 10, 0) == 3
    with pytest.raises(ValueError, match="database has no labels"):
        adg.majority_classify(q, adg.PointCloud(db.data), 3, 0)


def test_majority_classify_ties_deterministic(oracle):
    db = adg.PointCloud(np.arange(4, dtype=np.float64).reshape(4, 1), [5, 5, 9, 9])
    q = np.array([[1.5]])
    first = adg.majority_classify(q, db, 4, 31337)
    assert first in (5, 9)
    assert all(adg.majority_classify(q, db, 4, 31337) == first for _ in range(5))
    assert first == oracle.majority_classify(q, db.data, db.labels, 4, 31337)


def test_graph_symmetrized_union():
    cloud = np.array([[0.0, 0.0], [1.0, 0.0], [10.0, 0.0]])
    g = adg.build_knn_graph(cloud, 1)
    assert [(e.u, e.v) for e in g.edges] == [(0, 1), (1, 2)]
    assert all(e.weight == 1.0 for e in g.edges)


def test_graph_saturates(oracle):
    g = adg.build_knn_graph(oracle.gaussian_cloud(9, 3, 3), 8)
    assert len(g.edges) == 9 * 8 // 2


def test_graph_duplicates_no_self_loops():
    cloud = np.array([[1.0, 1.0], [1.0, 1.0], [5.0, 5.0], [5.0, 5.0]])
    g = adg.build_knn_graph(cloud, 1)
    assert all(e.u < e.v and e.weight > 0.0 for e in g.edges)
    assert any(e.u == 0 and e.v == 1 for e in g.edges)
    with pytest.raises(ValueError, match=r"build_knn_graph: k = 4 outside \[1, n\)"):
        adg.build_knn_graph(cloud, 4)


def test_graph_gaussian_weights(oracle):
    g = adg.build_knn_graph(oracle.gaussian_cloud(30, 4, 4), 3, adg.EdgeWeighting.gaussian)
    assert all(0.0 < e.weight <= 1.0 for e in g.edges)


# ------------------------------------------------------ parity with the oracle
@pytest.mark.parametrize("n,d,k,weighting", [(700, 20, 5, "binary"), (300, 33, 12, "gaussian"),
                                             (200, 7, 160, "binary")])
def test_graph_matches_oracle(oracle, n, d, k, weighting):
    cloud = oracle.gaussian_cloud(n, d, n + k)
    cloud[5] = cloud[17]  # an exact duplicate pair
    g = adg.build_knn_graph(cloud, k, adg.EdgeWeighting[weighting])
    ref = oracle.build_knn_graph(cloud, k, weighting)
    assert [(e.u, e.v) for e in g.edges] == [(u, v) for u, v, _ in ref]
    for e, (_, _, w) in zip(g.edges, ref):
        assert abs(e.weight - w) <= 1e-12


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_knn_batch_large_matches_oracle(oracle, dtype):
    """5000 x 64 database (79 tiles), 200 queries (4 query blocks), k = 30."""
    import torch
    rng = np.random.default_rng(3)
    db = rng.standard_normal((5000, 64)).astype(np.float32)
    qs = rng.standard_normal((200, 64)).astype(np.float32)
    tdb, tq = torch.from_numpy(db).cuda(), torch.from_numpy(qs).cuda()
    if dtype == "bf16":
        tdb, tq = tdb.to(torch.bfloat16), tq.to(torch.bfloat16)
    idx, dist = adg.knn_query_batch(tdb, tq, 30)
    dbh = tdb.double().cpu().numpy()
    qh = tq.double().cpu().numpy()
    for t in range(0, 200, 7):
        same_lists(list(zip(idx[t].tolist(), dist[t].tolist())), oracle.knn_query(dbh, qh[t], 30))


# --------------------------------------- tensor-core graph path (n >= 4096)
def _graph_cols(g):
    return g.edges.u.copy(), g.edges.v.copy(), g.edges.weight.copy()


def _tc_and_simt(monkeypatch, cloud, k, weighting):
    g = adg.build_knn_graph(cloud, k, adg.EdgeWeighting[weighting])
    assert adg.api.last_knn_engine() == "tensor"
    monkeypatch.setenv("ADG_KNN_SIMT", "1")
    s = adg.build_knn_graph(cloud, k, adg.EdgeWeighting[weighting])
    assert adg.api.last_knn_engine() == "simt"
    monkeypatch.delenv("ADG_KNN_SIMT")
    return _graph_cols(g), _graph_cols(s)


def _clustered(n, d, seed, dtype=np.float32):
    rng = np.random.default_rng(seed)
    centres = rng.standard_normal((40, d)) * 4.0
    x = centres[rng.integers(0, 40, n)] + rng.standard_normal((n, d)) * 0.3
    x[rng.integers(0, n, 300)] = x[rng.integers(0, n, 300)]  # exact duplicates
    return x.astype(dtype)


@pytest.mark.parametrize("case", ["gauss_f32", "clustered_dups_f32", "integer_ties_f32", "f64_d37",
                                  "k63"])
def test_graph_tensor_path_equals_simt(monkeypatch, case):
    """The candidate screen + exact refine gives bit-identical graphs to the
    fp64 SIMT tiles: same edges, same weights (same distances, same ties)."""
    rng = np.random.default_rng(11)
    k, w = 10, "gaussian"
    if case == "gauss_f32":
        x = rng.standard_normal((6000, 96)).astype(np.float32)
    elif case == "clustered_dups_f32":
        x, k = _clustered(5000, 40, 2), 7
    elif case == "integer_ties_f32":  # coordinates in {0..3}: massive exact ties
        x, k, w = rng.integers(0, 4, (4500, 12)).astype(np.float32), 5, "binary"
    elif case == "f64_d37":
        x = _clustered(4200, 37, 3, np.float64)
    else:
        x, k, w = rng.standard_normal((4096, 24)).astype(np.float32), 63, "binary"
    (gu, gv, gw), (su, sv, sw) = _tc_and_simt(monkeypatch, x, k, w)
    assert np.array_equal(gu, su) and np.array_equal(gv, sv)
    assert np.array_equal(gw.view(np.uint64), sw.view(np.uint64))


def test_graph_tensor_path_bf16_device_input(monkeypatch):
    import torch
    x = torch.from_numpy(_clustered(4500, 64, 4)).cuda().to(torch.bfloat16)
    (gu, gv, gw), (su, sv, sw) = _tc_and_simt(monkeypatch, x, 12, "binary")
    assert np.array_equal(gu, su) and np.array_equal(gv, sv) and np.array_equal(gw, sw)


def test_graph_tensor_path_matches_oracle(oracle):
    """n = 4096 through the tensor path against the oracle's restatement."""
    cloud = oracle.gaussian_cloud(4096, 16, 21)
    cloud[5] = cloud[17]
    g = adg.build_knn_graph(cloud, 6, adg.EdgeWeighting.gaussian)
    assert adg.api.last_knn_engine() == "tensor"
    ref = oracle.build_knn_graph(cloud, 6, "gaussian")
    assert [(e.u, e.v) for e in g.edges] == [(u, v) for u, v, _ in ref]
    assert np.allclose(g.edges.weight, np.array([w for _, _, w in ref]), rtol=0, atol=1e-12)

"""oracle.py -- Python face of the ADAgIO CPU oracle.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, as the checker -- never by the
product package (paper_1609_05388_b200), which fails loudly without its CUDA
library instead of falling back to anything here.

* ``liboracle.so`` (oracle/adagio_oracle.c) restates, in fp64 C, the
  reference's rng.hpp, jl.cpp, dataset.cpp center, embed.cpp transform and the
  whole of distortion.cpp evaluate (block order, Neumaier, zero rule, binning),
  plus the argmax extension (lowest linear pair index on exact ties).
* The spectral step lives in Eigen in the reference (BDCSVD / HouseholderQR,
  proj/src/spectral.cpp:42-101; Eigen >= 3.3, un-vendored, unpinned --
  proj/CMakeLists.txt:12).  It is restated here with numpy/LAPACK: gesdd for
  BDCSVD (same math, not the same bits) and Householder QR (geqrf) for thin_q.
  Only span(Q) matters for the randomized backend, so QR sign
  conventions drop out.  Parity of the exact basis at BASELINE sizes is
  therefore pinned only through the reference's own property tests
  (proj/tests/test_spectral.cpp) and the spectral gaps -- see DESIGN.md.

Parity pins: tests/golden/rng_golden.json is produced by the reference's own
rng.hpp compiled from /root/reference (oracle/Makefile target ``ref``); the
known-answer tests of proj/tests/test_{distortion,embed,jl,spectral}.cpp are
restated in tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    """Compile liboracle.so (and oracle/_ref when the reference is present)."""
    subprocess.check_call(["make", "-s", "-C", _HERE])
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.check_call(["make", "-s", "-C", _HERE, "ref"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        u64, i64, dbl, i32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        P = ctypes.c_void_p
        L.or_mix64.restype = u64
        L.or_mix64.argtypes = [u64]
        L.or_fnv1a64.restype = u64
        L.or_fnv1a64.argtypes = [ctypes.c_char_p, i64]
        L.or_derive_seed.restype = u64
        L.or_derive_seed.argtypes = [u64, ctypes.c_char_p]
        L.or_hash_position.restype = u64
        L.or_hash_position.argtypes = [u64, u64, u64]
        L.or_rademacher_sign.restype = dbl
        L.or_rademacher_sign.argtypes = [u64, u64, u64]
        L.or_rng_u64.argtypes = [u64, i64, P]
        L.or_rng_below.argtypes = [u64, u64, i64, P]
        L.or_rng_normal.argtypes = [u64, i64, P]
        L.or_sample_jl.restype = i32
        L.or_sample_jl.argtypes = [i64, i64, u64, P]
        L.or_jl_dimension.restype = i64
        L.or_jl_dimension.argtypes = [i64, dbl, dbl]
        L.or_center.argtypes = [P, i64, i64, P, P]
        L.or_transform_all.argtypes = [P, P, i64, P, i64, i64, P, i64, P, i32]
        L.or_evaluate.restype = i32
        L.or_evaluate.argtypes = [P, i64, i64, P, i64, i64, i32, u64, u64, i32, dbl, u64, i32,
                                  P, P, dbl, P, i64, i64]
        L.or_evaluate_f32.restype = i32
        L.or_evaluate_f32.argtypes = [P, i64, i64, P, i64, i32, dbl, i32, P, P, i64, i64]
        L.or_decode_pair.argtypes = [u64, u64, P, P]
        L.or_evaluate_f32_sampled.restype = i32
        L.or_evaluate_f32_sampled.argtypes = [P, i64, i64, P, i64, u64, u64, i32, dbl, i32, P, P]
        L.or_edge_band_counts.restype = i32
        L.or_edge_band_counts.argtypes = [P, P, i64, i64, i64, P, P, dbl, dbl, i32, dbl, i32, P]
        L.or_sample_pair_indices.restype = i32
        L.or_sample_pair_indices.argtypes = [u64, u64, u64, P]
        L.or_pair_distortion.restype = dbl
        L.or_pair_distortion.argtypes = [P, P, P, P, i64, i64]
        L.or_naive_distortion.argtypes = [P, i64, i64, P, i64, P, P, P, P]
        _lib = L
    return _lib


class _Report(ctypes.Structure):
    _fields_ = [("max_distortion", ctypes.c_double), ("mean_distortion", ctypes.c_double),
                ("n_pairs_evaluated", ctypes.c_uint64), ("n_zero_distance_pairs", ctypes.c_uint64),
                ("argmax_i", ctypes.c_uint64), ("argmax_j", ctypes.c_uint64),
                ("hist_bins", ctypes.c_int32), ("sampled", ctypes.c_int32),
                ("hist_max", ctypes.c_double), ("sample_seed", ctypes.c_uint64)]


@dataclass
class OracleReport:
    max_distortion: float
    mean_distortion: float
    histogram: np.ndarray
    hist_bins: int
    hist_max: float
    n_pairs_evaluated: int
    n_zero_distance_pairs: int
    sampled: bool
    sample_seed: int | None
    argmax: tuple | None
    edge_near: np.ndarray | None = field(default=None)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ rng.hpp
def mix64(x):
    return int(lib().or_mix64(x))


def fnv1a64(s: str):
    b = s.encode()
    return int(lib().or_fnv1a64(b, len(b)))


def derive_seed(seed, purpose: str):
    return int(lib().or_derive_seed(seed, purpose.encode()))


def hash_position(seed, i, j):
    return int(lib().or_hash_position(seed, i, j))


def rademacher_sign(seed, i, j):
    return float(lib().or_rademacher_sign(seed, i, j))


def rng_u64(seed, count):
    out = np.zeros(count, np.uint64)
    lib().or_rng_u64(seed, count, _p(out))
    return out


def rng_below(seed, bound, count):
    out = np.zeros(count, np.uint64)
    lib().or_rng_below(seed, bound, count, _p(out))
    return out


def rng_normal(seed, count):
    out = np.zeros(count, np.float64)
    lib().or_rng_normal(seed, count, _p(out))
    return out


def gaussian_cloud(n, d, seed):
    """proj/tests/test_util.hpp:17-24 (row-major SeededRng normals)."""
    return rng_normal(seed, n * d).reshape(n, d)


def low_rank_cloud(n, d, rank, seed):
    """proj/tests/test_util.hpp:28-40."""
    g = rng_normal(seed, rank * d + n * rank)
    directions = g[: rank * d].reshape(rank, d)
    coefficients = g[rank * d:].reshape(n, rank)
    return coefficients @ directions


# ------------------------------------------------------------------ jl.cpp
def sample_jl(k, d, seed):
    out = np.zeros((k, d), np.float64)
    if lib().or_sample_jl(k, d, seed, _p(out)) != 0:
        raise ValueError("sample_jl: k and d must be >= 1")
    return out


def jl_dimension(n_points, epsilon, gamma):
    v = int(lib().or_jl_dimension(n_points, epsilon, gamma))
    if v < 0:
        raise ValueError("jl_dimension: invalid arguments")
    return v


# ------------------------------------------------------------- dataset.cpp
def center(X):
    X = _c64(X)
    n, d = X.shape
    mean = np.zeros(d)
    cen = np.zeros_like(X)
    lib().or_center(_p(X), n, d, _p(mean), _p(cen))
    return cen, mean


# ------------------------------------------------------------ spectral.cpp
def _normalize_row_signs(rows):
    """proj/src/spectral.cpp:21-27 (first max-|.| entry made positive)."""
    rows = rows.copy()
    for i in range(rows.shape[0]):
        idx = int(np.argmax(np.abs(rows[i])))  # numpy argmax keeps the first max
        if rows[i, idx] < 0.0:
            rows[i] = -rows[i]
    return rows


def exact_top_svd(X, s):
    """proj/src/spectral.cpp:42-62 with LAPACK gesdd standing in for BDCSVD."""
    X = _c64(X)
    n, d = X.shape
    if s < 1 or s > min(n, d):
        raise ValueError(f"exact_top_svd: s = {s} outside [1, {min(n, d)}]")
    if not np.all(np.isfinite(X)):
        raise FloatingPointError("exact_top_svd: input contains non-finite values")
    _, sig, vt = np.linalg.svd(X, full_matrices=False)
    return _normalize_row_signs(vt[:s]), sig


def randomized_top_svd(X, s, oversampling=10, power_iters=2, seed=0):
    """proj/src/spectral.cpp:64-101 (Halko range finder; thin_q = Householder QR)."""
    X = _c64(X)
    n, d = X.shape
    max_rank = min(n, d)
    if s < 1 or oversampling < 0 or s + oversampling > max_rank:
        raise ValueError(f"randomized_top_svd: need 1 <= s and s + oversampling <= {max_rank}")
    w = s + oversampling
    test = rng_normal(seed, d * w).reshape(d, w)  # filled row-major, spectral.cpp:79-82
    q = np.linalg.qr(X @ test)[0]
    for _ in range(power_iters):
        co = np.linalg.qr(X.T @ q)[0]
        q = np.linalg.qr(X @ co)[0]
    projected = q.T @ X
    _, sig, vt = np.linalg.svd(projected, full_matrices=False)
    return _normalize_row_signs(vt[:s]), sig[:s]


# --------------------------------------------------------------- embed.cpp
def principal_basis(centered, s, backend, seed):
    """proj/src/embed.cpp:29-56."""
    n, d = centered.shape
    if s == 0:
        return np.zeros((0, d))
    max_rank = min(n, d)
    if s <= max_rank:
        if backend == "randomized":
            return randomized_top_svd(centered, s, min(10, max_rank - s), 2,
                                      derive_seed(seed, "spectral"))[0]
        return exact_top_svd(centered, s)[0]
    _, _, vt = np.linalg.svd(centered, full_matrices=True)
    return _normalize_row_signs(vt[:s])


def fit_with_split(X, s, k, backend="exact", seed=0):
    """proj/src/embed.cpp:115-141 -> (mean, P, S)."""
    X = _c64(X)
    cen, mean = center(X)
    P = principal_basis(cen, s, backend, seed)
    S = sample_jl(k, X.shape[1], derive_seed(seed, "jl"))
    return mean, P, S


def fit(X, target_dim, backend="exact", seed=0):
    """proj/src/embed.cpp:105-113 (s = floor(r/2), k = r - s)."""
    return fit_with_split(X, target_dim // 2, target_dim - target_dim // 2, backend, seed)


def transform_all(mean, P, S, X, threads=0):
    X = _c64(X)
    n, d = X.shape
    s, k = P.shape[0], S.shape[0]
    out = np.zeros((n, s + k))
    P = _c64(P) if s else np.zeros((0, d))
    lib().or_transform_all(_p(_c64(mean)), _p(P), s, _p(_c64(S)), k, d, _p(X), n, _p(out),
                           threads)
    return out


# ---------------------------------------------------------- distortion.cpp
def evaluate(orig, emb, all_pairs=True, m=0, sample_seed=0, hist_bins=50, hist_max=1.0,
             pairs_per_block=16384, threads=0, edge_band=0.0, row_range=None):
    orig = _c64(orig)
    emb = _c64(emb)
    n, d = orig.shape
    r = emb.shape[1]
    rep = _Report()
    hist = np.zeros(max(hist_bins, 0) + 1, np.uint64)
    edge = np.zeros(2 * max(hist_bins, 1), np.uint64) if edge_band > 0 else None
    rb, re = (0, n) if row_range is None else row_range
    rc = lib().or_evaluate(_p(orig), n, d, _p(emb), emb.shape[0], r, int(all_pairs), m,
                           sample_seed, hist_bins, hist_max, pairs_per_block, threads,
                           ctypes.byref(rep), _p(hist), edge_band,
                           _p(edge) if edge is not None else None, rb, re)
    if rc != 0:
        raise ValueError("evaluate: invalid arguments")
    am = None if rep.argmax_i == 2**64 - 1 else (int(rep.argmax_i), int(rep.argmax_j))
    out = OracleReport(rep.max_distortion, rep.mean_distortion, hist, hist_bins, hist_max,
                       int(rep.n_pairs_evaluated), int(rep.n_zero_distance_pairs),
                       bool(rep.sampled), int(rep.sample_seed) if rep.sampled else None, am,
                       edge[:hist_bins] if edge is not None else None)
    out.edge_near10 = edge[hist_bins:] if edge is not None else None  # within 10 * edge_band
    return out


def screen_shift_norms(A, sample=4096):
    """Squared row norms after the GPU SCREEN's centring shift (the column
    mean of rows 0, step, 2 step, ... with step = ceil(n / 4096), as
    column_means_sampled in csrc/adg_embed.cu) -- test infrastructure."""
    A64 = np.asarray(A, np.float64)
    n = A64.shape[0]
    step = max(1, -(-n // sample))
    mu = A64[::step].mean(axis=0)
    C = A64 - mu
    return np.einsum("ij,ij->i", C, C)


def screen_rel_eps(d, r):
    """The SCREEN engine's error coefficient (csrc/adg_screen.cu, setup):
    (3 * K16 + 64) * 2^-24 with K16 = ceil(d / 16) + ceil(r / 16)."""
    k16 = -(-d // 16) + -(-r // 16)
    return (3.0 * k16 + 64.0) * 2.0 ** -24


def edge_band_counts(X, Y, hist_bins=50, hist_max=1.0, frac=0.25, threads=0):
    """Per bin edge q = 1..hist_bins: pairs whose exact value lies within the
    SCREEN's rigorous per-pair error bound of edge q, and within frac of it
    (the exact-histogram mode's band) -- TEST INFRASTRUCTURE bounding how far
    the SCREEN histogram may differ from the reference's."""
    X = np.ascontiguousarray(X, np.float32)
    Y = np.ascontiguousarray(Y, np.float32)
    n, d = X.shape
    r = Y.shape[1]
    nx = np.ascontiguousarray(screen_shift_norms(X))
    ny = np.ascontiguousarray(screen_shift_norms(Y))
    out = np.zeros(2 * hist_bins, np.uint64)
    rc = lib().or_edge_band_counts(_p(X), _p(Y), n, d, r, _p(nx), _p(ny), screen_rel_eps(d, r),
                                   frac, hist_bins, hist_max, threads, _p(out))
    if rc != 0:
        raise ValueError("edge_band_counts: invalid arguments")
    return out[:hist_bins], out[hist_bins:]


def evaluate_f32(orig, emb, hist_bins=50, hist_max=1.0, threads=0, row_range=None):
    """Same algorithm reading fp32 rows (exactly widened); for the CPU baseline."""
    orig = np.ascontiguousarray(orig, np.float32)
    emb = np.ascontiguousarray(emb, np.float32)
    n, d = orig.shape
    rep = _Report()
    hist = np.zeros(hist_bins + 1, np.uint64)
    rb, re = (0, n) if row_range is None else row_range
    lib().or_evaluate_f32(_p(orig), n, d, _p(emb), emb.shape[1], hist_bins, hist_max, threads,
                          ctypes.byref(rep), _p(hist), rb, re)
    am = None if rep.argmax_i == 2**64 - 1 else (int(rep.argmax_i), int(rep.argmax_j))
    return OracleReport(rep.max_distortion, rep.mean_distortion, hist, hist_bins, hist_max,
                        int(rep.n_pairs_evaluated), int(rep.n_zero_distance_pairs), False, None, am)


def evaluate_f32_sampled(orig, emb, m, sample_seed, hist_bins=50, hist_max=1.0, threads=0):
    """The reference's sampled mode (distortion.cpp:90-103, :151-154) on fp32
    clouds read in place (exactly widened), for BASELINE-size parity checks."""
    orig = np.ascontiguousarray(orig, np.float32)
    emb = np.ascontiguousarray(emb, np.float32)
    n, d = orig.shape
    rep = _Report()
    hist = np.zeros(hist_bins + 1, np.uint64)
    rc = lib().or_evaluate_f32_sampled(_p(orig), n, d, _p(emb), emb.shape[1], m, sample_seed,
                                       hist_bins, hist_max, threads, ctypes.byref(rep), _p(hist))
    if rc != 0:
        raise ValueError("evaluate: invalid arguments")
    am = None if rep.argmax_i == 2**64 - 1 else (int(rep.argmax_i), int(rep.argmax_j))
    return OracleReport(rep.max_distortion, rep.mean_distortion, hist, hist_bins, hist_max,
                        int(rep.n_pairs_evaluated), int(rep.n_zero_distance_pairs), True,
                        int(sample_seed), am)


def decode_pair(p, n):
    i, j = ctypes.c_uint64(), ctypes.c_uint64()
    lib().or_decode_pair(p, n, ctypes.byref(i), ctypes.byref(j))
    return int(i.value), int(j.value)


def sample_pair_indices(total, m, seed):
    out = np.zeros(m, np.uint64)
    if lib().or_sample_pair_indices(total, m, seed, _p(out)) != 0:
        raise ValueError("sample size outside range")
    return out


def pair_distortion(x, y, fx, fy):
    x, y, fx, fy = (_c64(v) for v in (x, y, fx, fy))
    v = lib().or_pair_distortion(_p(x), _p(y), _p(fx), _p(fy), x.size, fx.size)
    if v < 0:
        raise ValueError("pair_distortion: coincident points")
    return float(v)


def naive_distortion(orig, emb):
    orig, emb = _c64(orig), _c64(emb)
    mx, mean = ctypes.c_double(), ctypes.c_double()
    ev, zp = ctypes.c_uint64(), ctypes.c_uint64()
    lib().or_naive_distortion(_p(orig), orig.shape[0], orig.shape[1], _p(emb), emb.shape[1],
                              ctypes.byref(mx), ctypes.byref(mean), ctypes.byref(ev),
                              ctypes.byref(zp))
    return mx.value, mean.value, int(ev.value), int(zp.value)


# --------------------------------------------------------------- sweep.cpp
def split_energy_cloud(n, d, core, core_energy, seed):
    """proj/tests/test_util.hpp:44-54."""
    cloud = gaussian_cloud(n, d, seed)
    core_scale = np.sqrt(core_energy / float(core))
    tail_scale = np.sqrt((1.0 - core_energy) / float(d - core))
    cloud[:, :core] *= core_scale
    cloud[:, core:] *= tail_scale
    return cloud


METHODS = ("adagio_exact", "adagio_randomized", "pca", "jl", "external")


def _embed_cell(centered, cache, method, r, seed, external_map):
    """proj/src/sweep.cpp:60-137 (embed_cell); cache = [full-rank rows or None]."""
    n, d = centered.shape
    max_rank = min(n, d)

    def prefix(s):
        if cache[0] is None:  # sweep.cpp:33-39: full usable rank, computed once
            cache[0] = exact_top_svd(centered, max_rank)[0]
        return cache[0][:s]

    if method == "pca":
        return centered @ prefix(min(r, max_rank)).T
    if method == "jl":
        return centered @ sample_jl(r, d, derive_seed(seed, "jl")).T
    if method == "external":
        if external_map is None:
            raise ValueError("sweep: method external needs an embedding matrix")
        if external_map.shape[1] != d:
            raise ValueError(f"sweep: external matrix has {external_map.shape[1]} columns, "
                             f"cloud has {d}")
        return centered @ np.asarray(external_map, np.float64).T
    s, k = r // 2, r - r // 2
    if method == "adagio_exact" and s <= max_rank:
        P = prefix(s) if s else np.zeros((0, d))
        S = sample_jl(k, d, derive_seed(seed, "jl"))
        return transform_all(np.zeros(d), P, S, centered)
    mean, P, S = fit_with_split(centered, s, k,
                                "exact" if method == "adagio_exact" else "randomized", seed)
    return transform_all(mean, P, S, centered)


def tradeoff(cloud, dims, methods, seeds, all_pairs=True, m=0, sample_seed=0,
             external_map=None):
    """proj/src/sweep.cpp:161-201 -> [(method, target_dim, seed, max_distortion)]."""
    cloud = _c64(cloud)
    n, d = cloud.shape
    if len(dims) == 0:
        raise ValueError("tradeoff: dims must be non-empty")
    for r in dims:
        if r < 1 or r > d:
            raise ValueError(f"tradeoff: dim {r} outside [1, {d}]")
    centered, _ = center(cloud)
    cache = [None]
    rows = []
    for method in methods:
        cell_dims = list(dims) if method != "external" else [
            external_map.shape[0] if external_map is not None else 0]
        for r in cell_dims:
            for seed in seeds:
                emb = _embed_cell(centered, cache, method, r, seed, external_map)
                rep = evaluate(centered, emb, all_pairs=all_pairs, m=m, sample_seed=sample_seed)
                rows.append((method, r, seed, rep.max_distortion))
    return rows


def min_dim_for_distortion(cloud, method, delta, seed, r_min, r_max):
    """proj/src/sweep.cpp:203-265 -> (target_dim, achieved_distortion, achieved,
    monotone, probed dict)."""
    cloud = _c64(cloud)
    n, d = cloud.shape
    if not (0.0 < delta < 1.0):
        raise ValueError("min_dim_for_distortion: delta must lie in (0, 1)")
    if r_min < 1 or r_min > r_max or r_max > d:
        raise ValueError("min_dim_for_distortion: need 1 <= r_min <= r_max <= d")
    if method == "external":
        raise ValueError("min_dim_for_distortion: external maps have a fixed dimension")
    centered, _ = center(cloud)
    cache = [None]
    probed = {}

    def probe(r):
        if r not in probed:
            emb = _embed_cell(centered, cache, method, r, seed, None)
            probed[r] = evaluate(centered, emb).max_distortion
        return probed[r]

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
    monotone, previous = True, -1.0
    for r in sorted(probed):
        if previous >= 0.0 and probed[r] > previous + 1e-12:
            monotone = False
        previous = probed[r]
    return res[0], res[1], res[2], monotone, probed


# ---------------------------------------------------------- downstream.cpp
def nearest_rows(cloud, query, k, skip=-1):
    """proj/src/downstream.cpp:24-40: the k smallest (distance, index) pairs,
    distance = fp64 norm of (row - query), ties toward the smaller index."""
    cloud = _c64(cloud)
    dist = np.sqrt(((cloud - np.asarray(query, np.float64)[None, :]) ** 2).sum(axis=1))
    idx = np.arange(cloud.shape[0])
    if skip >= 0:
        keep = idx != skip
        dist, idx = dist[keep], idx[keep]
    order = np.lexsort((idx, dist))[:k]  # by distance, then index
    return [(int(idx[t]), float(dist[t])) for t in order]


def knn_query(database, query, k):
    """proj/src/downstream.cpp:49-60"""
    database = _c64(database)
    if k < 1 or k > database.shape[0]:
        raise ValueError(f"knn_query: k = {k} outside [1, {database.shape[0]}]")
    if len(query) != database.shape[1]:
        raise ValueError("knn_query: query dimension mismatch")
    return nearest_rows(database, query, k)


def majority_classify(queries, database, labels, k, tie_seed):
    """proj/src/downstream.cpp:62-88"""
    if labels is None:
        raise ValueError("majority_classify: database has no labels")
    queries = _c64(queries)
    if queries.shape[0] == 0:
        raise ValueError("majority_classify: no query descriptors")
    counts = {}
    for q in queries:
        for idx, _ in knn_query(database, q, k):
            counts[int(labels[idx])] = counts.get(int(labels[idx]), 0) + 1
    best = max(counts.values())
    tied = sorted(lbl for lbl, c in counts.items() if c == best)
    if len(tied) == 1:
        return tied[0]
    return tied[int(rng_below(tie_seed, len(tied), 1)[0])]


def build_knn_graph(cloud, k, weighting="binary"):
    """proj/src/downstream.cpp:90-137 -> [(u, v, weight)] sorted by (u, v)."""
    cloud = _c64(cloud)
    n = cloud.shape[0]
    if k < 1 or k >= n:
        raise ValueError(f"build_knn_graph: k = {k} outside [1, n)")
    lists = [nearest_rows(cloud, cloud[u], k, u) for u in range(n)]
    sigma = 0.0
    if weighting == "gaussian":
        dists = sorted(dd for lst in lists for _, dd in lst)
        sigma = dists[len(dists) // 2]
    edges = {}
    for u in range(n):
        for v, dist in lists[u]:
            key = (min(u, v), max(u, v))
            w = 1.0
            if weighting == "gaussian" and sigma > 0.0:
                w = float(np.exp(-dist * dist / (sigma * sigma)))
            edges.setdefault(key, w)  # std::map::emplace keeps the first
    return [(a, b, w) for (a, b), w in sorted(edges.items())]

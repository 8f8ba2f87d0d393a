"""Brute-force k-NN and the k-NN graph: proj/include/adagio/downstream.hpp /
proj/src/downstream.cpp:24-137, over the C ABI (adg_knn_query,
adg_majority_classify, adg_build_knn_graph; kernels in csrc/adg_knn.cu).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

from . import _lib
from .api import InvalidArgument, PointCloud, _ctx_for, _data, _matrix, _Operand


class EdgeWeighting(enum.IntEnum):
    """proj/include/adagio/downstream.hpp:29"""
    binary = 0
    gaussian = 1


@dataclass
class Edge:
    u: int
    v: int
    weight: float = 1.0


class EdgeList:
    """Sequence view of a graph's edges over numpy columns (u < v, weight);
    Edge objects are built on access, so million-edge graphs stay arrays."""

    def __init__(self, u, v, w):
        self.u, self.v, self.weight = u, v, w

    def __len__(self):
        return int(self.u.shape[0])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[t] for t in range(*i.indices(len(self)))]
        return Edge(int(self.u[i]), int(self.v[i]), float(self.weight[i]))

    def __iter__(self):
        for t in range(len(self)):
            yield Edge(int(self.u[t]), int(self.v[t]), float(self.weight[t]))


@dataclass
class KnnGraph:
    """proj/include/adagio/downstream.hpp:14-25 (edges: sequence of Edge,
    backed by the numpy columns edges.u / edges.v / edges.weight)."""
    n: int = 0
    k: int = 0
    edges: EdgeList = field(default_factory=lambda: EdgeList(np.zeros(0, np.int32),
                                                             np.zeros(0, np.int32),
                                                             np.zeros(0)))


def knn_query_batch(database, queries, k: int) -> Tuple[np.ndarray, np.ndarray]:
    """knn_query for every row of `queries`: (indices, distances), each
    (nq, k), ascending by (distance, index) per row."""
    db = _matrix(_data(database), "database")
    q = _matrix(_data(queries), "queries")
    ctx, _ = _ctx_for(db, q)
    nq = q.shape[0]
    idx = np.zeros((nq, max(k, 1)), np.int64)
    dist = np.zeros((nq, max(k, 1)), np.float64)
    _lib.check(_lib.load().adg_knn_query(ctx, db.ptr, db.code, db.shape[0], db.shape[1], q.ptr,
                                         q.code, nq, q.shape[1], int(k), idx.ctypes.data,
                                         dist.ctypes.data))
    return idx[:, :k], dist[:, :k]


def knn_query(database, query, k: int) -> List[Tuple[int, float]]:
    """proj/src/downstream.cpp:49-60: the k nearest database rows by Euclidean
    distance, ascending, distance ties toward the smaller index."""
    qv = np.asarray(query.detach().cpu() if hasattr(query, "detach") else query, np.float64)
    if qv.ndim != 1:
        raise InvalidArgument("knn_query: query must be a vector")
    idx, dist = knn_query_batch(database, qv.reshape(1, -1), k)
    return [(int(i), float(d)) for i, d in zip(idx[0], dist[0])]


def majority_classify(query_descriptors, database: PointCloud, k: int, tie_seed: int) -> int:
    """proj/src/downstream.cpp:62-88: modal label of the pooled k-NN label
    multiset of all query descriptors; ties resolved by SeededRng(tie_seed)."""
    labels = database.labels if isinstance(database, PointCloud) else None
    lab = None if labels is None else np.ascontiguousarray(np.asarray(labels, np.int32))
    db = _matrix(_data(database), "database")
    q = _matrix(_data(query_descriptors), "queries")
    ctx, _ = _ctx_for(db, q)
    out = ctypes.c_int32()
    _lib.check(_lib.load().adg_majority_classify(
        ctx, q.ptr, q.code, q.shape[0], q.shape[1], db.ptr, db.code, db.shape[0], db.shape[1],
        lab.ctypes.data if lab is not None else None, int(k), int(tie_seed) & (2**64 - 1),
        ctypes.byref(out)))
    return int(out.value)


def build_knn_graph(cloud, k: int, weighting: EdgeWeighting = EdgeWeighting.binary) -> KnnGraph:
    """proj/src/downstream.cpp:90-137: symmetrised-union k-NN graph, edges
    sorted by (u, v), binary or Gaussian (sigma = median k-NN distance)."""
    x = _matrix(_data(cloud))
    n = x.shape[0]
    ctx, _ = _ctx_for(x)
    cap = max(n * max(int(k), 1), 1)
    buf = np.empty(cap, dtype=np.dtype([("u", "<i4"), ("v", "<i4"), ("w", "<f8")]))
    written = ctypes.c_int64()
    _lib.check(_lib.load().adg_build_knn_graph(
        ctx, x.ptr, x.code, n, x.shape[1], int(k), int(weighting),
        buf.ctypes.data_as(ctypes.POINTER(_lib.KnnEdgeC)), cap, ctypes.byref(written)))
    b = buf[: written.value]
    return KnnGraph(n, int(k), EdgeList(b["u"].copy(), b["v"].copy(), b["w"].copy()))

"""Dimension-distortion sweeps: proj/include/adagio/sweep.hpp / proj/src/sweep.cpp.

Thin mirror of the reference API over the C ABI (adg_tradeoff,
adg_min_dim_for_distortion, adg_sweep_csv): the cloud stays on the device for
the whole sweep, every cell is one fused transform plus the max-only
distortion evaluator (paper_1609_05388_b200/csrc/adg_sweep.cu).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .api import PairSampling, _ctx_for, _data, _matrix

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


class Method(enum.IntEnum):
    """proj/include/adagio/sweep.hpp:12 (same order as adg_method)."""
    adagio_exact = 0
    adagio_randomized = 1
    pca = 2
    jl = 3
    external = 4


def method_name(method: Method) -> str:
    """proj/src/sweep.cpp:142-150"""
    return _lib.load().adg_method_name(int(method)).decode()


def method_from_name(name: str) -> Method:
    """proj/src/sweep.cpp:152-159 (unknown names -> InvalidArgument)."""
    out = ctypes.c_int32()
    _lib.check(_lib.load().adg_method_from_name(name.encode(), ctypes.byref(out)))
    return Method(out.value)


@dataclass
class SweepRow:
    """proj/include/adagio/sweep.hpp:19-28"""
    method: Method
    target_dim: int
    seed: int
    max_distortion: float
    fit_seconds: float
    eval_seconds: float


@dataclass
class MinDimResult:
    """proj/include/adagio/sweep.hpp:38-43"""
    target_dim: int
    achieved_distortion: float
    achieved: bool
    monotone: bool
    # instrumentation (not in the reference): dimensions probed, and how many
    # were re-evaluated exactly because their [L, U] bracket could not decide
    probes: int = field(default=0, compare=False)
    probes_refined: int = field(default=0, compare=False)


def _mode(mode: Optional[PairSampling]):
    mode = mode or PairSampling.all()
    return _lib.PairSamplingC(1 if mode.all_pairs else 0, 0, int(mode.m), int(mode.seed) & (2**64 - 1))


def tradeoff(cloud, dims: Sequence[int], methods: Sequence[Method], seeds: Sequence[int],
             eval_mode: Optional[PairSampling] = None, external_map=None) -> List[SweepRow]:
    """proj/src/sweep.cpp:161-201: one row per (method, dim, seed); method
    external evaluates external_map (r x d) once per seed, ignoring dims."""
    x = _matrix(_data(cloud))
    n, d = x.shape
    ctx, _ = _ctx_for(x)
    dims_a = np.ascontiguousarray(np.asarray(list(dims), np.int64))
    meth_a = np.ascontiguousarray(np.asarray([int(m) for m in methods], np.int32))
    seed_a = np.ascontiguousarray(np.asarray([int(s) & (2**64 - 1) for s in seeds], np.uint64))
    ext, er, ec = None, 0, 0
    if external_map is not None:
        if torch is not None and isinstance(external_map, torch.Tensor):
            ext = external_map.detach().to(torch.float64).contiguous()
        else:
            ext = np.ascontiguousarray(np.asarray(external_map, np.float64))
        er, ec = int(ext.shape[0]), int(ext.shape[1])
    count = sum((1 if int(m) == Method.external else len(dims_a)) * len(seed_a) for m in meth_a)
    rows = (_lib.SweepRowC * max(count, 1))()
    written = ctypes.c_int64()
    ps = _mode(eval_mode)
    ext_ptr = None
    if ext is not None:
        ext_ptr = ext.data_ptr() if (torch is not None and isinstance(ext, torch.Tensor)) else ext.ctypes.data
    _lib.check(_lib.load().adg_tradeoff(
        ctx, x.ptr, x.code, n, d, dims_a.ctypes.data if dims_a.size else None, len(dims_a),
        meth_a.ctypes.data if meth_a.size else None, len(meth_a),
        seed_a.ctypes.data if seed_a.size else None, len(seed_a), ctypes.byref(ps), ext_ptr, er, ec,
        rows, max(count, 1), ctypes.byref(written)))
    return [SweepRow(Method(r.method), int(r.target_dim), int(r.seed), float(r.max_distortion),
                     float(r.fit_seconds), float(r.eval_seconds)) for r in rows[: written.value]]


def min_dim_for_distortion(cloud, method: Method, delta: float, seed: int, r_min: int,
                           r_max: int) -> MinDimResult:
    """proj/src/sweep.cpp:203-265"""
    x = _matrix(_data(cloud))
    n, d = x.shape
    ctx, _ = _ctx_for(x)
    out = _lib.MinDimC()
    _lib.check(_lib.load().adg_min_dim_for_distortion(ctx, x.ptr, x.code, n, d, int(method),
                                                      float(delta), int(seed) & (2**64 - 1),
                                                      int(r_min), int(r_max), ctypes.byref(out)))
    return MinDimResult(int(out.target_dim), float(out.achieved_distortion), bool(out.achieved),
                        bool(out.monotone), int(out.probes), int(out.probes_refined))


def sweep_csv(rows: Sequence[SweepRow]) -> str:
    """proj/src/sweep.cpp:267-278"""
    arr = (_lib.SweepRowC * max(len(rows), 1))()
    for i, r in enumerate(rows):
        arr[i] = _lib.SweepRowC(int(r.method), 0, int(r.target_dim), int(r.seed) & (2**64 - 1),
                                float(r.max_distortion), float(r.fit_seconds), float(r.eval_seconds))
    L = _lib.load()
    nbytes = L.adg_sweep_csv(arr, len(rows), None, 0)
    buf = ctypes.create_string_buffer(nbytes + 1)
    L.adg_sweep_csv(arr, len(rows), buf, nbytes + 1)
    return buf.value.decode()

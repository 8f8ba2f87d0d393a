"""Python mirror of the reference's public C++ API (namespace adagio).

Same names, argument meaning, defaults and error behaviour as
proj/include/adagio/{embed,distortion,spectral,jl,dataset,rng}.hpp, backed by
libadg.so (include/adg.h): every numeric step runs in the sm_100a kernels of
this package.  Arrays may be numpy (host) or torch CUDA tensors (device,
zero-copy); results come back on the side the inputs came from.

Reference type -> here:
  PointCloud{data, labels}        -> PointCloud (data: n x d array)
  AdagioModel{mean, basis, sketch, seed, backend} -> AdagioModel
  OrthonormalBasis{rows}, SpectralSummary{singular_values, approximate}
  JlMatrix{entries, seed}, PairSampling, DistortionReport (+ argmax extension)
  std::invalid_argument -> InvalidArgument (a ValueError), NumericError, IoError.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Any, Optional

import numpy as np

from . import _lib
from ._lib import CudaError, InvalidArgument, IoError, NumericError  # noqa: F401

try:  # torch is the device-memory / stream plumbing, not the product
    import torch
except Exception:  # pragma: no cover
    torch = None


# --------------------------------------------------------------- types
class SpectralBackend(IntEnum):
    """proj/include/adagio/embed.hpp:12"""
    exact = 0
    randomized = 1


@dataclass
class PointCloud:
    """proj/include/adagio/point_cloud.hpp:20-24"""
    data: Any
    labels: Optional[list] = None

    def n(self):
        return int(self.data.shape[0])

    def d(self):
        return int(self.data.shape[1])

    def has_labels(self):
        return self.labels is not None


@dataclass
class OrthonormalBasis:
    """proj/include/adagio/spectral.hpp:11-17"""
    rows: Any

    def s(self):
        return int(self.rows.shape[0])

    def d(self):
        return int(self.rows.shape[1])


@dataclass
class SpectralSummary:
    """proj/include/adagio/spectral.hpp:21-24"""
    singular_values: Any
    approximate: bool = False


@dataclass
class JlMatrix:
    """proj/include/adagio/jl.hpp:12-18"""
    entries: Any
    seed: int = 0

    def k(self):
        return int(self.entries.shape[0])

    def d(self):
        return int(self.entries.shape[1])


@dataclass
class CenteringInfo:
    """proj/include/adagio/dataset.hpp:12-14"""
    mean: Any


@dataclass
class AdagioModel:
    """proj/include/adagio/embed.hpp:17-28"""
    mean: Any
    basis: OrthonormalBasis
    sketch: JlMatrix
    seed: int = 0
    backend: SpectralBackend = SpectralBackend.exact

    def d(self):
        return self.sketch.d()

    def s(self):
        return self.basis.s()

    def k(self):
        return self.sketch.k()

    def target_dim(self):
        return self.s() + self.k()

    def __getstate__(self):  # the cached device transform plan does not pickle
        st = dict(self.__dict__)
        st.pop("_adg_plan", None)
        return st


@dataclass
class PairSampling:
    """proj/include/adagio/distortion.hpp:16-25"""
    all_pairs: bool = True
    m: int = 0
    seed: int = 0

    @staticmethod
    def all():
        return PairSampling()

    @staticmethod
    def sample(m, seed):
        return PairSampling(False, int(m), int(seed))


@dataclass
class DistortionReport:
    """proj/include/adagio/distortion.hpp:32-42, plus argmax (lowest (i, j)
    among exact ties; None when nothing was evaluated) and engine info."""
    max_distortion: float = 0.0
    mean_distortion: float = 0.0
    histogram: Any = field(default_factory=lambda: np.zeros(0, np.uint64))
    hist_bins: int = 0
    hist_max: float = 0.0
    n_pairs_evaluated: int = 0
    n_zero_distance_pairs: int = 0
    sampled: bool = False
    sample_seed: Optional[int] = None
    argmax: Optional[tuple] = None
    engine: str = "exact"
    candidate_rows: int = 0
    screen_error_bound: float = 0.0
    edge_pairs: int = 0


# ------------------------------------------------------------ plumbing
_DT = {np.dtype(np.float64): _lib.ADG_F64, np.dtype(np.float32): _lib.ADG_F32}


class _Operand:
    """A read-only array handed to the C ABI (host numpy or device torch)."""

    def __init__(self, a, allow_bf16=True):
        self.device = None
        if torch is not None and isinstance(a, torch.Tensor):
            t = a.detach()
            if t.dtype == torch.float64:
                code = _lib.ADG_F64
            elif t.dtype == torch.float32:
                code = _lib.ADG_F32
            elif t.dtype == torch.bfloat16 and allow_bf16:
                code = _lib.ADG_BF16
            else:
                t = t.to(torch.float64)
                code = _lib.ADG_F64
            t = t.contiguous()
            self.keep = t
            self.ptr = t.data_ptr()
            self.code = code
            self.shape = tuple(t.shape)
            if t.is_cuda:
                self.device = t.device
        else:
            arr = np.asarray(a)
            if arr.dtype not in _DT:
                arr = arr.astype(np.float64)
            arr = np.ascontiguousarray(arr)
            self.keep = arr
            self.ptr = arr.ctypes.data
            self.code = _DT[arr.dtype]
            self.shape = arr.shape


def _matrix(a, name="data"):
    op = _Operand(a)
    if len(op.shape) != 2:
        raise InvalidArgument(f"{name}: expected a 2-D (n x d) array, got shape {op.shape}")
    return op


def _ctx_for(*ops):
    dev = next((o.device for o in ops if o is not None and o.device is not None), None)
    idx = dev.index if dev is not None and dev.index is not None else 0
    if dev is None and torch is not None and torch.cuda.is_available():
        idx = torch.cuda.current_device()
    ctx = _lib.context(idx)
    if dev is not None:
        s = torch.cuda.current_stream(dev).cuda_stream
        # handle 0 is the legacy default stream; NULL would mean "the context's
        # own (non-blocking) stream", which is not ordered with torch's work
        s = s or _lib.CUDA_STREAM_LEGACY
        key = ("stream", idx)
        if getattr(_ctx_for, "_streams", {}).get(key) != s:
            _lib.check(_lib.load().adg_ctx_set_stream(ctx, ctypes.c_void_p(s)))
            _ctx_for._streams = {**getattr(_ctx_for, "_streams", {}), key: s}
    return ctx, dev


def _alloc(shape, dev, dtype=np.float64):
    if dev is not None:
        tdt = torch.float64 if dtype == np.float64 else torch.float32
        t = torch.empty(shape, dtype=tdt, device=dev)
        return t, t.data_ptr()
    a = np.empty(shape, dtype=dtype)
    return a, a.ctypes.data


def _ptr(x):
    if x is None:
        return None
    if torch is not None and isinstance(x, torch.Tensor):
        return x.data_ptr()
    return x.ctypes.data


def _f64(x, dev):
    """Model constants as fp64 on the side of the data."""
    if dev is not None:
        if isinstance(x, torch.Tensor):
            return x.to(device=dev, dtype=torch.float64).contiguous()
        return torch.as_tensor(np.ascontiguousarray(x, np.float64), device=dev)
    if torch is not None and isinstance(x, torch.Tensor):
        return x.detach().cpu().to(torch.float64).numpy()
    return np.ascontiguousarray(x, np.float64)


def _data(c):
    return c.data if isinstance(c, PointCloud) else c


def _labels(c):
    return c.labels if isinstance(c, PointCloud) else None


# ------------------------------------------------------------- rng.hpp
def derive_seed(seed: int, purpose: str) -> int:
    """proj/include/adagio/rng.hpp:30-32"""
    return int(_lib.load().adg_derive_seed(seed & (2**64 - 1), purpose.encode()))


# -------------------------------------------------------------- jl.cpp
def sample_jl(k: int, d: int, seed: int, device=None) -> JlMatrix:
    """proj/src/jl.cpp:13-36 (bit-exact Rademacher entries +-1/sqrt(k))."""
    if k < 1 or d < 1:
        raise InvalidArgument("sample_jl: k and d must be >= 1")
    dev = torch.device(device) if device is not None else None
    ctx = _lib.context(dev.index or 0 if dev is not None else 0)
    out, p = _alloc((k, d), dev)
    _lib.check(_lib.load().adg_sample_jl(ctx, k, d, seed & (2**64 - 1), p))
    return JlMatrix(out, seed)


def jl_dimension(n_points: int, epsilon: float, gamma: float) -> int:
    """proj/src/jl.cpp:38-50"""
    out = ctypes.c_int64()
    _lib.check(_lib.load().adg_jl_dimension(n_points, epsilon, gamma, ctypes.byref(out)))
    return int(out.value)


# --------------------------------------------------------- dataset.cpp
def center(cloud):
    """proj/src/dataset.cpp:209-216 -> (centered PointCloud, CenteringInfo)."""
    x = _matrix(_data(cloud))
    n, d = x.shape
    ctx, dev = _ctx_for(x)
    mean, pm = _alloc((d,), dev)
    if dev is not None:
        cen = torch.empty_like(x.keep)
        pc = cen.data_ptr()
    else:
        cen = np.empty_like(x.keep)
        pc = cen.ctypes.data
    _lib.check(_lib.load().adg_center(ctx, x.ptr, x.code, n, d, pm, pc))
    return PointCloud(cen, _labels(cloud)), CenteringInfo(mean)


# -------------------------------------------------------- spectral.cpp
def exact_top_svd(cloud, s: int, n_sigma: Optional[int] = None):
    """proj/src/spectral.cpp:42-62.  n_sigma: how many singular values to
    return (default: all min(n, d), like the reference's summary)."""
    x = _matrix(_data(cloud))
    n, d = x.shape
    ctx, dev = _ctx_for(x)
    ns = min(n, d) if n_sigma is None else int(n_sigma)
    ns = max(0, min(ns, min(n, d)))
    basis, pb = _alloc((max(s, 0), d), dev)
    sig, ps = _alloc((ns,), dev)
    _lib.check(_lib.load().adg_exact_top_svd(ctx, x.ptr, x.code, n, d, s, pb,
                                             ps if ns else None, ns))
    return OrthonormalBasis(basis), SpectralSummary(sig, False)


def randomized_top_svd(cloud, s: int, oversampling: int = 10, power_iters: int = 2,
                       seed: int = 0):
    """proj/src/spectral.cpp:64-101"""
    x = _matrix(_data(cloud))
    n, d = x.shape
    ctx, dev = _ctx_for(x)
    basis, pb = _alloc((max(s, 0), d), dev)
    sig, ps = _alloc((max(s, 0),), dev)
    _lib.check(_lib.load().adg_randomized_top_svd(ctx, x.ptr, x.code, n, d, s, oversampling,
                                                  power_iters, seed & (2**64 - 1), pb, ps))
    return OrthonormalBasis(basis), SpectralSummary(sig, True)


# ----------------------------------------------------------- embed.cpp
def fit_with_split(cloud, s: int, k: int, backend=SpectralBackend.exact, seed: int = 0):
    """proj/src/embed.cpp:115-141"""
    x = _matrix(_data(cloud))
    n, d = x.shape
    ctx, dev = _ctx_for(x)
    backend = SpectralBackend(backend)
    mean, pm = _alloc((d,), dev)
    basis, pb = _alloc((max(s, 0), d), dev)
    sketch, pk = _alloc((max(k, 0), d), dev)
    _lib.check(_lib.load().adg_fit_with_split(ctx, x.ptr, x.code, n, d, s, k, int(backend),
                                              seed & (2**64 - 1), pm, pb, pk))
    return AdagioModel(mean, OrthonormalBasis(basis), JlMatrix(sketch, derive_seed(seed, "jl")),
                       seed, backend)


def fit(cloud, target_dim: int, backend=SpectralBackend.exact, seed: int = 0):
    """proj/src/embed.cpp:105-113 (s = floor(r/2), k = r - s)."""
    d = _matrix(_data(cloud)).shape[1]
    n = _matrix(_data(cloud)).shape[0]
    if target_dim < 2 or target_dim > d:
        raise InvalidArgument(f"fit: target_dim = {target_dim} outside [2, {d}]")
    if n < 2:
        raise InvalidArgument("fit: need at least 2 points")
    return fit_with_split(cloud, target_dim // 2, target_dim - target_dim // 2, backend, seed)


class _TransformPlan:
    """adg_transform_plan for one model on one device (W and its tf32 split
    prepared once); destroyed with the model."""

    def __init__(self, ctx, model, dev, code):
        mean = _f64(model.mean, dev)
        basis = _f64(model.basis.rows, dev)
        sketch = _f64(model.sketch.entries, dev)
        self.h = ctypes.c_void_p()
        self._lib = _lib.load()
        _lib.check(self._lib.adg_transform_plan_create(
            ctx, _ptr(mean), _ptr(basis) if model.s() else None, model.s(), _ptr(sketch), model.k(),
            model.d(), code, ctypes.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self._lib.adg_transform_plan_destroy(self.h)
            self.h = ctypes.c_void_p()


def _model_plan(model, ctx, dev, code):
    """The model's cached plan when its arrays are device tensors, keyed by the
    tensors' identity and version counters (the entry holds the tensors, so an
    address cannot be reused under it); None otherwise."""
    if dev is None or torch is None:
        return None
    arrays = (model.mean, model.basis.rows, model.sketch.entries)
    if not all(isinstance(a, torch.Tensor) for a in arrays):
        return None
    key = (str(dev), code == _lib.ADG_F64, tuple((id(a), a._version) for a in arrays))
    ent = model.__dict__.get("_adg_plan")
    if ent is not None and ent[0] == key:
        return ent[1]
    plan = _TransformPlan(ctx, model, dev, code)
    model.__dict__["_adg_plan"] = (key, plan, arrays)
    return plan


def transform_all(model: AdagioModel, cloud, out_dtype=None) -> PointCloud:
    """proj/src/embed.cpp:161-181 (labels carried along).  out_dtype defaults
    to float64 for fp64 input (the reference's type) and float32 otherwise."""
    x = _matrix(_data(cloud))
    n, d = x.shape
    if d != model.d():
        raise InvalidArgument(f"transform_all: cloud dimension {d}, model expects {model.d()}")
    ctx, dev = _ctx_for(x)
    if out_dtype is None:
        out_dtype = np.float64 if x.code == _lib.ADG_F64 else np.float32
    oc = _lib.ADG_F64 if out_dtype == np.float64 else _lib.ADG_F32
    y, py = _alloc((n, model.target_dim()), dev, np.float64 if oc == _lib.ADG_F64 else np.float32)
    plan = _model_plan(model, ctx, dev, x.code)
    if plan is not None:
        _lib.check(_lib.load().adg_transform_plan_run(plan.h, x.ptr, x.code, n, py, oc))
        return PointCloud(y, _labels(cloud))
    mean = _f64(model.mean, dev)
    basis = _f64(model.basis.rows, dev)
    sketch = _f64(model.sketch.entries, dev)
    _lib.check(_lib.load().adg_transform_all(ctx, _ptr(mean), _ptr(basis) if model.s() else None,
                                             model.s(), _ptr(sketch), model.k(), d, x.ptr, x.code,
                                             n, py, oc))
    return PointCloud(y, _labels(cloud))


def save_model(model: AdagioModel, path: str) -> None:
    """proj/src/embed.cpp:183-202: ADG1 little-endian model file, bit-exact."""
    import struct
    mean = np.ascontiguousarray(_host64(model.mean), "<f8")
    P = np.ascontiguousarray(_host64(model.basis.rows), "<f8").reshape(model.s(), model.d())
    S = np.ascontiguousarray(_host64(model.sketch.entries), "<f8")
    try:
        with open(path, "wb") as f:
            f.write(b"ADG1" + struct.pack("<IIIIBQ", 1, model.d(), model.s(), model.k(),
                                          int(model.backend), int(model.seed) & (2**64 - 1)))
            f.write(mean.tobytes() + P.tobytes() + S.tobytes())
    except OSError as e:
        raise IoError(f"model: cannot write {path}") from e


def load_model(path: str) -> AdagioModel:
    """proj/src/embed.cpp:204-239 (same validation and messages)."""
    import struct
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError as e:
        raise IoError(f"model: cannot open {path}") from e
    if len(blob) < 4 or blob[:4] != b"ADG1":
        raise IoError(f"model: bad magic in {path}")
    if len(blob) < 8:
        raise IoError(f"model: truncated file {path}")
    (version,) = struct.unpack_from("<I", blob, 4)
    if version != 1:
        raise IoError(f"model: unsupported version {version} in {path}")
    if len(blob) < 20:
        raise IoError(f"model: truncated file {path}")
    d, s, k = struct.unpack_from("<III", blob, 8)
    if d == 0 or k == 0:
        raise IoError(f"model: invalid dimensions in {path}")
    if len(blob) < 21:
        raise IoError(f"model: truncated file {path}")
    tag = blob[20]
    if tag > 1:
        raise IoError(f"model: unknown backend tag in {path}")
    need = 29 + 8 * (d + s * d + k * d)
    if len(blob) < need:
        raise IoError(f"model: truncated file {path}")
    (seed,) = struct.unpack_from("<Q", blob, 21)
    vals = np.frombuffer(blob, "<f8", d + s * d + k * d, 29).astype(np.float64)
    mean, P, S = vals[:d].copy(), vals[d:d + s * d].reshape(s, d).copy(), vals[d + s * d:].reshape(k, d).copy()
    return AdagioModel(mean, OrthonormalBasis(P), JlMatrix(S, derive_seed(seed, "jl")), int(seed),
                       SpectralBackend(tag))


def _host64(x):
    if torch is not None and isinstance(x, torch.Tensor):
        return x.detach().cpu().to(torch.float64).numpy()
    return np.asarray(x, np.float64)


def transform(model: AdagioModel, w):
    """proj/src/embed.cpp:143-159 (one vector)."""
    w_arr = w if (torch is not None and isinstance(w, torch.Tensor)) else np.asarray(w, np.float64)
    if w_arr.shape[-1] != model.d() or len(w_arr.shape) != 1:
        raise InvalidArgument(f"transform: vector has dimension {w_arr.shape[-1]}, model expects "
                              f"{model.d()}")
    return transform_all(model, w_arr.reshape(1, -1), out_dtype=np.float64).data.reshape(-1)


# ------------------------------------------------------ distortion.cpp
_ENGINE_NAMES = {0: "auto", 1: "exact", 2: "screen", 3: "screen_exact_hist"}


def _report(rep: _lib.Report, hist) -> DistortionReport:
    am = None if rep.argmax_i == 2**64 - 1 else (int(rep.argmax_i), int(rep.argmax_j))
    return DistortionReport(rep.max_distortion, rep.mean_distortion, hist, rep.hist_bins,
                            rep.hist_max, int(rep.n_pairs_evaluated),
                            int(rep.n_zero_distance_pairs), bool(rep.sampled),
                            int(rep.sample_seed) if rep.sampled else None, am,
                            _ENGINE_NAMES.get(rep.engine, "?"), int(rep.candidate_rows),
                            float(rep.screen_error_bound), int(rep.edge_pairs))


def evaluate(original, embedded, mode: PairSampling = None, hist_bins: int = 50,
             hist_max: float = 1.0, pairs_per_block: int = 16384, engine: str = "auto"):
    """proj/src/distortion.cpp:113-192.  engine: "auto" | "exact" | "screen" |
    "screen_exact_hist" (include/adg.h adg_engine)."""
    mode = mode or PairSampling.all()
    x = _matrix(_data(original), "original")
    y = _matrix(_data(embedded), "embedded")
    ctx, _ = _ctx_for(x, y)
    rep = _lib.Report()
    hist = np.zeros(max(hist_bins, 1) + 1, np.uint64)
    ps = _lib.PairSamplingC(1 if mode.all_pairs else 0, 0, int(mode.m), int(mode.seed) & (2**64 - 1))
    _lib.check(_lib.load().adg_evaluate(ctx, x.ptr, x.code, x.shape[0], x.shape[1], y.ptr, y.code,
                                        y.shape[0], y.shape[1], ctypes.byref(ps), hist_bins,
                                        float(hist_max), pairs_per_block, _lib.ENGINES[engine],
                                        ctypes.byref(rep), hist.ctypes.data))
    return _report(rep, hist[: hist_bins + 1])


def distort_model(model: AdagioModel, original, mode: PairSampling = None, hist_bins: int = 50,
                  hist_max: float = 1.0, engine: str = "auto", return_embedded: bool = False,
                  out_dtype=None):
    """proj/tools/adagio_main.cpp:192-224 (run_distort --model): evaluate(original,
    transform_all(model, original), mode, hist_bins, hist_max) with the original
    staged to the device once and the embedding kept in HBM (adg_distort_model).
    Returns the report, or (report, embedded PointCloud) with return_embedded."""
    mode = mode or PairSampling.all()
    x = _matrix(_data(original), "original")
    n, d = x.shape
    if d != model.d():
        raise InvalidArgument(f"transform_all: cloud dimension {d}, model expects {model.d()}")
    ctx, dev = _ctx_for(x)
    if out_dtype is None:
        out_dtype = np.float64 if x.code == _lib.ADG_F64 else np.float32
    oc = _lib.ADG_F64 if out_dtype == np.float64 else _lib.ADG_F32
    mean = _f64(model.mean, dev)
    basis = _f64(model.basis.rows, dev)
    sketch = _f64(model.sketch.entries, dev)
    y, py = (None, None)
    if return_embedded:
        y, py = _alloc((n, model.target_dim()), dev, np.float64 if oc == _lib.ADG_F64 else np.float32)
    rep = _lib.Report()
    hist = np.zeros(max(hist_bins, 1) + 1, np.uint64)
    ps = _lib.PairSamplingC(1 if mode.all_pairs else 0, 0, int(mode.m), int(mode.seed) & (2**64 - 1))
    _lib.check(_lib.load().adg_distort_model(
        ctx, _ptr(mean), _ptr(basis) if model.s() else None, model.s(), _ptr(sketch), model.k(), d,
        x.ptr, x.code, n, ctypes.byref(ps), hist_bins, float(hist_max), _lib.ENGINES[engine],
        ctypes.byref(rep), hist.ctypes.data, py, oc))
    report = _report(rep, hist[: hist_bins + 1])
    return (report, PointCloud(y, _labels(original))) if return_embedded else report


def max_distortion(original, embedded) -> float:
    """proj/src/distortion.cpp:194-196 (adg_max_distortion: all pairs; large
    jobs run the max-only SCREEN evaluator, same value as evaluate().max)."""
    x = _matrix(_data(original), "original")
    y = _matrix(_data(embedded), "embedded")
    if x.shape[0] != y.shape[0]:
        raise InvalidArgument(f"evaluate: cloud sizes differ ({x.shape[0]} vs {y.shape[0]})")
    ctx, _ = _ctx_for(x, y)
    out = ctypes.c_double()
    _lib.check(_lib.load().adg_max_distortion(ctx, x.ptr, x.code, x.shape[0], x.shape[1], y.ptr,
                                              y.code, y.shape[1], ctypes.byref(out)))
    return float(out.value)


def pair_distortion(x, y, fx, fy) -> float:
    """proj/src/distortion.cpp:107-111 (coincident points -> InvalidArgument)."""
    xs = [np.ascontiguousarray(np.asarray(v, np.float64).reshape(-1)) for v in (x, y, fx, fy)]
    ctx = _lib.context(0)
    out = ctypes.c_double()
    _lib.check(_lib.load().adg_pair_distortion(ctx, xs[0].ctypes.data, xs[1].ctypes.data,
                                               xs[0].size, xs[2].ctypes.data, xs[3].ctypes.data,
                                               xs[2].size, ctypes.byref(out)))
    return float(out.value)


def _to_c_report(r: DistortionReport):
    rep = _lib.Report()
    rep.max_distortion, rep.mean_distortion = r.max_distortion, r.mean_distortion
    rep.n_pairs_evaluated, rep.n_zero_distance_pairs = r.n_pairs_evaluated, r.n_zero_distance_pairs
    rep.hist_bins, rep.hist_max, rep.sampled = r.hist_bins, r.hist_max, int(r.sampled)
    rep.sample_seed = r.sample_seed or 0
    rep.argmax_i, rep.argmax_j = r.argmax if r.argmax else (2**64 - 1, 2**64 - 1)
    h = np.ascontiguousarray(r.histogram, np.uint64)
    return rep, h


def report_to_json(report: DistortionReport) -> dict:
    """proj/src/distortion.cpp:198-215 (all fields of distort.schema.json)."""
    rep, h = _to_c_report(report)
    L = _lib.load()
    n = L.adg_report_to_json(ctypes.byref(rep), h.ctypes.data, None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    L.adg_report_to_json(ctypes.byref(rep), h.ctypes.data, buf, n + 1)
    return json.loads(buf.value.decode())


def histogram_csv(report: DistortionReport) -> str:
    """proj/src/distortion.cpp:217-230"""
    rep, h = _to_c_report(report)
    L = _lib.load()
    n = L.adg_histogram_csv(ctypes.byref(rep), h.ctypes.data, None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    L.adg_histogram_csv(ctypes.byref(rep), h.ctypes.data, buf, n + 1)
    return buf.value.decode()


def kernel_launch_count(device: int = 0) -> int:
    return int(_lib.load().adg_kernel_launch_count(_lib.context(device)))


def last_knn_engine(device: int = 0) -> str:
    """Engine of the last k-NN call: "none", "simt" or "tensor"."""
    return ("none", "simt", "tensor")[int(_lib.load().adg_last_knn_engine(_lib.context(device)))]


def last_screen_kernel_ms(device: int = 0) -> float:
    return float(_lib.load().adg_last_screen_kernel_ms(_lib.context(device)))


def last_screen_orig_passes(device: int = 0) -> int:
    """MMA passes of the last SCREEN evaluation over the original coordinates
    (1: exact fp16 planes, e.g. nearly centred bf16 input; 3: split)."""
    return int(_lib.load().adg_last_screen_orig_passes(_lib.context(device)))

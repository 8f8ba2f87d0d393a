"""The C-ABI library without a GPU: it loads, exports every symbol include/adg.h
declares, its host-side helpers agree with the oracle, and compute entry
points fail loudly (no CPU fallback) when no device is present."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import _lib
from paper_1609_05388_b200 import datasets as ds

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# proj/docs/schemas/distort.schema.json required keys (distortion.cpp:198-215)
DISTORT_KEYS = ["max_distortion", "mean_distortion", "hist_bins", "hist_max", "histogram",
                "n_pairs_evaluated", "n_zero_distance_pairs", "sampled", "sample_seed"]


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "adg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adg_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    L = _lib.load()
    decl = declared_symbols()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTS) == decl


def test_abi_version_and_seeds(oracle):
    L = _lib.load()
    assert L.adg_abi_version() == 2
    for seed in [0, 1, 99, 2**64 - 1]:
        for purpose in ["jl", "spectral", "sampling"]:
            assert adg.derive_seed(seed, purpose) == oracle.derive_seed(seed, purpose)


def test_jl_dimension_host(oracle):
    assert adg.jl_dimension(800, 0.2, 0.01) == 4148
    assert adg.jl_dimension(400, 0.5, 0.01) == 797
    assert adg.jl_dimension(100, 0.3, 0.05) == 1357
    with pytest.raises(adg.InvalidArgument, match="epsilon"):
        adg.jl_dimension(10, 1.0, 0.01)
    with pytest.raises(ValueError):
        adg.jl_dimension(1, 0.3, 0.01)


def test_report_json_and_csv_layout():
    rep = adg.DistortionReport(0.25, 0.125, np.array([3, 2, 1, 0, 0, 1], np.uint64), 5, 1.0, 7, 2,
                               False, None, (1, 4))
    j = adg.report_to_json(rep)
    for k in DISTORT_KEYS:
        assert k in j
    assert j["sample_seed"] is None and len(j["histogram"]) == 6
    assert j["argmax_i"] == 1 and j["argmax_j"] == 4
    csv = adg.histogram_csv(rep)
    assert csv.startswith("bin_left,bin_right,count\n")
    assert csv.count("\n") == 7 and "inf" in csv
    rep.sampled, rep.sample_seed = True, 123
    assert adg.report_to_json(rep)["sample_seed"] == 123


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    x = np.zeros((4, 3))
    with pytest.raises(adg.CudaError):
        adg.evaluate(x, x)
    with pytest.raises(adg.CudaError):
        adg.sample_jl(2, 3, 0)


def test_partials_struct_matches_header():
    src = open(os.path.join(ROOT, "include", "adg.h")).read()
    body = src[src.index("typedef struct {\n  uint64_t* hist;"):src.index("} adg_eval_partials;")]
    fields = re.findall(r"\b([a-z_]+);", body)
    assert fields == [f for f, _ in _lib.Partials._fields_]
    rep_body = src[src.index("typedef struct {\n  double max_distortion;"):src.index("} adg_report;")]
    rfields = re.findall(r"\b([a-z_]+);", rep_body)
    assert rfields == [f for f, _ in _lib.Report._fields_]


def test_datasets_shapes_and_determinism():
    a = ds.c1_low_rank()
    b = ds.c1_low_rank()
    assert a.shape == (2000, 256) and a.dtype == np.float32 and np.array_equal(a, b)
    c = ds.c2_blobs()
    assert c.shape == (1000, 256) and abs(float(c.max()) - 1.0) < 0.05
    x = ds.c3_mnist_like(n=512)
    assert x.shape == (512, 784) and x.min() >= 0.0 and x.max() <= 1.0
    img = x.reshape(-1, 28, 28)
    assert np.all(img[:, :4, :] == 0) and np.all(img[:, 24:, :] == 0)

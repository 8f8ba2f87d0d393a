"""B200-native ADAgIO hot path: fit -> embed -> all-pairs distortion.

Drop-in for the reference's C++ API (proj/include/adagio/*.hpp) through the
C ABI in include/adg.h (libadg.so, hand-written sm_100a CUDA).  The Python
surface in api.py mirrors the reference's names; dist.py shards the
distortion evaluator across GPUs with torch.distributed (NCCL).
"""
from .api import (  # noqa: F401
    AdagioModel, CenteringInfo, CudaError, DistortionReport, InvalidArgument, IoError, JlMatrix,
    NumericError, OrthonormalBasis, PairSampling, PointCloud, SpectralBackend, SpectralSummary,
    center, derive_seed, distort_model, evaluate, exact_top_svd, fit, fit_with_split, histogram_csv,
    jl_dimension, load_model, max_distortion, pair_distortion, randomized_top_svd, report_to_json,
    save_model,
    sample_jl, transform, transform_all)
from .sweep import (  # noqa: F401
    MinDimResult, Method, SweepRow, method_from_name, method_name, min_dim_for_distortion,
    sweep_csv, tradeoff)
from .downstream import (  # noqa: F401
    Edge, EdgeWeighting, KnnGraph, build_knn_graph, knn_query, knn_query_batch, majority_classify)
from .dataset_io import csv_string, load_csv, load_idx, sample_points, save_csv  # noqa: F401

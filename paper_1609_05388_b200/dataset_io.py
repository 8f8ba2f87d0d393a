"""Data formats around the path: proj/include/adagio/dataset.hpp I/O,
restated from proj/src/dataset.cpp:20-245 (host code -- parsing and file
formats, no device work).

* load_csv / csv_string / save_csv: the reference's CSV dialect (fields
  trimmed of blanks, optional header, optional label column, %.17g so a
  reload is bit-exact) with its IoError messages.  Numbers follow
  std::from_chars' general syntax (no leading '+', no '_' separators);
  Python's float() then gives the same correctly rounded double.
* load_idx: MNIST IDX (big-endian magic 0x00000803 / 0x00000801).
* sample_points: partial Fisher-Yates with SeededRng.below (rng.hpp).
"""
from __future__ import annotations

import math
import re
import struct
from typing import Optional

import numpy as np

from .api import InvalidArgument, IoError, PointCloud

_NUM = re.compile(r"-?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?\Z")
_SPECIAL = re.compile(r"-?(?:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)\Z", re.IGNORECASE)


def _trim(s: str) -> str:
    """proj/src/dataset.cpp:21-25"""
    return s.lstrip(" \t").rstrip(" \t\r")


def _field(f: str, row: int, col: int) -> float:
    """proj/src/dataset.cpp:38-52"""
    if _SPECIAL.match(f):
        raise IoError(f"csv: non-finite value at row {row}, column {col}")
    if not f or not _NUM.match(f):
        raise IoError(f"csv: non-numeric field '{f}' at row {row}, column {col}")
    v = float(f)
    if not math.isfinite(v):  # overflow to inf
        raise IoError(f"csv: non-finite value at row {row}, column {col}")
    return v


def load_csv(path: str, has_header: bool = False, label_column: Optional[int] = None) -> PointCloud:
    """proj/src/dataset.cpp:72-121"""
    try:
        fh = open(path, "r", newline="")
    except OSError as e:
        raise IoError(f"csv: cannot open {path}") from e
    rows, labels = [], []
    expected = 0
    with fh:
        for line_no, line in enumerate(fh, start=1):
            line = line.rstrip("\n")
            if has_header and line_no == 1:
                continue
            if not _trim(line):
                continue
            fields = [_trim(f) for f in line.split(",")]
            if expected == 0:
                expected = len(fields)
                if label_column is not None and not (0 <= label_column < expected):
                    raise IoError(f"csv: label column {label_column} out of range for {expected} columns")
            elif len(fields) != expected:
                raise IoError(f"csv: row {line_no} has {len(fields)} fields, expected {expected}")
            row = []
            for c, f in enumerate(fields):
                v = _field(f, line_no, c + 1)
                if label_column is not None and c == label_column:
                    if v < 0.0 or v != math.floor(v) or v > 2147483647.0:
                        raise IoError(f"csv: label must be a non-negative integer at row {line_no}, "
                                      f"column {c + 1}")
                    labels.append(int(v))
                else:
                    row.append(v)
            rows.append(row)
    if not rows:
        raise IoError(f"csv: no data rows in {path}")
    if not rows[0]:
        raise IoError(f"csv: no feature columns in {path}")
    return PointCloud(np.asarray(rows, np.float64), labels if label_column is not None else None)


def csv_string(cloud: PointCloud, with_labels: bool = True) -> str:
    """proj/src/dataset.cpp:123-141 (%.17g: a reload is bit-exact)."""
    data = np.asarray(cloud.data, np.float64) if not hasattr(cloud.data, "cpu") else \
        cloud.data.detach().cpu().double().numpy()
    emit = with_labels and cloud.labels is not None
    out = []
    for i in range(data.shape[0]):
        line = ",".join("%.17g" % v for v in data[i])
        if emit:
            line += "," + str(int(cloud.labels[i]))
        out.append(line + "\n")
    return "".join(out)


def save_csv(cloud: PointCloud, path: str, with_labels: bool = True) -> None:
    """proj/src/dataset.cpp:143-148"""
    try:
        with open(path, "w", newline="") as f:
            f.write(csv_string(cloud, with_labels))
    except OSError as e:
        raise IoError(f"csv: cannot write {path}") from e


def _be_u32(fh, path):
    b = fh.read(4)
    if len(b) != 4:
        raise IoError(f"idx: truncated header in {path}")
    return struct.unpack(">I", b)[0]


def load_idx(images_path: str, labels_path: Optional[str] = None) -> PointCloud:
    """proj/src/dataset.cpp:150-207"""
    try:
        fh = open(images_path, "rb")
    except OSError as e:
        raise IoError(f"idx: cannot open {images_path}") from e
    with fh:
        if _be_u32(fh, images_path) != 0x00000803:
            raise IoError(f"idx: wrong magic in {images_path} (expected 0x00000803)")
        count, rows, cols = (_be_u32(fh, images_path) for _ in range(3))
        if count == 0 or rows == 0 or cols == 0:
            raise IoError(f"idx: empty image file {images_path}")
        pixels = count * rows * cols
        payload = fh.read(pixels)
        if len(payload) != pixels:
            raise IoError(f"idx: truncated image payload in {images_path}")
    data = np.frombuffer(payload, np.uint8).reshape(count, rows * cols).astype(np.float64)
    labels = None
    if labels_path is not None:
        try:
            lf = open(labels_path, "rb")
        except OSError as e:
            raise IoError(f"idx: cannot open {labels_path}") from e
        with lf:
            if _be_u32(lf, labels_path) != 0x00000801:
                raise IoError(f"idx: wrong magic in {labels_path} (expected 0x00000801)")
            lcount = _be_u32(lf, labels_path)
            if lcount != count:
                raise IoError(f"idx: image/label count mismatch ({count} images, {lcount} labels)")
            lb = lf.read(lcount)
            if len(lb) != lcount:
                raise IoError(f"idx: truncated label payload in {labels_path}")
        labels = [int(v) for v in lb]
    return PointCloud(data, labels)


def _rng(seed):
    state = [seed & (2**64 - 1)]
    M = 2**64 - 1

    def nxt():
        state[0] = (state[0] + 0x9E3779B97F4A7C15) & M
        z = state[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    def below(bound):
        limit = (bound * (M // bound)) & M
        v = nxt()
        while v >= limit:
            v = nxt()
        return v % bound

    return below


def sample_points(cloud: PointCloud, m: int, seed: int) -> PointCloud:
    """proj/src/dataset.cpp:218-245"""
    data = cloud.data
    n = int(data.shape[0])
    if m < 1 or m > n:
        raise InvalidArgument(f"sample_points: m = {m} outside [1, {n}]")
    index = list(range(n))
    below = _rng(seed)
    for i in range(m):
        off = below(n - i)
        index[i], index[i + off] = index[i + off], index[i]
    pick = index[:m]
    if hasattr(data, "index_select"):
        import torch
        out = data.index_select(0, torch.as_tensor(pick, device=data.device))
    else:
        out = np.asarray(data)[pick]
    labels = [cloud.labels[i] for i in pick] if cloud.labels is not None else None
    return PointCloud(out, labels)

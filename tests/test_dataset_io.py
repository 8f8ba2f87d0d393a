"""Data formats either side of the path (proj/src/dataset.cpp:20-245), CPU
only: the Python mirror and the C++ facade (include/adagio_b200.hpp) read and
write the same files with the reference's rules and messages, mirroring
proj/tests/test_dataset.cpp (CSV round trip bit-exact, header/label column,
ragged / non-numeric / non-finite rejection with positions, IDX parsing,
sample_points determinism).
"""
import os
import struct
import subprocess

import numpy as np
import pytest

import paper_1609_05388_b200 as adg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_csv_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    data = rng.standard_normal((7, 5)) * 10.0 ** rng.integers(-30, 30, (7, 5))
    data[0, 0] = 0.1
    data[1, 1] = -0.0
    cloud = adg.PointCloud(data, [3, 0, 1, 4, 1, 5, 9])
    p = str(tmp_path / "c.csv")
    adg.save_csv(cloud, p)
    back = adg.load_csv(p, label_column=5)
    assert np.array_equal(back.data.view(np.uint64), data.view(np.uint64))
    assert back.labels == cloud.labels
    assert adg.csv_string(adg.PointCloud(data[:1, :2])) == "0.10000000000000001,%.17g\n" % data[0, 1]


def test_csv_header_blank_lines_and_trim(tmp_path):
    p = tmp_path / "h.csv"
    p.write_text("a,b,label\n 1.5 ,\t2,0\r\n\n3,4e2 , 7\n")
    c = adg.load_csv(str(p), has_header=True, label_column=2)
    assert c.data.tolist() == [[1.5, 2.0], [3.0, 400.0]] and c.labels == [0, 7]


@pytest.mark.parametrize("text,msg", [
    ("1,2\n3\n", "csv: row 2 has 1 fields, expected 2"),
    ("1,x\n", "csv: non-numeric field 'x' at row 1, column 2"),
    ("1,+2\n", "csv: non-numeric field '+2' at row 1, column 2"),
    ("1,\n", "csv: non-numeric field '' at row 1, column 2"),
    ("1,inf\n", "csv: non-finite value at row 1, column 2"),
    ("nan,1\n", "csv: non-finite value at row 1, column 1"),
    ("1,1e400\n", "csv: non-finite value at row 1, column 2"),
    ("\n \n", "csv: no data rows in"),
])
def test_csv_rejections(tmp_path, text, msg):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(adg.IoError, match=msg.replace("+", r"\+")):
        adg.load_csv(str(p))


def test_csv_label_rules(tmp_path):
    p = tmp_path / "l.csv"
    p.write_text("1,2.5\n")
    with pytest.raises(adg.IoError, match="label must be a non-negative integer at row 1, column 2"):
        adg.load_csv(str(p), label_column=1)
    with pytest.raises(adg.IoError, match="label column 2 out of range for 2 columns"):
        adg.load_csv(str(p), label_column=2)
    p.write_text("3\n")
    with pytest.raises(adg.IoError, match="no feature columns"):
        adg.load_csv(str(p), label_column=0)
    with pytest.raises(adg.IoError, match="cannot open"):
        adg.load_csv(str(tmp_path / "missing.csv"))


def _write_idx(tmp_path, count=3, rows=2, cols=2, magic=0x803, lmagic=0x801, lcount=None):
    img = tmp_path / "img.idx"
    lab = tmp_path / "lab.idx"
    pix = bytes(range(count * rows * cols))
    img.write_bytes(struct.pack(">IIII", magic, count, rows, cols) + pix)
    lab.write_bytes(struct.pack(">II", lmagic, count if lcount is None else lcount) + bytes(range(count)))
    return str(img), str(lab)


def test_idx(tmp_path):
    img, lab = _write_idx(tmp_path)
    c = adg.load_idx(img, lab)
    assert c.data.shape == (3, 4) and c.data[2].tolist() == [8.0, 9.0, 10.0, 11.0] and c.labels == [0, 1, 2]
    img, _ = _write_idx(tmp_path, magic=0x802)
    with pytest.raises(adg.IoError, match="wrong magic"):
        adg.load_idx(img)
    img, lab = _write_idx(tmp_path, lcount=2)
    with pytest.raises(adg.IoError, match=r"image/label count mismatch \(3 images, 2 labels\)"):
        adg.load_idx(img, lab)


def test_sample_points():
    c = adg.PointCloud(np.arange(40, dtype=np.float64).reshape(20, 2), list(range(20)))
    a = adg.sample_points(c, 7, 11)
    b = adg.sample_points(c, 7, 11)
    assert np.array_equal(a.data, b.data) and a.labels == b.labels
    assert len(set(a.labels)) == 7 and all(a.data[i, 0] == 2 * a.labels[i] for i in range(7))
    with pytest.raises(ValueError, match=r"sample_points: m = 21 outside \[1, 20\]"):
        adg.sample_points(c, 21, 0)


CPP = r'''
#include "adagio_b200.hpp"
#include <iostream>
int main(int argc, char** argv) {
  adagio::PointCloud c = adagio::load_csv(argv[1], false, 5);
  adagio::save_csv(c, argv[2]);
  adagio::PointCloud s = adagio::sample_points(c, 4, 11);
  for (int i = 0; i < 4; ++i) std::cout << (*s.labels)[i] << " ";
  std::cout << "\n";
  try { adagio::load_csv(argv[3]); } catch (const adagio::IoError& e) { std::cout << e.what() << "\n"; }
  adagio::PointCloud m = adagio::load_idx(argv[4], std::string(argv[5]));
  std::cout << m.n() << " " << m.d() << " " << m.data(2, 3) << " " << (*m.labels)[2] << "\n";
  return 0;
}
'''


def test_cpp_facade_io_matches_python(tmp_path):
    src = tmp_path / "io.cpp"
    src.write_text(CPP)
    exe = str(tmp_path / "io")
    libdir = os.path.join(ROOT, "paper_1609_05388_b200")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), str(src),
                           "-L", libdir, "-ladg", f"-Wl,-rpath,{libdir}", "-o", exe])
    rng = np.random.default_rng(5)
    data = rng.standard_normal((9, 5)) * 1e3
    cloud = adg.PointCloud(data, [int(v) for v in rng.integers(0, 50, 9)])
    a = str(tmp_path / "a.csv")
    adg.save_csv(cloud, a)
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2\n3,x\n")
    img, lab = _write_idx(tmp_path)
    out = subprocess.run([exe, a, str(tmp_path / "b.csv"), str(bad), img, lab], capture_output=True,
                         text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.splitlines()
    assert (tmp_path / "b.csv").read_text() == open(a).read()  # byte-identical re-serialisation
    assert [int(v) for v in lines[0].split()] == adg.sample_points(cloud, 4, 11).labels
    assert lines[1] == "csv: non-numeric field 'x' at row 2, column 2"
    assert lines[2] == "3 4 11 2"

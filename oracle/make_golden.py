"""Freeze golden vectors for the GPU box (TEST INFRASTRUCTURE ONLY).

rng_golden.json: output of the reference's own rng.hpp (compiled from
/root/reference by `make -C oracle ref`), so tests can pin both the oracle
restatement and the CUDA counter-hash / Box-Muller kernels bit-for-bit without
the reference being present.  Run here (the reference is mounted only in this
container):  python oracle/make_golden.py
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main():
    subprocess.check_call(["make", "-s", "-C", HERE, "ref"])
    out = subprocess.check_output([os.path.join(HERE, "_ref", "ref_rng")]).decode()
    doc = json.loads(out)
    doc["_provenance"] = ("printed by oracle/ref_rng_driver.cpp compiled against "
                          "/root/reference/proj/include/adagio/rng.hpp (unmodified)")
    path = os.path.join(ROOT, "tests", "golden", "rng_golden.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    sys.exit(main())

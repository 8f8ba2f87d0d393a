import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1609_05388_b200 import _lib
from oracle import oracle
X = oracle.gaussian_cloud(6000, 48, 4).astype(np.float32)
Y = (X.astype(np.float64) @ oracle.sample_jl(12, 48, 5).T).astype(np.float32)
L = _lib.load()
rep = _lib.Report()
hist = np.zeros(51, np.uint64)
devs = (ctypes.c_int32 * 1)(0)
print("calling", flush=True)
st = L.adg_evaluate_multi(1, devs, X.ctypes.data, _lib.ADG_F32, X.shape[0], X.shape[1],
                          Y.ctypes.data, _lib.ADG_F32, Y.shape[0], Y.shape[1], None, 50,
                          1.0, _lib.ENGINES["screen"], ctypes.byref(rep), hist.ctypes.data)
print("status", st, rep.max_distortion, flush=True)
comms = (_lib.Collectives * 1)()
print("nccl", L.adg_comm_nccl_create_all(1, devs, comms), flush=True)
print(L.adg_last_error())

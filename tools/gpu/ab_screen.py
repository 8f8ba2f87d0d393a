"""A/B of the screen kernel time between two builds of libadg.so (profiling
aid): C3 job (X, Y on the device), adg_evaluate SCREEN, median of the
CUDA-event screen-kernel times, builds alternated in separate processes."""
import ctypes, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def child(lib, reps, engine):
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from paper_1609_05388_b200 import datasets as ds
    L = ctypes.CDLL(lib)
    P, i64 = ctypes.c_void_p, ctypes.c_int64
    L.adg_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
    L.adg_evaluate.argtypes = [P, P, ctypes.c_int, i64, i64, P, ctypes.c_int, i64, i64, P,
                               ctypes.c_int, ctypes.c_double, ctypes.c_uint64, ctypes.c_int, P, P]
    L.adg_last_screen_kernel_ms.restype = ctypes.c_double
    L.adg_last_screen_kernel_ms.argtypes = [P]
    L.adg_ctx_set_stream.argtypes = [P, P]
    ctx = P()
    assert L.adg_ctx_create(0, ctypes.byref(ctx)) == 0
    L.adg_ctx_set_stream(ctx, P(1))
    X = torch.from_numpy(ds.c3_mnist_like()).cuda()
    W = torch.randn(784, 50, device="cuda", dtype=torch.float64) / 28
    Y = (X.double() @ W).float().contiguous()
    rep = (ctypes.c_uint8 * 256)()
    hist = np.zeros(51, np.uint64)
    flush = torch.empty(64 << 20, device="cuda")
    ts = []
    for k in range(reps + 2):
        flush.zero_()
        st = L.adg_evaluate(ctx, X.data_ptr(), 1, 60000, 784, Y.data_ptr(), 1, 60000, 50, None, 50, 1.0,
                            16384, engine, ctypes.byref(rep), hist.ctypes.data)
        assert st == 0, st
        if k >= 2:
            ts.append(L.adg_last_screen_kernel_ms(ctx))
    ts.sort()
    print(json.dumps({"lib": os.path.basename(lib), "engine": engine, "median_ms": ts[len(ts) // 2],
                      "min_ms": ts[0]}), flush=True)

if __name__ == "__main__":
    if sys.argv[1] == "child":
        child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    else:
        libs = sys.argv[1:]
        for rnd in range(3):
            for lib in libs:
                eng = 2
                if ":" in lib:
                    lib, eng = lib.split(":")
                subprocess.run([sys.executable, __file__, "child", lib, "15", str(eng)])

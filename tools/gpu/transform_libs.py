"""Cold-L2 transform_all time per library build (profiling aid): ADG_LIB per child."""
import os, sys, subprocess, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import torch
    import paper_1609_05388_b200 as adg
    from paper_1609_05388_b200 import datasets as ds
    X = torch.from_numpy(ds.c3_mnist_like()).cuda()
    m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(15):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); adg.transform_all(m, X); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(os.environ.get("ADG_LIB", "default"), "ms median %.4f" % statistics.median(ts[3:]), flush=True)
else:
    for rnd in range(2):
        for lib in sys.argv[1:]:
            subprocess.run([sys.executable, __file__, "child"], env={**os.environ, "ADG_LIB": lib})

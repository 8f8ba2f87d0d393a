import os, sys, time, statistics
sys.path.insert(0, "/root/repo")
import torch, torch.distributed as tdist
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds, dist, _lib
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29535")
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
tdist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
X = torch.from_numpy(ds.c3_mnist_like()).to(dev)
model = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(model, X).data.clone()
busy = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
def hostt(fn, reps=30):
    ts = []
    for _ in range(reps):
        busy.zero_(); busy.zero_()  # keep the GPU busy so enqueue never waits on idle
        t = time.perf_counter(); fn(); ts.append((time.perf_counter() - t) * 1e3)
    torch.cuda.synchronize()
    return statistics.median(ts)
print("transform_all host ms", hostt(lambda: adg.transform_all(model, X[:7500])))
x = adg.api._matrix(X[:7500]); ctx, d_ = adg.api._ctx_for(x)
plan = adg.api._model_plan(model, ctx, d_, x.code)
yb = torch.empty((7500, 50), device=dev)
L = _lib.load()
print("plan_run ctypes host ms", hostt(lambda: L.adg_transform_plan_run(plan.h, x.ptr, x.code, 7500, yb.data_ptr(), _lib.ADG_F32)))
print("torch.empty host ms", hostt(lambda: torch.empty((7500, 50), device=dev)))
print("_matrix host ms", hostt(lambda: adg.api._matrix(X[:7500])))
print("Plan create host ms", hostt(lambda: dist.Plan(X, Y, 50, 1.0).close()))
torch.cuda.synchronize()
p = dist.Plan(X, Y, 50, 1.0)
torch.cuda.set_sync_debug_mode("warn")
import warnings
with warnings.catch_warnings(record=True) as w:
    warnings.simplefilter("always")
    dist.reduce_partials(p.partials())
    print("sync warnings in reduce:", [str(x.message)[:100] for x in w])
torch.cuda.set_sync_debug_mode(0)
print("reduce host ms", hostt(lambda: dist.reduce_partials(p.partials())))
print("partials host ms", hostt(lambda: p.partials()))
print("finalize host ms", hostt(lambda: p.finalize(), reps=10))
tdist.destroy_process_group()

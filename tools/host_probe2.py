"""Host time of each collective / op of dist.reduce_partials while the GPU
is busy (profiling aid: which call blocks the host?)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as tdist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29536")
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
tdist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
busy = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
a = torch.zeros(100000, dtype=torch.float64, device=dev)
b = torch.zeros(120000, dtype=torch.float32, device=dev)
c = torch.zeros(8194, dtype=torch.int32, device=dev)
out = torch.empty(8194, dtype=torch.int32, device=dev)
ops = {
    "all_reduce f64 SUM": lambda: tdist.all_reduce(a),
    "all_reduce f32 MAX": lambda: tdist.all_reduce(b, op=tdist.ReduceOp.MAX),
    "all_gather_into_tensor": lambda: tdist.all_gather_into_tensor(out, c),
    "torch.cat": lambda: torch.cat([a, a]),
    "cumsum": lambda: torch.cumsum(c.long(), 0),
    "index_copy": lambda: torch.zeros(10, 2, device=dev).index_copy_(0, torch.arange(10, device=dev), torch.ones(10, 2, device=dev)),
    "where/any": lambda: torch.where((c > 3).any(), c.sum(), c.sum()),
}
for name, fn in ops.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        busy.zero_(); busy.zero_()
        t = time.perf_counter(); fn(); ts.append((time.perf_counter() - t) * 1e3)
    torch.cuda.synchronize()
    ts.sort()
    print(f"{name:28s} host {ts[5]:.4f} ms", flush=True)
tdist.destroy_process_group()

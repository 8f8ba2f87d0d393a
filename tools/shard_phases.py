"""Phase split of one sharded evaluate (rank 0 of W) on one GPU, as the
stream sees it: CUDA events between plan creation (operand prep), the
tile-range screen, the partial exchange and the finalize, no syncs in
between; host enqueue times beside them (profiling aid)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as tdist
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
from paper_1609_05388_b200 import dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29534")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
tdist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
X = torch.from_numpy(ds.c3_mnist_like()).to(dev)
model = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(model, X).data.clone()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
names = ["transform", "create", "run", "reduce", "finalize"]
for W in [int(a) for a in sys.argv[1:]] or [1, 8]:
    dev_ms = {k: [] for k in names}
    host_ms = {k: [] for k in names}
    r0, r1 = dist.shard_rows(X.shape[0], W, 0)
    for it in range(8):
        flush.zero_()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        t = [time.perf_counter()]
        ev[0].record()
        adg.transform_all(model, X[r0:r1]); ev[1].record(); t.append(time.perf_counter())
        plan = dist.Plan(X, Y, 50, 1.0); ev[2].record(); t.append(time.perf_counter())
        t0, t1 = dist.shard_range(plan.num_tiles, W, 0)
        plan.run(t0, t1); ev[3].record(); t.append(time.perf_counter())
        if W > 1:
            plan.reduce()
        ev[4].record(); t.append(time.perf_counter())
        rep = plan.finalize(); ev[5].record(); t.append(time.perf_counter())
        torch.cuda.synchronize()
        plan.close()
        if it >= 3:
            for i, k in enumerate(names):
                dev_ms[k].append(ev[i].elapsed_time(ev[i + 1]))
                host_ms[k].append((t[i + 1] - t[i]) * 1e3)
    print(f"W={W} device: " + ", ".join(f"{k} {statistics.median(v):.3f}" for k, v in dev_ms.items())
          + " ms | host enqueue: " + ", ".join(f"{k} {statistics.median(v):.3f}" for k, v in host_ms.items()),
          flush=True)
tdist.destroy_process_group()

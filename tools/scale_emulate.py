"""Per-rank step time of the N-GPU bench on ONE GPU: a 1-rank NCCL group runs
rank 0's share of an N-rank job (row shard of the embedding + 1/N of the
pair tiles + the partial-statistics exchange + the replicated finalize).
No peer traffic, so the collectives here cost only their launch latency;
the result bounds the strong-scaling efficiency from the per-rank side.
Profiling aid, not the bench."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as tdist
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
from paper_1609_05388_b200 import dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
tdist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
Ws = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
reps = 7 if cfg == "c3" else 3
if cfg == "c3":
    X = torch.from_numpy(ds.c3_mnist_like()).to(dev)
    r = 50
else:
    X = ds.make(cfg)
    r = ds.CONFIGS[cfg][2]
n = X.shape[0]
model = adg.fit(X, r, adg.SpectralBackend.exact, 0)
Yfull = adg.transform_all(model, X).data.clone()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for W in Ws:
    ev = dist.ShardedEvaluator(W, 0)
    r0, r1 = dist.shard_rows(n, W, 0)
    Xl = X[r0:r1]

    def step():
        Yl = adg.transform_all(model, Xl).data  # this rank's rows (timed)
        Y = Yfull if W > 1 else Yl  # the all-gather's result (its transfer is not emulated)
        return ev.evaluate(X, Y, hist_bins=50)

    for _ in range(2):
        step()
    ts, wall, kern = [], [], []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        t = time.perf_counter()
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        wall.append((time.perf_counter() - t) * 1e3)
        ts.append(e0.elapsed_time(e1))
        kern.append(adg.api.last_screen_kernel_ms(0))
    print(f"{cfg} W={W}: step {statistics.median(ts):.3f} ms (events), wall {statistics.median(wall):.3f} ms, "
          f"screen {statistics.median(kern):.3f} ms", flush=True)
tdist.destroy_process_group()

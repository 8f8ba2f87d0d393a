"""Per-rank step time of the N-GPU bench on ONE GPU (profiling aid, not the
bench): rank 0's share of an N-rank step -- the embedding of its n/N rows,
the operand prep of all rows (plan refresh), the screen of its 1/N of the
tile list, the library's exchange (adg_eval_plan_exchange) and the finalize.
The exchange runs its real code path over Rank0Collectives: world = N, but
the other ranks contribute nothing (reductions are no-ops, gathers leave
their blocks empty), so collectives cost only their call overhead; NVLink
transfer time is added from a stated budget, not measured.  CUDA events
around each phase on the plan's stream; median of `reps` steps, L2 flushed
before each.

  python tools/scale_emulate.py [c3|c4|c5] [W ...]
"""
import ctypes, json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import _lib, dist
from paper_1609_05388_b200 import datasets as ds


class Rank0Collectives:
    def __init__(self, world):
        self.world, self.rank, self.error = world, 0, None
        self._ar = _lib.ALL_REDUCE_FN(lambda u, b, c, o, s: 0)
        self._ag = _lib.ALL_GATHER_FN(self._gather)
        self.c = _lib.Collectives(world, 0, None, self._ar, self._ag)

    def _gather(self, user, send, recv, nbytes, stream):
        r = dist._view(recv, self.world * nbytes, "|u1", "cuda:0")
        r.zero_()
        r[:nbytes].copy_(dist._view(send, nbytes, "|u1", "cuda:0"))
        return 0


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    Ws = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
    reps = 7 if cfg == "c3" else 3
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    X = torch.from_numpy(ds.c3_mnist_like()).to(dev) if cfg == "c3" else ds.make(cfg)
    r = ds.CONFIGS[cfg][2]
    n = X.shape[0]
    model = adg.fit(X, r, adg.SpectralBackend.exact, 0)
    Y = adg.transform_all(model, X).data.clone()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    plan = dist.Plan(X, Y, 50)
    out = {"config": cfg, "n": n, "rows": []}
    base = None
    for W in Ws:
        coll = Rank0Collectives(W)
        r0, r1 = dist.shard_rows(n, W, 0)
        t0, t1 = plan.shard(W, 0)
        names = ["embed", "prep", "screen", "exchange", "finalize"]
        samples = {k: [] for k in names + ["step"]}
        for it in range(reps + 2):
            flush.zero_()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
            ev[0].record()
            adg.transform_all(model, X[r0:r1])  # this rank's rows; Y's all-gather is not emulated
            ev[1].record()
            plan.refresh()                       # operand prep of every row
            ev[2].record()
            plan.run(t0, t1)
            ev[3].record()
            if W > 1:
                plan.exchange(coll)
            ev[4].record()
            rep = plan.finalize()
            ev[5].record()
            torch.cuda.synchronize()
            if it < 2:
                continue
            for k, nm in enumerate(names):
                samples[nm].append(ev[k].elapsed_time(ev[k + 1]))
            samples["step"].append(ev[0].elapsed_time(ev[-1]))
        row = {"W": W, **{k: statistics.median(v) for k, v in samples.items()}}
        base = base or row["step"]
        row["speedup"] = base / row["step"]
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
    plan.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()

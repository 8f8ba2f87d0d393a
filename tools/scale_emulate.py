"""Per-rank step time of the N-GPU bench on ONE GPU (profiling aid, not the
bench): rank 0's share of an N-rank step -- the embedding of its n/N rows,
the operand prep of all rows (plan refresh), the screen of its 1/N of the
tile list, the library's exchange (adg_eval_plan_exchange) and the finalize,
timed with CUDA events on the plan's stream.

The other ranks are replayed, not run: a full single-plan pass over all
tiles is taken first, and the exchange of that full state is recorded once
per rank (Recorder collectives: each rank's own refine-chunk block is what it
would send).  In the timed step, rank 0 screens only its own tiles and the
Replay collectives hand its exchange the recorded result of every
reduction and gather -- exactly the buffers N real ranks would produce -- so
the finalize does the real rank's work.  Collectives cost their call
overhead plus one device copy each; the NVLink transfer itself (~1 MB at C3:
~5-20 us on NVLink 5) is not included.  Median of `reps` steps, L2 flushed
before each.

  python tools/scale_emulate.py [c3|c4|c5] [W ...]
"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import _lib, dist
from paper_1609_05388_b200 import datasets as ds


def _bytes_view(ptr, nbytes):
    return dist._view(ptr, nbytes, "|u1", "cuda:0")


_ELEM = {_lib.ADG_SUM_U64: 8, _lib.ADG_SUM_F64: 8, _lib.ADG_MAX_F32: 4, _lib.ADG_MAX_U64: 8}


class Recorder:
    """Leaves every buffer as it is (the plan holds the full state) and
    records it; the gather records this rank's block."""

    def __init__(self, world, rank):
        self.world, self.rank, self.error = world, rank, None
        self.reduced, self.blocks = [], []
        self._ar = _lib.ALL_REDUCE_FN(self._reduce)
        self._ag = _lib.ALL_GATHER_FN(self._gather)
        self.c = _lib.Collectives(world, rank, None, self._ar, self._ag)

    def _reduce(self, user, buf, count, op, stream):
        self.reduced.append(_bytes_view(buf, count * _ELEM[int(op)]).clone())
        return 0

    def _gather(self, user, send, recv, nbytes, stream):
        self.blocks.append(_bytes_view(send, nbytes).clone())
        return 0


class Replay:
    """gathered[g] = every rank's block of the exchange's g-th gather, concatenated."""

    def __init__(self, world, reduced, gathered):
        self.world, self.rank, self.error = world, 0, None
        self.reduced, self.gathered, self.k, self.g = reduced, gathered, 0, 0
        self._ar = _lib.ALL_REDUCE_FN(self._reduce)
        self._ag = _lib.ALL_GATHER_FN(self._gather)
        self.c = _lib.Collectives(world, 0, None, self._ar, self._ag)

    def _reduce(self, user, buf, count, op, stream):
        src = self.reduced[self.k]
        self.k += 1
        _bytes_view(buf, src.numel()).copy_(src)
        return 0

    def _gather(self, user, send, recv, nbytes, stream):
        src = self.gathered[self.g]
        self.g += 1
        _bytes_view(recv, src.numel()).copy_(src)
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
    # WARM=1: queue one 4096^3 matmul (~0.1 ms) right before each timed step.
    # A short step that starts from an idle GPU runs its first ~0.1 ms slower
    # (C3's W = 8 screen share: 0.87 ms cold, 0.78 ms warm; the 6 ms one-GPU
    # step is unaffected, tools/gpu/warm_probe.py)
    WARM = os.environ.get("WARM") == "1"
    warm = torch.randn(4096, 4096, device=dev)
    plan = dist.Plan(X, Y, 50)
    T = plan.num_tiles
    out = {"config": cfg, "n": n, "rows": []}
    base = None
    names = ["embed", "prep", "screen", "exchange", "finalize"]
    for W in Ws:
        replay = None
        if W > 1:  # record the full state's exchange, once per rank
            per_rank, reduced = [], None
            for k in range(W):
                plan.refresh()
                plan.run(0, T)
                rec = Recorder(W, k)
                plan.exchange(rec)
                torch.cuda.synchronize()
                per_rank.append(rec.blocks)
                reduced = reduced or rec.reduced
            gathered = [torch.cat([per_rank[k][g] for k in range(W)]) for g in range(len(per_rank[0]))]
            replay = Replay(W, reduced, gathered)
        r0, r1 = dist.shard_rows(n, W, 0)
        t0, t1 = plan.shard(W, 0)
        samples = {k: [] for k in names + ["step"]}
        for it in range(reps + 2):
            flush.zero_()
            torch.cuda.synchronize()
            if WARM:  # a busy tensor-core kernel right before the step (steady-state clocks)
                warm @ warm
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
            ev[0].record()
            adg.transform_all(model, X[r0:r1])  # this rank's rows; Y's all-gather is not emulated
            ev[1].record()
            plan.refresh()                       # operand prep of every row
            ev[2].record()
            plan.run(t0, t1)
            ev[3].record()
            if replay is not None:
                replay.k = replay.g = 0
                plan.exchange(replay)
            ev[4].record()
            rep = plan.finalize()
            ev[5].record()
            torch.cuda.synchronize()
            if it < 2:
                continue
            for k, nm in enumerate(names):
                samples[nm].append(ev[k].elapsed_time(ev[k + 1]))
            samples["step"].append(ev[0].elapsed_time(ev[-1]))
        row = {"W": W, **{k: statistics.median(v) for k, v in samples.items()},
               "max": rep.max_distortion, "argmax": rep.argmax, "candidate_rows": rep.candidate_rows}
        base = base or row["step"]
        row["speedup"] = base / row["step"]
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
    plan.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()

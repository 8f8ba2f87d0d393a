"""In-process stand-in for a multi-GPU job on one GPU (TEST INFRASTRUCTURE).

`world` host threads, each with its own context and plan on cuda:0, exchange
through LocalCollectives: an adg_collectives whose callbacks rendezvous the
ranks' device buffers and combine them with torch (SUM / MAX / rank-order
concatenation).  The library's exchange (adg_eval_plan_exchange) and
finalize run exactly as under NCCL; the ranks' kernels never wait on each
other (the rendezvous is on the host, after each rank's stream is drained).
"""
import threading

import numpy as np
import torch

from paper_1609_05388_b200 import _lib, dist


class _Hub:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.error = None


class LocalCollectives:
    def __init__(self, hub, rank):
        self.hub, self.rank, self.world = hub, rank, hub.world
        self.error = None
        self._ar = _lib.ALL_REDUCE_FN(self._all_reduce)
        self._ag = _lib.ALL_GATHER_FN(self._all_gather)
        self.c = _lib.Collectives(self.world, rank, None, self._ar, self._ag)

    def _all_reduce(self, user, buf, count, op, stream):
        try:
            torch.cuda.synchronize()
            np_dtype, typestr = dist._RED_DTYPE[int(op)]
            t = dist._view(buf, count, typestr, "cuda:0")
            h = self.hub
            h.slots[self.rank] = t.clone()
            h.barrier.wait()
            stack = torch.stack(h.slots)
            red = stack.max(0).values if op in (_lib.ADG_MAX_F32, _lib.ADG_MAX_U64) else stack.sum(0)
            h.barrier.wait()
            t.copy_(red)
            torch.cuda.synchronize()
            return 0
        except Exception as e:
            self.error = e
            return 1

    def _all_gather(self, user, send, recv, nbytes, stream):
        try:
            torch.cuda.synchronize()
            s = dist._view(send, nbytes, "|u1", "cuda:0")
            r = dist._view(recv, self.world * nbytes, "|u1", "cuda:0")
            h = self.hub
            h.slots[self.rank] = s.clone()
            h.barrier.wait()
            r.copy_(torch.cat(h.slots))
            h.barrier.wait()
            torch.cuda.synchronize()
            return 0
        except Exception as e:
            self.error = e
            return 1


def sharded_reports(X, Y, world, bins=50, hist_max=1.0, engine="screen"):
    """Every rank's report of a `world`-rank sharded evaluation on cuda:0."""
    hub = _Hub(world)
    reps, errs = [None] * world, [None] * world

    def rank_main(rank):
        try:
            plan = dist.Plan(X, Y, bins, hist_max)
            try:
                plan.set_engine(engine)
                plan.run(*plan.shard(world, rank))
                plan.exchange(LocalCollectives(hub, rank))
                reps[rank] = plan.finalize()
            finally:
                plan.close()
        except Exception as e:  # pragma: no cover - surfaced below
            errs[rank] = e
            hub.barrier.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return reps


def assert_same_report(a, b):
    assert a.max_distortion == b.max_distortion and a.mean_distortion == b.mean_distortion
    assert a.argmax == b.argmax and a.n_zero_distance_pairs == b.n_zero_distance_pairs
    assert a.n_pairs_evaluated == b.n_pairs_evaluated
    assert np.array_equal(np.asarray(a.histogram), np.asarray(b.histogram))
    assert a.edge_pairs == b.edge_pairs

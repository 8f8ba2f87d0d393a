"""The sharded evaluator's product path with more than one rank.

Two processes share cuda:0 and exchange over gloo: dist.ShardedEvaluator ->
adg_eval_plan_shard / _run / _exchange (the library's one exchange, over
dist.TorchCollectives, host-staged) / _finalize.  The ranks' kernels never
wait on one another (the exchange is host-level), so one GPU stands in for
two.  Every report must equal the one-GPU adg.evaluate bit for bit -- the
reference's thread-count invariance (proj/include/adagio/parallel.hpp:8-11,
proj/tests/acceptance.cpp:448-502).  Also: the single-process GPU-count knob
(adg_evaluate_multi) and the native NCCL communicator at one rank.
"""
import ctypes
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cloud(kind):
    from oracle import oracle
    if kind == "gauss":
        X = oracle.gaussian_cloud(6000, 48, 3).astype(np.float32)
    else:  # many coincident rows: near-coincident lists on every rank
        X = oracle.gaussian_cloud(6000, 48, 4).astype(np.float32)
        X[3000:3400] = X[:400]
        X[5000:5100] = X[100]
    Y = (X.astype(np.float64) @ oracle.sample_jl(12, 48, 5).T).astype(np.float32)
    return X, Y


CASES = [("gauss", "screen", 50), ("dups", "screen", 50), ("gauss", "screen_exact_hist", 50),
         ("gauss", "screen_exact_hist", 1000)]


def _worker(rank, world, port, out_q, env, cases):
    os.environ.update(env)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as tdist
    from paper_1609_05388_b200 import dist
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for kind, engine, bins in cases:
            X, Y = _cloud(kind)
            ev = dist.ShardedEvaluator()
            rep = ev.evaluate(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), hist_bins=bins,
                              engine=engine)
            ev.close()
            res.append(((kind, engine, bins), rep.max_distortion, rep.mean_distortion, rep.argmax,
                        np.asarray(rep.histogram).copy(), rep.n_zero_distance_pairs, rep.edge_pairs))
        out_q.put((rank, res))
    finally:
        tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(world, env, cases=CASES):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, env, cases)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


def _single(kind, engine, bins=50):
    import torch
    import paper_1609_05388_b200 as adg
    X, Y = _cloud(kind)
    return adg.evaluate(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), hist_bins=bins,
                        engine=engine)


def _same(a, rep):
    key, mx, mean, am, hist, zero, edges = a
    assert mx == rep.max_distortion and mean == rep.mean_distortion, key
    assert am == rep.argmax and zero == rep.n_zero_distance_pairs, key
    assert np.array_equal(hist, rep.histogram), key
    assert edges == rep.edge_pairs, key


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_evaluator_bit_identical(world):
    out = _run_ranks(world, {})
    for kind, engine, bins in CASES:
        ref = _single(kind, engine, bins)
        for r in range(world):
            got = [x for x in out[r] if x[0] == (kind, engine, bins)][0]
            _same(got, ref)
    dups = _single("dups", "screen")
    assert dups.n_zero_distance_pairs > 0


@pytest.mark.timeout(900)
def test_sharded_evaluator_edge_overflow_redo():
    """An edge list over its capacity on a rank: every rank redoes the
    histogram in tile chunks, and the report is unchanged."""
    import torch
    import paper_1609_05388_b200 as adg
    case = ("gauss", "screen_exact_hist", 1000)
    out = _run_ranks(2, {"ADG_EDGE_CAP": "30000"}, [case])
    ref = _single(*case)
    assert ref.edge_pairs > 2 * 30000  # more than the cap on some rank
    for r in range(2):
        _same(out[r][0], ref)


def test_evaluate_multi_one_gpu_and_nccl_comm():
    """The C++ GPU-count knob (adg_evaluate_multi) at one device equals
    adg.evaluate; NCCL loads and builds a one-rank communicator."""
    import torch
    import paper_1609_05388_b200 as adg
    from paper_1609_05388_b200 import _lib
    X, Y = _cloud("dups")
    ref = _single("dups", "screen")
    L = _lib.load()
    rep = _lib.Report()
    hist = np.zeros(51, np.uint64)
    devs = (ctypes.c_int32 * 1)(0)
    _lib.check(L.adg_evaluate_multi(1, devs, X.ctypes.data, _lib.ADG_F32, X.shape[0], X.shape[1],
                                    Y.ctypes.data, _lib.ADG_F32, Y.shape[0], Y.shape[1], None, 50,
                                    1.0, _lib.ENGINES["screen"], ctypes.byref(rep), hist.ctypes.data))
    assert rep.max_distortion == ref.max_distortion and rep.mean_distortion == ref.mean_distortion
    assert np.array_equal(hist, ref.histogram)
    comms = (_lib.Collectives * 1)()
    _lib.check(L.adg_comm_nccl_create_all(1, devs, comms))
    assert comms[0].world == 1 and comms[0].rank == 0
    _lib.check(L.adg_comm_nccl_destroy(ctypes.byref(comms[0])))

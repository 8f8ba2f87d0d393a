"""Multi-rank host logic of the sharded evaluator on CPU (gloo, world size 2).

The per-tile statistics come from an exact numpy stand-in for the screen
(test infrastructure); what is under test is the rank partition and the
transport the library's exchange (adg_eval_plan_exchange) runs over:
dist.TorchCollectives' C callbacks, called through ctypes exactly as the
library calls them (in-place SUM / MAX all-reduces, a rank-order all-gather),
on host buffers.  The reduced partials of a 2-rank run must equal the 1-rank
partials bit for bit, so every rank's finalize sees the same inputs and the
report cannot depend on the GPU count.  The exchange itself (C++, device
buffers) is run end to end by tests/test_gpu_dist.py.
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from paper_1609_05388_b200 import _lib, dist

BM = dist.BN  # column block of a pair tile (160)
PM = dist.PM  # row block of a pair tile (256)
SLOTS = 40  # (256 / 32) row slots x (160 / 32) column slots per tile (emulation)


def tile_partials(X, Y, tiles, t0, t1, bins=20, hist_max=1.0, cap=4096):
    """Exact fp64 stand-in for the screen over tiles [t0, t1)."""
    n = X.shape[0]
    hist = np.zeros(bins + 1, np.int64)
    sums = np.zeros(SLOTS * len(tiles), np.float64)
    rmax = np.zeros(n, np.float32)
    rbound = np.zeros(n, np.float32)
    near = []
    for t in range(t0, t1):
        I2, J = int(tiles[t]) >> 16, int(tiles[t]) & 0xFFFF
        for i in range(I2 * PM, min((I2 + 1) * PM, n)):
            for j in range(max(J * BM, i + 1), min((J + 1) * BM, n)):
                o = np.sum((X[i] - X[j]) ** 2)
                if o == 0.0:
                    near.append((i, j))
                    continue
                v = abs(np.sqrt(np.sum((Y[i] - Y[j]) ** 2)) / np.sqrt(o) - 1.0)
                hist[min(int(v / hist_max * bins), bins) if v < hist_max else bins] += 1
                slot = t * SLOTS + ((i % PM) // 32) + 8 * ((j % BM) // 32)
                sums[slot] += v
                rmax[i] = max(rmax[i], np.float32(v))
                rbound[i] = max(rbound[i], np.float32(v + 1e-6))
    pairs = np.zeros(2 * cap, np.int32)
    for k, (i, j) in enumerate(near):
        pairs[2 * k], pairs[2 * k + 1] = i, j
    return {"hist": torch.from_numpy(hist), "tile_sums": torch.from_numpy(sums),
            "row_max": torch.from_numpy(rmax), "row_bound": torch.from_numpy(rbound),
            "near_pairs": torch.from_numpy(pairs),
            "near_count": torch.tensor([len(near)], dtype=torch.int64), "near_capacity": cap}


def make_data():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((300, 6))
    X[17] = X[3]          # duplicates -> near-coincident list on different ranks
    X[290] = X[3]
    Y = X @ rng.standard_normal((6, 3)) / np.sqrt(3)
    return X, Y


def _ptr(a):
    return a.ctypes.data


def exchange_host(coll, parts, block=1024):
    """The library's exchange sequence (csrc/adg_api.cu plan_exchange and
    near_regather) over coll's C callbacks on host numpy partials: SUM hist,
    SUM tile sums, MAX [row_max | row_bound], then the near-coincident lists
    all-gathered in fixed blocks and concatenated in rank order (the merge
    kernel's rule); a list longer than the block -> MAX of the counts and a
    second gather sized by it; a total over the capacity -> overflow mark.
    (The refine-chunk gather moves opaque bytes: covered on the GPU.)"""
    c = coll.c
    hist = parts["hist"].numpy()
    assert c.all_reduce(None, _ptr(hist), hist.size, _lib.ADG_SUM_U64, None) == 0
    sums = parts["tile_sums"].numpy()
    assert c.all_reduce(None, _ptr(sums), sums.size, _lib.ADG_SUM_F64, None) == 0
    rows = np.concatenate([parts["row_max"].numpy(), parts["row_bound"].numpy()])
    assert c.all_reduce(None, _ptr(rows), rows.size, _lib.ADG_MAX_F32, None) == 0
    n = parts["row_max"].numel()
    parts["row_max"].copy_(torch.from_numpy(rows[:n]))
    parts["row_bound"].copy_(torch.from_numpy(rows[n:]))
    mine = int(parts["near_count"].item())
    cap = parts["near_capacity"]
    own = parts["near_pairs"].numpy()[: 2 * min(mine, cap)].copy()

    def gather(g):
        blk = np.zeros(2 * g + 2, np.int32)
        blk[0] = mine if mine <= g else g + 1
        m = min(mine, g)
        blk[2: 2 + 2 * m] = own[: 2 * m]
        allb = np.zeros(coll.world * (2 * g + 2), np.int32)
        assert c.all_gather(None, _ptr(blk), _ptr(allb), blk.nbytes, None) == 0
        return allb.reshape(coll.world, 2 * g + 2)

    g = min(cap, block)
    allb = gather(g)
    counts = allb[:, 0].astype(np.int64)
    if (counts > g).any():  # second, sized gather
        most = np.array([mine], np.int64)
        assert c.all_reduce(None, _ptr(most), 1, _lib.ADG_MAX_U64, None) == 0
        if most[0] > cap:
            parts["near_count"][0] = int(most[0])
            return
        g = int(most[0])
        allb = gather(g)
        counts = allb[:, 0].astype(np.int64)
    if counts.sum() > cap:
        parts["near_count"][0] = cap + 1
        return
    merged = np.concatenate([allb[w, 2: 2 + 2 * counts[w]] for w in range(coll.world)])
    parts["near_pairs"][: merged.size] = torch.from_numpy(merged)
    parts["near_count"][0] = int(counts.sum())


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, Y = make_data()
        tiles = dist.tile_list(X.shape[0])
        t0, t1 = dist.shard_range(len(tiles), world, rank)
        parts = tile_partials(X, Y, tiles, t0, t1)
        coll = dist.TorchCollectives(device="cpu")
        assert (coll.world, coll.rank) == (world, rank) and coll.staged
        exchange_host(coll, parts)
        c = int(parts["near_count"].item())
        near = parts["near_pairs"][: 2 * c].numpy().reshape(-1, 2)
        out_q.put((rank, parts["hist"].numpy().copy(), parts["tile_sums"].numpy().copy(),
                   parts["row_max"].numpy().copy(), parts["row_bound"].numpy().copy(),
                   sorted(map(tuple, near.tolist()))))
    finally:
        tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_tile_list_and_shards():
    for n in [1, 2, 100, 300, 1000, 5000, 20000]:
        tl = dist.tile_list(n)
        pairs = {(int(t) >> 16, int(t) & 0xFFFF) for t in tl}
        assert len(tl) == len(pairs)
        # exactly the (row block, column block) combinations holding some pair i < j
        T, T2 = -(-n // BM), -(-n // PM)
        want = {(i2, j) for i2 in range(T2) for j in range(T)
                if min((j + 1) * BM, n) - 1 > i2 * PM}
        assert want <= pairs  # every combination holding a pair is listed, once
        assert all(min((j + 1) * BM, n) - 1 <= i2 * PM for i2, j in pairs - want)  # extras are empty
        for world in [1, 2, 3, 8]:
            rngs = [dist.shard_range(len(tl), world, r) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == len(tl)
            assert all(rngs[k][1] == rngs[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in rngs]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.timeout(300)
def test_two_rank_reduction_equals_single_rank():
    X, Y = make_data()
    tiles = dist.tile_list(X.shape[0])
    ref = tile_partials(X, Y, tiles, 0, len(tiles))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_near = sorted(map(tuple, ref["near_pairs"][: 2 * int(ref["near_count"])].numpy()
                          .reshape(-1, 2).tolist()))
    assert len(ref_near) == 3
    for _, h, s, rm, rb, near in results:
        assert np.array_equal(h, ref["hist"].numpy())
        assert np.array_equal(s, ref["tile_sums"].numpy())      # bitwise: one writer per slot
        assert np.array_equal(rm, ref["row_max"].numpy())
        assert np.array_equal(rb, ref["row_bound"].numpy())
        assert near == ref_near


# ------------------------------------------------- row-sharded fit (8e step 1)
def _cpu_fit_ops():
    """Oracle stand-ins for the three per-shard kernels (column sums, centred
    Gram, solve on the total Gram) so the exchange runs on CPU under gloo."""
    from oracle import oracle as o

    def colsum(x, ctx, dev):
        return x.sum(dim=0, dtype=torch.float64)

    def gram(x, ctx, dev, mean, backend):
        c = x.double() - mean
        return c.T @ c

    def solve(G, n_total, s, k, backend, seed, ctx, dev):
        w, v = np.linalg.eigh(G.numpy())
        P = o._normalize_row_signs(v[:, ::-1][:, :s].T.copy())
        S = o.sample_jl(k, G.shape[0], o.derive_seed(seed, "jl"))
        return torch.from_numpy(P), torch.from_numpy(S)

    return {"colsum": colsum, "gram": gram, "solve": solve}


def _fit_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dist._FIT_OPS.update(_cpu_fit_ops())
        X = _fit_cloud()
        n = X.shape[0]
        r0, r1 = dist.shard_rows(n, world, rank)
        Xl = torch.from_numpy(X[r0:r1])
        model = dist.fit_sharded(Xl, n, 8, seed=3)
        Xall = dist.all_gather_rows(Xl, n)
        lab = torch.arange(r0, r1, dtype=torch.int64)[:, None].repeat(1, 3)
        lab_all = dist.all_gather_rows(lab, n)
        out_q.put((rank, model.mean.numpy().copy(), model.basis.rows.numpy().copy(),
                   model.sketch.entries.numpy().copy(), Xall.numpy().copy(), lab_all.numpy().copy()))
    finally:
        tdist.destroy_process_group()


def _fit_cloud():
    from oracle import oracle as o
    return o.low_rank_cloud(301, 24, 5, 11) + 3.0  # off-centre, uneven shards at world 2 and 3


def test_shard_rows_cover():
    for n in [0, 1, 2, 7, 301, 60000]:
        for world in [1, 2, 3, 8]:
            rngs = [dist.shard_rows(n, world, r) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == n
            assert all(rngs[k][1] == rngs[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in rngs]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fit_matches_whole_cloud(world):
    from oracle import oracle as o
    X = _fit_cloud()
    mean_ref, P_ref, S_ref = o.fit(X, 8, "exact", 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fit_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    means = [r[1] for r in results]
    for _, mean, P, S, Xall, lab in results:
        assert np.array_equal(mean, means[0])             # identical model on every rank
        np.testing.assert_allclose(mean, mean_ref, rtol=1e-14, atol=1e-14)
        # same principal subspace and the reference's sign rule
        np.testing.assert_allclose(P, P_ref, atol=1e-10)
        assert np.array_equal(S, S_ref)                   # JL entries bit-exact
        assert np.array_equal(Xall, X)                    # uneven all-gather in rank order
        assert np.array_equal(lab[:, 0], np.arange(X.shape[0]))


def _overflow_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, Y = make_data()
        tiles = dist.tile_list(X.shape[0])
        t0, t1 = dist.shard_range(len(tiles), world, rank)
        coll = dist.TorchCollectives(device="cpu")
        res = []
        for cap in (1, 2, 8):  # plan capacity of the near-coincident list
            parts = tile_partials(X, Y, tiles, t0, t1, cap=max(cap, 8))
            parts["near_capacity"] = cap
            mine = int(parts["near_count"].item())  # > cap: the screen's own overflow mark
            exchange_host(coll, parts, block=1)  # block 1: the second, sized gather runs too
            res.append((cap, mine, int(parts["near_count"].item())))
        # a failing collective is reported, not raised through C
        bad = np.zeros(3, np.float32)
        assert coll.c.all_reduce(None, bad.ctypes.data, 3, 99, None) == 1 and coll.error is not None
        out_q.put((rank, res))
    finally:
        tdist.destroy_process_group()


@pytest.mark.timeout(300)
def test_near_list_exchange_overflow_marks_plan():
    """Any rank's list over the plan's capacity, or a total above it, leaves
    near_count > capacity on every rank, which sends every finalize to the
    chunked redo (csrc/adg_api.cu plan_rechunk)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overflow_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for idx, cap in enumerate((1, 2, 8)):
        mine = [results[r][idx][1] for r in range(2)]
        got = [results[r][idx][2] for r in range(2)]
        assert got[0] == got[1]
        if sum(mine) > cap:
            assert got[0] > cap
        else:
            assert got[0] == sum(mine) == 3


def test_screen_band_rule():
    # planes of ktot fp16 columns: C3 (832 + 64), C4 (960 + 64), C5 (4096 + 128)
    assert dist.screen_band(896) == 32 and dist.screen_band(1024) == 32
    assert dist.screen_band(4224) == 16
    assert dist.screen_band(65536) == 4
    for n in (1000, 5000):
        for band in (8, 16, 32):
            tl = dist.tile_list(n, band)
            assert len(set(tl.tolist())) == len(tl) == len(dist.tile_list(n))

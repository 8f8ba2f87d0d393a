"""Multi-GPU sharding of the hot path, one process per GPU.

1. Fit (`fit_sharded`): the cloud is row-sharded (`shard_rows`).  Each rank
   sums its shard's columns, the d sums are all-reduced and divided by the
   total row count (the reference's colwise mean, proj/src/dataset.cpp:211),
   each rank forms the fp64 Gram of its centred shard, the d x d Grams are
   all-reduced (SUM), and every rank runs the identical subspace solve and JL
   sample on the total (adg_fit_from_gram) -> the same model on every rank.
2. Embedding (`transform_sharded`): each rank embeds its own rows, then one
   all-gather assembles the n x r embedding on every rank (`all_gather_rows`,
   also used once to replicate X for the pair space).
3. Distortion (`ShardedEvaluator`): every rank holds the whole
point set (replicated, as the pair space needs all rows), builds the same
SCREEN plan (adg_eval_plan_*: identical tile list), screens a contiguous range
of the tile list, then the partial statistics are combined with one exchange:

  hist, tile_sums          all_reduce SUM   (each tile slot written by one rank,
                                             so the fp64 sums are exact copies)
  row_max, row_bound       all_reduce MAX
  near-coincident pairs    all_gather + concatenation (finalize sorts them)

and every rank runs the deterministic finalize (exact fp64 refine of the max
band, ordered reductions) on identical inputs -> the report is bit-identical
for any number of GPUs, mirroring the reference's thread-count invariance
(proj/include/adagio/parallel.hpp:8-11, proj/tests/acceptance.cpp:448-502).

The reduction helpers operate on plain torch tensors, so the same code runs
with the gloo backend on CPU in the tests (the fit's three per-shard kernels
are looked up through `_FIT_OPS`, so those tests can stand the oracle in for
them on CPU).
"""
from __future__ import annotations

import ctypes

import numpy as np

try:
    import torch
    import torch.distributed as tdist
except Exception:  # pragma: no cover
    torch = None
    tdist = None

from . import _lib
from .api import (_matrix, _ctx_for, _report, AdagioModel, OrthonormalBasis, JlMatrix,
                  SpectralBackend, derive_seed, transform_all)

BAND = 32  # must match SC_BAND in csrc/adg_screen_kernel.cuh
GATHER_PAIRS = 4096  # near-coincident pairs per rank carried by the exchange


PM, BN = 256, 160  # must match SC_PM / SC_BN in csrc/adg_screen_kernel.cuh


def screen_band(ktot: int) -> int:
    """Replica of screen_band (csrc/adg_screen.cu): row blocks per band, halved
    from BAND while the band's hi + lo rows of ktot fp16 columns exceed 72 MB."""
    band = BAND
    while band > 4 and band * PM * 4 * ktot > (72 << 20):
        band //= 2
    return band


def tile_list(n: int, band: int = BAND) -> np.ndarray:
    """Host replica of build_tile_list (csrc/adg_screen.cu) for n points:
    pair tiles of a 256-row block I2 and a 160-column block J with
    J >= floor(256 I2 / 160) (the upper triangle with its diagonal tiles), in
    bands of `band` row blocks (screen_band(ktot)), packed (I2 << 16) | J."""
    T, T2 = -(-n // BN), -(-n // PM)
    out = []
    for B0 in range(0, T2, band):
        B1 = min(B0 + band, T2)
        for J in range(B0 * PM // BN, T):
            for I2 in range(B0, B1):
                if I2 * PM // BN <= J:
                    out.append((I2 << 16) | J)
    return np.asarray(out, np.uint32)


def shard_range(num_tiles: int, world: int, rank: int):
    """Contiguous, balanced tile range of `rank` (covers [0, num_tiles) exactly)."""
    return num_tiles * rank // world, num_tiles * (rank + 1) // world


def shard_rows(n: int, world: int, rank: int):
    """Contiguous, balanced row range [r0, r1) of `rank` for an n-row cloud."""
    return n * rank // world, n * (rank + 1) // world


def all_gather_rows(local, n_total: int, group=None):
    """Concatenate the per-rank row blocks of a cloud sharded by `shard_rows`
    (uneven blocks allowed) in rank order: one all_gather_into_tensor of the
    blocks padded to the largest, then the padding dropped."""
    world = tdist.get_world_size(group)
    if world == 1:
        return local
    counts = [shard_rows(n_total, world, r)[1] - shard_rows(n_total, world, r)[0]
              for r in range(world)]
    mx = max(counts)
    rank = tdist.get_rank(group)
    if local.shape[0] != counts[rank]:
        raise ValueError(f"all_gather_rows: rank {rank} holds {local.shape[0]} rows, "
                         f"shard_rows gives {counts[rank]}")
    tail = tuple(local.shape[1:])
    src = local.contiguous()
    if src.shape[0] != mx:
        pad = torch.zeros((mx,) + tail, dtype=local.dtype, device=local.device)
        pad[: src.shape[0]] = src
        src = pad
    out = torch.empty((world * mx,) + tail, dtype=local.dtype, device=local.device)
    tdist.all_gather_into_tensor(out, src, group=group)
    if all(c == mx for c in counts):
        return out
    return torch.cat([out[r * mx: r * mx + counts[r]] for r in range(world)])


# ------------------------------------------------------------ sharded fit
def _colsum_dev(x, ctx, dev):
    n, d = x.shape
    out = torch.empty(d, dtype=torch.float64, device=dev)
    _lib.check(_lib.load().adg_column_sums(ctx, x.ptr, x.code, n, d, out.data_ptr()))
    return out


def _gram_dev(x, ctx, dev, mean, backend):
    n, d = x.shape
    out = torch.empty((d, d), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().adg_gram(ctx, x.ptr, x.code, n, d, mean.data_ptr(), int(backend),
                                    out.data_ptr()))
    return out


def _solve_dev(gram, n_total, s, k, backend, seed, ctx, dev):
    d = gram.shape[0]
    basis = torch.empty((max(s, 0), d), dtype=torch.float64, device=dev)
    sketch = torch.empty((k, d), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().adg_fit_from_gram(ctx, gram.data_ptr(), n_total, d, s, k, int(backend),
                                             seed & (2**64 - 1),
                                             basis.data_ptr() if s > 0 else None,
                                             sketch.data_ptr()))
    return basis, sketch


# the three per-shard steps of the fit: (column sums, centred Gram, solve)
_FIT_OPS = {"colsum": _colsum_dev, "gram": _gram_dev, "solve": _solve_dev}


def fit_with_split_sharded(X_local, n_total: int, s: int, k: int,
                           backend=SpectralBackend.exact, seed: int = 0, group=None):
    """proj/src/embed.cpp:115-141 over a row-sharded cloud: this rank holds
    rows shard_rows(n_total, world, rank) of X.  Returns the same
    AdagioModel on every rank; at world size 1 it is bit-identical to
    api.fit_with_split."""
    backend = SpectralBackend(backend)
    ops = _FIT_OPS
    if ops["colsum"] is _colsum_dev:
        x = _matrix(X_local)
        ctx, dev = _ctx_for(x)
    else:  # CPU test stand-ins
        x, ctx, dev = X_local, None, X_local.device
    d = x.shape[1]
    sums = ops["colsum"](x, ctx, dev)
    if tdist.is_initialized() and tdist.get_world_size(group) > 1:
        tdist.all_reduce(sums, op=tdist.ReduceOp.SUM, group=group)
    # colwise().mean() = sum / n: a tensor divisor keeps torch's true IEEE
    # division (a scalar divisor becomes a reciprocal multiply)
    mean = sums / torch.full_like(sums, float(n_total))
    gram = ops["gram"](x, ctx, dev, mean, backend)
    if tdist.is_initialized() and tdist.get_world_size(group) > 1:
        tdist.all_reduce(gram, op=tdist.ReduceOp.SUM, group=group)
    basis, sketch = ops["solve"](gram, n_total, s, k, backend, seed, ctx, dev)
    assert mean.shape[0] == d
    return AdagioModel(mean, OrthonormalBasis(basis), JlMatrix(sketch, derive_seed(seed, "jl")),
                       seed, backend)


def fit_sharded(X_local, n_total: int, target_dim: int, backend=SpectralBackend.exact,
                seed: int = 0, group=None):
    """proj/src/embed.cpp:105-113 (s = floor(r/2), k = r - s) over a row-sharded cloud."""
    d = X_local.shape[1]
    if target_dim < 2 or target_dim > d:
        raise _lib.InvalidArgument(f"fit: target_dim = {target_dim} outside [2, {d}]")
    if n_total < 2:
        raise _lib.InvalidArgument("fit: need at least 2 points")
    return fit_with_split_sharded(X_local, n_total, target_dim // 2, target_dim - target_dim // 2,
                                  backend, seed, group)


def transform_sharded(model, X_local, n_total: int, group=None):
    """proj/src/embed.cpp:161-181 over a row-sharded cloud: each rank embeds its
    own rows, one all-gather returns the whole n x r embedding on every rank."""
    Y_local = transform_all(model, X_local).data
    if not tdist.is_initialized():
        return Y_local
    return all_gather_rows(Y_local, n_total, group)


def reduce_partials(parts: dict, group=None):
    """Combine per-rank partials in place, on the device and without a host
    round trip: three collectives whatever the world size.  parts: hist
    (int64), tile_sums (float64), row_max / row_bound (float32), near_pairs
    (int32, 2*cap), near_count (int64 [1]), near_capacity (int).

      [tile_sums | hist]   one float64 all_reduce SUM.  Exact: every tile slot
                           has one writer (the other ranks add 0.0) and the
                           counts stay below 2^53.
      [row_max | row_bound] one float32 all_reduce MAX.
      near-coincident list  one all_gather of a fixed block per rank
                           ([count, pad, pairs...], at most GATHER_PAIRS pairs),
                           compacted in rank order by a prefix sum; a rank
                           over the block (or the total over the plan's
                           capacity) marks the list overflowed, and the
                           finalize then runs the exact engine."""
    SUM, MAX = tdist.ReduceOp.SUM, tdist.ReduceOp.MAX
    hist, sums = parts["hist"], parts["tile_sums"]
    nb = hist.numel()
    buf = torch.cat([sums, hist.to(torch.float64)])
    tdist.all_reduce(buf, op=SUM, group=group)
    sums.copy_(buf[: sums.numel()])
    hist.copy_(buf[sums.numel():].to(torch.int64))
    rm, rb = parts["row_max"], parts["row_bound"]
    mx = torch.cat([rm, rb])
    tdist.all_reduce(mx, op=MAX, group=group)
    rm.copy_(mx[: rm.numel()])
    rb.copy_(mx[rm.numel():])

    cap = int(parts["near_capacity"])
    world = tdist.get_world_size(group)
    g = min(cap, GATHER_PAIRS)
    pairs, cnt = parts["near_pairs"], parts["near_count"]
    dev = pairs.device
    block = torch.zeros(2 + 2 * g, dtype=torch.int32, device=dev)
    c = cnt.clamp(max=g + 1)
    block[0:1] = c.to(torch.int32)
    block[2:] = pairs[: 2 * g]
    allb = torch.empty(world * (2 + 2 * g), dtype=torch.int32, device=dev)
    tdist.all_gather_into_tensor(allb, block, group=group)
    allb = allb.view(world, 2 + 2 * g)
    counts = allb[:, 0].to(torch.int64)
    total = counts.sum()
    over = (counts > g).any() | (total > cap)
    k = torch.arange(g, device=dev)
    offs = torch.cumsum(counts, 0) - counts
    valid = k[None, :] < counts.clamp(max=g)[:, None]
    dst = torch.where(valid, offs[:, None] + k[None, :], torch.full_like(k[None, :], world * g))
    out = torch.zeros(world * g + 1, 2, dtype=torch.int32, device=dev)
    out.index_copy_(0, dst.reshape(-1), allb[:, 2:].reshape(world * g, 2))
    m = min(world * g, cap)
    pairs[: 2 * m] = out[:m].reshape(-1)
    cnt.copy_(torch.where(over, torch.full_like(total, cap + 1), total).reshape(1))
    return parts


class _CAI:
    """Expose a raw device pointer to torch via __cuda_array_interface__."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _view(ptr, count, typestr, device, dtype=None):
    t = torch.as_tensor(_CAI(ptr, count, typestr), device=device)
    return t.view(dtype) if dtype is not None else t


class Plan:
    """A SCREEN evaluation plan on this rank's GPU (adg_eval_plan_*)."""

    def __init__(self, X, Y, hist_bins=50, hist_max=1.0):
        self.x = _matrix(X, "original")
        self.y = _matrix(Y, "embedded")
        if self.x.shape[0] != self.y.shape[0]:
            raise _lib.InvalidArgument(
                f"evaluate: cloud sizes differ ({self.x.shape[0]} vs {self.y.shape[0]})")
        self.ctx, self.dev = _ctx_for(self.x, self.y)
        self.L = _lib.load()
        self.h = ctypes.c_void_p()
        n, d = self.x.shape
        _lib.check(self.L.adg_eval_plan_create(self.ctx, self.x.ptr, self.x.code, n, d, self.y.ptr,
                                               self.y.code, self.y.shape[1], hist_bins,
                                               float(hist_max), ctypes.byref(self.h)))
        p = _lib.Partials()
        _lib.check(self.L.adg_eval_plan_partials(self.h, ctypes.byref(p)))
        self.p = p
        self.hist_bins = hist_bins
        self.num_tiles = int(p.num_tiles)

    def partials(self):
        p, dev = self.p, self.dev
        return {"hist": _view(p.hist, self.hist_bins + 1, "<i8", dev),
                "tile_sums": _view(p.tile_sums, p.tile_slots * p.num_tiles, "<f8", dev),
                "row_max": _view(p.row_max, p.n, "<f4", dev),
                "row_bound": _view(p.row_bound, p.n, "<f4", dev),
                "near_pairs": _view(p.near_pairs, 2 * p.near_capacity, "<i4", dev),
                "near_count": _view(p.near_count, 1, "<i8", dev),
                "near_capacity": int(p.near_capacity)}

    def run(self, t0, t1):
        _lib.check(self.L.adg_eval_plan_run(self.h, int(t0), int(t1)))

    def reduce(self, group=None):
        """reduce_partials on the plan's own buffers: hist and tile sums SUM
        in place, the contiguous [row_max | row_bound] MAX in place, and the
        near-coincident list packed / all-gathered / merged by two library
        kernels -- four collectives and two kernels, all stream-ordered."""
        p, dev = self.p, self.dev
        SUM, MAX = tdist.ReduceOp.SUM, tdist.ReduceOp.MAX
        tdist.all_reduce(_view(p.hist, self.hist_bins + 1, "<i8", dev), op=SUM, group=group)
        tdist.all_reduce(_view(p.tile_sums, p.tile_slots * p.num_tiles, "<f8", dev), op=SUM, group=group)
        tdist.all_reduce(_view(p.row_max, 2 * p.n, "<f4", dev), op=MAX, group=group)  # row_bound follows
        world = tdist.get_world_size(group)
        g = int(min(p.near_capacity, GATHER_PAIRS))
        block = torch.empty(2 * g + 2, dtype=torch.int32, device=dev)
        _lib.check(self.L.adg_eval_plan_near_pack(self.h, block.data_ptr(), g))
        blocks = torch.empty(world * (2 * g + 2), dtype=torch.int32, device=dev)
        tdist.all_gather_into_tensor(blocks, block, group=group)
        _lib.check(self.L.adg_eval_plan_near_merge(self.h, blocks.data_ptr(), world, g))

    def reset(self):
        _lib.check(self.L.adg_eval_plan_reset(self.h))

    def refresh(self):
        """Reset and re-prepare from the same device buffers (new contents)."""
        _lib.check(self.L.adg_eval_plan_refresh(self.h))

    def finalize(self):
        rep = _lib.Report()
        hist = np.zeros(self.hist_bins + 1, np.uint64)
        _lib.check(self.L.adg_eval_plan_finalize(self.h, ctypes.byref(rep), hist.ctypes.data))
        return _report(rep, hist)

    def close(self):
        if self.h:
            self.L.adg_eval_plan_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedEvaluator:
    """evaluate(all pairs) sharded over the ranks of the default group."""

    def __init__(self, world=None, rank=None, group=None):
        self.group = group
        self.world = world if world is not None else tdist.get_world_size(group)
        self.rank = rank if rank is not None else tdist.get_rank(group)

    def _plan(self, X, Y, hist_bins, hist_max):
        """The previous call's plan when X / Y are the same device buffers
        (shape, dtype) on the same stream -- refreshed from their current
        contents, without re-allocation -- else a new plan."""
        key = None
        if torch is not None and isinstance(X, torch.Tensor) and isinstance(Y, torch.Tensor) and X.is_cuda:
            key = (X.data_ptr(), tuple(X.shape), X.dtype, Y.data_ptr(), tuple(Y.shape), Y.dtype,
                   int(hist_bins), float(hist_max), torch.cuda.current_stream(X.device).cuda_stream)
        cached = getattr(self, "_cached", None)
        if key is not None and cached is not None and cached[0] == key:
            _ctx_for(_matrix(X), _matrix(Y))  # (re)bind the context to this stream
            cached[1].refresh()
            return cached[1]
        if cached is not None:
            cached[1].close()
            self._cached = None
        plan = Plan(X, Y, hist_bins, hist_max)
        direct = (torch.float32, torch.float64, torch.bfloat16)
        if (key is not None and X.is_contiguous() and Y.is_contiguous() and X.dtype in direct
                and Y.dtype in direct):
            # the plan reads X / Y in place (no converted copies), so it need
            # not keep them alive: a later call passing live tensors at the
            # same addresses refreshes from them, any other call rebuilds
            plan.x = plan.y = None
            self._cached = (key, plan)
        return plan

    def evaluate(self, X, Y, hist_bins=50, hist_max=1.0):
        plan = self._plan(X, Y, hist_bins, hist_max)
        try:
            t0, t1 = shard_range(plan.num_tiles, self.world, self.rank)
            plan.run(t0, t1)
            if self.world > 1:
                # stream-ordered: the collectives queue behind the screen on
                # torch's current stream (the plan's stream) and the finalize
                # behind them -- no host round trip until the finalize's own
                plan.reduce(self.group)
            return plan.finalize()
        finally:
            if getattr(self, "_cached", None) is None or self._cached[1] is not plan:
                plan.close()

    def close(self):
        cached = getattr(self, "_cached", None)
        if cached is not None:
            cached[1].close()
            self._cached = None

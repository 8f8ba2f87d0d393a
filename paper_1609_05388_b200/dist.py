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
3. Distortion (`ShardedEvaluator`): every rank holds the whole point set
   (replicated, as the pair space needs all rows), builds the same SCREEN plan
   (adg_eval_plan_*: identical tile list), screens its contiguous range of the
   tile list (adg_eval_plan_shard), and the ranks combine their partials with
   the library's one exchange, adg_eval_plan_exchange (include/adg.h):

     [edge pairs | hist]      all_reduce SUM (u64)
     tile_sums                all_reduce SUM (f64; one writer per slot: exact)
     [row_max | row_bound]    all_reduce MAX (f32)
     best row's exact refine  its j chunks split over the ranks, all_gather
     near-coincident pairs    all_gather of fixed 1024-pair blocks + rank-order
                              merge (gathered again, sized by the largest list,
                              at the finalize when a list is longer)

   over collectives this module provides (`TorchCollectives`: torch.distributed,
   device buffers under NCCL, host-staged under gloo) or NCCL driven natively
   by the library (`NcclCollectives`).  Every rank then runs the
   deterministic finalize (exact fp64 refine of the max band, ordered
   reductions) on identical inputs -> the report is bit-identical for any
   number of GPUs, mirroring the reference's thread-count invariance
   (proj/include/adagio/parallel.hpp:8-11, proj/tests/acceptance.cpp:448-502).

The fit's reductions operate on plain torch tensors, so the same code runs
with the gloo backend on CPU in the tests (its three per-shard kernels are
looked up through `_FIT_OPS`, so those tests can stand the oracle in for them
on CPU); `TorchCollectives` also serves host pointers, which the CPU tests use.
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


class _CAI:
    """Expose a raw device pointer to torch via __cuda_array_interface__."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _view(ptr, count, typestr, device, dtype=None):
    t = torch.as_tensor(_CAI(ptr, count, typestr), device=device)
    return t.view(dtype) if dtype is not None else t


_RED_DTYPE = {_lib.ADG_SUM_U64: (np.int64, "<i8"), _lib.ADG_SUM_F64: (np.float64, "<f8"),
              _lib.ADG_MAX_F32: (np.float32, "<f4"), _lib.ADG_MAX_U64: (np.int64, "<i8")}


def _tensor_at(ptr, count, np_dtype, typestr, device):
    """A torch view of `count` elements at a raw pointer: device memory via
    __cuda_array_interface__, host memory via a numpy buffer."""
    if device is not None and torch.device(device).type == "cuda":
        return _view(ptr, count, typestr, device)
    ctype = {np.int64: ctypes.c_int64, np.float64: ctypes.c_double, np.float32: ctypes.c_float,
             np.uint8: ctypes.c_uint8}[np_dtype]
    return torch.from_numpy(np.ctypeslib.as_array((ctype * int(count)).from_address(int(ptr))))


class TorchCollectives:
    """adg_collectives over torch.distributed.  NCCL: the buffers are reduced
    in place on the device (torch's collectives are ordered with its current
    stream, which the plan's context is bound to).  Other backends (gloo):
    host-staged -- each buffer is copied to the host, reduced and copied back.
    Counts are exchanged as int64 (they stay below 2^63)."""

    def __init__(self, group=None, device=None):
        self.group = group
        self.device = device
        self.world = tdist.get_world_size(group)
        self.rank = tdist.get_rank(group)
        self.staged = tdist.get_backend(group) != "nccl"
        self.error = None
        self._ar = _lib.ALL_REDUCE_FN(self._all_reduce)
        self._ag = _lib.ALL_GATHER_FN(self._all_gather)
        self.c = _lib.Collectives(self.world, self.rank, None, self._ar, self._ag)

    def _all_reduce(self, user, buf, count, op, stream):
        try:
            np_dtype, typestr = _RED_DTYPE[int(op)]
            t = _tensor_at(buf, count, np_dtype, typestr, self.device)
            rop = tdist.ReduceOp.MAX if op in (_lib.ADG_MAX_F32, _lib.ADG_MAX_U64) else tdist.ReduceOp.SUM
            if self.staged and t.is_cuda:
                h = t.cpu()
                tdist.all_reduce(h, op=rop, group=self.group)
                t.copy_(h)
            else:
                tdist.all_reduce(t, op=rop, group=self.group)
            return 0
        except Exception as e:  # reported through the library as ADG_ENCCL
            self.error = e
            return 1

    def _all_gather(self, user, send, recv, nbytes, stream):
        try:
            s = _tensor_at(send, nbytes, np.uint8, "|u1", self.device)
            r = _tensor_at(recv, self.world * nbytes, np.uint8, "|u1", self.device)
            if self.staged and s.is_cuda:
                hr = torch.empty(self.world * nbytes, dtype=torch.uint8)
                tdist.all_gather_into_tensor(hr, s.cpu(), group=self.group)
                r.copy_(hr)
            else:
                tdist.all_gather_into_tensor(r, s, group=self.group)
            return 0
        except Exception as e:
            self.error = e
            return 1


class NcclCollectives:
    """adg_collectives over an NCCL communicator the library drives itself
    (adg_comm_nccl_create): rank 0 draws the unique id, torch.distributed
    broadcasts it."""

    def __init__(self, ctx, group=None):
        L = _lib.load()
        world, rank = tdist.get_world_size(group), tdist.get_rank(group)
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _lib.check(L.adg_nccl_unique_id(uid))
        box = [bytes(uid)]
        tdist.broadcast_object_list(box, src=tdist.get_global_rank(group, 0) if group else 0,
                                    group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(box[0])
        self.c = _lib.Collectives()
        _lib.check(L.adg_comm_nccl_create(ctx, world, rank, uid, ctypes.byref(self.c)))
        self.world, self.rank = world, rank

    def close(self):
        if self.c.user:
            _lib.check(_lib.load().adg_comm_nccl_destroy(ctypes.byref(self.c)))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


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

    def set_engine(self, engine="screen"):
        _lib.check(self.L.adg_eval_plan_set_engine(self.h, _lib.ENGINES[engine]))

    def shard(self, world, rank):
        b, e = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(self.L.adg_eval_plan_shard(self.h, world, rank, ctypes.byref(b), ctypes.byref(e)))
        return b.value, e.value

    def exchange(self, coll):
        """adg_eval_plan_exchange over `coll` (TorchCollectives / NcclCollectives)."""
        st = self.L.adg_eval_plan_exchange(self.h, ctypes.byref(coll.c))
        err = getattr(coll, "error", None)
        if err is not None:
            coll.error = None
            raise _lib.CollectiveError(f"eval_plan_exchange: {err!r}") from err
        _lib.check(st)

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
    """evaluate(all pairs) sharded over the ranks of `group`.
    collectives: "torch" (torch.distributed: NCCL or host-staged gloo) or
    "nccl" (a communicator the library drives natively)."""

    def __init__(self, group=None, collectives="torch"):
        self.group = group
        up = tdist is not None and tdist.is_available() and tdist.is_initialized()
        self.world = tdist.get_world_size(group) if up else 1  # no process group: one rank
        self.rank = tdist.get_rank(group) if up else 0
        self.kind = collectives
        self._coll = None

    def _collectives(self, plan):
        if self.world == 1:
            return None
        if self._coll is None:
            if self.kind == "nccl":
                self._coll = NcclCollectives(plan.ctx, self.group)
            else:
                self._coll = TorchCollectives(self.group, plan.dev)
        return self._coll

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

    def evaluate(self, X, Y, hist_bins=50, hist_max=1.0, engine="screen"):
        plan = self._plan(X, Y, hist_bins, hist_max)
        try:
            plan.set_engine(engine)
            t0, t1 = plan.shard(self.world, self.rank)
            plan.run(t0, t1)
            coll = self._collectives(plan)
            if coll is not None:
                # stream-ordered behind the screen; one host read (the largest
                # near-coincident count sizes the gather)
                plan.exchange(coll)
            return plan.finalize()
        finally:
            if getattr(self, "_cached", None) is None or self._cached[1] is not plan:
                plan.close()

    def close(self):
        cached = getattr(self, "_cached", None)
        if cached is not None:
            cached[1].close()
            self._cached = None
        if isinstance(self._coll, NcclCollectives):
            self._coll.close()
        self._coll = None

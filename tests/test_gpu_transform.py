"""transform_all across the shapes that select different kernel paths:

* the streamed kernel (16-byte aligned rows: d % 4 == 0 for fp32, d % 8 == 0
  for bf16) with full and ragged last K chunks, 1..2 column blocks, and row
  counts around the 64-row tile;
* the general kernel (unaligned rows or a misaligned device view);
* fp64 input (fp64 compute path).

Reference: the oracle's transform_all (proj/src/embed.cpp:161-181) in fp64 on
the same (exactly widened) input values, relative Frobenius <= 1e-4 as for
the fit/transform parity tests.
"""
import numpy as np
import pytest

import paper_1609_05388_b200 as adg

pytestmark = pytest.mark.gpu

EMBED_TOL = 1e-4


def _model(d, s, k, seed):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((d, s)))
    mean = rng.normal(3.0, 1.0, d)
    basis = adg.OrthonormalBasis(np.ascontiguousarray(q.T))
    sketch = adg.sample_jl(k, d, adg.derive_seed(seed, "jl"))
    return adg.AdagioModel(mean=mean, basis=basis, sketch=sketch, seed=seed)


def _check(model, Xh, Y):
    Yref = _oracle_transform(model, Xh)
    Yh = Y.double().cpu().numpy() if hasattr(Y, "cpu") else np.asarray(Y, np.float64)
    assert Yh.shape == Yref.shape
    err = np.linalg.norm(Yh - Yref) / max(np.linalg.norm(Yref), 1e-300)
    assert err <= EMBED_TOL, err


def _oracle_transform(model, Xh):
    from oracle import oracle as orc
    return orc.transform_all(np.asarray(model.mean, np.float64), np.asarray(model.basis.rows, np.float64),
                             np.asarray(model.sketch.entries, np.float64), Xh)


@pytest.mark.parametrize("n,d,s,k", [
    (1, 64, 3, 2),        # single row
    (63, 128, 8, 8),      # < one row tile
    (65, 132, 10, 6),     # ragged last K chunk (132 = 2*64 + 4)
    (1000, 784, 25, 25),  # C3 shape family, RN = 64
    (777, 256, 60, 60),   # RN = 128
    (300, 192, 100, 100), # two column blocks
    (129, 96, 4, 4),      # RN = 16
])
def test_transform_f32_streamed(n, d, s, k):
    import torch
    model = _model(d, s, k, n + d)
    rng = np.random.default_rng(n)
    X = torch.from_numpy(rng.normal(3.0, 2.0, (n, d)).astype(np.float32)).cuda()
    _check(model, X.double().cpu().numpy(), adg.transform_all(model, X).data)


@pytest.mark.parametrize("n,d", [(500, 131), (200, 3), (70, 66)])
def test_transform_f32_unaligned_rows(n, d):
    import torch
    model = _model(d, 2, 3, d)
    X = torch.from_numpy(np.random.default_rng(d).normal(0.0, 1.0, (n, d)).astype(np.float32)).cuda()
    _check(model, X.double().cpu().numpy(), adg.transform_all(model, X).data)


def test_transform_misaligned_view():
    import torch
    n, d = 300, 128
    model = _model(d, 6, 6, 5)
    base = torch.from_numpy(np.random.default_rng(1).normal(0.0, 1.0, n * d + 1).astype(np.float32)).cuda()
    X = base[1:].view(n, d)  # 4-byte offset: general kernel
    _check(model, X.double().cpu().numpy(), adg.transform_all(model, X).data)


@pytest.mark.parametrize("n,d,s,k", [(400, 1024, 32, 32), (130, 136, 5, 7), (90, 100, 4, 4)])
def test_transform_bf16(n, d, s, k):
    import torch
    model = _model(d, s, k, 11)
    X = torch.from_numpy(np.random.default_rng(2).normal(1.0, 1.0, (n, d)).astype(np.float32))
    X = X.to(torch.bfloat16).cuda()
    _check(model, X.double().cpu().numpy(), adg.transform_all(model, X).data)


def test_transform_f64():
    n, d = 200, 96
    model = _model(d, 5, 5, 3)
    X = np.random.default_rng(3).normal(0.0, 1.0, (n, d))
    Y = adg.transform_all(model, X).data
    Yref = _oracle_transform(model, X)
    assert np.max(np.abs(np.asarray(Y) - Yref)) <= 1e-10 * np.max(np.abs(Yref))


def test_device_output_ordered_with_torch_stream():
    """Device-resident results are produced on torch's current stream (also
    when that is the legacy default stream, handle 0): reading them right away
    through torch, without any explicit synchronisation, sees the final values."""
    import torch
    n, d = 20000, 784
    model = _model(d, 25, 25, 9)
    X = torch.from_numpy(np.random.default_rng(5).normal(0.0, 1.0, (n, d)).astype(np.float32)).cuda()
    Yref = _oracle_transform(model, X[:64].double().cpu().numpy())
    for _ in range(3):
        Y = adg.transform_all(model, X).data
        head = Y[:64].double().cpu().numpy()  # no torch.cuda.synchronize()
        assert np.linalg.norm(head - Yref) / np.linalg.norm(Yref) <= EMBED_TOL
        del Y
    with torch.cuda.stream(torch.cuda.Stream()):
        Y = adg.transform_all(model, X).data
        head = Y[:64].double().cpu().numpy()
    assert np.linalg.norm(head - Yref) / np.linalg.norm(Yref) <= EMBED_TOL


def test_transform_host_input_matches_device():
    import torch
    n, d = 640, 784
    model = _model(d, 25, 25, 7)
    Xh = np.random.default_rng(4).normal(0.0, 1.0, (n, d)).astype(np.float32)
    Yd = adg.transform_all(model, torch.from_numpy(Xh).cuda()).data.cpu().numpy()
    Yh = np.asarray(adg.transform_all(model, Xh).data)
    assert np.array_equal(Yd, Yh)


def test_cached_plan_matches_one_shot_and_tracks_model_changes():
    """transform_all with a device-resident model reuses one adg_transform_plan
    (W built once); results are bit-identical to the one-shot ABI (a host
    model takes that path), and an in-place change of the model invalidates
    the cached plan."""
    import copy
    import pickle

    import torch
    rng = np.random.default_rng(7)
    X = torch.from_numpy(rng.standard_normal((3000, 200)).astype(np.float32)).cuda()
    m = adg.fit(X, 24, adg.SpectralBackend.exact, 3)
    host = adg.AdagioModel(m.mean.cpu().numpy(), adg.OrthonormalBasis(m.basis.rows.cpu().numpy()),
                           adg.JlMatrix(m.sketch.entries.cpu().numpy()), 3)
    y1 = adg.transform_all(m, X).data
    assert "_adg_plan" in m.__dict__
    plan = m.__dict__["_adg_plan"][1]
    y2 = adg.transform_all(m, X).data
    assert m.__dict__["_adg_plan"][1] is plan  # reused
    ref = adg.transform_all(host, X).data
    assert "_adg_plan" not in host.__dict__
    assert torch.equal(y1, ref) and torch.equal(y2, ref)
    m.mean.add_(1.0)  # in place: version counter moves
    y3 = adg.transform_all(m, X).data
    assert m.__dict__["_adg_plan"][1] is not plan
    host.mean = host.mean + 1.0
    assert torch.equal(y3, adg.transform_all(host, X).data)
    # fp64 input gets its own (fp64) plan; the model still pickles and copies
    y4 = adg.transform_all(m, X.double()).data
    assert y4.dtype == torch.float64
    assert torch.allclose(y4.float(), y3, rtol=1e-5, atol=1e-5)
    m2 = pickle.loads(pickle.dumps(copy.copy(m)))
    assert "_adg_plan" not in m2.__dict__ and torch.equal(m2.mean, m.mean)

"""Seeded synthetic stand-ins for the BASELINE.json configs C1-C5.

The reference's headline data (MNIST) is not available offline; BASELINE.json
fixes the shapes, dtypes and value distributions, and these generators
reproduce them from fixed seeds (numpy PCG64 for C1-C3, which are also the
CPU-oracle parity configs; torch on the target device for the large C4/C5).
Nothing here is copied from any dataset.  SURVEY.md 8(d) lists the
ambiguities resolved below (blob interior, mask location, perturbation scale).
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    # name: (n, d, target_dim, hist_bins, dtype)
    "c1": (2000, 256, 30, 100, "f32"),
    "c2": (1000, 256, 20, 50, "f32"),
    "c3": (60000, 784, 50, 50, "f32"),
    "c4": (1000000, 960, 64, 50, "f32"),
    "c5": (200000, 4096, 128, 50, "bf16"),
}


def _orthonormal(rng, rows, cols):
    q, r = np.linalg.qr(rng.standard_normal((rows, cols)))
    return q * np.sign(np.diag(r))  # unique orthonormal factor


def c1_low_rank(n=2000, d=256, rank=10, noise=0.01, seed=1):
    """x = U z + e, U d x 10 orthonormal, z ~ N(0, I), e ~ N(0, noise^2 I); fp32."""
    rng = np.random.default_rng(seed)
    U = _orthonormal(rng, d, rank)
    Z = rng.standard_normal((n, rank))
    E = noise * rng.standard_normal((n, d))
    return (Z @ U.T + E).astype(np.float32)


def c2_blobs(n=1000, side=16, sigma=1.5, grid=32, lo=1.5, hi=13.5):
    """16x16 isotropic Gaussian blob (amplitude 1) centred on a uniform 32x32
    sub-pixel grid over the interior [lo, hi]^2; first n centres in row-major
    order; images flattened row-major; fp32 (deterministic, no seed)."""
    ticks = lo + (hi - lo) * np.arange(grid) / (grid - 1)
    cy, cx = np.meshgrid(ticks, ticks, indexing="ij")
    cy, cx = cy.reshape(-1)[:n], cx.reshape(-1)[:n]
    r = np.arange(side, dtype=np.float64)
    dy = (r[None, :, None] - cy[:, None, None]) ** 2
    dx = (r[None, None, :] - cx[:, None, None]) ** 2
    img = np.exp(-(dy + dx) / (2.0 * sigma * sigma))
    return img.reshape(n, side * side).astype(np.float32)


def c3_mnist_like(n=60000, side=28, classes=10, rank=20, pert=0.15, noise=0.05, seed=3,
                  return_labels=False):
    """MNIST-shaped synthetic: 10 prototypes with a 20x20 centre mask (rows/cols
    4..23) ~40% active with U(0.5, 1), border 0; sample = prototype + pert * B_c z
    (B_c orthonormal 784 x 20 supported on the mask, z ~ N(0, I_20)) + N(0, noise^2),
    clamped to [0, 1], border re-zeroed; uniform labels; fp32."""
    rng = np.random.default_rng(seed)
    d = side * side
    mask2 = np.zeros((side, side), bool)
    mask2[4:24, 4:24] = True
    mask = mask2.reshape(-1)
    midx = np.nonzero(mask)[0]
    protos = np.zeros((classes, d))
    bases = np.zeros((classes, d, rank))
    for c in range(classes):
        active = rng.random(midx.size) < 0.4
        protos[c, midx[active]] = rng.uniform(0.5, 1.0, active.sum())
        bases[c][midx] = _orthonormal(rng, midx.size, rank)
    labels = rng.integers(0, classes, n)
    X = np.empty((n, d), np.float32)
    chunk = 8192
    for s in range(0, n, chunk):
        lab = labels[s:s + chunk]
        z = rng.standard_normal((lab.size, rank))
        x = protos[lab] + pert * np.einsum("ndr,nr->nd", bases[lab], z)
        x += noise * rng.standard_normal((lab.size, d))
        np.clip(x, 0.0, 1.0, out=x)
        x[:, ~mask] = 0.0
        X[s:s + chunk] = x
    return (X, labels) if return_labels else X


def c4_power_law(n=1000000, d=960, exponent=0.8, seed=4, device="cuda"):
    """x = V diag(i^-0.8) g, V random orthonormal d x d, g ~ N(0, I); fp32 (torch)."""
    import torch
    gen = torch.Generator(device=device).manual_seed(seed)
    V, _ = torch.linalg.qr(torch.randn(d, d, generator=gen, device=device, dtype=torch.float64))
    scale = torch.arange(1, d + 1, device=device, dtype=torch.float64) ** (-exponent)
    M = (V * scale).T.contiguous()  # rows: g @ M = (V diag(s) g)^T
    out = torch.empty(n, d, device=device, dtype=torch.float32)
    for s in range(0, n, 65536):
        m = min(65536, n - s)
        g = torch.randn(m, d, generator=gen, device=device, dtype=torch.float64)
        out[s:s + m] = (g @ M).float()
    return out


def c5_mixture(n=200000, d=4096, comps=256, sub=128, mean_var=4.0, noise=0.1, seed=5,
               device="cuda"):
    """256-component Gaussian mixture: means B u_c (B d x 128 orthonormal,
    u_c ~ N(0, 4 I)), uniform component, + N(0, 0.1^2 I_d); stored bf16 (torch)."""
    import torch
    gen = torch.Generator(device=device).manual_seed(seed)
    B, _ = torch.linalg.qr(torch.randn(d, sub, generator=gen, device=device,
                                       dtype=torch.float64))
    means = (torch.randn(comps, sub, generator=gen, device=device, dtype=torch.float64)
             * mean_var ** 0.5) @ B.T
    lab = torch.randint(0, comps, (n,), generator=gen, device=device)
    out = torch.empty(n, d, device=device, dtype=torch.bfloat16)
    for s in range(0, n, 16384):
        m = min(16384, n - s)
        x = means[lab[s:s + m]] + noise * torch.randn(m, d, generator=gen, device=device,
                                                       dtype=torch.float64)
        out[s:s + m] = x.to(torch.bfloat16)
    return out


def make(name, **kw):
    return {"c1": c1_low_rank, "c2": c2_blobs, "c3": c3_mnist_like, "c4": c4_power_law,
            "c5": c5_mixture}[name](**kw)

import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_1609_05388_b200 as adg
rng = np.random.default_rng(0)
X = rng.standard_normal((3000, 500)) @ np.diag(np.linspace(3, 0.1, 500))
import os
for ns in (0, 500):  # 0: subspace iteration, block 152 (grid Cholesky); 500: full grid Jacobi
    basis, _ = adg.exact_top_svd(torch.from_numpy(X).cuda(), 60, n_sigma=ns)
    B = basis.rows.cpu().numpy()
    Xc = X - X.mean(0)
    _, s, vt = np.linalg.svd(Xc, full_matrices=False)
    print(ns, "nan", np.isnan(B).any(), "proj err", np.abs(np.abs((B * vt[:60]).sum(1)) - 1).max())
if len(sys.argv) > 1:
    from paper_1609_05388_b200 import datasets as ds
    Xt = torch.from_numpy(ds.c3_mnist_like()).cuda()
    Xc = (Xt.double() - Xt.double().mean(0)).float().contiguous()
    for s_, src in ((200, Xt), (100, Xc), (150, Xc), (200, Xc)):
        basis, _ = adg.exact_top_svd(src, s_, n_sigma=0)
        B = basis.rows.double()
        G = B @ B.T
        print(s_, "nan", bool(torch.isnan(B).any()), "orth err", float((G - torch.eye(s_, device=G.device, dtype=G.dtype)).abs().max()),
              "row norms", B.norm(dim=1)[:3].tolist())
sys.exit(0)
print("nan", np.isnan(B).any(), "norm", np.linalg.norm(B, axis=1)[:5])
Xc = X - X.mean(0)
_, s, vt = np.linalg.svd(Xc, full_matrices=False)
print("proj err", np.abs(np.abs((B * vt[:60]).sum(1)) - 1).max())

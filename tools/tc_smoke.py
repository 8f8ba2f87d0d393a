import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1609_05388_b200 as adg
from oracle import oracle as orc
orc.lib()
rng = np.random.default_rng(0)
for (n, d, s, k) in [(300, 64, 3, 5), (1000, 784, 25, 25), (129, 100, 50, 60)]:
    q, _ = np.linalg.qr(rng.standard_normal((d, s)))
    mean = rng.normal(3.0, 1.0, d)
    m = adg.AdagioModel(mean, adg.OrthonormalBasis(np.ascontiguousarray(q.T)), adg.sample_jl(k, d, 5), 0)
    X = torch.from_numpy(rng.normal(3.0, 2.0, (n, d)).astype(np.float32)).cuda()
    Y = adg.transform_all(m, X).data.double().cpu().numpy()
    ref = orc.transform_all(mean, np.ascontiguousarray(q.T), np.asarray(m.sketch.entries), X.double().cpu().numpy())
    print(n, d, s + k, "relerr", np.linalg.norm(Y - ref) / np.linalg.norm(ref), flush=True)

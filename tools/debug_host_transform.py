import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_05388_b200 as adg
from oracle import oracle as orc
orc.lib()

def model(d, s, k, seed):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((d, s)))
    return adg.AdagioModel(mean=rng.normal(3.0, 1.0, d), basis=adg.OrthonormalBasis(np.ascontiguousarray(q.T)),
                           sketch=adg.sample_jl(k, d, adg.derive_seed(seed, "jl")), seed=seed)

def ref(m, X):
    return orc.transform_all(np.asarray(m.mean), np.asarray(m.basis.rows), np.asarray(m.sketch.entries), X)

# step 1: misaligned view (general kernel)
n, d = 300, 128
m1 = model(d, 6, 6, 5)
base = torch.from_numpy(np.random.default_rng(1).normal(0.0, 1.0, n * d + 1).astype(np.float32)).cuda()
X1 = base[1:].view(n, d)
Y1 = adg.transform_all(m1, X1).data
print("misaligned err", np.linalg.norm(Y1.double().cpu().numpy() - ref(m1, X1.double().cpu().numpy())))
# step 2
n, d = 640, 784
m2 = model(d, 25, 25, 7)
Xh = np.random.default_rng(4).normal(0.0, 1.0, (n, d)).astype(np.float32)
Yr = ref(m2, Xh.astype(np.float64))
Yd_t = adg.transform_all(m2, torch.from_numpy(Xh).cuda()).data
Yd_nosync = Yd_t.cpu().numpy()
torch.cuda.synchronize()
Yd_sync = Yd_t.cpu().numpy()
Yh = np.asarray(adg.transform_all(m2, Xh).data)
f = lambda A: np.linalg.norm(A - Yr) / np.linalg.norm(Yr)
print("dev nosync", f(Yd_nosync), "dev sync", f(Yd_sync), "host", f(Yh))
print("torch stream", torch.cuda.current_stream().cuda_stream)

"""Debug aid: does min_dim_for_distortion(pca, rank 200) leave X intact?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import Method, datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
h0 = float(X.double().abs().sum())
warm = len(sys.argv) > 1
if warm:
    adg.min_dim_for_distortion(X[:5000], Method.pca, 0.5, 0, 1, 20)
    print("after warm-up", float(X.double().abs().sum()) - h0, flush=True)
r = adg.min_dim_for_distortion(X, Method.pca, 0.5, 0, 1, 200)
torch.cuda.synchronize()
print(r, "X delta", float(X.double().abs().sum()) - h0, flush=True)

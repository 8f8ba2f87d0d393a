"""One exact fit of a rank-200 basis on C3 (the PCA sweep's basis cache) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import Method, datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
adg.tradeoff(X, [200], [Method.pca], [0])
torch.cuda.synchronize()
print("ok")

import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
adg.fit(X, 50, adg.SpectralBackend.exact, 0)
torch.cuda.synchronize()
print("ok")

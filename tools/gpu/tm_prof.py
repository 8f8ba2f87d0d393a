import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
adg.transform_all(m, X); torch.cuda.synchronize()
for dbg in sys.argv[1:]:
    print("== debug", dbg, flush=True)
    os.environ["ADG_TM_DEBUG"] = dbg
    adg.transform_all(m, X); torch.cuda.synchronize()

"""One config-3 CSC SpMM at 256 images (fused CSC check + apply) and one at 64
images (CSC check + apply), for an ncu capture."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

k = 3
kern = np.random.default_rng(0).standard_normal(9).astype(np.float32)
t = sp.build_transform(sp.Kernel(3, kern), sp.ConvSpec(1024, 1024, 3, 1, 1), layout=1)
X = torch.randn(256, t.cols, device="cuda")
Y = torch.empty(256, t.rows, device="cuda")
sp.spmm(t, X, Y)
sp.spmm(t, X[:64], Y[:64])
torch.cuda.synchronize()
print(t.last_kernel)

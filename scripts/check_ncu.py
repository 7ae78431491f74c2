"""Config 4 (4096^2 k7 s2 p3) at 8 images: one spmm per layout (CSR then CSC),
for an ncu capture of the two check kernels."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

kern = np.random.default_rng(0).standard_normal(49).astype(np.float32)
X = torch.randn(8, 4096 * 4096, device="cuda")
Y = torch.empty(8, 2048 * 2048, device="cuda")
for layout in (0, 1):
    t = sp.build_transform(sp.Kernel(7, kern), sp.ConvSpec(4096, 4096, 7, 2, 3), layout=layout)
    sp.spmm(t, X, Y)
    torch.cuda.synchronize()
    print(t.last_kernel)
    t.close()

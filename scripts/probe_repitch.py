"""One batched apply on an odd width, for an ncu launch list (repitch pass +
band kernels):  ncu --metrics gpu__time_duration.sum python scripts/probe_repitch.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

for spec, b in (((1023, 1023, 3, 1, 1), 64), ((257, 193, 3, 2, 1), 256)):
    k = spec[2]
    t = sp.build_transform(sp.Kernel(k, np.random.default_rng(0).standard_normal(k * k).astype(np.float32)),
                           sp.ConvSpec(*spec))
    X = torch.randn(b, t.cols, device="cuda")
    Y = torch.empty(b, t.rows, device="cuda")
    for _ in range(2):
        sp.spmm(t, X, Y)
    torch.cuda.synchronize()
    print(spec, t.last_kernel)

"""One config-3-shape spmm call per kernel flavour (dense / one zero tap), for an ncu launch list."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp
spec = sp.ConvSpec(1024, 1024, 3, 1, 1)
X = torch.randn(256, 1024 * 1024, device="cuda")
Y = torch.empty(256, 1024 * 1024, device="cuda")
k = np.random.default_rng(0).standard_normal(9).astype(np.float32)
kz = k.copy(); kz[4] = 0.0
for kern in (k, kz):
    t = sp.build_transform(sp.Kernel(3, kern), spec)
    for _ in range(3):
        sp.spmm(t, X, Y)
    torch.cuda.synchronize()

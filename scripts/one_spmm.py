import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp
spec = tuple(int(v) for v in sys.argv[1:6]); b = int(sys.argv[6]); fused = sys.argv[7]
m, n, k, s, p = spec
kern = np.random.default_rng(0).standard_normal(k * k).astype(np.float32)
t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec))
X = torch.randn(b, t.cols, device="cuda"); Y = torch.empty(b, t.rows, device="cuda")
with sp.options(fused=fused):
    sp.spmm(t, X, Y)
torch.cuda.synchronize(); print("ok", t.last_kernel)

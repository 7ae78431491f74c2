import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp
spec = sp.ConvSpec(1024, 1024, 3, 1, 1)
X = torch.randn(256, 1024 * 1024, device="cuda"); Y = torch.empty(256, 1024 * 1024, device="cuda")
t = sp.build_transform(sp.Kernel(3, np.random.default_rng(0).standard_normal(9).astype(np.float32)), spec)
p, i, v = t.export(); g = sp.Transform.from_host(t.rows, t.cols, p, i[:t.nnz], v[:t.nnz])
for _ in range(2): sp.spmm(g, X, Y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): sp.spmm(g, X, Y)
e1.record(); torch.cuda.synchronize()
print(sys.argv[1], e0.elapsed_time(e1) / 5 * 1e3, g.last_kernel)

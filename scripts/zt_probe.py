import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp
def timeit(t, X, Y, n=10):
    for _ in range(3): sp.spmm(t, X, Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): sp.spmm(t, X, Y)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
spec = sp.ConvSpec(1024, 1024, 3, 1, 1)
rng = np.random.default_rng(0)
X = torch.randn(256, 1024 * 1024, device="cuda")
Y = torch.empty(256, 1024 * 1024, device="cuda")
k = rng.standard_normal(9).astype(np.float32)
t = sp.build_transform(sp.Kernel(3, k), spec)
print("dense", timeit(t, X, Y), t.last_kernel)
kz = k.copy(); kz[4] = 0.0
tz = sp.build_transform(sp.Kernel(3, kz), spec)
print("zero-tap", timeit(tz, X, Y), tz.last_kernel)
p, i, v = t.export()
g = sp.Transform.from_host(t.rows, t.cols, p, i[:t.nnz], v[:t.nnz])
print("generic", timeit(g, X, Y, 3), g.last_kernel)

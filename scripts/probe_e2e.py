import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp
t = sp.build_transform(sp.Kernel(3, np.random.default_rng(0).standard_normal(9).astype(np.float32)), sp.ConvSpec(1024, 1024, 3, 1, 1))
Xh = torch.randn(256, t.cols).pin_memory(); Yh = torch.empty(256, t.rows).pin_memory()
sp.convolve_batch(t, Xh, Yh)
for r in range(5):
    t0 = time.perf_counter(); sp.convolve_batch(t, Xh, Yh); print("e2e ms", (time.perf_counter() - t0) * 1e3, flush=True)
Xd = Xh.cuda(); print("parity", torch.equal(sp.spmm(t, Xd).cpu(), Yh))

import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp
def tm(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 1)
for spec in [(257,193,3,2,1),(257,193,3,1,1),(257,193,5,3,4),(257,193,1,1,0),(256,192,3,2,1),(256,196,3,2,1),(1024,1021,3,1,1)]:
    k = spec[2]
    kern = np.random.default_rng(0).standard_normal(k*k).astype(np.float32)
    t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec))
    for b in (256, 32):
        X = torch.randn(b, t.cols, device="cuda"); Y = torch.empty(b, t.rows, device="cuda")
        r = {}
        for f in ("0", "1"):
            with sp.options(fused=f):
                r[f] = tm(lambda: sp.spmm(t, X, Y))
        print(spec, b, r, flush=True)

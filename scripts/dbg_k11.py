import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp
for spec in [(131, 196, 11, 1, 0), (131, 196, 11, 1, 10), (64, 96, 11, 1, 0), (131, 196, 7, 1, 3)]:
    m, n, k, s, p = spec
    kern = np.random.default_rng(0).standard_normal(k * k).astype(np.float32)
    t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec))
    X = torch.randn(4, t.cols, device="cuda")
    with sp.options(fused="0"):
        sp.spmm(t, X)
    torch.cuda.synchronize()
    f = t.band_check_flags()
    no = (n + 2 * p - k) // s + 1
    print(spec, "segments", f.size, "failed", np.nonzero(f == 0)[0].tolist()[:20], "no", no, flush=True)

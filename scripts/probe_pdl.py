"""Back-to-back applies with option pdl = auto (apply and check as programmatic
dependents), apply_only, off: config 3 (fp32 fused, fp32 two-kernel, fp64) and
config 4, CUDA-event mean over 20 calls."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402


def run(t, X, Y, fn, pdl, fused="auto"):
    with sp.options(pdl=pdl, fused=fused):
        for _ in range(3):
            fn(t, X, Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn(t, X, Y)
        e1.record()
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / 20


for name, spec, b, dt, fused in (("c3 fused", (1024, 1024, 3, 1, 1), 256, torch.float32, "auto"),
                                 ("c3 two-kernel", (1024, 1024, 3, 1, 1), 256, torch.float32, "0"),
                                 ("c3 fp64", (1024, 1024, 3, 1, 1), 256, torch.float64, "auto"),
                                 ("c4 b=8", (4096, 4096, 7, 2, 3), 8, torch.float32, "auto"),
                                 ("c4 b=64", (4096, 4096, 7, 2, 3), 64, torch.float32, "auto")):
    k = spec[2]
    t = sp.build_transform(sp.Kernel(k, np.random.default_rng(0).standard_normal(k * k).astype(np.float32)),
                           sp.ConvSpec(*spec))
    X = torch.randn(b, t.cols, device="cuda", dtype=dt)
    Y = torch.empty(b, t.rows, device="cuda", dtype=dt)
    fn = sp.spmm_f64 if dt == torch.float64 else sp.spmm
    res = [(p, round(run(t, X, Y, lambda a, x, y: fn(a, x, y), p, fused), 1)) for p in ("auto", "apply_only", "off", "auto", "apply_only")]
    print(name, res, t.last_kernel, flush=True)
    del X, Y
    t.close()
    torch.cuda.empty_cache()

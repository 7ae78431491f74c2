"""Band forms by geometry: fused vs two-kernel (option fused), dense and
zero-tap (pruned) kernels, CSR and CSC storage, 1024^2 images.
    python scripts/ab_zt.py [dense|zt|both]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402


def tm(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 1)


which = sys.argv[1] if len(sys.argv) > 1 else "both"
for spec, zt in [(sp_, z) for sp_ in ((1024, 1024, 3, 1, 1), (1024, 1024, 5, 1, 2), (1024, 1024, 3, 2, 1),
                                      (1024, 1024, 5, 2, 2), (1024, 1024, 1, 1, 0), (1024, 1024, 2, 2, 0))
                 for z in (False, True) if which == "both" or (which == "zt") == z]:
    k = spec[2]
    kern = np.random.default_rng(0).standard_normal(k * k).astype(np.float32)
    if zt:
        if k == 1:
            continue
        kern[1] = 0.0
    for layout in (0, 1):
        t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec), layout=layout)
        for b in (256, 32):
            X = torch.randn(b, t.cols, device="cuda")
            Y = torch.empty(b, t.rows, device="cuda")
            r = {}
            for f in ("0", "1"):
                with sp.options(fused=f):
                    r[f] = (tm(lambda: sp.spmm(t, X, Y)), t.last_kernel)
            print(spec, "zt" if zt else "dense", "csc" if layout else "csr", b, r, flush=True)
            del X, Y
        t.close()

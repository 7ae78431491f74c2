"""Event-timed apply of CSC transforms (check + blocked apply) against the same
geometry in CSR: config 4 (8 images) and config 3 (256 images), plus s = 2 / 3
shapes.  L2 flushed between reps."""
import sys

import numpy as np
import torch

import os
sys.path.insert(0, os.environ.get("AB_ROOT", "."))
import paper_2411_19419_b200 as sp  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for spec, b in (((4096, 4096, 7, 2, 3), 8), ((1024, 1024, 3, 1, 1), 256), ((2048, 2048, 5, 2, 2), 32),
                ((2048, 2048, 7, 3, 3), 32), ((2048, 2048, 3, 2, 1), 64)):
    k = spec[2]
    kern = sp.Kernel(k, np.random.default_rng(0).standard_normal(k * k).astype(np.float32))
    out = {}
    for lay in (0, 1):
        t = sp.build_transform(kern, sp.ConvSpec(*spec), layout=lay)
        X = torch.randn(b, t.cols, device="cuda")
        Y = torch.empty(b, t.rows, device="cuda")
        out["csr" if lay == 0 else "csc"] = (timed(lambda: sp.spmm(t, X, Y)), t.last_kernel, t.band_check_status())
        del t, X, Y
        torch.cuda.empty_cache()
    print(spec, b, {k_: (round(v[0], 1), v[1], v[2][1]) for k_, v in out.items()}, flush=True)

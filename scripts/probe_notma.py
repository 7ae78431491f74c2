"""Event-timed batched applies on image widths whose rows are not 16-byte
pitched, 256 images, L2 scrubbed between reps.  REPITCH=off keeps the cp.async
element staging (default: a 16-byte pitched copy + TMA); AB_ROOT selects another
checkout's build for an A/B."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("AB_ROOT", "."))
import paper_2411_19419_b200 as sp  # noqa: E402

scrub = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
if os.environ.get("REPITCH"):
    sp.set_option("repitch", os.environ["REPITCH"])


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        scrub.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for spec in ((257, 193, 11, 1, 10), (257, 193, 5, 1, 4), (257, 193, 3, 1, 1), (257, 193, 3, 2, 1), (257, 193, 5, 3, 2),
             (255, 255, 7, 1, 3), (1023, 1023, 3, 1, 1)):
    k = spec[2]
    kern = sp.Kernel(k, np.random.default_rng(0).standard_normal(k * k).astype(np.float32))
    t = sp.build_transform(kern, sp.ConvSpec(*spec))
    b = 256 if spec[0] < 1000 else 64
    X = torch.randn(b, t.cols, device="cuda")
    Y = torch.empty(b, t.rows, device="cuda")
    us = timed(lambda: sp.spmm(t, X, Y))
    print(spec, b, f"{us:.1f} us", t.last_kernel, flush=True)
    del X, Y
    t.close()

"""Config 3 apply time against batch size (fused form and the two-kernel
form), event-timed back to back with L2 scrubbed between reps -- the fixed
per-call cost the N = 8 slice (32 images) pays.  Run under
`ncu --metrics gpu__time_duration.sum` for the per-kernel split."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

scrub = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
spec = (1024, 1024, 3, 1, 1)
t = sp.build_transform(sp.Kernel(3, np.random.default_rng(0).standard_normal(9).astype(np.float32)),
                       sp.ConvSpec(*spec))
reps = int(os.environ.get("REPS", "10"))
for fused, pdl in (("1", "auto"), ("1", "off"), ("0", "auto"), ("0", "off")):
    for b in (1 * 0 + 8, 16, 32, 64, 128, 256):
        X = torch.randn(b, t.cols, device="cuda")
        Y = torch.empty(b, t.rows, device="cuda")
        with sp.options(fused=fused, pdl=pdl):
            for _ in range(2):
                sp.spmm(t, X, Y)
            ts = []
            for _ in range(reps):
                scrub.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sp.spmm(t, X, Y)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            # back to back (the bench's protocol: K calls in one event window)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                sp.spmm(t, X, Y)
            e1.record()
            torch.cuda.synchronize()
            b2b = e0.elapsed_time(e1) * 1e3 / reps
        us = float(np.median(ts))
        alg = 8 * t.nnz + 4 * (t.rows + 1) + 4 * b * (t.cols + t.rows)
        print(f"fused={fused} pdl={pdl:4s} b={b:4d} single {us:8.1f} us  back-to-back {b2b:8.1f} us "
              f"({alg / b2b / 1e3:5.0f} GB/s)  {t.last_kernel}", flush=True)
        del X, Y

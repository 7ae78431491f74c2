#!/usr/bin/env python
"""A/B of the CSR build kernels (option build): device time of the build
(median of N; CUDA events behind a GPU sleep, so host enqueue latency is
excluded) for fp32 taps and exact double taps, and the arrays checked equal
to the default kernel's.   python scripts/build_ab.py [N] [variants...]"""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
variants = sys.argv[2:] or ["persist", "block"]
st = torch.cuda.Stream()
for name, spec in (("c3", (1024, 1024, 3, 1, 1)), ("c2", (512, 512, 5, 2, 2)), ("c4", (4096, 4096, 7, 2, 3))):
    k = spec[2]
    for exact in (False, True):
        kv = np.random.default_rng(0).standard_normal(k * k)
        if not exact:
            kv = kv.astype(np.float32).astype(np.float64)
        kern = sp.Kernel(k, kv)
        ref = None
        for v in variants:
            with sp.options(build=v):
                ts = []
                for i in range(N + 3):
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.stream(st):
                        torch.cuda._sleep(2_000_000)
                        e0.record(st)
                        t = sp.build_transform(kern, sp.ConvSpec(*spec), stream=st)
                        e1.record(st)
                    torch.cuda.synchronize()
                    if i >= 3:
                        ts.append(e0.elapsed_time(e1) * 1e3)
                    if i < N + 2:
                        t.close()
            arrs = t.export()
            same = "" if ref is None else (" same" if all(np.array_equal(a.view(np.uint64) if a.dtype == np.float64 else a,
                                                                          b.view(np.uint64) if b.dtype == np.float64 else b)
                                                           for a, b in zip(arrs, ref)) else " DIFFERENT")
            ref = ref if ref is not None else arrs
            t.close()
            print(f"{name} exact={int(exact)} {v:8s} {statistics.median(ts):8.1f} us  (min {min(ts):.1f}){same}",
                  flush=True)

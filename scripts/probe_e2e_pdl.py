"""spconv_convolve_host on config 3 (256 pinned images in, 256 out) with the
band apply's programmatic dependent launch on (auto) and off."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

t = sp.build_transform(sp.Kernel(3, np.random.default_rng(0).standard_normal(9).astype(np.float32)),
                       sp.ConvSpec(1024, 1024, 3, 1, 1))
X = torch.randn(256, t.cols).pin_memory()
Y = torch.empty(256, t.rows).pin_memory()
for rep in range(2):
    for pdl in ("auto", "off"):
        with sp.options(pdl=pdl):
            sp.convolve_batch(t, X, Y)
            ts = []
            for _ in range(4):
                t0 = time.perf_counter()
                sp.convolve_batch(t, X, Y)
                ts.append(time.perf_counter() - t0)
        print(pdl, f"{np.median(ts) * 1e3:.2f} ms", t.last_kernel, flush=True)
